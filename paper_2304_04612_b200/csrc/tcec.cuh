// tcec.cuh — the B-operand side of TCEC-SGEMM (Eqs 5-9):
// C_F32 ~ A_low B_low + (dA_low B_low + A_low dB_low) x 2^-11 for FP32 A and B. A is split in the
// mainloop's splitter exactly as for SHGEMM (Eqs 14-15); B is small next to A in the products this
// serves (Q^T A of RSVD line 3, the RP-HOSVD core contractions), so it is split ONCE per call into a
// column-major FP16 buffer [B_low | dB_low] that the mainloop's Omega stager streams by TMA.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>
#include "split.cuh"

namespace shg {

// B element (l, j) at B[l * sbk + j * sbn] (k x n). Writes H[j * ldh + l] = B_low(l, j) and
// H[(noff + j) * ldh + l] = dB_low(l, j) for j < noff (zeros for n <= j < noff), l < k.
// 32 x 32 tiles through shared memory so both the read (either layout) and the write are coalesced.
__global__ void split_b_kernel(const float* __restrict__ B, int64_t k, int64_t n, int64_t sbk, int64_t sbn,
                               uint16_t* __restrict__ H, int64_t ldh, int64_t noff) {
    __shared__ float tile[32][33];   // [l - l0][j - j0]
    const int64_t tl = (k + 31) / 32, tj = (noff + 31) / 32;
    const int tx = threadIdx.x, ty = threadIdx.y;
    for (int64_t tb = blockIdx.x; tb < tl * tj; tb += gridDim.x) {
        const int64_t l0 = (tb % tl) * 32, j0 = (tb / tl) * 32;
        for (int y = ty; y < 32; y += blockDim.y) {
            int64_t l, j;
            int r, c;
            if (sbk == 1) { l = l0 + tx; j = j0 + y; r = tx; c = y; }
            else { l = l0 + y; j = j0 + tx; r = y; c = tx; }
            tile[r][c] = (l < k && j < n) ? B[l * sbk + j * sbn] : 0.0f;
        }
        __syncthreads();
        for (int y = ty; y < 32; y += blockDim.y) {
            const int64_t l = l0 + tx, j = j0 + y;
            if (l < k && j < noff) {
                uint32_t h, lo;
                split2(tile[tx][y], 0.0f, h, lo);      // Eqs 14-15 (the same split as A's)
                H[j * ldh + l] = static_cast<uint16_t>(h & 0xFFFFu);
                H[(noff + j) * ldh + l] = static_cast<uint16_t>(lo & 0xFFFFu);
            }
        }
        __syncthreads();
    }
}

// Correctness-only TCEC-SGEMM on CUDA cores (misaligned inputs): per 64-k chunk the products
// A_low B_low and the correction dA_low B_low + A_low dB_low are accumulated with FMA, and the
// chunk's A_low B_low + 2^-11 correction is added with RN into the FP32 result.
// A element (i, l) at A[i * sa_row + l * sa_col]; H as written by split_b_kernel.
__global__ void tcec_simt_kernel(int64_t m, int64_t n, int64_t k, const float* __restrict__ A, int64_t sa_row,
                                 int64_t sa_col, const uint16_t* __restrict__ H, int64_t ldh, int64_t noff,
                                 float* __restrict__ C, int64_t ldc) {
    const int64_t total = m * n;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = t / n, j = t - (t / n) * n;
        const float* a = A + i * sa_row;
        const uint16_t* bh = H + j * ldh;
        const uint16_t* bl = H + (noff + j) * ldh;
        float acc = 0.0f;
        for (int64_t k0 = 0; k0 < k; k0 += 64) {
            const int64_t k1 = k0 + 64 < k ? k0 + 64 : k;
            // chunk sums in FP64 (exact FP16 x FP16 products, one rounding per chunk), as in
            // shgemm_simt_kernel (DESIGN R26)
            double s_hh = 0.0, s_c = 0.0;
            for (int64_t l = k0; l < k1; ++l) {
                uint32_t h, lo;
                split2(a[l * sa_col], 0.0f, h, lo);
                const double ah = __half2float(__ushort_as_half(static_cast<uint16_t>(h & 0xFFFFu)));
                const double al = __half2float(__ushort_as_half(static_cast<uint16_t>(lo & 0xFFFFu)));
                const double bhf = __half2float(__ushort_as_half(bh[l]));
                const double blf = __half2float(__ushort_as_half(bl[l]));
                s_hh = __fma_rn(ah, bhf, s_hh);
                s_c = __fma_rn(al, bhf, s_c);
                s_c = __fma_rn(ah, blf, s_c);
            }
            acc = __fadd_rn(acc, __double2float_rn(__fma_rn(s_c, 4.8828125e-4, s_hh)));
        }
        C[i * ldc + j] = acc;
    }
}

}  // namespace shg

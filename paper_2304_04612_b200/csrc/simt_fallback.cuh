// simt_fallback.cuh — correctness-only SHGEMM on CUDA cores, used when the tensor-core path's
// TMA alignment preconditions fail (base pointers not 16-B aligned, lda % 4 != 0, ldo % 8 != 0).
// Same numerics contract as the mainloop: Eqs 14-16 with the hi+lo partial
// of every 64-k chunk (summed in FP64, one rounding to FP32) folded with RN into an FP32 accumulator
// (RZ avoidance).
#pragma once
#include <cstdint>
#include <cuda_fp16.h>
#include "split.cuh"

namespace shg {

// A element (i, l) at A[i * sa_row + l * sa_col] (row-major: sa_row = lda, sa_col = 1;
// M-major: sa_row = 1, sa_col = lda). Omega element (l, j) at Om[l * so_k + j * so_n] (column-major:
// so_k = 1, so_n = ldo; row-major: so_k = ldo, so_n = 1).
__global__ void shgemm_simt_kernel(int64_t m, int64_t n, int64_t k, const float* __restrict__ A, int64_t sa_row,
                                   int64_t sa_col, const uint16_t* __restrict__ Om, int64_t so_k, int64_t so_n,
                                   float* __restrict__ Y, int64_t ldc, int* nonfinite, bool tf32) {
    const int64_t total = m * n;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = t / n, j = t - (t / n) * n;
        const float* a = A + i * sa_row;
        const uint16_t* w = Om + j * so_n;
        float acc = 0.0f;
        for (int64_t k0 = 0; k0 < k; k0 += 64) {
            const int64_t k1 = k0 + 64 < k ? k0 + 64 : k;
            // the chunk's hi and lo sums in FP64: every product of two FP16 (or TF32) values is exact
            // there and 64 of them sum with a relative error below 2^-47, so the chunk costs ONE
            // rounding to FP32 (like the tensor cores' fused K-step, not k-1 sequential FP32 roundings,
            // which exceed the c5 elementwise bar at small k: round-2 edge fuzz, DESIGN R26)
            double s_hi = 0.0, s_lo = 0.0;
            for (int64_t l = k0; l < k1; ++l) {
                float hf, lf;
                if (tf32) {   // SHGEMM-TF32 split
                    uint32_t h0, h1, l0, l1;
                    split_tf32_x2(a[l * sa_col], 0.0f, h0, h1, l0, l1);
                    hf = __uint_as_float(h0);
                    lf = __uint_as_float(l0);
                } else {
                    uint32_t h, lo;
                    split2(a[l * sa_col], 0.0f, h, lo);
                    hf = __half2float(__ushort_as_half(static_cast<uint16_t>(h & 0xFFFFu)));
                    lf = __half2float(__ushort_as_half(static_cast<uint16_t>(lo & 0xFFFFu)));
                }
                const double wf = static_cast<double>(__half2float(__ushort_as_half(w[l * so_k])));
                s_hi = __fma_rn(static_cast<double>(hf), wf, s_hi);
                s_lo = __fma_rn(static_cast<double>(lf), wf, s_lo);
            }
            acc = __fadd_rn(acc, __double2float_rn(__fma_rn(s_lo, 4.8828125e-4, s_hi)));
        }
        Y[i * ldc + j] = acc;
        if (nonfinite && !isfinite(acc)) atomicOr(nonfinite, 1);
    }
}

// SHGEMM-TF32's B operand: Omega's FP16 values widened exactly to FP32/TF32 bit patterns (P:498:
// "converted to TF32 ... before input to Tensor Cores"; tcgen05 reads B from shared memory, so the
// widening is done once in global memory instead of per tile in registers). Input element (r, j)
// at Om[r * so_k + j * so_n] (either layout); output column-major k x n (ldo32).
__global__ void widen_omega_kernel(const uint16_t* __restrict__ Om, int64_t k, int64_t n, int64_t so_k, int64_t so_n,
                                   float* __restrict__ Om32, int64_t ldo32) {
    const int64_t total = k * n;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t j = t / k, r = t - (t / k) * k;
        Om32[j * ldo32 + r] = __half2float(__ushort_as_half(Om[r * so_k + j * so_n]));
    }
}

// A ROW-major Omega (element (l, j) at Om[l * ldo + j]) copied bit for bit into the
// column-major layout (Ot[j * ldt + l]) that the tensor-core path streams as its K-major B operand
// (tcgen05 reads B from shared memory through TMA, which cannot transpose 2-byte elements). 32 x 32
// tiles through shared memory: both the reads (along j) and the writes (along l) are coalesced.
// blockDim = (32, 8); rows l in [k, ldt) are not written.
__global__ void transpose_omega_kernel(const uint16_t* __restrict__ Om, int64_t k, int64_t n, int64_t ldo,
                                       uint16_t* __restrict__ Ot, int64_t ldt) {
    __shared__ uint16_t tile[32][33];
    const int64_t tk_n = (k + 31) / 32, tn_n = (n + 31) / 32;
    const int tx = static_cast<int>(threadIdx.x), ty = static_cast<int>(threadIdx.y);
    for (int64_t t = blockIdx.x; t < tk_n * tn_n; t += gridDim.x) {
        const int64_t tk = t / tn_n, tn = t - tk * tn_n;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t l = tk * 32 + ty + 8 * i, j = tn * 32 + tx;
            tile[ty + 8 * i][tx] = (l < k && j < n) ? Om[l * ldo + j] : uint16_t(0);
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t j = tn * 32 + ty + 8 * i, l = tk * 32 + tx;
            if (l < k && j < n) Ot[j * ldt + l] = tile[tx][ty + 8 * i];
        }
        __syncthreads();
    }
}

// The same widening from the k-tiled FP16 Omega (64-row tiles: (r/64)*n*64 + j*64 + r%64) into a
// k-tiled FP32 copy of 32-row tiles ((r/32)*n*32 + j*32 + r%32: one SW128 TMA box row per TF32
// k-half); rows k .. 32*ceil(k/32)-1 of the last tile are 0.
__global__ void widen_omega_tiled_kernel(const uint16_t* __restrict__ Om, int64_t k, int64_t n,
                                         float* __restrict__ Om32) {
    const int64_t kp = (k + 31) / 32 * 32;
    const int64_t total = kp * n;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t j = t / kp, r = t - j * kp;
        const float v = r < k ? __half2float(__ushort_as_half(Om[(r >> 6) * n * 64 + j * 64 + (r & 63)])) : 0.0f;
        Om32[(r >> 5) * n * 32 + j * 32 + (r & 31)] = v;
    }
}

}  // namespace shg

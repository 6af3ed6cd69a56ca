// split.cuh — the in-kernel FP32 -> (FP16 hi, FP16 lo) split of Eqs 14-15:
//   A_low  = toLow(A_F32)                                   (RN ties-to-even)
//   dA_low = toLow((A_F32 - toF32(A_low)) * 2^11)
// so that A_F32 ~= A_low + dA_low * 2^-11 (Eq 16). The subtraction is exact for
// |a| in the FP16 range and the x2^11 is an exact exponent shift; both are written as explicit
// _rn ops in exactly this order (no contraction into an fma) so |a| >= 65520 gives hi = +-inf,
// lo = -+inf like the definition (the FP16-range failure mode of PAPER.md:495, :705-706).
#pragma once
#include <cstdint>
#include <cuda_fp16.h>

namespace shg {

// two FP32 values -> packed FP16x2 hi and lo (low half = first value)
__device__ __forceinline__ void split2(float a0, float a1, uint32_t& hi, uint32_t& lo) {
    const __half2 h = __floats2half2_rn(a0, a1);               // cvt.rn.f16x2.f32
    const float2 hf = __half22float2(h);
    const float r0 = __fmul_rn(__fsub_rn(a0, hf.x), 2048.0f);
    const float r1 = __fmul_rn(__fsub_rn(a1, hf.y), 2048.0f);
    const __half2 l = __floats2half2_rn(r0, r1);
    hi = *reinterpret_cast<const uint32_t*>(&h);
    lo = *reinterpret_cast<const uint32_t*>(&l);
}

// Same split with the residual arithmetic done as packed f32x2 (sub.rn / mul.rn .f32x2 = FADD2 /
// FMUL2 on sm_100): identical IEEE RN results per lane, 3 instead of 4 ALU ops per element.
__device__ __forceinline__ void split2_x2(float a0, float a1, uint32_t& hi, uint32_t& lo) {
    const __half2 h = __floats2half2_rn(a0, a1);
    const float2 hf = __half22float2(h);
    float r0, r1;
    asm("{\n\t.reg .b64 x, y, z;\n\t"
        "mov.b64 x, {%2, %3};\n\t"
        "mov.b64 y, {%4, %5};\n\t"
        "sub.rn.f32x2 x, x, y;\n\t"
        "mov.b64 z, {%6, %6};\n\t"
        "mul.rn.f32x2 x, x, z;\n\t"
        "mov.b64 {%0, %1}, x;\n\t}\n"
        : "=f"(r0), "=f"(r1)
        : "f"(a0), "f"(a1), "f"(hf.x), "f"(hf.y), "f"(2048.0f));
    const __half2 l = __floats2half2_rn(r0, r1);
    hi = *reinterpret_cast<const uint32_t*>(&h);
    lo = *reinterpret_cast<const uint32_t*>(&l);
}

// SHGEMM-TF32 split (Eqs 14-15 with toLow = TF32): hi = cvt.rn.tf32(a),
// lo = cvt.rn.tf32((a - hi) * 2^11); TF32 values as FP32 bit patterns (the tensor core reads the
// top 19 bits). a - hi is exact and x 2^11 an exponent shift (packed f32x2 ops, RN per lane).
__device__ __forceinline__ uint32_t cvt_rn_tf32(float a) {
    uint32_t r;
    asm("cvt.rn.tf32.f32 %0, %1;" : "=r"(r) : "f"(a));
    return r;
}

__device__ __forceinline__ void split_tf32_x2(float a0, float a1, uint32_t& h0, uint32_t& h1, uint32_t& l0,
                                              uint32_t& l1) {
    h0 = cvt_rn_tf32(a0);
    h1 = cvt_rn_tf32(a1);
    float r0, r1;
    asm("{\n\t.reg .b64 x, y, z;\n\t"
        "mov.b64 x, {%2, %3};\n\t"
        "mov.b64 y, {%4, %5};\n\t"
        "sub.rn.f32x2 x, x, y;\n\t"
        "mov.b64 z, {%6, %6};\n\t"
        "mul.rn.f32x2 x, x, z;\n\t"
        "mov.b64 {%0, %1}, x;\n\t}\n"
        : "=f"(r0), "=f"(r1)
        : "f"(a0), "f"(a1), "f"(__uint_as_float(h0)), "f"(__uint_as_float(h1)), "f"(2048.0f));
    l0 = cvt_rn_tf32(r0);
    l1 = cvt_rn_tf32(r1);
}

// Elementwise split, for the test ABI shg_debug_split (split2_x2: the mainloop's device function).
static __global__ void debug_split_kernel(const float* __restrict__ a, int64_t count, uint16_t* __restrict__ hi,
                                   uint16_t* __restrict__ lo) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; 2 * t < count;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = 2 * t;
        const float a0 = a[i];
        const float a1 = (i + 1 < count) ? a[i + 1] : 0.0f;
        uint32_t h, l;
        split2_x2(a0, a1, h, l);
        hi[i] = static_cast<uint16_t>(h & 0xFFFFu);
        lo[i] = static_cast<uint16_t>(l & 0xFFFFu);
        if (i + 1 < count) {
            hi[i + 1] = static_cast<uint16_t>(h >> 16);
            lo[i + 1] = static_cast<uint16_t>(l >> 16);
        }
    }
}

// Elementwise TF32 split, for the test ABI shg_debug_split_tf32 (the mainloop's device function).
static __global__ void debug_split_tf32_kernel(const float* __restrict__ a, int64_t count, uint32_t* __restrict__ hi,
                                        uint32_t* __restrict__ lo) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; 2 * t < count;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = 2 * t;
        const float a0 = a[i];
        const float a1 = (i + 1 < count) ? a[i + 1] : 0.0f;
        uint32_t h0, h1, l0, l1;
        split_tf32_x2(a0, a1, h0, h1, l0, l1);
        hi[i] = h0;
        lo[i] = l0;
        if (i + 1 < count) {
            hi[i + 1] = h1;
            lo[i + 1] = l1;
        }
    }
}

}  // namespace shg

// internal.cuh — plumbing shared by api.cu and the kernel-instantiation units (tc_f16.cu,
// tc_tf32.cu, compiled in parallel): error/launch bookkeeping, the BN switch, and the templated
// launch of the tcgen05 mainloop. Not part of the C ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <mutex>

#include "../../include/shgemm.h"
#include "shgemm_sm100.cuh"

namespace shg_api {

extern std::atomic<uint64_t> g_launches;     // kernels launched by this library (shg_launch_count)
extern thread_local char g_err[256];         // message of the last SHG_ERR_CUDA (shg_last_error)
shg_status_t cuda_fail(cudaError_t e, const char* what);

#define SHG_CUDA(call)                                              \
    do {                                                            \
        cudaError_t e_ = (call);                                    \
        if (e_ != cudaSuccess) return shg_api::cuda_fail(e_, #call); \
    } while (0)

constexpr int kBNs[] = {32, 64, 96, 128, 144, 160, 192, 224, 256, 272, 288};
// wide tiles (one N tile for 256 < n <= 288): SHGEMM-FP16 only
constexpr bool wide_bn(int bn) { return bn > 256; }

#define SHG_BN_SWITCH(bn, EXPR)                                  \
    switch (bn) {                                                \
        case 32: { constexpr int BN_ = 32; EXPR; }               \
        case 64: { constexpr int BN_ = 64; EXPR; }               \
        case 96: { constexpr int BN_ = 96; EXPR; }               \
        case 128: { constexpr int BN_ = 128; EXPR; }             \
        case 144: { constexpr int BN_ = 144; EXPR; }             \
        case 160: { constexpr int BN_ = 160; EXPR; }             \
        case 192: { constexpr int BN_ = 192; EXPR; }             \
        case 224: { constexpr int BN_ = 224; EXPR; }             \
        default: { constexpr int BN_ = 256; EXPR; }              \
    }

// CTA pairs (cta_group::2) are instantiated for BN >= 128, where Omega traffic matters
constexpr bool pair_ok(int bn) { return bn >= 128; }

inline bool valid_bn(int bn) {
    for (int b : kBNs) if (b == bn) return true;
    return false;
}

template <int BN, bool MMAJOR, bool PAIR, bool TF32, bool TCEC = false, bool OMGEN = false, int NPA = 1>
shg_status_t launch_tc(const CUtensorMap& mapA, const CUtensorMap& mapB0, const CUtensorMap& mapB1,
                       const shg::KParams& kp, int grid, cudaStream_t stream) {
    using CF = shg::Cfg<BN, PAIR, TF32, TCEC>;
    auto kern = shg::shgemm_sm100_kernel<BN, MMAJOR, PAIR, TF32, TCEC, OMGEN, NPA>;
    static std::once_flag flags[64];
    int dev = 0;
    cudaGetDevice(&dev);
    cudaError_t attr_err = cudaSuccess;
    std::call_once(flags[std::min(std::max(dev, 0), 63)], [&]() {
        attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::kSmemBytes);
    });
    if (attr_err != cudaSuccess) return cuda_fail(attr_err, "cudaFuncSetAttribute");
    if constexpr (!PAIR) {
        // plain launch: a cluster-dimension attribute (even 1x1x1) takes a slower launch path
        kern<<<grid, shg::threads_for<OMGEN>(), CF::kSmemBytes, stream>>>(mapA, mapB0, mapB1, kp);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        SHG_CUDA(cudaGetLastError());
        return SHG_OK;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(shg::threads_for<OMGEN>());
    cfg.dynamicSmemBytes = CF::kSmemBytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = PAIR ? 2 * NPA : 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // The grid is persistent: every cluster must be co-resident, or the clusters that do not fit
    // run as a second wave. Clusters must sit in one GPC, so fewer than #SMs / (2 NPA) may fit (GPC
    // sizes are not multiples of the cluster size): clamp to the occupancy query. (The kernel reads its unit count from
    // gridDim, so a stream-K schedule follows the clamped grid.)
    static int max_clusters[64];
    static std::once_flag occ_flags[64];
    const int di = std::min(std::max(dev, 0), 63);
    std::call_once(occ_flags[di], [&]() {
        int nc = 0;
        if (cudaOccupancyMaxActiveClusters(&nc, kern, &cfg) != cudaSuccess) {
            (void)cudaGetLastError();
            nc = 0;
        }
        max_clusters[di] = nc;
    });
    constexpr int kCl = PAIR ? 2 * NPA : 1;
    if (max_clusters[di] > 0 && grid > max_clusters[di] * kCl) cfg.gridDim = dim3(max_clusters[di] * kCl);
    SHG_CUDA(cudaLaunchKernelEx(&cfg, kern, mapA, mapB0, mapB1, kp));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return SHG_OK;
}

template <bool MMAJOR, bool PAIR, bool TF32>
shg_status_t dispatch_bn(int bn, const CUtensorMap& a, const CUtensorMap& b0, const CUtensorMap& b1,
                         const shg::KParams& kp, int grid, cudaStream_t s) {
    if constexpr (PAIR) {
        switch (bn) {
            case 128: return launch_tc<128, MMAJOR, true, TF32>(a, b0, b1, kp, grid, s);
            case 144: return launch_tc<144, MMAJOR, true, TF32>(a, b0, b1, kp, grid, s);
            case 160: return launch_tc<160, MMAJOR, true, TF32>(a, b0, b1, kp, grid, s);
            case 192: return launch_tc<192, MMAJOR, true, TF32>(a, b0, b1, kp, grid, s);
            case 224: return launch_tc<224, MMAJOR, true, TF32>(a, b0, b1, kp, grid, s);
            case 256: return launch_tc<256, MMAJOR, true, TF32>(a, b0, b1, kp, grid, s);
            case 272: if constexpr (!TF32) return launch_tc<272, MMAJOR, true, false>(a, b0, b1, kp, grid, s);
                      return SHG_ERR_INVALID_VALUE;
            case 288: if constexpr (!TF32) return launch_tc<288, MMAJOR, true, false>(a, b0, b1, kp, grid, s);
                      return SHG_ERR_INVALID_VALUE;
            default: return SHG_ERR_INVALID_VALUE;
        }
    } else {
        if constexpr (!TF32) {
            if (bn == 272) return launch_tc<272, MMAJOR, false, false>(a, b0, b1, kp, grid, s);
            if (bn == 288) return launch_tc<288, MMAJOR, false, false>(a, b0, b1, kp, grid, s);
        }
        if (wide_bn(bn)) return SHG_ERR_INVALID_VALUE;
        SHG_BN_SWITCH(bn, return (launch_tc<BN_, MMAJOR, false, TF32>(a, b0, b1, kp, grid, s)))
    }
}

// TCEC-SGEMM: two B tiles per stage, so single CTAs stop at BN = 128 (smem); pairs cover 128..256
constexpr int kTcecMaxBnSingle = 128;

// Defined in tc_f16.cu / tc_tf32.cu / tc_tcec.cu (one instantiation set per translation unit).
shg_status_t dispatch_tc_f16(int bn, bool mmajor, bool pair, const CUtensorMap& a, const CUtensorMap& b0,
                             const CUtensorMap& b1, const shg::KParams& kp, int grid, cudaStream_t s);
shg_status_t dispatch_tc_f16_mmajor(int bn, bool pair, const CUtensorMap& a, const CUtensorMap& b0,
                                    const CUtensorMap& b1, const shg::KParams& kp, int grid, cudaStream_t s);
shg_status_t dispatch_tc_tf32(int bn, bool mmajor, bool pair, const CUtensorMap& a, const CUtensorMap& b0,
                              const CUtensorMap& b1, const shg::KParams& kp, int grid, cudaStream_t s);
shg_status_t dispatch_tc_tcec(int bn, bool mmajor, bool pair, const CUtensorMap& a, const CUtensorMap& b0,
                              const CUtensorMap& b1, const shg::KParams& kp, int grid, cudaStream_t s);
// SHGEMM-FP16 single CTAs with cooperative in-kernel Omega generation (tc_f16_gen.cu), BN <= 192
shg_status_t dispatch_tc_f16_gen(int bn, bool mmajor, const CUtensorMap& a, const CUtensorMap& b0,
                                 const CUtensorMap& b1, const shg::KParams& kp, int grid, cudaStream_t s);
constexpr int kOmGenMaxBn = shg::kOmGenMaxBnKernel;
// SHGEMM-FP16 K-major CTA pairs with A multicast across npa = 2 or 4 pairs of a cluster (tc_f16_amc.cu)
shg_status_t dispatch_tc_f16_amc(int bn, int npa, const CUtensorMap& a, const CUtensorMap& b0, const CUtensorMap& b1,
                                 const shg::KParams& kp, int grid, cudaStream_t s);
}  // namespace shg_api

// probes.cu — tcgen05 semantics probe. The paper's error analysis rests on the
// A100 tensor-core accumulation properties it lists at PAPER.md:505-512 ("confirmed theoretically
// or empirically through small numerical experiments"). This kernel lets the tests run the
// same kind of small experiments on B200: a single 128 x n x 64 UMMA with chosen FP16 inputs and a
// chosen FP32 accumulator preload, so RN-vs-RZ, alignment width and the scale-input-d semantics the
// mainloop relies on can be measured instead of assumed.
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include "ptx.cuh"
#include "../../include/shgemm.h"

namespace shg {

__global__ void __launch_bounds__(128, 1)
probe_umma_kernel(const uint16_t* __restrict__ A, const uint16_t* __restrict__ B, int n,
                  const float* __restrict__ Dinit, int mode, int nsteps, float* __restrict__ Dout) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t* base = smem_raw + ((1024u - (raw_addr & 1023u)) & 1023u);
    uint8_t* sA = base;                 // 128 rows x 128 B
    uint8_t* sB = base + 128 * 128;     // n rows x 128 B
    uint64_t* bar = reinterpret_cast<uint64_t*>(sB + 256 * 128);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
    const int t = threadIdx.x;
    const uint32_t warp = warp_id();

    // K-major SWIZZLE_128B canonical layout: row r at r*128, 16-B chunk c at (c ^ (r & 7)) * 16
    for (int r = t; r < 128 + n; r += 128) {
        const uint16_t* src = r < 128 ? A + r * 64 : B + (r - 128) * 64;
        uint8_t* dst = r < 128 ? sA + r * 128 : sB + (r - 128) * 128;
        for (int c = 0; c < 8; ++c) {
            const uint4 v = *reinterpret_cast<const uint4*>(src + 8 * c);
            *reinterpret_cast<uint4*>(dst + ((c ^ (r & 7)) * 16)) = v;
        }
    }
    fence_proxy_async_smem();
    if (t == 0) { mbar_init(bar, 1); fence_mbar_init(); }
    if (warp == 0) tmem_alloc<256>(tslot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tslot;
    const uint32_t lane_base = (32u * warp) << 16;

    if (Dinit != nullptr) {
        for (int c = 0; c < n; c += 16) {
            float v[16];
            for (int i = 0; i < 16; ++i) v[i] = Dinit[t * n + c + i];
            tmem_st16(tbase + lane_base + c, v);
        }
        tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    if (warp == 0) {
        if (elect_one()) {
            const uint32_t idesc = idesc_f16_f32(128, static_cast<uint32_t>(n));
            const uint64_t ad = sw128_kmajor_desc(smem_u32(sA));
            const uint64_t bd = sw128_kmajor_desc(smem_u32(sB));
            for (int j = 0; j < nsteps; ++j) {
                if (j == 0 && mode == 1) {
                    mma_f16_ss_scaled<11>(tbase, ad, bd, idesc);
                } else {
                    const uint32_t acc = (j > 0 || Dinit != nullptr) ? 1u : 0u;
                    mma_f16_ss(tbase, ad + 2 * j, bd + 2 * j, idesc, acc);
                }
            }
            tc_commit(bar);
        }
        __syncwarp();
    }
    mbar_wait(bar, 0);
    tc_fence_after();
    for (int c = 0; c < n; c += 16) {
        float v[16];
        tmem_ld16(tbase + lane_base + c, v);
        tmem_ld_wait();
        for (int i = 0; i < 16; ++i) Dout[t * n + c + i] = v[i];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<256>(tbase);
    }
}

}  // namespace shg

extern "C" shg_status_t shg_probe_umma(const uint16_t* A, const uint16_t* B, int n, const float* D_init,
                                       int mode, int nsteps, float* D_out, shg_stream_t stream) {
    if (!A || !B || !D_out || n < 16 || n > 256 || (n % 16) || nsteps < 1 || nsteps > 4 || mode < 0 || mode > 1)
        return SHG_ERR_INVALID_VALUE;
    if (mode == 1 && D_init == nullptr) return SHG_ERR_INVALID_VALUE;
    const int smem = 1024 + 128 * 128 + 256 * 128 + 64;
    cudaError_t e = cudaFuncSetAttribute(shg::probe_umma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return SHG_ERR_CUDA;
    shg::probe_umma_kernel<<<1, 128, smem, reinterpret_cast<cudaStream_t>(stream)>>>(A, B, n, D_init, mode, nsteps, D_out);
    e = cudaGetLastError();
    return e == cudaSuccess ? SHG_OK : SHG_ERR_CUDA;
}

// ------------------------------------------------------------------ MMA throughput microbenchmark
// Every CTA (1 per SM) issues `iters` tcgen05.mma.cta_group::1.kind::f16 128 x n x 16 back to back
// on resident operands (A from TMEM when ts != 0, else from smem; B from smem) into a TMEM
// accumulator, optionally while `lsu_warps` other warps stream LDS.128/STS.128 over a 64 KB smem
// region (to emulate the splitter's shared-memory traffic). out[blockIdx.x] = cycles / MMA.
namespace shg {
__global__ void __launch_bounds__(256, 1)
probe_mma_rate_kernel(int n, int iters, int ts, int lsu_warps, float* out, int nacc) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t* base = smem_raw + ((1024u - (raw_addr & 1023u)) & 1023u);
    uint8_t* sA = base;                  // 128 rows x 128 B
    uint8_t* sB = base + 16384;          // 256 rows x 128 B
    uint8_t* scratch = base + 16384 + 32768;   // 64 KB for LSU traffic
    uint64_t* bar = reinterpret_cast<uint64_t*>(scratch + 65536);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
    volatile uint32_t* stop = tslot + 1;
    const uint32_t warp = warp_id();
    for (int i = threadIdx.x; i < (16384 + 32768 + 65536) / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(base)[i] = make_uint4(0x3C003C00u, 0x3C003C00u, 0, 0);
    fence_proxy_async_smem();
    if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); *stop = 0; }
    if (warp == 0) tmem_alloc<512>(tslot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tslot;
    if (warp == 0) {
        if (elect_one()) {
            const uint32_t idesc = idesc_f16_f32(128, static_cast<uint32_t>(n));
            const uint64_t ad = sw128_kmajor_desc(smem_u32(sA));
            const uint64_t bd = sw128_kmajor_desc(smem_u32(sB));
            const long long t0 = clock64();
            for (int i = 0; i < iters; ++i) {
                const uint32_t j = static_cast<uint32_t>(i & 3);
                const uint32_t d = tbase + static_cast<uint32_t>((i % nacc) * n);
                if (ts) {
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n"
                                 ::"r"(d), "r"(tbase + 448 + 8 * j), "l"(bd + 2 * j), "r"(idesc) : "memory");
                } else {
                    mma_f16_ss(d, ad + 2 * j, bd + 2 * j, idesc, 1u);
                }
            }
            tc_commit(bar);
            mbar_wait(bar, 0);
            const long long t1 = clock64();
            out[blockIdx.x] = static_cast<float>(t1 - t0) / static_cast<float>(iters);
            *stop = 1;
        }
        __syncwarp();
    } else if (static_cast<int>(warp) <= lsu_warps) {
        // stream LDS.128 + STS.128 over the scratch region until the MMA warp finishes
        const int t = threadIdx.x - 32;
        uint4 acc = make_uint4(0, 0, 0, 0);
        while (*stop == 0) {
#pragma unroll 4
            for (int i = 0; i < 16; ++i) {
                const int idx = ((i * 224 + t) % 4096);
                uint4 v = reinterpret_cast<const uint4*>(scratch)[idx];
                acc.x ^= v.x; acc.y += v.y;
                reinterpret_cast<uint4*>(scratch)[(idx + 2048) % 4096] = acc;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tbase); }
}
}  // namespace shg

extern "C" shg_status_t shg_probe_mma_rate(int n, int iters, int ts, int lsu_warps, float* out, int grid,
                                           shg_stream_t stream) {
    // lsu_warps >= 8 encodes the number of independent accumulators: nacc = lsu_warps >> 3
    const int nacc = lsu_warps >= 8 ? (lsu_warps >> 3) : 1;
    lsu_warps &= 7;
    if (!out || n < 16 || n > 256 || (n % 16) || iters < 1 || grid < 1 || nacc * n > 448)
        return SHG_ERR_INVALID_VALUE;
    const int smem = 1024 + 16384 + 32768 + 65536 + 64;
    cudaError_t e = cudaFuncSetAttribute(shg::probe_mma_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return SHG_ERR_CUDA;
    shg::probe_mma_rate_kernel<<<grid, 256, smem, reinterpret_cast<cudaStream_t>(stream)>>>(n, iters, ts, lsu_warps, out, nacc);
    return cudaGetLastError() == cudaSuccess ? SHG_OK : SHG_ERR_CUDA;
}

// ------------------------------------------------------------------ cta_group::2 MMA rate
// Clusters of 2 CTAs; the leader issues `iters` tcgen05.mma.cta_group::2.kind::f16 with M = 256
// (128 rows per CTA), N = n, K = 16, A from TMEM (ts) or smem, B halves (n/2 rows) in each CTA's
// smem. out[cluster] = cycles per MMA instruction (each does 256 x n x 16 MACs on two SMs).
namespace shg {
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
probe_mma2_rate_kernel(int n, int iters, int ts, float* out) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t* base = smem_raw + ((1024u - (raw_addr & 1023u)) & 1023u);
    uint8_t* sA = base;                  // 128 rows x 128 B
    uint8_t* sB = base + 16384;          // up to 128 rows x 128 B (n/2 rows)
    uint64_t* bar = reinterpret_cast<uint64_t*>(base + 32768);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const uint32_t warp = warp_id();
    for (int i = threadIdx.x; i < 32768 / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(base)[i] = make_uint4(0x3C003C00u, 0x3C003C00u, 0, 0);
    fence_proxy_async_smem();
    if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    tc_fence_after();
    const uint32_t tbase = *tslot;
    if (rank == 0 && warp == 0) {
        if (elect_one()) {
            const uint32_t idesc = idesc_f16_f32(256, static_cast<uint32_t>(n));
            const uint64_t ad = sw128_kmajor_desc(smem_u32(sA));
            const uint64_t bd = sw128_kmajor_desc(smem_u32(sB));
            const long long t0 = clock64();
            for (int i = 0; i < iters; ++i) {
                const uint32_t j = static_cast<uint32_t>(i & 3);
                if (ts) {
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                                 "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n"
                                 ::"r"(tbase), "r"(tbase + 448 + 8 * j), "l"(bd + 2 * j), "r"(idesc) : "memory");
                } else {
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                                 "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
                                 ::"r"(tbase), "l"(ad + 2 * j), "l"(bd + 2 * j), "r"(idesc) : "memory");
                }
            }
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                         ::"r"(smem_u32(bar)), "h"(static_cast<uint16_t>(3)) : "memory");
            mbar_wait(bar, 0);
            const long long t1 = clock64();
            uint32_t cid;
            asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
            out[cid] = static_cast<float>(t1 - t0) / static_cast<float>(iters);
        }
        __syncwarp();
    } else if (rank == 1 && threadIdx.x == 0) {
        mbar_wait(bar, 0);
    }
    tc_fence_before();
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
    }
}
}  // namespace shg

extern "C" shg_status_t shg_probe_mma2_rate(int n, int iters, int ts, float* out, int clusters, shg_stream_t stream) {
    if (!out || n < 32 || n > 256 || (n % 32) || iters < 1 || clusters < 1) return SHG_ERR_INVALID_VALUE;
    const int smem = 1024 + 32768 + 64;
    cudaError_t e = cudaFuncSetAttribute(shg::probe_mma2_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return SHG_ERR_CUDA;
    shg::probe_mma2_rate_kernel<<<2 * clusters, 128, smem, reinterpret_cast<cudaStream_t>(stream)>>>(n, iters, ts, out);
    return cudaGetLastError() == cudaSuccess ? SHG_OK : SHG_ERR_CUDA;
}

// ------------------------------------------------------------------ MMA energy probe (diagnostics)
// Same tensor work split into `parts` MMAs per K step (N = n / parts each) on random FP16 data
// (A from TMEM, B from smem, both filled with hashed values in [-1, 1)), so that a long run under
// the power cap shows whether the N-split of the mainloop (two parts of N = 128 for BN = 256) costs
// energy: out[cluster] = clock64 cycles of the issuing loop.
namespace shg {
__device__ __forceinline__ uint32_t probe_hash(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}
__device__ __forceinline__ uint32_t rand_h2(uint32_t x) {
    const uint32_t h = probe_hash(x);
    const __half2 v = __floats2half2_rn(static_cast<float>(h & 0xFFFF) * (2.0f / 65536.0f) - 1.0f,
                                        static_cast<float>(h >> 16) * (2.0f / 65536.0f) - 1.0f);
    return *reinterpret_cast<const uint32_t*>(&v);
}

__global__ void __launch_bounds__(128, 1) probe_mma_energy_kernel(int n, int parts, int iters, long long* out) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t* base = smem_raw + ((1024u - (raw_addr & 1023u)) & 1023u);
    uint8_t* sB = base;                                   // 128 rows x 128 B (n/2 rows used)
    uint64_t* bar = reinterpret_cast<uint64_t*>(base + 16384);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const uint32_t warp = warp_id();
    for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(sB)[i] = rand_h2(static_cast<uint32_t>(i) * 2654435761u + rank);
    fence_proxy_async_smem();
    if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    tc_fence_after();
    const uint32_t tbase = *tslot;
    {   // A operand: TMEM columns 256..511 of this warp's lane quarter, random FP16 pairs
        const uint32_t lane_addr = (32u * (warp & 3u)) << 16;
        for (int c = 0; c < 256; c += 16) {
            uint32_t r[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) r[i] = rand_h2((threadIdx.x * 977u + c + i) * 40503u + rank * 7u);
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
                "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                ::"r"(tbase + lane_addr + 256 + c), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]),
                  "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]),
                  "r"(r[14]), "r"(r[15]) : "memory");
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    tc_fence_after();
    if (rank == 0 && warp == 0) {
        if (elect_one()) {
            const int w = n / parts;
            const uint32_t idesc = idesc_f16_f32(256, static_cast<uint32_t>(w));
            const uint64_t bd = sw128_kmajor_desc(smem_u32(sB));
            const long long t0 = clock64();
            for (int i = 0; i < iters; ++i) {
                const uint32_t j = static_cast<uint32_t>(i & 3);
                const uint32_t a = tbase + 256 + 8 * j + ((i & 4) ? 32u : 0u) + ((i & 8) ? 64u : 0u);
                for (int q = 0; q < parts; ++q) {
                    const uint64_t b = bd + static_cast<uint64_t>((q * (w / 2) * 128) >> 4) + 2 * j;
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                                 "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n"
                                 ::"r"(tbase + q * w), "r"(a), "l"(b), "r"(idesc) : "memory");
                }
            }
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                         ::"r"(smem_u32(bar)), "h"(static_cast<uint16_t>(3)) : "memory");
            mbar_wait(bar, 0);
            uint32_t cid;
            asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
            out[cid] = clock64() - t0;
        }
        __syncwarp();
    } else if (rank == 1 && threadIdx.x == 0) {
        mbar_wait(bar, 0);
    }
    tc_fence_before();
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
    }
}
}  // namespace shg

extern "C" shg_status_t shg_probe_mma_energy(int n, int parts, int iters, long long* out, int clusters,
                                             shg_stream_t stream) {
    if (!out || parts < 1 || parts > 2 || n % (32 * parts) || n < 32 || n > 256 || iters < 1 || clusters < 1)
        return SHG_ERR_INVALID_VALUE;
    const int smem = 1024 + 16384 + 64;
    cudaError_t e = cudaFuncSetAttribute(shg::probe_mma_energy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return SHG_ERR_CUDA;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * clusters);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = reinterpret_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, shg::probe_mma_energy_kernel, n, parts, iters, out);
    return e == cudaSuccess ? SHG_OK : SHG_ERR_CUDA;
}

// Box-Muller probe: the generator's radius and angle functions (omega.cuh) evaluated on given
// Philox words, so the tests can compare them with the oracle over every 24-bit code.
#include "omega.cuh"
namespace shg {
__global__ void probe_boxmuller_kernel(const uint32_t* __restrict__ words, int64_t count, float* __restrict__ r,
                                       float* __restrict__ c, float* __restrict__ s) {
    // words 2t and 2t + 1 go through the two lanes of the generator's packed radius / angle (an odd
    // last word is paired with itself)
    const int64_t npair = (count + 1) / 2;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < npair; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i0 = 2 * t, i1 = (2 * t + 1 < count) ? 2 * t + 1 : 2 * t;
        const uint32_t w0 = words[i0], w1 = words[i1];
        float2 cv, sv;
        omega::bm_angle2(w0, w1, cv, sv);
        const float2 rv = omega::bm_radius2(w0, w1);
        r[i0] = rv.x;
        c[i0] = cv.x;
        s[i0] = sv.x;
        if (i1 != i0) {
            r[i1] = rv.y;
            c[i1] = cv.y;
            s[i1] = sv.y;
        }
    }
}
}  // namespace shg

extern "C" shg_status_t shg_probe_boxmuller(const uint32_t* words, int64_t count, float* r, float* c, float* s,
                                            shg_stream_t stream) {
    if (count < 0 || (count > 0 && (!words || !r || !c || !s))) return SHG_ERR_INVALID_VALUE;
    if (count == 0) return SHG_OK;
    shg::probe_boxmuller_kernel<<<148 * 8, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(words, count, r, c, s);
    return cudaGetLastError() == cudaSuccess ? SHG_OK : SHG_ERR_CUDA;
}

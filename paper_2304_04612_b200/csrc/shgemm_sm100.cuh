// shgemm_sm100.cuh — the SHGEMM mainloop for B200 (sm_100a): Y = A_F32 . Omega_F16.
//
// Paper: Eqs 14-17 split each FP32 element of A into FP16 hi/lo and run
// hi.Omega and lo.Omega on the tensor cores; the hi product's accumulation is moved onto the
// FP32 RN units to avoid the tensor cores' RZ accumulation.
// The A100 design (WMMA, RN add after every f_k = 8 mma) is prior art, not the
// blueprint; this kernel re-derives it for tcgen05:
//
//  * A stager   : TMA (3-D map, SWIZZLE_128B) streams 128 x 64 FP32 tiles into an SA-deep ring.
//  * Splitter   : 4 warps read the FP32 tile from smem, apply split2 (Eqs 14-15) and write hi and
//                 lo in the UMMA K-major SW128 layout into an SB-deep ring (+ fence.proxy.async).
//  * Omega      : TMA streams the 64 x BN FP16 tile (K-major) into the same SB ring slot.
//  * MMA        : one thread issues, per 64-k stage, 4 lo MMAs (D := lo.Omega) and 4 hi MMAs, the
//                 first with scale-input-d = 11 (D := hi.Omega + D * 2^-11) — so D holds the
//                 stage's hi.Omega + 2^-11 lo.Omega (Eq 16) in an FP32 TMEM accumulator.
//                 Two D buffers (2 x BN TMEM columns) alternate between stages.
//  * Promotion  : 8 epilogue warps tcgen05.ld each finished D and add it with RN (add.rn.f32)
//                 into a register accumulator: the RZ-avoidance of PAPER.md:587 applied per
//                 K_c = 64 chunk instead of per A100 mma (and to lo too: reading c4-2).
//  * Epilogue   : after the last stage, the RN accumulator is written to Y (row-major) with
//                 128-bit stores, masked on ragged edges; split-K tiles write to a workspace
//                 plane that splitk_reduce_kernel sums in fixed order.
//
// One CTA per SM (smem-bound), persistent over tiles (m-block, k-split, n-block), n fastest.
#pragma once
#include <cstdint>
#include <cuda.h>
#include "ptx.cuh"
#include "split.cuh"

namespace shg {

constexpr int kBM = 128;                 // UMMA M (cta_group::1)
constexpr int kBK = 64;                  // k per stage: one 128-B swizzle row of FP16
constexpr int kA32StageBytes = kBM * kBK * 4;   // 32 KB (two 16 KB TMA boxes of 32 FP32 columns)
constexpr int kHLStageBytes = kBM * kBK * 2 * 2; // hi 16 KB + lo 16 KB
constexpr int kThreads = 512;
constexpr int kWarpProdA = 4, kWarpMMA = 5, kWarpProdB = 6;
constexpr int kEpiWarp0 = 8;
constexpr int kSmemLimit = 232448;       // max dynamic smem per block on sm_100

struct KParams {
    int64_t m, n, k;
    int64_t k_inner;        // S: contiguous k run of the A view (k for a plain matrix)
    int32_t num_kb;         // ceil(k / 64)
    int32_t m_tiles, n_tiles, splits;
    float* out;             // Y, or the split-K workspace when splits > 1
    int64_t ldo_out;        // leading dimension of out (elements)
    int64_t split_stride;   // elements between split planes (workspace)
    int32_t vec_store;      // out rows 16-B aligned and ldo_out % 4 == 0
    int* nonfinite;         // optional flag (set to 1 on any non-finite output)
};

__host__ __device__ constexpr uint32_t tmem_cols_for(uint32_t cols) {
    return cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
}

template <int BN>
struct Cfg {
    static constexpr int kOmStageBytes = BN * kBK * 2;
    static constexpr int SB = 2;
    static constexpr int kBarBytes = 256;
    static constexpr int SA_fit = (kSmemLimit - 1024 - kBarBytes - SB * (kHLStageBytes + kOmStageBytes)) / kA32StageBytes;
    static constexpr int SA = SA_fit > 4 ? 4 : SA_fit;
    static constexpr int kSmemBytes = 1024 + SA * kA32StageBytes + SB * (kHLStageBytes + kOmStageBytes) + kBarBytes;
    static constexpr uint32_t kTmemCols = tmem_cols_for(2 * BN);
    static constexpr int C = BN / 2;     // accumulator columns per epilogue thread
    static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "UMMA N for M=128");
    static_assert(SA >= 2, "smem");
    static_assert(kSmemBytes <= kSmemLimit, "smem");
};

__device__ __forceinline__ void tile_coords(int tile, const KParams& p, int& m_blk, int& s, int& n_blk) {
    const int per_m = p.splits * p.n_tiles;
    m_blk = tile / per_m;
    const int rem = tile - m_blk * per_m;
    s = rem / p.n_tiles;
    n_blk = rem - s * p.n_tiles;
}

__device__ __forceinline__ void kb_range(int s, const KParams& p, int& lo, int& hi) {
    lo = static_cast<int>((static_cast<int64_t>(s) * p.num_kb) / p.splits);
    hi = static_cast<int>((static_cast<int64_t>(s + 1) * p.num_kb) / p.splits);
}

__device__ __forceinline__ void advance(uint32_t& stage, uint32_t& phase, uint32_t n) {
    if (++stage == n) { stage = 0; phase ^= 1u; }
}

template <int BN>
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
shgemm_sm100_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                    const KParams p) {
    using CF = Cfg<BN>;
    constexpr int SA = CF::SA, SB = CF::SB, C = CF::C;
    constexpr int kOm = CF::kOmStageBytes;

    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t* base = smem_raw + ((1024u - (raw_addr & 1023u)) & 1023u);
    uint8_t* a32 = base;
    uint8_t* hl = a32 + SA * kA32StageBytes;
    uint8_t* om = hl + SB * kHLStageBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(om + SB * kOm);
    uint64_t* a_full = bars;
    uint64_t* a_empty = a_full + SA;
    uint64_t* hl_full = a_empty + SA;
    uint64_t* om_full = hl_full + SB;
    uint64_t* b_empty = om_full + SB;
    uint64_t* acc_full = b_empty + SB;
    uint64_t* acc_empty = acc_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const uint32_t warp = warp_id();
    const uint32_t lane = threadIdx.x & 31u;

    if (threadIdx.x == 0) {
        for (int i = 0; i < SA; ++i) { mbar_init(&a_full[i], 1); mbar_init(&a_empty[i], 4); }
        for (int i = 0; i < SB; ++i) {
            mbar_init(&hl_full[i], 4); mbar_init(&om_full[i], 1); mbar_init(&b_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) { mbar_init(&acc_full[i], 1); mbar_init(&acc_empty[i], 8); }
        fence_mbar_init();
    }
    if (warp == kWarpProdA && lane == 0) {
        tma_prefetch_desc(&mapA);
        tma_prefetch_desc(&mapB);
    }
    if (warp == kWarpMMA) tmem_alloc<CF::kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int num_tiles = p.m_tiles * p.splits * p.n_tiles;

    if (warp < 4) {
        // ============================================================ splitter (Eqs 14-15)
        asm volatile("setmaxnreg.dec.sync.aligned.u32 64;");
        const int t = threadIdx.x;                       // 0..127
        const int w = t >> 5, l = t & 31;
        const int r = 32 * w + 8 * (l >> 3) + (l & 7);   // tile row owned by this thread
        const int rx = r & 7;                            // SW128 XOR term of this row
        uint32_t sa = 0, pa = 0, sb = 0, pb = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            int m_blk, s, n_blk, kb0, kb1;
            tile_coords(tile, p, m_blk, s, n_blk);
            kb_range(s, p, kb0, kb1);
            for (int kb = kb0; kb < kb1; ++kb) {
                mbar_wait(&a_full[sa], pa);
                mbar_wait(&b_empty[sb], pb ^ 1u);
                const uint8_t* src = a32 + sa * kA32StageBytes + r * 128;
                uint8_t* dhi = hl + sb * kHLStageBytes + r * 128;
                uint8_t* dlo = dhi + kHLStageBytes / 2;
#pragma unroll
                for (int c = 0; c < 8; ++c) {            // FP16 16-B chunk c = k 8c .. 8c+7
                    const uint8_t* box = src + (c >> 2) * (kA32StageBytes / 2);
                    const int f0 = ((2 * (c & 3)) ^ rx) * 16;
                    const int f1 = ((2 * (c & 3) + 1) ^ rx) * 16;
                    const float4 x0 = *reinterpret_cast<const float4*>(box + f0);
                    const float4 x1 = *reinterpret_cast<const float4*>(box + f1);
                    uint4 h, lo;
                    split8(x0, x1, h, lo);
                    const int dc = (c ^ rx) * 16;
                    *reinterpret_cast<uint4*>(dhi + dc) = h;
                    *reinterpret_cast<uint4*>(dlo + dc) = lo;
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (l == 0) {
                    mbar_arrive(&hl_full[sb]);
                    mbar_arrive(&a_empty[sa]);
                }
                advance(sa, pa, SA);
                advance(sb, pb, SB);
            }
        }
    } else if (warp < 8) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 64;");
        if (warp == kWarpProdA) {
            // ======================================================== A stager (TMA, FP32)
            if (elect_one()) {
                const uint64_t pol = policy_evict_first();
                uint32_t sa = 0, pa = 0;
                for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                    int m_blk, s, n_blk, kb0, kb1;
                    tile_coords(tile, p, m_blk, s, n_blk);
                    kb_range(s, p, kb0, kb1);
                    const int m0 = m_blk * kBM;
                    for (int kb = kb0; kb < kb1; ++kb) {
                        mbar_wait(&a_empty[sa], pa ^ 1u);
                        mbar_arrive_expect_tx(&a_full[sa], kA32StageBytes);
                        const int64_t kk = static_cast<int64_t>(kb) * kBK;
                        const int c0 = static_cast<int>(kk % p.k_inner);
                        const int c2 = static_cast<int>(kk / p.k_inner);
                        uint8_t* dst = a32 + sa * kA32StageBytes;
                        tma_load_3d(dst, &mapA, &a_full[sa], c0, m0, c2, pol);
                        tma_load_3d(dst + kA32StageBytes / 2, &mapA, &a_full[sa], c0 + 32, m0, c2, pol);
                        advance(sa, pa, SA);
                    }
                }
            }
        } else if (warp == kWarpProdB) {
            // ======================================================== Omega stager (TMA, FP16)
            if (elect_one()) {
                const uint64_t pol = policy_evict_last();
                uint32_t sb = 0, pb = 0;
                for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                    int m_blk, s, n_blk, kb0, kb1;
                    tile_coords(tile, p, m_blk, s, n_blk);
                    kb_range(s, p, kb0, kb1);
                    const int n0 = n_blk * BN;
                    for (int kb = kb0; kb < kb1; ++kb) {
                        mbar_wait(&b_empty[sb], pb ^ 1u);
                        mbar_arrive_expect_tx(&om_full[sb], kOm);
                        tma_load_2d(om + sb * kOm, &mapB, &om_full[sb], kb * kBK, n0, pol);
                        advance(sb, pb, SB);
                    }
                }
            }
        } else if (warp == kWarpMMA) {
            // ======================================================== MMA issuer (tcgen05)
            constexpr uint32_t idesc = idesc_f16_f32(kBM, BN);
            uint32_t sb = 0, pb = 0, buf = 0, pacc = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                int m_blk, s, n_blk, kb0, kb1;
                tile_coords(tile, p, m_blk, s, n_blk);
                kb_range(s, p, kb0, kb1);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&acc_empty[buf], pacc ^ 1u);
                    mbar_wait(&hl_full[sb], pb);
                    mbar_wait(&om_full[sb], pb);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t d = tmem_base + buf * BN;
                        const uint64_t ahi = sw128_kmajor_desc(smem_u32(hl + sb * kHLStageBytes));
                        const uint64_t alo = sw128_kmajor_desc(smem_u32(hl + sb * kHLStageBytes + kHLStageBytes / 2));
                        const uint64_t bd = sw128_kmajor_desc(smem_u32(om + sb * kOm));
                        // D := lo . Omega   (4 x K=16; +32 B per step inside the 128-B swizzle row)
#pragma unroll
                        for (int j = 0; j < 4; ++j) mma_f16_ss(d, alo + 2 * j, bd + 2 * j, idesc, j > 0 ? 1u : 0u);
                        // D := hi . Omega + D * 2^-11, then accumulate the rest of hi
                        mma_f16_ss_scaled<11>(d, ahi, bd, idesc);
#pragma unroll
                        for (int j = 1; j < 4; ++j) mma_f16_ss(d, ahi + 2 * j, bd + 2 * j, idesc, 1u);
                        tc_commit(&b_empty[sb]);
                        tc_commit(&acc_full[buf]);
                    }
                    __syncwarp();
                    advance(sb, pb, SB);
                    advance(buf, pacc, 2);
                }
            }
        }
    } else {
        // ============================================================ RN promotion + epilogue
        asm volatile("setmaxnreg.inc.sync.aligned.u32 192;");
        const int q = static_cast<int>(warp & 3u);           // TMEM lane quarter (warp_id % 4)
        const int h = static_cast<int>((warp - kEpiWarp0) >> 2);  // column half
        const uint32_t lane_base = static_cast<uint32_t>(32 * q) << 16;
        uint32_t buf = 0, pacc = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            int m_blk, s, n_blk, kb0, kb1;
            tile_coords(tile, p, m_blk, s, n_blk);
            kb_range(s, p, kb0, kb1);
            float acc[C];
#pragma unroll
            for (int i = 0; i < C; ++i) acc[i] = 0.0f;
            for (int kb = kb0; kb < kb1; ++kb) {
                mbar_wait(&acc_full[buf], pacc);
                tc_fence_after();
                const uint32_t taddr = tmem_base + lane_base + buf * BN + h * C;
#pragma unroll
                for (int c = 0; c < C; c += 32) {
                    constexpr int kMax = 32;
                    float v[4][8];
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (c + 8 * u < C) tmem_ld8<BN>(taddr + c + 8 * u, v[u]);
                    tmem_ld_wait();
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int i = 0; i < 8; ++i)
                            if (c + 8 * u < C) acc[c + 8 * u + i] = __fadd_rn(acc[c + 8 * u + i], v[u][i]);
                    (void)kMax;
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&acc_empty[buf]);
                advance(buf, pacc, 2);
            }
            // ---- store the tile rows owned by this thread
            const int64_t row = static_cast<int64_t>(m_blk) * kBM + 32 * q + static_cast<int>(lane);
            const int64_t col0 = static_cast<int64_t>(n_blk) * BN + h * C;
            if (row < p.m && col0 < p.n) {
                float* dst = p.out + static_cast<int64_t>(s) * p.split_stride + row * p.ldo_out + col0;
                const int64_t valid = p.n - col0;
                bool bad = false;
                if (p.vec_store && valid >= C) {
#pragma unroll
                    for (int i = 0; i < C; i += 4)
                        *reinterpret_cast<float4*>(dst + i) = make_float4(acc[i], acc[i + 1], acc[i + 2], acc[i + 3]);
                } else {
#pragma unroll
                    for (int i = 0; i < C; ++i)
                        if (i < valid) dst[i] = acc[i];
                }
                if (p.nonfinite) {
#pragma unroll
                    for (int i = 0; i < C; ++i)
                        if (i < valid && !isfinite(acc[i])) bad = true;
                    if (bad) atomicOr(p.nonfinite, 1);
                }
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == kWarpMMA) {
        tc_fence_after();
        tmem_dealloc<CF::kTmemCols>(tmem_base);
    }
}

// Fixed-order (s = 0..S-1) RN sum of split-K partial planes (a8 of SURVEY §8a; deterministic).
__global__ void splitk_reduce_kernel(const float* __restrict__ ws, int splits, int64_t m, int64_t n,
                                     int64_t ld_ws, int64_t split_stride, float* __restrict__ Y, int64_t ldc,
                                     int* nonfinite) {
    const int64_t total = m * n;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = t / n, j = t - (t / n) * n;
        float acc = ws[i * ld_ws + j];
        for (int s = 1; s < splits; ++s) acc = __fadd_rn(acc, ws[s * split_stride + i * ld_ws + j]);
        Y[i * ldc + j] = acc;
        if (nonfinite && !isfinite(acc)) atomicOr(nonfinite, 1);
    }
}

}  // namespace shg

// api.cu — the C ABI of include/shgemm.h: validation, planning (tile N, split-K, grid),
// TMA tensor-map encoding (cuTensorMapEncodeTiled through cudaGetDriverEntryPoint, no -lcuda),
// and kernel launches. No torch types cross this boundary.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "../../include/shgemm.h"
#include "internal.cuh"
#include "omega.cuh"
#include "probe_tma.cuh"
#include "shgemm_sm100.cuh"
#include "simt_fallback.cuh"
#include "split.cuh"
#include "tcec.cuh"

namespace shg_api {

std::atomic<uint64_t> g_launches{0};
thread_local char g_err[256] = "";

shg_status_t cuda_fail(cudaError_t e, const char* what) {
    std::snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
    return SHG_ERR_CUDA;
}

}  // namespace shg_api

namespace {

using namespace shg_api;

struct DevInfo {
    int sms = 0;
    int major = 0, minor = 0;
    bool ok = false;
};

DevInfo& dev_info() {
    static DevInfo infos[64];
    static std::once_flag flags[64];
    int dev = 0;
    cudaGetDevice(&dev);
    dev = std::min(std::max(dev, 0), 63);
    std::call_once(flags[dev], [dev]() {
        DevInfo& d = infos[dev];
        cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&d.major, cudaDevAttrComputeCapabilityMajor, dev);
        cudaDeviceGetAttribute(&d.minor, cudaDevAttrComputeCapabilityMinor, dev);
        d.ok = (d.major == 10 && d.minor == 0);
        // stream-ordered scratch (split-K planes, B splits, Omega of project()) comes from the default
        // pool: keep freed blocks in the pool instead of returning them to the OS at every sync
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        (void)cudaGetLastError();
    });
    return infos[dev];
}

// ------------------------------------------------------------------ TMA encode
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    static std::once_flag flag;
    std::call_once(flag, []() {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    return fn;
}

// A view: dims {S (k inner), M, P (k outer)}, strides (bytes) {row, slab}; box {32, 128, 1}
bool encode_a(CUtensorMap* map, const float* A, int64_t S, int64_t M, int64_t P, int64_t row_stride_el,
              int64_t slab_stride_el) {
    EncodeFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(S), static_cast<cuuint64_t>(M), static_cast<cuuint64_t>(P)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(row_stride_el) * 4, static_cast<cuuint64_t>(slab_stride_el) * 4};
    cuuint32_t box[3] = {32, 128, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(A), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Same view as a 4-D map {32, S/32, M, P} (S % 32 == 0), box {32, 2, 128, 1}: TMA walks the box
// row by row, 256 B per row visit (twice encode_a's 128 B). Measured with shg_probe_tma_read on a
// 1024 x 2^20 matrix: 4.5 TB/s for 128-B row visits vs 7.1 TB/s for 256-B (6.4 vs 7.1 at 256-KB
// row strides) — each row visit costs a DRAM page / TLB lookup, so fewer, longer visits stream
// faster (profiles/r01_tma_probe.jsonl).
bool encode_a_rowpair(CUtensorMap* map, const float* A, int64_t S, int64_t M, int64_t P, int64_t row_stride_el,
                      int64_t slab_stride_el) {
    EncodeFn fn = encode_fn();
    if (!fn || S % 32) return false;
    cuuint64_t dims[4] = {32, static_cast<cuuint64_t>(S / 32), static_cast<cuuint64_t>(M), static_cast<cuuint64_t>(P)};
    cuuint64_t strides[3] = {128, static_cast<cuuint64_t>(row_stride_el) * 4, static_cast<cuuint64_t>(slab_stride_el) * 4};
    cuuint32_t box[4] = {32, 2, 128, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(A), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// TF32 copy of Omega (column-major k x n FP32 bit patterns, ldo32 % 4 == 0): dims {k, n}, box {32 k, rows}
bool encode_b32(CUtensorMap* map, const float* Om32, int64_t k, int64_t n, int64_t ldo32, int rows) {
    EncodeFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(n)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldo32) * 4};
    cuuint32_t box[2] = {32, static_cast<cuuint32_t>(rows)};
    cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(Om32), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Omega (column-major k x n == n rows of ldo halves): dims {k, n}, box {64 k, rows}
bool encode_b(CUtensorMap* map, const uint16_t* Om, int64_t k, int64_t n, int64_t ldo, int rows) {
    EncodeFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(n)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldo) * 2};
    cuuint32_t box[2] = {64, static_cast<cuuint32_t>(rows)};
    cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<uint16_t*>(Om), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// k-tiled FP32 (TF32) copy of Omega (widen_omega_tiled_kernel): dims {32, n, ceil(k/32)}, box {32 k, rows, 1}
bool encode_b32_tiled(CUtensorMap* map, const float* Om32, int64_t k, int64_t n, int rows) {
    EncodeFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {32, static_cast<cuuint64_t>(n), static_cast<cuuint64_t>((k + 31) / 32)};
    cuuint64_t strides[2] = {128, static_cast<cuuint64_t>(n) * 128};
    cuuint32_t box[3] = {32, static_cast<cuuint32_t>(rows), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(Om32), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// k-tiled Omega (gen_omega_f16_tiled): dims {64, n, ceil(k/64)}, box {64 k, rows, 1} — each 64-k
// box is ONE contiguous run of rows x 128 B (the column-major box visits rows 128 B at a time, ldo*2
// bytes apart: 2 MiB apart for an RP-HOSVD unfolding with k = 2^20, one DRAM page per visit)
bool encode_b_tiled(CUtensorMap* map, const uint16_t* Om, int64_t k, int64_t n, int rows) {
    EncodeFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(n), static_cast<cuuint64_t>((k + 63) / 64)};
    cuuint64_t strides[2] = {128, static_cast<cuuint64_t>(n) * 128};
    cuuint32_t box[3] = {64, static_cast<cuuint32_t>(rows), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<uint16_t*>(Om), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ------------------------------------------------------------------ planning
template <int B> using CfgPair = shg::Cfg<B, true, false>;
template <int B> using CfgSingle = shg::Cfg<B, false, false>;
template <int B> using CfgPairT = shg::Cfg<B, true, true>;
template <int B> using CfgSingleT = shg::Cfg<B, false, true>;
template <int B> using CfgPairC = shg::Cfg<B, true, false, true>;
template <int B> using CfgSingleC = shg::Cfg<B < 128 ? B : 128, false, false, true>;
#define SHG_CFG_FIELD(bn, pair, tf32, FIELD)                                                              \
    if (!tf32 && bn == 272) return pair ? shg::Cfg<272, true>::FIELD : shg::Cfg<272, false>::FIELD;      \
    if (!tf32 && bn == 288) return pair ? shg::Cfg<288, true>::FIELD : shg::Cfg<288, false>::FIELD;      \
    if (tf32 && pair) { SHG_BN_SWITCH(bn, return CfgPairT<BN_>::FIELD) }                                  \
    if (tf32) { SHG_BN_SWITCH(bn, return CfgSingleT<BN_>::FIELD) }                                        \
    if (pair) { SHG_BN_SWITCH(bn, return CfgPair<BN_>::FIELD) }                                           \
    SHG_BN_SWITCH(bn, return CfgSingle<BN_>::FIELD)

int smem_for(int bn, bool pair, bool tf32) { SHG_CFG_FIELD(bn, pair, tf32, kSmemBytes) }
int sa_for(int bn, bool pair, bool tf32) { SHG_CFG_FIELD(bn, pair, tf32, SA) }
int so_for(int bn, bool pair, bool tf32) { SHG_CFG_FIELD(bn, pair, tf32, SO) }
int r0_for(int bn, bool pair, bool tf32) { SHG_CFG_FIELD(bn, pair, tf32, R0) }
int r1_for(int bn, bool pair, bool tf32) { SHG_CFG_FIELD(bn, pair, tf32, R1) }
// TCEC-SGEMM configurations (pairs: BN >= 128; single CTAs: BN <= 128)
#define SHG_CFG_FIELD_TCEC(bn, pair, FIELD)                                                              \
    if (pair && bn == 272) return shg::Cfg<272, true, false, true>::FIELD;                                \
    if (pair && bn == 288) return shg::Cfg<288, true, false, true>::FIELD;                                \
    if (pair) { SHG_BN_SWITCH(bn, return CfgPairC<(BN_ < 128 ? 128 : BN_)>::FIELD) }                      \
    SHG_BN_SWITCH(bn, return CfgSingleC<BN_>::FIELD)
int smem_for_tcec(int bn, bool pair) { SHG_CFG_FIELD_TCEC(bn, pair, kSmemBytes) }
int sa_for_tcec(int bn, bool pair) { SHG_CFG_FIELD_TCEC(bn, pair, SA) }
int so_for_tcec(int bn, bool pair) { SHG_CFG_FIELD_TCEC(bn, pair, SO) }
int r0_for_tcec(int bn, bool pair) { SHG_CFG_FIELD_TCEC(bn, pair, R0) }
int r1_for_tcec(int bn, bool pair) { SHG_CFG_FIELD_TCEC(bn, pair, R1) }

struct Plan {
    int path = 0;  // 0 tc, 1 simt, 2 trivial
    int bn = 0, n_tiles = 0, m_tiles = 0, splits = 1, grid = 0, num_kb = 0;
    bool pair = false;
    bool tf32 = false;        // SHGEMM-TF32 (tune->tc == SHG_TC_TF32)
    bool tcec = false;        // TCEC-SGEMM (FP32 B split into B_low / dB_low)
    bool sk = false;          // stream-K schedule (KParams::sk): equal k-ranges per SM (pair), in-kernel fix-up
    int npa = 1;              // CTA pairs per cluster sharing each A stage by TMA multicast (NPA > 1)
    int64_t sk_planes = 0;    // stream-K: bytes of the partial planes (the counters follow, 256-B aligned)
    // workspace = [split-K planes, 256-B aligned][TF32 copy of Omega | TCEC split of B]
    int64_t ws_bytes = 0, ld_ws = 0, sk_bytes = 0, om_bytes = 0, ldo32 = 0;
    int64_t ldh = 0, noff = 0;  // TCEC: split B column-major, ld ldh; dB_low starts at column noff
    int64_t ldt = 0;            // row-major FP16 Omega: leading dimension of its column-major copy
};

int64_t up256(int64_t b) { return (b + 255) / 256 * 256; }

// Cooperative in-kernel Omega generation request (project(): k-tiled Omega generated by the
// mainloop's epilogue warps instead of a separate gen_omega launch)
struct OmGen {
    uint64_t seed;
    uint32_t stream_id;
    int dist;
    uint32_t thr;
    int64_t row0;           // spec row of local row 0 (multiple of 4)
    uint32_t* flags;        // ceil(k/64) zero-initialised ready flags
};
int omgen_mode();           // shg_set_inkernel_omega's setting (below)

// Stream-K is chosen automatically only on the HBM side of the roofline (BN <= kSkAutoMaxBn), where
// a partly idle last wave of whole tiles cannot keep HBM busy: measured interleaved under the 1000 W
// cap (profiles/r02_ab_streamk2.jsonl), m = k = 32768: n = 128 0.863 -> 0.749 ms, n = 64 0.694 ->
// 0.653, n = 96 0.685 -> 0.646. On the tensor side the idle wave is paid back by the power cap
// (profiles/r02_ab_streamk.jsonl: cfg2's projection 0.297 vs 0.298 ms, n = 192 0.970 vs 0.992), and
// short-wide split-K shapes (cfg3's unfoldings) stay split (r02_ab_streamk3.jsonl).
constexpr bool kSkAuto = true;
constexpr int kSkAutoMaxBn = 160;
constexpr double kSkMinWaveEff = 0.92;   // ... and whole tiles would leave the last wave < 92% busy

// A multicast chosen automatically (tune->a_mcast == 0): 2 pairs per cluster whenever the N tiles
// pair up. Measured in steady state under the 1000 W cap (blocks of >= 1.5 s back-to-back calls per
// variant, interleaved, profiles/r02_ab_amc_steady.jsonl): m = k = 32768 n = 512 2.12 -> 1.97 ms,
// n = 1024 3.91 -> 3.82; m = 2^21, k = 4096, n = 512 18.5 -> 17.0, n = 1024 36.4 -> 33.6 (4 pairs
// per cluster: 33.0, and 3.91 at 32768^2): A is read once per cluster instead of once per N tile,
// and the SM clock under the cap rises from 0.95-1.05 to 1.16-1.27 GHz, more than paying for the
// 132 of 148 SMs that clusters of 4 CTAs occupy. shg_set_a_mcast() overrides the default per process.
std::atomic<int> g_amc_default{0};      // 0 auto, 1 off, 2 / 4 (where eligible)
inline int auto_amcast(int n_tiles) {
    const int g = g_amc_default.load(std::memory_order_relaxed);
    if (g == 1 || g == 2 || g == 4) return g;
    return (n_tiles >= 2 && n_tiles % 2 == 0) ? 2 : 1;
}


// om_rm: Omega is row-major; the FP16 tensor-core path then reads a column-major copy
// made in the workspace by transpose_omega_kernel (TF32 widens either layout directly)
Plan make_plan(int64_t m, int64_t n, int64_t k, bool fast_ok, const shg_tune_t* tune, int sms, bool tcec = false,
               bool om_rm = false, bool allow_sk = true, bool a_kmajor = true) {
    Plan pl;
    pl.tf32 = !tcec && tune && tune->tc == SHG_TC_TF32;
    pl.tcec = tcec;
    if (m == 0 || n == 0 || k == 0) { pl.path = 2; return pl; }
    if (tcec) {   // the B split runs on every path
        pl.ldh = (k + 7) / 8 * 8;
    }
    if (!fast_ok || (tune && tune->force_simt)) {
        pl.path = 1;
        if (tcec) {
            pl.noff = n;
            pl.om_bytes = 2 * pl.noff * pl.ldh * 2;
            pl.ws_bytes = pl.om_bytes;
        }
        return pl;
    }
    pl.path = 0;
    // CTA pair: halves Omega's L2->SMEM traffic per SM (the power-cap lever at BN >= 128); needs > 128 rows
    const int pair_mode = tune ? tune->pair : 0;   // 0 auto, 1 force on, 2 force off
    const bool want_pair = (pair_mode == 0 && m > shg::kBM) || pair_mode == 1;
    // TCEC stages two B tiles: single CTAs stop at BN = 128; wide tiles (BN 272 / 288) are FP16-only
    const int max_bn = (tcec && !want_pair) ? kTcecMaxBnSingle : 256;
    if (tune && tune->bn > 0 && valid_bn(tune->bn)) {
        pl.bn = tune->bn;
        if (pl.bn > max_bn && !(wide_bn(pl.bn) && !pl.tf32 && (!tcec || want_pair))) { pl.path = -1; return pl; }
        pl.n_tiles = static_cast<int>((n + pl.bn - 1) / pl.bn);
    } else {
        pl.n_tiles = static_cast<int>((n + max_bn - 1) / max_bn);
        // SHGEMM-FP16, 256 < n <= 288: ONE wide tile (BN 272 / 288) instead of two of <= 144, so A
        // streams once: 0.29 vs 0.35 ms at cfg2, 11.1 vs 16.0 ms at m = 2^21 (profiles/r01_ab_wide.jsonl).
        // Not for n > 288: two wide tiles of 272 measured slower than three of 192 at n = 544.
        // TCEC-SGEMM likewise when it runs as CTA pairs (RSVD line 3: n = p + s = 272).
        if (!pl.tf32 && (!tcec || want_pair) && n > 256 && n <= 288) pl.n_tiles = 1;
        const int64_t need = (n + pl.n_tiles - 1) / pl.n_tiles;
        pl.bn = 288;
        for (int b : kBNs) if (b >= need) { pl.bn = b; break; }
    }
    pl.pair = pair_ok(pl.bn) && want_pair;
    // Omega multicast across CTA pairs of a cluster was removed in round 2 (no steady-state gain,
    // DESIGN.md §5): 0 and 1 mean unicast, anything else is rejected
    const int mc = tune ? tune->omega_mcast : 0;
    if (mc < 0 || mc > 1) { pl.path = -1; return pl; }
    const int sk_mode = tune ? tune->stream_k : 0;   // 0 auto, 1 force on, 2 off
    if (sk_mode < 0 || sk_mode > 2) { pl.path = -1; return pl; }
    const int tile_m = pl.pair ? 2 * shg::kBM : shg::kBM;
    int cap = (tune && tune->max_ctas > 0) ? tune->max_ctas : sms;
    const int cl = pl.pair ? 2 : 1;                 // CTAs per cluster (= per work unit)
    cap = std::max(cl, cap / cl * cl);
    const int slots = std::max(1, cap / cl);        // concurrent tiles (work units)
    pl.m_tiles = static_cast<int>((m + tile_m - 1) / tile_m);
    pl.num_kb = static_cast<int>((k + shg::kBK - 1) / shg::kBK);
    const int64_t mn_tiles = static_cast<int64_t>(pl.m_tiles) * pl.n_tiles;
    // stream-K (KParams::sk): when whole tiles quantise badly onto the units (the last wave mostly
    // idle) but there are at least half as many tiles as units; one N tile (the N tiles of an
    // m-block then share A in L2 by running together); >= 4 k-blocks per unit
    const int64_t waves = (mn_tiles + slots - 1) / slots;
    const double wave_eff = static_cast<double>(mn_tiles) / static_cast<double>(waves * slots);
    const bool sk_fits = allow_sk && pl.n_tiles == 1 && mn_tiles * pl.num_kb >= int64_t(4) * slots &&
                         !(tune && tune->split_k > 1);
    pl.sk = sk_fits && (sk_mode == 1 || (kSkAuto && sk_mode == 0 && pl.bn <= kSkAutoMaxBn &&
                                          wave_eff < kSkMinWaveEff && 2 * mn_tiles >= slots && pl.num_kb >= 16));
    if (sk_mode == 1 && !sk_fits) { pl.path = -1; return pl; }
    int splits = 1;
    const bool amc_req = tune && tune->a_mcast >= 2;   // an explicit A multicast request keeps whole tiles
    if (tune && tune->split_k > 0) {
        splits = tune->split_k;
    } else if (!pl.sk && !amc_req && mn_tiles < slots && pl.num_kb >= 16) {
        // fill the SMs with k-splits, keeping >= 4 k-blocks (256 k) per split; not for k < 1024,
        // where the partial planes and the extra reduce launch cost more than the idle SMs
        // (cfg1, 512 x 512 x 32: split 1/2/4/8 all within 2 us, profiles/r01_small_split.jsonl)
        splits = static_cast<int>(std::max<int64_t>(1, slots / mn_tiles));
        splits = static_cast<int>(std::min<int64_t>(splits, std::max<int64_t>(1, pl.num_kb / 4)));
    }
    splits = std::max(1, std::min(splits, pl.num_kb));
    pl.splits = splits;
    const int64_t tiles = mn_tiles * splits;
    pl.grid = pl.sk ? slots * cl : static_cast<int>(std::min<int64_t>(tiles * cl, cap));
    pl.grid = std::max(cl, pl.grid / cl * cl);
    // A multicast (tune->a_mcast; shgemm_sm100_kernel<..., NPA>): clusters of NPA pairs share each A
    // stage across NPA N tiles of one m-block. Decided after splits / stream-K, which it does not
    // change (it needs neither), so the workspace is the same with or without it.
    const int amc = tune ? tune->a_mcast : 0;      // 0 auto, 1 off, 2 / 4 pairs per cluster
    if (amc < 0 || amc == 3 || amc > 4) { pl.path = -1; return pl; }
    const int npa_want = amc >= 2 ? amc : (amc == 1 ? 1 : auto_amcast(pl.n_tiles));
    if (npa_want > 1) {
        const bool amc_ok = pl.pair && !pl.tf32 && !tcec && a_kmajor && !pl.sk && splits == 1 &&
                            !wide_bn(pl.bn) && (pl.bn == 128 || pl.bn == 192 || pl.bn == 256) &&
                            pl.n_tiles % npa_want == 0 && pl.n_tiles >= npa_want;
        if (amc_ok) {
            pl.npa = npa_want;
            const int cln = 2 * pl.npa;
            const int64_t groups = static_cast<int64_t>(pl.m_tiles) * (pl.n_tiles / pl.npa);
            const int capn = std::max(cln, cap / cln * cln);
            pl.grid = static_cast<int>(std::min<int64_t>(groups * cln, capn));
        } else if (amc >= 2) {
            pl.path = -1;
            return pl;
        }
    }
    if (splits > 1) {
        pl.ld_ws = (n + 3) / 4 * 4;
        pl.sk_bytes = static_cast<int64_t>(splits) * m * pl.ld_ws * 4;
    } else if (pl.sk) {
        // 2 partial slots per unit x CTAs per unit x (BN x 128) floats, then one counter per tile and CTA
        pl.sk_planes = up256(static_cast<int64_t>(2) * (pl.grid / cl) * cl * pl.bn * shg::kBM * 4);
        pl.sk_bytes = pl.sk_planes + up256(mn_tiles * cl * 4);
    }
    if (pl.tf32) {   // Omega widened once to TF32 (exact) for the tensor cores' smem operand
        pl.ldo32 = (k + 3) / 4 * 4;
        pl.om_bytes = (k + 31) / 32 * 32 * n * 4;   // column-major (ldo32) or 32-k tiles
    }
    if (pl.tcec) {   // [B_low | pad | dB_low | pad], each n_tiles * BN columns (pads zeroed)
        pl.noff = static_cast<int64_t>(pl.n_tiles) * pl.bn;
        pl.om_bytes = 2 * pl.noff * pl.ldh * 2;
    } else if (om_rm && !pl.tf32) {   // column-major copy of a row-major Omega (ldt % 8 == 0: TMA pitch)
        pl.ldt = (k + 7) / 8 * 8;
        pl.om_bytes = n * pl.ldt * 2;
    }
    pl.ws_bytes = (pl.om_bytes ? up256(pl.sk_bytes) : pl.sk_bytes) + pl.om_bytes;
    return pl;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }


// M-major A (element (i, l) at A[l * lda + i]): 2-D map {M, K}, box {128 rows, 64 k}, no swizzle
// (512 contiguous bytes per k-line; rows >= M zero-filled)
bool encode_a_mmajor(CUtensorMap* map, const float* A, int64_t M, int64_t K, int64_t lda) {
    EncodeFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(M), static_cast<cuuint64_t>(K)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(lda) * 4};
    cuuint32_t box[2] = {128, 64};
    cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(A), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int grid_for(int64_t work, int threads) {
    const int sms = std::max(1, dev_info().sms);
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((work + threads - 1) / threads, int64_t(sms) * 16)));
}

// gen_omega_kernel's 2-D grid: columns over y, 256-thread row-block strips over x, ~16 blocks/SM
dim3 omega_grid(int64_t nq, int64_t n) {
    const int sms = std::max(1, dev_info().sms);
    const int64_t y = std::min<int64_t>(std::max<int64_t>(n, 1), 65535);
    const int64_t x = std::max<int64_t>(1, std::min<int64_t>((nq + 255) / 256, (int64_t(sms) * 16 + y - 1) / y));
    return dim3(static_cast<unsigned>(x), static_cast<unsigned>(y));
}

// Generic A view used by shgemm (plain matrix) and project (unfoldings):
// K-major : element (row, kk) at A[(kk / S) * slab + row * row_stride + kk % S];
// M-major : element (row, kk) at A[kk * row_stride + row]   (S = k, P = 1, slab unused).
struct AView {
    const float* A;
    int64_t S, P, row_stride, slab;
    bool mmajor = false;
};

// B32 != nullptr selects TCEC-SGEMM: B element (l, j) at B32[l * sbk + j * sbn] (FP32), Om unused.
// om_rm: Om is ROW-major (element (l, j) at Om[l * ldo + j]); otherwise column-major (Om[j * ldo + l])
// or, with om_tiled, the k-tiled layout of gen_omega_f16_tiled.
shg_status_t run_shgemm(int64_t m, int64_t n, int64_t k, const AView& av, const uint16_t* Om, int64_t ldo,
                        float* Y, int64_t ldc, const shg_tune_t* tune, void* ws, size_t ws_bytes, int* nonfinite,
                        cudaStream_t stream, const float* B32 = nullptr, int64_t sbk = 0, int64_t sbn = 0,
                        bool om_tiled = false, const OmGen* og = nullptr, bool om_rm = false) {
    const bool tcec = B32 != nullptr;
    if (om_rm && (om_tiled || tcec)) return SHG_ERR_INVALID_VALUE;
    if (om_tiled && tcec) return SHG_ERR_INVALID_VALUE;
    if (m == 0 || n == 0) return SHG_OK;
    if (k == 0) {
        SHG_CUDA(cudaMemset2DAsync(Y, ldc * sizeof(float), 0, n * sizeof(float), m, stream));
        return SHG_OK;
    }
    DevInfo& d = dev_info();
    if (!d.ok) return SHG_ERR_UNSUPPORTED_DEVICE;
    const bool plain = (av.P == 1 && av.S == k);
    // a row-major Omega is copied (transposed) into the workspace first, so its alignment and ldo do not matter
    const bool om_ok = tcec || om_rm || (aligned16(Om) && ldo % 8 == 0);
    const bool fast_ok = aligned16(av.A) && om_ok && (av.row_stride % 4 == 0) && (av.slab % 4 == 0) &&
                         (plain || av.S % 32 == 0) && encode_fn() != nullptr &&
                         k < (int64_t(1) << 31) && av.S < (int64_t(1) << 31) && m < (int64_t(1) << 31);
    Plan pl = make_plan(m, n, k, fast_ok, tune, d.sms, tcec, om_rm, og == nullptr, !av.mmajor);
    if (pl.path < 0) return SHG_ERR_INVALID_VALUE;
    if (pl.path == 1 && tcec) {
        if (!plain) return SHG_ERR_INVALID_VALUE;
        void* own = nullptr;
        uint16_t* H = static_cast<uint16_t*>(ws);
        if (ws && ws_bytes < static_cast<size_t>(pl.ws_bytes)) return SHG_ERR_WORKSPACE;
        if (!ws) {
            SHG_CUDA(cudaMallocAsync(&own, pl.ws_bytes, stream));
            H = static_cast<uint16_t*>(own);
        }
        shg::split_b_kernel<<<grid_for(((k + 31) / 32) * ((pl.noff + 31) / 32) * 256, 256), dim3(32, 8), 0, stream>>>(
            B32, k, n, sbk, sbn, H, pl.ldh, pl.noff);
        const int64_t sa_row = av.mmajor ? 1 : av.row_stride, sa_col = av.mmajor ? av.row_stride : 1;
        shg::tcec_simt_kernel<<<grid_for(m * n, 256), 256, 0, stream>>>(m, n, k, av.A, sa_row, sa_col, H, pl.ldh,
                                                                       pl.noff, Y, ldc);
        g_launches.fetch_add(2, std::memory_order_relaxed);
        const cudaError_t e = cudaGetLastError();
        if (own) cudaFreeAsync(own, stream);
        if (e != cudaSuccess) return cuda_fail(e, "tcec_simt_kernel");
        return SHG_OK;
    }
    if (pl.path == 1) {
        // callers materialise non-plain views first; the CUDA-core fallback reads column-major Omega
        if (!plain || om_tiled) return SHG_ERR_INVALID_VALUE;
        const int64_t sa_row = av.mmajor ? 1 : av.row_stride, sa_col = av.mmajor ? av.row_stride : 1;
        shg::shgemm_simt_kernel<<<grid_for(m * n, 256), 256, 0, stream>>>(
            m, n, k, av.A, sa_row, sa_col, Om, om_rm ? ldo : 1, om_rm ? 1 : ldo, Y, ldc, nonfinite, pl.tf32);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        SHG_CUDA(cudaGetLastError());
        return SHG_OK;
    }
    CUtensorMap mapA, mapB0, mapB1;
    // K-major A stage layout: 256-B row visits (encode_a_rowpair) when rows are >= 2 MiB apart, i.e.
    // every row of a 128-row box sits in its own 2-MiB page (measured on 1024 x 2^20: 1.24 -> 0.79
    // ms); at shorter strides the two-box layout measured 3-15% faster (profiles/r01_ab_abox.jsonl)
    const int a_box = tune ? tune->a_box : 0;     // 0 auto, 1 128-B row visits, 2 256-B row visits
    // the 4-D box spans two 32-k chunks: inside one slab only if S % 64 == 0 (or a plain matrix)
    const bool rowpair_ok = !av.mmajor && av.S % 32 == 0 && (plain || av.S % 64 == 0);
    const bool rowpair = rowpair_ok && (a_box == 2 || (a_box == 0 && av.row_stride * 4 >= (int64_t(2) << 20)));
    if (a_box == 2 && !rowpair_ok) return SHG_ERR_INVALID_VALUE;
    const bool enc_ok = av.mmajor ? encode_a_mmajor(&mapA, av.A, m, k, av.row_stride)
                        : rowpair ? encode_a_rowpair(&mapA, av.A, av.S, m, av.P, av.row_stride, av.slab)
                                  : encode_a(&mapA, av.A, av.S, m, av.P, av.row_stride, av.slab);
    if (!enc_ok) {
        std::snprintf(g_err, sizeof(g_err), "cuTensorMapEncodeTiled(A) failed");
        return SHG_ERR_CUDA;
    }
    // workspace: caller's (checked) or stream-ordered scratch, freed on every exit below
    uint8_t* wsb = nullptr;
    void* own_ws = nullptr;
    if (pl.ws_bytes > 0) {
        if (ws && ws_bytes >= static_cast<size_t>(pl.ws_bytes)) {
            wsb = static_cast<uint8_t*>(ws);
        } else if (ws) {
            return SHG_ERR_WORKSPACE;
        } else {
            SHG_CUDA(cudaMallocAsync(&own_ws, pl.ws_bytes, stream));
            wsb = static_cast<uint8_t*>(own_ws);
        }
    }
    auto finish = [&](shg_status_t st) -> shg_status_t {
        if (own_ws) {
            const cudaError_t e = cudaFreeAsync(own_ws, stream);
            if (st == SHG_OK && e != cudaSuccess) return cuda_fail(e, "cudaFreeAsync");
        }
        return st;
    };
    // Omega operand: FP16 as given (SHGEMM-FP16), or its exact TF32 widening (SHGEMM-TF32),
    // or TCEC-SGEMM's [B_low | dB_low] split of an FP32 B (Eqs 5-9)
    const int rows0 = pl.pair ? (tcec ? r0_for_tcec(pl.bn, true) : r0_for(pl.bn, true, pl.tf32))
                              : (wide_bn(pl.bn) ? r0_for(pl.bn, false, false) : pl.bn);
    const int r1 = tcec ? r1_for_tcec(pl.bn, pl.pair) : r1_for(pl.bn, pl.pair, pl.tf32);
    const int rows1 = r1 > 0 ? r1 : rows0;         // one N part (R1 == 0): mapB1 unused
    bool encb_ok;
    if (tcec) {
        uint16_t* H = reinterpret_cast<uint16_t*>(wsb + up256(pl.sk_bytes));
        shg::split_b_kernel<<<grid_for(((k + 31) / 32) * ((pl.noff + 31) / 32) * 256, 256), dim3(32, 8), 0, stream>>>(
            B32, k, n, sbk, sbn, H, pl.ldh, pl.noff);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        if (cudaGetLastError() != cudaSuccess) return finish(cuda_fail(cudaErrorLaunchFailure, "split_b_kernel"));
        encb_ok = encode_b(&mapB0, H, k, 2 * pl.noff, pl.ldh, rows0) && encode_b(&mapB1, H, k, 2 * pl.noff, pl.ldh, rows1);
    } else if (pl.tf32) {
        float* om32 = reinterpret_cast<float*>(wsb + up256(pl.sk_bytes));
        if (om_tiled) {
            shg::widen_omega_tiled_kernel<<<grid_for((k + 31) / 32 * 32 * n, 256), 256, 0, stream>>>(Om, k, n, om32);
        } else {
            shg::widen_omega_kernel<<<grid_for(k * n, 256), 256, 0, stream>>>(Om, k, n, om_rm ? ldo : 1,
                                                                            om_rm ? 1 : ldo, om32, pl.ldo32);
        }
        g_launches.fetch_add(1, std::memory_order_relaxed);
        if (cudaGetLastError() != cudaSuccess) return finish(cuda_fail(cudaErrorLaunchFailure, "widen_omega_kernel"));
        encb_ok = om_tiled ? encode_b32_tiled(&mapB0, om32, k, n, rows0) && encode_b32_tiled(&mapB1, om32, k, n, rows1)
                           : encode_b32(&mapB0, om32, k, n, pl.ldo32, rows0) &&
                                 encode_b32(&mapB1, om32, k, n, pl.ldo32, rows1);
    } else if (om_tiled) {
        encb_ok = encode_b_tiled(&mapB0, Om, k, n, rows0) && encode_b_tiled(&mapB1, Om, k, n, rows1);
    } else if (om_rm) {
        uint16_t* Ot = reinterpret_cast<uint16_t*>(wsb + up256(pl.sk_bytes));
        const int64_t tiles = ((k + 31) / 32) * ((n + 31) / 32);
        const int sms = std::max(1, d.sms);
        shg::transpose_omega_kernel<<<static_cast<int>(std::min<int64_t>(tiles, int64_t(sms) * 8)), dim3(32, 8), 0,
                                      stream>>>(Om, k, n, ldo, Ot, pl.ldt);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        if (cudaGetLastError() != cudaSuccess) return finish(cuda_fail(cudaErrorLaunchFailure, "transpose_omega_kernel"));
        encb_ok = encode_b(&mapB0, Ot, k, n, pl.ldt, rows0) && encode_b(&mapB1, Ot, k, n, pl.ldt, rows1);
    } else {
        encb_ok = encode_b(&mapB0, Om, k, n, ldo, rows0) && encode_b(&mapB1, Om, k, n, ldo, rows1);
    }
    if (!encb_ok) {
        std::snprintf(g_err, sizeof(g_err), "cuTensorMapEncodeTiled(Omega) failed");
        return finish(SHG_ERR_CUDA);
    }
    shg::KParams kp{};
    kp.m = m; kp.n = n; kp.k = k;
    kp.k_inner = av.S;
    kp.num_kb = pl.num_kb;
    kp.m_tiles = pl.m_tiles; kp.n_tiles = pl.n_tiles; kp.splits = pl.splits;
    kp.a_rowpair = rowpair ? 1 : 0;
    kp.b_lo_col = static_cast<int32_t>(pl.noff);
    kp.om_tiled = om_tiled ? 1 : 0;
    const bool gen = og != nullptr;
    kp.sk = pl.sk ? 1 : 0;
    if (pl.sk) {
        kp.sk_total = static_cast<int64_t>(pl.m_tiles) * pl.n_tiles * pl.num_kb;
        kp.sk_ws = reinterpret_cast<float*>(wsb);
        kp.sk_cnt = reinterpret_cast<uint32_t*>(wsb + pl.sk_planes);
        const cudaError_t e = cudaMemsetAsync(kp.sk_cnt, 0, static_cast<size_t>(pl.sk_bytes - pl.sk_planes), stream);
        if (e != cudaSuccess) return finish(cuda_fail(e, "cudaMemsetAsync(stream-K counters)"));
    }
    if (gen) {   // the caller checked om_gen_ok() on this plan
        if (!om_tiled || pl.pair || pl.tf32 || tcec || pl.n_tiles != 1 || pl.bn > kOmGenMaxBn ||
            static_cast<int64_t>(pl.m_tiles) * pl.splits > pl.grid)
            return finish(SHG_ERR_INVALID_VALUE);
        SHG_CUDA(cudaMemsetAsync(og->flags, 0, static_cast<size_t>(pl.num_kb) * 4, stream));
        kp.om_gen = omgen_mode() == 2 ? 2 : 1;
        kp.om_dist = og->dist;
        kp.om_stream = og->stream_id;
        kp.om_thr = og->thr;
        kp.om_seed = og->seed;
        kp.om_q0 = og->row0 / 4;
        kp.om_buf = const_cast<uint16_t*>(Om);
        kp.om_flags = og->flags;
    }
    kp.dbg = tune ? static_cast<uint32_t>(tune->debug_flags) : 0u;
    kp.prof = tune ? reinterpret_cast<long long*>(tune->prof) : nullptr;
    if (pl.splits > 1) {
        float* wsf = reinterpret_cast<float*>(wsb);
        kp.out = wsf;
        kp.ldo_out = pl.ld_ws;
        kp.split_stride = m * pl.ld_ws;
        kp.vec_store = aligned16(wsf) ? 1 : 0;
        kp.nonfinite = nullptr;
    } else {
        kp.out = Y;
        kp.ldo_out = ldc;
        kp.split_stride = 0;
        kp.vec_store = (aligned16(Y) && ldc % 4 == 0) ? 1 : 0;
        kp.nonfinite = nonfinite;
    }
    shg_status_t st = gen ? dispatch_tc_f16_gen(pl.bn, av.mmajor, mapA, mapB0, mapB1, kp, pl.grid, stream)
                      : tcec      ? dispatch_tc_tcec(pl.bn, av.mmajor, pl.pair, mapA, mapB0, mapB1, kp, pl.grid, stream)
                      : pl.tf32 ? dispatch_tc_tf32(pl.bn, av.mmajor, pl.pair, mapA, mapB0, mapB1, kp, pl.grid, stream)
                      : pl.npa > 1 ? dispatch_tc_f16_amc(pl.bn, pl.npa, mapA, mapB0, mapB1, kp, pl.grid, stream)
                                : dispatch_tc_f16(pl.bn, av.mmajor, pl.pair, mapA, mapB0, mapB1, kp, pl.grid, stream);
    if (st != SHG_OK) return finish(st);
    if (pl.splits > 1) {
        shg::splitk_reduce_kernel<<<grid_for(m * n, 256), 256, 0, stream>>>(kp.out, pl.splits, m, n, pl.ld_ws,
                                                                          kp.split_stride, Y, ldc, nonfinite);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return finish(cuda_fail(e, "splitk_reduce_kernel"));
    }
    return finish(SHG_OK);
}

// In-kernel Omega generation for project(): ON by default since round 2 — with
// dedicated generator warps, the packed-f32x2 generator and the stager's generate-on-timeout fallback
// it is faster than the separate generator launch on cfg3 and does not depend on
// co-residency; shg_set_inkernel_omega(0) or SHG_OMGEN=0 selects the separate generator.
// 2 = tests only: the generator warps stay idle, every tile comes from the stagers' fallback.
std::atomic<int> g_omgen{-1};
int omgen_mode() {
    int v = g_omgen.load(std::memory_order_relaxed);
    if (v < 0) {
        const char* e = std::getenv("SHG_OMGEN");
        v = (e && e[0] == '0') ? 0 : 1;
        g_omgen.store(v, std::memory_order_relaxed);
    }
    return v;
}
bool omgen_enabled() { return omgen_mode() != 0; }

uint32_t sparse_threshold(int dist, int64_t k_total) {
    if (dist == SHG_DIST_SPARSE3) return 715827882u;
    if (dist == SHG_DIST_VERYSPARSE) {
        double t = std::floor(2147483648.0 / std::sqrt(static_cast<double>(k_total)));
        if (t > 2147483648.0) t = 2147483648.0;
        return static_cast<uint32_t>(t);
    }
    return 0u;
}


// ------------------------------------------------------------------ host-streaming support
int64_t host_chunk_rows(int64_t m, int64_t k, int64_t chunk_rows) {
    int64_t r = chunk_rows > 0 ? chunk_rows : (int64_t(256) << 20) / (std::max<int64_t>(k, 1) * 4);
    r = std::max<int64_t>(128, (r + 127) / 128 * 128);
    if (m > 0) r = std::min(r, (m + 127) / 128 * 128);
    return r;
}

// Device workspace of shgemm_host: [column-major copy of a row-major Omega][2 x (A chunk, Y chunk,
// split-K scratch)]. The split-K scratch is sized for EVERY chunk height up to `chunk` (a short last
// chunk has fewer m-tiles, may plan more splits and need more scratch than a full one); heights
// that round up to the same multiple of 128 share the plan's split count and need no more bytes
// than that multiple, so the multiples of 128 cover all heights.
struct HostWs {
    int64_t chunk, lda_s, ldy_s, ldt;
    size_t om_bytes, a_bytes, y_bytes, sk_bytes, total;
};

HostWs host_ws(int64_t m, int64_t n, int64_t k, int64_t chunk_rows, bool om_rm) {
    HostWs w{};
    w.chunk = host_chunk_rows(m, k, chunk_rows);
    w.lda_s = (k + 3) / 4 * 4;
    w.ldy_s = (n + 3) / 4 * 4;
    w.ldt = (k + 7) / 8 * 8;
    auto up = [](size_t b) { return (b + 255) / 256 * 256; };
    w.om_bytes = om_rm ? up(static_cast<size_t>(n * w.ldt * 2)) : 0;
    w.a_bytes = up(static_cast<size_t>(w.chunk * w.lda_s * 4));
    w.y_bytes = up(static_cast<size_t>(w.chunk * w.ldy_s * 4));
    shg_tune_t col{};
    col.omega_layout = SHG_OMEGA_COL_MAJOR;
    size_t sk = 0;
    const int sms = std::max(1, dev_info().sms);
    // split-K scratch only exists while the m-tiles do not fill the SMs (<= sms x 256 rows); past
    // that a height can only plan stream-K, whose planes do not depend on it and whose counters
    // grow with it: bounded by the forced stream-K plan of the full chunk
    const int64_t scan = std::min<int64_t>(w.chunk, int64_t(sms) * 256 + 256);
    for (int64_t rows = 128; rows <= scan; rows += 128)
        sk = std::max(sk, static_cast<size_t>(make_plan(rows, n, k, true, &col, sms).ws_bytes));
    sk = std::max(sk, static_cast<size_t>(make_plan(w.chunk, n, k, true, &col, sms).ws_bytes));
    shg_tune_t col_sk = col;
    col_sk.stream_k = 1;
    const Plan psk = make_plan(w.chunk, n, k, true, &col_sk, sms);
    if (psk.path == 0) sk = std::max(sk, static_cast<size_t>(psk.ws_bytes));
    w.sk_bytes = up(sk);
    w.total = w.om_bytes + 2 * (w.a_bytes + w.y_bytes + w.sk_bytes);
    return w;
}

bool omega_layout_ok(const shg_tune_t* t) {
    return !t || t->omega_layout == SHG_OMEGA_ROW_MAJOR || t->omega_layout == SHG_OMEGA_COL_MAJOR;
}
bool omega_row_major(const shg_tune_t* t) { return !t || t->omega_layout == SHG_OMEGA_ROW_MAJOR; }

}  // namespace

extern "C" {

shg_status_t gen_omega_f16_ex(int64_t k, int64_t n, uint64_t seed, int dist, uint32_t stream_id, int64_t row0,
                              int64_t k_total, uint16_t* Omega, int64_t ldo, int layout, shg_stream_t stream) {
    if (k < 0 || n < 0 || row0 < 0 || dist < 0 || dist > 3) return SHG_ERR_INVALID_VALUE;
    if (layout != SHG_OMEGA_ROW_MAJOR && layout != SHG_OMEGA_COL_MAJOR) return SHG_ERR_INVALID_VALUE;
    if (k == 0 || n == 0) return SHG_OK;
    if (!Omega || ldo < (layout == SHG_OMEGA_ROW_MAJOR ? n : k)) return SHG_ERR_INVALID_VALUE;
    if (dist == SHG_DIST_VERYSPARSE && k_total < 1) return SHG_ERR_INVALID_VALUE;
    const int64_t nq = ((row0 + k - 1) >> 2) - (row0 >> 2) + 1;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (layout == SHG_OMEGA_ROW_MAJOR) {
        const int sms = std::max(1, dev_info().sms);
        const int64_t gx = (n + 31) / 32;
        const int64_t gy = std::max<int64_t>(1, std::min<int64_t>((nq + 7) / 8, (int64_t(sms) * 16 + gx - 1) / gx));
        if (gx > 2147483647 || gy > 65535) return SHG_ERR_INVALID_VALUE;
        shg::omega::gen_omega_rowmajor_kernel<<<dim3(static_cast<unsigned>(gx), static_cast<unsigned>(gy)), dim3(32, 8),
                                                0, s>>>(k, n, seed, stream_id, row0, dist,
                                                        sparse_threshold(dist, k_total), Omega, ldo);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        SHG_CUDA(cudaGetLastError());
        return SHG_OK;
    }
    const bool vec = ((reinterpret_cast<uintptr_t>(Omega) & 7u) == 0) && (ldo % 4 == 0) && (row0 % 4 == 0);
    shg::omega::gen_omega_kernel<<<omega_grid(nq, n), 256, 0, s>>>(k, n, seed, stream_id, row0, dist,
                                                                  sparse_threshold(dist, k_total), Omega, ldo, vec);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    SHG_CUDA(cudaGetLastError());
    return SHG_OK;
}

shg_status_t gen_omega_f16_tiled(int64_t k, int64_t n, uint64_t seed, int dist, uint32_t stream_id, int64_t row0,
                                 int64_t k_total, uint16_t* Omega, shg_stream_t stream) {
    if (k < 0 || n < 0 || row0 < 0 || dist < 0 || dist > 3) return SHG_ERR_INVALID_VALUE;
    if (k == 0 || n == 0) return SHG_OK;
    if (!Omega) return SHG_ERR_INVALID_VALUE;
    if (dist == SHG_DIST_VERYSPARSE && k_total < 1) return SHG_ERR_INVALID_VALUE;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (k % 64) {   // rows k .. 64*ceil(k/64)-1 of the last tile are zero
        SHG_CUDA(cudaMemsetAsync(Omega + (k / 64) * n * 64, 0, static_cast<size_t>(n) * 64 * 2, s));
    }
    const bool vec = ((reinterpret_cast<uintptr_t>(Omega) & 7u) == 0) && (row0 % 4 == 0);
    const int64_t nq = ((row0 + k - 1) >> 2) - (row0 >> 2) + 1;
    shg::omega::gen_omega_kernel<<<omega_grid(nq, n), 256, 0, s>>>(k, n, seed, stream_id, row0, dist,
                                                                  sparse_threshold(dist, k_total), Omega, 0, vec, n);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    SHG_CUDA(cudaGetLastError());
    return SHG_OK;
}

shg_status_t shgemm_tiled(int64_t m, int64_t n, int64_t k, const float* A, int64_t lda, const uint16_t* Omega_tiled,
                          float* Y, int64_t ldc, const shg_tune_t* tune, void* workspace, size_t workspace_bytes,
                          int* nonfinite_flag, shg_stream_t stream) {
    if (m < 0 || n < 0 || k < 0) return SHG_ERR_INVALID_VALUE;
    if (m == 0 || n == 0) return SHG_OK;
    if (!Y || ldc < n) return SHG_ERR_INVALID_VALUE;
    if (k > 0 && (!A || !Omega_tiled || lda < k)) return SHG_ERR_INVALID_VALUE;
    if (tune && ((tune->bn > 0 && !valid_bn(tune->bn)) || (tune->tc != SHG_TC_FP16 && tune->tc != SHG_TC_TF32)))
        return SHG_ERR_INVALID_VALUE;
    AView av{A, k, 1, lda, lda * std::max<int64_t>(m, 1)};
    return run_shgemm(m, n, k, av, Omega_tiled, 8, Y, ldc, tune, workspace, workspace_bytes, nonfinite_flag,
                      reinterpret_cast<cudaStream_t>(stream), nullptr, 0, 0, true);
}

shg_status_t gen_omega_f16(int64_t k, int64_t n, uint64_t seed, int dist, uint16_t* Omega, int64_t ldo,
                           shg_stream_t stream) {
    return gen_omega_f16_ex(k, n, seed, dist, 0u, 0, k, Omega, ldo, SHG_OMEGA_ROW_MAJOR, stream);
}

shg_status_t shgemm_ex(int64_t m, int64_t n, int64_t k, const float* A, int64_t lda, const uint16_t* Omega,
                       int64_t ldo, float* Y, int64_t ldc, const shg_tune_t* tune, void* workspace,
                       size_t workspace_bytes, int* nonfinite_flag, shg_stream_t stream) {
    if (m < 0 || n < 0 || k < 0) return SHG_ERR_INVALID_VALUE;
    if (m == 0 || n == 0) return SHG_OK;
    if (!Y || ldc < n) return SHG_ERR_INVALID_VALUE;
    if (!omega_layout_ok(tune)) return SHG_ERR_INVALID_VALUE;
    const bool om_rm = omega_row_major(tune);
    if (k > 0 && (!A || !Omega || lda < k || ldo < (om_rm ? n : k))) return SHG_ERR_INVALID_VALUE;
    if (tune && tune->bn > 0 && !valid_bn(tune->bn)) return SHG_ERR_INVALID_VALUE;
    if (tune && tune->tc != SHG_TC_FP16 && tune->tc != SHG_TC_TF32) return SHG_ERR_INVALID_VALUE;
    AView av{A, k, 1, lda, lda * std::max<int64_t>(m, 1)};
    return run_shgemm(m, n, k, av, Omega, ldo, Y, ldc, tune, workspace, workspace_bytes, nonfinite_flag,
                      reinterpret_cast<cudaStream_t>(stream), nullptr, 0, 0, false, nullptr, om_rm);
}

shg_status_t shgemm(int64_t m, int64_t n, int64_t k, const float* A, int64_t lda, const uint16_t* Omega,
                    int64_t ldo, float* Y, int64_t ldc, shg_stream_t stream) {
    return shgemm_ex(m, n, k, A, lda, Omega, ldo, Y, ldc, nullptr, nullptr, 0, nullptr, stream);
}

shg_status_t shgemm_tf32(int64_t m, int64_t n, int64_t k, const float* A, int64_t lda, const uint16_t* Omega,
                         int64_t ldo, float* Y, int64_t ldc, shg_stream_t stream) {
    shg_tune_t tt{};
    tt.tc = SHG_TC_TF32;
    return shgemm_ex(m, n, k, A, lda, Omega, ldo, Y, ldc, &tt, nullptr, 0, nullptr, stream);
}

shg_status_t shgemm_at(int64_t m, int64_t n, int64_t k, const float* At, int64_t ldat, const uint16_t* Omega,
                       int64_t ldo, float* Y, int64_t ldc, const shg_tune_t* tune, void* workspace,
                       size_t workspace_bytes, int* nonfinite_flag, shg_stream_t stream) {
    if (m < 0 || n < 0 || k < 0) return SHG_ERR_INVALID_VALUE;
    if (m == 0 || n == 0) return SHG_OK;
    if (!Y || ldc < n) return SHG_ERR_INVALID_VALUE;
    if (!omega_layout_ok(tune)) return SHG_ERR_INVALID_VALUE;
    const bool om_rm = omega_row_major(tune);
    if (k > 0 && (!At || !Omega || ldat < m || ldo < (om_rm ? n : k))) return SHG_ERR_INVALID_VALUE;
    if (tune && tune->bn > 0 && !valid_bn(tune->bn)) return SHG_ERR_INVALID_VALUE;
    if (tune && tune->tc != SHG_TC_FP16 && tune->tc != SHG_TC_TF32) return SHG_ERR_INVALID_VALUE;
    AView av{At, k, 1, ldat, 0, true};
    return run_shgemm(m, n, k, av, Omega, ldo, Y, ldc, tune, workspace, workspace_bytes, nonfinite_flag,
                      reinterpret_cast<cudaStream_t>(stream), nullptr, 0, 0, false, nullptr, om_rm);
}

shg_status_t tcec_sgemm_ex(int64_t m, int64_t n, int64_t k, const float* A, int64_t lda, int a_layout, const float* B,
                           int64_t ldb, int b_layout, float* C, int64_t ldc, const shg_tune_t* tune, void* workspace,
                           size_t workspace_bytes, shg_stream_t stream) {
    if (m < 0 || n < 0 || k < 0) return SHG_ERR_INVALID_VALUE;
    if ((a_layout != SHG_LAYOUT_K_MAJOR && a_layout != SHG_LAYOUT_MN_MAJOR) ||
        (b_layout != SHG_LAYOUT_K_MAJOR && b_layout != SHG_LAYOUT_MN_MAJOR))
        return SHG_ERR_INVALID_VALUE;
    if (m == 0 || n == 0) return SHG_OK;
    if (!C || ldc < n) return SHG_ERR_INVALID_VALUE;
    if (k > 0) {
        if (!A || !B) return SHG_ERR_INVALID_VALUE;
        if (lda < (a_layout == SHG_LAYOUT_K_MAJOR ? k : m)) return SHG_ERR_INVALID_VALUE;
        if (ldb < (b_layout == SHG_LAYOUT_K_MAJOR ? k : n)) return SHG_ERR_INVALID_VALUE;
    }
    if (tune && tune->bn > 0 && !valid_bn(tune->bn)) return SHG_ERR_INVALID_VALUE;
    const AView av = a_layout == SHG_LAYOUT_K_MAJOR ? AView{A, k, 1, lda, lda * std::max<int64_t>(m, 1)}
                                                    : AView{A, k, 1, lda, 0, true};
    const int64_t sbk = b_layout == SHG_LAYOUT_K_MAJOR ? 1 : ldb;
    const int64_t sbn = b_layout == SHG_LAYOUT_K_MAJOR ? ldb : 1;
    return run_shgemm(m, n, k, av, nullptr, 8, C, ldc, tune, workspace, workspace_bytes, nullptr,
                      reinterpret_cast<cudaStream_t>(stream), B ? B : reinterpret_cast<const float*>(C), sbk, sbn);
}

shg_status_t tcec_sgemm(int64_t m, int64_t n, int64_t k, const float* A, int64_t lda, int a_layout, const float* B,
                        int64_t ldb, int b_layout, float* C, int64_t ldc, shg_stream_t stream) {
    return tcec_sgemm_ex(m, n, k, A, lda, a_layout, B, ldb, b_layout, C, ldc, nullptr, nullptr, 0, stream);
}

size_t tcec_sgemm_workspace_size(int64_t m, int64_t n, int64_t k, const shg_tune_t* tune) {
    if (m <= 0 || n <= 0 || k <= 0) return 0;
    const Plan pl = make_plan(m, n, k, true, tune, std::max(1, dev_info().sms), true);
    return pl.path < 0 ? 0 : static_cast<size_t>(pl.ws_bytes);
}

shg_status_t tcec_plan(int64_t m, int64_t n, int64_t k, const shg_tune_t* tune, shg_plan_t* out) {
    if (!out || m < 0 || n < 0 || k < 0) return SHG_ERR_INVALID_VALUE;
    const Plan pl = make_plan(m, n, k, true, tune, std::max(1, dev_info().sms), true);
    if (pl.path < 0) return SHG_ERR_INVALID_VALUE;
    std::memset(out, 0, sizeof(*out));
    out->path = pl.path;
    out->bn = pl.bn; out->n_tiles = pl.n_tiles; out->m_tiles = pl.m_tiles; out->split_k = pl.splits;
    out->grid = pl.grid;
    out->tc = SHG_TC_TCEC;
    if (pl.path == 0) {
        out->stages_a = sa_for_tcec(pl.bn, pl.pair);
        out->stages_b = so_for_tcec(pl.bn, pl.pair);
        out->smem_bytes = smem_for_tcec(pl.bn, pl.pair);
        out->cta_pair = pl.pair ? 1 : 0;
        out->stream_k = pl.sk ? 1 : 0;
        out->omega_mcast = 1;
        out->a_mcast = 1;
        out->kernels = 2 + (pl.splits > 1 ? 1 : 0);
    }
    out->workspace_bytes = pl.ws_bytes;
    return SHG_OK;
}

size_t shg_workspace_size(int64_t m, int64_t n, int64_t k, const shg_tune_t* tune) {
    if (m <= 0 || n <= 0 || k <= 0) return 0;
    const Plan pl = make_plan(m, n, k, true, tune, std::max(1, dev_info().sms), false, omega_row_major(tune));
    return static_cast<size_t>(pl.ws_bytes);
}

shg_status_t shg_plan(int64_t m, int64_t n, int64_t k, const shg_tune_t* tune, shg_plan_t* out) {
    if (!out || m < 0 || n < 0 || k < 0) return SHG_ERR_INVALID_VALUE;
    const int sms = std::max(1, dev_info().sms);
    if (!omega_layout_ok(tune)) return SHG_ERR_INVALID_VALUE;
    const Plan pl = make_plan(m, n, k, true, tune, sms, false, omega_row_major(tune));
    if (pl.path < 0) return SHG_ERR_INVALID_VALUE;
    std::memset(out, 0, sizeof(*out));
    out->path = pl.path;
    out->bn = pl.bn; out->n_tiles = pl.n_tiles; out->m_tiles = pl.m_tiles; out->split_k = pl.splits;
    out->grid = pl.grid;
    if (pl.path == 0) {
        out->stages_a = sa_for(pl.bn, pl.pair, pl.tf32);
        out->stages_b = so_for(pl.bn, pl.pair, pl.tf32);
        out->smem_bytes = smem_for(pl.bn, pl.pair, pl.tf32);
        out->cta_pair = pl.pair ? 1 : 0;
        out->tc = pl.tf32 ? SHG_TC_TF32 : SHG_TC_FP16;
        out->omega_mcast = 1;
        out->stream_k = pl.sk ? 1 : 0;
        out->a_mcast = pl.npa;
        out->kernels = 1 + (pl.splits > 1 ? 1 : 0) + (pl.tf32 || pl.ldt > 0 ? 1 : 0);
    } else {
        out->kernels = pl.path == 1 ? 1 : (k == 0 && m > 0 && n > 0 ? 0 : 0);
    }
    out->workspace_bytes = pl.ws_bytes;
    return SHG_OK;
}

size_t shg_project_workspace_size_ex(int ndim, const int64_t* dims, int mode, int64_t n, int tc) {
    if (ndim < 1 || ndim > 8 || !dims || mode < 0 || mode >= ndim || n <= 0) return 0;
    if (tc != SHG_TC_FP16 && tc != SHG_TC_TF32) return 0;
    int64_t K = 1, P = 1, S = 1;
    for (int i = 0; i < ndim; ++i) {
        if (i != mode) K *= dims[i];
        if (i < mode) P *= dims[i];
        if (i > mode) S *= dims[i];
    }
    const int64_t M = dims[mode];
    // Omega: k-tiled (FP16) or column-major (TF32) — n * round64(K) halves covers both
    size_t bytes = static_cast<size_t>((n * ((K + 63) / 64 * 64) * 2 + 255) / 256 * 256);
    bytes += static_cast<size_t>(up256((K + 63) / 64 * 4));       // in-kernel generation flags
    const bool needs_copy = !(mode == 0 || S == 1 || S % 32 == 0);
    if (needs_copy) bytes += static_cast<size_t>((M * ((K + 3) / 4 * 4) * 4 + 255) / 256 * 256);
    shg_tune_t tt{};
    tt.tc = tc;
    bytes += shg_workspace_size(M, n, K, &tt);
    return bytes;
}

size_t shg_project_workspace_size(int ndim, const int64_t* dims, int mode, int64_t n) {
    return shg_project_workspace_size_ex(ndim, dims, mode, n, SHG_TC_FP16);
}

namespace {
// project_shard's body; om_given != nullptr: Omega_(mode) supplied by the caller in the k-tiled
// layout (project_omega), no generation
shg_status_t project_impl(const float* A, int ndim, const int64_t* dims, int mode, int64_t n, uint64_t seed,
                          int dist, int tc, int64_t omega_row0, int64_t k_total, float* W, int64_t ldw,
                          void* workspace, size_t workspace_bytes, shg_stream_t stream, const uint16_t* om_given) {
    if (!A || !dims || !W || ndim < 1 || ndim > 8 || mode < 0 || mode >= ndim || n < 0 || ldw < n)
        return SHG_ERR_INVALID_VALUE;
    if (omega_row0 < 0) return SHG_ERR_INVALID_VALUE;
    if (dist < 0 || dist > 3 || (tc != SHG_TC_FP16 && tc != SHG_TC_TF32)) return SHG_ERR_INVALID_VALUE;
    for (int i = 0; i < ndim; ++i) if (dims[i] < 1) return SHG_ERR_INVALID_VALUE;
    if (n == 0) return SHG_OK;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int64_t K = 1, P = 1, S = 1;
    for (int i = 0; i < ndim; ++i) {
        if (i != mode) K *= dims[i];
        if (i < mode) P *= dims[i];
        if (i > mode) S *= dims[i];
    }
    const int64_t M = dims[mode];
    const size_t need = shg_project_workspace_size_ex(ndim, dims, mode, n, tc);
    void* own = nullptr;
    uint8_t* ws = static_cast<uint8_t*>(workspace);
    if (!ws) {
        SHG_CUDA(cudaMallocAsync(&own, need, s));
        ws = static_cast<uint8_t*>(own);
    } else if (workspace_bytes < need) {
        return SHG_ERR_WORKSPACE;
    }
    const int64_t ldo = (K + 7) / 8 * 8;
    uint16_t* Om = reinterpret_cast<uint16_t*>(ws);
    size_t off = static_cast<size_t>((n * ((K + 63) / 64 * 64) * 2 + 255) / 256 * 256);
    uint32_t* gen_flags = reinterpret_cast<uint32_t*>(ws + off);
    off += static_cast<size_t>(up256((K + 63) / 64 * 4));
    // SHGEMM-FP16 streams Omega in the k-tiled layout: an unfolding's K reaches 2^20 (cfg3), where
    // each column-major 64-k box would visit n rows 2 MiB apart (measured: the Omega stream, not A,
    // bounded mode 0 at 0.90 ms; 0.69 ms without it)
    bool om_tiled = false;   // decided below, once the A view is known
    auto finish = [&](shg_status_t st) -> shg_status_t {
        if (own) {
            const cudaError_t e = cudaFreeAsync(own, s);
            if (st == SHG_OK && e != cudaSuccess) return cuda_fail(e, "cudaFreeAsync");
        }
        return st;
    };
    if (k_total < 1) k_total = omega_row0 + K;
    if (k_total < omega_row0 + K) return finish(SHG_ERR_INVALID_VALUE);
    AView av{A, K, 1, K, K * M};
    if (mode == 0) {
        av = AView{A, K, 1, K, K * M};
    } else if (S % 32 == 0) {
        // A[p][r][s] -> unfold[r][p*S + s]: 3-D view {S, M, P}, row stride S, slab stride M*S
        av = AView{A, S, P, S, M * S};
    } else if (S == 1) {
        // last mode: unfold[r][c] = A[c * M + r], i.e. the M-major view of a (K x M) row-major
        // matrix — read in place by the M-major stager (no transpose copy)
        av = AView{A, K, 1, M, 0, true};
    } else {
        // middle mode with S % 64 != 0: materialise the unfolding slab by slab (S-wide row blocks)
        float* T = reinterpret_cast<float*>(ws + off);
        const int64_t ldt = (K + 3) / 4 * 4;
        off += static_cast<size_t>((M * ldt * 4 + 255) / 256 * 256);
        for (int64_t p = 0; p < P; ++p) {
            const cudaError_t e = cudaMemcpy2DAsync(T + p * S, ldt * 4, A + p * M * S, S * 4, S * 4, M,
                                                    cudaMemcpyDeviceToDevice, s);
            if (e != cudaSuccess) return finish(cuda_fail(e, "cudaMemcpy2DAsync"));
        }
        av = AView{T, K, 1, ldt, ldt * M};
    }
    // the tcgen05 path will run (same predicate as run_shgemm's fast path) -> k-tiled Omega
    const bool plain_view = (av.P == 1 && av.S == K);
    om_tiled = aligned16(av.A) && av.row_stride % 4 == 0 && av.slab % 4 == 0 &&
               (plain_view || av.S % 32 == 0);
    shg_tune_t tt{};
    tt.tc = tc;
    // By default (shg_set_inkernel_omega) Omega is generated INSIDE the projection kernel when every
    // tile of the plan fits the grid at once (one tile per CTA) and the tiles are single CTAs of
    // BN <= 128: the m_tiles CTAs that share a k range each generate 1/m_tiles of its Omega tiles
    // with their generator warps (no separate gen_omega launch, no Omega traffic before the GEMM);
    // a stager whose tile is late generates it itself (acquire_or_generate), so residency is a
    // performance condition, not a correctness one
    bool om_gen = false;
    if (om_tiled && tc == SHG_TC_FP16 && omega_row0 % 4 == 0 && omgen_enabled()) {
        const Plan pl = make_plan(M, n, K, true, &tt, std::max(1, dev_info().sms), false, false, false);
        om_gen = pl.path == 0 && !pl.pair && pl.n_tiles == 1 && pl.bn <= kOmGenMaxBn &&
                 static_cast<int64_t>(pl.m_tiles) * pl.splits <= pl.grid;
    }
    shg_status_t st = SHG_OK;
    if (om_given) {                  // caller's k-tiled Omega: the tcgen05 path must read it
        if (!om_tiled) return finish(SHG_ERR_INVALID_VALUE);
        om_gen = false;
        Om = const_cast<uint16_t*>(om_given);
    } else if (!om_gen) {
        st = om_tiled ? gen_omega_f16_tiled(K, n, seed, dist, static_cast<uint32_t>(mode), omega_row0, k_total, Om,
                                            stream)
                      : gen_omega_f16_ex(K, n, seed, dist, static_cast<uint32_t>(mode), omega_row0, k_total, Om,
                                         ldo, SHG_OMEGA_COL_MAJOR, stream);
        if (st != SHG_OK) return finish(st);
    } else if (dist == SHG_DIST_VERYSPARSE && k_total < 1) {
        return finish(SHG_ERR_INVALID_VALUE);
    }
    const OmGen og{seed, static_cast<uint32_t>(mode), dist, sparse_threshold(dist, k_total), omega_row0, gen_flags};
    void* sk = ws + off;
    const size_t sk_bytes = need - off;
    st = run_shgemm(M, n, K, av, Om, ldo, W, ldw, &tt, sk_bytes ? sk : nullptr, sk_bytes, nullptr, s, nullptr, 0, 0,
                    om_tiled, om_gen ? &og : nullptr);
    return finish(st);
}
}  // namespace

shg_status_t project_shard(const float* A, int ndim, const int64_t* dims, int mode, int64_t n, uint64_t seed,
                           int dist, int tc, int64_t omega_row0, int64_t k_total, float* W, int64_t ldw,
                           void* workspace, size_t workspace_bytes, shg_stream_t stream) {
    return project_impl(A, ndim, dims, mode, n, seed, dist, tc, omega_row0, k_total, W, ldw, workspace,
                        workspace_bytes, stream, nullptr);
}

shg_status_t project_omega(const float* A, int ndim, const int64_t* dims, int mode, int64_t n,
                           const uint16_t* Omega_tiled, float* W, int64_t ldw, void* workspace, size_t workspace_bytes,
                           shg_stream_t stream) {
    if (!Omega_tiled) return SHG_ERR_INVALID_VALUE;
    return project_impl(A, ndim, dims, mode, n, 0, SHG_DIST_GAUSSIAN, SHG_TC_FP16, 0, 0, W, ldw, workspace,
                        workspace_bytes, stream, Omega_tiled);
}

shg_status_t project_ex(const float* A, int ndim, const int64_t* dims, int mode, int64_t n, uint64_t seed, int dist,
                        int tc, float* W, int64_t ldw, void* workspace, size_t workspace_bytes, shg_stream_t stream) {
    return project_shard(A, ndim, dims, mode, n, seed, dist, tc, 0, 0, W, ldw, workspace, workspace_bytes, stream);
}

shg_status_t project(const float* A, int ndim, const int64_t* dims, int mode, int64_t n, uint64_t seed, int dist,
                     float* W, int64_t ldw, void* workspace, size_t workspace_bytes, shg_stream_t stream) {
    return project_ex(A, ndim, dims, mode, n, seed, dist, SHG_TC_FP16, W, ldw, workspace, workspace_bytes, stream);
}

size_t shg_host_workspace_size(int64_t n, int64_t k, int64_t chunk_rows, int omega_layout) {
    if (n <= 0 || k <= 0) return 0;
    if (omega_layout != SHG_OMEGA_ROW_MAJOR && omega_layout != SHG_OMEGA_COL_MAJOR) return 0;
    return host_ws(0, n, k, chunk_rows, omega_layout == SHG_OMEGA_ROW_MAJOR).total;
}

shg_status_t shgemm_host(int64_t m, int64_t n, int64_t k, const float* A_host, int64_t lda, const uint16_t* Omega,
                         int64_t ldo, int omega_layout, float* Y_host, int64_t ldc, int64_t chunk_rows,
                         void* workspace, size_t workspace_bytes, shg_stream_t stream) {
    if (m < 0 || n < 0 || k < 0 || chunk_rows < 0) return SHG_ERR_INVALID_VALUE;
    if (omega_layout != SHG_OMEGA_ROW_MAJOR && omega_layout != SHG_OMEGA_COL_MAJOR) return SHG_ERR_INVALID_VALUE;
    const bool om_rm = omega_layout == SHG_OMEGA_ROW_MAJOR;
    if (m == 0 || n == 0) return SHG_OK;
    if (!Y_host || ldc < n || (k > 0 && (!A_host || !Omega || lda < k || ldo < (om_rm ? n : k))))
        return SHG_ERR_INVALID_VALUE;
    cudaStream_t us = reinterpret_cast<cudaStream_t>(stream);
    if (k == 0) {
        for (int64_t i = 0; i < m; ++i) std::memset(Y_host + i * ldc, 0, n * sizeof(float));
        return SHG_OK;
    }
    const HostWs w = host_ws(m, n, k, chunk_rows, om_rm);
    if (workspace && workspace_bytes < w.total) return SHG_ERR_WORKSPACE;
    // per-call side streams and events: concurrent calls (other threads, other user streams) share no
    // library state, so one call's record/wait can never order another call's work
    cudaStream_t side[2] = {nullptr, nullptr};
    cudaEvent_t ev_start = nullptr, ev_done[2] = {nullptr, nullptr};
    void* own = nullptr;
    bool joined = false;
    // every exit after the first enqueue goes through here: the user stream waits for whatever the
    // side streams have enqueued (so no copy into the workspace or the caller's buffers is still in
    // flight once the caller synchronises `stream`), owned scratch is freed on `stream`, and the
    // streams / events are released (destroying them with work pending is legal; the work completes)
    auto cleanup = [&](shg_status_t st) -> shg_status_t {
        for (int b = 0; b < 2; ++b) {
            if (side[b] && ev_done[b] && !joined) {
                if (cudaEventRecord(ev_done[b], side[b]) == cudaSuccess) cudaStreamWaitEvent(us, ev_done[b], 0);
            }
        }
        joined = true;
        if (own) {
            const cudaError_t e = cudaFreeAsync(own, us);
            if (st == SHG_OK && e != cudaSuccess) st = cuda_fail(e, "cudaFreeAsync");
        }
        for (int b = 0; b < 2; ++b) {
            if (side[b]) cudaStreamDestroy(side[b]);
            if (ev_done[b]) cudaEventDestroy(ev_done[b]);
        }
        if (ev_start) cudaEventDestroy(ev_start);
        return st;
    };
    auto fail = [&](cudaError_t e, const char* what) { return cleanup(cuda_fail(e, what)); };
    cudaError_t e = cudaSuccess;
    for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
        e = cudaStreamCreateWithFlags(&side[b], cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_done[b], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming);
    if (e != cudaSuccess) return fail(e, "shgemm_host stream/event creation");
    uint8_t* ws = static_cast<uint8_t*>(workspace);
    if (!ws) {
        e = cudaMallocAsync(&own, w.total, us);
        if (e != cudaSuccess) return fail(e, "cudaMallocAsync");
        ws = static_cast<uint8_t*>(own);
    }
    // a row-major Omega is transposed ONCE into the column-major layout the chunks stream
    const uint16_t* Om = Omega;
    int64_t ldo_c = ldo;
    if (om_rm) {
        uint16_t* Ot = reinterpret_cast<uint16_t*>(ws);
        const int64_t tiles = ((k + 31) / 32) * ((n + 31) / 32);
        shg::transpose_omega_kernel<<<static_cast<int>(std::min<int64_t>(tiles, int64_t(std::max(1, dev_info().sms)) * 8)),
                                      dim3(32, 8), 0, us>>>(Omega, k, n, ldo, Ot, w.ldt);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        e = cudaGetLastError();
        if (e != cudaSuccess) return fail(e, "transpose_omega_kernel");
        Om = Ot;
        ldo_c = w.ldt;
    }
    if ((e = cudaEventRecord(ev_start, us)) != cudaSuccess) return fail(e, "cudaEventRecord");
    for (int b = 0; b < 2; ++b)
        if ((e = cudaStreamWaitEvent(side[b], ev_start, 0)) != cudaSuccess) return fail(e, "cudaStreamWaitEvent");
    shg_tune_t col{};
    col.omega_layout = SHG_OMEGA_COL_MAJOR;
    const int64_t nchunks = (m + w.chunk - 1) / w.chunk;
    for (int64_t c = 0; c < nchunks; ++c) {
        const int b = static_cast<int>(c & 1);
        cudaStream_t s = side[b];
        uint8_t* base = ws + w.om_bytes + b * (w.a_bytes + w.y_bytes + w.sk_bytes);
        float* As = reinterpret_cast<float*>(base);
        float* Ys = reinterpret_cast<float*>(base + w.a_bytes);
        void* sk = w.sk_bytes ? base + w.a_bytes + w.y_bytes : nullptr;
        const int64_t r0 = c * w.chunk;
        const int64_t rows = std::min(w.chunk, m - r0);
        e = cudaMemcpy2DAsync(As, w.lda_s * 4, A_host + r0 * lda, lda * 4, k * 4, rows, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return fail(e, "cudaMemcpy2DAsync(H2D)");
        const shg_status_t st = shgemm_ex(rows, n, k, As, w.lda_s, Om, ldo_c, Ys, w.ldy_s, &col, sk, w.sk_bytes,
                                          nullptr, reinterpret_cast<shg_stream_t>(s));
        if (st != SHG_OK) return cleanup(st);
        e = cudaMemcpy2DAsync(Y_host + r0 * ldc, ldc * 4, Ys, w.ldy_s * 4, n * 4, rows, cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) return fail(e, "cudaMemcpy2DAsync(D2H)");
    }
    return cleanup(SHG_OK);
}

shg_status_t shg_probe_tma_read(const float* A, int64_t m, int64_t k, int64_t lda, int layout, int box_k,
                                int box_rows, int splits, int grid, unsigned long long* bytes_out,
                                shg_stream_t stream) {
    if (!A || !bytes_out || m < 128 || k < 32 || lda < k || layout < 0 || layout > 2 || box_rows < 1 ||
        box_rows > 128 || 128 % box_rows || box_k < 1 || splits < 1 || grid < 1)
        return SHG_ERR_INVALID_VALUE;
    if (static_cast<int64_t>(box_k) * box_rows * 4 > shg::kProbeStageBytes) return SHG_ERR_INVALID_VALUE;
    if ((layout != 0 && (box_k % 32)) || (layout == 0 && (box_k > 256 || box_k % 4)) || (layout == 1 && box_k != 32))
        return SHG_ERR_INVALID_VALUE;
    if (layout == 2 && (box_k / 32 > 256 || k % 32)) return SHG_ERR_INVALID_VALUE;
    EncodeFn fn = encode_fn();
    if (!fn) return SHG_ERR_CUDA;
    CUtensorMap map;
    CUresult r;
    if (layout == 2) {
        cuuint64_t dims[3] = {32, static_cast<cuuint64_t>(k / 32), static_cast<cuuint64_t>(m)};
        cuuint64_t strides[2] = {128, static_cast<cuuint64_t>(lda) * 4};
        cuuint32_t box[3] = {32, static_cast<cuuint32_t>(box_k / 32), static_cast<cuuint32_t>(box_rows)};
        cuuint32_t estr[3] = {1, 1, 1};
        r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(A), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(m)};
        cuuint64_t strides[1] = {static_cast<cuuint64_t>(lda) * 4};
        cuuint32_t box[2] = {static_cast<cuuint32_t>(box_k), static_cast<cuuint32_t>(box_rows)};
        cuuint32_t estr[2] = {1, 1};
        r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(A), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, layout == 1 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) return SHG_ERR_INVALID_VALUE;
    const int smem = shg::kProbeStages * shg::kProbeStageBytes + 1024 + 64;
    SHG_CUDA(cudaFuncSetAttribute(shg::probe_tma_read_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int m_tiles = static_cast<int>(m / 128);
    const int num_ks = static_cast<int>(k / box_k);
    shg::probe_tma_read_kernel<<<grid, 32, smem, reinterpret_cast<cudaStream_t>(stream)>>>(
        map, layout, box_k, box_rows, m_tiles, splits, num_ks, bytes_out);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    SHG_CUDA(cudaGetLastError());
    return SHG_OK;
}

shg_status_t shg_debug_split(const float* a, int64_t count, uint16_t* hi, uint16_t* lo, shg_stream_t stream) {
    if (count < 0 || (count > 0 && (!a || !hi || !lo))) return SHG_ERR_INVALID_VALUE;
    if (count == 0) return SHG_OK;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    shg::debug_split_kernel<<<grid_for((count + 1) / 2, 256), 256, 0, s>>>(a, count, hi, lo);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    SHG_CUDA(cudaGetLastError());
    return SHG_OK;
}

shg_status_t shg_debug_split_tf32(const float* a, int64_t count, uint32_t* hi, uint32_t* lo, shg_stream_t stream) {
    if (count < 0 || (count > 0 && (!a || !hi || !lo))) return SHG_ERR_INVALID_VALUE;
    if (count == 0) return SHG_OK;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    shg::debug_split_tf32_kernel<<<grid_for((count + 1) / 2, 256), 256, 0, s>>>(a, count, hi, lo);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    SHG_CUDA(cudaGetLastError());
    return SHG_OK;
}

shg_status_t shg_synth_f32(int kind, uint64_t seed, uint32_t stream_id, int64_t m, int64_t k, int64_t row0,
                           float* A, int64_t lda, shg_stream_t stream) {
    if (kind < 0 || kind > 1 || m < 0 || k < 0 || row0 < 0) return SHG_ERR_INVALID_VALUE;
    if (m == 0 || k == 0) return SHG_OK;
    if (!A || lda < k) return SHG_ERR_INVALID_VALUE;
    const bool vec = aligned16(A) && (lda % 4 == 0);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int64_t work = ((k + 3) / 4) * m;
    shg::omega::synth_f32_kernel<<<grid_for(work, 256), 256, 0, s>>>(kind, seed, stream_id, m, k, row0, A, lda, vec);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    SHG_CUDA(cudaGetLastError());
    return SHG_OK;
}

uint64_t shg_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

const char* shg_last_error(void) { return g_err; }

int shg_device_supported(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return 0;
    return dev_info().ok ? 1 : 0;
}

void shg_set_inkernel_omega(int on) { g_omgen.store(on == 2 ? 2 : (on ? 1 : 0), std::memory_order_relaxed); }
int shg_get_inkernel_omega(void) { return omgen_mode(); }

int shg_set_a_mcast(int npa) {
    if (npa != 0 && npa != 1 && npa != 2 && npa != 4) return -1;
    return g_amc_default.exchange(npa, std::memory_order_relaxed);
}

const char* shg_version(void) { return "shgemm-b200 0.2.0 sm_100a"; }

}  // extern "C"

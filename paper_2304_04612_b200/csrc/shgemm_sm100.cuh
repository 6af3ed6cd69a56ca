// shgemm_sm100.cuh — the SHGEMM mainloop for B200 (sm_100a): Y = A_F32 . Omega_F16.
//
// Paper: Eqs 14-17 split each FP32 element of A into FP16 hi/lo and run
// hi.Omega and lo.Omega on the tensor cores; the hi product's accumulation is moved onto the
// FP32 RN units to avoid the tensor cores' RZ accumulation.
// The A100 design (WMMA, RN add after every f_k = 8 mma) is prior art, not the
// blueprint; this kernel re-derives it for tcgen05:
//
//  * A stager   : TMA streams 128 x 64 FP32 tiles (K-major: 3-D map, or M-major: 2-D map) into an
//                 SA-deep smem ring (SWIZZLE_128B).
//  * Splitter   : 8 warps (2 per TMEM lane quarter, one per 32-k half) read their rows of the FP32
//                 tile (conflict-free shared loads through the swizzle), apply split2 (Eqs 14-15)
//                 with packed f32x2 arithmetic, and write hi and lo straight into TENSOR MEMORY with
//                 tcgen05.st — the MMA takes A from TMEM, so hi/lo never touch shared memory.
//  * Omega      : TMA streams the 64-k Omega tiles (K-major SW128) of a chunk into smem.
//  * Chunks     : K_c = 128 = 2 stages; a chunk slot = 2 TMEM A stages + 2 Omega smem stages, with
//                 ONE ready barrier (splitter arrivals + the Omega TMA bytes) and ONE empty barrier
//                 (tcgen05.commit) — every mbarrier wait costs ~90 cycles on the MMA thread.
//  * MMA        : one thread issues, per chunk and per N-part (H0 + H1 = BN columns), 8 lo MMAs
//                 (D := sum lo.Omega) then 8 hi MMAs, the first with scale-input-d = 11
//                 (D := hi.Omega + D * 2^-11), so D holds hi.Omega + 2^-11 lo.Omega (Eq 16) for
//                 the chunk. Part accumulators rotate through NSLOT TMEM slots.
//  * Promotion  : 8 epilogue warps (4 lane quarters x 2 column halves) tcgen05.ld each finished D and
//                 add it with RN (add.rn.f32x2) into register accumulators: the RZ-avoidance of
//                 PAPER.md:587 applied per K_c = 128 chunk (and to lo as well: reading R2).
//  * Epilogue   : after the last chunk, the RN accumulators are written to Y (row-major) with
//                 128-bit stores, masked on ragged edges; split-K tiles write to a workspace plane
//                 that splitk_reduce_kernel sums in fixed order.
//  * PAIR       : optional CTA pair (cluster of 2, tcgen05.mma.cta_group::2, M = 256): each CTA
//                 splits its own 128 rows and holds HALF of every Omega part tile, the leader issues
//                 the MMAs for both — Omega's L2->SMEM traffic per SM halves (measured: Omega
//                 traffic costs ~1/3 of the clock under the 1000 W power cap).
//
// One CTA (or CTA pair) per SM (pair), persistent over tiles (m-block, k-split, n-block), n fastest.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include "omega.cuh"
#include "ptx.cuh"
#include "split.cuh"

namespace shg {

constexpr int kBM = 128;                          // rows per CTA (UMMA M per CTA)
constexpr int kBK = 64;                           // k per stage: one 128-B swizzle row of FP16
constexpr int kA32StageBytes = kBM * kBK * 4;     // 32 KB
constexpr int kNumSplitWarps = 8;                 // warps 0..7
constexpr int kEpiWarp0 = 8;                      // warps 8..15
constexpr int kWarpProdA = 16, kWarpMMA = 17, kWarpProdB = 18;   // warp 19 idle
constexpr int kThreads = 640;
// OMGEN kernels (in-kernel Omega) add 8 generator warps (20..27): 896 threads, 72 registers each at
// launch; the roles then take splitter 256 x 56 + epilogue 256 x 104 + control 128 x 32 + generator
// 256 x 72 = 63488 of the 64512 (BN <= kOmGenMaxBnKernel keeps the epilogue's accumulators in 104)
constexpr int kThreadsGen = 896;
constexpr int kWarpGen0 = 20;
constexpr int kOmGenMaxBnKernel = 128;
template <bool OMGEN> constexpr int threads_for() { return OMGEN ? kThreadsGen : kThreads; }
// Register budget: setmaxnreg moves registers inside the CTA's own pool (640 threads x 96 = 61440):
// splitter 256 x 56 + epilogue 256 x 168 + control 128 x 32 = 61440.
constexpr int kSmemLimit = 232448;                // max dynamic smem per block on sm_100
constexpr int kTmemCols = 512;
constexpr uint32_t kPeerBitMask = 0xFEFFFFFFu;    // shared::cluster address of the even CTA's copy

struct KParams {
    int64_t m, n, k;
    int64_t k_inner;        // S: contiguous k run of the A view (k for a plain matrix)
    int32_t num_kb;         // ceil(k / 64)
    int32_t m_tiles, n_tiles, splits;   // m_tiles counts 128-row (single) or 256-row (pair) tiles
    int32_t a_rowpair;      // K-major A stage layout: 0 = two boxes {32 k, 128 rows} (k-half major,
                            // 128 B fetched per row visit), 1 = one 4-D box {32, 2, 128 rows, 1}
                            // (row major, 256 B per row visit; needs k_inner % 32 == 0)
    float* out;             // Y, or the split-K workspace when splits > 1
    int64_t ldo_out;        // leading dimension of out (elements)
    int64_t split_stride;   // elements between split planes (workspace)
    int32_t vec_store;      // out rows 16-B aligned and ldo_out % 4 == 0
    int32_t b_lo_col;       // TCEC: column (n) coordinate of dB_low in the B tensor maps (B_low at 0)
    int32_t om_tiled;       // Omega in the k-tiled layout (3-D maps {64, n_pad, k/64}; SHGEMM-FP16 only)
    // Cooperative in-kernel Omega (om_gen = 1; single CTAs, one tile per CTA, n_tiles == 1): the
    // generator warps (20..27) of the CTA (m_blk, s) generate the k-tiles t of split s with
    // (t - first tile of s) % m_tiles == m_blk into om_buf (k-tiled layout) and release flag[t];
    // the Omega stager acquires flag[t] before its TMA. Every tile is generated once, by one of the
    // m_tiles CTAs that read it — or, if that CTA has not published it within kOmGenHelpNs (it may
    // not be resident yet), by the waiting stager itself (same bits), so no CTA's progress depends
    // on another CTA being resident. om_gen = 2 (tests): the generator warps stay idle and every
    // tile takes that fallback.
    int32_t om_gen;
    int32_t om_dist;
    uint32_t om_stream, om_thr;
    uint64_t om_seed;
    int64_t om_q0;          // Philox block of local row 0 (global row / 4; rows are 4-aligned)
    uint16_t* om_buf;
    uint32_t* om_flags;
    int* nonfinite;         // optional flag (set to 1 on any non-finite output)
    // Stream-K schedule (sk = 1; splits == 1): T = m_tiles * n_tiles * num_kb k-block iterations cut
    // into gridDim/CL equal ranges (next_piece); partial pieces publish their sums in sk_ws
    // (2 slots per unit x CTAs per unit x BN x 128 floats) and count them in sk_cnt (one zeroed
    // uint32 per tile and CTA of the unit); the last piece of a tile sums the slots in k order.
    int32_t sk;
    int64_t sk_total;
    float* sk_ws;
    uint32_t* sk_cnt;
    uint32_t dbg;           // diagnostics: bit0 skip promotion loads, bit1 skip split math, bit2 skip MMAs,
                            //              bit3 skip the Omega TMA, bit4 Omega TMA always loads k-tile 0
                            //              (same transfers, constant B data), bit5 A TMA always loads
                            //              k-block 0 of its rows (L2 hits, no HBM stream)
                            //              (results are wrong when dbg != 0)
    long long* prof;        // diagnostics: per-CTA wait-cycle counters [gridDim.x][16] (ProfSlot)
};

// Per-CTA diagnostic counters (cycles unless noted), written only when KParams::prof != nullptr.
enum ProfSlot {
    kProfTotal = 0, kProfMmaAccEmpty, kProfMmaHlFull, kProfMmaOmFull, kProfSplitAFull, kProfSplitBEmpty,
    kProfEpiAccFull, kProfProdAEmpty, kProfProdBEmpty, kProfSplitBusy, kProfEpiStore, kProfStages, kProfSlots = 16
};

// Every pipeline wait is bounded: a wait that spins ~2^22 times (seconds) traps, so a deadlock
// becomes a launch error instead of a hung GPU. Building with -DSHG_WATCHDOG_PRINT also reports
// which barrier (smem offset), parity, CTA and warp stalled (a printf call costs registers).
__device__ __forceinline__ void watchdog_report(uint64_t* bar, uint32_t parity) {
#ifdef SHG_WATCHDOG_PRINT
    printf("shgemm watchdog: block %d warp %d lane %d stuck on mbarrier smem+0x%x parity %u\n", blockIdx.x,
           threadIdx.x / 32, threadIdx.x % 32, smem_u32(bar), parity);
#else
    (void)bar;
    (void)parity;
#endif
    asm volatile("trap;");
}

// try_wait with cluster-scope acquire (barriers that receive arrivals from the peer CTA)
__device__ __forceinline__ bool mbar_try_wait_cluster(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}\n"
        : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    return ok != 0;
}

// CLUSTER selects acquire.cluster. The pair path does NOT use it: its remote arrivals are relaxed
// (they carry no data) and acquire.cluster emits CCTL.IVALL (an L1 invalidate) on every success.
template <bool CLUSTER = false>
__device__ __forceinline__ void mbar_wait_prof(uint64_t* bar, uint32_t parity, long long& acc) {
    const long long t0 = clock64();
    uint32_t spins = 0;
    while (!(CLUSTER ? mbar_try_wait_cluster(bar, parity) : mbar_try_wait(bar, parity))) {
        if (++spins == (1u << 22)) watchdog_report(bar, parity);
    }
    acc += clock64() - t0;
}

// arrive on the copy of `bar` (a local smem address) in CTA `cta` of the cluster. RELAXED, because
// these arrivals publish no generic-proxy memory, only the completion of the arriving thread's own
// tensor-memory accesses, and that completion is established by blocking waits BEFORE the arrive:
//  (1) ch_ready (follower splitter -> leader MMA): the follower's tcgen05.st of hi/lo into its TMEM
//      are followed by tcgen05.wait::st, which does not return until every prior tcgen05.st of the
//      thread has completed (the values are in TMEM); then tcgen05.fence::before_thread_sync orders
//      those tcgen05 ops before the arrive, the arrive can only execute after the wait returned, the
//      leader's try_wait observes the phase it completes, and tcgen05.fence::after_thread_sync keeps
//      the leader's tcgen05.mma (which reads the follower's TMEM half) from being issued before that
//      observation. Causality runs st-complete -> arrive -> phase flip -> wait returns -> MMA issue.
//  (2) acc_empty (follower epilogue -> leader MMA): tcgen05.ld of the accumulator, then
//      tcgen05.wait::ld (the values are in registers) -> fence::before_thread_sync -> arrive; the
//      leader's next MMA into that slot is issued after its wait + fence::after_thread_sync, so the
//      overwrite cannot reach the slot before the reads completed (write-after-read).
// Neither handoff carries data through shared or global memory, so no release/acquire is needed
// for visibility; a .release.cluster arrive would emit MEMBAR.ALL.GPU (measured ~1000 cycles per
// handoff on the MMA thread's critical path). The Omega TMA bytes (complete_tx on the leader's
// barrier) and the MMA completions (tcgen05.commit multicast) are hardware arrivals that fire only
// after their data has landed / their operand reads have finished. (compute-sanitizer racecheck
// does not model TMEM; this argument plus the bitwise parity suite are the evidence.)
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, uint32_t cta) {
    asm volatile(
        "{\n\t.reg .b32 ra;\n\t"
        "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
        "mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [ra];\n\t}\n"
        ::"r"(smem_u32(bar)), "r"(cta) : "memory");
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// TF32 = false: SHGEMM-FP16 (kind::f16, hi/lo packed 2 per 32-bit TMEM column, Omega FP16 in smem).
// TF32 = true : SHGEMM-TF32 (kind::tf32, one hi or lo element per TMEM column,
//               Omega as TF32 (the exactly widened FP16 values) in smem, two 128-B k-halves a stage).
// TCEC = true: TCEC-SGEMM (Eqs 5-9; NEXT-2): A split in-kernel exactly as for
//               SHGEMM-FP16; B (FP32) pre-split into FP16 B_low / dB_low, whose tiles sit side by
//               side in each Omega smem stage (NB = 2); per chunk the MMA issuer accumulates
//               dA_low.B_low + A_low.dB_low, then folds it under A_low.B_low with scale-input-d = 11.
template <int BN, bool PAIR, bool TF32 = false, bool TCEC = false>
struct Cfg {
    // FP16: K_c = 128, one promotion chunk = 2 stages of 64 k; TMEM: 4 A stages (2 chunks of hi/lo,
    // 64 columns each) + accumulator slots. TF32: a stage's hi/lo take 128 columns, so K_c = 64 =
    // one stage and 2 chunk slots. N is covered by 2 part-MMAs of widths W + WLAST = BN so that the
    // drain of one part overlaps the MMAs of the other.
    // WIDE (SHGEMM-FP16, 256 < BN <= 288): one N tile covers n = 257..288 (e.g. RSVD's p + s = 272)
    // so A streams once; two accumulator parts of up to 144 columns leave 192 TMEM columns for A,
    // hence K_c = 64 (one stage per chunk) and 3 chunk slots.
    static constexpr bool WIDE = BN > 256;
    static constexpr int KC = (TF32 || WIDE) ? 1 : 2;      // stages per promotion chunk
    static constexpr int AST = TF32 ? 128 : 64;            // TMEM columns per A stage (hi, then lo)
    static constexpr int EB = TF32 ? 4 : 2;                // Omega bytes per element in smem
    static constexpr int KSTEP = TF32 ? 8 : 16;            // UMMA K per instruction
    static constexpr int NMMA = kBK / KSTEP;               // MMAs per stage per operand (hi or lo)
    // chunk slots (TMEM A + Omega smem); TF32 with BN <= 64 has the TMEM for a third (the ring is
    // only one stage deep per slot there, and the splitter must not wait on the MMAs every stage)
    static constexpr int NCH = ((TF32 && BN <= 64) || WIDE) ? 3 : 2;
    // N parts: 2 (drain of one overlaps the MMAs of the other), or 1 for TF32 with BN <= 64, whose
    // MMA thread is issue-bound (8 K steps a stage: half the instructions with one part of N = BN)
    static constexpr int NQ = (TF32 && BN <= 64) ? 1 : 2;
    static constexpr int W = NQ == 1 ? BN : ((BN / 2) + 15) / 16 * 16;    // width of part 0
    static constexpr int WLAST = NQ == 1 ? BN : BN - W;                     // width of the last part
    static constexpr int SB = NCH * KC;                    // TMEM A stage slots
    static constexpr int ABASE = kTmemCols - SB * AST;
    static constexpr int NSLOT_fit = ABASE / W;
    static constexpr int NSLOT_MAX = TF32 ? 8 : 4;             // TF32 chunks are half as long: more slack
    static constexpr int NSLOT = NSLOT_fit > NSLOT_MAX ? NSLOT_MAX : NSLOT_fit;
    static constexpr int SO = NCH * KC;                    // Omega smem stages
    static constexpr int R0 = PAIR ? W / 2 : W;            // Omega rows of part 0 held by this CTA
    static constexpr int R1 = NQ == 1 ? 0 : (PAIR ? WLAST / 2 : WLAST);   // ... of part 1
    static constexpr int NB = TCEC ? 2 : 1;                // B tiles per stage (TCEC: B_low, then dB_low)
    static constexpr int kOmTileBytes = (R0 + R1) * kBK * EB;   // TF32: [k-half][R0 + R1 rows][128 B]
    static constexpr int kOmStageBytes = NB * kOmTileBytes;
    static constexpr int kTileM = PAIR ? 2 * kBM : kBM;   // rows per (pair) tile
    static constexpr int kBarBytes = 512;
    static constexpr int SA_fit = (kSmemLimit - 1024 - kBarBytes - SO * kOmStageBytes) / kA32StageBytes;
    static constexpr int SA = SA_fit > 6 ? 6 : SA_fit;
    static constexpr int kSmemBytes = 1024 + SA * kA32StageBytes + SO * kOmStageBytes + kBarBytes;
    static_assert(BN % 16 == 0 && BN >= 32 && BN <= (TF32 ? 256 : 288) && (!TCEC || !WIDE || PAIR), "BN");
    static_assert(WLAST >= 16 && WLAST % 16 == 0 && (W <= 128 || NQ == 1 || (WIDE && W <= 144)), "UMMA N parts");
    static_assert(!PAIR || (R0 % 8 == 0 && R1 % 8 == 0), "pair halves must be whole 8-row core groups");
    static_assert(NSLOT >= NQ, "TMEM accumulator slots");
    static_assert(SA >= 2 && kSmemBytes <= kSmemLimit, "smem");
    static_assert(!(TF32 && TCEC), "TCEC-SGEMM is instantiated for FP16 tensor cores only");
};

// ------------------------------------------------------------------ work schedule
// A CTA (pair) = one work unit of `units` = gridDim.x / CL; every role of the CTA walks the same
// sequence of pieces, each a contiguous k-block range [kb0, kb0 + nkb) of one output tile.
//  * Tiles (KParams::sk == 0): tiles (m-block, k-split, n-block), n fastest, are dealt round robin
//    (tile = unit + it * units); split s covers k-blocks [s*num_kb/S, (s+1)*num_kb/S) (an interleaved
//    assignment, k-block s + it*S, was measured slower on 4-MB-strided rows).
//  * Stream-K (sk == 1): the T = tiles * num_kb k-block iterations, tile-major, are cut into `units`
//    equal contiguous ranges [u*T/U, (u+1)*T/U), so every SM pair gets the same work (no partly idle
//    last wave: 64 pair tiles of RSVD's projection on 74 pairs would otherwise leave 14% of the
//    tensor cores idle). A range covers the tail of one tile, whole tiles, and the head of another;
//    the pieces of a tile that one unit does not cover completely are PARTIAL and are summed by the
//    epilogue of whichever of them finishes last (sk_fixup), in fixed k order.
struct Piece {
    int m_blk, n_blk, s;
    int kb0, nkb;      // global first k-block, k-block count
    int64_t tile;      // output tile (m_blk * n_tiles + n_blk) (stream-K)
    int slot;          // stream-K partial-plane slot (2 per unit: its first / last piece), -1 = whole tile
};

// This unit's stream-K range [g0, g1) of k-block iterations and its first tile, computed once per CTA
// (64-bit divisions stay out of the roles' loops: the control warps run with 32 registers)
struct SkRange {
    int64_t g0, g1, t0;
};

__device__ __forceinline__ SkRange sk_range(const KParams& p, int unit, int units) {
    SkRange r{0, 0, 0};
    if (p.sk) {
        r.g0 = static_cast<int64_t>(unit) * p.sk_total / units;
        r.g1 = static_cast<int64_t>(unit + 1) * p.sk_total / units;
        r.t0 = r.g0 / p.num_kb;
    }
    return r;
}

// NPA > 1 (A multicast, see the kernel): a unit is a cluster of NPA pairs that take one m-block and
// NPA consecutive N tiles together (the planner guarantees n_tiles % NPA == 0); pair pr of the
// cluster gets N tile ng * NPA + pr of the unit's N group ng.
template <int NPA = 1>
__device__ __forceinline__ bool next_piece(const KParams& p, int unit, int units, const SkRange& sr, int it,
                                           Piece& w, int pr = 0) {
    if (!p.sk) {
        const int tile = unit + it * units;
        const int ngr = NPA == 1 ? p.n_tiles : p.n_tiles / NPA;
        if (tile >= p.m_tiles * p.splits * ngr) return false;
        const int per_m = p.splits * ngr;
        w.m_blk = tile / per_m;
        const int rem = tile - w.m_blk * per_m;
        w.s = rem / ngr;
        w.n_blk = NPA == 1 ? rem - w.s * ngr : (rem - w.s * ngr) * NPA + pr;
        w.kb0 = static_cast<int>((static_cast<int64_t>(w.s) * p.num_kb) / p.splits);
        w.nkb = static_cast<int>((static_cast<int64_t>(w.s + 1) * p.num_kb) / p.splits) - w.kb0;
        w.tile = tile;
        w.slot = -1;
        return true;
    }
    // stream-K (the planner guarantees n_tiles == 1 and splits == 1): tile = m-block
    const int64_t K = p.num_kb;
    const int64_t tau = sr.t0 + it;
    const int64_t lo = tau * K > sr.g0 ? tau * K : sr.g0, hi = (tau + 1) * K < sr.g1 ? (tau + 1) * K : sr.g1;
    if (lo >= hi) return false;
    w.tile = tau;
    w.m_blk = static_cast<int>(tau);
    w.n_blk = 0;
    w.s = 0;
    w.kb0 = static_cast<int>(lo - tau * K);
    w.nkb = static_cast<int>(hi - lo);
    w.slot = (w.kb0 == 0 && w.nkb == K) ? -1 : 2 * unit + (it == 0 ? 0 : 1);
    return true;
}

// stream-K: the unit whose range holds k-block iteration x (the largest u with u*T/U <= x)
__device__ __forceinline__ int sk_unit_of(int64_t x, int64_t T, int units) {
    return static_cast<int>(((x + 1) * units - 1) / T);
}

__device__ __forceinline__ void advance(uint32_t& stage, uint32_t& phase, uint32_t n) {
    if (++stage == n) { stage = 0; phase ^= 1u; }
}

// D[tmem] (+)= A[tmem] * B[smem]  (A operand from tensor memory, "TS" form), 1 CTA or CTA pair,
// kind::f16 (SHGEMM-FP16) or kind::tf32 (SHGEMM-TF32)
#define SHG_MMA_TS(GROUP, KIND)                                                                  \
    asm volatile("{\n\t.reg .pred p;\n\t"                                                     \
                 "setp.ne.b32 p, %4, 0;\n\t"                                                     \
                 "tcgen05.mma.cta_group::" GROUP ".kind::" KIND " [%0], [%1], %2, %3, p;\n\t}\n"  \
                 ::"r"(tmem_d), "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory")
#define SHG_MMA_TS_SCALE11(GROUP, KIND)                                                             \
    asm volatile("{\n\t.reg .pred p;\n\t"                                                        \
                 "setp.ne.b32 p, 1, 0;\n\t"                                                         \
                 "tcgen05.mma.cta_group::" GROUP ".kind::" KIND " [%0], [%1], %2, %3, p, 11;\n\t}\n" \
                 ::"r"(tmem_d), "r"(tmem_a), "l"(bdesc), "r"(idesc) : "memory")

template <bool PAIR, bool TF32>
__device__ __forceinline__ void mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
    if constexpr (PAIR && TF32) SHG_MMA_TS("2", "tf32");
    else if constexpr (PAIR) SHG_MMA_TS("2", "f16");
    else if constexpr (TF32) SHG_MMA_TS("1", "tf32");
    else SHG_MMA_TS("1", "f16");
}

// D[tmem] = A[tmem] * B[smem] + D * 2^-11  (scale-input-d = 11, sm_100a)
template <bool PAIR, bool TF32>
__device__ __forceinline__ void mma_ts_scale11(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc) {
    if constexpr (PAIR && TF32) SHG_MMA_TS_SCALE11("2", "tf32");
    else if constexpr (PAIR) SHG_MMA_TS_SCALE11("2", "f16");
    else if constexpr (TF32) SHG_MMA_TS_SCALE11("1", "tf32");
    else SHG_MMA_TS_SCALE11("1", "f16");
}

// completion of this thread's prior tcgen05 ops -> one arrive on `bar` in every CTA of `mask`
// (a pair: its two CTAs; an Omega-multicast cluster: all CTAs for the chunk-slot release)
template <bool PAIR>
__device__ __forceinline__ void commit_to(uint64_t* bar, uint16_t mask = 3) {
    if constexpr (PAIR) {
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
            ::"r"(smem_u32(bar)), "h"(mask) : "memory");
    } else {
        tc_commit(bar);
    }
}

// Omega tile load; in a pair the transaction bytes land on the leader's (even CTA's) barrier.
// tiled: Omega in the k-tiled layout (KParams::om_tiled), a 3-D map {64, n, k/64}: the box of a
// 64-k stage is one contiguous run of rows x 128 B instead of one 128-B visit per column.
template <bool PAIR, bool TF32 = false>
__device__ __forceinline__ void tma_load_omega(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                               int32_t c1, uint64_t policy, bool tiled = false) {
    if (tiled) {   // FP16: 64-k tiles; TF32 (the exact FP32 widening): 32-k tiles
        const int32_t t0 = TF32 ? (c0 & 31) : (c0 & 63), t2 = TF32 ? (c0 >> 5) : (c0 >> 6);
        if constexpr (PAIR) {
            asm volatile(
                "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                " [%0], [%1, {%3, %4, %5}], [%2], %6;"
                ::"r"(smem_u32(smem_dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & kPeerBitMask),
                  "r"(t0), "r"(c1), "r"(t2), "l"(policy)
                : "memory");
        } else {
            tma_load_3d(smem_dst, map, bar, t0, c1, t2, policy);
        }
        return;
    }
    if constexpr (PAIR) {
        asm volatile(
            "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
            " [%0], [%1, {%3, %4}], [%2], %5;"
            ::"r"(smem_u32(smem_dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & kPeerBitMask),
              "r"(c0), "r"(c1), "l"(policy)
            : "memory");
    } else {
        tma_load_2d(smem_dst, map, bar, c0, c1, policy);
    }
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
        ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
          "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// (a, b) += (c, d) with one add.rn.f32x2 (IEEE RN per lane; FADD2 on sm_100)
__device__ __forceinline__ void add2_rn(float& a, float& b, float c, float d) {
    asm("{\n\t.reg .b64 x, y;\n\t"
        "mov.b64 x, {%0, %1};\n\t"
        "mov.b64 y, {%2, %3};\n\t"
        "add.rn.f32x2 x, x, y;\n\t"
        "mov.b64 {%0, %1}, x;\n\t}\n"
        : "+f"(a), "+f"(b)
        : "f"(c), "f"(d));
}

// RN promotion adds: packed add.rn.f32x2 (FADD2) by default; -DSHG_EPI_SCALAR for add.rn.f32.
#ifdef SHG_EPI_SCALAR
#define ADD_PAIR(a, b, c, d) do { (a) = __fadd_rn((a), (c)); (b) = __fadd_rn((b), (d)); } while (0)
#else
#define ADD_PAIR(a, b, c, d) add2_rn((a), (b), (c), (d))
#endif

// ------------------------------------------------------------------ cooperative Omega (om_gen)

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
__device__ __forceinline__ void gen_bar() { asm volatile("bar.sync 2, 256;" ::: "memory"); }

// 64-k tile t of the k-tiled Omega (rows 64t..64t+63 of this operand, all n columns) by the 256
// generator threads (tid 0..255): OMEGA_SPEC blocks q = om_q0 + 16t + ql; rows >= k written as 0.
__device__ __forceinline__ void gen_omega_tile(const KParams& p, int64_t t, int tid, int nthr = 256) {
    const omega::Keys keys = omega::philox_keys(p.om_seed);
    uint16_t* tile = p.om_buf + t * p.n * 64;
    const int nb = 16 * static_cast<int>(p.n);
    for (int b = tid; b < nb; b += nthr) {
        const int ql = b & 15;
        const int64_t j = b >> 4;
        const int64_t r0 = t * 64 + 4 * ql;
        uint2 v = make_uint2(0u, 0u);
        if (r0 < p.k) {
            v = omega::omega4p(keys, p.om_stream, p.om_dist, p.om_thr, static_cast<uint64_t>(p.om_q0 + t * 16 + ql),
                               static_cast<uint32_t>(j));
            if (r0 + 3 >= p.k) {          // rows >= k of the last tile are +0
                if (r0 + 1 >= p.k) v.x &= 0xFFFFu;
                if (r0 + 2 >= p.k) v.y = 0u;
                else v.y &= 0xFFFFu;
            }
        }
        *reinterpret_cast<uint2*>(tile + j * 64 + 4 * ql) = v;
    }
    // the tile is read by other CTAs' TMA (async proxy): order these generic writes before the release
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ void release_flag(uint32_t* f) {
    __threadfence();
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(1u) : "memory");
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// The Omega stager's wait for k-tile t (one thread). Normally the tile's generator CTA publishes it
// within microseconds; if the flag is still clear after kOmGenHelpNs, that CTA may not be resident
// (another kernel holds its SM, e.g. a second in-kernel-Omega projection on another stream whose
// stagers wait in turn), so this thread generates the tile itself — the same bits, written to the
// same place (a concurrent write by the generator CTA stores identical values) — and publishes it.
// No CTA then waits on another being scheduled: the kernel completes whatever else runs.
constexpr uint64_t kOmGenHelpNs = 200000;
static __device__ unsigned long long g_om_helped;   // tiles generated by the fallback (tests read it)
__device__ __forceinline__ void acquire_or_generate(const KParams& p, int64_t t) {
    const uint32_t* f = p.om_flags + t;
    uint64_t t0 = 0;
    for (uint32_t spins = 0;; ++spins) {
        uint32_t v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if (v != 0) break;
        if ((spins & 63u) == 0) {
            const uint64_t now = globaltimer_ns();
            if (t0 == 0) {
                t0 = now;
            } else if (now - t0 > kOmGenHelpNs) {
                gen_omega_tile(p, t, 0, 1);           // ends with fence.proxy.async.global
                release_flag(p.om_flags + t);
                atomicAdd(&g_om_helped, 1ull);
                break;
            }
        }
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// MMAJOR = false: A is K-major (row-major m x k, or a 3-D K-major view of an unfolding); each stage
//                 is two TMA boxes of 32 k x 128 rows.
// MMAJOR = true : A is M-major (element (i, l) at A[l * lda + i], e.g. the last-mode unfolding of a
//                 C-order tensor); each stage is ONE unswizzled TMA box of 128 rows x 64 k (512 B per
//                 k-line: the former four 32-row SW128 boxes fetched 128 B per visit of lines up to
//                 4 MB apart), and the splitter gathers its row's k values with conflict-free 32-bit
//                 loads (a warp's 32 rows are one 128-B run) — no transpose copy.
// PAIR          : CTA pair (launch with cluster dims (2,1,1)); see the header comment.
// TF32          : SHGEMM-TF32 (Cfg's header); mapB0/B1 then describe the FP32 (TF32) copy of Omega.
// TCEC          : TCEC-SGEMM (Cfg's header): two B tiles per stage, three MMA groups per chunk.
// OMGEN         : cooperative in-kernel Omega (KParams::om_gen; single CTAs, SHGEMM-FP16, k-tiled Omega,
//                 one tile per CTA): compiled only into the instantiations project() uses for it, so
//                 the other kernels' epilogues carry no generator registers.
// NPA > 1       : A multicast (SHGEMM-FP16 K-major CTA pairs, several N tiles): a cluster of NPA pairs
//                 (2 * NPA CTAs) takes one m-block and NPA N tiles, one per pair. Each A stage is
//                 fetched ONCE per cluster and row half: the even pair's CTA of that half (the issuer)
//                 multicasts it into the same ring slot of the NPA CTAs holding those rows, which
//                 split it locally. A peer's stager arms its own a_full for the bytes and then
//                 arrives on the issuer's a_empty, so the issuer's a_empty phase of a slot's use u
//                 completes only when every destination has consumed use u and armed use u + 1 (the
//                 issuer waits for NPA - 1 such arrivals besides its own 8 splitter warps). A comes from L2/HBM once instead of NPA times
//                 (the A100 design loads A mnk/b_n times).
template <int BN, bool MMAJOR, bool PAIR, bool TF32 = false, bool TCEC = false, bool OMGEN = false, int NPA = 1>
__global__ void __launch_bounds__(threads_for<OMGEN>(), 1)
shgemm_sm100_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB0,
                    const __grid_constant__ CUtensorMap mapB1, const KParams p) {
    using CF = Cfg<BN, PAIR, TF32, TCEC>;
    constexpr int SA = CF::SA, NQ = CF::NQ, W = CF::W, WLAST = CF::WLAST;
    constexpr int NSLOT = CF::NSLOT, ABASE = CF::ABASE;
    // epilogue mapping (below): both groups drain half of every part for wide tiles and for one-part
    // tiles (TF32 BN <= 64, where group 1 would otherwise idle); else one part per group
    constexpr bool SPLITH = CF::WIDE || NQ == 1;
    constexpr int kOm = CF::kOmStageBytes;
    constexpr int NCH = CF::NCH, KC = CF::KC;
    constexpr int SO = CF::SO;
    constexpr int AST = CF::AST, NMMA = CF::NMMA;

    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t* base = smem_raw + ((1024u - (raw_addr & 1023u)) & 1023u);
    uint8_t* a32 = base;
    uint8_t* om = a32 + SA * kA32StageBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(om + SO * kOm);
    uint64_t* a_full = bars;                 // TMA A landed                        (count 1 + tx)
    uint64_t* a_empty = a_full + SA;         // splitters done reading              (count 8)
    uint64_t* ch_ready = a_empty + SA;       // chunk hi/lo in TMEM + Omega in smem (leader: count 8|16 + 1|2 + tx)
    uint64_t* ch_empty = ch_ready + NCH;     // MMAs done with the chunk slot       (tcgen05.commit)
    uint64_t* acc_full = ch_empty + NCH;     // D slot complete                     (tcgen05.commit)
    uint64_t* acc_empty = acc_full + NSLOT;  // D slot drained                      (leader: 4|8 warps, SPLITH 8|16)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + NSLOT);
    uint32_t* sk_flag = tmem_slot + 1;       // stream-K: "this CTA sums the tile" (epilogue broadcast)

    const uint32_t warp = warp_id();
    const uint32_t lane = threadIdx.x & 31u;
    static_assert(!OMGEN || (!PAIR && !TF32 && !TCEC && BN <= kOmGenMaxBnKernel), "in-kernel Omega: single-CTA SHGEMM-FP16");
    static_assert(NPA == 1 || (PAIR && !MMAJOR && !TF32 && !TCEC && !OMGEN && !CF::WIDE), "A multicast: FP16 K-major pairs");
    constexpr int CL = PAIR ? 2 * NPA : 1;                        // CTAs per cluster
    const uint32_t crk = PAIR ? cluster_ctarank() : 0u;
    const uint32_t crank = crk & 1u;                              // rank in the pair: 0 = leader (issues the MMAs)
    const int pr = static_cast<int>(crk >> 1);                    // pair of the cluster (NPA > 1)
    const uint32_t lead = 2u * static_cast<uint32_t>(pr);         // cluster rank of the pair's leader
    const uint16_t pair_mask = static_cast<uint16_t>(3u << lead);
    const int unit = static_cast<int>(blockIdx.x) / CL;           // this CTA's (pair's / cluster's) work unit
    const int units = static_cast<int>(gridDim.x) / CL;
    const SkRange sr = sk_range(p, unit, units);
    constexpr int kPair = PAIR ? 2 : 1;
    const bool a_issuer = NPA == 1 || pr == 0;

    if (threadIdx.x == 0) {
        for (int i = 0; i < SA; ++i) {
            mbar_init(&a_full[i], 1);
            mbar_init(&a_empty[i], kNumSplitWarps + ((NPA > 1 && a_issuer) ? NPA - 1 : 0));
        }
        for (int i = 0; i < NCH; ++i) {
            mbar_init(&ch_ready[i], kPair * (kNumSplitWarps + 1));
            mbar_init(&ch_empty[i], 1);
        }
        for (int i = 0; i < NSLOT; ++i) { mbar_init(&acc_full[i], 1); mbar_init(&acc_empty[i], (SPLITH ? 8 : 4) * kPair); }
        fence_mbar_init();
    }
    if (warp == kWarpProdA && lane == 0) {
        tma_prefetch_desc(&mapA);
        tma_prefetch_desc(&mapB0);
        tma_prefetch_desc(&mapB1);
    }
    if (warp == kWarpMMA) {
        if constexpr (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                         ::"r"(smem_u32(tmem_slot)), "n"(kTmemCols) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        } else {
            tmem_alloc<kTmemCols>(tmem_slot);
        }
    }
    tc_fence_before();
    if constexpr (PAIR) cluster_sync_all(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const long long t_kernel0 = clock64();

    if (warp < kNumSplitWarps) {
        // ============================================================ splitter (Eqs 14-15) -> TMEM
        asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
        const int q = static_cast<int>(warp & 3u);        // TMEM lane quarter = rows 32q..32q+31
        const int kh = static_cast<int>(warp >> 2);       // k half of the stage: 32kh .. 32kh+31
        const int r = 32 * q + static_cast<int>(lane);    // tile row (of this CTA) owned by this thread
        // this thread's 128-B line of the stage and its SW128 XOR term (line index & 7)
        const int a_line = p.a_rowpair ? 2 * r + kh : kh * kBM + r;
        const int rx = a_line & 7;
        const uint32_t lane_addr = static_cast<uint32_t>(32 * q) << 16;
        uint32_t sa = 0, pa = 0, cs = 0, pc = 0;
        long long w_a = 0, w_b = 0, stages = 0;
        const long long t_begin = clock64();
        const bool skip_math = (p.dbg & 2u) != 0;
        Piece wk;
        for (int it = 0; next_piece<NPA>(p, unit, units, sr, it, wk, pr); ++it) {
            const int m_blk = wk.m_blk, n_blk = wk.n_blk, kb0 = 0, kb1 = wk.nkb;
            (void)m_blk;
            (void)n_blk;
            for (int kb = kb0; kb < kb1; kb += KC) {
                const int nst = (kb1 - kb) < KC ? (kb1 - kb) : KC;
#pragma unroll
                for (int t = 0; t < KC; ++t) {
                    if (t < nst) {
                        ++stages;
                        // (1) read and split this thread's 32 k of its row (overlaps the MMAs that
                        //     still use the chunk slot about to be overwritten)
                        mbar_wait_prof(&a_full[sa], pa, w_a);
                        if constexpr (TF32) {
                            // 32 k of this row -> 64 TMEM words (32 hi + 32 lo): two rounds of 16 k,
                            // each stored before the next is read (56-register budget); the wait for
                            // the chunk slot sits after the first round's split, which it overlaps
                            const uint32_t col = tmem_base + lane_addr + ABASE + (cs * KC + t) * AST + kh * 32;
#pragma unroll
                            for (int rd = 0; rd < 2; ++rd) {
                                uint32_t hi[16], lo[16];
                                if (!skip_math) {
                                    if constexpr (MMAJOR) {
                                        // unswizzled [64 k][128 rows] stage: this thread's row r at
                                        // word r of every 512-B k-line (a warp reads one 128-B run)
                                        const float* colp = reinterpret_cast<const float*>(a32 + sa * kA32StageBytes) + r;
#pragma unroll
                                        for (int i = 0; i < 8; ++i) {
                                            const int k0 = 32 * kh + 16 * rd + 2 * i;
                                            split_tf32_x2(colp[k0 * kBM], colp[(k0 + 1) * kBM], hi[2 * i], hi[2 * i + 1],
                                                          lo[2 * i], lo[2 * i + 1]);
                                        }
                                    } else {
                                        const uint8_t* src = a32 + sa * kA32StageBytes + a_line * 128;
#pragma unroll
                                        for (int c = 0; c < 2; ++c) {
                                            const int pc0 = 4 * rd + 2 * c;
                                            const float4 x0 = *reinterpret_cast<const float4*>(src + ((pc0 ^ rx) * 16));
                                            const float4 x1 = *reinterpret_cast<const float4*>(src + (((pc0 + 1) ^ rx) * 16));
                                            split_tf32_x2(x0.x, x0.y, hi[8 * c + 0], hi[8 * c + 1], lo[8 * c + 0], lo[8 * c + 1]);
                                            split_tf32_x2(x0.z, x0.w, hi[8 * c + 2], hi[8 * c + 3], lo[8 * c + 2], lo[8 * c + 3]);
                                            split_tf32_x2(x1.x, x1.y, hi[8 * c + 4], hi[8 * c + 5], lo[8 * c + 4], lo[8 * c + 5]);
                                            split_tf32_x2(x1.z, x1.w, hi[8 * c + 6], hi[8 * c + 7], lo[8 * c + 6], lo[8 * c + 7]);
                                        }
                                    }
                                }
                                if (rd == 0 && t == 0) {
                                    mbar_wait_prof(&ch_empty[cs], pc ^ 1u, w_b);
                                    tc_fence_after();
                                }
                                if (!skip_math) {
                                    tmem_st16(col + 16 * rd, hi);
                                    tmem_st16(col + 64 + 16 * rd, lo);
                                }
                            }
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&a_empty[sa]);
                            advance(sa, pa, SA);
                        } else {
                        uint32_t hi[16], lo[16];
                        if (!skip_math && MMAJOR) {
                            // unswizzled [64 k][128 rows] stage (one TMA box, 512 B per k-line):
                            // this thread's row r is word r of every k-line; a warp's 32 rows are
                            // one conflict-free 128-B run
                            const float* colp = reinterpret_cast<const float*>(a32 + sa * kA32StageBytes) + r;
#pragma unroll
                            for (int i = 0; i < 16; ++i) {       // k pairs 32kh + 2i, +1
                                const int k0 = 32 * kh + 2 * i;
                                split2_x2(colp[k0 * kBM], colp[(k0 + 1) * kBM], hi[i], lo[i]);
                            }
                        } else if (!skip_math) {
                            const uint8_t* src = a32 + sa * kA32StageBytes + a_line * 128;
#pragma unroll
                            for (int c = 0; c < 4; ++c) {        // 8 k per chunk of the row
                                const float4 x0 = *reinterpret_cast<const float4*>(src + (((2 * c) ^ rx) * 16));
                                const float4 x1 = *reinterpret_cast<const float4*>(src + (((2 * c + 1) ^ rx) * 16));
                                split2_x2(x0.x, x0.y, hi[4 * c + 0], lo[4 * c + 0]);
                                split2_x2(x0.z, x0.w, hi[4 * c + 1], lo[4 * c + 1]);
                                split2_x2(x1.x, x1.y, hi[4 * c + 2], lo[4 * c + 2]);
                                split2_x2(x1.z, x1.w, hi[4 * c + 3], lo[4 * c + 3]);
                            }
                        }
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&a_empty[sa]);
                        advance(sa, pa, SA);
                        // (2) hand hi/lo to the tensor cores through TMEM
                        if (t == 0) {
                            mbar_wait_prof(&ch_empty[cs], pc ^ 1u, w_b);
                            tc_fence_after();
                        }
                        if (!skip_math) {
                            const uint32_t col = tmem_base + lane_addr + ABASE + (cs * KC + t) * AST + kh * 16;
                            tmem_st16(col, hi);
                            tmem_st16(col + 32, lo);
                        }
                        }   // FP16
                    }
                }
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if constexpr (PAIR) mbar_arrive_cluster(&ch_ready[cs], lead);
                    else mbar_arrive(&ch_ready[cs]);
                }
                advance(cs, pc, NCH);
            }
        }
        if (p.prof && threadIdx.x == 0) {
            long long* pr = p.prof + blockIdx.x * kProfSlots;
            pr[kProfSplitAFull] = w_a;
            pr[kProfSplitBEmpty] = w_b;
            pr[kProfSplitBusy] = clock64() - t_begin - w_a - w_b;
            pr[kProfStages] = stages;
        }
    } else if (warp < kEpiWarp0 + 8) {
        // ============================================================ RN promotion + epilogue
        // SPLITH (wide tiles): each N part's accumulator is drained by BOTH epilogue groups, group h
        // taking the h-th half of its columns, so a part's slot is released after half the per-warp
        // TMEM loads (the next stage's MMAs wait on it; K_c = 64 there). Otherwise group h drains
        // all of part h, which overlaps the other part's MMAs (measured 2.7% faster at BN = 256).
        if constexpr (OMGEN) asm volatile("setmaxnreg.inc.sync.aligned.u32 104;");
        else asm volatile("setmaxnreg.inc.sync.aligned.u32 168;");
        const int q = static_cast<int>(warp & 3u);                       // TMEM lane quarter (warp_id % 4)
        const int h = static_cast<int>((warp - kEpiWarp0) >> 2);         // epilogue group
        const uint32_t lane_addr = static_cast<uint32_t>(32 * q) << 16;
        // per group: the column span of each part it drains (HP0: part 0 / all but the last,
        // HPL: the last part) and its accumulator count
        constexpr int HP0 = SPLITH ? W / 2 : W, HPL = SPLITH ? WLAST / 2 : WLAST;
        constexpr int NACC = SPLITH ? HP0 + (NQ > 1 ? HPL : 0) : W;
        static_assert(HP0 % 8 == 0 && HPL % 8 == 0, "drained spans must be whole tcgen05.ld x8 groups");
        // parts drained by this group: SPLITH all of them (its half of each), else part h only
        auto mine = [&](int part) { return SPLITH || part == h; };
        uint32_t stage = 0;
        uint32_t e_use0 = 0, e_use1 = 0;   // WIDE: drains per accumulator slot (= part)
        long long w_full = 0, t_store = 0;
        const bool skip_ld = (p.dbg & 1u) != 0;
        const int etid = static_cast<int>(threadIdx.x) - kEpiWarp0 * 32;   // 0..255
        Piece wk;
        for (int it = 0; next_piece<NPA>(p, unit, units, sr, it, wk, pr); ++it) {
            const int m_blk = wk.m_blk, n_blk = wk.n_blk, kb0 = 0, kb1 = wk.nkb;
            (void)m_blk;
            (void)n_blk;
            float acc[NACC];
#pragma unroll
            for (int i = 0; i < NACC; ++i) acc[i] = 0.0f;
            for (int kb = kb0; kb < kb1; kb += CF::KC, ++stage) {   // one promotion per K_c chunk
#pragma unroll
                for (int part = 0; part < NQ; ++part) {
                    if (!mine(part)) continue;
                    // WIDE: part q is promoted on stages with (local stage + q) odd and on the
                    // piece's last stage, in the same pairing as the MMA issuer's
                    if (CF::WIDE && !((((kb - kb0) + part) & 1) == 1 || kb + 1 == kb1)) continue;
                    const int hw = (part == NQ - 1) ? HPL : HP0;       // this group's columns of the part
                    const int aoff = SPLITH ? part * HP0 : 0;
                    const uint32_t g = stage * NQ + part;
                    const uint32_t slot = CF::WIDE ? static_cast<uint32_t>(part) : g % NSLOT;
                    const uint32_t par = CF::WIDE ? ((part ? e_use1 : e_use0) & 1u) : ((g / NSLOT) & 1u);
                    if (CF::WIDE) {
                        if (part) ++e_use1;
                        else ++e_use0;
                    }
                    mbar_wait_prof(&acc_full[slot], par, w_full);
                    tc_fence_after();
                    const uint32_t taddr = tmem_base + lane_addr + slot * W + (SPLITH ? h * hw : 0);
                    if (!skip_ld) {
                        // 16 columns per wait (two tcgen05.ld in flight)
#pragma unroll
                        for (int c = 0; c < HP0; c += 16) {
                            if (c < hw) {
                                float v[2][8];
#pragma unroll
                                for (int u = 0; u < 2; ++u)
                                    if (c + 8 * u < hw) tmem_ld8(taddr + c + 8 * u, v[u]);
                                tmem_ld_wait();
#pragma unroll
                                for (int u = 0; u < 2; ++u)
#pragma unroll
                                    for (int i = 0; i < 8; i += 2)
                                        if (c + 8 * u < hw)
                                            ADD_PAIR(acc[aoff + c + 8 * u + i], acc[aoff + c + 8 * u + i + 1],
                                                     v[u][i], v[u][i + 1]);
                            }
                        }
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        if constexpr (PAIR) mbar_arrive_cluster(&acc_empty[slot], lead);
                        else mbar_arrive(&acc_empty[slot]);
                    }
                }
            }
            const long long ts0 = clock64();
            if (wk.slot >= 0) {
                // ---- stream-K partial piece (sk_fixup): publish this piece's sums in its slot's plane
                // (column-major 128-row planes per CTA half: a warp's 32 rows are one 128-B run), count
                // it, and the tile's LAST piece to arrive reads all of them back and sums them in
                // ascending k order (deterministic; nobody waits, so no co-residency is assumed)
                const int r_in = 32 * q + static_cast<int>(lane);
                const int64_t plane_el = static_cast<int64_t>(BN) * kBM;
                float* mine_pl = p.sk_ws + (static_cast<int64_t>(wk.slot) * kPair + crank) * plane_el + r_in;
#pragma unroll
                for (int part = 0; part < NQ; ++part) {
                    if (!mine(part)) continue;
                    const int hw = (part == NQ - 1) ? HPL : HP0;
                    const int aoff = SPLITH ? part * HP0 : 0;
                    const int c0 = part * W + (SPLITH ? h * hw : 0);
#pragma unroll
                    for (int i = 0; i < HP0; ++i)
                        if (i < hw) __stcg(mine_pl + static_cast<int64_t>(c0 + i) * kBM, acc[aoff + i]);
                }
                __threadfence();
                epi_bar();
                const int64_t K = p.num_kb, T = p.sk_total;
                const int u0 = sk_unit_of(wk.tile * K, T, units), u1 = sk_unit_of(wk.tile * K + K - 1, T, units);
                if (etid == 0) {
                    const uint32_t old = atomicAdd(p.sk_cnt + wk.tile * kPair + crank, 1u);
                    *sk_flag = (old + 1 == static_cast<uint32_t>(u1 - u0 + 1)) ? 1u : 0u;
                }
                epi_bar();
                if (*reinterpret_cast<volatile uint32_t*>(sk_flag) == 0u) {
                    t_store += clock64() - ts0;
                    continue;
                }
                __threadfence();
                // column groups of 8 outer (unrolled), the tile's pieces inner: 8 live sums, so the
                // fix-up adds no register pressure to the epilogue's accumulators
#pragma unroll
                for (int part = 0; part < NQ; ++part) {
                    if (!mine(part)) continue;
                    const int hw = (part == NQ - 1) ? HPL : HP0;
                    const int aoff = SPLITH ? part * HP0 : 0;
                    const int c0 = part * W + (SPLITH ? h * hw : 0);
#pragma unroll
                    for (int i = 0; i < HP0; i += 8) {
                        if (i < hw) {
                            float t8[8];
                            for (int u = u0; u <= u1; ++u) {
                                // unit u's piece of this tile is its first piece iff u's range starts
                                // inside the tile: floor(u*T/U) >= tile*K  <=>  u*T >= tile*K*U
                                const int sl = 2 * u + (static_cast<int64_t>(u) * T >= wk.tile * K * units ? 0 : 1);
                                const float* pl = p.sk_ws + (static_cast<int64_t>(sl) * kPair + crank) * plane_el + r_in +
                                                  static_cast<int64_t>(c0 + i) * kBM;
#pragma unroll
                                for (int e = 0; e < 8; ++e) {
                                    const float v = __ldcg(pl + e * kBM);
                                    t8[e] = (u == u0) ? v : __fadd_rn(t8[e], v);
                                }
                            }
#pragma unroll
                            for (int e = 0; e < 8; ++e) acc[aoff + i + e] = t8[e];
                        }
                    }
                }
            }
            // ---- store the tile rows owned by this thread (its half of every part's columns)
            const int64_t row = static_cast<int64_t>(m_blk) * CF::kTileM + static_cast<int64_t>(crank) * kBM + 32 * q +
                                static_cast<int>(lane);
            if (row < p.m) {
#pragma unroll
                for (int part = 0; part < NQ; ++part) {
                    if (!mine(part)) continue;
                    const int hw = (part == NQ - 1) ? HPL : HP0;
                    const int aoff = SPLITH ? part * HP0 : 0;
                    const int64_t col0 = static_cast<int64_t>(n_blk) * BN + part * W + (SPLITH ? h * hw : 0);
                    if (col0 >= p.n) continue;
                    float* dst = p.out + static_cast<int64_t>(wk.s) * p.split_stride + row * p.ldo_out + col0;
                    const int64_t valid = (p.n - col0) < hw ? (p.n - col0) : hw;
                    bool bad = false;
                    if (p.vec_store && valid == hw) {
#pragma unroll
                        for (int i = 0; i < HP0; i += 4)
                            if (i < hw)
                                *reinterpret_cast<float4*>(dst + i) =
                                    make_float4(acc[aoff + i], acc[aoff + i + 1], acc[aoff + i + 2], acc[aoff + i + 3]);
                    } else {
#pragma unroll
                        for (int i = 0; i < HP0; ++i)
                            if (i < valid) dst[i] = acc[aoff + i];
                    }
                    if (p.nonfinite) {
#pragma unroll
                        for (int i = 0; i < HP0; ++i)
                            if (i < valid && !isfinite(acc[aoff + i])) bad = true;
                        if (bad) atomicOr(p.nonfinite, 1);
                    }
                }
            }
            t_store += clock64() - ts0;
        }
        if (p.prof && warp == kEpiWarp0 && lane == 0) {
            long long* pr = p.prof + blockIdx.x * kProfSlots;
            pr[kProfEpiAccFull] = w_full;
            pr[kProfEpiStore] = t_store;
        }
    } else if (OMGEN && warp >= kWarpGen0) {
        // ============================================================ Omega generator (OMGEN)
        // cooperative in-kernel Omega (p.om_gen): the CTA (m_blk, s) generates the 64-k tiles
        // kb0s + m_blk + i * m_tiles of its split into the k-tiled buffer, in increasing k, and
        // releases each tile's flag; the Omega stagers of the split's m_tiles CTAs acquire the flags
        // before their TMA. Generation never waits on anything, so every flag is eventually set.
        asm volatile("setmaxnreg.dec.sync.aligned.u32 72;");
        const int gtid = static_cast<int>(threadIdx.x) - kWarpGen0 * 32;   // 0..255
        Piece wk;
        for (int it = 0; next_piece<NPA>(p, unit, units, sr, it, wk, pr); ++it) {
            const int64_t kb0s = wk.kb0;
            for (int64_t t = kb0s + wk.m_blk; t < kb0s + wk.nkb && p.om_gen == 1; t += p.m_tiles) {
                gen_omega_tile(p, t, gtid);
                gen_bar();
                if (gtid == 0) release_flag(p.om_flags + t);
            }
        }
    } else {
        // (one count for the four control warps: ptxas allocates the code after a setmaxnreg for the
        // count it sees there, so warp-dependent counts before shared code would over-allocate the
        // warps given fewer; the Omega stager's rare fallback generation spills instead)
        asm volatile("setmaxnreg.dec.sync.aligned.u32 32;");
        if (warp == kWarpProdA) {
            // ======================================================== A stager (TMA, FP32, own rows)
            if (elect_one()) {
                // A is streamed once: evict_first, unless several N tiles of an m-block read the same
                // A stages (n > BN). Those tiles are consecutive in the n-fastest tile order, so
                // they run concurrently on neighbouring CTAs; evict_normal keeps a stage in L2
                // until its last reader has fetched it, so A comes from HBM once instead of
                // n_tiles times (PAPER.md:652 counts mnk/b_n loads of A on the A100 design).
                // (NPA > 1: one cluster covers NPA N tiles, so only n_tiles > NPA re-reads A.)
                const uint64_t pol = p.n_tiles > NPA ? policy_evict_normal() : policy_evict_first();
                // A multicast: the CTAs of this row half in every pair of the cluster
                uint16_t a_mask = 0;
#pragma unroll
                for (int j = 0; j < NPA; ++j) a_mask |= static_cast<uint16_t>(1u << (crank + 2u * j));
                uint32_t sa = 0, pa = 0;
                uint32_t n_st = 0;     // stages staged so far (NPA > 1: the first SA are first uses)
                long long w = 0;
                Piece wk;
                for (int it = 0; next_piece<NPA>(p, unit, units, sr, it, wk, pr); ++it) {
                    const int m_blk = wk.m_blk, n_blk = wk.n_blk, kb0 = 0, kb1 = wk.nkb;
                    (void)m_blk;
                    (void)n_blk;
                    const int m0 = m_blk * CF::kTileM + static_cast<int>(crank) * kBM;
                    for (int kb = kb0; kb < kb1; ++kb, ++n_st) {
                        mbar_wait_prof(&a_empty[sa], pa ^ 1u, w);
                        mbar_arrive_expect_tx(&a_full[sa], kA32StageBytes);
                        if (NPA > 1 && !a_issuer) {
                            // slot free (its previous use consumed) and armed: tell the issuer of this
                            // row half, whose multicast fills it. The arrival completes the issuer's
                            // a_empty phase of that PREVIOUS use, which is what the issuer waits on
                            // before the next multicast into the slot; a slot's first use needs none
                            // (the issuer does not wait then, and bytes landing before the arm count
                            // in the same a_full phase). Relaxed: the arrive publishes no memory, and
                            // the splitters' reads of the slot completed before their own arrivals.
                            if (n_st >= static_cast<uint32_t>(SA)) mbar_arrive_cluster(&a_empty[sa], crank);
                            advance(sa, pa, SA);
                            continue;
                        }
                        const int64_t kk = (p.dbg & 32u) ? 0 : static_cast<int64_t>((wk.kb0 + (kb))) * kBK;
                        const int c0 = static_cast<int>(kk % p.k_inner);
                        const int c2 = static_cast<int>(kk / p.k_inner);
                        uint8_t* dst = a32 + sa * kA32StageBytes;
                        if constexpr (NPA > 1) {
                            if (p.a_rowpair) {
                                tma_load_4d_mc(dst, &mapA, &a_full[sa], 0, c0 >> 5, m0, c2, a_mask, pol);
                            } else {
                                const int64_t kk2 = kk + 32;
                                const bool wrap = kk2 < p.k && (c0 + 32) >= p.k_inner;
                                tma_load_3d_mc(dst, &mapA, &a_full[sa], c0, m0, c2, a_mask, pol);
                                tma_load_3d_mc(dst + kA32StageBytes / 2, &mapA, &a_full[sa],
                                               wrap ? static_cast<int>(kk2 % p.k_inner) : c0 + 32, m0,
                                               wrap ? static_cast<int>(kk2 / p.k_inner) : c2, a_mask, pol);
                            }
                        } else if (MMAJOR) {
                            // 2-D map {M (inner), K}, no swizzle: one box of 128 rows x 64 k, each
                            // k-line 512 contiguous bytes (4 KB-4 MB apart in HBM: one visit per line)
                            tma_load_2d(dst, &mapA, &a_full[sa], m0, static_cast<int>(kk), pol);
                        } else if (p.a_rowpair) {
                            // 4-D map {32, S/32, M, P}: one box of 128 rows x (2 x 32 k), row major
                            tma_load_4d(dst, &mapA, &a_full[sa], 0, c0 >> 5, m0, c2, pol);
                        } else {
                            // two 32-k halves; the second continues in the next slab when the
                            // view's contiguous run S ends mid-stage (S % 32 == 0 unfoldings). Past
                            // the last k it stays in dim 0 (zero-filled there: a box wholly outside
                            // the OUTER dimension never completed its transaction bytes)
                            const int64_t kk2 = kk + 32;
                            const bool wrap = kk2 < p.k && (c0 + 32) >= p.k_inner;
                            tma_load_3d(dst, &mapA, &a_full[sa], c0, m0, c2, pol);
                            tma_load_3d(dst + kA32StageBytes / 2, &mapA, &a_full[sa],
                                        wrap ? static_cast<int>(kk2 % p.k_inner) : c0 + 32, m0,
                                        wrap ? static_cast<int>(kk2 / p.k_inner) : c2, pol);
                        }
                        advance(sa, pa, SA);
                    }
                }
                if (p.prof) p.prof[blockIdx.x * kProfSlots + kProfProdAEmpty] = w;
            }
        } else if (warp == kWarpProdB) {
            // ======================================================== Omega stager (TMA, FP16)
            // per stage and per N-part one box: part 0 rows [n0 + crank*R0, +R0), part 1 rows
            // [n0 + W + crank*R1, +R1) (pair: each CTA holds its half of every part)
            if (elect_one()) {
                const uint64_t pol = policy_evict_last();
                const bool tiled = p.om_tiled != 0;
                uint32_t cs = 0, pc = 0;
                long long w = 0;
                Piece wk;
                for (int it = 0; next_piece<NPA>(p, unit, units, sr, it, wk, pr); ++it) {
                    const int m_blk = wk.m_blk, n_blk = wk.n_blk, kb0 = 0, kb1 = wk.nkb;
                    (void)m_blk;
                    (void)n_blk;
                    const int n0 = n_blk * BN;
                    for (int kb = kb0; kb < kb1; kb += KC) {
                        const int nst = (kb1 - kb) < KC ? (kb1 - kb) : KC;
                        mbar_wait_prof(&ch_empty[cs], pc ^ 1u, w);
                        const bool skip = (p.dbg & 8u) != 0;      // diagnostics: stale Omega (power study)
                        if (crank == 0) {
                            mbar_arrive_expect_tx(&ch_ready[cs], skip ? 0u : static_cast<uint32_t>(kPair * nst * kOm));
                        } else {
                            mbar_arrive_cluster(&ch_ready[cs], lead);
                        }
                        if (!skip) {
                            for (int t = 0; t < nst; ++t) {
                                const int kcoord = (p.dbg & 16u) ? 0 : (wk.kb0 + (kb + t)) * kBK;
                                if constexpr (OMGEN) acquire_or_generate(p, kcoord / kBK);   // generated in-kernel
                                // FP16: one 128-B box row = 64 k; TF32: two k-halves of 32 k
#pragma unroll
                                for (int hh = 0; hh < (TF32 ? 2 : 1); ++hh) {
                                    uint8_t* dst = om + (cs * KC + t) * kOm + hh * (CF::R0 + CF::R1) * 128;
                                    const int kc = kcoord + 32 * hh;
#pragma unroll
                                    for (int bt = 0; bt < CF::NB; ++bt) {   // TCEC: B_low tile, then dB_low
                                        uint8_t* d2 = dst + bt * CF::kOmTileBytes;
                                        const int nb0 = n0 + bt * p.b_lo_col;
                                        if constexpr (PAIR) {
                                            tma_load_omega<PAIR, TF32>(d2, &mapB0, &ch_ready[cs], kc,
                                                                 nb0 + static_cast<int>(crank) * CF::R0, pol, tiled);
                                            tma_load_omega<PAIR, TF32>(d2 + CF::R0 * 128, &mapB1, &ch_ready[cs], kc,
                                                                 nb0 + W + static_cast<int>(crank) * CF::R1, pol, tiled);
                                        } else if constexpr (CF::WIDE) {   // > 256 rows: one box per part
                                            tma_load_omega<PAIR, TF32>(d2, &mapB0, &ch_ready[cs], kc, nb0, pol, tiled);
                                            tma_load_omega<PAIR, TF32>(d2 + CF::R0 * 128, &mapB1, &ch_ready[cs], kc, nb0 + W, pol,
                                                                 tiled);
                                        } else {   // the two parts are contiguous rows: one box of BN rows (mapB0)
                                            tma_load_omega<PAIR, TF32>(d2, &mapB0, &ch_ready[cs], kc, nb0, pol, tiled);
                                        }
                                    }
                                }
                            }
                        }
                        advance(cs, pc, NCH);
                    }
                }
                if (p.prof) p.prof[blockIdx.x * kProfSlots + kProfProdBEmpty] = w;
            }
        } else if (warp == kWarpMMA && crank == 0) {
            // ======================================================== MMA issuer (tcgen05, A from TMEM)
            uint32_t cs = 0, pc = 0, g = 0;
            long long w_acc = 0, w_hl = 0, w_om = 0;
            const bool skip_mma = (p.dbg & 4u) != 0;
            // wide tiles: per-slot use counts (part 0 every stage, part 1 every second stage)
            uint32_t u0 = 0, u1 = 0;
            Piece wk;
            for (int it = 0; next_piece<NPA>(p, unit, units, sr, it, wk, pr); ++it) {
                const int m_blk = wk.m_blk, n_blk = wk.n_blk, kb0 = 0, kb1 = wk.nkb;
                (void)m_blk;
                (void)n_blk;
                if constexpr (CF::WIDE) {
                    // WIDE (KC = 1, 3 stage slots): each part is folded and promoted every TWO
                    // stages (K_c = 128 per part: lo MMAs of stages s and s+1 accumulate, then hi of
                    // s with scale-input-d = 11 and hi of s+1), the parts staggered by one stage so
                    // that one part (<= 144 columns) is drained per stage instead of all 272: the
                    // wide tile is bound by the TMEM read port otherwise. A stage slot
                    // is released one stage later (when both parts have consumed it).
                    auto part_mmas = [&](int part, uint32_t a_st, uint64_t b_st, int kind, bool first) {
                        // kind 0: lo (+ TCEC's A_low . dB_low); kind 1: hi, first with scale-input-d
                        const uint32_t d = tmem_base + part * W;
                        const uint32_t idesc = idesc_f16_f32(CF::kTileM, part ? WLAST : W);
                        const uint64_t b = b_st + static_cast<uint64_t>(((part ? CF::R0 : 0) * 128) >> 4);
                        if (kind == 0) {
#pragma unroll
                            for (int j = 0; j < NMMA; ++j)
                                mma_ts<PAIR, false>(d, a_st + AST / 2 + 8 * j, b + static_cast<uint64_t>(2 * j), idesc,
                                                    (first && j == 0) ? 0u : 1u);
                            if constexpr (TCEC) {
#pragma unroll
                                for (int j = 0; j < NMMA; ++j)
                                    mma_ts<PAIR, false>(d, a_st + 8 * j,
                                                        b + static_cast<uint64_t>(CF::kOmTileBytes >> 4) +
                                                            static_cast<uint64_t>(2 * j),
                                                        idesc, 1u);
                            }
                        } else {
#pragma unroll
                            for (int j = 0; j < NMMA; ++j) {
                                const uint32_t a = a_st + 8 * j;
                                const uint64_t bb = b + static_cast<uint64_t>(2 * j);
                                if (first && j == 0) mma_ts_scale11<PAIR, false>(d, a, bb, idesc);
                                else mma_ts<PAIR, false>(d, a, bb, idesc, 1u);
                            }
                        }
                    };
                    // part q folds and promotes PAIRS of stages, part 0 closing on odd local stages
                    // and part 1 on even ones (stage 0 alone), and both on the piece's last stage:
                    // one part is drained per stage, with two stages of MMAs to hide it
                    bool pend0 = false, pend1 = false;
                    uint32_t cs_prev = 0, a_prev = 0;
                    uint64_t b_prev = 0;
                    for (int kb = kb0; kb < kb1; ++kb) {
                        mbar_wait_prof(&ch_ready[cs], pc, w_hl);
                        const uint32_t a_cur = tmem_base + ABASE + cs * AST;
                        const uint64_t b_cur = sw128_kmajor_desc(smem_u32(om + cs * kOm));
                        const bool last = kb + 1 == kb1;
                        // the part that closes at this stage goes FIRST: its drain then has the other
                        // part's MMAs of this stage and the next one's (~1200 cycles) to hide behind
                        // before it is reused (closing it last left ~300 cycles: the MMA waited on
                        // acc_empty every other stage, profiles/r02_diag_wide2.jsonl)
                        const int cfirst = ((kb - kb0) & 1) ? 0 : 1;
#pragma unroll
                        for (int qi = 0; qi < 2; ++qi) {
                            const int q = qi ^ cfirst;
                            bool& pend = q ? pend1 : pend0;
                            uint32_t& u = q ? u1 : u0;
                            const bool close = (((kb - kb0) + q) & 1) == 1 || last;
                            if (!pend) {
                                mbar_wait_prof(&acc_empty[q], (u & 1u) ^ 1u, w_acc);
                                tc_fence_after();
                            }
                            if (elect_one()) {
                                if (!skip_mma) {
                                    part_mmas(q, a_cur, b_cur, 0, !pend);
                                    if (close) {
                                        if (pend) {
                                            part_mmas(q, a_prev, b_prev, 1, true);
                                            part_mmas(q, a_cur, b_cur, 1, false);
                                        } else {
                                            part_mmas(q, a_cur, b_cur, 1, true);
                                        }
                                    }
                                }
                                if (close) commit_to<PAIR>(&acc_full[q], pair_mask);
                            }
                            __syncwarp();
                            if (close) {
                                ++u;
                                pend = false;
                            } else {
                                pend = true;
                            }
                        }
                        // the previous stage is now consumed by both parts; the last one too at the end
                        if (elect_one()) {
                            if (kb > kb0) commit_to<PAIR>(&ch_empty[cs_prev], pair_mask);
                            if (last) commit_to<PAIR>(&ch_empty[cs], pair_mask);
                        }
                        __syncwarp();
                        cs_prev = cs;
                        a_prev = a_cur;
                        b_prev = b_cur;
                        advance(cs, pc, NCH);
                    }
                    continue;
                }
                for (int kb = kb0; kb < kb1; kb += KC) {
                    const int nst = (kb1 - kb) < KC ? (kb1 - kb) : KC;   // stages in this chunk
                    mbar_wait_prof(&ch_ready[cs], pc, w_hl);
                    const uint32_t a_base = tmem_base + ABASE + cs * KC * AST;
                    const uint64_t b_base = sw128_kmajor_desc(smem_u32(om + cs * KC * kOm));
#pragma unroll
                    for (int part = 0; part < NQ; ++part, ++g) {
                        const uint32_t slot = g % NSLOT;
                        mbar_wait_prof(&acc_empty[slot], ((g / NSLOT) & 1u) ^ 1u, w_acc);
                        tc_fence_after();
                        if (elect_one()) {
                            if (!skip_mma) {
                                const uint32_t d = tmem_base + slot * W;
                                const uint32_t idesc = TF32 ? idesc_tf32_f32(CF::kTileM, part == NQ - 1 ? WLAST : W)
                                                            : idesc_f16_f32(CF::kTileM, part == NQ - 1 ? WLAST : W);
                                const uint64_t b = b_base + static_cast<uint64_t>(((part ? CF::R0 : 0) * 128) >> 4);
                                // K step j of a stage: 32 B into a 128-B swizzle row; TF32 steps 4..7
                                // are in the second k-half box, (R0 + R1) rows further on
                                auto boff = [](int j) -> uint64_t {
                                    return TF32 ? static_cast<uint64_t>((((j >> 2) * (CF::R0 + CF::R1) * 128) >> 4) + 2 * (j & 3))
                                                : static_cast<uint64_t>(2 * j);
                                };
                                // D := sum over the chunk's stages of lo . Omega  (Eq 16's dA_low term)
#pragma unroll
                                for (int t = 0; t < KC; ++t)
                                    if (t < nst)
#pragma unroll
                                        for (int j = 0; j < NMMA; ++j)
                                            mma_ts<PAIR, TF32>(d, a_base + t * AST + AST / 2 + 8 * j,
                                                               b + static_cast<uint64_t>((t * kOm) >> 4) + boff(j), idesc,
                                                               (t > 0 || j > 0) ? 1u : 0u);
                                // TCEC (Eq 9): D += A_low . dB_low, so D = dA_low B_low + A_low dB_low
                                if constexpr (TCEC) {
#pragma unroll
                                    for (int t = 0; t < KC; ++t)
                                        if (t < nst)
#pragma unroll
                                            for (int j = 0; j < NMMA; ++j)
                                                mma_ts<PAIR, TF32>(d, a_base + t * AST + 8 * j,
                                                                   b + static_cast<uint64_t>((t * kOm + CF::kOmTileBytes) >> 4) + boff(j),
                                                                   idesc, 1u);
                                }
                                // D := hi . Omega + D * 2^-11 (first step), then the rest of hi
#pragma unroll
                                for (int t = 0; t < KC; ++t)
                                    if (t < nst)
#pragma unroll
                                        for (int j = 0; j < NMMA; ++j) {
                                            const uint32_t a = a_base + t * AST + 8 * j;
                                            const uint64_t bb = b + static_cast<uint64_t>((t * kOm) >> 4) + boff(j);
                                            if (t == 0 && j == 0) mma_ts_scale11<PAIR, TF32>(d, a, bb, idesc);
                                            else mma_ts<PAIR, TF32>(d, a, bb, idesc, 1u);
                                        }
                            }
                            commit_to<PAIR>(&acc_full[slot], pair_mask);
                        }
                        __syncwarp();
                    }
                    if (elect_one()) commit_to<PAIR>(&ch_empty[cs], pair_mask);
                    __syncwarp();
                    advance(cs, pc, NCH);
                }
            }
            if (p.prof && lane == 0) {
                long long* pr = p.prof + blockIdx.x * kProfSlots;
                pr[kProfMmaAccEmpty] = w_acc;
                pr[kProfMmaHlFull] = w_hl;
                pr[kProfMmaOmFull] = w_om;
            }
        }
    }

    tc_fence_before();
    if constexpr (PAIR) cluster_sync_all(); else __syncthreads();
    if (p.prof && threadIdx.x == 0) p.prof[blockIdx.x * kProfSlots + kProfTotal] = clock64() - t_kernel0;
    if (warp == kWarpMMA) {
        tc_fence_after();
        if constexpr (PAIR) {
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(kTmemCols)
                         : "memory");
        } else {
            tmem_dealloc<kTmemCols>(tmem_base);
        }
    }
}

// Fixed-order (s = 0..S-1) RN sum of split-K partial planes (a8 of SURVEY §8a; deterministic).
static __global__ void splitk_reduce_kernel(const float* __restrict__ ws, int splits, int64_t m, int64_t n,
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

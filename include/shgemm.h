/*
 * shgemm.h — C ABI of the B200 (sm_100a) SHGEMM random-projection library (libshgemm.so).
 *
 * Paper: H. Ootomo, R. Yokota, "Mixed-precision random projection for RandNLA on Tensor Cores"
 * (arXiv 2304.04612), /root/reference/PAPER.md, cited as P:<line>.
 *
 * The library computes the paper's one data-parallel hot path, the random projection
 * Y = A . Omega (Eq 1; Alg 1 line 1; Alg 2 line 2), with A in FP32 and
 * Omega a random matrix stored in FP16, by SHGEMM (Eqs 14-17): every FP32
 * element of A is split in-kernel into an FP16 hi and a 2^11-scaled FP16 lo part, both products
 * run on the tensor cores, and accumulation is promoted to round-to-nearest FP32 adds
 * (P:36-37).
 *
 * Conventions for every call
 *  - Pointers named A/Omega/Y/W/workspace/hi/lo are DEVICE pointers (CUDA global memory) unless
 *    the name says host. The caller owns every buffer; the library keeps no allocation past a call
 *    (project() without a workspace uses stream-ordered cudaMallocAsync/cudaFreeAsync).
 *  - All work is enqueued asynchronously on `stream` (a cudaStream_t; NULL = legacy default).
 *    Argument errors are returned synchronously and nothing is enqueued; faults inside kernels
 *    surface at the caller's next synchronization (CUDA convention).
 *  - Layouts: A is row-major m x k with leading dimension lda >= k
 *    (elements); Y is row-major m x n, ldc >= n. Omega (k x n, FP16 stored as uint16_t bit
 *    patterns) is ROW-major by default, Omega[i][j] at Omega[i*ldo + j] with ldo >= n — the layout
 *    of shgemm() and gen_omega_f16(). The _ex calls also take it COLUMN-major
 *    (SHG_OMEGA_COL_MAJOR: Omega[i][j] at Omega[j*ldo + i], ldo >= k), which is the tensor cores'
 *    K-major B operand and is streamed by TMA as is; a row-major Omega is first transposed into
 *    that layout in the workspace (transpose_omega_kernel, 4kn bytes of traffic, one launch).
 *    Both layouts give bitwise-identical Y. The layout is always explicit (an argument or
 *    shg_tune_t.omega_layout), never guessed from ldo: for n == k both leading dimensions are valid.
 *  - Tensor-core fast path preconditions: A, Y 16-byte aligned, lda % 4 == 0; a column-major
 *    Omega also 16-byte aligned with ldo % 8 == 0 (TMA row pitch multiple of 16 B). Otherwise a
 *    CUDA-core fallback with the same numerics contract runs (slower).
 *  - Numerical exceptions are not errors: |a| >= 65520 overflows the FP16 hi part to +-inf and
 *    the affected Y rows become non-finite — the paper's expected SHGEMM-FP16 failure on
 *    A_Cauchy. NaN propagates. The _ex variants can raise a device flag.
 *  - Determinism: identical inputs, shapes and tunables give bitwise-identical Y (fixed-order
 *    split-K reduction, no atomics on data).
 *  - Requires a compute-capability 10.0 device (B200); otherwise SHG_ERR_UNSUPPORTED_DEVICE.
 */
#ifndef SHGEMM_H_
#define SHGEMM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *shg_stream_t; /* == cudaStream_t */

typedef enum {
    SHG_OK = 0,
    SHG_ERR_INVALID_VALUE = 1,      /* bad dimension, leading dimension, mode or NULL pointer */
    SHG_ERR_UNSUPPORTED_DEVICE = 2, /* current device is not sm_100 */
    SHG_ERR_CUDA = 3,               /* a CUDA runtime/driver call failed; see shg_last_error() */
    SHG_ERR_WORKSPACE = 4           /* caller workspace smaller than required */
} shg_status_t;

/* Omega distributions (OMEGA_SPEC.md §3-4). Gaussian N(0,1) rounded RN to FP16;
 * sparse sign matrices of Eq 7 without the sqrt(s) factor. */
typedef enum {
    SHG_DIST_GAUSSIAN = 0,
    SHG_DIST_RADEMACHER = 1,  /* s = 1 */
    SHG_DIST_SPARSE3 = 2,     /* s = 3 (Achlioptas) */
    SHG_DIST_VERYSPARSE = 3   /* s = sqrt(k) (Li et al.), k = rows of the full Omega */
} shg_dist_t;

/* Tensor-core kind of the SHGEMM ("two kinds of SGEMM"). */
typedef enum {
    SHG_TC_FP16 = 0,  /* SHGEMM-FP16: toLow = FP16 (Eqs 14-17); |A| < 65520 (FP16 range) */
    SHG_TC_TF32 = 1,  /* SHGEMM-TF32: toLow = TF32 (e8m10): the full FP32 exponent range, Omega
                         widened exactly to TF32; half the FP16 tensor-core rate */
    SHG_TC_TCEC = 2   /* reported in shg_plan_t.tc by tcec_plan only: TCEC-SGEMM (Eqs 5-9) */
} shg_tc_t;

/* Operand layouts for tcec_sgemm. For A (m x k): K_MAJOR = row-major, element (i, l) at
 * A[i * lda + l], lda >= k; MN_MAJOR = element (i, l) at A[l * lda + i], lda >= m (A given as its
 * k x m row-major transpose). For B (k x n): K_MAJOR = column-major, element (l, j) at
 * B[j * ldb + l], ldb >= k; MN_MAJOR = row-major, element (l, j) at B[l * ldb + j], ldb >= n. */
typedef enum { SHG_LAYOUT_K_MAJOR = 0, SHG_LAYOUT_MN_MAJOR = 1 } shg_layout_t;

/* Omega layouts (k x n FP16). ROW_MAJOR is SURVEY §8(b)'s: Omega[i][j] at Omega[i*ldo + j],
 * ldo >= n. COL_MAJOR: Omega[i][j] at Omega[j*ldo + i], ldo >= k (the kernel's native K-major
 * operand: no transpose pass). Any other value: SHG_ERR_INVALID_VALUE. */
typedef enum { SHG_OMEGA_ROW_MAJOR = 0, SHG_OMEGA_COL_MAJOR = 1 } shg_omega_layout_t;

/* Tunables for shgemm_ex. Zero-initialise for the heuristics. */
typedef struct {
    int32_t bn;          /* N tile (multiple of 16, <= 256); 0 = heuristic */
    int32_t split_k;     /* number of k splits; 0 = heuristic, 1 = none */
    int32_t max_ctas;    /* persistent grid size cap; 0 = number of SMs */
    int32_t force_simt;  /* 1 = force the CUDA-core fallback (tests) */
    /* Diagnostics only (results are WRONG when debug_flags != 0): bit0 skip the TMEM->register
     * promotion loads, bit1 skip the splitter arithmetic, bit2 skip the MMAs, bit3 skip the Omega
     * loads, bit4 load Omega k-tile 0 for every stage (constant B data), bit5 load A's k-block 0 of
     * its rows for every stage (L2 hits instead of the HBM stream). */
    int32_t debug_flags;
    int32_t pair;        /* CTA pairs (tcgen05.mma.cta_group::2): 0 auto (BN >= 128 and m > 128), 1 on, 2 off */
    int32_t a_box;       /* row-major A staging: 0 auto (2 if k % 32 == 0 and lda >= 2 MiB, else 1), 1 two TMA boxes of
                            {32 k, 128 rows} per stage (128 B per row visit), 2 one box of
                            {2 x 32 k, 128 rows} (256 B per row visit; needs k % 32 == 0, else
                            SHG_ERR_INVALID_VALUE). Ignored for M-major A (shgemm_at). */
    int32_t tc;          /* shg_tc_t: SHG_TC_FP16 (0, default) or SHG_TC_TF32; selects the kernel, not a
                            tuning: the results differ (TF32 keeps |a| >= 65520 finite) */
    int32_t omega_mcast; /* 0 or 1 (Omega stages are loaded per CTA pair). The round-1 option of multicasting
                            them to 2-4 pairs of a cluster was measured without a steady-state gain and
                            removed; other values: SHG_ERR_INVALID_VALUE. */
    /* Diagnostics: device int64[grid * 16] per-CTA wait-cycle counters (layout in
     * csrc/shgemm_sm100.cuh, enum ProfSlot), or NULL. */
    int64_t *prof;
    int32_t omega_layout; /* shg_omega_layout_t of the Omega argument: SHG_OMEGA_ROW_MAJOR (0, default;
                             ldo >= n) or SHG_OMEGA_COL_MAJOR (ldo >= k). A NULL tune means row-major. */
    int32_t stream_k;     /* work schedule: 0 auto, 1 stream-K, 2 whole tiles. Stream-K cuts the
                             (tile, k-block) iterations into one equal contiguous range per SM (pair)
                             and sums the partial tiles in-kernel in fixed k order (deterministic).
                             Auto uses it on the HBM side (BN <= 160) when whole tiles would leave the
                             last wave < 92% busy (one N tile, >= half as many tiles as SMs (pairs),
                             k >= 1024): e.g. m = k = 32768, n = 128, 15% faster. Needs
                             one N tile, no split_k > 1 and >= 4 k-blocks per unit: otherwise
                             SHG_ERR_INVALID_VALUE. Row shards of one Y are bitwise equal to the
                             unsharded Y only under whole tiles (stream-K's sums depend on the grid). */
    int32_t a_mcast;      /* A multicast: 0 auto, 1 off, 2 or 4 = CTA pairs per cluster that take one m-block
                             and that many N tiles together, each A stage fetched once per cluster and
                             multicast by TMA to the CTAs holding its rows (A read once for n_tiles ==
                             a_mcast; PAPER.md:652 counts the A100 design's mnk/b_n loads of A). Needs
                             SHGEMM-FP16 CTA pairs, K-major A (shgemm / project, not shgemm_at), BN in
                             {128, 192, 256}, n_tiles % a_mcast == 0, no split-K and no stream-K:
                             otherwise SHG_ERR_INVALID_VALUE. Bitwise-identical Y (the arithmetic is
                             unchanged). */
} shg_tune_t;

/* Plan the library would use for an (m, n, k) shgemm on the current device. */
typedef struct {
    int32_t path;        /* 0 = tcgen05 mainloop, 1 = SIMT fallback, 2 = trivial (no GEMM) */
    int32_t bn, n_tiles, m_tiles, split_k, grid, stages_a, stages_b, smem_bytes;
    int32_t kernels;     /* kernel launches one call makes */
    int32_t cta_pair;    /* 1 if the mainloop runs as CTA pairs (cluster of 2, cta_group::2) */
    int32_t tc;          /* shg_tc_t the plan runs */
    int32_t omega_mcast; /* always 1 (no Omega multicast) */
    int32_t stream_k;    /* 1 if the plan uses the stream-K schedule (shg_tune_t.stream_k) */
    int64_t workspace_bytes;
    int32_t a_mcast;     /* CTA pairs per cluster sharing each A stage (shg_tune_t.a_mcast); 1 = none */
} shg_plan_t;

/* ---------------------------------------------------------------------------------------------
 * shgemm — Y[m x n] = A[m x k] . Omega[k x n] by SHGEMM-FP16 (Eqs 14-17).
 *   m, n, k  >= 0. m == 0 or n == 0: no-op. k == 0: Y = 0.
 *   A        device, row-major, lda >= max(k,1).   Omega device, ROW-major, ldo >= max(n,1).
 *   Y        device, row-major, ldc >= max(n,1); overwritten (beta = 0).
 *   Errors   SHG_ERR_INVALID_VALUE for negative sizes, short leading dimensions or NULL pointers
 *            (nothing enqueued); SHG_ERR_UNSUPPORTED_DEVICE off sm_100; SHG_ERR_CUDA on a failed launch.
 * Scratch (the column-major copy of Omega the tensor cores read; split-K planes when the heuristic
 * splits k) is stream-ordered cudaMallocAsync memory freed on `stream`.
 * ------------------------------------------------------------------------------------------- */
shg_status_t shgemm(int64_t m, int64_t n, int64_t k, const float *A, int64_t lda, const uint16_t *Omega,
                    int64_t ldo, float *Y, int64_t ldc, shg_stream_t stream);

/* shgemm by SHGEMM-TF32: Eqs 14-17 with toLow = TF32 (RN ties-to-even), so
 * any finite FP32 A below (2 - 2^-11) * 2^127 is accepted (A_Cauchy of P:699-706 stays finite).
 * Same arguments and layouts as shgemm (row-major Omega, ldo >= n); Omega stays FP16 in memory and
 * is widened exactly to TF32 in stream-ordered scratch (k x n x 4 bytes) for the tensor cores. */
shg_status_t shgemm_tf32(int64_t m, int64_t n, int64_t k, const float *A, int64_t lda, const uint16_t *Omega,
                         int64_t ldo, float *Y, int64_t ldc, shg_stream_t stream);

/* shgemm with tunables (tune->tc selects SHGEMM-FP16 or -TF32; tune->omega_layout the Omega
 * layout, row-major when tune is NULL), caller workspace (>= shg_workspace_size bytes for the same
 * tune, or NULL), and an optional device int flag set to 1 if any output is non-finite (never
 * cleared by the library). */
shg_status_t shgemm_ex(int64_t m, int64_t n, int64_t k, const float *A, int64_t lda, const uint16_t *Omega,
                       int64_t ldo, float *Y, int64_t ldc, const shg_tune_t *tune, void *workspace,
                       size_t workspace_bytes, int *nonfinite_flag, shg_stream_t stream);

/* shgemm_ex for an M-major A ("A transposed"): element (i, l) of A is At[l * ldat + i], i.e. At is
 * the k x m row-major transpose of A, ldat >= m (fast path: At 16-B aligned, ldat % 4 == 0). This
 * is how project() reads the last-mode unfolding of a C-order tensor in place. Omega layout from
 * tune->omega_layout as for shgemm_ex. */
shg_status_t shgemm_at(int64_t m, int64_t n, int64_t k, const float *At, int64_t ldat, const uint16_t *Omega,
                       int64_t ldo, float *Y, int64_t ldc, const shg_tune_t *tune, void *workspace,
                       size_t workspace_bytes, int *nonfinite_flag, shg_stream_t stream);

/* Bytes of workspace shgemm_ex needs for (m, n, k) with `tune` (NULL = heuristics, row-major Omega):
 * split-K partial planes, plus the TF32 copy of Omega when tune->tc == SHG_TC_TF32, or the
 * column-major copy of a row-major FP16 Omega. */
size_t shg_workspace_size(int64_t m, int64_t n, int64_t k, const shg_tune_t *tune);

/* Fill *plan for (m, n, k) with `tune` (NULL = heuristics), without launching anything. */
shg_status_t shg_plan(int64_t m, int64_t n, int64_t k, const shg_tune_t *tune, shg_plan_t *plan);

/* ---------------------------------------------------------------------------------------------
 * tcec_sgemm — C[m x n] = A[m x k] . B[k x n] for FP32 A AND FP32 B by TCEC-SGEMM, the authors'
 * error-corrected single-precision GEMM on FP16 tensor cores (Eqs 5-9; SURVEY §8f
 * NEXT-2): A_low = toLow(A), dA_low = toLow((A - A_low) * 2^11), likewise for B (RN to FP16,
 * P:190), and C ~ A_low.B_low + (dA_low.B_low + A_low.dB_low) * 2^-11 (Eq 9; dA_low.dB_low is
 * dropped), accumulated per 128-k chunk on the tensor cores and added with RN on the CUDA cores
 * (P:181). It serves the RandNLA pipelines' other FP32 products: B = Q^T A (Alg 1 line 3, P:129;
 * computed as B^T = A^T Q with an MN_MAJOR A) and the RP-HOSVD core contractions (Alg 2 line 5).
 *   m, n, k  >= 0. m == 0 or n == 0: no-op. k == 0: C = 0.
 *   A, B     device FP32 in the shg_layout_t given by a_layout / b_layout (see shg_layout_t).
 *   C        device, row-major, ldc >= n; overwritten (beta = 0).
 *   Range: as SHGEMM-FP16, |a|, |b| >= 65520 overflow to non-finite C; entries below 2^-14
 *   lose relative precision in their FP16 parts (absolute error <= ~2^-36 |other operand|).
 *   Error: |C - AB| <~ ((k/8) + 3) u |A||B| elementwise (u = 2^-24), the SGEMM level.
 * B is split once per call (split_b_kernel) into stream-ordered scratch, or into `workspace`
 * (>= tcec_sgemm_workspace_size bytes) with tcec_sgemm_ex. Fast path: A 16-B aligned and
 * lda % 4 == 0 (B has no alignment requirement); otherwise a CUDA-core fallback (same contract).
 * Errors: SHG_ERR_INVALID_VALUE for negative sizes, bad layouts, short leading dimensions, NULL
 * pointers with k > 0, or tune->bn > 128 with single CTAs (TCEC stages two B tiles).
 * ------------------------------------------------------------------------------------------- */
shg_status_t tcec_sgemm(int64_t m, int64_t n, int64_t k, const float *A, int64_t lda, int a_layout,
                        const float *B, int64_t ldb, int b_layout, float *C, int64_t ldc, shg_stream_t stream);

/* tcec_sgemm with tunables (bn, split_k, max_ctas, pair, a_box, force_simt; tc ignored) and a
 * caller workspace (NULL = stream-ordered scratch). */
shg_status_t tcec_sgemm_ex(int64_t m, int64_t n, int64_t k, const float *A, int64_t lda, int a_layout,
                           const float *B, int64_t ldb, int b_layout, float *C, int64_t ldc,
                           const shg_tune_t *tune, void *workspace, size_t workspace_bytes, shg_stream_t stream);

size_t tcec_sgemm_workspace_size(int64_t m, int64_t n, int64_t k, const shg_tune_t *tune);

/* Plan of a tcec_sgemm call (plan->tc = SHG_TC_TCEC). */
shg_status_t tcec_plan(int64_t m, int64_t n, int64_t k, const shg_tune_t *tune, shg_plan_t *plan);

/* ---------------------------------------------------------------------------------------------
 * gen_omega_f16 — Omega[i][j] = OMEGA_SPEC(seed, stream_id = 0, dist, i, j) for 0 <= i < k,
 * 0 <= j < n (the random matrix of Eq 1 / Alg 1 line 1, drawn in FP32 and rounded RN
 * to FP16), written ROW-major with ldo >= n (FP16 bits). Bit-identical to the CPU oracle.
 * Errors: SHG_ERR_INVALID_VALUE for negative sizes, dist outside shg_dist_t, ldo < n or NULL Omega.
 * ------------------------------------------------------------------------------------------- */
shg_status_t gen_omega_f16(int64_t k, int64_t n, uint64_t seed, int dist, uint16_t *Omega, int64_t ldo,
                           shg_stream_t stream);

/* As gen_omega_f16 with an explicit Philox stream id, a row offset (local row r holds spec row
 * row0 + r; used for K-sharding), the full-Omega row count k_total for SHG_DIST_VERYSPARSE, and the
 * output layout (shg_omega_layout_t: ROW_MAJOR ldo >= n, COL_MAJOR ldo >= k). */
shg_status_t gen_omega_f16_ex(int64_t k, int64_t n, uint64_t seed, int dist, uint32_t stream_id,
                              int64_t row0, int64_t k_total, uint16_t *Omega, int64_t ldo, int layout,
                              shg_stream_t stream);

/* project() with Omega_(mode) supplied by the caller, already generated in the k-tiled layout by
 * gen_omega_f16_tiled(K, n, seed, dist, stream_id = mode, ...) with K = prod_{j != mode} dims[j] —
 * so the generation can run earlier / on another stream (the RSVD/RP-HOSVD harness overlaps it with
 * the previous mode's QR). SHGEMM-FP16; needs the tcgen05 path (16-B aligned A view), otherwise
 * SHG_ERR_INVALID_VALUE. Workspace as project(). */
shg_status_t project_omega(const float *A, int ndim, const int64_t *dims, int mode, int64_t n,
                           const uint16_t *Omega_tiled, float *W, int64_t ldw, void *workspace,
                           size_t workspace_bytes, shg_stream_t stream);

/* gen_omega_f16_ex into the K-TILED layout that project() streams: rows i of Omega are grouped in
 * tiles of 64 (t = i / 64), each tile stored as n contiguous 128-byte rows (one per column j):
 * element (i, j) at Omega[(i / 64) * n * 64 + j * 64 + i % 64]. Omega holds ceil(k/64) * n * 64
 * halves; rows k .. 64*ceil(k/64)-1 of the last tile are written as +0. The same values as
 * gen_omega_f16_ex(k, n, seed, dist, stream_id, row0, k_total). Why: a column-major 64-k TMA box
 * visits n rows 2*ldo bytes apart (2 MiB for an RP-HOSVD unfolding, k = 2^20); a tiled box is one
 * contiguous run of n x 128 bytes. */
shg_status_t gen_omega_f16_tiled(int64_t k, int64_t n, uint64_t seed, int dist, uint32_t stream_id, int64_t row0,
                                 int64_t k_total, uint16_t *Omega, shg_stream_t stream);

/* shgemm_ex (tune->tc: SHG_TC_FP16, or SHG_TC_TF32 which widens the tiles to a 32-k-tiled FP32
 * copy) reading a k-tiled Omega written by gen_omega_f16_tiled(k, n, ...). Needs the tcgen05 fast
 * path (A 16-B aligned, lda % 4 == 0); otherwise SHG_ERR_INVALID_VALUE (the CUDA-core fallback
 * reads column-major Omega only). */
shg_status_t shgemm_tiled(int64_t m, int64_t n, int64_t k, const float *A, int64_t lda, const uint16_t *Omega_tiled,
                          float *Y, int64_t ldc, const shg_tune_t *tune, void *workspace, size_t workspace_bytes,
                          int *nonfinite_flag, shg_stream_t stream);

/* ---------------------------------------------------------------------------------------------
 * project — W[I_mode x n] = A'_(mode) . Omega_(mode) (Alg 2 line 2). With an aligned A
 * view, Omega_(mode) is generated in the k-tiled layout (gen_omega_f16_tiled) — by default inside
 * the projection kernel when the plan has one tile per CTA (shg_set_inkernel_omega), else by a
 * separate gen_omega launch; the bits of Omega and W are the same either way.
 *   A        device, C-order tensor with ndim dims (1 <= ndim <= 8), dims[i] >= 1.
 *   mode     0 <= mode < ndim. The unfolding's column index is the C-order linear index over the
 *            remaining modes in ascending order (== torch.movedim(A, mode, 0).reshape(I_mode, -1)).
 *   Omega_(mode) = gen_omega_f16_ex(K = prod_{j != mode} dims[j], n, seed, dist,
 *            stream_id = mode, row0 = 0, k_total = K).
 *   W        device, row-major I_mode x n, ldw >= n.
 *   workspace  device scratch of >= shg_project_workspace_size(...) bytes, or NULL (then the
 *            library allocates stream-ordered memory and frees it on `stream`).
 * ------------------------------------------------------------------------------------------- */
shg_status_t project(const float *A, int ndim, const int64_t *dims, int mode, int64_t n, uint64_t seed,
                     int dist, float *W, int64_t ldw, void *workspace, size_t workspace_bytes,
                     shg_stream_t stream);

size_t shg_project_workspace_size(int ndim, const int64_t *dims, int mode, int64_t n);

/* project with the tensor-core kind `tc` (shg_tc_t); project() == project_ex(..., SHG_TC_FP16, ...). */
shg_status_t project_ex(const float *A, int ndim, const int64_t *dims, int mode, int64_t n, uint64_t seed,
                        int dist, int tc, float *W, int64_t ldw, void *workspace, size_t workspace_bytes,
                        shg_stream_t stream);

size_t shg_project_workspace_size_ex(int ndim, const int64_t *dims, int mode, int64_t n, int tc);

/* project_ex for a SLAB of a larger tensor (K-sharded RP-HOSVD): A is
 * this rank's C-order piece with dims `dims`, and its mode-`mode` unfolding's K_local columns are
 * columns [omega_row0, omega_row0 + K_local) of the full tensor's unfolding, so W is multiplied with
 * rows [omega_row0, omega_row0 + K_local) of the full Omega_(mode) = gen_omega_f16_ex(k_total, n,
 * seed, dist, stream_id = mode). Summing W over the slabs (one all-reduce) gives the full W.
 * k_total = 0 means omega_row0 + K_local (matters only for SHG_DIST_VERYSPARSE). Workspace as
 * project_ex (shg_project_workspace_size_ex of the LOCAL dims). omega_row0 < 0 or
 * k_total < omega_row0 + K_local: SHG_ERR_INVALID_VALUE. */
shg_status_t project_shard(const float *A, int ndim, const int64_t *dims, int mode, int64_t n, uint64_t seed,
                           int dist, int tc, int64_t omega_row0, int64_t k_total, float *W, int64_t ldw,
                           void *workspace, size_t workspace_bytes, shg_stream_t stream);

/* ---------------------------------------------------------------------------------------------
 * shgemm_host — Y = A . Omega with A and Y in HOST memory (pinned for overlap; pageable works but
 * serialises), Omega on the device in `omega_layout` (shg_omega_layout_t). A is streamed to the
 * device in row chunks of `chunk_rows` (0 = heuristic) through two staging buffers: H2D copy of
 * chunk c+1 and D2H copy of chunk c-1 overlap the SHGEMM of chunk c on two side streams created
 * for this call and ordered after / before `stream` by events created for this call, so
 * concurrent calls from several host threads (on their own streams) do not serialise on shared
 * library state. workspace: device scratch >= shg_host_workspace_size(n, k, chunk_rows,
 * omega_layout) bytes (covers every chunk height up to chunk_rows, including a short last chunk),
 * or NULL (stream-ordered allocation). Returns when everything is enqueued; synchronize `stream`.
 * On an error after work was enqueued, the side streams are still joined to `stream` and owned
 * scratch is freed on it before returning.
 * ------------------------------------------------------------------------------------------- */
shg_status_t shgemm_host(int64_t m, int64_t n, int64_t k, const float *A_host, int64_t lda,
                         const uint16_t *Omega, int64_t ldo, int omega_layout, float *Y_host, int64_t ldc,
                         int64_t chunk_rows, void *workspace, size_t workspace_bytes, shg_stream_t stream);

size_t shg_host_workspace_size(int64_t n, int64_t k, int64_t chunk_rows, int omega_layout);

/* ---------------------------------------------------------------------------------------------
 * Test / bench support (not part of the method).
 * ------------------------------------------------------------------------------------------- */
/* Elementwise split of Eqs 14-15 with the SAME device function the mainloop uses:
 * hi[t], lo[t] = FP16 bits of toLow(a[t]) and toLow((a[t] - hi) * 2^11). Device pointers. */
shg_status_t shg_debug_split(const float *a, int64_t count, uint16_t *hi, uint16_t *lo, shg_stream_t stream);

/* Elementwise SHGEMM-TF32 split with the mainloop's device function: hi[t], lo[t] = FP32 bit
 * patterns of RN_tf32(a[t]) and RN_tf32((a[t] - hi) * 2^11) (low 13 bits zero). Device pointers. */
shg_status_t shg_debug_split_tf32(const float *a, int64_t count, uint32_t *hi, uint32_t *lo, shg_stream_t stream);

/* Synthetic FP32 input of OMEGA_SPEC §6 (kind 0 Gaussian, 1 uniform [0,1)):
 * A[i*lda + l] = synth(seed, stream_id, global row row0 + i, column l), 0 <= i < m, 0 <= l < k. */
shg_status_t shg_synth_f32(int kind, uint64_t seed, uint32_t stream_id, int64_t m, int64_t k, int64_t row0,
                           float *A, int64_t lda, shg_stream_t stream);

/* TMA read-bandwidth probe (diagnostics): `grid` CTAs stream the full 128-row
 * m-blocks of A (device, m x k FP32, row stride lda) into shared memory with TMA only, in the
 * mainloop's tile order (m-block major, `splits` contiguous k ranges). Box per load:
 *   layout 0: 2-D {box_k, box_rows}, no swizzle (box_k <= 256, multiple of 4)
 *   layout 1: 2-D {32, box_rows}, 128-B swizzle (the mainloop's A box)
 *   layout 2: 3-D {32, box_k/32, box_rows} over dims {32, k/32, m}, 128-B swizzle
 * box_k * box_rows * 4 <= 32768, 128 % box_rows == 0. Adds the bytes loaded to *bytes_out (device
 * u64). Time it with events on `stream`. */
shg_status_t shg_probe_tma_read(const float *A, int64_t m, int64_t k, int64_t lda, int layout, int box_k,
                                int box_rows, int splits, int grid, unsigned long long *bytes_out,
                                shg_stream_t stream);

/* project()/project_shard() with SHGEMM-FP16: generate Omega_(mode) INSIDE the projection kernel
 * (on = 1, the default since round 2) instead of a separate gen_omega launch, when the plan has
 * one tile per CTA and single-CTA tiles of BN <= 128 ("fused in-producer
 * Omega"): the m-tiles that share a k range each generate 1/m_tiles of its k-tiled Omega with
 * dedicated generator warps and publish per-tile flags that the Omega stager acquires; a stager
 * whose tile is not published within 200 us generates it itself (same bits), so the kernel never
 * depends on another CTA being resident. Same bits as gen_omega_f16_tiled either way. on = 0: the
 * separate generator; on = 2 (tests): the generator warps stay idle and every tile comes from the
 * stagers' fallback. Process-wide; SHG_OMGEN=0 sets the default to the separate generator.
 * shg_get_inkernel_omega returns the current setting. */
void shg_set_inkernel_omega(int on);
int shg_get_inkernel_omega(void);
/* Test support: how many k-tiles of Omega the stagers' generate-on-timeout fallback has produced in
 * this process so far (synchronous read of a device counter; UINT64_MAX on a CUDA error). */
uint64_t shg_inkernel_omega_fallbacks(void);

/* Process-wide default of shg_tune_t.a_mcast for calls whose tune leaves it 0 (and for project(),
 * tcec paths excluded): 0 = the automatic rule (2 pairs per cluster when the N tiles pair up,
 * DESIGN.md §5), 1 = off, 2 or 4 = that many pairs per cluster where the plan is eligible (silently
 * off where not). Returns the previous value, or -1 (unchanged) for any other npa. */
int shg_set_a_mcast(int npa);

/* Number of kernels this library has launched in this process (monotonic). */
uint64_t shg_launch_count(void);

/* Message of the last SHG_ERR_CUDA in this thread ("" if none). */
const char *shg_last_error(void);

/* 1 if the current device can run the tcgen05 path (cc 10.0), else 0. */
int shg_device_supported(void);

/* Library version, e.g. "shgemm-b200 0.2.0 sm_100a". */
const char *shg_version(void);

/* Tensor-core semantics probe: ONE CTA runs tcgen05.mma.cta_group::1.kind::f16
 * with M = 128, N = n (16 <= n <= 256, n % 16 == 0), K = 64 (four K=16 instructions) on
 *   A  device, 128 x 64 FP16 bits, row-major (K-contiguous);  B  device, n x 64 FP16 bits, row-major;
 *   D_init device 128 x n FP32 row-major preloaded into TMEM with tcgen05.st, or NULL (D starts
 *          undefined and the first instruction runs with enable-input-d = 0);
 *   mode 0: D = D_init + sum_{j<nsteps} A_j B_j^T                 (j = 16-wide K step)
 *   mode 1: D = D_init * 2^-11 + sum_{j<nsteps} A_j B_j^T   (first instruction has scale-input-d = 11)
 *   nsteps 1..4 instructions; D_out device 128 x n FP32 row-major. */
shg_status_t shg_probe_umma(const uint16_t *A, const uint16_t *B, int n, const float *D_init, int mode,
                            int nsteps, float *D_out, shg_stream_t stream);

/* MMA-rate microbenchmark: `grid` CTAs each issue `iters` back-to-back
 * 128 x n x 16 kind::f16 MMAs (A from TMEM if ts, else smem) while `lsu_warps` warps stream
 * shared-memory loads/stores (lsu_warps bits 0-2) into (lsu_warps >> 3, min 1) rotating
 * accumulators; out[cta] (device floats) = cycles per MMA. */
shg_status_t shg_probe_mma_rate(int n, int iters, int ts, int lsu_warps, float *out, int grid,
                                shg_stream_t stream);

/* Same for tcgen05.mma.cta_group::2 (clusters of 2 CTAs, M = 256, n % 32 == 0): out[cluster] =
 * cycles per pair-MMA instruction (256 x n x 16 MACs on two SMs). */
shg_status_t shg_probe_mma2_rate(int n, int iters, int ts, float *out, int clusters, shg_stream_t stream);

/* MMA energy probe: `clusters` CTA pairs each issue `iters` K steps of
 * cta_group::2 kind::f16 MMAs (M = 256, A from TMEM, B from smem, random FP16 data), each K step
 * split into `parts` (1 or 2) MMAs of N = n / parts; out[cluster] (device int64) = clock64 cycles
 * of the issuing loop. Timed with events under the power cap it measures tensor work per joule. */
shg_status_t shg_probe_mma_energy(int n, int parts, int iters, long long *out, int clusters, shg_stream_t stream);

/* Box-Muller probe (OMEGA_SPEC §3.1-3.2, the Gaussian Omega of PAPER.md:448-451): for each of
 * `count` Philox output words w (device uint32), r[i] = the generator's radius sqrt(-2 ln(((w >> 8) + 1)
 * 2^-24)) and (c[i], s[i]) = its cos/sin of 2 pi (w >> 8) 2^-24, computed by the SAME device functions
 * gen_omega* use (device float outputs, caller-owned). Lets a test compare the generator's
 * transcendental steps with the oracle over all 2^24 codes. count = 0 is a no-op;
 * SHG_ERR_INVALID_VALUE for count < 0 or NULL pointers. */
shg_status_t shg_probe_boxmuller(const uint32_t *words, int64_t count, float *r, float *c, float *s,
                                 shg_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* SHGEMM_H_ */

/*
 * oracle.c — plain, slow, obviously-correct CPU oracle for the SHGEMM random projection.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library. The product path (paper_2304_04612_b200/) never
 * links, imports or calls it, and shares no code with it.
 *
 * What it computes, each function citing the passage it follows (PAPER.md = /root/reference/PAPER.md,
 * "P:n" = line n; OMEGA_SPEC.md is this repo's written reading of the Ω generator):
 *   orc_philox4x32_10   OMEGA_SPEC §1 (Philox4x32-10, Salmon et al. 2011)
 *   orc_f32_to_f16_rn   RN ties-to-even conversion, P:190 ("we use RN for the rounding")
 *   orc_omega_f16       OMEGA_SPEC §2-4; Gaussian Ω N(0,1) rounded RN to FP16,
 *                       sparse sign Ω (Eq 7, without sqrt(s))
 *   orc_split           Eqs 14-15: hi = toLow(A), lo = toLow((A - toF32(hi)) * 2^11)
 *   orc_gemm_y64        C_F64 of Fig 5: sum_l (double)A[i][l] * (double)Ω[l][j]
 *   orc_gemm_y32        naive single-precision GEMM (the "SGEMM" comparator of P:613):
 *                       acc = fmaf(A[i][l], Ω[l][j], acc), sequential in l
 *   orc_gemm_ysplit64   Eq 16 evaluated exactly in FP64: sum_l (hi + lo*2^-11) * Ω[l][j]
 *   orc_gemm_y64_f32b / orc_gemm_y32_f32b   the same two GEMMs with an FP32 B (k x n, column-major)
 *   orc_gemm_ytcec64    TCEC-SGEMM, Eq 9 in FP64:
 *                       sum_l [ahi*bhi + (alo*bhi + ahi*blo) * 2^-11], hi/lo from orc_split
 *   orc_f32_to_tf32_rn  RN ties-to-even to TF32 (e8m10), as FP32 bits with 13 zero low bits
 *   orc_split_tf32      Eqs 14-15 with toLow = TF32: the SHGEMM-TF32 variant of P:494-498
 *   orc_gemm_ysplit64_tf32  Eq 16 in FP64 with the TF32 hi/lo
 *   orc_unif_f32 / orc_gauss_f32   counter-based synthetic-input generator (same Philox, §6 of
 *                       OMEGA_SPEC), fp32 outputs, for regenerating sampled rows of device-made inputs
 *
 * Built with -O2 -ffp-contract=off (no -ffast-math): every float op is the IEEE op written.
 * Parity status: every function here is pinned by tests/test_oracle_*.py.
 */
#include <stdint.h>
#include <string.h>
#include <math.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ bit helpers */
static inline uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static inline float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

/* ------------------------------------------------------------------ Philox4x32-10 (OMEGA_SPEC §1) */
void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* ------------------------------------------------------------------ FP16 conversions (RN) */
/* Right-shift a non-negative integer by s bits, rounding to nearest, ties to even. */
static uint32_t rshift_rne(uint32_t v, int s) {
    if (s <= 0) return v;
    if (s >= 32) return 0;  /* only reached for v < 2^24 and s >= 26: always < half */
    uint32_t q = v >> s;
    uint32_t rem = v & ((1u << s) - 1u);
    uint32_t half = 1u << (s - 1);
    if (rem > half || (rem == half && (q & 1u))) q += 1u;
    return q;
}

uint16_t orc_f32_to_f16_rn(float f) {
    uint32_t x = f2u(f);
    uint16_t sign = (uint16_t)((x >> 16) & 0x8000u);
    uint32_t ax = x & 0x7FFFFFFFu;
    if (ax > 0x7F800000u) return (uint16_t)(sign | 0x7E00u);      /* NaN (payload not kept) */
    if (ax == 0x7F800000u) return (uint16_t)(sign | 0x7C00u);     /* inf */
    uint32_t E = ax >> 23;                 /* biased fp32 exponent */
    uint32_t mant = ax & 0x7FFFFFu;
    if (E == 0) return sign;               /* fp32 subnormal (< 2^-126): rounds to +-0 */
    uint32_t sig = mant | 0x800000u;       /* 24-bit significand, value = sig * 2^(E-150) */
    int e = (int)E - 127;                  /* unbiased exponent */
    if (e >= 16) return (uint16_t)(sign | 0x7C00u);
    if (e >= -14) {
        /* normal fp16 candidate: keep 11 significant bits */
        uint32_t q = rshift_rne(sig, 13);  /* in [2^10, 2^11] */
        int he = e + 15;
        if (q == (1u << 11)) { q >>= 1; he += 1; }
        if (he >= 31) return (uint16_t)(sign | 0x7C00u);
        return (uint16_t)(sign | ((uint32_t)he << 10) | (q & 0x3FFu));
    }
    /* subnormal fp16: value / 2^-24 = sig * 2^(E-150+24) = sig >> (126 - E) */
    int s = 126 - (int)E;
    uint32_t q = rshift_rne(sig, s);       /* may round up to 2^10 = smallest normal: encoding works */
    return (uint16_t)(sign | q);
}

float orc_f16_to_f32(uint16_t h) {
    uint32_t sign = ((uint32_t)h & 0x8000u) << 16;
    uint32_t he = ((uint32_t)h >> 10) & 0x1Fu;
    uint32_t hm = (uint32_t)h & 0x3FFu;
    if (he == 0x1F) return u2f(sign | 0x7F800000u | (hm << 13));
    if (he == 0) {
        if (hm == 0) return u2f(sign);
        /* subnormal: hm * 2^-24, exact in fp32 */
        float v = (float)hm * u2f(0x33800000u); /* 2^-24 */
        return u2f(sign | f2u(v));
    }
    return u2f(sign | ((he - 15 + 127) << 23) | (hm << 13));
}

/* ------------------------------------------------------------------ Box–Muller pieces (OMEGA_SPEC §3) */
#define SQRT2_F  0x3FB504F3u
#define LN2_F    0x3F317218u
#define L3_F     0x3F2AAAABu
#define L5_F     0x3ECCCCCDu
#define L7_F     0x3E924925u
#define L9_F     0x3E638E39u
#define S1_F     0x3FC90FDBu
#define S3_F     0xBF255DE7u
#define S5_F     0x3DA335E3u
#define S7_F     0xBB996966u
#define S9_F     0x39283C1Au
#define C2_F     0xBF9DE9E6u
#define C4_F     0x3E81E0F8u
#define C6_F     0xBCAAE9E4u
#define C8_F     0x3A70FA83u
#define C10_F    0xB7D368F9u

/* ln(na * 2^-24) for na in [1, 2^24] (OMEGA_SPEC §3.1). */
float orc_ln_spec(uint32_t na) {
    int e = 31 - __builtin_clz(na);
    float m = (float)na * u2f((uint32_t)(127 - e) << 23);    /* exact */
    if (m > u2f(SQRT2_F)) { m = m * 0.5f; e = e + 1; }
    float s = (m - 1.0f) / (m + 1.0f);
    float z = s * s;
    float p = fmaf(u2f(L9_F), z, u2f(L7_F));
    p = fmaf(p, z, u2f(L5_F));
    p = fmaf(p, z, u2f(L3_F));
    p = fmaf(p, z, 2.0f);
    float lnm = s * p;
    return fmaf((float)(e - 24), u2f(LN2_F), lnm);
}

/* radius sqrt(-2 ln u) from the first word of a pair */
float orc_radius_spec(uint32_t xa) {
    uint32_t na = (xa >> 8) + 1u;
    float L = orc_ln_spec(na);
    return sqrtf(-2.0f * L);
}

/* (cos θ, sin θ), θ = 2π (xb >> 8) 2^-24 (OMEGA_SPEC §3.2) */
void orc_sincos_spec(uint32_t xb, float *c_out, float *s_out) {
    uint32_t quad = xb >> 30;
    uint32_t f = (xb >> 8) & 0x3FFFFFu;
    int swap = f > (1u << 21);
    uint32_t h = swap ? ((1u << 22) - f) : f;
    float x = (float)h * u2f(0x34800000u);   /* 2^-22, exact */
    float x2 = x * x;
    float ps = fmaf(u2f(S9_F), x2, u2f(S7_F));
    ps = fmaf(ps, x2, u2f(S5_F));
    ps = fmaf(ps, x2, u2f(S3_F));
    ps = fmaf(ps, x2, u2f(S1_F));
    float sv = x * ps;
    float pc = fmaf(u2f(C10_F), x2, u2f(C8_F));
    pc = fmaf(pc, x2, u2f(C6_F));
    pc = fmaf(pc, x2, u2f(C4_F));
    pc = fmaf(pc, x2, u2f(C2_F));
    float cv = fmaf(pc, x2, 1.0f);
    float sg = swap ? cv : sv;
    float cg = swap ? sv : cv;
    float c, s;
    switch (quad) {
        case 0: c = cg; s = sg; break;
        case 1: c = -sg; s = cg; break;
        case 2: c = -cg; s = -sg; break;
        default: c = sg; s = -cg; break;
    }
    *c_out = c; *s_out = s;
}

/* Gaussian pair in fp32: (r cos θ, r sin θ) */
static void gauss_pair_f32(uint32_t xa, uint32_t xb, float *za, float *zb) {
    float r = orc_radius_spec(xa);
    float c, s;
    orc_sincos_spec(xb, &c, &s);
    *za = r * c;
    *zb = r * s;
}

/* ------------------------------------------------------------------ Ω (OMEGA_SPEC §2-5) */
enum { ORC_GAUSSIAN = 0, ORC_RADEMACHER = 1, ORC_SPARSE3 = 2, ORC_VERYSPARSE = 3 };

static void philox_block(uint64_t seed, uint32_t stream_id, uint64_t q, uint32_t j, uint32_t x[4]) {
    uint32_t ctr[4] = { (uint32_t)(q & 0xFFFFFFFFu), j, stream_id, (uint32_t)(q >> 32) };
    uint32_t key[2] = { (uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32) };
    orc_philox4x32_10(ctr, key, x);
}

uint32_t orc_sparse_threshold(int dist, int64_t k_total) {
    if (dist == ORC_SPARSE3) return 715827882u;                 /* floor(2^31 / 3) */
    if (dist == ORC_VERYSPARSE) {
        double s = sqrt((double)k_total);
        double t = floor(2147483648.0 / s);
        if (t > 2147483648.0) t = 2147483648.0;
        return (uint32_t)t;
    }
    return 0u;
}

/* Value of Ω[i][j] as FP16 bits. k_total only matters for the very-sparse threshold. */
uint16_t orc_omega_element(uint64_t seed, uint32_t stream_id, int dist, int64_t k_total,
                           uint64_t i, uint32_t j) {
    uint32_t x[4];
    philox_block(seed, stream_id, i >> 2, j, x);
    uint32_t w = (uint32_t)(i & 3u);
    if (dist == ORC_GAUSSIAN) {
        float za, zb;
        if (w < 2) gauss_pair_f32(x[0], x[1], &za, &zb);
        else       gauss_pair_f32(x[2], x[3], &za, &zb);
        return orc_f32_to_f16_rn((w & 1u) ? zb : za);
    }
    uint32_t xw = x[w];
    if (dist == ORC_RADEMACHER) return (xw >> 31) ? 0xBC00u : 0x3C00u;
    uint32_t T = orc_sparse_threshold(dist, k_total);
    if ((xw >> 1) < T) return (xw & 1u) ? 0xBC00u : 0x3C00u;
    return 0x0000u;
}

/* Column-major k x n: Omega[j*ldo + r] = Ω[row0 + r][j]. k_total = rows of the full Ω. */
void orc_omega_f16(int64_t k, int64_t n, uint64_t seed, uint32_t stream_id, int64_t row0,
                   int dist, int64_t k_total, uint16_t *omega, int64_t ldo) {
    #pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < n; ++j)
        for (int64_t r = 0; r < k; ++r)
            omega[j * ldo + r] = orc_omega_element(seed, stream_id, dist, k_total,
                                                   (uint64_t)(row0 + r), (uint32_t)j);
}

/* ------------------------------------------------------------------ split (Eqs 14-15) */
void orc_split(const float *a, int64_t count, uint16_t *hi, uint16_t *lo) {
    for (int64_t t = 0; t < count; ++t) {
        uint16_t h = orc_f32_to_f16_rn(a[t]);
        float hf = orc_f16_to_f32(h);
        float resid = a[t] - hf;              /* exact for |a| in the FP16 range */
        float scaled = resid * 2048.0f;       /* x 2^11, exact */
        hi[t] = h;
        lo[t] = orc_f32_to_f16_rn(scaled);
    }
}

/* ------------------------------------------------------------------ TF32 (SHGEMM-TF32) */
/* RN ties-to-even of an FP32 value to TF32 = e8m10: the sign and 8-bit exponent are kept,
 * the 23-bit fraction is rounded to its top 10 bits. On the FP32 encoding this is: drop the low 13
 * bits, and add one unit of bit 13 when the dropped part exceeds half of it, or equals half and
 * the kept part is odd. The carry may run into the exponent (correct: the next binade, or +-inf
 * from the largest finite binade). Infinities pass through; NaNs stay NaN (quiet bit set). */
uint32_t orc_f32_to_tf32_rn(float f) {
    uint32_t x = f2u(f);
    uint32_t sign = x & 0x80000000u, ax = x & 0x7FFFFFFFu;
    if (ax > 0x7F800000u) return x | 0x00400000u;          /* NaN */
    if (ax == 0x7F800000u) return x;                       /* inf */
    uint32_t dropped = ax & 0x1FFFu, kept = ax & ~0x1FFFu;
    if (dropped > 0x1000u || (dropped == 0x1000u && (kept & 0x2000u))) kept += 0x2000u;
    return sign | kept;
}

/* Eqs 14-15 with toLow = TF32: hi = RN_tf32(a), lo = RN_tf32((a - hi) * 2^11).
 * a - hi is exact (hi is a rounding of a to fewer bits of the same binade or the next one up) and
 * x 2^11 is an exact exponent shift, except at the TF32 overflow edge (hi = +-inf, lo = -+inf). */
void orc_split_tf32(const float *a, int64_t count, uint32_t *hi, uint32_t *lo) {
    for (int64_t t = 0; t < count; ++t) {
        uint32_t h = orc_f32_to_tf32_rn(a[t]);
        float resid = a[t] - u2f(h);
        float scaled = resid * 2048.0f;
        hi[t] = h;
        lo[t] = orc_f32_to_tf32_rn(scaled);
    }
}

/* ------------------------------------------------------------------ GEMMs (A row-major m x k, Ω column-major) */
/* Ω as a k x n row-major fp32/fp64 copy so the inner loop over j is contiguous. */
static float *omega_rows_f32(int64_t k, int64_t n, const uint16_t *omega, int64_t ldo) {
    float *w = (float *)malloc(sizeof(float) * (size_t)(k * n > 0 ? k * n : 1));
    for (int64_t l = 0; l < k; ++l)
        for (int64_t j = 0; j < n; ++j)
            w[l * n + j] = orc_f16_to_f32(omega[j * ldo + l]);
    return w;
}

/* Y64[i][j] = sum_{l=0}^{k-1} (double)A[i][l] * (double)Ω[l][j], l ascending (Fig 5's C_F64).
 * rows: optional list of nrows row indices of A (NULL = all m rows); Y row r <- A row rows[r]. */
void orc_gemm_y64(int64_t nrows, const int64_t *rows, int64_t n, int64_t k,
                  const float *A, int64_t lda, const uint16_t *omega, int64_t ldo,
                  double *Y, int64_t ldy) {
    float *w = omega_rows_f32(k, n, omega, ldo);
    #pragma omp parallel
    {
        double *acc = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
        #pragma omp for schedule(dynamic, 4)
        for (int64_t r = 0; r < nrows; ++r) {
            const float *a = A + (rows ? rows[r] : r) * lda;
            for (int64_t j = 0; j < n; ++j) acc[j] = 0.0;
            for (int64_t l = 0; l < k; ++l) {
                double al = (double)a[l];
                const float *wl = w + l * n;
                for (int64_t j = 0; j < n; ++j) acc[j] = acc[j] + al * (double)wl[j];
            }
            for (int64_t j = 0; j < n; ++j) Y[r * ldy + j] = acc[j];
        }
        free(acc);
    }
    free(w);
}

/* Y32[i][j]: acc = 0.0f; for l ascending: acc = fmaf(A[i][l], Ω[l][j], acc). Naive FP32. */
void orc_gemm_y32(int64_t nrows, const int64_t *rows, int64_t n, int64_t k,
                  const float *A, int64_t lda, const uint16_t *omega, int64_t ldo,
                  float *Y, int64_t ldy) {
    float *w = omega_rows_f32(k, n, omega, ldo);
    #pragma omp parallel
    {
        float *acc = (float *)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
        #pragma omp for schedule(dynamic, 4)
        for (int64_t r = 0; r < nrows; ++r) {
            const float *a = A + (rows ? rows[r] : r) * lda;
            for (int64_t j = 0; j < n; ++j) acc[j] = 0.0f;
            for (int64_t l = 0; l < k; ++l) {
                float al = a[l];
                const float *wl = w + l * n;
                for (int64_t j = 0; j < n; ++j) acc[j] = fmaf(al, wl[j], acc[j]);
            }
            for (int64_t j = 0; j < n; ++j) Y[r * ldy + j] = acc[j];
        }
        free(acc);
    }
    free(w);
}

/* Y_split64[i][j] = sum_l ((double)hi + (double)lo * 2^-11) * (double)Ω[l][j]  (Eq 16 in FP64) */
void orc_gemm_ysplit64(int64_t nrows, const int64_t *rows, int64_t n, int64_t k,
                       const float *A, int64_t lda, const uint16_t *omega, int64_t ldo,
                       double *Y, int64_t ldy) {
    float *w = omega_rows_f32(k, n, omega, ldo);
    #pragma omp parallel
    {
        double *acc = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
        #pragma omp for schedule(dynamic, 4)
        for (int64_t r = 0; r < nrows; ++r) {
            const float *a = A + (rows ? rows[r] : r) * lda;
            for (int64_t j = 0; j < n; ++j) acc[j] = 0.0;
            for (int64_t l = 0; l < k; ++l) {
                uint16_t h, lo;
                orc_split(&a[l], 1, &h, &lo);
                double rec = (double)orc_f16_to_f32(h) + (double)orc_f16_to_f32(lo) * (1.0 / 2048.0);
                const float *wl = w + l * n;
                for (int64_t j = 0; j < n; ++j) acc[j] = acc[j] + rec * (double)wl[j];
            }
            for (int64_t j = 0; j < n; ++j) Y[r * ldy + j] = acc[j];
        }
        free(acc);
    }
    free(w);
}

/* Eq 16 in FP64 with the TF32 split (SHGEMM-TF32) */
void orc_gemm_ysplit64_tf32(int64_t nrows, const int64_t *rows, int64_t n, int64_t k,
                       const float *A, int64_t lda, const uint16_t *omega, int64_t ldo,
                       double *Y, int64_t ldy) {
    float *w = omega_rows_f32(k, n, omega, ldo);
    #pragma omp parallel
    {
        double *acc = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
        #pragma omp for schedule(dynamic, 4)
        for (int64_t r = 0; r < nrows; ++r) {
            const float *a = A + (rows ? rows[r] : r) * lda;
            for (int64_t j = 0; j < n; ++j) acc[j] = 0.0;
            for (int64_t l = 0; l < k; ++l) {
                uint32_t h, lo;
                orc_split_tf32(&a[l], 1, &h, &lo);
                double rec = (double)u2f(h) + (double)u2f(lo) * (1.0 / 2048.0);
                const float *wl = w + l * n;
                for (int64_t j = 0; j < n; ++j) acc[j] = acc[j] + rec * (double)wl[j];
            }
            for (int64_t j = 0; j < n; ++j) Y[r * ldy + j] = acc[j];
        }
        free(acc);
    }
    free(w);
}

/* ------------------------------------------------------------------ synthetic fp32 inputs (OMEGA_SPEC §6) */
/* Element (i, l) of an m x k input, i = row, l = column, generated like Ω with l in the role of
 * the Philox row index: q = l >> 2, ctr = (q lo, i, stream_id, q hi). Gaussian: as §3 but kept in
 * fp32 (no FP16 rounding). Uniform [0,1): ((x_w >> 8) * 2^-24). */
float orc_gauss_f32(uint64_t seed, uint32_t stream_id, uint64_t i, uint64_t l) {
    uint32_t x[4];
    philox_block(seed, stream_id, l >> 2, (uint32_t)i, x);
    uint32_t w = (uint32_t)(l & 3u);
    float za, zb;
    if (w < 2) gauss_pair_f32(x[0], x[1], &za, &zb);
    else       gauss_pair_f32(x[2], x[3], &za, &zb);
    return (w & 1u) ? zb : za;
}

float orc_unif_f32(uint64_t seed, uint32_t stream_id, uint64_t i, uint64_t l) {
    uint32_t x[4];
    philox_block(seed, stream_id, l >> 2, (uint32_t)i, x);
    return (float)(x[l & 3u] >> 8) * u2f(0x33800000u);
}

/* Rows `rows[0..nrows)` of the synthetic matrix, each of length k, into out (row-major, ld = k). */
void orc_synth_rows_f32(int kind, uint64_t seed, uint32_t stream_id, int64_t nrows,
                        const int64_t *rows, int64_t k, float *out) {
    #pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < nrows; ++r)
        for (int64_t l = 0; l < k; ++l)
            out[r * k + l] = kind == 0 ? orc_gauss_f32(seed, stream_id, (uint64_t)rows[r], (uint64_t)l)
                                       : orc_unif_f32(seed, stream_id, (uint64_t)rows[r], (uint64_t)l);
}

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------------ batch helpers (for the pins) */
void orc_ln_spec_batch(const uint32_t *na, int64_t count, float *out) {
    #pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < count; ++t) out[t] = orc_ln_spec(na[t]);
}

void orc_radius_spec_batch(const uint32_t *xa, int64_t count, float *out) {
    #pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < count; ++t) out[t] = orc_radius_spec(xa[t]);
}

void orc_sincos_spec_batch(const uint32_t *xb, int64_t count, float *c, float *s) {
    #pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < count; ++t) orc_sincos_spec(xb[t], &c[t], &s[t]);
}

void orc_f32_to_f16_batch(const float *x, int64_t count, uint16_t *out) {
    #pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < count; ++t) out[t] = orc_f32_to_f16_rn(x[t]);
}

/* Gaussian fp32 pre-rounding values z for column j, rows row0..row0+count-1 (stream, seed). */
void orc_gauss_column_f32(uint64_t seed, uint32_t stream_id, uint32_t j, int64_t row0,
                          int64_t count, float *out) {
    #pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < count; ++t) {
        uint64_t i = (uint64_t)(row0 + t);
        uint32_t x[4];
        philox_block(seed, stream_id, i >> 2, j, x);
        uint32_t w = (uint32_t)(i & 3u);
        float za, zb;
        if (w < 2) gauss_pair_f32(x[0], x[1], &za, &zb);
        else       gauss_pair_f32(x[2], x[3], &za, &zb);
        out[t] = (w & 1u) ? zb : za;
    }
}

/* ------------------------------------------------------------------ FP32 x FP32 GEMMs (TCEC-SGEMM) */
/* B: k x n FP32, column-major (element (l, j) at B[j * ldb + l]). Products of two FP32 values are
 * exact in binary64 (24 + 24 significant bits <= 53). */
static double *b_rows_f64(int64_t k, int64_t n, const float *B, int64_t ldb) {
    double *w = (double *)malloc(sizeof(double) * (size_t)(k * n > 0 ? k * n : 1));
    for (int64_t l = 0; l < k; ++l)
        for (int64_t j = 0; j < n; ++j) w[l * n + j] = (double)B[j * ldb + l];
    return w;
}

void orc_gemm_y64_f32b(int64_t nrows, const int64_t *rows, int64_t n, int64_t k,
                       const float *A, int64_t lda, const float *B, int64_t ldb, double *Y, int64_t ldy) {
    double *w = b_rows_f64(k, n, B, ldb);
    #pragma omp parallel
    {
        double *acc = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
        #pragma omp for schedule(dynamic, 4)
        for (int64_t r = 0; r < nrows; ++r) {
            const float *a = A + (rows ? rows[r] : r) * lda;
            for (int64_t j = 0; j < n; ++j) acc[j] = 0.0;
            for (int64_t l = 0; l < k; ++l) {
                double al = (double)a[l];
                const double *wl = w + l * n;
                for (int64_t j = 0; j < n; ++j) acc[j] = acc[j] + al * wl[j];
            }
            for (int64_t j = 0; j < n; ++j) Y[r * ldy + j] = acc[j];
        }
        free(acc);
    }
    free(w);
}

/* naive FP32: acc = fmaf(A[i][l], B[l][j], acc), l ascending */
void orc_gemm_y32_f32b(int64_t nrows, const int64_t *rows, int64_t n, int64_t k,
                       const float *A, int64_t lda, const float *B, int64_t ldb, float *Y, int64_t ldy) {
    float *w = (float *)malloc(sizeof(float) * (size_t)(k * n > 0 ? k * n : 1));
    for (int64_t l = 0; l < k; ++l)
        for (int64_t j = 0; j < n; ++j) w[l * n + j] = B[j * ldb + l];
    #pragma omp parallel
    {
        float *acc = (float *)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
        #pragma omp for schedule(dynamic, 4)
        for (int64_t r = 0; r < nrows; ++r) {
            const float *a = A + (rows ? rows[r] : r) * lda;
            for (int64_t j = 0; j < n; ++j) acc[j] = 0.0f;
            for (int64_t l = 0; l < k; ++l) {
                float al = a[l];
                const float *wl = w + l * n;
                for (int64_t j = 0; j < n; ++j) acc[j] = fmaf(al, wl[j], acc[j]);
            }
            for (int64_t j = 0; j < n; ++j) Y[r * ldy + j] = acc[j];
        }
        free(acc);
    }
    free(w);
}

/* TCEC-SGEMM (Eqs 5-9): both operands split by Eqs 14-15's FP16 split (orc_split),
 * C ~ A_low B_low + (dA_low B_low + A_low dB_low) 2^-11, each term evaluated exactly in FP64 and
 * summed over l ascending. The dA_low dB_low term is absent (Eq 9). */
void orc_gemm_ytcec64(int64_t nrows, const int64_t *rows, int64_t n, int64_t k,
                      const float *A, int64_t lda, const float *B, int64_t ldb, double *Y, int64_t ldy) {
    double *bh = (double *)malloc(sizeof(double) * (size_t)(k * n > 0 ? k * n : 1));
    double *bl = (double *)malloc(sizeof(double) * (size_t)(k * n > 0 ? k * n : 1));
    for (int64_t l = 0; l < k; ++l)
        for (int64_t j = 0; j < n; ++j) {
            uint16_t h, lo;
            orc_split(&B[j * ldb + l], 1, &h, &lo);
            bh[l * n + j] = (double)orc_f16_to_f32(h);
            bl[l * n + j] = (double)orc_f16_to_f32(lo);
        }
    #pragma omp parallel
    {
        double *acc = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
        #pragma omp for schedule(dynamic, 4)
        for (int64_t r = 0; r < nrows; ++r) {
            const float *a = A + (rows ? rows[r] : r) * lda;
            for (int64_t j = 0; j < n; ++j) acc[j] = 0.0;
            for (int64_t l = 0; l < k; ++l) {
                uint16_t h, lo;
                orc_split(&a[l], 1, &h, &lo);
                double ah = (double)orc_f16_to_f32(h), al = (double)orc_f16_to_f32(lo);
                for (int64_t j = 0; j < n; ++j) {
                    double hh = ah * bh[l * n + j];
                    double corr = al * bh[l * n + j] + ah * bl[l * n + j];
                    acc[j] = acc[j] + (hh + corr * (1.0 / 2048.0));
                }
            }
            for (int64_t j = 0; j < n; ++j) Y[r * ldy + j] = acc[j];
        }
        free(acc);
    }
    free(bh);
    free(bl);
}

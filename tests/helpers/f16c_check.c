/* Exhaustive pin of the oracle's software FP32->FP16 RN conversion against the x86 F16C
 * hardware instruction vcvtps2ph (round-to-nearest-even), over all 2^32 FP32 bit patterns.
 * Test helper only; links against oracle/liboracle.so. All NaN outputs count as equal. */
#include <stdint.h>
#include <string.h>
#include <immintrin.h>

extern uint16_t orc_f32_to_f16_rn(float f);

static int is_nan16(uint16_t h) { return (h & 0x7C00u) == 0x7C00u && (h & 0x3FFu) != 0; }

/* Returns the number of mismatches in [lo, hi) (hi exclusive, as uint64). First mismatch in *first. */
uint64_t f16c_mismatches(uint64_t lo, uint64_t hi, uint32_t *first) {
    uint64_t bad = 0;
    uint32_t firstbad = 0;
    #pragma omp parallel for reduction(+:bad) schedule(static)
    for (uint64_t u = lo; u < hi; ++u) {
        uint32_t bits = (uint32_t)u;
        float f;
        memcpy(&f, &bits, 4);
        uint16_t ref = (uint16_t)_cvtss_sh(f, _MM_FROUND_TO_NEAREST_INT);
        uint16_t got = orc_f32_to_f16_rn(f);
        if (got != ref && !(is_nan16(got) && is_nan16(ref))) {
            bad++;
            firstbad = bits;
        }
    }
    *first = firstbad;
    return bad;
}

/* Exhaustive pin of the oracle's FP32 -> TF32 RN conversion (orc_f32_to_tf32_rn) by an independent
 * route: TF32 and FP16 both keep 10 fraction bits, so for a NORMAL FP32 x = y * 2^e (y in [1, 2))
 * RN_tf32(x) = RN_f16(y) * 2^e, with RN_f16 done by the F16C instruction and the scalings exact
 * (ldexpf; an overflow to 2^128 gives +-inf, as RN requires). FP32 subnormals x = q * 2^-149 round
 * at the fixed quantum 2^-136: RN_tf32(x) = round_half_even(q / 2^13) * 2^-136, done in integers.
 * Zeros and infinities map to themselves; NaN must stay NaN. */
extern uint32_t orc_f32_to_tf32_rn(float f);
#include <math.h>

static uint32_t tf32_ref(uint32_t bits) {
    uint32_t sign = bits & 0x80000000u, ax = bits & 0x7FFFFFFFu;
    if (ax >= 0x7F800000u) return bits;                     /* inf / NaN (NaN compared by class) */
    if (ax == 0) return bits;
    if (ax < 0x00800000u) {                                  /* subnormal: q * 2^-149 */
        uint32_t q = ax, hi = q >> 13, rem = q & 0x1FFFu;
        if (rem > 0x1000u || (rem == 0x1000u && (hi & 1u))) hi += 1u;
        return sign | (hi << 13);
    }
    float x, r;
    memcpy(&x, &ax, 4);
    int e;
    float y = frexpf(x, &e);                                 /* x = y * 2^e, y in [0.5, 1) */
    y = ldexpf(y, 1); e -= 1;                                /* y in [1, 2) */
    uint16_t h = (uint16_t)_cvtss_sh(y, _MM_FROUND_TO_NEAREST_INT);
    float hy = _cvtsh_ss(h);
    r = ldexpf(hy, e);
    uint32_t rb;
    memcpy(&rb, &r, 4);
    return sign | rb;
}

uint64_t tf32_mismatches(uint64_t lo, uint64_t hi, uint32_t *first) {
    uint64_t bad = 0;
    uint32_t firstbad = 0;
    #pragma omp parallel for reduction(+:bad) schedule(static)
    for (uint64_t u = lo; u < hi; ++u) {
        uint32_t bits = (uint32_t)u;
        float f;
        memcpy(&f, &bits, 4);
        uint32_t ref = tf32_ref(bits), got = orc_f32_to_tf32_rn(f);
        int nan_ref = (ref & 0x7FFFFFFFu) > 0x7F800000u, nan_got = (got & 0x7FFFFFFFu) > 0x7F800000u;
        if (nan_ref || nan_got) {
            if (nan_ref != nan_got) { bad++; firstbad = bits; }
        } else if (got != ref) {
            bad++;
            firstbad = bits;
        }
    }
    *first = firstbad;
    return bad;
}

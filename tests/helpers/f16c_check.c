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

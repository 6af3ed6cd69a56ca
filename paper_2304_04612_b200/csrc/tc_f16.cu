// tc_f16.cu — instantiations of the tcgen05 mainloop for SHGEMM-FP16 with K-major A (all BN x
// {single CTA, CTA pair}); M-major A is in tc_f16_mm.cu. Separate translation units so the build
// compiles them in parallel.
#include "internal.cuh"

namespace shg_api {

shg_status_t dispatch_tc_f16(int bn, bool mmajor, bool pair, const CUtensorMap& a, const CUtensorMap& b0,
                             const CUtensorMap& b1, const shg::KParams& kp, int grid, cudaStream_t s) {
    if (!valid_bn(bn) || (pair && !pair_ok(bn))) return SHG_ERR_INVALID_VALUE;
    if (mmajor) return dispatch_tc_f16_mmajor(bn, pair, a, b0, b1, kp, grid, s);
    return pair ? dispatch_bn<false, true, false>(bn, a, b0, b1, kp, grid, s)
                : dispatch_bn<false, false, false>(bn, a, b0, b1, kp, grid, s);
}

}  // namespace shg_api

// tc_tf32.cu — instantiations of the tcgen05 mainloop for SHGEMM-TF32 (all BN x {K-major,
// M-major} x {single CTA, CTA pair}); a separate translation unit so the build compiles it in parallel.
#include "internal.cuh"

namespace shg_api {

shg_status_t dispatch_tc_tf32(int bn, bool mmajor, bool pair, const CUtensorMap& a, const CUtensorMap& b0,
                             const CUtensorMap& b1, const shg::KParams& kp, int grid, cudaStream_t s) {
    if (!valid_bn(bn) || (pair && !pair_ok(bn))) return SHG_ERR_INVALID_VALUE;
    if (mmajor) return pair ? dispatch_bn<true, true, true>(bn, a, b0, b1, kp, grid, s)
                            : dispatch_bn<true, false, true>(bn, a, b0, b1, kp, grid, s);
    return pair ? dispatch_bn<false, true, true>(bn, a, b0, b1, kp, grid, s)
                : dispatch_bn<false, false, true>(bn, a, b0, b1, kp, grid, s);
}

}  // namespace shg_api

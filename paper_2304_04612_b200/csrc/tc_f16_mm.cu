// tc_f16_mm.cu — SHGEMM-FP16 mainloop instantiations for M-major A (shgemm_at, last-mode
// unfoldings of project()); see tc_f16.cu.
#include "internal.cuh"

namespace shg_api {

shg_status_t dispatch_tc_f16_mmajor(int bn, bool pair, const CUtensorMap& a, const CUtensorMap& b0,
                                    const CUtensorMap& b1, const shg::KParams& kp, int grid, cudaStream_t s) {
    return pair ? dispatch_bn<true, true, false>(bn, a, b0, b1, kp, grid, s)
                : dispatch_bn<true, false, false>(bn, a, b0, b1, kp, grid, s);
}

}  // namespace shg_api

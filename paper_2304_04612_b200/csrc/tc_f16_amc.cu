// tc_f16_amc.cu — SHGEMM-FP16 K-major CTA-pair mainloop with each A stage multicast to the NPA = 2 / 4
// pairs of a cluster that cover NPA N tiles of one m-block (shgemm_sm100_kernel<..., NPA>, DESIGN.md §5
// "A read once"); its own translation unit so the build compiles it in parallel.
#include "internal.cuh"

namespace shg_api {

namespace {
template <int NPA>
shg_status_t dispatch(int bn, const CUtensorMap& a, const CUtensorMap& b0, const CUtensorMap& b1,
                      const shg::KParams& kp, int grid, cudaStream_t s) {
    switch (bn) {
        case 128: return launch_tc<128, false, true, false, false, false, NPA>(a, b0, b1, kp, grid, s);
        case 192: return launch_tc<192, false, true, false, false, false, NPA>(a, b0, b1, kp, grid, s);
        case 256: return launch_tc<256, false, true, false, false, false, NPA>(a, b0, b1, kp, grid, s);
        default: return SHG_ERR_INVALID_VALUE;
    }
}
}  // namespace

shg_status_t dispatch_tc_f16_amc(int bn, int npa, const CUtensorMap& a, const CUtensorMap& b0, const CUtensorMap& b1,
                                 const shg::KParams& kp, int grid, cudaStream_t s) {
    if (npa == 2) return dispatch<2>(bn, a, b0, b1, kp, grid, s);
    if (npa == 4) return dispatch<4>(bn, a, b0, b1, kp, grid, s);
    return SHG_ERR_INVALID_VALUE;
}

}  // namespace shg_api

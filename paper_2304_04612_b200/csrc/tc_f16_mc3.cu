// tc_f16_mc3.cu — SHGEMM-FP16 CTA-pair mainloop with every Omega stage multicast to 3 pairs of a
// cluster (shgemm_sm100_kernel<..., NP = 2>); its own translation unit so the build compiles it in parallel.
#include "internal.cuh"

namespace shg_api {

namespace {
template <bool MMAJOR>
shg_status_t dispatch(int bn, const CUtensorMap& a, const CUtensorMap& b0, const CUtensorMap& b1,
                      const shg::KParams& kp, int grid, cudaStream_t s) {
    switch (bn) {
        case 128: return launch_tc<128, MMAJOR, true, false, false, 3>(a, b0, b1, kp, grid, s);
        case 144: return launch_tc<144, MMAJOR, true, false, false, 3>(a, b0, b1, kp, grid, s);
        case 160: return launch_tc<160, MMAJOR, true, false, false, 3>(a, b0, b1, kp, grid, s);
        case 192: return launch_tc<192, MMAJOR, true, false, false, 3>(a, b0, b1, kp, grid, s);
        case 224: return launch_tc<224, MMAJOR, true, false, false, 3>(a, b0, b1, kp, grid, s);
        case 256: return launch_tc<256, MMAJOR, true, false, false, 3>(a, b0, b1, kp, grid, s);
        default: return SHG_ERR_INVALID_VALUE;
    }
}
}  // namespace

shg_status_t dispatch_tc_f16_mc3(int bn, bool mmajor, const CUtensorMap& a, const CUtensorMap& b0,
                                 const CUtensorMap& b1, const shg::KParams& kp, int grid, cudaStream_t s) {
    return mmajor ? dispatch<true>(bn, a, b0, b1, kp, grid, s) : dispatch<false>(bn, a, b0, b1, kp, grid, s);
}

}  // namespace shg_api

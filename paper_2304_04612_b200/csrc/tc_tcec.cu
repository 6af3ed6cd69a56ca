// tc_tcec.cu — instantiations of the tcgen05 mainloop for TCEC-SGEMM (Eqs 5-9):
// single CTAs for BN <= 128 and CTA pairs for BN >= 128, K-major and M-major A.
#include "internal.cuh"

namespace shg_api {

namespace {

template <bool MMAJOR>
shg_status_t dispatch_single(int bn, const CUtensorMap& a, const CUtensorMap& b0, const CUtensorMap& b1,
                             const shg::KParams& kp, int grid, cudaStream_t s) {
    switch (bn) {
        case 32: return launch_tc<32, MMAJOR, false, false, true>(a, b0, b1, kp, grid, s);
        case 64: return launch_tc<64, MMAJOR, false, false, true>(a, b0, b1, kp, grid, s);
        case 96: return launch_tc<96, MMAJOR, false, false, true>(a, b0, b1, kp, grid, s);
        case 128: return launch_tc<128, MMAJOR, false, false, true>(a, b0, b1, kp, grid, s);
        default: return SHG_ERR_INVALID_VALUE;
    }
}

template <bool MMAJOR>
shg_status_t dispatch_pair(int bn, const CUtensorMap& a, const CUtensorMap& b0, const CUtensorMap& b1,
                           const shg::KParams& kp, int grid, cudaStream_t s) {
    switch (bn) {
        case 128: return launch_tc<128, MMAJOR, true, false, true>(a, b0, b1, kp, grid, s);
        case 144: return launch_tc<144, MMAJOR, true, false, true>(a, b0, b1, kp, grid, s);
        case 160: return launch_tc<160, MMAJOR, true, false, true>(a, b0, b1, kp, grid, s);
        case 192: return launch_tc<192, MMAJOR, true, false, true>(a, b0, b1, kp, grid, s);
        case 224: return launch_tc<224, MMAJOR, true, false, true>(a, b0, b1, kp, grid, s);
        case 256: return launch_tc<256, MMAJOR, true, false, true>(a, b0, b1, kp, grid, s);
        case 272: return launch_tc<272, MMAJOR, true, false, true>(a, b0, b1, kp, grid, s);
        case 288: return launch_tc<288, MMAJOR, true, false, true>(a, b0, b1, kp, grid, s);
        default: return SHG_ERR_INVALID_VALUE;
    }
}

}  // namespace

shg_status_t dispatch_tc_tcec(int bn, bool mmajor, bool pair, const CUtensorMap& a, const CUtensorMap& b0,
                              const CUtensorMap& b1, const shg::KParams& kp, int grid, cudaStream_t s) {
    if (pair) return mmajor ? dispatch_pair<true>(bn, a, b0, b1, kp, grid, s) : dispatch_pair<false>(bn, a, b0, b1, kp, grid, s);
    return mmajor ? dispatch_single<true>(bn, a, b0, b1, kp, grid, s) : dispatch_single<false>(bn, a, b0, b1, kp, grid, s);
}

}  // namespace shg_api

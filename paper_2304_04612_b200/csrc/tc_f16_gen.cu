// tc_f16_gen.cu — SHGEMM-FP16 single-CTA mainloop with cooperative in-kernel Omega generation
// (shgemm_sm100_kernel<..., OMGEN = true>, used by project() for the unfoldings); its own translation
// unit so the build compiles it in parallel.
#include "internal.cuh"

namespace shg_api {

namespace {
template <bool MMAJOR>
shg_status_t dispatch(int bn, const CUtensorMap& a, const CUtensorMap& b0, const CUtensorMap& b1,
                      const shg::KParams& kp, int grid, cudaStream_t s) {
    switch (bn) {
        case 32: return launch_tc<32, MMAJOR, false, false, false, true>(a, b0, b1, kp, grid, s);
        case 64: return launch_tc<64, MMAJOR, false, false, false, true>(a, b0, b1, kp, grid, s);
        case 96: return launch_tc<96, MMAJOR, false, false, false, true>(a, b0, b1, kp, grid, s);
        case 128: return launch_tc<128, MMAJOR, false, false, false, true>(a, b0, b1, kp, grid, s);
        default: return SHG_ERR_INVALID_VALUE;
    }
}
}  // namespace

shg_status_t dispatch_tc_f16_gen(int bn, bool mmajor, const CUtensorMap& a, const CUtensorMap& b0,
                                 const CUtensorMap& b1, const shg::KParams& kp, int grid, cudaStream_t s) {
    return mmajor ? dispatch<true>(bn, a, b0, b1, kp, grid, s) : dispatch<false>(bn, a, b0, b1, kp, grid, s);
}

}  // namespace shg_api

// test support: number of Omega tiles the stagers' fallback has generated in this process
extern "C" uint64_t shg_inkernel_omega_fallbacks(void) {
    unsigned long long v = 0;
    if (cudaMemcpyFromSymbol(&v, shg::g_om_helped, sizeof(v)) != cudaSuccess) return ~0ull;
    return v;
}

// dispatch.cu — picks the kernel instantiation for the robot's DoF: exact-N
// kernels (no per-joint guards) for the benchmarked chains n = 7, 8, 14 and
// the paper's Table II DoFs 12, 18, 24, and NMAX-bounded kernels (uniform
// `j < n` guards) for every other n <= 32.
#include <cstdlib>

#include "hjcd_internal.h"

namespace hjcd {

int poccd_nmax(int n) {   // must match launch_poccd's choice below
    switch (n) {
        case 7: case 8: case 12: case 14: case 18: case 24: return n;
        default: return n <= 8 ? 8 : (n <= 16 ? 16 : 32);
    }
}

// K17: the two-seeds-per-thread packed kernel for the stop-rule launch with
// fused seeds at n <= 8 (HJCD_POCCD_X2=0 in the environment selects the
// one-seed-per-thread kernel, for A/B measurements)
static bool use_x2(int n) {
    static const int env = [] {
        const char* e = std::getenv("HJCD_POCCD_X2");
        return e ? std::atoi(e) : 1;
    }();
    return env != 0 && n <= 8;
}

bool poccd_uses_x2(int n, bool ccd_early_exit) { return ccd_early_exit && use_x2(n); }

int poccd_cluster_ctas(int M, int n) {
    int nt, CL;
    if (use_x2(n)) texit_shape_x2(M, nt, CL);
    else texit_shape(M, poccd_nmax(n), nt, CL);
    return CL;
}

cudaError_t launch_poccd(const DevRobot& rb, const DevCfg& c, const float* targets, int T,
                         const float* seeds, float* theta, float* cost, float* ep, float* eo,
                         int32_t* iters, cudaStream_t s, TraceOut trace, uint32_t* ready) {
    if (c.ccd_early_exit && !seeds && use_x2(rb.n)) {
        if (rb.n == 7) return launch_poccd_x2_t<7, true>(rb, c, targets, T, theta, cost, ep, eo, iters, trace, ready, s);
        if (rb.n == 8) return launch_poccd_x2_t<8, true>(rb, c, targets, T, theta, cost, ep, eo, iters, trace, ready, s);
        return launch_poccd_x2_t<8, false>(rb, c, targets, T, theta, cost, ep, eo, iters, trace, ready, s);
    }
    switch (rb.n) {   // exact instantiations for the benchmarked chains, bounded ones otherwise
        case 7: return launch_poccd_t<7, true>(rb, c, targets, T, seeds, theta, cost, ep, eo, iters, trace, ready, s);
        case 8: return launch_poccd_t<8, true>(rb, c, targets, T, seeds, theta, cost, ep, eo, iters, trace, ready, s);
        case 12: return launch_poccd_t<12, true>(rb, c, targets, T, seeds, theta, cost, ep, eo, iters, trace, ready, s);
        case 14: return launch_poccd_t<14, true>(rb, c, targets, T, seeds, theta, cost, ep, eo, iters, trace, ready, s);
        case 18: return launch_poccd_t<18, true>(rb, c, targets, T, seeds, theta, cost, ep, eo, iters, trace, ready, s);
        case 24: return launch_poccd_t<24, true>(rb, c, targets, T, seeds, theta, cost, ep, eo, iters, trace, ready, s);
        default: break;
    }
    if (rb.n <= 8) return launch_poccd_t<8, false>(rb, c, targets, T, seeds, theta, cost, ep, eo, iters, trace, ready, s);
    if (rb.n <= 16) return launch_poccd_t<16, false>(rb, c, targets, T, seeds, theta, cost, ep, eo, iters, trace, ready, s);
    return launch_poccd_t<32, false>(rb, c, targets, T, seeds, theta, cost, ep, eo, iters, trace, ready, s);
}

template <class T>
cudaError_t launch_pjik_coop(const DevRobotT<T>& rb, const DevCfg& c, const float* targets, int T_,
                             const float* seeds, T* theta, T* ep, T* eo, int32_t* counts, int32_t* iters,
                             cudaStream_t s, const StageLink& link) {
    if (c.copies * c.K > 256 || 2 * c.A + 2 > 64) return cudaErrorInvalidConfiguration;
    switch (rb.n) {   // exact instantiations for the benchmarked chains, bounded ones otherwise
        case 7: return launch_coop_t<T, 7, true>(rb, c, targets, T_, seeds, theta, ep, eo, counts, iters, s, link);
        case 8: return launch_coop_t<T, 8, true>(rb, c, targets, T_, seeds, theta, ep, eo, counts, iters, s, link);
        case 14: return launch_coop_t<T, 14, true>(rb, c, targets, T_, seeds, theta, ep, eo, counts, iters, s, link);
        default: break;
    }
    if constexpr (sizeof(T) == 4) {   // Table II DoFs (fp32 polish only)
        switch (rb.n) {
            case 12: return launch_coop_t<T, 12, true>(rb, c, targets, T_, seeds, theta, ep, eo, counts, iters, s, link);
            case 18: return launch_coop_t<T, 18, true>(rb, c, targets, T_, seeds, theta, ep, eo, counts, iters, s, link);
            case 24: return launch_coop_t<T, 24, true>(rb, c, targets, T_, seeds, theta, ep, eo, counts, iters, s, link);
            default: break;
        }
    }
    if (rb.n <= 8) return launch_coop_t<T, 8, false>(rb, c, targets, T_, seeds, theta, ep, eo, counts, iters, s, link);
    if (rb.n <= 16) return launch_coop_t<T, 16, false>(rb, c, targets, T_, seeds, theta, ep, eo, counts, iters, s, link);
    return launch_coop_t<T, 32, false>(rb, c, targets, T_, seeds, theta, ep, eo, counts, iters, s, link);
}
template cudaError_t launch_pjik_coop<float>(const DevRobotT<float>&, const DevCfg&, const float*, int, const float*,
                                             float*, float*, float*, int32_t*, int32_t*, cudaStream_t,
                                             const StageLink&);

cudaError_t launch_pjik64(const DevRobotT<double>& rb, const DevCfg& c, const float* targets, int T,
                          const float* seeds, double* theta, double* ep, double* eo, int32_t* counts,
                          int32_t* iters, cudaStream_t s) {
    return launch_pjik_coop<double>(rb, c, targets, T, seeds, theta, ep, eo, counts, iters, s, StageLink());
}

cudaError_t launch_pjik(const DevRobot& rb, const DevCfg& c, const float* targets, int T,
                        const float* seeds, float* theta, float* ep, float* eo, int32_t* counts,
                        int32_t* iters, cudaStream_t s, const StageLink& link) {
    // one CTA per target, warp-cooperative cascade (pjik_coop.cuh), for both
    // the per-target stop rule and the per-seed break
    return launch_pjik_coop(rb, c, targets, T, seeds, theta, ep, eo, counts, iters, s, link);
}

cudaError_t launch_ccd(const DevRobot& rb, const DevCfg& c, const float* targets, int T, const float* seeds,
                       float* theta, float* ep, int32_t* iters, cudaStream_t s) {
    if (rb.n == 7) return launch_ccd_t<7, true>(rb, c, targets, T, seeds, theta, ep, iters, s);
    if (rb.n <= 8) return launch_ccd_t<8, false>(rb, c, targets, T, seeds, theta, ep, iters, s);
    if (rb.n <= 16) return launch_ccd_t<16, false>(rb, c, targets, T, seeds, theta, ep, iters, s);
    return launch_ccd_t<32, false>(rb, c, targets, T, seeds, theta, ep, iters, s);
}

}  // namespace hjcd

// hjcd_internal.h — structures shared by the host C-ABI code and the kernels
// of libhjcd.so (never by the oracle).  The robot and the config travel to the
// device as __grid_constant__ kernel parameters, i.e. in the constant bank:
// every lane reads the same joint at the same time (uniform loop index), so
// each access is a broadcast and FFMAs take the constants as direct operands.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/hjcd.h"

namespace hjcd {

// One DoF joint after canonicalisation (host, fp64 -> S):
//   T_i = T_{i-1} * F_i * Rz(theta_i)        (revolute)
//   T_i = T_{i-1} * F_i * Tz(theta_i)        (prismatic)
// F_i = [R | t] (R row-major).  P_i = translation of T_{i-1} F_i, z_i = its
// third rotation column, which equal the paper's P_i, z_i (Eq. 7).
template <class S>
struct DevJointT {
    S R[9];
    S t[3];
    S lo, hi;
    int32_t type;  // HJCD_REVOLUTE / HJCD_PRISMATIC
    int32_t pad;
};

template <class S>
struct DevRobotT {
    int32_t n;
    uint32_t pmask;      // bit j set: DoF joint j is prismatic
    int32_t pad[2];
    DevJointT<S> j[HJCD_MAX_DOF];
    S eeR[9];
    S eet[3];
};
using DevJoint = DevJointT<float>;
using DevRobot = DevRobotT<float>;   // the fp32 kernels; DevRobotT<double> for the fp64 polish

struct DevCfg {
    int32_t M, K, B, ccd_iters, lm_iters, A, copies, repl_noise_all, target_early_exit, ccd_early_exit;
    float eps_p_coarse, eps_o_coarse, eps_p_fine, eps_o_fine;
    float gamma, delta0, delta_rho, delta_min;
    float sigma_ccd, sigma_rep, sigma_lm;
    float lambda, d_floor, R, inv_beta;
    float w_p, w_o, succ_p, succ_o, tau_deg;
    uint32_t key0, key1;
    int64_t tid_offset;
};

// Philox purposes (R30)
enum : uint32_t { P_INIT = 1, P_PERTURB = 2, P_REPL = 3, P_PJPERT = 4 };

// per-instantiation launchers (templates in poccd.cuh / pjik_coop.cuh,
// explicitly instantiated one or two per inst_*.cu so nvcc runs in parallel)
template <int NMAX, bool EXACT>
cudaError_t launch_poccd_t(const DevRobot& rb, const DevCfg& c, const float* targets, int T,
                           const float* seeds, float* theta, float* cost, float* ep, float* eo,
                           int32_t* iters, uint32_t* trace, cudaStream_t s);
template <int NMAX, bool EXACT>
cudaError_t launch_ccd_t(const DevRobot& rb, const DevCfg& c, const float* targets, int T, const float* seeds,
                         float* theta, float* ep, int32_t* iters, cudaStream_t s);
template <class T, int NMAX, bool EXACT>
cudaError_t launch_coop_t(const DevRobotT<T>& rb, const DevCfg& c, const float* targets, int T_,
                          const float* seeds, T* theta, T* ep, T* eo, int32_t* counts, int32_t* iters,
                          cudaStream_t s);

// launchers (dispatch.cu, select.cu); all asynchronous on `s`
cudaError_t launch_fk(const DevRobot& rb, const float* q, int N, float* pose7, float* jac,
                      cudaStream_t s);
cudaError_t launch_poccd(const DevRobot& rb, const DevCfg& c, const float* targets, int T,
                         const float* seeds, float* theta, float* cost, float* ep, float* eo,
                         int32_t* iters, cudaStream_t s, uint32_t* trace = nullptr);
cudaError_t launch_ccd(const DevRobot& rb, const DevCfg& c, const float* targets, int T, const float* seeds,
                       float* theta, float* ep, int32_t* iters, cudaStream_t s);
cudaError_t launch_select_replicate(const DevRobot& rb, const DevCfg& c, const float* cost,
                                    const float* theta, int T, float* seeds, int32_t* kept,
                                    cudaStream_t s);
cudaError_t launch_pjik(const DevRobot& rb, const DevCfg& c, const float* targets, int T,
                        const float* seeds, float* theta, float* ep, float* eo, int32_t* counts,
                        int32_t* iters, cudaStream_t s);
template <class T>
cudaError_t launch_pjik_coop(const DevRobotT<T>& rb, const DevCfg& c, const float* targets, int T_,
                             const float* seeds, T* theta, T* ep, T* eo, int32_t* counts, int32_t* iters,
                             cudaStream_t s);
cudaError_t launch_select_topn(const DevRobot& rb, const DevCfg& c, const float* targets, int T, const float* theta,
                               const float* ep_all, const float* eo_all, int N, float* q_out, float* pos_err,
                               float* ori_err, int32_t* idx, int32_t* status, cudaStream_t s);
cudaError_t launch_mmd(const float* X, int N, const float* Y, int N2, int n, int T, float* mmd2, float* bw,
                       cudaStream_t s);
template <class T>
cudaError_t launch_select_best(const DevRobot& rb, const DevCfg& c, const float* targets, int T_,
                               const T* theta, const T* ep_all, const T* eo_all, T* q_out, T* pos_err,
                               T* ori_err, int32_t* status, cudaStream_t s);
// fp64 polish: the same PJ-IK on DevRobotT<double>
cudaError_t launch_pjik64(const DevRobotT<double>& rb, const DevCfg& c, const float* targets, int T,
                          const float* seeds, double* theta, double* ep, double* eo, int32_t* counts,
                          int32_t* iters, cudaStream_t s);

}  // namespace hjcd

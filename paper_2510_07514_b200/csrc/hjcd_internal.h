// hjcd_internal.h — structures shared by the host C-ABI code and the kernels
// of libhjcd.so (never by the oracle).  The robot and the config travel to the
// device as __grid_constant__ kernel parameters, i.e. in the constant bank:
// every lane reads the same joint at the same time (uniform loop index), so
// each access is a broadcast and FFMAs take the constants as direct operands.
#pragma once
#include <atomic>
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
    uint32_t rx;         // 1: every DoF joint's F_j rotation is Rx(alpha) (DH twist; R[0] = 1,
                         //    R[1] = R[2] = R[3] = R[6] = 0 exactly in this precision): DESIGN K11
    int32_t pad;
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

// Decision trace of the PO-CCD kernel (hjcd_poccd_trace): the decision word
// of every seed-iteration [T][M][ccd_iters], and optionally theta at the start
// of every iteration [T][M][ccd_iters + 1][n] (the replay resynchronises on it)
struct TraceOut {
    uint32_t* words = nullptr;
    float* theta = nullptr;
};

// Dependent launch of PJ-IK on PO-CCD inside hjcd_solve (K10). With
// ready != nullptr the PO-CCD lockstep kernel adds 1 to ready[t] (release, gpu
// scope) when a CTA of target t's cluster has written its seeds, and the PJ-IK
// kernel, launched as a programmatic dependent (it may start while PO-CCD still
// runs), waits in each CTA until ready[t] == need, then does Alg. 2 l.2-8 (top-K
// + replicate) for its target itself from cost / theta before polishing.
struct StageLink {
    uint32_t* ready = nullptr;     // [T], zeroed before the PO-CCD launch
    const float* cost = nullptr;   // stage-1 cost [T][M]
    const float* theta = nullptr;  // stage-1 theta [T][n][M]
    uint32_t need = 0;             // CTAs per PO-CCD cluster
    int32_t Mpad = 0;              // M rounded up to a power of two >= 2
    // readiness polls (~0.5 us apart) before a waiting PJ-IK CTA traps instead
    // of hanging (a stage 1 that cannot complete); scaled with the PO-CCD budget
    unsigned long long spin_limit = 0;
    // K26: pop the targets in PO-CCD stop-iteration order (else blockIdx order)
    int32_t order = 0;
    // not part of the link: PJ-IK decision words [T][B][lm_iters] and theta at
    // the start of every iteration [T][B][lm_iters + 1][n], or nullptr
    // (hjcd_pjik_trace; word format in include/hjcd.h), for any launch
    uint32_t* trace = nullptr;
    float* trace_theta = nullptr;
};

// seeds per CTA (nt) and CTAs per cluster (CL) of the PO-CCD lockstep launch:
// 128-thread CTAs (32 for M < 128), 256 for the 12- and 14-joint kernels
// (measured: C4 -7 %; no change at 7-8 joints; the 16/18-joint kernels need
// 170 registers, i.e. 3 CTAs of 128), up to 16 CTAs per cluster (non-portable
// size above 8).  nmax: the kernel's joint bound (poccd_nmax).
constexpr int poccd_cta(int nmax) { return (nmax > 8 && nmax <= 14) ? 256 : 128; }
inline void texit_shape(int M, int nmax, int& nt, int& CL) {
    const int big = poccd_cta(nmax);
    nt = M < 128 ? (M + 31) / 32 * 32 : (M < big ? 128 : big);
    CL = (M + nt - 1) / nt;
}

// the packed two-seeds-per-thread launch (K17): threads per CTA and CTAs per cluster
inline void texit_shape_x2(int M, int& nt, int& CL) {
    const int pairs = (M + 1) / 2;
    nt = pairs < 128 ? (pairs + 31) / 32 * 32 : 128;
    CL = (pairs + nt - 1) / nt;
}

// DESIGN K26: the polish order.  hjcd_solve's PO-CCD clusters push each
// finished target onto a lock-free stack keyed by its stop iteration k*
// (R12b), and every PJ-IK CTA pops the ready target of the smallest k*: the
// targets whose polish runs longest are the ones whose stage 1 stopped
// earliest (scripts/slow_predict.py), so they start first instead of wherever
// their index puts them in the polish grid.  Only the schedule changes (each
// target's arithmetic depends on its index alone).  K30: the stacks are
// sharded (target t in shard t mod kReadyShards, a claiming CTA starts at
// shard blockIdx mod kReadyShards), so concurrent claims rarely race on one
// head; the order is then k*-first within a shard, and the shards drain at
// the same rate.  Layout after ready[T]: next[T] (stack links, t + 1; 0 =
// end), head[shards][buckets] (t + 1 of the top; 0 = empty), pushed, popped;
// all zeroed with ready.  Each target is pushed once and popped once, so the
// stacks have no ABA problem.
constexpr int kReadyBuckets = 64;
#ifndef HJCD_READY_SHARDS
#define HJCD_READY_SHARDS 16
#endif
constexpr int kReadyShards = HJCD_READY_SHARDS;
constexpr int kReadyHeads = kReadyShards * kReadyBuckets;
constexpr int kReadyWords = kReadyHeads + 2;   // + pushed, popped counts

__device__ __forceinline__ void ready_push(uint32_t* ready, int T, int t, int kstar) {
    uint32_t* nxt = ready + T;
    uint32_t* head = ready + 2 * T + (t % kReadyShards) * kReadyBuckets +
                     (kstar < kReadyBuckets - 1 ? kstar : kReadyBuckets - 1);
    __threadfence();   // the cluster's seeds (fenced by every CTA before its count) before the link
    uint32_t h = *(volatile uint32_t*)head;
    for (;;) {
        *(volatile uint32_t*)(nxt + t) = h;
        __threadfence();
        const uint32_t prev = atomicCAS(head, h, (uint32_t)t + 1u);
        if (prev == h) break;
        h = prev;
    }
    atomicAdd(ready + 2 * T + kReadyHeads, 1u);   // pushed
}

// one warp: the lowest non-empty bucket's top in the first non-empty shard
// from `shard0` on, popped; -1 if every stack is empty right now.  The result
// is warp-uniform.
__device__ __forceinline__ int ready_pop_warp(uint32_t* ready, int T, int shard0) {
    uint32_t* nxt = ready + T;
    uint32_t* heads = ready + 2 * T;
    const int lane = (int)(threadIdx.x & 31);
    // one word pair polled while nothing is queued (the heads only when a pop can succeed)
    const uint32_t pushed = *(volatile uint32_t*)(heads + kReadyHeads);
    const uint32_t popped = *(volatile uint32_t*)(heads + kReadyHeads + 1);
    if (pushed == popped) return -1;
    for (int sh = 0; sh < kReadyShards;) {
        uint32_t* head = heads + ((shard0 + sh) % kReadyShards) * kReadyBuckets;
        const uint32_t h0 = *(volatile uint32_t*)(head + lane);
        const uint32_t h1 = *(volatile uint32_t*)(head + 32 + lane);
        const unsigned m0 = __ballot_sync(0xffffffffu, h0 != 0u), m1 = __ballot_sync(0xffffffffu, h1 != 0u);
        if (!(m0 | m1)) {   // this shard is empty: the next one
            ++sh;
            continue;
        }
        const int b = m0 ? __ffs(m0) - 1 : 32 + __ffs(m1) - 1;
        int got = -2;   // -2: lost a race, rescan this shard
        if (lane == (b & 31)) {
            uint32_t h = b < 32 ? h0 : h1;
            while (h != 0u) {
                const uint32_t nx = *(volatile uint32_t*)(nxt + (h - 1u));
                const uint32_t prev = atomicCAS(head + b, h, nx);
                if (prev == h) { got = (int)(h - 1u); break; }
                h = prev;
            }
        }
        if (got >= 0) atomicAdd(heads + kReadyHeads + 1, 1u);   // popped
        got = __shfl_sync(0xffffffffu, got, b & 31);
        if (got >= 0) {
            __threadfence();
            return got;
        }
    }
    return -1;
}

#ifdef HJCD_PROBE
// A/B diagnostic build only: %globaltimer stamps of the K10 schedule, stored
// after the readiness counts: [5][T] = PO-CCD first CTA start, last CTA end,
// PJ-IK CTA start, end of its wait, CTA end (ns)
__device__ __forceinline__ unsigned long long probe_now() {
    unsigned long long v;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
    return v;
}
__device__ __forceinline__ unsigned long long* probe_base(uint32_t* ready, int T) {
    return (unsigned long long*)(ready + ((2 * T + kReadyWords + 63) & ~63));   // after the K26 queue
}
#endif

// Kernel attributes (shared-memory opt-in, non-portable cluster size) are
// per device: `done` is one call site's bitmask of devices already set.
// Setting an attribute twice is harmless, so a race only repeats the call.
template <class Fn>
inline cudaError_t once_per_device(std::atomic<unsigned long long>& done, Fn&& fn) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    if ((e = fn()) != cudaSuccess) return e;
    done.fetch_or(bit, std::memory_order_acq_rel);
    return cudaSuccess;
}

// Philox purposes (R30)
enum : uint32_t { P_INIT = 1, P_PERTURB = 2, P_REPL = 3, P_PJPERT = 4 };

// per-instantiation launchers (templates in poccd.cuh / pjik_coop.cuh,
// explicitly instantiated one or two per inst_*.cu so nvcc runs in parallel)
template <int NMAX, bool EXACT>
cudaError_t launch_poccd_t(const DevRobot& rb, const DevCfg& c, const float* targets, int T,
                           const float* seeds, float* theta, float* cost, float* ep, float* eo,
                           int32_t* iters, TraceOut trace, uint32_t* ready, cudaStream_t s);
template <int NMAX, bool EXACT>
cudaError_t launch_ccd_t(const DevRobot& rb, const DevCfg& c, const float* targets, int T, const float* seeds,
                         float* theta, float* ep, int32_t* iters, cudaStream_t s);
template <class T, int NMAX, bool EXACT>
cudaError_t launch_coop_t(const DevRobotT<T>& rb, const DevCfg& c, const float* targets, int T_,
                          const float* seeds, T* theta, T* ep, T* eo, int32_t* counts, int32_t* iters,
                          cudaStream_t s, const StageLink& link);

template <int NMAX, bool EXACT>
cudaError_t launch_poccd_x2_t(const DevRobot& rb, const DevCfg& c, const float* targets, int T, float* theta,
                              float* cost, float* ep, float* eo, int32_t* iters, TraceOut trace, uint32_t* ready,
                              cudaStream_t s);

// the joint bound NMAX of the PO-CCD kernel launch_poccd picks for n DoF (dispatch.cu)
int poccd_nmax(int n);
// CTAs per target cluster of launch_poccd's stop-rule launch (M seeds, n DoF,
// fused Philox seeds): the readiness count the dependent PJ-IK waits for (K10)
int poccd_cluster_ctas(int M, int n);
// true if hjcd_solve's PO-CCD stage runs k_poccd_x2 (K17) for n DoF
bool poccd_uses_x2(int n, bool ccd_early_exit);

// launchers (dispatch.cu, select.cu); all asynchronous on `s`
cudaError_t launch_fk(const DevRobot& rb, const float* q, int N, float* pose7, float* jac,
                      cudaStream_t s, bool sfu = false);
cudaError_t launch_poccd(const DevRobot& rb, const DevCfg& c, const float* targets, int T,
                         const float* seeds, float* theta, float* cost, float* ep, float* eo,
                         int32_t* iters, cudaStream_t s, TraceOut trace = TraceOut(), uint32_t* ready = nullptr);
cudaError_t launch_ccd(const DevRobot& rb, const DevCfg& c, const float* targets, int T, const float* seeds,
                       float* theta, float* ep, int32_t* iters, cudaStream_t s);
cudaError_t launch_select_replicate(const DevRobot& rb, const DevCfg& c, const float* cost,
                                    const float* theta, int T, float* seeds, int32_t* kept,
                                    cudaStream_t s);
cudaError_t launch_pjik(const DevRobot& rb, const DevCfg& c, const float* targets, int T,
                        const float* seeds, float* theta, float* ep, float* eo, int32_t* counts,
                        int32_t* iters, cudaStream_t s, const StageLink& link = StageLink());
template <class T>
cudaError_t launch_pjik_coop(const DevRobotT<T>& rb, const DevCfg& c, const float* targets, int T_,
                             const float* seeds, T* theta, T* ep, T* eo, int32_t* counts, int32_t* iters,
                             cudaStream_t s, const StageLink& link);
cudaError_t launch_select_topn(const DevRobot& rb, const DevCfg& c, const float* targets, int T, const float* theta,
                               const float* ep_all, const float* eo_all, int N, float* q_out, float* pos_err,
                               float* ori_err, int32_t* idx, int32_t* status, cudaStream_t s);
cudaError_t launch_mmd(const float* X, int N, const float* Y, int N2, int n, int T, float* mmd2, float* bw,
                       cudaStream_t s);
template <class T>
cudaError_t launch_select_best(const DevRobot& rb, const DevCfg& c, const float* targets, int T_,
                               const T* theta, const T* ep_all, const T* eo_all, T* q_out, T* pos_err,
                               T* ori_err, int32_t* status, cudaStream_t s);
// fp64 pose error of fp32 configurations on the fp64 chain (hjcd_pose_error_f64)
cudaError_t launch_pose_error64(const DevRobotT<double>& rb, const float* q, const float* targets, int N,
                                double* pos_err, double* ori_err, cudaStream_t s);
// fp64 polish: the same PJ-IK on DevRobotT<double>
cudaError_t launch_pjik64(const DevRobotT<double>& rb, const DevCfg& c, const float* targets, int T,
                          const float* seeds, double* theta, double* ep, double* eo, int32_t* counts,
                          int32_t* iters, cudaStream_t s);

}  // namespace hjcd

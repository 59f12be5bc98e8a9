/*
 * hjcd.h — C ABI of libhjcd.so, the B200 (sm_100a) hot path of HJCD-IK
 * (arXiv 2510.07514; "P:NNN" = line of the paper's PAPER.md).
 *
 * Problem (Eq. 2; constraints Eq. 3): given a serial chain and
 * target poses P_t in SE(3), find theta* with f(theta*) = P_t and
 * theta_min <= theta* <= theta_max.  The general g(theta) >= 0 of Eq. 3 is out
 * of scope.  Method (Alg. 2): PO-CCD over M seeds per target
 * (Alg. 3) -> top-K + noisy replication to B seeds (Alg. 2 l.2-8,
 * P:177-186) -> PJ-IK polish (Alg. 4) -> best of B.
 *
 * Conventions (every entry point):
 *   - Plain C types only; no exceptions cross the ABI; every call returns an
 *     hjcd_status.  Argument/shape errors are detected synchronously on the
 *     host BEFORE any launch; kernels are then enqueued on `stream` and the
 *     call returns without synchronising (except hjcd_solve_host).
 *   - Ownership: the library owns only hjcd_robot handles.  Every array is
 *     caller-owned; pointers documented "device" must be device memory of the
 *     current CUDA device (e.g. torch tensors), "host" pointers host memory.
 *     Scratch space is a caller-provided device workspace sized by
 *     hjcd_workspace_size().
 *   - Layouts are C row-major with the shapes given in brackets; all
 *     floating point is fp32 (the kernels compute in fp32 on the FP32 ALUs).
 *   - Pose layout: [px, py, pz, qw, qx, qy, qz] (metres, unit quaternion,
 *     Hamilton convention, scalar first).
 *   - Determinism: results are a pure function of (robot, config, targets,
 *     global target ids = target_index_offset + row).  Random numbers are
 *     Philox4x32-10 keyed by config.rng_seed with counter
 *     (global target id, seed id, purpose << 24 | iteration, draw block), so
 *     results do not depend on T-chunking or on the number of GPUs.
 *   - A robot handle is immutable: it may be shared across threads, streams
 *     and devices (it carries no device memory; the chain travels in the
 *     kernel parameters).  Concurrent calls need distinct workspaces.
 */
#ifndef HJCD_H_
#define HJCD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* hjcd_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
    HJCD_OK = 0,
    HJCD_E_INVALID_ARG = 1, /* null pointer, bad size, K > M, K > B, lo > hi, ... */
    HJCD_E_UNSUPPORTED = 2, /* dof > HJCD_MAX_DOF, unsupported option */
    HJCD_E_CUDA = 3,        /* a CUDA runtime error (see hjcd_last_cuda_error) */
    HJCD_E_WORKSPACE = 4,   /* workspace too small, misaligned (< 256 B), or in use by a
                               solve still in flight on another stream */
    HJCD_E_NOMEM = 5        /* host allocation failed */
} hjcd_status;

#define HJCD_MAX_DOF 32

/* Per-target result status written by hjcd_solve (Alg. 4 l.18). */
enum {
    HJCD_TARGET_CONVERGED = 0,  /* |r_p| < eps_p_fine and |omega| < eps_o_fine */
    HJCD_TARGET_SUCCESS = 1,    /* not fine-converged but within succ_p / succ_o */
    HJCD_TARGET_NOT_CONVERGED = 2, /* best effort returned */
    HJCD_TARGET_INVALID = 3     /* | |q| - 1 | > 1e-3 or non-finite target; q = 0, errors = +inf */
};

typedef enum { HJCD_REVOLUTE = 0, HJCD_PRISMATIC = 1, HJCD_FIXED = 2 } hjcd_joint_type;

/* One joint of a serial chain, base -> tip (D1; P:44-48 limits, P:69 axes).
 * The joint's frame is parent * origin; it then rotates about (revolute) or
 * translates along (prismatic) `axis`, expressed in that frame.
 * origin_quat_wxyz must be unit (+-1e-6); axis non-zero (normalised here);
 * lo <= hi (radians, or metres for prismatic); revolute limits within +-1e4 rad
 * (the kernels' joint sincos range).  Fixed joints are folded. */
typedef struct {
    int32_t type;
    double origin_xyz[3];
    double origin_quat_wxyz[4];
    double axis[3];
    double lo, hi;
} hjcd_joint;

typedef struct hjcd_robot hjcd_robot; /* opaque, immutable */

/* Create a robot from `num_joints` joints + end-effector offset (relative to
 * the last joint frame).  Validates (E_INVALID_ARG) and canonicalises every
 * DoF joint to "fixed transform F_i, then rotation about / translation along
 * local z" in fp64, stored in fp32.  dof must be 1..HJCD_MAX_DOF
 * (E_UNSUPPORTED otherwise).  *out receives a new handle. */
hjcd_status hjcd_robot_create(const hjcd_joint* joints, int32_t num_joints,
                              const double ee_xyz[3], const double ee_quat_wxyz[4],
                              hjcd_robot** out);

/* DoF extension ("adding replicated revolute joints and links"; DESIGN.md
 * R34): cyclic replication of r's DoF joints (origin, axis, limits) before the
 * end effector until target_dof.  E_INVALID_ARG if target_dof < dof. */
hjcd_status hjcd_robot_extend(const hjcd_robot* r, int32_t target_dof, hjcd_robot** out);
void hjcd_robot_destroy(hjcd_robot* r);
int32_t hjcd_robot_dof(const hjcd_robot* r);
/* joint limits of the DoF joints as stored (fp32), host arrays [dof] */
hjcd_status hjcd_robot_limits(const hjcd_robot* r, float* lo, float* hi);

/* Algorithm parameters (Alg. 2-4 headers P:175); defaults and the
 * reading behind each are in DESIGN.md "Readings" (R-numbers). */
typedef struct {
    int32_t M, K, B;               /* seeds, retained, polish batch: 1 <= K <= M, K <= B (Alg. 2);
                                      floor(B/K)*K <= 256 (one CTA per target in PJ-IK) */
    int32_t ccd_iters, lm_iters;   /* iteration budgets I_c (Alg. 3), I_l (Alg. 4) (R28) */
    int32_t target_early_exit;     /* PJ-IK stop rule (Alg. 4 l.18; R26b): 1 = a target stops at the
                                      first iteration in which ANY of its polish seeds passes the fine
                                      test (deterministic); 0 = every seed
                                      runs until it converges or lm_iters (per-seed freeze) */
    int32_t ccd_early_exit;        /* PO-CCD stop rule (R12b): 1 = a target's M seeds stop at the
                                      first iteration in which ANY of them passes the coarse test (one
                                      thread-block cluster per target, deterministic, needs M <= 2048);
                                      0 = every seed runs until it converges or ccd_iters */
    float eps_p_coarse, eps_o_coarse; /* epsilon [m], nu [rad], Alg. 3 l.14 (R12) */
    float eps_p_fine, eps_o_fine;  /* varepsilon [m], upsilon [rad], Alg. 4 l.18 (R26) */
    float gamma;                   /* improvement threshold, Alg. 3 l.11 (R10) */
    float delta0, delta_rho, delta_min; /* delta(k) = max(delta_min, delta0 rho^k), Eq. 11 (R5) */
    float sigma_ccd, sigma_rep, sigma_lm; /* isotropic N(0, sigma^2) std devs (R11, R15, R25) */
    float lambda, d_floor, R, beta; /* Eq. 12 damping, D floor, trust radius, line-search base (R20-R22) */
    int32_t A;                     /* line-search depth: alphas 1 .. beta^-A (Eq. 13) */
    float w_p, w_o;                /* residual weights inside W (R17) and the ranking cost (R14) */
    float succ_p, succ_o;          /* reporting thresholds for status 1 */
    float tau_deg;                 /* CCD degenerate-projection threshold [m] (R4) */
    int32_t repl_noise_all;        /* 1 = noise on every replica (literal Alg. 2 l.8), 0 = copy 0 clean (R15) */
    uint64_t rng_seed;             /* Philox key */
    int64_t target_index_offset;   /* global id of targets[0] (RNG counter; multi-GPU shards) */
} hjcd_config;

void hjcd_config_default(hjcd_config* c);

/* Bytes of device workspace hjcd_solve needs for T targets (a multiple of 256). */
hjcd_status hjcd_workspace_size(const hjcd_robot* r, int32_t T, const hjcd_config* c, size_t* bytes);
/* Bytes hjcd_solve_host needs: hjcd_workspace_size + device staging of I/O. */
hjcd_status hjcd_workspace_size_host(const hjcd_robot* r, int32_t T, const hjcd_config* c,
                                     size_t* bytes);

/* HJCD-IK (Alg. 2) for T >= 1 targets.
 *   targets  device [T][7] fp32 (pose layout above); q normalised when
 *            | |q| - 1 | <= 1e-3, else the row gets status 3.
 *   q_out    device [T][dof]   theta* (best polished seed, R27)
 *   pos_err  device [T]        |P_t - P_ee(theta*)| metres
 *   ori_err  device [T]        |omega(theta*)| radians (Eq. 5)
 *   status   device [T]        HJCD_TARGET_*
 *   workspace device, >= hjcd_workspace_size bytes, 256-byte aligned; one
 *            solve at a time per workspace (it holds the stage-1 seeds and,
 *            with the per-target PO-CCD stop rule, per-target readiness
 *            counts).  A solve on another stream while the last solve that
 *            used this workspace (through this library, any solve entry point)
 *            is still in flight returns HJCD_E_WORKSPACE; the same stream is
 *            stream-ordered and always allowed; during CUDA-graph capture the
 *            check is skipped.  If a polish CTA still waits more than ~30 s
 *            (x ccd_iters/64) for its target's stage 1 (e.g. a workspace shared
 *            with another process), it executes a device trap rather than
 *            hang: that is a sticky error that loses the CUDA context of the
 *            whole process (every later CUDA call in it, torch's included,
 *            fails).
 * Asynchronous on `stream`: a memset of the readiness counts, the PO-CCD
 * kernel, PJ-IK as its programmatic dependent launch (it starts on each target
 * as soon as that target's stage 1 is in memory, K10; for
 * 2 x SMs < T <= 5000 its CTAs take the ready targets in order of their
 * PO-CCD stop iteration, smallest first, K26/K30) and the best select; for
 * T >= 5000 at >= 12 DoF the staged sequence of hjcd_solve_timed (K33).  Results are
 * bitwise those of hjcd_solve_timed's staged sequence. */
hjcd_status hjcd_solve(const hjcd_robot* r, const hjcd_config* c, const float* targets, int32_t T,
                       float* q_out, float* pos_err, float* ori_err, int32_t* status,
                       void* workspace, size_t workspace_bytes, hjcd_stream_t stream);

/* hjcd_solve that also records stage boundaries for live per-kernel timing:
 * events = NULL (then exactly hjcd_solve) or an array of 5 caller-created
 * CUDA events (cudaEvent_t, created with timing enabled), recorded on `stream`
 * before PO-CCD, after PO-CCD, after top-K/replicate, after PJ-IK and after
 * best-select; with events the stages run as separate, serialised kernels. */
hjcd_status hjcd_solve_timed(const hjcd_robot* r, const hjcd_config* c, const float* targets, int32_t T,
                             float* q_out, float* pos_err, float* ori_err, int32_t* status,
                             void* workspace, size_t workspace_bytes, hjcd_stream_t stream,
                             void* const* events);

/* The solution BATCH ("the return of multiple local optima"; §V-C
 * keeps "the best 50 joint configurations"): Alg. 2 with the final
 * best-select replaced by the best N <= floor(B/K)*K polished seeds of each
 * target, in R27 order (fine-converged first, then the cost c of R14, then
 * slot), so entry 0 is hjcd_solve's answer.
 *   q_out [T][N][dof], pos_err/ori_err [T][N] device out; status [T] of entry 0.
 *   workspace as hjcd_solve. */
hjcd_status hjcd_solve_batch(const hjcd_robot* r, const hjcd_config* c, const float* targets, int32_t T,
                             int32_t N, float* q_out, float* pos_err, float* ori_err, int32_t* status,
                             void* workspace, size_t workspace_bytes, hjcd_stream_t stream);

/* fp64 polish (R29b): PO-CCD, top-K and replication
 * in fp32 as hjcd_solve (stage 1 only needs the coarse tolerance), then PJ-IK
 * and best-select in fp64 on an fp64 copy of the chain, so the fine tolerances
 * can go to SPEC's 1e-9 m / 1e-8 rad.  Outputs are fp64: q_out [T][dof],
 * pos_err/ori_err [T] (device); status [T] as hjcd_solve.  Workspace: device,
 * >= hjcd_workspace_size_f64 bytes, 256-byte aligned.  The fp64 polish keeps
 * per-seed records in shared memory: with dof > 16, floor(B/K)*K <= 160
 * (227 KB per CTA), otherwise HJCD_E_CUDA ("invalid configuration"). */
hjcd_status hjcd_workspace_size_f64(const hjcd_robot* r, int32_t T, const hjcd_config* c, size_t* bytes);
hjcd_status hjcd_solve_f64(const hjcd_robot* r, const hjcd_config* c, const float* targets, int32_t T,
                           double* q_out, double* pos_err, double* ori_err, int32_t* status,
                           void* workspace, size_t workspace_bytes, hjcd_stream_t stream);

/* The same with HOST buffers (same shapes): copies targets host->device,
 * solves, copies results device->host, and synchronises `stream` before
 * returning.  workspace: device, >= hjcd_workspace_size_host bytes. */
hjcd_status hjcd_solve_host(const hjcd_robot* r, const hjcd_config* c, const float* targets_host,
                            int32_t T, float* q_host, float* pos_err_host, float* ori_err_host,
                            int32_t* status_host, void* workspace, size_t workspace_bytes,
                            hjcd_stream_t stream);

/* ---- stage entry points (tests, tracing; same conventions; device pointers) ---- */

/* hjcd_fk with the joint sines / cosines from the SFU (__sincosf), the
 * variant the PO-CCD kernel runs (K5: coarse stage only); same
 * layouts and errors as hjcd_fk.  For parity testing of that FK. */
hjcd_status hjcd_fk_sfu(const hjcd_robot* r, const float* q, int32_t N, float* pose7, float* jac,
                        hjcd_stream_t stream);

/* Pose error of given joint configurations, evaluated in fp64 on the fp64
 * copy of the chain: pos_err = |P_t - P_ee(q)| (Eq. 4) and ori_err = |omega|
 * (Eq. 5, R1) with the fp32 configuration widened exactly.  Lets a caller
 * decide success at 1 mm / 1 deg from the returned theta rather than from the
 * solver's own fp32 errors (SURVEY §8(d) "Success").
 *   q [N][dof] f32, targets [N][7] f32 in (device); pos_err, ori_err [N] f64
 *   out (device).  An invalid target row (S2) gives +inf.  Asynchronous. */
hjcd_status hjcd_pose_error_f64(const hjcd_robot* r, const float* q, const float* targets, int32_t N,
                                double* pos_err, double* ori_err, hjcd_stream_t stream);

/* Batched FK (Eq. 1) + geometric Jacobian (Eq. 7) for N configurations.
 *   q     [N][dof]; pose7 [N][7] (w >= 0); jac [N][6][dof] or NULL
 *   (rows 0-2 linear, 3-5 angular; prismatic columns [z; 0]). */
hjcd_status hjcd_fk(const hjcd_robot* r, const float* q, int32_t N, float* pose7, float* jac,
                    hjcd_stream_t stream);

/* PO-CCD (Alg. 3) for T targets x c->M seeds.
 *   seeds  [T][dof][M] initial theta, or NULL = Philox uniform in limits (Alg. 3 l.2-3)
 *   theta  [T][dof][M] out; cost [T][M] out: w_p^2 |r_p|^2 + w_o^2 |omega|^2 (R14)
 *   pos_err, ori_err [T][M] out or NULL; iters [T][M] out or NULL (updates applied;
 *   with c->ccd_early_exit every seed of a target reports the target's k*, R12b,
 *   and M <= 2048, else E_UNSUPPORTED). */
hjcd_status hjcd_poccd(const hjcd_robot* r, const hjcd_config* c, const float* targets, int32_t T,
                       const float* seeds, float* theta, float* cost, float* pos_err,
                       float* ori_err, int32_t* iters, hjcd_stream_t stream);

/* hjcd_poccd that also records every seed's decisions (parity tests: the
 * oracle replays them in fp64): trace [T][M][c->ccd_iters]
 * uint32, one word per iteration k that updated the seed (entries past its
 * iteration count are left unwritten):
 *   bits 0-4 jp, 5-9 jo (Alg. 3 l.9 argmins), bit 10 same joint and the
 *   orientation step taken (l.10), bit 11 accepted (l.11), bits 12-13 / 14-15
 *   the sign of the position / orientation step at jp / jo (0 zero,
 *   1 positive, 2 negative).
 *   theta_hist [T][M][ccd_iters + 1][dof] out (device) or NULL: each seed's
 *   theta at the start of every iteration it ran (entry k = the state the
 *   decision of word k was taken at; entry iters = the returned theta); the
 *   decision replay restarts the oracle from it at every iteration, so fp32
 *   drift cannot accumulate into the comparison. */
hjcd_status hjcd_poccd_trace(const hjcd_robot* r, const hjcd_config* c, const float* targets, int32_t T,
                             const float* seeds, float* theta, float* cost, float* pos_err,
                             float* ori_err, int32_t* iters, uint32_t* trace, float* theta_hist,
                             hjcd_stream_t stream);

/* Classic position-only CCD (Alg. 1), the baseline PO-CCD extends
 * (ablation): T targets x c->M seeds, joints swept tip to root,
 * signed projected-angle steps (Eqs. 8-9; R3, R4) clamped to the limits (R7);
 * a seed stops when |P_ee - P_t| < c->eps_p_coarse (Alg. 1 l.7, R12) or after
 * c->ccd_iters sweeps.  Orientation is ignored (position-only IK).
 *   seeds [T][dof][M] or NULL (the PO-CCD Philox seeds, R30);
 *   theta [T][dof][M] out; pos_err [T][M] out or NULL; iters [T][M] out or NULL. */
hjcd_status hjcd_ccd(const hjcd_robot* r, const hjcd_config* c, const float* targets, int32_t T,
                     const float* seeds, float* theta, float* pos_err, int32_t* iters,
                     hjcd_stream_t stream);

/* Top-K by (cost, seed index) + floor(B/K) replicas (Alg. 2 l.2-8; R14, R15).
 *   cost [T][M], theta [T][dof][M] in; polish_seeds [T][B][dof] out (slot
 *   b = copy*K + rank; slots >= floor(B/K)*K are NaN); kept_idx [T][K] out or NULL.
 *   Requires M <= 8192. */
hjcd_status hjcd_select_replicate(const hjcd_robot* r, const hjcd_config* c, const float* cost,
                                  const float* theta, int32_t T, float* polish_seeds,
                                  int32_t* kept_idx, hjcd_stream_t stream);

/* PJ-IK (Alg. 4) for T targets x c->B seeds (slots >= floor(B/K)*K skipped).
 *   seeds [T][B][dof] in; theta [T][B][dof] out (may alias seeds);
 *   pos_err, ori_err [T][B] out; step_counts [T][B][4] (LM, dogleg, single,
 *   perturb) out or NULL; iters [T][B] out or NULL. */
hjcd_status hjcd_pjik(const hjcd_robot* r, const hjcd_config* c, const float* targets, int32_t T,
                      const float* seeds, float* theta, float* pos_err, float* ori_err,
                      int32_t* step_counts, int32_t* iters, hjcd_stream_t stream);

/* hjcd_pjik that also records every seed's decision at every iteration
 * (parity testing: the oracle replays these decisions in fp64).
 *   trace [T][B][lm_iters] out, device, caller-owned; one word per
 *   (target, polish slot, iteration k) at which that seed took a step
 *   (words past a seed's iteration count, and slots >= floor(B/K)*K, are left
 *   unwritten):
 *   bits 0-1 the branch that moved the seed: 0 the LM step (Alg. 4 l.3-9,
 *   Eq. 12-13), 1 the dogleg step (l.10-12, Eqs. 14-15), 2 the
 *   single-coordinate step (l.13-16, Eq. 16), 3 the perturbation (l.17);
 *   bits 2-6 the line-search index a (step beta^-a; 0 for dogleg and
 *   perturbation); bits 8-12 the single-coordinate index i* (branch 2 only);
 *   bit 15 set (a step was taken).
 *   theta_hist [T][B][lm_iters + 1][dof] out (device) or NULL: each seed's
 *   theta at the start of every iteration it ran, as in hjcd_poccd_trace.
 *   Same errors as hjcd_pjik. */
hjcd_status hjcd_pjik_trace(const hjcd_robot* r, const hjcd_config* c, const float* targets, int32_t T,
                            const float* seeds, float* theta, float* pos_err, float* ori_err,
                            int32_t* step_counts, int32_t* iters, uint32_t* trace, float* theta_hist,
                            hjcd_stream_t stream);

/* Best-of-B selection (Alg. 2 l.9-10, R27): fine-converged seeds first, then
 * argmin_b w_p^2 pe^2 + w_o^2 oe^2, ties -> lowest b; writes
 * q_out/pos_err/ori_err/status as hjcd_solve does. */
hjcd_status hjcd_select_best(const hjcd_robot* r, const hjcd_config* c, const float* targets,
                             int32_t T, const float* theta, const float* pos_err_all,
                             const float* ori_err_all, float* q_out, float* pos_err,
                             float* ori_err, int32_t* status, hjcd_stream_t stream);

/* PJ-IK (Alg. 4) in fp64 (the stage of hjcd_solve_f64): fp32 seeds [T][B][dof]
 * in; theta [T][B][dof], pos_err/ori_err [T][B] fp64 out; step_counts and
 * iters as hjcd_pjik. */
hjcd_status hjcd_pjik_f64(const hjcd_robot* r, const hjcd_config* c, const float* targets, int32_t T,
                          const float* seeds, double* theta, double* pos_err, double* ori_err,
                          int32_t* step_counts, int32_t* iters, hjcd_stream_t stream);

/* Best N of the B polished seeds per target (the stage of hjcd_solve_batch):
 * theta [T][B][dof], pos_err_all/ori_err_all [T][B] in; q_out [T][N][dof],
 * pos_err/ori_err [T][N], idx [T][N] (slot, or -1 for an invalid target; may be
 * NULL) out.  1 <= N <= floor(B/K)*K. */
hjcd_status hjcd_select_topn(const hjcd_robot* r, const hjcd_config* c, const float* targets, int32_t T,
                             const float* theta, const float* pos_err_all, const float* ori_err_all,
                             int32_t N, float* q_out, float* pos_err, float* ori_err, int32_t* idx,
                             hjcd_stream_t stream);

/* Solution-set diversity (§V-C, Table III; R36): for each of T pairs
 * of point sets X [T][N][dim], Y [T][N2][dim] (device, fp32), the biased
 * V-statistic MMD^2 = mean k(x,x') + mean k(y,y') - 2 mean k(x,y) with the
 * Gaussian kernel k(a,b) = exp(-|a-b|^2 / (2 h^2)), h = median of the pairwise
 * distances over X u Y (h is written to bandwidth [T] if non-NULL).
 * N, N2 >= 1, N + N2 <= 256 (E_UNSUPPORTED), 1 <= dim <= 32.  MMD = sqrt(max(0, MMD^2)). */
hjcd_status hjcd_mmd(const float* X, int32_t N, const float* Y, int32_t N2, int32_t dim, int32_t T,
                     float* mmd2, float* bandwidth, hjcd_stream_t stream);

const char* hjcd_status_string(hjcd_status s);

/* The name of the PO-CCD kernel hjcd_solve launches for this robot and config
 * ("k_poccd_x2": two seeds per thread, packed fp32, K17; "k_poccd"
 * otherwise), for profilers and roofline reports.  Static storage; "" on NULL. */
const char* hjcd_poccd_kernel(const hjcd_robot* r, const hjcd_config* c);
/* text of the last CUDA error seen by this thread's calls ("" if none) */
const char* hjcd_last_cuda_error(void);
/* library / build identification, e.g. "hjcd 0.1 sm_100a" */
const char* hjcd_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HJCD_H_ */

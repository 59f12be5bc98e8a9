// hjcd_capi.cu — host side of the C ABI (include/hjcd.h): robot validation and
// canonicalisation (fp64), config validation, workspace carving and the
// stream-ordered launch sequence of hjcd_solve (Alg. 2).
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <unordered_map>
#include <vector>

#include "hjcd_internal.h"

using namespace hjcd;

struct hjcd_robot {
    std::vector<hjcd_joint> joints;   // as given (for extend)
    double ee_xyz[3];
    double ee_quat[4];
    int dof;
    DevRobot dev;
    DevRobotT<double> dev64;   // the same chain in fp64 (hjcd_solve_f64)
};

namespace {

thread_local std::string g_cuda_err;

hjcd_status cuda_fail(cudaError_t e) {
    g_cuda_err = cudaGetErrorString(e);
    (void)cudaGetLastError();   // clear a non-sticky error so the next call does not inherit it
    return HJCD_E_CUDA;
}

// ---------------------------------------------------------------- fp64 rigid transforms
struct Rt {
    double R[9];   // row-major
    double t[3];
};

Rt rt_identity() {
    Rt a = {{1, 0, 0, 0, 1, 0, 0, 0, 1}, {0, 0, 0}};
    return a;
}

Rt rt_mul(const Rt& a, const Rt& b) {
    Rt c;
    for (int r = 0; r < 3; ++r) {
        for (int k = 0; k < 3; ++k)
            c.R[3 * r + k] = a.R[3 * r] * b.R[k] + a.R[3 * r + 1] * b.R[3 + k] + a.R[3 * r + 2] * b.R[6 + k];
        c.t[r] = a.R[3 * r] * b.t[0] + a.R[3 * r + 1] * b.t[1] + a.R[3 * r + 2] * b.t[2] + a.t[r];
    }
    return c;
}

Rt rt_transpose_rot(const Rt& a) {   // inverse of a pure rotation
    Rt c = rt_identity();
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k) c.R[3 * r + k] = a.R[3 * k + r];
    return c;
}

Rt rt_from_pose(const double xyz[3], const double q[4]) {
    double w = q[0], x = q[1], y = q[2], z = q[3];
    double nq = std::sqrt(w * w + x * x + y * y + z * z);
    w /= nq; x /= nq; y /= nq; z /= nq;
    Rt a;
    a.R[0] = 1 - 2 * (y * y + z * z); a.R[1] = 2 * (x * y - w * z); a.R[2] = 2 * (x * z + w * y);
    a.R[3] = 2 * (x * y + w * z); a.R[4] = 1 - 2 * (x * x + z * z); a.R[5] = 2 * (y * z - w * x);
    a.R[6] = 2 * (x * z - w * y); a.R[7] = 2 * (y * z + w * x); a.R[8] = 1 - 2 * (x * x + y * y);
    a.t[0] = xyz[0]; a.t[1] = xyz[1]; a.t[2] = xyz[2];
    return a;
}

// a rotation C with C e_z = a (a unit)
Rt rot_z_to(const double a[3]) {
    Rt C = rt_identity();
    if (a[2] > 1.0 - 1e-15) return C;
    if (a[2] < -1.0 + 1e-15) {   // Rx(pi)
        C.R[4] = -1; C.R[8] = -1;
        return C;
    }
    // axis k = e_z x a / |.|, angle acos(a_z)
    double kx = -a[1], ky = a[0];
    double s = std::sqrt(kx * kx + ky * ky);
    kx /= s; ky /= s;
    double c = a[2], sn = s, v = 1 - c;
    C.R[0] = c + kx * kx * v; C.R[1] = kx * ky * v;      C.R[2] = ky * sn;
    C.R[3] = ky * kx * v;     C.R[4] = c + ky * ky * v;  C.R[5] = -kx * sn;
    C.R[6] = -ky * sn;        C.R[7] = kx * sn;          C.R[8] = c;
    return C;
}

template <class S>
void store(const Rt& a, S R[9], S t[3]) {
    for (int i = 0; i < 9; ++i) R[i] = (S)a.R[i];
    for (int i = 0; i < 3; ++i) t[i] = (S)a.t[i];
}

bool finite3(const double* v, int k) {
    for (int i = 0; i < k; ++i)
        if (!std::isfinite(v[i])) return false;
    return true;
}

hjcd_status build_robot(const hjcd_joint* joints, int32_t num, const double ee_xyz[3],
                        const double ee_quat[4], hjcd_robot** out) {
    if (!joints || num < 1 || !ee_xyz || !ee_quat || !out) return HJCD_E_INVALID_ARG;
    int dof = 0;
    for (int i = 0; i < num; ++i) {
        const hjcd_joint& j = joints[i];
        if (j.type != HJCD_REVOLUTE && j.type != HJCD_PRISMATIC && j.type != HJCD_FIXED) return HJCD_E_INVALID_ARG;
        if (!finite3(j.origin_xyz, 3) || !finite3(j.origin_quat_wxyz, 4)) return HJCD_E_INVALID_ARG;
        const double* q = j.origin_quat_wxyz;
        double nq = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
        if (std::fabs(nq - 1.0) > 1e-6) return HJCD_E_INVALID_ARG;
        if (j.type != HJCD_FIXED) {
            if (!finite3(j.axis, 3)) return HJCD_E_INVALID_ARG;
            double na = std::sqrt(j.axis[0] * j.axis[0] + j.axis[1] * j.axis[1] + j.axis[2] * j.axis[2]);
            if (!(na > 1e-9)) return HJCD_E_INVALID_ARG;
            if (!std::isfinite(j.lo) || !std::isfinite(j.hi) || j.lo > j.hi) return HJCD_E_INVALID_ARG;
            // the kernels' joint sincos is accurate for |theta| <= 1e4 (kin.cuh sincos_b)
            if (j.type == HJCD_REVOLUTE && (std::fabs(j.lo) > 1e4 || std::fabs(j.hi) > 1e4)) return HJCD_E_INVALID_ARG;
            dof++;
        }
    }
    if (!finite3(ee_xyz, 3) || !finite3(ee_quat, 4)) return HJCD_E_INVALID_ARG;
    {
        double nq = std::sqrt(ee_quat[0] * ee_quat[0] + ee_quat[1] * ee_quat[1] + ee_quat[2] * ee_quat[2] +
                              ee_quat[3] * ee_quat[3]);
        if (std::fabs(nq - 1.0) > 1e-6) return HJCD_E_INVALID_ARG;
    }
    if (dof < 1 || dof > HJCD_MAX_DOF) return dof < 1 ? HJCD_E_INVALID_ARG : HJCD_E_UNSUPPORTED;

    hjcd_robot* r = new (std::nothrow) hjcd_robot;
    if (!r) return HJCD_E_NOMEM;
    r->joints.assign(joints, joints + num);
    for (int i = 0; i < 3; ++i) r->ee_xyz[i] = ee_xyz[i];
    for (int i = 0; i < 4; ++i) r->ee_quat[i] = ee_quat[i];
    r->dof = dof;
    std::memset(&r->dev, 0, sizeof(DevRobot));
    std::memset(&r->dev64, 0, sizeof(r->dev64));
    r->dev.n = dof;
    r->dev64.n = dof;
    // Canonicalise: Rot(a, th) = C Rz(th) C^T with C e_z = a; fold C^T and any
    // fixed joints into the next joint's fixed transform F (or the ee).
    Rt acc = rt_identity();
    int d = 0;
    for (int i = 0; i < num; ++i) {
        const hjcd_joint& j = joints[i];
        acc = rt_mul(acc, rt_from_pose(j.origin_xyz, j.origin_quat_wxyz));
        if (j.type == HJCD_FIXED) continue;
        double na = std::sqrt(j.axis[0] * j.axis[0] + j.axis[1] * j.axis[1] + j.axis[2] * j.axis[2]);
        double a[3] = {j.axis[0] / na, j.axis[1] / na, j.axis[2] / na};
        Rt C = rot_z_to(a);
        Rt F = rt_mul(acc, C);
        DevJoint& dj = r->dev.j[d];
        store(F, dj.R, dj.t);
        dj.lo = (float)j.lo;
        dj.hi = (float)j.hi;
        dj.type = j.type;
        DevJointT<double>& dd = r->dev64.j[d];
        store(F, dd.R, dd.t);
        // fp64 limits = the fp32 ones widened, so both precisions clamp to the same box
        dd.lo = (double)dj.lo;
        dd.hi = (double)dj.hi;
        dd.type = j.type;
        if (j.type == HJCD_PRISMATIC) { r->dev.pmask |= 1u << d; r->dev64.pmask |= 1u << d; }
        acc = rt_transpose_rot(C);
        d++;
    }
    // K11: the DH-twist pattern F_j.R = Rx(alpha_j), tested on the stored values
#ifndef HJCD_NO_RX   // (A/B builds only)
    r->dev.rx = r->dev64.rx = 1u;
#endif
    for (int k = 0; k < dof; ++k) {
        const float* R = r->dev.j[k].R;
        const double* R64 = r->dev64.j[k].R;
        if (!(R[0] == 1.f && R[1] == 0.f && R[2] == 0.f && R[3] == 0.f && R[6] == 0.f)) r->dev.rx = 0u;
        if (!(R64[0] == 1.0 && R64[1] == 0.0 && R64[2] == 0.0 && R64[3] == 0.0 && R64[6] == 0.0)) r->dev64.rx = 0u;
    }
    Rt E = rt_mul(acc, rt_from_pose(ee_xyz, ee_quat));
    store(E, r->dev.eeR, r->dev.eet);
    store(E, r->dev64.eeR, r->dev64.eet);
    *out = r;
    return HJCD_OK;
}

hjcd_status make_cfg(const hjcd_robot* r, const hjcd_config* c, DevCfg* d) {
    if (!r || !c) return HJCD_E_INVALID_ARG;
    if (c->M < 1 || c->K < 1 || c->B < 1 || c->K > c->M || c->K > c->B) return HJCD_E_INVALID_ARG;
    if (c->ccd_iters < 0 || c->lm_iters < 0 || c->A < 0) return HJCD_E_INVALID_ARG;
    if (c->target_early_exit != 0 && c->target_early_exit != 1) return HJCD_E_INVALID_ARG;
    if ((c->B / c->K) * c->K > 256 || c->A > 31) return HJCD_E_UNSUPPORTED;   // one CTA per target (K6)
    if (c->ccd_early_exit != 0 && c->ccd_early_exit != 1) return HJCD_E_INVALID_ARG;
    if (!(c->beta > 1.f) || !(c->lambda > 0.f) || !(c->d_floor > 0.f) || !(c->R > 0.f)) return HJCD_E_INVALID_ARG;
    if (!(c->eps_p_coarse > 0.f) || !(c->eps_o_coarse > 0.f) || !(c->eps_p_fine > 0.f) ||
        !(c->eps_o_fine > 0.f))
        return HJCD_E_INVALID_ARG;
    if (!(c->sigma_ccd >= 0.f) || !(c->sigma_rep >= 0.f) || !(c->sigma_lm >= 0.f)) return HJCD_E_INVALID_ARG;
    if (!(c->delta_min >= 0.f) || !(c->delta0 >= 0.f) || !(c->delta_rho > 0.f)) return HJCD_E_INVALID_ARG;
    if (!(c->tau_deg >= 0.f) || !(c->gamma >= 0.f) || !(c->w_p >= 0.f) || !(c->w_o >= 0.f)) return HJCD_E_INVALID_ARG;
    d->M = c->M; d->K = c->K; d->B = c->B;
    d->ccd_iters = c->ccd_iters; d->lm_iters = c->lm_iters; d->A = c->A;
    d->copies = c->B / c->K;
    d->repl_noise_all = c->repl_noise_all ? 1 : 0;
    d->target_early_exit = c->target_early_exit;
    d->ccd_early_exit = c->ccd_early_exit;
    d->eps_p_coarse = c->eps_p_coarse; d->eps_o_coarse = c->eps_o_coarse;
    d->eps_p_fine = c->eps_p_fine; d->eps_o_fine = c->eps_o_fine;
    d->gamma = c->gamma; d->delta0 = c->delta0; d->delta_rho = c->delta_rho; d->delta_min = c->delta_min;
    d->sigma_ccd = c->sigma_ccd; d->sigma_rep = c->sigma_rep; d->sigma_lm = c->sigma_lm;
    d->lambda = c->lambda; d->d_floor = c->d_floor; d->R = c->R; d->inv_beta = 1.f / c->beta;
    d->w_p = c->w_p; d->w_o = c->w_o; d->succ_p = c->succ_p; d->succ_o = c->succ_o;
    d->tau_deg = c->tau_deg;
    d->key0 = (uint32_t)c->rng_seed;
    d->key1 = (uint32_t)(c->rng_seed >> 32);
    d->tid_offset = c->target_index_offset;
    return HJCD_OK;
}

// the PO-CCD stop rule keeps a target's M seeds in one cluster of <= 16 x 128 threads
hjcd_status check_poccd(const hjcd_config* c) {
    return (c->ccd_early_exit && c->M > 2048) ? HJCD_E_UNSUPPORTED : HJCD_OK;
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// One solve at a time per workspace (hjcd.h): the host remembers, per workspace
// address, the stream of its last solve and an event recorded after that
// solve's launches.  A solve on ANOTHER stream while that event is pending
// would share the stage-1 buffers and readiness counts of a solve in flight;
// it is refused with HJCD_E_WORKSPACE instead of racing (or, in the dependent
// launch, waiting on counts the other solve resets).  The same stream is
// stream-ordered and always allowed; graph capture is left to the caller.
struct WsUse {
    cudaStream_t s = nullptr;
    cudaEvent_t ev = nullptr;
    int dev = -1;
};
std::mutex g_ws_mu;
std::unordered_map<const void*, WsUse> g_ws;

bool capturing(cudaStream_t s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return cs != cudaStreamCaptureStatusNone;
}

hjcd_status ws_acquire(const void* ws, cudaStream_t s) {
    if (capturing(s)) return HJCD_OK;
    std::lock_guard<std::mutex> lk(g_ws_mu);
    auto it = g_ws.find(ws);
    if (it == g_ws.end() || it->second.s == s || !it->second.ev) return HJCD_OK;
    cudaError_t e = cudaEventQuery(it->second.ev);
    if (e == cudaErrorNotReady) return HJCD_E_WORKSPACE;
    if (e != cudaSuccess) (void)cudaGetLastError();
    return HJCD_OK;
}

void ws_release(const void* ws, cudaStream_t s) {
    if (capturing(s)) return;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) { (void)cudaGetLastError(); return; }
    std::lock_guard<std::mutex> lk(g_ws_mu);
    WsUse& u = g_ws[ws];
    if (u.ev && u.dev != dev) { cudaEventDestroy(u.ev); u.ev = nullptr; }
    if (!u.ev && cudaEventCreateWithFlags(&u.ev, cudaEventDisableTiming) != cudaSuccess) {
        (void)cudaGetLastError();
        u.ev = nullptr;
        return;
    }
    u.dev = dev;
    u.s = s;
    if (cudaEventRecord(u.ev, s) != cudaSuccess) (void)cudaGetLastError();
}

// acquired for the scope of one solve's launches; marks the workspace busy on
// `s` until the work enqueued in that scope completes
struct WsScope {
    const void* ws;
    cudaStream_t s;
    ~WsScope() { ws_release(ws, s); }
};

struct Layout {
    size_t theta1, cost1, seeds2, ep2, eo2, ready, total;
};

constexpr int kOrderMaxTargets = 5000;   // (A/B: HJCD_ORDER_MAX)

Layout layout(int dof, long long T, const hjcd_config* c) {
    Layout L;
    size_t off = 0;
    L.theta1 = off; off += align256((size_t)T * dof * c->M * sizeof(float));
    L.cost1 = off;  off += align256((size_t)T * c->M * sizeof(float));
    L.seeds2 = off; off += align256((size_t)T * c->B * dof * sizeof(float));
    L.ep2 = off;    off += align256((size_t)T * c->B * sizeof(float));
    L.eo2 = off;    off += align256((size_t)T * c->B * sizeof(float));
    // K10 per-target PO-CCD completion counts [T], then the K26 polish-order
    // stacks (next [T], heads [shards][buckets], pushed, popped)
    L.ready = off;  off += align256((size_t)((2 * T + kReadyWords + 63) & ~63) * sizeof(uint32_t));
#ifdef HJCD_PROBE
    off += align256(5 * (size_t)T * 8);
#endif
    L.total = off;
    return L;
}

#ifdef HJCD_PROBE
unsigned long long* g_probe = nullptr;
int g_probe_T = 0;
#endif

// hjcd_solve's launch sequence without stage events (DESIGN K10): PO-CCD
// (lockstep clusters) counts each target's finished CTAs into `ready`; PJ-IK is
// its programmatic dependent and starts on a target as soon as that target's
// stage 1 is done, doing top-K + replication in its prologue, so the polish
// of early targets overlaps the tail of PO-CCD. Needs the per-target PO-CCD
// stop rule (R12b, one cluster per target); the per-seed break uses the
// staged sequence. `final` launches Alg. 2 l.10 (best-select or best-N).
template <class Final>
cudaError_t solve_linked(const hjcd_robot* r, const DevCfg& d, const float* targets, int T, const Layout& L,
                         char* ws, cudaStream_t s, Final final) {
    float* theta1 = (float*)(ws + L.theta1);
    float* cost1 = (float*)(ws + L.cost1);
    float* seeds2 = (float*)(ws + L.seeds2);
    float* ep2 = (float*)(ws + L.ep2);
    float* eo2 = (float*)(ws + L.eo2);
    cudaError_t e;
    if (!d.ccd_early_exit) {
        if ((e = launch_poccd(r->dev, d, targets, T, nullptr, theta1, cost1, nullptr, nullptr, nullptr, s)) !=
                cudaSuccess ||
            (e = launch_select_replicate(r->dev, d, cost1, theta1, T, seeds2, nullptr, s)) != cudaSuccess ||
            (e = launch_pjik(r->dev, d, targets, T, seeds2, seeds2, ep2, eo2, nullptr, nullptr, s)) != cudaSuccess)
            return e;
        return final(seeds2, ep2, eo2);
    }
    StageLink link;
    link.ready = (uint32_t*)(ws + L.ready);
    link.cost = cost1;
    link.theta = theta1;
    link.need = (uint32_t)poccd_cluster_ctas(d.M, r->dof);
    link.spin_limit = (1ull << 26) * (unsigned long long)(1 + d.ccd_iters / 64);
    link.Mpad = 2;
    while (link.Mpad < d.M) link.Mpad <<= 1;
    // K26: the stop-iteration order (C2 -2 %, 300 targets -9 %, 2000 -8 %,
    // 4000 -6 %); with every polish CTA resident at once (<= 2 per SM) the
    // order is moot and the pops only add traffic (100 targets +12 %); from
    // ~10k targets the tail is amortised and the claims cost about what the
    // order gains (Panda -1 %, Fetch-like 0, 14-DoF +1 %), so those run in
    // target order.  The sharded stacks (K30) keep the claims free of
    // contention: profiles/r02t_k26_polish_order_ab.log, r02y_*
    int dev = 0, nsm = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaGetLastError();
    static const int order_max = [] {   // A/B override of the K26 batch bound
        const char* v = std::getenv("HJCD_ORDER_MAX");
        return v ? std::atoi(v) : kOrderMaxTargets;
    }();
    link.order = (T > 2 * nsm && T <= order_max) ? 1 : 0;
#ifdef HJCD_PROBE
    g_probe = (unsigned long long*)(link.ready + ((2 * T + kReadyWords + 63) & ~63));
    g_probe_T = T;
    if ((e = cudaMemsetAsync(g_probe, 0xff, (size_t)T * 8, s)) != cudaSuccess ||
        (e = cudaMemsetAsync(g_probe + T, 0, 4 * (size_t)T * 8, s)) != cudaSuccess)
        return e;
#endif
    if ((e = cudaMemsetAsync(link.ready, 0, (size_t)(2 * T + kReadyWords) * sizeof(uint32_t), s)) != cudaSuccess ||
        (e = launch_poccd(r->dev, d, targets, T, nullptr, theta1, cost1, nullptr, nullptr, nullptr, s, TraceOut(),
                          link.ready)) != cudaSuccess ||
        (e = launch_pjik(r->dev, d, targets, T, nullptr, seeds2, ep2, eo2, nullptr, nullptr, s, link)) != cudaSuccess)
        return e;
    return final(seeds2, ep2, eo2);
}

struct Layout64 {
    size_t theta1, cost1, seeds2, theta64, ep64, eo64, total;
};

Layout64 layout64(int dof, long long T, const hjcd_config* c) {
    Layout64 L;
    size_t off = 0;
    L.theta1 = off;  off += align256((size_t)T * dof * c->M * sizeof(float));
    L.cost1 = off;   off += align256((size_t)T * c->M * sizeof(float));
    L.seeds2 = off;  off += align256((size_t)T * c->B * dof * sizeof(float));
    L.theta64 = off; off += align256((size_t)T * c->B * dof * sizeof(double));
    L.ep64 = off;    off += align256((size_t)T * c->B * sizeof(double));
    L.eo64 = off;    off += align256((size_t)T * c->B * sizeof(double));
    L.total = off;
    return L;
}

size_t host_staging(int dof, long long T) {
    return align256((size_t)T * 7 * 4) + align256((size_t)T * dof * 4) + 3 * align256((size_t)T * 4);
}

}  // namespace

extern "C" {

#ifdef HJCD_PROBE
// A/B diagnostic build only: copies the last linked solve's [5][T] stamps
int hjcd_debug_probe(unsigned long long* host, int T) {
    if (!g_probe || T != g_probe_T) return -1;
    return (int)cudaMemcpy(host, g_probe, 5 * (size_t)T * 8, cudaMemcpyDeviceToHost);
}
#endif

hjcd_status hjcd_robot_create(const hjcd_joint* joints, int32_t num_joints, const double ee_xyz[3],
                              const double ee_quat_wxyz[4], hjcd_robot** out) {
    return build_robot(joints, num_joints, ee_xyz, ee_quat_wxyz, out);
}

hjcd_status hjcd_robot_extend(const hjcd_robot* r, int32_t target_dof, hjcd_robot** out) {
    if (!r || !out) return HJCD_E_INVALID_ARG;
    if (target_dof < r->dof) return HJCD_E_INVALID_ARG;
    if (target_dof > HJCD_MAX_DOF) return HJCD_E_UNSUPPORTED;
    // cyclic replicas of the DoF joints (R34) go before the end-effector
    // offset, which includes any trailing run of FIXED joints (SPEC extend_dof)
    std::vector<hjcd_joint> base;
    for (const hjcd_joint& j : r->joints)
        if (j.type != HJCD_FIXED) base.push_back(j);
    size_t tail = r->joints.size();
    while (tail > 0 && r->joints[tail - 1].type == HJCD_FIXED) --tail;
    std::vector<hjcd_joint> all(r->joints.begin(), r->joints.begin() + tail);
    int d = r->dof;
    for (size_t i = 0; d < target_dof; ++i, ++d) all.push_back(base[i % base.size()]);
    all.insert(all.end(), r->joints.begin() + tail, r->joints.end());
    return build_robot(all.data(), (int32_t)all.size(), r->ee_xyz, r->ee_quat, out);
}

void hjcd_robot_destroy(hjcd_robot* r) { delete r; }

int32_t hjcd_robot_dof(const hjcd_robot* r) { return r ? r->dof : 0; }

hjcd_status hjcd_robot_limits(const hjcd_robot* r, float* lo, float* hi) {
    if (!r || !lo || !hi) return HJCD_E_INVALID_ARG;
    for (int j = 0; j < r->dof; ++j) { lo[j] = r->dev.j[j].lo; hi[j] = r->dev.j[j].hi; }
    return HJCD_OK;
}

void hjcd_config_default(hjcd_config* c) {
    if (!c) return;
    std::memset(c, 0, sizeof(*c));
    c->M = 1000; c->K = 50; c->B = 100;            // R16
    c->ccd_iters = 64; c->lm_iters = 128;          // R28
    c->target_early_exit = 1;                           // R26b
    c->ccd_early_exit = 1;                              // R12b
    c->eps_p_coarse = 5e-3f; c->eps_o_coarse = 5e-2f;   // R12
    c->eps_p_fine = 1e-6f; c->eps_o_fine = 1e-5f;       // R26
    c->gamma = 1e-6f;                                   // R10
    c->delta0 = 1.f; c->delta_rho = 0.98f; c->delta_min = 0.1f;   // R5
    c->sigma_ccd = 0.05f; c->sigma_rep = 0.02f; c->sigma_lm = 0.05f;   // R11, R15, R25
    c->lambda = 1e-3f; c->d_floor = 1e-8f; c->R = 0.5f; c->beta = 2.f; c->A = 8;   // R20-R22
    c->w_p = 1.f; c->w_o = 0.5f;                        // R17
    c->succ_p = 1e-3f; c->succ_o = 0.017453292519943295f;
    c->tau_deg = 1e-5f;                                 // R4
    c->repl_noise_all = 0;                              // R15
    c->rng_seed = 0;
    c->target_index_offset = 0;
}

hjcd_status hjcd_workspace_size(const hjcd_robot* r, int32_t T, const hjcd_config* c, size_t* bytes) {
    if (!r || !c || !bytes || T < 1) return HJCD_E_INVALID_ARG;
    DevCfg d;
    hjcd_status st = make_cfg(r, c, &d);
    if (st != HJCD_OK) return st;
    if ((st = check_poccd(c)) != HJCD_OK) return st;
    *bytes = layout(r->dof, T, c).total;
    return HJCD_OK;
}

hjcd_status hjcd_workspace_size_host(const hjcd_robot* r, int32_t T, const hjcd_config* c, size_t* bytes) {
    hjcd_status st = hjcd_workspace_size(r, T, c, bytes);
    if (st != HJCD_OK) return st;
    *bytes += host_staging(r->dof, T);
    return HJCD_OK;
}

hjcd_status hjcd_solve(const hjcd_robot* r, const hjcd_config* c, const float* targets, int32_t T,
                       float* q_out, float* pos_err, float* ori_err, int32_t* status, void* workspace,
                       size_t workspace_bytes, hjcd_stream_t stream) {
    return hjcd_solve_timed(r, c, targets, T, q_out, pos_err, ori_err, status, workspace, workspace_bytes,
                            stream, nullptr);
}

hjcd_status hjcd_solve_timed(const hjcd_robot* r, const hjcd_config* c, const float* targets, int32_t T,
                             float* q_out, float* pos_err, float* ori_err, int32_t* status, void* workspace,
                             size_t workspace_bytes, hjcd_stream_t stream, void* const* events) {
    if (!r || !c || !targets || T < 1 || !q_out || !pos_err || !ori_err || !status || !workspace)
        return HJCD_E_INVALID_ARG;
    DevCfg d;
    hjcd_status st = make_cfg(r, c, &d);
    if (st != HJCD_OK) return st;
    if (c->M > 8192) return HJCD_E_UNSUPPORTED;
    if ((st = check_poccd(c)) != HJCD_OK) return st;
    Layout L = layout(r->dof, T, c);
    if (workspace_bytes < L.total || ((uintptr_t)workspace & 255)) return HJCD_E_WORKSPACE;
    char* ws = (char*)workspace;
    float* theta1 = (float*)(ws + L.theta1);
    float* cost1 = (float*)(ws + L.cost1);
    float* seeds2 = (float*)(ws + L.seeds2);
    float* ep2 = (float*)(ws + L.ep2);
    float* eo2 = (float*)(ws + L.eo2);
    cudaStream_t s = (cudaStream_t)stream;
    if ((st = ws_acquire(workspace, s)) != HJCD_OK) return st;
    WsScope busy{workspace, s};
    cudaError_t e;
    auto mark = [&](int i) -> cudaError_t {
        return (events && events[i]) ? cudaEventRecord((cudaEvent_t)events[i], s) : cudaSuccess;
    };
    // K33: at >= 12 DoF and >= 5000 targets the staged sequence is faster than
    // the dependent launch (C4: 35.9 vs 36.3 ms): the 14-DoF polish CTAs
    // (255 registers) overlapping PO-CCD's last wave and doing the top-K
    // themselves cost more than the separate top-K kernel
    const bool staged = T >= 5000 && r->dof >= 12;
    if (!events && !staged) {   // DESIGN K10: PJ-IK as a dependent launch of PO-CCD
        e = solve_linked(r, d, targets, T, L, ws, s, [&](const float* th, const float* ep, const float* eo) {
            return launch_select_best(r->dev, d, targets, T, th, ep, eo, q_out, pos_err, ori_err, status, s);
        });
        return e == cudaSuccess ? HJCD_OK : cuda_fail(e);
    }
    // stage events requested (or K33): the staged sequence, one kernel per stage
    if ((e = mark(0)) != cudaSuccess) return cuda_fail(e);
    // Alg. 2 l.1: PO-CCD over M seeds per target
    if ((e = launch_poccd(r->dev, d, targets, T, nullptr, theta1, cost1, nullptr, nullptr, nullptr, s)) != cudaSuccess ||
        (e = mark(1)) != cudaSuccess)
        return cuda_fail(e);
    // Alg. 2 l.2-8: top-K + replicate
    if ((e = launch_select_replicate(r->dev, d, cost1, theta1, T, seeds2, nullptr, s)) != cudaSuccess ||
        (e = mark(2)) != cudaSuccess)
        return cuda_fail(e);
    // Alg. 2 l.9 / Alg. 4: PJ-IK, in place on the replicated seeds
    if ((e = launch_pjik(r->dev, d, targets, T, seeds2, seeds2, ep2, eo2, nullptr, nullptr, s)) != cudaSuccess ||
        (e = mark(3)) != cudaSuccess)
        return cuda_fail(e);
    // Alg. 2 l.10: best of B
    if ((e = launch_select_best(r->dev, d, targets, T, seeds2, ep2, eo2, q_out, pos_err, ori_err, status, s)) !=
            cudaSuccess ||
        (e = mark(4)) != cudaSuccess)
        return cuda_fail(e);
    return HJCD_OK;
}

hjcd_status hjcd_solve_batch(const hjcd_robot* r, const hjcd_config* c, const float* targets, int32_t T, int32_t N,
                             float* q_out, float* pos_err, float* ori_err, int32_t* status, void* workspace,
                             size_t workspace_bytes, hjcd_stream_t stream) {
    if (!r || !c || !targets || T < 1 || !q_out || !pos_err || !ori_err || !status || !workspace)
        return HJCD_E_INVALID_ARG;
    DevCfg d;
    hjcd_status st = make_cfg(r, c, &d);
    if (st != HJCD_OK) return st;
    if (N < 1 || N > d.copies * d.K) return HJCD_E_INVALID_ARG;
    if (c->M > 8192) return HJCD_E_UNSUPPORTED;
    if ((st = check_poccd(c)) != HJCD_OK) return st;
    Layout L = layout(r->dof, T, c);
    if (workspace_bytes < L.total || ((uintptr_t)workspace & 255)) return HJCD_E_WORKSPACE;
    char* ws = (char*)workspace;
    cudaStream_t s = (cudaStream_t)stream;
    if ((st = ws_acquire(workspace, s)) != HJCD_OK) return st;
    WsScope busy{workspace, s};
    cudaError_t e = solve_linked(r, d, targets, T, L, ws, s, [&](const float* th, const float* ep, const float* eo) {
        return launch_select_topn(r->dev, d, targets, T, th, ep, eo, N, q_out, pos_err, ori_err, nullptr, status, s);
    });
    return e == cudaSuccess ? HJCD_OK : cuda_fail(e);
}

hjcd_status hjcd_workspace_size_f64(const hjcd_robot* r, int32_t T, const hjcd_config* c, size_t* bytes) {
    if (!r || !c || !bytes || T < 1) return HJCD_E_INVALID_ARG;
    DevCfg d;
    hjcd_status st = make_cfg(r, c, &d);
    if (st != HJCD_OK) return st;
    if ((st = check_poccd(c)) != HJCD_OK) return st;
    *bytes = layout64(r->dof, T, c).total;
    return HJCD_OK;
}

hjcd_status hjcd_solve_f64(const hjcd_robot* r, const hjcd_config* c, const float* targets, int32_t T,
                           double* q_out, double* pos_err, double* ori_err, int32_t* status, void* workspace,
                           size_t workspace_bytes, hjcd_stream_t stream) {
    if (!r || !c || !targets || T < 1 || !q_out || !pos_err || !ori_err || !status || !workspace)
        return HJCD_E_INVALID_ARG;
    DevCfg d;
    hjcd_status st = make_cfg(r, c, &d);
    if (st != HJCD_OK) return st;
    if (c->M > 8192) return HJCD_E_UNSUPPORTED;
    if ((st = check_poccd(c)) != HJCD_OK) return st;
    Layout64 L = layout64(r->dof, T, c);
    if (workspace_bytes < L.total || ((uintptr_t)workspace & 255)) return HJCD_E_WORKSPACE;
    char* ws = (char*)workspace;
    float* theta1 = (float*)(ws + L.theta1);
    float* cost1 = (float*)(ws + L.cost1);
    float* seeds2 = (float*)(ws + L.seeds2);
    double* th64 = (double*)(ws + L.theta64);
    double* ep64 = (double*)(ws + L.ep64);
    double* eo64 = (double*)(ws + L.eo64);
    cudaStream_t s = (cudaStream_t)stream;
    if ((st = ws_acquire(workspace, s)) != HJCD_OK) return st;
    WsScope busy{workspace, s};
    cudaError_t e;
    // stage 1 and the hand-over in fp32 (PO-CCD only needs the coarse
    // tolerance), stage 2 and the answer in fp64 on the fp64 chain (f1)
    if ((e = launch_poccd(r->dev, d, targets, T, nullptr, theta1, cost1, nullptr, nullptr, nullptr, s)) != cudaSuccess ||
        (e = launch_select_replicate(r->dev, d, cost1, theta1, T, seeds2, nullptr, s)) != cudaSuccess ||
        (e = launch_pjik64(r->dev64, d, targets, T, seeds2, th64, ep64, eo64, nullptr, nullptr, s)) != cudaSuccess ||
        (e = launch_select_best(r->dev, d, targets, T, (const double*)th64, (const double*)ep64, (const double*)eo64,
                                q_out, pos_err, ori_err, status, s)) != cudaSuccess)
        return cuda_fail(e);
    return HJCD_OK;
}

hjcd_status hjcd_pjik_f64(const hjcd_robot* r, const hjcd_config* c, const float* targets, int32_t T,
                          const float* seeds, double* theta, double* pos_err, double* ori_err, int32_t* step_counts,
                          int32_t* iters, hjcd_stream_t stream) {
    if (!r || !c || !targets || T < 1 || !seeds || !theta || !pos_err || !ori_err) return HJCD_E_INVALID_ARG;
    DevCfg d;
    hjcd_status st = make_cfg(r, c, &d);
    if (st != HJCD_OK) return st;
    cudaError_t e = launch_pjik64(r->dev64, d, targets, T, seeds, theta, pos_err, ori_err, step_counts, iters,
                                  (cudaStream_t)stream);
    return e == cudaSuccess ? HJCD_OK : cuda_fail(e);
}

hjcd_status hjcd_select_topn(const hjcd_robot* r, const hjcd_config* c, const float* targets, int32_t T,
                             const float* theta, const float* pos_err_all, const float* ori_err_all, int32_t N,
                             float* q_out, float* pos_err, float* ori_err, int32_t* idx, hjcd_stream_t stream) {
    if (!r || !c || !targets || T < 1 || !theta || !pos_err_all || !ori_err_all || !q_out || !pos_err || !ori_err)
        return HJCD_E_INVALID_ARG;
    DevCfg d;
    hjcd_status st = make_cfg(r, c, &d);
    if (st != HJCD_OK) return st;
    if (N < 1 || N > d.copies * d.K) return HJCD_E_INVALID_ARG;
    cudaError_t e = launch_select_topn(r->dev, d, targets, T, theta, pos_err_all, ori_err_all, N, q_out, pos_err,
                                       ori_err, idx, nullptr, (cudaStream_t)stream);
    return e == cudaSuccess ? HJCD_OK : cuda_fail(e);
}

hjcd_status hjcd_mmd(const float* X, int32_t N, const float* Y, int32_t N2, int32_t dim, int32_t T, float* mmd2,
                     float* bandwidth, hjcd_stream_t stream) {
    if (!X || !Y || !mmd2 || N < 1 || N2 < 1 || T < 1 || dim < 1 || dim > HJCD_MAX_DOF) return HJCD_E_INVALID_ARG;
    if (N + N2 > 256) return HJCD_E_UNSUPPORTED;
    cudaError_t e = launch_mmd(X, N, Y, N2, dim, T, mmd2, bandwidth, (cudaStream_t)stream);
    return e == cudaSuccess ? HJCD_OK : cuda_fail(e);
}

hjcd_status hjcd_solve_host(const hjcd_robot* r, const hjcd_config* c, const float* targets_host, int32_t T,
                            float* q_host, float* pos_err_host, float* ori_err_host, int32_t* status_host,
                            void* workspace, size_t workspace_bytes, hjcd_stream_t stream) {
    if (!r || !c || !targets_host || T < 1 || !q_host || !pos_err_host || !ori_err_host || !status_host ||
        !workspace)
        return HJCD_E_INVALID_ARG;
    size_t need = 0;
    hjcd_status st = hjcd_workspace_size(r, T, c, &need);
    if (st != HJCD_OK) return st;
    const size_t stage = host_staging(r->dof, T);
    if (workspace_bytes < need + stage || ((uintptr_t)workspace & 255)) return HJCD_E_WORKSPACE;
    char* io = (char*)workspace + need;
    float* tg = (float*)io;            io += align256((size_t)T * 7 * 4);
    float* q = (float*)io;             io += align256((size_t)T * r->dof * 4);
    float* pe = (float*)io;            io += align256((size_t)T * 4);
    float* oe = (float*)io;            io += align256((size_t)T * 4);
    int32_t* stt = (int32_t*)io;
    cudaStream_t s = (cudaStream_t)stream;
    if ((st = ws_acquire(workspace, s)) != HJCD_OK) return st;
    cudaError_t e;
    if ((e = cudaMemcpyAsync(tg, targets_host, (size_t)T * 7 * 4, cudaMemcpyHostToDevice, s)) != cudaSuccess)
        return cuda_fail(e);
    st = hjcd_solve(r, c, tg, T, q, pe, oe, stt, workspace, need, stream);
    if (st != HJCD_OK) return st;
    if ((e = cudaMemcpyAsync(q_host, q, (size_t)T * r->dof * 4, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
        (e = cudaMemcpyAsync(pos_err_host, pe, (size_t)T * 4, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
        (e = cudaMemcpyAsync(ori_err_host, oe, (size_t)T * 4, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
        (e = cudaMemcpyAsync(status_host, stt, (size_t)T * 4, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
        return cuda_fail(e);
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e);
    return HJCD_OK;
}

hjcd_status hjcd_fk(const hjcd_robot* r, const float* q, int32_t N, float* pose7, float* jac,
                    hjcd_stream_t stream) {
    if (!r || !q || N < 1 || !pose7) return HJCD_E_INVALID_ARG;
    cudaError_t e = launch_fk(r->dev, q, N, pose7, jac, (cudaStream_t)stream);
    return e == cudaSuccess ? HJCD_OK : cuda_fail(e);
}

hjcd_status hjcd_fk_sfu(const hjcd_robot* r, const float* q, int32_t N, float* pose7, float* jac,
                        hjcd_stream_t stream) {
    if (!r || !q || N < 1 || !pose7) return HJCD_E_INVALID_ARG;
    cudaError_t e = launch_fk(r->dev, q, N, pose7, jac, (cudaStream_t)stream, true);
    return e == cudaSuccess ? HJCD_OK : cuda_fail(e);
}

hjcd_status hjcd_pose_error_f64(const hjcd_robot* r, const float* q, const float* targets, int32_t N,
                                double* pos_err, double* ori_err, hjcd_stream_t stream) {
    if (!r || !q || !targets || N < 1 || !pos_err || !ori_err) return HJCD_E_INVALID_ARG;
    cudaError_t e = launch_pose_error64(r->dev64, q, targets, N, pos_err, ori_err, (cudaStream_t)stream);
    return e == cudaSuccess ? HJCD_OK : cuda_fail(e);
}

hjcd_status hjcd_poccd(const hjcd_robot* r, const hjcd_config* c, const float* targets, int32_t T,
                       const float* seeds, float* theta, float* cost, float* pos_err, float* ori_err,
                       int32_t* iters, hjcd_stream_t stream) {
    if (!r || !c || !targets || T < 1 || !theta || !cost) return HJCD_E_INVALID_ARG;
    DevCfg d;
    hjcd_status st = make_cfg(r, c, &d);
    if (st != HJCD_OK) return st;
    if ((st = check_poccd(c)) != HJCD_OK) return st;
    cudaError_t e = launch_poccd(r->dev, d, targets, T, seeds, theta, cost, pos_err, ori_err, iters,
                                 (cudaStream_t)stream);
    return e == cudaSuccess ? HJCD_OK : cuda_fail(e);
}

hjcd_status hjcd_ccd(const hjcd_robot* r, const hjcd_config* c, const float* targets, int32_t T, const float* seeds,
                     float* theta, float* pos_err, int32_t* iters, hjcd_stream_t stream) {
    if (!r || !c || !targets || T < 1 || !theta) return HJCD_E_INVALID_ARG;
    DevCfg d;
    hjcd_status st = make_cfg(r, c, &d);
    if (st != HJCD_OK) return st;
    cudaError_t e = launch_ccd(r->dev, d, targets, T, seeds, theta, pos_err, iters, (cudaStream_t)stream);
    return e == cudaSuccess ? HJCD_OK : cuda_fail(e);
}

hjcd_status hjcd_poccd_trace(const hjcd_robot* r, const hjcd_config* c, const float* targets, int32_t T,
                             const float* seeds, float* theta, float* cost, float* pos_err, float* ori_err,
                             int32_t* iters, uint32_t* trace, float* theta_hist, hjcd_stream_t stream) {
    if (!r || !c || !targets || T < 1 || !theta || !cost || !trace) return HJCD_E_INVALID_ARG;
    DevCfg d;
    hjcd_status st = make_cfg(r, c, &d);
    if (st != HJCD_OK) return st;
    if ((st = check_poccd(c)) != HJCD_OK) return st;
    TraceOut tr;
    tr.words = trace;
    tr.theta = theta_hist;
    cudaError_t e = launch_poccd(r->dev, d, targets, T, seeds, theta, cost, pos_err, ori_err, iters,
                                 (cudaStream_t)stream, tr);
    return e == cudaSuccess ? HJCD_OK : cuda_fail(e);
}

hjcd_status hjcd_select_replicate(const hjcd_robot* r, const hjcd_config* c, const float* cost,
                                  const float* theta, int32_t T, float* polish_seeds, int32_t* kept_idx,
                                  hjcd_stream_t stream) {
    if (!r || !c || !cost || !theta || T < 1 || !polish_seeds) return HJCD_E_INVALID_ARG;
    DevCfg d;
    hjcd_status st = make_cfg(r, c, &d);
    if (st != HJCD_OK) return st;
    if (c->M > 8192) return HJCD_E_UNSUPPORTED;
    cudaError_t e = launch_select_replicate(r->dev, d, cost, theta, T, polish_seeds, kept_idx, (cudaStream_t)stream);
    return e == cudaSuccess ? HJCD_OK : cuda_fail(e);
}

hjcd_status hjcd_pjik(const hjcd_robot* r, const hjcd_config* c, const float* targets, int32_t T,
                      const float* seeds, float* theta, float* pos_err, float* ori_err, int32_t* step_counts,
                      int32_t* iters, hjcd_stream_t stream) {
    if (!r || !c || !targets || T < 1 || !seeds || !theta || !pos_err || !ori_err) return HJCD_E_INVALID_ARG;
    DevCfg d;
    hjcd_status st = make_cfg(r, c, &d);
    if (st != HJCD_OK) return st;
    cudaError_t e = launch_pjik(r->dev, d, targets, T, seeds, theta, pos_err, ori_err, step_counts, iters,
                                (cudaStream_t)stream);
    return e == cudaSuccess ? HJCD_OK : cuda_fail(e);
}

hjcd_status hjcd_pjik_trace(const hjcd_robot* r, const hjcd_config* c, const float* targets, int32_t T,
                            const float* seeds, float* theta, float* pos_err, float* ori_err, int32_t* step_counts,
                            int32_t* iters, uint32_t* trace, float* theta_hist, hjcd_stream_t stream) {
    if (!r || !c || !targets || T < 1 || !seeds || !theta || !pos_err || !ori_err || !trace)
        return HJCD_E_INVALID_ARG;
    DevCfg d;
    hjcd_status st = make_cfg(r, c, &d);
    if (st != HJCD_OK) return st;
    StageLink extra;
    extra.trace = trace;
    extra.trace_theta = theta_hist;
    cudaError_t e = launch_pjik(r->dev, d, targets, T, seeds, theta, pos_err, ori_err, step_counts, iters,
                                (cudaStream_t)stream, extra);
    return e == cudaSuccess ? HJCD_OK : cuda_fail(e);
}

hjcd_status hjcd_select_best(const hjcd_robot* r, const hjcd_config* c, const float* targets, int32_t T,
                             const float* theta, const float* pos_err_all, const float* ori_err_all, float* q_out,
                             float* pos_err, float* ori_err, int32_t* status, hjcd_stream_t stream) {
    if (!r || !c || !targets || T < 1 || !theta || !pos_err_all || !ori_err_all || !q_out || !pos_err ||
        !ori_err || !status)
        return HJCD_E_INVALID_ARG;
    DevCfg d;
    hjcd_status st = make_cfg(r, c, &d);
    if (st != HJCD_OK) return st;
    cudaError_t e = launch_select_best(r->dev, d, targets, T, theta, pos_err_all, ori_err_all, q_out, pos_err,
                                       ori_err, status, (cudaStream_t)stream);
    return e == cudaSuccess ? HJCD_OK : cuda_fail(e);
}

const char* hjcd_status_string(hjcd_status s) {
    switch (s) {
        case HJCD_OK: return "ok";
        case HJCD_E_INVALID_ARG: return "invalid argument";
        case HJCD_E_UNSUPPORTED: return "unsupported";
        case HJCD_E_CUDA: return "CUDA error";
        case HJCD_E_WORKSPACE: return "workspace too small, misaligned, or in use on another stream";
        case HJCD_E_NOMEM: return "out of host memory";
    }
    return "unknown status";
}

const char* hjcd_poccd_kernel(const hjcd_robot* r, const hjcd_config* c) {
    if (!r || !c) return "";
    return poccd_uses_x2(r->dof, c->ccd_early_exit != 0) ? "k_poccd_x2" : "k_poccd";
}

const char* hjcd_last_cuda_error(void) { return g_cuda_err.c_str(); }

const char* hjcd_version(void) { return "hjcd 0.1 sm_100a"; }

}  // extern "C"

/*
 * hjcd_oracle.cpp — fp64 CPU ORACLE for HJCD-IK (arXiv 2510.07514).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * under paper_2510_07514_b200/csrc/; neither side includes the other.
 *
 * Written from PAPER.md ("P:NNN" = line of /root/reference/PAPER.md), plainly
 * and slowly, in fp64, following the paper's algorithms step by step:
 *   - FK as a literal product of 4x4 homogeneous matrices (Eq. 1);
 *   - geometric Jacobian columns [z_i x (P_ee - P_i); z_i] (Eq. 7);
 *   - quaternion error (Eq. 5) and angle-axis form (Eq. 10);
 *   - CCD projections and angle, literal normalise/project/arccos form
 *     (Eqs. 8-9);
 *   - PO-CCD (Alg. 3) scoring every candidate by a FULL FK of
 *     theta + dtheta*e_j (literal P:222), NOT the rigid-rotation shortcut the
 *     GPU uses;
 *   - top-K by stable sort + replication (Alg. 2 l.2-8);
 *   - PJ-IK (Alg. 4) solving the literal n x n weighted normal
 *     equations (Eq. 12) by Cholesky, NOT the GPU's 6x6
 *     push-through form; dogleg (Eqs. 14-15), single-coordinate
 *     (Eq. 16) and perturbation fallbacks.
 * Where the paper is silent/garbled the reading is the one recorded in
 * DESIGN.md "Readings" (R-numbers; the same ids as SURVEY.md §8(c) C1-C35).
 *
 * Random numbers: Philox4x32-10 (Random123 definition), counter-based, so both
 * sides draw the same uniforms (R30).  Uniform -> joint value is
 * evaluated in fp32 with an explicit fmaf so initial seeds are bitwise equal
 * (the one place fp32 appears here, by design); Gaussians via fp64 Box-Muller.
 *
 * Decision margins: every discrete decision (argmin, gamma test, convergence
 * test, line-search comparison, ...) records how far it was from flipping.  The
 * per-seed minimum lets the parity tests tell a genuine bug apart from an
 * fp32-vs-fp64 near-tie flip.
 */
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_MAXJ 64

extern "C" {

/* Robot as given by the user: a serial chain, base -> tip (D1).
 * type: 0 revolute, 1 prismatic, 2 fixed.  Only non-fixed joints are DoF. */
typedef struct {
    int32_t n;
    int32_t type[ORACLE_MAXJ];
    double origin_xyz[ORACLE_MAXJ][3];
    double origin_quat[ORACLE_MAXJ][4]; /* w x y z */
    double axis[ORACLE_MAXJ][3];
    double lo[ORACLE_MAXJ];
    double hi[ORACLE_MAXJ];
    double ee_xyz[3];
    double ee_quat[4];
} OracleRobot;

/* Algorithm parameters (Alg. 2-4 headers; defaults in
 * DESIGN.md R5, R11, R12, R15-R17, R20-R28). */
typedef struct {
    int32_t M, K, B;
    int32_t ccd_iters, lm_iters;
    double eps_p_coarse, eps_o_coarse;
    double eps_p_fine, eps_o_fine;
    double gamma, delta0, delta_rho, delta_min;
    double sigma_ccd, sigma_rep, sigma_lm;
    double lambda, d_floor, R, beta;
    int32_t A;
    double w_p, w_o;
    double succ_p, succ_o;
    double tau_deg;
    uint64_t rng_seed;
    int32_t repl_noise_all;
    int32_t target_early_exit;
    int32_t ccd_early_exit;
} OracleConfig;

} /* extern "C" */

namespace {

const double PI = 3.14159265358979323846;
const double INF = std::numeric_limits<double>::infinity();

/* ---------------- small fp64 linear algebra ---------------- */
struct V3 { double x, y, z; };
struct Qt { double w, x, y, z; };
struct H4 { double m[4][4]; };

V3 v3(double x, double y, double z) { V3 r = {x, y, z}; return r; }
V3 add(V3 a, V3 b) { return v3(a.x + b.x, a.y + b.y, a.z + b.z); }
V3 sub(V3 a, V3 b) { return v3(a.x - b.x, a.y - b.y, a.z - b.z); }
V3 scl(V3 a, double s) { return v3(a.x * s, a.y * s, a.z * s); }
double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
V3 cross(V3 a, V3 b) { return v3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x); }
double norm(V3 a) { return std::sqrt(dot(a, a)); }

H4 h_identity() {
    H4 h;
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) h.m[i][j] = (i == j) ? 1.0 : 0.0;
    return h;
}

H4 h_mul(const H4& a, const H4& b) {
    H4 c;
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
            double s = 0.0;
            for (int k = 0; k < 4; ++k) s += a.m[i][k] * b.m[k][j];
            c.m[i][j] = s;
        }
    return c;
}

/* rotation matrix of a unit quaternion (w,x,y,z) */
H4 h_from_pose(const double xyz[3], const double q_in[4]) {
    double w = q_in[0], x = q_in[1], y = q_in[2], z = q_in[3];
    double nq = std::sqrt(w * w + x * x + y * y + z * z);
    w /= nq; x /= nq; y /= nq; z /= nq;
    H4 h = h_identity();
    h.m[0][0] = 1 - 2 * (y * y + z * z); h.m[0][1] = 2 * (x * y - w * z);     h.m[0][2] = 2 * (x * z + w * y);
    h.m[1][0] = 2 * (x * y + w * z);     h.m[1][1] = 1 - 2 * (x * x + z * z); h.m[1][2] = 2 * (y * z - w * x);
    h.m[2][0] = 2 * (x * z - w * y);     h.m[2][1] = 2 * (y * z + w * x);     h.m[2][2] = 1 - 2 * (x * x + y * y);
    h.m[0][3] = xyz[0]; h.m[1][3] = xyz[1]; h.m[2][3] = xyz[2];
    return h;
}

/* Rodrigues rotation about unit axis a by angle t, as a 4x4 */
H4 h_rot_axis(V3 a, double t) {
    double na = norm(a);
    a = scl(a, 1.0 / na);
    double c = std::cos(t), s = std::sin(t), C = 1.0 - c;
    H4 h = h_identity();
    h.m[0][0] = c + a.x * a.x * C;       h.m[0][1] = a.x * a.y * C - a.z * s; h.m[0][2] = a.x * a.z * C + a.y * s;
    h.m[1][0] = a.y * a.x * C + a.z * s; h.m[1][1] = c + a.y * a.y * C;       h.m[1][2] = a.y * a.z * C - a.x * s;
    h.m[2][0] = a.z * a.x * C - a.y * s; h.m[2][1] = a.z * a.y * C + a.x * s; h.m[2][2] = c + a.z * a.z * C;
    return h;
}

H4 h_trans_axis(V3 a, double d) {
    double na = norm(a);
    H4 h = h_identity();
    h.m[0][3] = a.x / na * d; h.m[1][3] = a.y / na * d; h.m[2][3] = a.z / na * d;
    return h;
}

/* rotation matrix -> unit quaternion (Shepperd), canonical w >= 0 (D2) */
Qt quat_from_h(const H4& h) {
    double r00 = h.m[0][0], r11 = h.m[1][1], r22 = h.m[2][2];
    double tr = r00 + r11 + r22;
    Qt q;
    if (tr > 0) {
        double s = std::sqrt(tr + 1.0) * 2.0;
        q.w = 0.25 * s;
        q.x = (h.m[2][1] - h.m[1][2]) / s;
        q.y = (h.m[0][2] - h.m[2][0]) / s;
        q.z = (h.m[1][0] - h.m[0][1]) / s;
    } else if (r00 > r11 && r00 > r22) {
        double s = std::sqrt(1.0 + r00 - r11 - r22) * 2.0;
        q.w = (h.m[2][1] - h.m[1][2]) / s;
        q.x = 0.25 * s;
        q.y = (h.m[0][1] + h.m[1][0]) / s;
        q.z = (h.m[0][2] + h.m[2][0]) / s;
    } else if (r11 > r22) {
        double s = std::sqrt(1.0 + r11 - r00 - r22) * 2.0;
        q.w = (h.m[0][2] - h.m[2][0]) / s;
        q.x = (h.m[0][1] + h.m[1][0]) / s;
        q.y = 0.25 * s;
        q.z = (h.m[1][2] + h.m[2][1]) / s;
    } else {
        double s = std::sqrt(1.0 + r22 - r00 - r11) * 2.0;
        q.w = (h.m[1][0] - h.m[0][1]) / s;
        q.x = (h.m[0][2] + h.m[2][0]) / s;
        q.y = (h.m[1][2] + h.m[2][1]) / s;
        q.z = 0.25 * s;
    }
    double nq = std::sqrt(q.w * q.w + q.x * q.x + q.y * q.y + q.z * q.z);
    q.w /= nq; q.x /= nq; q.y /= nq; q.z /= nq;
    if (q.w < 0) { q.w = -q.w; q.x = -q.x; q.y = -q.y; q.z = -q.z; }
    return q;
}

/* Hamilton product a (x) b */
Qt qmul(Qt a, Qt b) {
    Qt r;
    r.w = a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z;
    r.x = a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y;
    r.y = a.w * b.y - a.x * b.z + a.y * b.w + a.z * b.x;
    r.z = a.w * b.z + a.x * b.y - a.y * b.x + a.z * b.w;
    return r;
}
Qt qconj(Qt a) { Qt r = {a.w, -a.x, -a.y, -a.z}; return r; }

/* ---------------- robot + FK ---------------- */
struct Robot {
    const OracleRobot* r;
    int dof;
    std::vector<int> dof_entry; /* dof index -> entry in r arrays */
};

Robot make_robot(const OracleRobot* r) {
    Robot rb;
    rb.r = r;
    rb.dof = 0;
    for (int i = 0; i < r->n; ++i)
        if (r->type[i] != 2) { rb.dof_entry.push_back(i); rb.dof++; }
    return rb;
}

struct Frames {
    std::vector<V3> P;  /* P_i: world position of joint i (Eq. 7) */
    std::vector<V3> z;  /* z_i: world axis of joint i (Eq. 7) */
    V3 pee;             /* end-effector position */
    Qt qee;             /* end-effector orientation, w >= 0 */
};

/* Eq. 1: P_ee = f(theta); literal product
 * T = Origin_1 * Joint_1(theta_1) * ... * Origin_n * Joint_n(theta_n) * EE. */
void fk(const Robot& rb, const double* theta, Frames& F) {
    const OracleRobot* r = rb.r;
    F.P.assign(rb.dof, v3(0, 0, 0));
    F.z.assign(rb.dof, v3(0, 0, 0));
    H4 T = h_identity();
    int d = 0;
    for (int i = 0; i < r->n; ++i) {
        T = h_mul(T, h_from_pose(r->origin_xyz[i], r->origin_quat[i]));
        if (r->type[i] == 2) continue;
        V3 a = v3(r->axis[i][0], r->axis[i][1], r->axis[i][2]);
        a = scl(a, 1.0 / norm(a));
        if (r->type[i] == 0) T = h_mul(T, h_rot_axis(a, theta[d]));
        else T = h_mul(T, h_trans_axis(a, theta[d]));
        F.P[d] = v3(T.m[0][3], T.m[1][3], T.m[2][3]);
        F.z[d] = v3(T.m[0][0] * a.x + T.m[0][1] * a.y + T.m[0][2] * a.z,
                    T.m[1][0] * a.x + T.m[1][1] * a.y + T.m[1][2] * a.z,
                    T.m[2][0] * a.x + T.m[2][1] * a.y + T.m[2][2] * a.z);
        d++;
    }
    T = h_mul(T, h_from_pose(r->ee_xyz, r->ee_quat));
    F.pee = v3(T.m[0][3], T.m[1][3], T.m[2][3]);
    F.qee = quat_from_h(T);
}

/* Eq. 7: J columns [z_i x (P_ee - P_i); z_i] (revolute);
 * prismatic extension [z_i; 0] (R32).  J row-major 6 x dof. */
void jacobian(const Robot& rb, const Frames& F, double* J) {
    int n = rb.dof;
    for (int d = 0; d < n; ++d) {
        int e = rb.dof_entry[d];
        V3 col_p, col_o;
        if (rb.r->type[e] == 0) {
            col_p = cross(F.z[d], sub(F.pee, F.P[d]));
            col_o = F.z[d];
        } else {
            col_p = F.z[d];
            col_o = v3(0, 0, 0);
        }
        J[0 * n + d] = col_p.x; J[1 * n + d] = col_p.y; J[2 * n + d] = col_p.z;
        J[3 * n + d] = col_o.x; J[4 * n + d] = col_o.y; J[5 * n + d] = col_o.z;
    }
}

/* Eq. 5: q_err = q_t (x) q_e^-1 = [w, v];
 * omega = 2 atan2(|v|, |w|)/|v| * v, with q_err canonicalised to w >= 0 first
 * (R1: the literal |w| with un-flipped v negates omega when w < 0). */
V3 quat_error(Qt qt, Qt qe) {
    Qt q = qmul(qt, qconj(qe));
    if (q.w < 0) { q.w = -q.w; q.x = -q.x; q.y = -q.y; q.z = -q.z; }
    V3 v = v3(q.x, q.y, q.z);
    double s = norm(v);
    if (s < 1e-300) return scl(v, 2.0 / q.w); /* smooth limit 2v/w */
    return scl(v, 2.0 * std::atan2(s, q.w) / s);
}

/* Eq. 10: phi = 2 arccos(w), a = v / sin(phi/2), after the w >= 0
 * canonicalisation (R2).  phi < 1e-9 => caller treats the update as zero. */
void angle_axis(Qt qt, Qt qe, double* phi, V3* a) {
    Qt q = qmul(qt, qconj(qe));
    if (q.w < 0) { q.w = -q.w; q.x = -q.x; q.y = -q.y; q.z = -q.z; }
    double w = std::min(1.0, q.w);
    *phi = 2.0 * std::acos(w);
    double s = std::sin(*phi / 2.0);
    if (*phi < 1e-9 || s <= 0) { *phi = 0; *a = v3(0, 0, 1); return; }
    *a = scl(v3(q.x, q.y, q.z), 1.0 / s);
}

/* ---------------- Philox4x32-10 (Random123), R30 ---------------- */
void philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
    uint32_t k[2] = {key_in[0], key_in[1]};
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k[0] += 0x9E3779B9u; k[1] += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c[0];
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c[2];
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c[1] ^ k[0];
        uint32_t n2 = hi0 ^ c[3] ^ k[1];
        c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    }
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

enum { P_INIT = 1, P_PERTURB = 2, P_REPL = 3, P_PJPERT = 4 };

/* u = ((x >> 9) + 0.5) * 2^-23: exact in fp32, strictly inside (0, 1) */
double u01(uint32_t x) { return ((double)(x >> 9) + 0.5) * (1.0 / 8388608.0); }

/* the 4 uniforms of draw block `blk` of stream (tid, sid, purpose, iter) */
void draw4(uint64_t seed, uint64_t tid, uint32_t sid, uint32_t purpose, uint32_t iter,
           uint32_t blk, double u[4]) {
    uint32_t ctr[4] = {(uint32_t)tid, sid, (purpose << 24) | (iter & 0xFFFFFFu), blk};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t o[4];
    philox4x32_10(ctr, key, o);
    for (int i = 0; i < 4; ++i) u[i] = u01(o[i]);
}

/* standard normals for joint d: block d/4, Box-Muller pairs (u0,u1),(u2,u3) */
double normal_for_joint(uint64_t seed, uint64_t tid, uint32_t sid, uint32_t purpose,
                        uint32_t iter, int d) {
    double u[4];
    draw4(seed, tid, sid, purpose, iter, (uint32_t)(d / 4), u);
    int e = d % 4;
    int pair = e / 2;
    double ua = u[2 * pair], ub = u[2 * pair + 1];
    double rr = std::sqrt(-2.0 * std::log(ua));
    return (e % 2 == 0) ? rr * std::cos(2.0 * PI * ub) : rr * std::sin(2.0 * PI * ub);
}

double clampd(double x, double lo, double hi) { return std::min(std::max(x, lo), hi); }

/* ---------------- target ---------------- */
struct Target { V3 p; Qt q; bool valid; };

/* S2 / R-target: read fp32 pose, normalise q if | |q| - 1 | <= 1e-3 else invalid */
Target read_target(const float* t7) {
    Target t;
    t.p = v3(t7[0], t7[1], t7[2]);
    double w = t7[3], x = t7[4], y = t7[5], z = t7[6];
    double nq = std::sqrt(w * w + x * x + y * y + z * z);
    t.valid = std::fabs(nq - 1.0) <= 1e-3 && std::isfinite(nq) &&
              std::isfinite(t.p.x) && std::isfinite(t.p.y) && std::isfinite(t.p.z);
    if (!(nq > 0)) nq = 1;
    t.q.w = w / nq; t.q.x = x / nq; t.q.y = y / nq; t.q.z = z / nq;
    if (t.q.w < 0) { t.q.w = -t.q.w; t.q.x = -t.q.x; t.q.y = -t.q.y; t.q.z = -t.q.z; }
    return t;
}

struct Err { double ep, eo; V3 rp, om; };

/* Eq. 4: r = [P_t - P_ee, omega] */
Err residual(const Frames& F, const Target& t) {
    Err e;
    e.rp = sub(t.p, F.pee);
    e.om = quat_error(t.q, F.qee);
    e.ep = norm(e.rp);
    e.eo = norm(e.om);
    return e;
}

/* margins of boolean combinations of threshold tests (see header) */
double margin_and(bool a, double ma, bool b, double mb) {
    if (a && b) return std::min(ma, mb);
    if (a && !b) return mb;
    if (!a && b) return ma;
    return std::max(ma, mb);
}
double margin_or(bool a, double ma, bool b, double mb) {
    if (a && b) return std::max(ma, mb);
    if (a && !b) return ma;
    if (!a && b) return mb;
    return std::min(ma, mb);
}

/* ---------------- CCD steps ---------------- */
/* Eqs. 8-9, literal: normalise, project onto the plane of r_j,
 * arccos of the normalised projections (magnitude) with the sign of the triple
 * product z.(u_proj x v_proj) (R3).  Degenerate projection (R4): the raw
 * projections |P_ee - P_j|_perp or |P_t - P_j|_perp below tau_deg => 0.
 * Also returns the distance of the degeneracy tests from tau (margin). */
double ccd_position_step(V3 Pj, V3 rj, V3 pee, V3 pt, double tau, double* margin) {
    V3 uraw = sub(pee, Pj), vraw = sub(pt, Pj);
    double rr = dot(rj, rj);
    V3 uraw_p = sub(uraw, scl(rj, dot(uraw, rj) / rr));
    V3 vraw_p = sub(vraw, scl(rj, dot(vraw, rj) / rr));
    double nu = norm(uraw_p), nv = norm(vraw_p);
    /* a projection norm within a decade of tau is a live decision; far from it
     * (e.g. the ee exactly on the axis, nu ~ 1e-17) it is structural */
    if (margin) {
        *margin = INF;
        if (nu > 0.1 * tau && nu < 10 * tau) *margin = std::fabs(nu - tau);
        if (nv > 0.1 * tau && nv < 10 * tau) *margin = std::min(*margin, std::fabs(nv - tau));
    }
    if (nu < tau || nv < tau) return 0.0;
    V3 u = scl(uraw, 1.0 / norm(uraw));
    V3 v = scl(vraw, 1.0 / norm(vraw));
    V3 ur = scl(rj, dot(u, rj) / rr);
    V3 vr = scl(rj, dot(v, rj) / rr);
    V3 up = sub(u, ur), vp = sub(v, vr);
    double c = dot(scl(vp, 1.0 / norm(vp)), scl(up, 1.0 / norm(up)));
    double mag = std::acos(clampd(c, -1.0, 1.0));
    double sgn = dot(rj, cross(up, vp));
    /* |dtheta| near pi: the sign (branch cut of the signed angle) is a decision */
    if (margin) *margin = std::min(*margin, PI - mag);
    return (sgn > 0) ? mag : (sgn < 0 ? -mag : 0.0);
}

/* delta(k) = max(delta_min, delta0 * rho^k) (R5) */
double delta_k(const OracleConfig& c, int k) {
    return std::max(c.delta_min, c.delta0 * std::pow(c.delta_rho, (double)k));
}

/* Eq. 11: dtheta = delta(k) sgn(a . r_j) phi, sgn(0) = 0 */
double ccd_orientation_step(double phi, V3 a, V3 rj, double dk) {
    if (phi <= 0) return 0.0;
    double s = dot(a, rj);
    double sg = (s > 0) ? 1.0 : (s < 0 ? -1.0 : 0.0);
    return dk * sg * phi;
}

/* ---------------- PO-CCD one seed (Alg. 3) ---------------- */
struct SeedOut { double ep, eo; int iters; double margin; };

/* Alg. 3 l.14, unsquared reading R12, checked at iteration start so a
 * seed on the answer stops with 0 updates: FK, residual, coarse test. */
bool po_ccd_check(const Robot& rb, const OracleConfig& c, const Target& tgt,
                  const std::vector<double>& th, Frames& F, Err& e, SeedOut& so) {
    fk(rb, th.data(), F);
    e = residual(F, tgt);
    bool cp = e.ep < c.eps_p_coarse, co = e.eo < c.eps_o_coarse;
    so.margin = std::min(so.margin, margin_and(cp, std::fabs(e.ep - c.eps_p_coarse), co,
                                               std::fabs(e.eo - c.eps_o_coarse)));
    so.ep = e.ep;
    so.eo = e.eo;
    return cp && co;
}

/* Alg. 3 l.6-13: one greedy orientation-aware update of seed `sid`
 * at iteration k (frames F and residual e at th), or a perturbation. */
void po_ccd_step(const Robot& rb, const OracleConfig& c, const Target& tgt, uint64_t tid,
                 uint32_t sid, int k, const Frames& F, const Err& e, std::vector<double>& th,
                 SeedOut& so, const uint32_t* forced = nullptr, double* gap = nullptr,
                 uint32_t* record = nullptr, int* gap_kind = nullptr) {
    const OracleRobot* r = rb.r;
    int n = rb.dof;
    Frames Fc;
    std::vector<double> thc(n), thh(n);
    double phi; V3 ahat;
    angle_axis(tgt.q, F.qee, &phi, &ahat);
    double dk = delta_k(c, k);
    /* the w >= 0 canonicalisation of q_err flips a (R1/R2) when w crosses 0 */
    if (phi > 0) so.margin = std::min(so.margin, std::fabs(std::cos(phi / 2.0)));
    std::vector<double> sp(n), sop(n), dp(n), dor(n);
    /* replay only: the other sign of each candidate step, its score, and how
     * near its sign is to a tie: the pi branch cut of Eq. 9 (pi - |step|),
     * sgn(a . r_j) of Eq. 11 near 0 (|a . r_j|), or a vanishing step (|step|) */
    std::vector<double> dpa, spa, doa, sopa, tp(n, INF), to(n, INF);
    if (forced) { dpa.assign(n, 0.0); spa.assign(n, 0.0); doa.assign(n, 0.0); sopa.assign(n, 0.0); }
    for (int j = 0; j < n; ++j) {
        int ent = rb.dof_entry[j];
        double lo = r->lo[ent], hi = r->hi[ent];
        /* position candidate (Eqs. 8-9); prismatic: z.(P_t - P_ee) (R32) */
        double stepp;
        if (r->type[ent] == 0) {
            double mdeg;
            stepp = ccd_position_step(F.P[j], F.z[j], F.pee, tgt.p, c.tau_deg, &mdeg);
            so.margin = std::min(so.margin, mdeg);
        } else {
            stepp = dot(F.z[j], sub(tgt.p, F.pee));
        }
        /* joint limits on candidates (R7) */
        dp[j] = clampd(th[j] + stepp, lo, hi) - th[j];
        thc = th; thc[j] = th[j] + dp[j];
        fk(rb, thc.data(), Fc);                     /* literal P:222: full FK */
        sp[j] = norm(sub(tgt.p, Fc.pee));
        if (forced) {
            dpa[j] = dp[j]; spa[j] = sp[j];
            if (r->type[ent] == 0 && stepp != 0.0) {
                /* the sign of Eq. 9's step is the sign of y = z.(u_p x v_p) =
                 * |u_p||v_p| sin(step): both of its ties (a vanishing step, and
                 * the +-pi branch cut) are y = 0, and a float evaluation of y
                 * errs by ~eps |u||v| (u = P_ee - P_j, v = P_t - P_j), so the
                 * tie distance is |y| / (|u||v|) */
                V3 u = sub(F.pee, F.P[j]), v = sub(tgt.p, F.P[j]);
                double rr = dot(F.z[j], F.z[j]);
                V3 up = sub(u, scl(F.z[j], dot(u, F.z[j]) / rr)), vp = sub(v, scl(F.z[j], dot(v, F.z[j]) / rr));
                tp[j] = std::fabs(std::sin(stepp)) * norm(up) * norm(vp) / (norm(u) * norm(v));
                dpa[j] = clampd(th[j] - stepp, lo, hi) - th[j];
                thc = th; thc[j] = th[j] + dpa[j];
                fk(rb, thc.data(), Fc);
                spa[j] = norm(sub(tgt.p, Fc.pee));
            }
        }
        /* orientation candidate (Eqs. 10-11); prismatic: 0 */
        double stepo = 0.0;
        if (r->type[ent] == 0) {
            stepo = ccd_orientation_step(phi, ahat, F.z[j], dk);
            if (phi > 0) so.margin = std::min(so.margin, std::fabs(dot(ahat, F.z[j])));
        }
        dor[j] = clampd(th[j] + stepo, lo, hi) - th[j];
        thc = th; thc[j] = th[j] + dor[j];
        fk(rb, thc.data(), Fc);
        sop[j] = norm(quat_error(tgt.q, Fc.qee));
        if (forced) {
            doa[j] = dor[j]; sopa[j] = sop[j];
            if (r->type[ent] == 0 && phi > 0) {
                to[j] = std::min(std::fabs(dot(ahat, F.z[j])), std::fabs(stepo));
                doa[j] = clampd(th[j] - stepo, lo, hi) - th[j];
                thc = th; thc[j] = th[j] + doa[j];
                fk(rb, thc.data(), Fc);
                sopa[j] = norm(quat_error(tgt.q, Fc.qee));
            }
        }
    }
    /* Alg. 3 l.9: argmin over joints, ties -> lower index (R6) */
    int jp = 0, jo = 0;
    for (int j = 1; j < n; ++j) {
        if (sp[j] < sp[jp]) jp = j;
        if (sop[j] < sop[jo]) jo = j;
    }
    for (int j = 0; j < n; ++j) {
        /* distance to the nearest competitor with a different outcome */
        if (j != jp && (dp[j] != 0.0 || dp[jp] != 0.0))
            so.margin = std::min(so.margin, std::fabs(sp[j] - sp[jp]));
        if (j != jo && (dor[j] != 0.0 || dor[jo] != 0.0))
            so.margin = std::min(so.margin, std::fabs(sop[j] - sop[jo]));
    }
    /* replay (oracle_po_ccd_replay): take the recorded argmins instead; the gap
     * is how much worse they score than this fp64 argmin */
    if (forced) {
        auto upd = [&](double g, int kind) { if (g > *gap) { *gap = g; *gap_kind = kind; } };
        auto code = [](double x) { return x > 0 ? 1u : (x < 0 ? 2u : 0u); };
        int fp = (int)(*forced & 31u), fo = (int)((*forced >> 5) & 31u);
        if (fp >= n || fo >= n) { *gap = INF; return; }
        /* the recorded step signs: a near-tie sign takes the other variant
         * (gap = the tie's distance); a sign no variant has costs |step| */
        unsigned cp = (*forced >> 12) & 3u, co = (*forced >> 14) & 3u;
        if (code(dp[fp]) != cp) {
            if (code(dpa[fp]) == cp) { upd(tp[fp], 6); dp[fp] = dpa[fp]; sp[fp] = spa[fp]; }
            else upd(std::fabs(dp[fp]), 6);
        }
        if (code(dor[fo]) != co) {
            if (code(doa[fo]) == co) { upd(to[fo], 7); dor[fo] = doa[fo]; sop[fo] = sopa[fo]; }
            else upd(std::fabs(dor[fo]), 7);
        }
        /* the best score any valid reading allows: a near-tie joint counts
         * with its worse variant */
        const double TIE = 1e-4;
        double bp = INF, bo = INF;
        for (int j = 0; j < n; ++j) {
            bp = std::min(bp, j != fp && tp[j] < TIE ? std::max(sp[j], spa[j]) : sp[j]);
            bo = std::min(bo, j != fo && to[j] < TIE ? std::max(sop[j], sopa[j]) : sop[j]);
        }
        upd(sp[fp] - bp, 1);
        upd(sop[fo] - bo, 2);
        jp = fp;
        jo = fo;
    }
    /* Alg. 3 l.10 + P:201: same joint -> larger |dtheta|, tie -> position (R8) */
    thh = th;
    bool ori_taken = false;
    if (jp == jo) {
        if (dp[jp] != dor[jo]) /* equal steps = same outcome, no decision */
            so.margin = std::min(so.margin, std::fabs(std::fabs(dp[jp]) - std::fabs(dor[jo])));
        bool take_p = std::fabs(dp[jp]) >= std::fabs(dor[jo]);
        if (forced && dp[jp] != dor[jo] && take_p == (((*forced >> 10) & 1u) != 0)) {
            if (std::fabs(std::fabs(dp[jp]) - std::fabs(dor[jo])) > *gap) {
                *gap = std::fabs(std::fabs(dp[jp]) - std::fabs(dor[jo]));
                *gap_kind = 3;
            }
            take_p = !take_p;
        }
        ori_taken = !take_p;
        if (take_p) thh[jp] = th[jp] + dp[jp];
        else thh[jo] = th[jo] + dor[jo];
    } else {
        thh[jp] = th[jp] + dp[jp];
        thh[jo] = th[jo] + dor[jo];
    }
    /* clamp after every applied update (R7): removes rounding overshoot */
    for (int j = 0; j < n; ++j) {
        int ent = rb.dof_entry[j];
        thh[j] = clampd(thh[j], r->lo[ent], r->hi[ent]);
    }
    fk(rb, thh.data(), Fc);
    Err eh = residual(Fc, tgt);
    /* Alg. 3 l.11 read as an improvement test on either space (R10) */
    double ip = e.ep - eh.ep, io = e.eo - eh.eo;
    bool ap = ip > c.gamma, ao = io > c.gamma;
    double macc = margin_or(ap, std::fabs(ip - c.gamma), ao, std::fabs(io - c.gamma));
    so.margin = std::min(so.margin, macc);
    bool accept = ap || ao;
    if (forced && accept != (((*forced >> 11) & 1u) != 0)) {
        if (macc > *gap) { *gap = macc; *gap_kind = 4; }
        accept = !accept;
    }
    if (record)   /* this oracle's own decisions, in hjcd_poccd_trace's word format */
        *record = (uint32_t)jp | ((uint32_t)jo << 5) | (ori_taken ? 1u << 10 : 0u) |
                  (accept ? 1u << 11 : 0u) | ((dp[jp] > 0 ? 1u : dp[jp] < 0 ? 2u : 0u) << 12) |
                  ((dor[jo] > 0 ? 1u : dor[jo] < 0 ? 2u : 0u) << 14);
    if (accept) {
        th = thh;
    } else {
        /* Alg. 3 l.13: theta + N(0, sigma_ccd^2 I), clamp (R11) */
        for (int j = 0; j < n; ++j) {
            int ent = rb.dof_entry[j];
            double g = normal_for_joint(c.rng_seed, tid, sid, P_PERTURB, (uint32_t)k, j);
            th[j] = clampd(th[j] + c.sigma_ccd * g, r->lo[ent], r->hi[ent]);
        }
    }
}

SeedOut seed_init() {
    SeedOut so;
    so.ep = so.eo = INF;
    so.iters = 0;
    so.margin = INF;
    return so;
}

/* Alg. 3 for ONE seed with a per-seed break (ccd_early_exit = 0) */
SeedOut po_ccd_seed(const Robot& rb, const OracleConfig& c, const Target& tgt, uint64_t tid,
                    uint32_t sid, std::vector<double>& th, uint32_t* record = nullptr) {
    SeedOut so = seed_init();
    Frames F;
    Err e;
    int k;
    for (k = 0;; ++k) {
        if (po_ccd_check(rb, c, tgt, th, F, e, so)) break;
        if (k == c.ccd_iters) break;
        po_ccd_step(rb, c, tgt, tid, sid, k, F, e, th, so, nullptr, nullptr, record ? record + k : nullptr);
    }
    so.iters = k;
    return so;
}

/* Alg. 3 for the M seeds of ONE target with the paper's stop rule ("once
 * a seed satisfies the position and orientation error thresholds ... the
 * parallel loop is broken and all samples are returned"; ccd_early_exit = 1,
 * DESIGN.md R12b).  The M seeds advance in lockstep (iteration loop outside,
 * seeds inside); the target stops at the first iteration at which any seed
 * passes the coarse test, every seed keeping its state after that many
 * iterations.  th_m: [M][n] in/out. */
void po_ccd_target(const Robot& rb, const OracleConfig& c, const Target& tgt, uint64_t tid, int M,
                   std::vector<std::vector<double>>& th_m, std::vector<SeedOut>& so,
                   uint32_t* record = nullptr) {
    so.assign(M, seed_init());
    std::vector<Frames> F(M);
    std::vector<Err> e(M);
    for (int k = 0;; ++k) {
        bool any = false;
        for (int m = 0; m < M; ++m) {
            bool cv = po_ccd_check(rb, c, tgt, th_m[m], F[m], e[m], so[m]);
            any = any || cv;
        }
        for (int m = 0; m < M; ++m) so[m].iters = k;
        if (any || k == c.ccd_iters) break;
        for (int m = 0; m < M; ++m)
            po_ccd_step(rb, c, tgt, tid, (uint32_t)m, k, F[m], e[m], th_m[m], so[m], nullptr, nullptr,
                        record ? record + (size_t)m * c.ccd_iters + k : nullptr);
    }
}

/* ---------------- classic CCD, one seed (Alg. 1) ----------------
 * Literal: joints j = n..1 (tip to root); for each, a FULL FK at the current
 * theta, Eqs. 8-9 (R3 sign, R4 degeneracy), clamp to the limits (R7), update;
 * after the sweep an FK and the test |P_ee - P_t| < eps (R12's unsquared
 * reading of Alg. 1 l.7, eps = eps_p_coarse), checked before each sweep. */
SeedOut ccd_seed(const Robot& rb, const OracleConfig& c, const Target& tgt, std::vector<double>& th) {
    const OracleRobot* r = rb.r;
    int n = rb.dof;
    SeedOut so = {INF, INF, 0, INF};
    Frames F;
    int k;
    for (k = 0;; ++k) {
        fk(rb, th.data(), F);
        so.ep = norm(sub(tgt.p, F.pee));
        if (so.ep < c.eps_p_coarse) break;
        if (k == c.ccd_iters) break;
        for (int j = n - 1; j >= 0; --j) {
            fk(rb, th.data(), F);                 /* literal: FK at the current theta */
            int ent = rb.dof_entry[j];
            double step;
            if (r->type[ent] == 0) step = ccd_position_step(F.P[j], F.z[j], F.pee, tgt.p, c.tau_deg, nullptr);
            else step = dot(F.z[j], sub(tgt.p, F.pee));
            th[j] = clampd(th[j] + step, r->lo[ent], r->hi[ent]);
        }
    }
    so.iters = k;
    return so;
}

/* uniform seed in limits (Alg. 3 l.2-3), fp32 fmaf on purpose (R30) */
void uniform_seed(const Robot& rb, uint64_t seed, uint64_t tid, uint32_t sid, double* th) {
    for (int j = 0; j < rb.dof; ++j) {
        int ent = rb.dof_entry[j];
        double u[4];
        draw4(seed, tid, sid, P_INIT, 0, (uint32_t)(j / 4), u);
        float lo = (float)rb.r->lo[ent], hi = (float)rb.r->hi[ent];
        float uf = (float)u[j % 4];
        th[j] = (double)std::fmaf(hi - lo, uf, lo);
    }
}

/* splitmix64 stream (replay variants only; the method's own draws are Philox) */
uint64_t splitmix64(uint64_t& x) {
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* u * 2^-23, u uniform in [-1, 1]: one fp32 rounding's relative size */
double ulp32_noise(uint64_t& st) {
    return ((double)(splitmix64(st) >> 11) * (2.0 / 9007199254740992.0) - 1.0) * std::ldexp(1.0, -23);
}

/* replay variants only (rng != NULL): every entry of a symmetric n x n matrix
 * scaled by (1 + one fp32 rounding), the size of the error a float
 * accumulation of its sums carries (the normal matrices of Eq. 12 and Eq. 14
 * can be ill-conditioned enough for that to matter) */
void perturb_sym(std::vector<double>& H, int n, uint64_t* rng) {
    if (!rng) return;
    for (int a = 0; a < n; ++a)
        for (int b = a; b < n; ++b) {
            double v = H[a * n + b] * (1.0 + ulp32_noise(*rng));
            H[a * n + b] = H[b * n + a] = v;
        }
}

/* ---------------- dense SPD solve (Cholesky), n x n ---------------- */
bool cholesky_solve(std::vector<double> A, int n, const double* b, double* x) {
    /* A = L L^T in place (lower) */
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j <= i; ++j) {
            double s = A[i * n + j];
            for (int k = 0; k < j; ++k) s -= A[i * n + k] * A[j * n + k];
            if (i == j) {
                if (!(s > 0)) return false;
                A[i * n + i] = std::sqrt(s);
            } else {
                A[i * n + j] = s / A[j * n + j];
            }
        }
    }
    std::vector<double> y(n);
    for (int i = 0; i < n; ++i) {
        double s = b[i];
        for (int k = 0; k < i; ++k) s -= A[i * n + k] * y[k];
        y[i] = s / A[i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = y[i];
        for (int k = i + 1; k < n; ++k) s -= A[k * n + i] * x[k];
        x[i] = s / A[i * n + i];
    }
    return true;
}

/* replay resynchronisation: the end-effector distance (m) and rotation angle
 * (rad) between FK(a) and FK(b): one step's fp32-vs-fp64 difference measured
 * where it matters (a joint whose axis passes near the end effector can differ
 * in angle without moving it) */
double task_distance(const Robot& rb, const double* a, const double* b) {
    Frames Fa, Fb;
    fk(rb, a, Fa);
    fk(rb, b, Fb);
    return std::max(norm(sub(Fa.pee, Fb.pee)), norm(quat_error(Fa.qee, Fb.qee)));
}

/* replay resynchronisation: the states "one fp32 ulp away" from theta_k at
 * which a recorded decision is also judged (a float evaluation cannot tell
 * them apart): every joint moved by u * 2^-23 * max(|theta_j|, 1 rad or m),
 * u uniform in [-1, 1] from a splitmix64 stream keyed by (seed row, k,
 * variant), then clamped into the limits */
const int REPLAY_VARIANTS = 4;
const double REPLAY_SPREAD_FACTOR = 10.0;

void perturb_ulp(const Robot& rb, std::vector<double>& th, uint64_t key) {
    uint64_t st = key;
    for (int j = 0; j < rb.dof; ++j) {
        int ent = rb.dof_entry[j];
        th[j] = clampd(th[j] + ulp32_noise(st) * std::max(std::fabs(th[j]), 1.0), rb.r->lo[ent], rb.r->hi[ent]);
    }
}

/* ---------------- PJ-IK pieces (Alg. 4) ---------------- */
/* rho = -r = [P_ee - P_t; -omega] (R19), 6-vector */
void rho_of(const Err& e, double rho[6]) {
    rho[0] = -e.rp.x; rho[1] = -e.rp.y; rho[2] = -e.rp.z;
    rho[3] = -e.om.x; rho[4] = -e.om.y; rho[5] = -e.om.z;
}

/* W (R17): diag(w_p I3, w_o I3) * diag(1 / (1 + |J_row_i|)) */
void weights(const OracleConfig& c, const double* J, int n, double W[6]) {
    for (int i = 0; i < 6; ++i) {
        double s = 0;
        for (int j = 0; j < n; ++j) s += J[i * n + j] * J[i * n + j];
        W[i] = (i < 3 ? c.w_p : c.w_o) / (1.0 + std::sqrt(s));
    }
}

double cost_w(const double W[6], const double rho[6]) {
    double s = 0;
    for (int i = 0; i < 6; ++i) s += (W[i] * rho[i]) * (W[i] * rho[i]);
    return 0.5 * s;
}

double norm6(const double v[6]) {
    double s = 0;
    for (int i = 0; i < 6; ++i) s += v[i] * v[i];
    return std::sqrt(s);
}

/* Eq. 12 with the missing W restored (R18), D = max(diag(J^T J),
 * d_floor) (R20): (J^T W^2 J + lambda D) dtheta = -J^T W^2 rho, literal n x n. */
bool lm_step(const OracleConfig& c, const double* J, int n, const double W[6],
             const double rho[6], double* dth, uint64_t* rng = nullptr) {
    std::vector<double> H(n * n, 0.0), g(n, 0.0);
    for (int a = 0; a < n; ++a) {
        for (int b = 0; b < n; ++b) {
            double s = 0;
            for (int i = 0; i < 6; ++i) s += J[i * n + a] * W[i] * W[i] * J[i * n + b];
            H[a * n + b] = s;
        }
        double d = 0;
        for (int i = 0; i < 6; ++i) d += J[i * n + a] * J[i * n + a];
        H[a * n + a] += c.lambda * std::max(d, c.d_floor);
        double s = 0;
        for (int i = 0; i < 6; ++i) s += J[i * n + a] * W[i] * W[i] * rho[i];
        g[a] = -s;
    }
    perturb_sym(H, n, rng);
    return cholesky_solve(H, n, g.data(), dth);
}

/* Eqs. 14-15, readings R23: GD = -alpha_c J^T rho (Cauchy alpha),
 * GN = -(J^T J + d_floor I)^-1 J^T rho, dtheta(tau) = tau GD + (1-tau) GN with
 * the smallest tau in [0,1] such that |dtheta(tau)| <= R; none -> GD scaled to
 * |.| = R.  Returns false on a zero gradient. */
bool dogleg_step(const OracleConfig& c, const double* J, int n, const double rho[6], double* dth,
                 uint64_t* rng = nullptr) {
    std::vector<double> g0(n, 0.0);
    double gg = 0;
    for (int a = 0; a < n; ++a) {
        double s = 0;
        for (int i = 0; i < 6; ++i) s += J[i * n + a] * rho[i];
        g0[a] = s;
        gg += s * s;
    }
    if (gg <= 1e-30) return false;
    double jg2 = 0;
    for (int i = 0; i < 6; ++i) {
        double s = 0;
        for (int a = 0; a < n; ++a) s += J[i * n + a] * g0[a];
        jg2 += s * s;
    }
    if (!(jg2 > 0)) return false;
    double alpha = gg / jg2;
    std::vector<double> gd(n), gn(n);
    for (int a = 0; a < n; ++a) gd[a] = -alpha * g0[a];
    std::vector<double> H(n * n, 0.0), rhs(n);
    for (int a = 0; a < n; ++a) {
        for (int b = 0; b < n; ++b) {
            double s = 0;
            for (int i = 0; i < 6; ++i) s += J[i * n + a] * J[i * n + b];
            H[a * n + b] = s;
        }
        H[a * n + a] += c.d_floor;
        rhs[a] = -g0[a];
    }
    perturb_sym(H, n, rng);
    if (!cholesky_solve(H, n, rhs.data(), gn.data())) return false;
    double ngn2 = 0;
    for (int a = 0; a < n; ++a) ngn2 += gn[a] * gn[a];
    double R2 = c.R * c.R;
    if (ngn2 <= R2) { for (int a = 0; a < n; ++a) dth[a] = gn[a]; return true; }
    /* |gn + tau (gd - gn)|^2 = R^2  ->  qa tau^2 + qb tau + qc = 0 */
    double qa = 0, qb = 0, qc = ngn2 - R2;
    for (int a = 0; a < n; ++a) {
        double d = gd[a] - gn[a];
        qa += d * d;
        qb += 2.0 * gn[a] * d;
    }
    double disc = qb * qb - 4.0 * qa * qc;
    if (qa > 0 && disc >= 0) {
        double tau = (-qb - std::sqrt(disc)) / (2.0 * qa);
        if (tau >= 0.0 && tau <= 1.0) {
            for (int a = 0; a < n; ++a) dth[a] = tau * gd[a] + (1.0 - tau) * gn[a];
            return true;
        }
    }
    double ngd = 0;
    for (int a = 0; a < n; ++a) ngd += gd[a] * gd[a];
    ngd = std::sqrt(ngd);
    for (int a = 0; a < n; ++a) dth[a] = gd[a] * (c.R / ngd);
    return true;
}

/* Eq. 16, reading R24: i* = argmax |g_i|, g = J^T W^2 rho; step
 * -sign(g_i*) min(|g_i*|, R) e_i*.  Returns i* or -1 on a zero gradient. */
int single_coord_step(const OracleConfig& c, const double* J, int n, const double W[6],
                      const double rho[6], double* dth, double* gap) {
    std::vector<double> g(n);
    for (int a = 0; a < n; ++a) {
        double s = 0;
        for (int i = 0; i < 6; ++i) s += J[i * n + a] * W[i] * W[i] * rho[i];
        g[a] = s;
    }
    int ist = 0;
    for (int a = 1; a < n; ++a)
        if (std::fabs(g[a]) > std::fabs(g[ist])) ist = a;
    if (gap) {
        double second = 0;
        for (int a = 0; a < n; ++a)
            if (a != ist) second = std::max(second, std::fabs(g[a]));
        *gap = (std::fabs(g[ist]) - second) / (std::fabs(g[ist]) + 1e-300);
    }
    for (int a = 0; a < n; ++a) dth[a] = 0;
    if (g[ist] == 0.0) return -1;
    double m = std::min(std::fabs(g[ist]), c.R);
    dth[ist] = (g[ist] > 0) ? -m : m;
    return ist;
}

double rel_gap(double a, double b, double floor_) {
    return std::fabs(a - b) / (std::fabs(a) + std::fabs(b) + floor_);
}

struct PolishOut { double ep, eo; int counts[4]; double margin; int iters; };

/* evaluate rho at clamp(theta + alpha * dth) */
void trial_point(const Robot& rb, const std::vector<double>& th, const double* dth, double alpha,
                 std::vector<double>& tt) {
    for (int j = 0; j < rb.dof; ++j) {
        int ent = rb.dof_entry[j];
        tt[j] = clampd(th[j] + alpha * dth[j], rb.r->lo[ent], rb.r->hi[ent]);
    }
}

/* Eq. 13, reading R22: first alpha in {1, 1/beta, ..., 1/beta^A}
 * with c_W(clamp(theta + alpha dth)) < c_W(theta), W frozen; returns index or -1 */
int line_search(const Robot& rb, const OracleConfig& c, const Target& tgt,
                const std::vector<double>& th, const double* dth, const double W[6], double c0,
                std::vector<double>& tt, double* margin) {
    Frames Ft;
    double alpha = 1.0;
    for (int a = 0; a <= c.A; ++a) {
        trial_point(rb, th, dth, alpha, tt);
        fk(rb, tt.data(), Ft);
        Err et = residual(Ft, tgt);
        double rho[6];
        rho_of(et, rho);
        double ct = cost_w(W, rho);
        if (margin) *margin = std::min(*margin, rel_gap(ct, c0, 1e-30));
        if (ct < c0) return a;
        alpha /= c.beta;
    }
    return -1;
}

/* Alg. 4 l.18 fine test at iteration start (R26); stores the residual */
bool pj_ik_check(const Robot& rb, const OracleConfig& c, const Target& tgt,
                 const std::vector<double>& th, Frames& F, Err& e, PolishOut& po) {
    fk(rb, th.data(), F);
    e = residual(F, tgt);
    bool cp = e.ep < c.eps_p_fine, co = e.eo < c.eps_o_fine;
    po.margin = std::min(po.margin, margin_and(cp, rel_gap(e.ep, c.eps_p_fine, 0), co,
                                               rel_gap(e.eo, c.eps_o_fine, 0)));
    /* omega's direction flips where the canonical q_err has w = 0 (|omega| = pi) */
    po.margin = std::min(po.margin, std::fabs(std::cos(e.eo / 2.0)));
    po.ep = e.ep;
    po.eo = e.eo;
    return cp && co;
}

/* PJ-IK decision word (the format of hjcd_pjik_trace, include/hjcd.h): the
 * branch that moved the seed (0 LM step, 1 dogleg, 2 single coordinate,
 * 3 perturbation) | alpha index a (step beta^-a) << 2 | single-coordinate
 * index i* << 8 | 1 << 15 (a step was taken; 0 = no step at this iteration) */
uint32_t pj_word(int kind, int a, int ist) {
    return (uint32_t)kind | ((uint32_t)a << 2) | ((uint32_t)ist << 8) | (1u << 15);
}

/* one iteration of Alg. 4 (l.3-17) for one seed, frames F and residual e at th */
void pj_ik_step(const Robot& rb, const OracleConfig& c, const Target& tgt, uint64_t tid,
                uint32_t bidx, int k, const Frames& F, const Err& e, std::vector<double>& th,
                PolishOut& po, uint32_t* record = nullptr) {
    const OracleRobot* r = rb.r;
    int n = rb.dof;
    Frames Ft;
    std::vector<double> J(6 * n), dth(n), tt(n);
    jacobian(rb, F, J.data());
    double W[6], rho[6];
    weights(c, J.data(), n, W);
    rho_of(e, rho);
    double c0 = cost_w(W, rho);
    /* LM step (Alg. 4 l.3-9) */
    bool ok = lm_step(c, J.data(), n, W, rho, dth.data());
    if (ok) {
        for (int j = 0; j < n; ++j) dth[j] = clampd(dth[j], -c.R, c.R); /* l.6, R21 */
        int a = line_search(rb, c, tgt, th, dth.data(), W, c0, tt, &po.margin);
        if (a >= 0) {
            th = tt; po.counts[0]++;
            if (record) *record = pj_word(0, a, 0);
            return;
        }
    }
    /* dogleg (l.10-12), acceptance on the unweighted |rho| (R23) */
    if (dogleg_step(c, J.data(), n, rho, dth.data())) {
        trial_point(rb, th, dth.data(), 1.0, tt);
        fk(rb, tt.data(), Ft);
        Err et = residual(Ft, tgt);
        double rt[6];
        rho_of(et, rt);
        double n0 = norm6(rho), nt = norm6(rt);
        po.margin = std::min(po.margin, rel_gap(nt, n0, 1e-30));
        if (nt < n0) {
            th = tt; po.counts[1]++;
            if (record) *record = pj_word(1, 0, 0);
            return;
        }
    }
    /* single coordinate (l.13-16) */
    double gap;
    int ist = single_coord_step(c, J.data(), n, W, rho, dth.data(), &gap);
    if (ist >= 0) {
        po.margin = std::min(po.margin, gap);
        int a = line_search(rb, c, tgt, th, dth.data(), W, c0, tt, &po.margin);
        if (a >= 0) {
            th = tt; po.counts[2]++;
            if (record) *record = pj_word(2, a, ist);
            return;
        }
    }
    /* perturbation (l.17, R25) */
    for (int j = 0; j < n; ++j) {
        int ent = rb.dof_entry[j];
        double g = normal_for_joint(c.rng_seed, tid, bidx, P_PJPERT, (uint32_t)k, j);
        th[j] = clampd(th[j] + c.sigma_lm * g, r->lo[ent], r->hi[ent]);
    }
    po.counts[3]++;
    if (record) *record = pj_word(3, 0, 0);
}

/* Decision replay of one Alg. 4 iteration (oracle_pj_ik_replay): the same
 * cascade as pj_ik_step, in fp64, but the branch, alpha index and
 * single-coordinate index are the RECORDED ones (word, pj_word format).  Every
 * cascade item before the recorded one must fail and the recorded one must
 * succeed; *gap grows by how far the fp64 comparison is from the recorded
 * outcome, in the units it compares: | |W rho_t| - |W rho_0| | for the
 * weighted-cost tests (Eq. 13, R22), | |rho_t| - |rho_0| | for the dogleg test
 * (R23), |g_i*| - |g_rec| for the single-coordinate argmax (Eq. 16, R24).
 * gap_kind: 1 LM trial, 2 dogleg trial, 3 single-coordinate index, 4
 * single-coordinate trial, 6 an invalid word. */
void pj_ik_step_replay(const Robot& rb, const OracleConfig& c, const Target& tgt, uint64_t tid,
                       uint32_t bidx, int k, const Frames& F, const Err& e, std::vector<double>& th,
                       PolishOut& po, uint32_t word, double* gap, int* gap_kind, uint64_t* rng = nullptr) {
    const OracleRobot* r = rb.r;
    int n = rb.dof;
    auto upd = [&](double g, int kind) { if (g > *gap) { *gap = g; *gap_kind = kind; } };
    int kind = (int)(word & 3u), af = (int)((word >> 2) & 31u), istf = (int)((word >> 8) & 31u);
    if (!(word & (1u << 15)) || (word >> 16) != 0 || af > c.A || istf >= n ||
        (kind == 1 && af != 0)) {
        upd(INF, 6);
        return;
    }
    Frames Ft;
    std::vector<double> J(6 * n), dth(n), tt(n);
    jacobian(rb, F, J.data());
    double W[6], rho[6];
    weights(c, J.data(), n, W);
    rho_of(e, rho);
    double c0 = cost_w(W, rho);
    /* the weighted cost at clamp(th + alpha dth) (Eq. 13, W frozen at th) */
    auto trial_cost = [&](const std::vector<double>& d, double alpha) {
        trial_point(rb, th, d.data(), alpha, tt);
        fk(rb, tt.data(), Ft);
        Err et = residual(Ft, tgt);
        double rt[6];
        rho_of(et, rt);
        return cost_w(W, rt);
    };
    auto depth = [&](double ct) { return std::fabs(std::sqrt(2.0 * ct) - std::sqrt(2.0 * c0)); };
    /* LM line search (l.3-9): items alpha_0 .. alpha_A */
    bool lm_ok = lm_step(c, J.data(), n, W, rho, dth.data(), rng);
    if (lm_ok)
        for (int j = 0; j < n; ++j) dth[j] = clampd(dth[j], -c.R, c.R);
    double alpha = 1.0;
    for (int a = 0; a <= c.A; ++a, alpha /= c.beta) {
        bool forced_here = kind == 0 && a == af;
        if (!lm_ok) {
            if (forced_here) { upd(INF, 1); return; }
            continue;
        }
        double ct = trial_cost(dth, alpha);
        if (forced_here) {
            if (!(ct < c0)) upd(depth(ct), 1);
            th = tt; po.counts[0]++;
            return;
        }
        if (ct < c0) upd(depth(ct), 1);   /* fp64 accepts an earlier item */
    }
    /* dogleg (l.10-12) */
    std::vector<double> dd(n);
    if (dogleg_step(c, J.data(), n, rho, dd.data(), rng)) {
        trial_point(rb, th, dd.data(), 1.0, tt);
        fk(rb, tt.data(), Ft);
        Err et = residual(Ft, tgt);
        double rt[6];
        rho_of(et, rt);
        double n0 = norm6(rho), nt = norm6(rt);
        if (kind == 1) {
            if (!(nt < n0)) upd(std::fabs(nt - n0), 2);
            th = tt; po.counts[1]++;
            return;
        }
        if (nt < n0) upd(std::fabs(nt - n0), 2);
    } else if (kind == 1) {
        upd(INF, 2);
        return;
    }
    /* single coordinate (l.13-16) at the recorded index */
    std::vector<double> g(n);
    for (int a = 0; a < n; ++a) {
        double s = 0;
        for (int i = 0; i < 6; ++i) s += J[i * n + a] * W[i] * W[i] * rho[i];
        g[a] = s;
    }
    int ist = 0;
    for (int a = 1; a < n; ++a)
        if (std::fabs(g[a]) > std::fabs(g[ist])) ist = a;
    bool sc_ok = g[ist] != 0.0;
    if (kind == 2) {
        upd(std::fabs(g[ist]) - std::fabs(g[istf]), 3);
        ist = istf;
        sc_ok = g[ist] != 0.0;
    }
    std::vector<double> ds(n, 0.0);
    if (sc_ok) {
        double m = std::min(std::fabs(g[ist]), c.R);
        ds[ist] = (g[ist] > 0) ? -m : m;
    }
    alpha = 1.0;
    for (int a = 0; a <= c.A; ++a, alpha /= c.beta) {
        bool forced_here = kind == 2 && a == af;
        if (!sc_ok) {
            if (forced_here) { upd(INF, 4); return; }
            continue;
        }
        double ct = trial_cost(ds, alpha);
        if (forced_here) {
            if (!(ct < c0)) upd(depth(ct), 4);
            th = tt; po.counts[2]++;
            return;
        }
        if (ct < c0) upd(depth(ct), 4);
    }
    /* perturbation (l.17, R25): every item above failed */
    for (int j = 0; j < n; ++j) {
        int ent = rb.dof_entry[j];
        double gn = normal_for_joint(c.rng_seed, tid, bidx, P_PJPERT, (uint32_t)k, j);
        th[j] = clampd(th[j] + c.sigma_lm * gn, r->lo[ent], r->hi[ent]);
    }
    po.counts[3]++;
}

PolishOut polish_init() {
    PolishOut po;
    po.margin = INF;
    po.ep = po.eo = INF;
    po.iters = 0;
    for (int i = 0; i < 4; ++i) po.counts[i] = 0;
    return po;
}

/* Alg. 4 for ONE seed with a per-seed break (target_early_exit = 0) */
PolishOut pj_ik_seed(const Robot& rb, const OracleConfig& c, const Target& tgt, uint64_t tid,
                     uint32_t bidx, std::vector<double>& th, uint32_t* record = nullptr) {
    PolishOut po = polish_init();
    Frames F;
    Err e;
    int k;
    for (k = 0;; ++k) {
        if (pj_ik_check(rb, c, tgt, th, F, e, po)) break;
        if (k == c.lm_iters) break;
        pj_ik_step(rb, c, tgt, tid, bidx, k, F, e, th, po, record ? record + k : nullptr);
    }
    po.iters = k;
    return po;
}

/* Alg. 4 for the `used` seeds of ONE target in the paper's loop order: the
 * iteration loop outside, the seeds inside.  target_early_exit = 1:
 * the target stops at the first iteration at which any seed passes the fine
 * test (Alg. 4 l.18 "break"), every seed keeping its state after
 * the same number of iterations (R26b).  th_bn: [used][n] in/out. */
void pj_ik_target(const Robot& rb, const OracleConfig& c, const Target& tgt, uint64_t tid, int used,
                  std::vector<std::vector<double>>& th_bn, std::vector<PolishOut>& po,
                  uint32_t* record = nullptr, int rec_stride_b = 0) {
    po.assign(used, polish_init());
    std::vector<Frames> F(used);
    std::vector<Err> e(used);
    for (int k = 0;; ++k) {
        bool any = false;
        for (int b = 0; b < used; ++b) {
            bool cv = pj_ik_check(rb, c, tgt, th_bn[b], F[b], e[b], po[b]);
            any = any || cv;
        }
        for (int b = 0; b < used; ++b) po[b].iters = k;
        if (any || k == c.lm_iters) break;
        for (int b = 0; b < used; ++b)
            pj_ik_step(rb, c, tgt, tid, (uint32_t)b, k, F[b], e[b], th_bn[b], po[b],
                       record ? record + (size_t)b * rec_stride_b + k : nullptr);
    }
}

/* c(theta) = w_p^2 |r_p|^2 + w_o^2 |omega|^2 (R14), used for ranking and best-select */
double rank_cost(const OracleConfig& c, double ep, double eo) {
    return c.w_p * c.w_p * ep * ep + c.w_o * c.w_o * eo * eo;
}

/* Alg. 2 l.2-8: K rounds of argmin-and-remove == the first K of a
 * stable sort by (cost, index); then floor(B/K) copies, copy-major order
 * b = copy * K + rank, copy 0 clean (R15), others + N(0, sigma_rep^2), clamp. */
void rank_and_replicate(const Robot& rb, const OracleConfig& c, uint64_t tid, const double* cost,
                        const double* theta_nm /* [n][M] */, double* seeds_bn /* [B][n] */,
                        int32_t* kept /* [K] */) {
    int M = c.M, K = c.K, n = rb.dof;
    std::vector<int> idx(M);
    for (int m = 0; m < M; ++m) idx[m] = m;
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return cost[a] < cost[b]; });
    for (int i = 0; i < K; ++i) kept[i] = idx[i];
    int copies = c.B / K;
    for (int b = 0; b < c.B; ++b) {
        if (b >= copies * K) { /* unused tail slots (B not a multiple of K) */
            for (int j = 0; j < n; ++j) seeds_bn[b * n + j] = std::numeric_limits<double>::quiet_NaN();
            continue;
        }
        int rank = b % K, cp = b / K;
        int src = idx[rank];
        for (int j = 0; j < n; ++j) {
            int ent = rb.dof_entry[j];
            double v = theta_nm[j * M + src];
            if (cp > 0 || c.repl_noise_all) {
                double g = normal_for_joint(c.rng_seed, tid, (uint32_t)b, P_REPL, 0, j);
                v = clampd(v + c.sigma_rep * g, rb.r->lo[ent], rb.r->hi[ent]);
            }
            seeds_bn[b * n + j] = v;
        }
    }
}

} /* namespace */

/* =========================== C entry points =========================== */
extern "C" {

int oracle_dof(const OracleRobot* r) { return make_robot(r).dof; }

void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    philox4x32_10(ctr, key, out);
}

/* batched FK (+ optional frames, Jacobian): theta [N][n] -> pose [N][7]
 * (px py pz qw qx qy qz, w >= 0), P/z [N][n][3], J [N][6][n] */
void oracle_fk(const OracleRobot* r, const double* theta, int32_t N, double* pose, double* Pf,
               double* zf, double* J) {
    Robot rb = make_robot(r);
    int n = rb.dof;
#pragma omp parallel for schedule(static)
    for (int s = 0; s < N; ++s) {
        Frames F;
        fk(rb, theta + (size_t)s * n, F);
        double* p = pose + (size_t)s * 7;
        p[0] = F.pee.x; p[1] = F.pee.y; p[2] = F.pee.z;
        p[3] = F.qee.w; p[4] = F.qee.x; p[5] = F.qee.y; p[6] = F.qee.z;
        for (int j = 0; j < n; ++j) {
            if (Pf) { double* q = Pf + ((size_t)s * n + j) * 3; q[0] = F.P[j].x; q[1] = F.P[j].y; q[2] = F.P[j].z; }
            if (zf) { double* q = zf + ((size_t)s * n + j) * 3; q[0] = F.z[j].x; q[1] = F.z[j].y; q[2] = F.z[j].z; }
        }
        if (J) jacobian(rb, F, J + (size_t)s * 6 * n);
    }
}

void oracle_quat_error(const double qt[4], const double qe[4], double omega[3]) {
    Qt a = {qt[0], qt[1], qt[2], qt[3]}, b = {qe[0], qe[1], qe[2], qe[3]};
    V3 w = quat_error(a, b);
    omega[0] = w.x; omega[1] = w.y; omega[2] = w.z;
}

void oracle_angle_axis(const double qt[4], const double qe[4], double* phi, double a[3]) {
    Qt x = {qt[0], qt[1], qt[2], qt[3]}, y = {qe[0], qe[1], qe[2], qe[3]};
    V3 ax;
    angle_axis(x, y, phi, &ax);
    a[0] = ax.x; a[1] = ax.y; a[2] = ax.z;
}

double oracle_ccd_position_step(const double Pj[3], const double rj[3], const double pee[3],
                                const double pt[3], double tau) {
    return ccd_position_step(v3(Pj[0], Pj[1], Pj[2]), v3(rj[0], rj[1], rj[2]),
                             v3(pee[0], pee[1], pee[2]), v3(pt[0], pt[1], pt[2]), tau, nullptr);
}

double oracle_ccd_orientation_step(const OracleConfig* c, const double qt[4], const double qe[4],
                                   const double rj[3], int32_t k) {
    Qt x = {qt[0], qt[1], qt[2], qt[3]}, y = {qe[0], qe[1], qe[2], qe[3]};
    double phi; V3 a;
    angle_axis(x, y, &phi, &a);
    return ccd_orientation_step(phi, a, v3(rj[0], rj[1], rj[2]), delta_k(*c, k));
}

/* LM / dogleg / single-coordinate / line-search units on explicit J, rho, W */
int32_t oracle_lm_step(const OracleConfig* c, const double* J, int32_t n, const double W[6],
                       const double rho[6], double* dth) {
    return lm_step(*c, J, n, W, rho, dth) ? 1 : 0;
}
int32_t oracle_dogleg_step(const OracleConfig* c, const double* J, int32_t n, const double rho[6],
                           double* dth) {
    return dogleg_step(*c, J, n, rho, dth) ? 1 : 0;
}
int32_t oracle_single_coord_step(const OracleConfig* c, const double* J, int32_t n,
                                 const double W[6], const double rho[6], double* dth) {
    return single_coord_step(*c, J, n, W, rho, dth, nullptr);
}
void oracle_weights(const OracleConfig* c, const double* J, int32_t n, double W[6]) {
    weights(*c, J, n, W);
}
/* line search at theta along dth toward target t7 with W frozen at theta */
int32_t oracle_line_search(const OracleRobot* r, const OracleConfig* c, const float* t7,
                           const double* theta, const double* dth) {
    Robot rb = make_robot(r);
    Target tgt = read_target(t7);
    std::vector<double> th(theta, theta + rb.dof), tt(rb.dof), J(6 * rb.dof);
    Frames F;
    fk(rb, th.data(), F);
    Err e = residual(F, tgt);
    jacobian(rb, F, J.data());
    double W[6], rho[6];
    weights(*c, J.data(), rb.dof, W);
    rho_of(e, rho);
    return line_search(rb, *c, tgt, th, dth, W, cost_w(W, rho), tt, nullptr);
}

void oracle_uniform_seeds(const OracleRobot* r, uint64_t seed, int64_t tid, int32_t M,
                          double* theta_nm /* [n][M] */) {
    Robot rb = make_robot(r);
    std::vector<double> th(rb.dof);
    for (int m = 0; m < M; ++m) {
        uniform_seed(rb, seed, (uint64_t)tid, (uint32_t)m, th.data());
        for (int j = 0; j < rb.dof; ++j) theta_nm[(size_t)j * M + m] = th[j];
    }
}

/* one standard normal of stream (tid, sid, purpose, iter) for joint d */
double oracle_normal(uint64_t seed, int64_t tid, uint32_t sid, uint32_t purpose, uint32_t iter,
                     int32_t d) {
    return normal_for_joint(seed, (uint64_t)tid, sid, purpose, iter, d);
}

/* PO-CCD stage (Alg. 3) for T targets x M seeds.
 * targets f32 [T][7]; seeds f64 [T][n][M] or NULL (Philox uniform);
 * out: theta f64 [T][n][M], cost f64 [T][M], ep/eo f64 [T][M], iters i32 [T][M],
 * margin f64 [T][M] (smallest absolute decision margin along the trajectory). */
void oracle_po_ccd(const OracleRobot* r, const OracleConfig* c, const float* targets, int32_t T,
                   int64_t tid_offset, const double* seeds, double* theta, double* cost,
                   double* ep, double* eo, int32_t* iters, double* margin, uint32_t* trace) {
    Robot rb = make_robot(r);
    int n = rb.dof, M = c->M;
    auto seed_of = [&](int t, int m, uint64_t tid, std::vector<double>& th) {
        if (seeds) for (int j = 0; j < n; ++j) th[j] = seeds[((size_t)t * n + j) * M + m];
        else uniform_seed(rb, c->rng_seed, tid, (uint32_t)m, th.data());
    };
    auto emit = [&](int t, int m, const std::vector<double>& th, const SeedOut& so) {
        for (int j = 0; j < n; ++j) theta[((size_t)t * n + j) * M + m] = th[j];
        size_t o = (size_t)t * M + m;
        if (cost) cost[o] = rank_cost(*c, so.ep, so.eo);
        if (ep) ep[o] = so.ep;
        if (eo) eo[o] = so.eo;
        if (iters) iters[o] = so.iters;
        if (margin) margin[o] = so.margin;
    };
    if (c->ccd_early_exit) {
#pragma omp parallel for schedule(dynamic, 1)
        for (int t = 0; t < T; ++t) {
            Target tgt = read_target(targets + (size_t)t * 7);
            uint64_t tid = (uint64_t)(tid_offset + t);
            std::vector<std::vector<double>> th(M, std::vector<double>(n));
            for (int m = 0; m < M; ++m) seed_of(t, m, tid, th[m]);
            std::vector<SeedOut> so;
            po_ccd_target(rb, *c, tgt, tid, M, th, so, trace ? trace + (size_t)t * M * c->ccd_iters : nullptr);
            for (int m = 0; m < M; ++m) emit(t, m, th[m], so[m]);
        }
        return;
    }
#pragma omp parallel for collapse(2) schedule(dynamic, 4)
    for (int t = 0; t < T; ++t) {
        for (int m = 0; m < M; ++m) {
            Target tgt = read_target(targets + (size_t)t * 7);
            uint64_t tid = (uint64_t)(tid_offset + t);
            std::vector<double> th(n);
            seed_of(t, m, tid, th);
            SeedOut so = po_ccd_seed(rb, *c, tgt, tid, (uint32_t)m, th,
                                     trace ? trace + ((size_t)t * M + m) * c->ccd_iters : nullptr);
            emit(t, m, th, so);
        }
    }
}

/* Decision replay of Alg. 3 (parity tests, DESIGN.md §4 "decision replay"):
 * every seed runs the GPU's iteration count iters [T][M] and, at each
 * iteration k, takes the GPU's recorded decisions trace [T][M][ccd_iters]
 * (hjcd_poccd_trace word: jp | jo << 5 | orientation-taken << 10 |
 * accepted << 11 | position / orientation step sign << 12 / 14) in place of
 * its own, with every candidate, score, step and
 * the perturbation computed here in fp64 exactly as in po_ccd_step.
 *   gap [T][M]: the largest amount by which a recorded decision is worse than
 *     this oracle's own (a score difference in m or rad, |dp| - |do| in rad,
 *     the distance of the gamma test from its threshold; 0 = all agree), and
 *     the depth inside the coarse box at an iteration the GPU continued;
 *   gap_at [T][M] (or NULL): 8 k + kind of that largest gap (kind 1 jp, 2 jo,
 *     3 same-joint choice, 4 gamma test, 5 continued inside the box, 6 / 7
 *     the sign of the position / orientation step), -1 none;
 *   stop_gap [T]: the distance outside the coarse box of the seed closest to
 *     it where the GPU stopped before ccd_iters (per target with
 *     ccd_early_exit, else the max over the seeds of their own); 0 if none.
 * theta f64 [T][n][M], ep/eo f64 [T][M] after the replay.
 * theta_hist f32 [T][M][ccd_iters + 1][n] or NULL: the GPU's theta at the
 *   start of every iteration (hjcd_poccd_trace).  Given, the replay is
 *   RESYNCHRONISED: iteration k starts from the GPU's theta_k instead of this
 *   oracle's own continuation, so every decision is judged at the exact state
 *   the GPU took it in and fp32 drift cannot accumulate.  A decision is also
 *   judged at REPLAY_VARIANTS states one fp32 ulp away from theta_k
 *   (perturb_ulp), and the smallest gap counts: fp32 cannot tell those states
 *   apart.  step_dev [T][M][3] (or NULL) receives, over k, (0) the largest
 *   task-space difference (task_distance: end-effector m / rotation rad)
 *   between this oracle's fp64 step from theta_k and the GPU's theta_{k+1}
 *   (one step's fp32-vs-fp64 difference under identical decisions), (1) the
 *   largest excess of that difference over REPLAY_SPREAD_FACTOR x the spread
 *   of the fp64 steps from the ulp-perturbed states (how well fp32 can
 *   determine the step at all: a step near a joint axis or a singular
 *   Jacobian is ill-conditioned), (2) the largest max_j |dtheta_j|. */
void oracle_po_ccd_replay(const OracleRobot* r, const OracleConfig* c, const float* targets, int32_t T,
                          int64_t tid_offset, const uint32_t* trace, const int32_t* iters,
                          double* theta, double* ep, double* eo, double* gap, double* stop_gap,
                          int32_t* gap_at, const float* theta_hist, double* step_dev) {
    Robot rb = make_robot(r);
    int n = rb.dof, M = c->M, I = c->ccd_iters;
#pragma omp parallel for schedule(dynamic, 1)
    for (int t = 0; t < T; ++t) {
        Target tgt = read_target(targets + (size_t)t * 7);
        uint64_t tid = (uint64_t)(tid_offset + t);
        double sg = c->ccd_early_exit ? INF : 0.0;
        bool stopped = false;
        for (int m = 0; m < M; ++m) {
            size_t o = (size_t)t * M + m;
            std::vector<double> th(n);
            uniform_seed(rb, c->rng_seed, tid, (uint32_t)m, th.data());
            SeedOut so = seed_init();
            Frames F;
            Err e;
            double g = 0.0, sd = 0.0, sdj = 0.0, sdx = -INF, spread = 0.0;
            int K = iters[o], kind = 0, at = -1;
            for (int k = 0;; ++k) {
                if (theta_hist && k <= I) {   /* resynchronise on the GPU's theta_k */
                    const float* h = theta_hist + (o * (size_t)(I + 1) + k) * n;
                    std::vector<double> hk(h, h + n);
                    if (k > 0) {
                        double dv = task_distance(rb, th.data(), hk.data());
                        sd = std::max(sd, dv);
                        sdx = std::max(sdx, dv - REPLAY_SPREAD_FACTOR * spread);
                        for (int j = 0; j < n; ++j) sdj = std::max(sdj, std::fabs(th[j] - hk[j]));
                    }
                    th = hk;
                }
                po_ccd_check(rb, *c, tgt, th, F, e, so);
                double inside = std::min(c->eps_p_coarse - e.ep, c->eps_o_coarse - e.eo);
                if (k == K) {
                    if (K < I) {
                        double outside = std::max(0.0, -inside);
                        stopped = true;
                        sg = c->ccd_early_exit ? std::min(sg, outside) : std::max(sg, outside);
                    }
                    break;
                }
                if (inside > g) { g = inside; at = 8 * k + 5; }
                const uint32_t* w = trace + o * I + k;
                std::vector<double> thk = th;
                double gk = 0.0;
                kind = 0;
                po_ccd_step(rb, *c, tgt, tid, (uint32_t)m, k, F, e, th, so, w, &gk, nullptr, &kind);
                spread = 0.0;
                if (theta_hist) {
                    /* the same decision one fp32 ulp away: the smallest gap over
                     * the variants counts, and the spread of their results
                     * measures how well fp32 can determine this step */
                    for (int v = 1; v <= REPLAY_VARIANTS; ++v) {
                        std::vector<double> tv = thk;
                        perturb_ulp(rb, tv, (o * 1024 + (uint64_t)k) * 8 + (uint64_t)v);
                        Frames Fv;
                        Err ev;
                        SeedOut sov = seed_init();
                        po_ccd_check(rb, *c, tgt, tv, Fv, ev, sov);
                        double gv = 0.0;
                        int kv = 0;
                        po_ccd_step(rb, *c, tgt, tid, (uint32_t)m, k, Fv, ev, tv, sov, w, &gv, nullptr, &kv);
                        if (gv < gk) { gk = gv; kind = kv; }
                        spread = std::max(spread, task_distance(rb, th.data(), tv.data()));
                    }
                }
                if (gk > g) { g = gk; at = 8 * k + kind; }
                if (!std::isfinite(g)) break;
            }
            for (int j = 0; j < n; ++j) theta[((size_t)t * n + j) * M + m] = th[j];
            ep[o] = so.ep;
            eo[o] = so.eo;
            gap[o] = g;
            if (gap_at) gap_at[o] = at;
            if (step_dev) { step_dev[3 * o] = sd; step_dev[3 * o + 1] = sdx; step_dev[3 * o + 2] = sdj; }
        }
        stop_gap[t] = stopped ? sg : 0.0;
    }
}

/* classic CCD (Alg. 1) for T targets x M seeds: seeds f64 [T][n][M] or NULL
 * (Philox uniform, as PO-CCD); out theta f64 [T][n][M], ep f64 [T][M], iters i32 [T][M] */
void oracle_ccd(const OracleRobot* r, const OracleConfig* c, const float* targets, int32_t T,
                int64_t tid_offset, const double* seeds, double* theta, double* ep, int32_t* iters) {
    Robot rb = make_robot(r);
    int n = rb.dof, M = c->M;
#pragma omp parallel for collapse(2) schedule(dynamic, 4)
    for (int t = 0; t < T; ++t) {
        for (int m = 0; m < M; ++m) {
            Target tgt = read_target(targets + (size_t)t * 7);
            uint64_t tid = (uint64_t)(tid_offset + t);
            std::vector<double> th(n);
            if (seeds) for (int j = 0; j < n; ++j) th[j] = seeds[((size_t)t * n + j) * M + m];
            else uniform_seed(rb, c->rng_seed, tid, (uint32_t)m, th.data());
            SeedOut so = ccd_seed(rb, *c, tgt, th);
            for (int j = 0; j < n; ++j) theta[((size_t)t * n + j) * M + m] = th[j];
            size_t o = (size_t)t * M + m;
            if (ep) ep[o] = so.ep;
            if (iters) iters[o] = so.iters;
        }
    }
}

/* top-K + replicate (Alg. 2 l.2-8): cost f64 [T][M], theta f64 [T][n][M] ->
 * polish seeds f64 [T][B][n], kept i32 [T][K] */
void oracle_select_replicate(const OracleRobot* r, const OracleConfig* c, const double* cost,
                             const double* theta, int32_t T, int64_t tid_offset, double* seeds,
                             int32_t* kept) {
    Robot rb = make_robot(r);
    int n = rb.dof;
#pragma omp parallel for schedule(static)
    for (int t = 0; t < T; ++t)
        rank_and_replicate(rb, *c, (uint64_t)(tid_offset + t), cost + (size_t)t * c->M,
                           theta + (size_t)t * n * c->M, seeds + (size_t)t * c->B * n,
                           kept + (size_t)t * c->K);
}

/* PJ-IK stage (Alg. 4): seeds f64 [T][B][n] -> theta f64 [T][B][n], ep/eo f64
 * [T][B], counts i32 [T][B][4] (LM, dogleg, single, perturb), margin f64 [T][B]
 * (smallest relative decision margin), iters i32 [T][B], trace u32
 * [T][B][lm_iters] or NULL (this oracle's own decision words, pj_word format;
 * 0 where no step was taken) */
void oracle_pj_ik(const OracleRobot* r, const OracleConfig* c, const float* targets, int32_t T,
                  int64_t tid_offset, const double* seeds, double* theta, double* ep, double* eo,
                  int32_t* counts, double* margin, int32_t* iters, uint32_t* trace) {
    Robot rb = make_robot(r);
    int n = rb.dof, B = c->B, I = c->lm_iters;
    int used = (c->B / c->K) * c->K;
    auto emit = [&](size_t o, const std::vector<double>& th, const PolishOut& po) {
        for (int j = 0; j < n; ++j) theta[o * n + j] = th[j];
        if (ep) ep[o] = po.ep;
        if (eo) eo[o] = po.eo;
        if (counts) for (int i = 0; i < 4; ++i) counts[o * 4 + i] = po.counts[i];
        if (margin) margin[o] = po.margin;
        if (iters) iters[o] = po.iters;
    };
    if (c->target_early_exit) {
#pragma omp parallel for schedule(dynamic, 1)
        for (int t = 0; t < T; ++t) {
            Target tgt = read_target(targets + (size_t)t * 7);
            std::vector<std::vector<double>> th(used);
            for (int b = 0; b < used; ++b) {
                size_t o = (size_t)t * B + b;
                th[b].assign(seeds + o * n, seeds + o * n + n);
            }
            std::vector<PolishOut> po;
            pj_ik_target(rb, *c, tgt, (uint64_t)(tid_offset + t), used, th, po,
                         trace ? trace + (size_t)t * B * I : nullptr, I);
            for (int b = 0; b < used; ++b) emit((size_t)t * B + b, th[b], po[b]);
        }
        return;
    }
#pragma omp parallel for collapse(2) schedule(dynamic, 2)
    for (int t = 0; t < T; ++t) {
        for (int b = 0; b < used; ++b) {
            Target tgt = read_target(targets + (size_t)t * 7);
            size_t o = (size_t)t * B + b;
            std::vector<double> th(seeds + o * n, seeds + o * n + n);
            PolishOut po = pj_ik_seed(rb, *c, tgt, (uint64_t)(tid_offset + t), (uint32_t)b, th,
                                      trace ? trace + o * I : nullptr);
            emit(o, th, po);
        }
    }
}

/* Decision replay of Alg. 4 (parity tests, DESIGN.md §4 "decision replay"):
 * every polish seed runs the GPU's iteration count iters [T][B] and, at each
 * iteration k, takes the GPU's recorded decision trace [T][B][lm_iters]
 * (hjcd_pjik_trace word = pj_word: branch | alpha index << 2 | i* << 8 |
 * 1 << 15) in place of its own, with J, W, every direction, trial and
 * perturbation computed here in fp64 as in pj_ik_step (pj_ik_step_replay).
 *   gap [T][B]: the largest amount by which a recorded decision is worse than
 *     this oracle's own (residual-norm units, see pj_ik_step_replay), and the
 *     depth inside the fine box (min(eps_p - ep, eps_o - eo)) at an iteration
 *     the GPU continued; 0 = all agree;
 *   gap_at [T][B] (or NULL): 8 k + kind of that largest gap (kinds of
 *     pj_ik_step_replay, 5 = continued inside the box), -1 none;
 *   stop_gap [T]: the distance outside the fine box of the seed closest to it
 *     where the GPU stopped before lm_iters (per target with
 *     target_early_exit, else the max over the seeds of their own); 0 if none.
 * theta f64 [T][B][n], ep/eo f64 [T][B], counts i32 [T][B][4] after the replay
 * (slots >= floor(B/K) K untouched).
 * theta_hist f32 [T][B][lm_iters + 1][n] or NULL: the GPU's theta at the
 *   start of every iteration (hjcd_pjik_trace); given, the replay is
 *   resynchronised on it at every iteration, judged also one ulp away (here
 *   the variants also carry one fp32 rounding in every entry of the normal
 *   matrices of the LM and dogleg solves, perturb_sym), and step_dev
 *   [T][B][3] (or NULL) receives the one-step differences, as in
 *   oracle_po_ccd_replay. */
void oracle_pj_ik_replay(const OracleRobot* r, const OracleConfig* c, const float* targets, int32_t T,
                         int64_t tid_offset, const double* seeds, const uint32_t* trace, const int32_t* iters,
                         double* theta, double* ep, double* eo, int32_t* counts, double* gap,
                         double* stop_gap, int32_t* gap_at, const float* theta_hist, double* step_dev) {
    Robot rb = make_robot(r);
    int n = rb.dof, B = c->B, I = c->lm_iters;
    int used = (c->B / c->K) * c->K;
#pragma omp parallel for schedule(dynamic, 1)
    for (int t = 0; t < T; ++t) {
        Target tgt = read_target(targets + (size_t)t * 7);
        uint64_t tid = (uint64_t)(tid_offset + t);
        double sg = c->target_early_exit ? INF : 0.0;
        bool stopped = false;
        for (int b = 0; b < used; ++b) {
            size_t o = (size_t)t * B + b;
            std::vector<double> th(seeds + o * n, seeds + o * n + n);
            PolishOut po = polish_init();
            Frames F;
            Err e;
            double g = 0.0, sd = 0.0, sdj = 0.0, sdx = -INF, spread = 0.0;
            int K = iters[o], kind = 0, at = -1;
            for (int k = 0;; ++k) {
                if (theta_hist && k <= I) {   /* resynchronise on the GPU's theta_k */
                    const float* h = theta_hist + (o * (size_t)(I + 1) + k) * n;
                    std::vector<double> hk(h, h + n);
                    if (k > 0) {
                        double dv = task_distance(rb, th.data(), hk.data());
                        sd = std::max(sd, dv);
                        sdx = std::max(sdx, dv - REPLAY_SPREAD_FACTOR * spread);
                        for (int j = 0; j < n; ++j) sdj = std::max(sdj, std::fabs(th[j] - hk[j]));
                    }
                    th = hk;
                }
                pj_ik_check(rb, *c, tgt, th, F, e, po);
                double inside = std::min(c->eps_p_fine - e.ep, c->eps_o_fine - e.eo);
                if (k == K) {
                    if (K < I) {
                        double outside = std::max(0.0, -inside);
                        stopped = true;
                        sg = c->target_early_exit ? std::min(sg, outside) : std::max(sg, outside);
                    }
                    break;
                }
                if (k >= I) { g = INF; at = 8 * k + 6; break; }   /* more iterations than the budget */
                if (inside > g) { g = inside; at = 8 * k + 5; }
                const uint32_t w = trace[o * I + k];
                std::vector<double> thk = th;
                double gk = 0.0;
                kind = 0;
                pj_ik_step_replay(rb, *c, tgt, tid, (uint32_t)b, k, F, e, th, po, w, &gk, &kind);
                spread = 0.0;
                if (theta_hist) {   /* as in oracle_po_ccd_replay */
                    for (int v = 1; v <= REPLAY_VARIANTS; ++v) {
                        std::vector<double> tv = thk;
                        perturb_ulp(rb, tv, (o * 1024 + (uint64_t)k) * 8 + (uint64_t)v);
                        Frames Fv;
                        Err ev;
                        PolishOut pov = polish_init();
                        pj_ik_check(rb, *c, tgt, tv, Fv, ev, pov);
                        double gv = 0.0;
                        int kv = 0;
                        uint64_t nrng = ((o * 1024 + (uint64_t)k) * 8 + (uint64_t)v) ^ 0x5bd1e995ull;
                        pj_ik_step_replay(rb, *c, tgt, tid, (uint32_t)b, k, Fv, ev, tv, pov, w, &gv, &kv, &nrng);
                        if (gv < gk) { gk = gv; kind = kv; }
                        spread = std::max(spread, task_distance(rb, th.data(), tv.data()));
                    }
                }
                if (gk > g) { g = gk; at = 8 * k + kind; }
                if (!std::isfinite(g)) break;
            }
            for (int j = 0; j < n; ++j) theta[o * n + j] = th[j];
            ep[o] = po.ep;
            eo[o] = po.eo;
            if (counts) for (int i = 0; i < 4; ++i) counts[o * 4 + i] = po.counts[i];
            gap[o] = g;
            if (gap_at) gap_at[o] = at;
            if (step_dev) { step_dev[3 * o] = sd; step_dev[3 * o + 1] = sdx; step_dev[3 * o + 2] = sdj; }
        }
        stop_gap[t] = stopped ? sg : 0.0;
    }
}

/* HJCD-IK (Alg. 2) end to end for T targets.
 * out: q f64 [T][n], pos_err/ori_err f64 [T], status i32 [T]
 * (0 converged at the fine tolerance, 1 success at succ_p/succ_o only,
 *  2 not converged, 3 invalid target). */
void oracle_solve(const OracleRobot* r, const OracleConfig* c, const float* targets, int32_t T,
                  int64_t tid_offset, double* q_out, double* pos_err, double* ori_err,
                  int32_t* status) {
    Robot rb = make_robot(r);
    int n = rb.dof, M = c->M, B = c->B, K = c->K;
#pragma omp parallel for schedule(dynamic, 1)
    for (int t = 0; t < T; ++t) {
        Target tgt = read_target(targets + (size_t)t * 7);
        uint64_t tid = (uint64_t)(tid_offset + t);
        if (!tgt.valid) {
            for (int j = 0; j < n; ++j) q_out[(size_t)t * n + j] = 0.0;
            pos_err[t] = INF; ori_err[t] = INF; status[t] = 3;
            continue;
        }
        /* stage 1: PO-CCD over M seeds */
        std::vector<double> theta_nm((size_t)n * M), cost(M);
        std::vector<std::vector<double>> th1(M, std::vector<double>(n));
        std::vector<SeedOut> so1(M);
        for (int m = 0; m < M; ++m) uniform_seed(rb, c->rng_seed, tid, (uint32_t)m, th1[m].data());
        if (c->ccd_early_exit) {
            po_ccd_target(rb, *c, tgt, tid, M, th1, so1);   /* P:203 stop rule (R12b) */
        } else {
            for (int m = 0; m < M; ++m) so1[m] = po_ccd_seed(rb, *c, tgt, tid, (uint32_t)m, th1[m]);
        }
        for (int m = 0; m < M; ++m) {
            for (int j = 0; j < n; ++j) theta_nm[(size_t)j * M + m] = th1[m][j];
            cost[m] = rank_cost(*c, so1[m].ep, so1[m].eo);
        }
        /* top-K + replicate */
        std::vector<double> seeds((size_t)B * n);
        std::vector<int32_t> kept(K);
        rank_and_replicate(rb, *c, tid, cost.data(), theta_nm.data(), seeds.data(), kept.data());
        /* stage 2: PJ-IK over the B polish seeds, best by c(theta) (R27) */
        int used = (B / K) * K;
        std::vector<std::vector<double>> th2(used);
        std::vector<PolishOut> po(used);
        for (int b = 0; b < used; ++b)
            th2[b].assign(seeds.begin() + (size_t)b * n, seeds.begin() + (size_t)b * n + n);
        if (c->target_early_exit) {
            pj_ik_target(rb, *c, tgt, tid, used, th2, po);
        } else {
            for (int b = 0; b < used; ++b) po[b] = pj_ik_seed(rb, *c, tgt, tid, (uint32_t)b, th2[b]);
        }
        /* R27: theta* = argmin over (not fine-converged, c), ties -> lowest slot:
         * a seed that passed Alg. 4 l.18 is the answer the break returns */
        int btier = 2;
        double best = INF;
        double bep = INF, beo = INF;
        std::vector<double> bth(n, 0.0);
        for (int b = 0; b < used; ++b) {
            int tier = (po[b].ep < c->eps_p_fine && po[b].eo < c->eps_o_fine) ? 0 : 1;
            double cb = rank_cost(*c, po[b].ep, po[b].eo);
            if (!(cb >= 0)) cb = INF;
            if (tier < btier || (tier == btier && cb < best)) {
                btier = tier; best = cb; bep = po[b].ep; beo = po[b].eo; bth = th2[b];
            }
        }
        for (int j = 0; j < n; ++j) q_out[(size_t)t * n + j] = bth[j];
        pos_err[t] = bep;
        ori_err[t] = beo;
        if (bep < c->eps_p_fine && beo < c->eps_o_fine) status[t] = 0;
        else if (bep < c->succ_p && beo < c->succ_o) status[t] = 1;
        else status[t] = 2;
    }
}

/* host threads for the OpenMP loops (bench.py's cpu_baseline times 1 and all) */
void oracle_set_num_threads(int32_t k) {
#ifdef _OPENMP
    if (k > 0) omp_set_num_threads(k);
#else
    (void)k;
#endif
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

} /* extern "C" */

#pragma once
// poccd_x2.cuh — k_poccd_x2: PO-CCD (Alg. 3) with the paper's stop
// rule (R12b) for TWO seeds per thread, every fp32 operation on the
// pair issued as ONE packed sm_100a instruction (FFMA2 / FMUL2 / FADD2 on
// (seed 2i, seed 2i + 1)); K17.
//
// Why: k_poccd is issue-bound (~70 % issue-active, FP32 pipe
// ~40 %), and half of its instructions are scalar fp32 add / mul / fma.  A
// packed instruction does the same per-lane arithmetic (same rounding) in one
// issue slot, so the seed pair costs one FP instruction where two seeds in two
// threads cost two.  Unlike packing joint pairs (K13, dropped), the data is born
// packed: the two seeds of a thread run the same chain in lockstep (R12b makes
// every seed of a target run the same number of iterations), so every
// per-seed value is naturally a (seed a, seed b) pair.  What stays per seed:
// SFU (sincos, rsqrt), comparisons and selects (argmins, clamps), Philox.
//
// Per seed the arithmetic is that of k_poccd<..., TEXIT = true, ...> up to the
// association of a few sums (the FK translation accumulates in FMAs) and the
// SFU forms of sqrt and of atan2's ratio (fp32-rounding-level differences;
// the decision replay judges the decisions), with one layout
// change: the frames (P_j, z_j) live only in
// shared memory, [joint][3][thread] float4 = {Px, Py}, {Pz, zx}, {zy, zz} of
// the pair, written by the FK and read back joint by joint by the candidate
// loop and the gamma test (keeping 2 x 6 n frame floats in registers would
// halve the occupancy).
//
// Mapping: the M seeds of a target live in one thread-block cluster of CL CTAs
// x nt threads; thread i of CTA rank r holds seeds m = 2 (r nt + i) and m + 1.
#include <cooperative_groups.h>
#include <cstdlib>

#include "kin.cuh"

namespace cg = cooperative_groups;

#ifndef HJCD_VOTE_RELAXED
#define HJCD_VOTE_RELAXED 1
#endif
// K40 (A/B): the two warp-voted branches of the iteration taken unconditionally
#ifndef HJCD_X2_UNIFORM
#define HJCD_X2_UNIFORM 1
#endif

namespace hjcd {
namespace px {

// ---- packed fp32 pairs (lane 0 = seed a, lane 1 = seed b)
__device__ __forceinline__ f2 operator+(f2 a, f2 b) { return add2(a, b); }
__device__ __forceinline__ f2 operator*(f2 a, f2 b) { return mul2(a, b); }
__device__ __forceinline__ f2 operator-(f2 a, f2 b) {
    f2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
    return r;
}
__device__ __forceinline__ f2 neg(f2 a) {
    float x, y;
    unpk2(a, x, y);
    return mk2(-x, -y);   // folded into the consumer's operand by ptxas
}
__device__ __forceinline__ float lo(f2 a) {
    float x, y;
    unpk2(a, x, y);
    return x;
}
__device__ __forceinline__ float hi(f2 a) {
    float x, y;
    unpk2(a, x, y);
    return y;
}
__device__ __forceinline__ float lane(f2 a, int s) { return s ? hi(a) : lo(a); }

struct V {
    f2 x, y, z;
};
__device__ __forceinline__ V operator+(V a, V b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ V operator-(V a, V b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ V scale(f2 s, V a) { return {s * a.x, s * a.y, s * a.z}; }
// a.x b.x + a.y b.y + a.z b.z, contracted as nvcc contracts the scalar dot3
__device__ __forceinline__ f2 dot(V a, V b) { return fma2(a.z, b.z, fma2(a.y, b.y, a.x * b.x)); }
// a x b, each component as the scalar cross3 contracts: a.y b.z - a.z b.y
__device__ __forceinline__ V cross(V a, V b) {
    return {fma2(a.y, b.z, neg(a.z * b.y)), fma2(a.z, b.x, neg(a.x * b.z)), fma2(a.x, b.y, neg(a.y * b.x))};
}
// a - s b
__device__ __forceinline__ V axpy_neg(V a, f2 s, V b) { return {fma2(neg(s), b.x, a.x), fma2(neg(s), b.y, a.y), fma2(neg(s), b.z, a.z)}; }
__device__ __forceinline__ V bcv(float3 a) { return {bc2(a.x), bc2(a.y), bc2(a.z)}; }

struct Q {
    f2 w, x, y, z;
};

// q_err = q_t (x) conj(q_e), canonicalised to w >= 0 (Eq. 5, R1), per lane
__device__ __forceinline__ Q quat_err2(Quat qt, Q qe) {
    Q r;
    r.w = fma2(bc2(qt.z), qe.z, fma2(bc2(qt.y), qe.y, fma2(bc2(qt.x), qe.x, bc2(qt.w) * qe.w)));
    r.x = fma2(bc2(qt.z), qe.y, fma2(bc2(-qt.y), qe.z, fma2(bc2(qt.x), qe.w, bc2(-qt.w) * qe.x)));
    r.y = fma2(bc2(qt.z), neg(qe.x), fma2(bc2(qt.y), qe.w, fma2(bc2(qt.x), qe.z, bc2(-qt.w) * qe.y)));
    r.z = fma2(bc2(qt.z), qe.w, fma2(bc2(qt.y), qe.x, fma2(bc2(-qt.x), qe.y, bc2(-qt.w) * qe.z)));
    const f2 sg = mk2(lo(r.w) < 0.f ? -1.f : 1.f, hi(r.w) < 0.f ? -1.f : 1.f);
    r.w = r.w * sg; r.x = r.x * sg; r.y = r.y * sg; r.z = r.z * sg;
    return r;
}

// kin.cuh quat_from_rot for the pair: the pivot choice per lane, the
// arithmetic packed (per lane the same operations)
__device__ __forceinline__ Q quat_from_rot2(const f2 (&R)[9]) {
    const f2 one = bc2(1.f);
    const f2 t0 = ((one + R[0]) + R[4]) + R[8];
    const f2 t1 = ((one + R[0]) - R[4]) - R[8];
    const f2 t2 = ((one - R[0]) + R[4]) - R[8];
    const f2 t3 = ((one - R[0]) - R[4]) + R[8];
    const f2 a = R[7] - R[5], b = R[2] - R[6], cc = R[3] - R[1];
    const f2 d = R[1] + R[3], e = R[2] + R[6], f = R[5] + R[7];
    const f2 tr = (R[0] + R[4]) + R[8];
    float t[2], qw[2], qx[2], qy[2], qz[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        const bool pw = lane(tr, s) > 0.f;
        const bool pxx = !pw && lane(R[0], s) > lane(R[4], s) && lane(R[0], s) > lane(R[8], s);
        const bool py = !pw && !pxx && lane(R[4], s) > lane(R[8], s);
        if (pw) { t[s] = lane(t0, s); qw[s] = lane(t0, s); qx[s] = lane(a, s); qy[s] = lane(b, s); qz[s] = lane(cc, s); }
        else if (pxx) { t[s] = lane(t1, s); qw[s] = lane(a, s); qx[s] = lane(t1, s); qy[s] = lane(d, s); qz[s] = lane(e, s); }
        else if (py) { t[s] = lane(t2, s); qw[s] = lane(b, s); qx[s] = lane(d, s); qy[s] = lane(t2, s); qz[s] = lane(f, s); }
        else { t[s] = lane(t3, s); qw[s] = lane(cc, s); qx[s] = lane(e, s); qy[s] = lane(f, s); qz[s] = lane(t3, s); }
    }
    const f2 is = bc2(0.5f) * mk2(rsqrtf(t[0]), rsqrtf(t[1]));
    Q q = {mk2(qw[0], qw[1]) * is, mk2(qx[0], qx[1]) * is, mk2(qy[0], qy[1]) * is, mk2(qz[0], qz[1]) * is};
    const f2 nn = fma2(q.z, q.z, fma2(q.y, q.y, fma2(q.x, q.x, q.w * q.w)));
    float i0 = rsqrtf(lo(nn)), i1 = rsqrtf(hi(nn));
    if (lo(q.w) < 0.f) i0 = -i0;
    if (hi(q.w) < 0.f) i1 = -i1;
    const f2 inv = mk2(i0, i1);
    q.w = q.w * inv; q.x = q.x * inv; q.y = q.y * inv; q.z = q.z * inv;
    return q;
}

// q_err (x) q(z, -d) for the pair (kin.cuh qerr_rotate)
__device__ __forceinline__ Q qerr_rotate2(Q q, V z, f2 c2, f2 s2) {
    Q r;
    const f2 vz = fma2(q.z, z.z, fma2(q.y, z.y, q.x * z.x));
    const f2 cx = fma2(q.y, z.z, neg(q.z * z.y)), cy = fma2(q.z, z.x, neg(q.x * z.z)),
             cz = fma2(q.x, z.y, neg(q.y * z.x));
    r.w = fma2(vz, s2, q.w * c2);
    const f2 sw = s2 * q.w;
    r.x = fma2(neg(s2), cx, fma2(neg(sw), z.x, c2 * q.x));
    r.y = fma2(neg(s2), cy, fma2(neg(sw), z.y, c2 * q.y));
    r.z = fma2(neg(s2), cz, fma2(neg(sw), z.z, c2 * q.z));
    return r;
}

// the end effector rotated about a joint axis by d (s2, c2 = sin, cos of d/2;
// up = the end effector's offset from the axis, zxu = z x (P_ee - P_j)):
// p - (2 s2 s2) up + (2 s2 c2) zxu, contracted as the scalar kernel's K3
__device__ __forceinline__ V rot_about(V p, V up, V zxu, f2 s2, f2 c2) {
    const f2 a = (bc2(2.f) * s2) * s2, b = (bc2(2.f) * s2) * c2;
    return {fma2(b, zxu.x, fma2(neg(a), up.x, p.x)), fma2(b, zxu.y, fma2(neg(a), up.y, p.y)),
            fma2(b, zxu.z, fma2(neg(a), up.z, p.z))};
}

// per-lane helpers
__device__ __forceinline__ f2 sqrt2(f2 a) { return mk2(sqrt_approx(lo(a)), sqrt_approx(hi(a))); }
// kin.cuh fast_atan2f for the pair: octant reduction per lane, the
// polynomial packed (per lane the same operations)
__device__ __forceinline__ f2 atan2_2(f2 y, f2 x) {
    float r[2], ax[2], ay[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        ax[s] = fabsf(lane(x, s));
        ay[s] = fabsf(lane(y, s));
        const float mx = fmaxf(ax[s], ay[s]), mn = fminf(ax[s], ay[s]);
        r[s] = mx > 0.f ? mn * rcp_approx(mx) : 0.f;
    }
    const f2 rr = mk2(r[0], r[1]);
    const f2 sq = rr * rr;
    f2 p = bc2(-0.00405456f);
    p = fma2(p, sq, bc2(0.02186293f));
    p = fma2(p, sq, bc2(-0.05591229f));
    p = fma2(p, sq, bc2(0.09642195f));
    p = fma2(p, sq, bc2(-0.13908629f));
    p = fma2(p, sq, bc2(0.19946566f));
    p = fma2(p, sq, bc2(-0.3332986f));
    p = fma2(p, sq, bc2(0.99999934f));
    const f2 a = p * rr;
    float o[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        float v = lane(a, s);
        v = (ay[s] > ax[s]) ? 1.57079637f - v : v;
        v = (lane(x, s) < 0.f) ? 3.14159274f - v : v;
        o[s] = copysignf(v, lane(y, s));
    }
    return mk2(o[0], o[1]);
}
__device__ __forceinline__ void sincos2(f2 a, f2& s, f2& c) {
    float s0, c0, s1, c1;
    __sincosf(lo(a), &s0, &c0);
    __sincosf(hi(a), &s1, &c1);
    s = mk2(s0, s1);
    c = mk2(c0, c1);
}
__device__ __forceinline__ f2 clamp2(f2 x, float l, float h) { return mk2(clampf(lo(x), l, h), clampf(hi(x), l, h)); }

// frames in shared memory: [joint][3][FR] float4 {Px_a, Px_b, Py_a, Py_b},
// {Pz_a, Pz_b, zx_a, zx_b}, {zy_a, zy_b, zz_a, zz_b}; the stride is the
// compile-time maximum CTA size, so every offset is an immediate
constexpr int FR = 128;
__device__ __forceinline__ void store_frame(float4* s, int j, V P, V Z) {
    float4* p = s + (3 * j) * FR + threadIdx.x;
    p[0] = make_float4(lo(P.x), hi(P.x), lo(P.y), hi(P.y));
    p[FR] = make_float4(lo(P.z), hi(P.z), lo(Z.x), hi(Z.x));
    p[2 * FR] = make_float4(lo(Z.y), hi(Z.y), lo(Z.z), hi(Z.z));
}
__device__ __forceinline__ void load_frame(const float4* s, int j, V& P, V& Z) {
    const float4* p = s + (3 * j) * FR + threadIdx.x;
    const float4 a = p[0], b = p[FR], c = p[2 * FR];
    P = {mk2(a.x, a.y), mk2(a.z, a.w), mk2(b.x, b.y)};
    Z = {mk2(b.z, b.w), mk2(c.x, c.y), mk2(c.z, c.w)};
}
// joint ja of lane 0 and joint jb of lane 1 (the winners differ per seed)
__device__ __forceinline__ void load_frame_lanes(const float4* s, int j0, int j1, V& P, V& Z) {
    const float4* p0 = s + (3 * j0) * FR + threadIdx.x;
    const float4* p1 = s + (3 * j1) * FR + threadIdx.x;
    const float4 a0 = p0[0], b0 = p0[FR], c0 = p0[2 * FR];
    const float4 a1 = p1[0], b1 = p1[FR], c1 = p1[2 * FR];
    P = {mk2(a0.x, a1.y), mk2(a0.z, a1.w), mk2(b0.x, b1.y)};
    Z = {mk2(b0.z, b1.w), mk2(c0.x, c1.y), mk2(c0.z, c1.w)};
}

}  // namespace px

// FK of the pair (Eq. 1; kin.cuh fk, general or REV = 2 DH-twist form), frames
// to shared memory; returns the end-effector position and orientation
template <int NMAX, bool EXACT, int REV>
__device__ __forceinline__ void fk_x2(const DevRobot& rb, const f2 (&th)[NMAX], float4* s_fr,
                                      px::V& pe, px::Q& qe) {
    using namespace px;
    f2 R[9] = {bc2(1.f), bc2(0.f), bc2(0.f), bc2(0.f), bc2(1.f), bc2(0.f), bc2(0.f), bc2(0.f), bc2(1.f)};
    f2 tx = bc2(0.f), ty = bc2(0.f), tz = bc2(0.f);
#pragma unroll
    for (int j = 0; j < NMAX; ++j) {
        if (EXACT || j < rb.n) {
            const DevJoint& J = rb.j[j];
            // t += R F_j.t, accumulated into t (three FMAs per component)
            tx = fma2(R[2], bc2(J.t[2]), fma2(R[1], bc2(J.t[1]), fma2(R[0], bc2(J.t[0]), tx)));
            ty = fma2(R[5], bc2(J.t[2]), fma2(R[4], bc2(J.t[1]), fma2(R[3], bc2(J.t[0]), ty)));
            tz = fma2(R[8], bc2(J.t[2]), fma2(R[7], bc2(J.t[1]), fma2(R[6], bc2(J.t[0]), tz)));
            f2 N[9];
            if constexpr (REV == 2) {
#pragma unroll
                for (int r = 0; r < 3; ++r) {
                    N[3 * r] = R[3 * r];
                    N[3 * r + 1] = fma2(R[3 * r + 2], bc2(J.R[7]), R[3 * r + 1] * bc2(J.R[4]));
                    N[3 * r + 2] = fma2(R[3 * r + 2], bc2(J.R[8]), R[3 * r + 1] * bc2(J.R[5]));
                }
            } else {
#pragma unroll
                for (int r = 0; r < 3; ++r)
#pragma unroll
                    for (int cc = 0; cc < 3; ++cc)
                        N[3 * r + cc] = fma2(R[3 * r + 2], bc2(J.R[6 + cc]),
                                             fma2(R[3 * r + 1], bc2(J.R[3 + cc]), R[3 * r] * bc2(J.R[cc])));
            }
            store_frame(s_fr, j, V{tx, ty, tz}, V{N[2], N[5], N[8]});
            if (REV || J.type == HJCD_REVOLUTE) {
                f2 s, c;
                sincos2(th[j], s, c);   // K5: SFU sines in the coarse stage
#pragma unroll
                for (int r = 0; r < 3; ++r) {
                    const f2 a = N[3 * r], b = N[3 * r + 1];
                    R[3 * r] = fma2(s, b, c * a);
                    R[3 * r + 1] = fma2(neg(s), a, c * b);
                    R[3 * r + 2] = N[3 * r + 2];
                }
            } else {
#pragma unroll
                for (int i = 0; i < 9; ++i) R[i] = N[i];
                tx = fma2(th[j], N[2], tx);
                ty = fma2(th[j], N[5], ty);
                tz = fma2(th[j], N[8], tz);
            }
        }
    }
    tx = fma2(R[2], bc2(rb.eet[2]), fma2(R[1], bc2(rb.eet[1]), fma2(R[0], bc2(rb.eet[0]), tx)));
    ty = fma2(R[5], bc2(rb.eet[2]), fma2(R[4], bc2(rb.eet[1]), fma2(R[3], bc2(rb.eet[0]), ty)));
    tz = fma2(R[8], bc2(rb.eet[2]), fma2(R[7], bc2(rb.eet[1]), fma2(R[6], bc2(rb.eet[0]), tz)));
    f2 E[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int cc = 0; cc < 3; ++cc)
            E[3 * r + cc] = fma2(R[3 * r + 2], bc2(rb.eeR[6 + cc]),
                                 fma2(R[3 * r + 1], bc2(rb.eeR[3 + cc]), R[3 * r] * bc2(rb.eeR[cc])));
    pe = {tx, ty, tz};
    qe = quat_from_rot2(E);
}

#ifndef HJCD_X2_MINB
#define HJCD_X2_MINB 4
#endif
template <int NMAX>
constexpr int poccd_x2_min_blocks() { return HJCD_X2_MINB; }

template <int NMAX, bool EXACT, int REV>
__global__ void __launch_bounds__(128, poccd_x2_min_blocks<NMAX>())
k_poccd_x2(const __grid_constant__ DevRobot rb, const __grid_constant__ DevCfg c,
           const float* __restrict__ targets, int T, float* __restrict__ theta_out, float* __restrict__ cost_out,
           float* __restrict__ ep_out, float* __restrict__ eo_out, int32_t* __restrict__ iters_out, int CL,
           const TraceOut trace, uint32_t* __restrict__ ready) {
    using namespace px;
    const int M = c.M;
    const int n = rb.n;
    const int nt = (int)blockDim.x;
    __shared__ int s_flag[3];
    extern __shared__ float4 s_fr[];   // [NMAX][3][FR] frames of the pair
    const int t = (int)(blockIdx.x / (unsigned)CL);
    const int m0 = 2 * ((int)(blockIdx.x - (unsigned)t * CL) * nt + (int)threadIdx.x);
    const bool act[2] = {m0 < M, m0 + 1 < M};
    // DESIGN K10: the dependent PJ-IK grid may be scheduled once every CTA of
    // this grid is resident or done
    if (ready) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x < 3) s_flag[threadIdx.x] = 0;
    cg::this_cluster().sync();   // flags initialised before any remote store
    const Target tg = load_target(targets + 7ll * t);
    const uint32_t tid = (uint32_t)(c.tid_offset + t);
    const V tp = bcv(tg.p);

    // ---- Alg. 3 l.2-3: theta ~ U(theta_min, theta_max) (fp32 fma: R30), per seed
    f2 th[NMAX];
    {
        float tl[2][NMAX];
#pragma unroll
        for (int s = 0; s < 2; ++s) {
#pragma unroll
            for (int blk = 0; blk < (NMAX + 3) / 4; ++blk) {
                if (EXACT || 4 * blk < n) {
                    uint4 r = draw(c, tid, (uint32_t)(m0 + s), P_INIT, 0u, (uint32_t)blk);
                    uint32_t x[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int j = 4 * blk + e;
                        if (j < NMAX && (EXACT || j < n)) {
                            const float l = rb.j[j].lo, h = rb.j[j].hi;
                            tl[s][j] = __fmaf_rn(__fsub_rn(h, l), u01(x[e]), l);
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int j = 0; j < NMAX; ++j) th[j] = (EXACT || j < n) ? mk2(tl[0][j], tl[1][j]) : bc2(0.f);
    }

    V pe;
    Q qe;
    f2 ep2 = bc2(0.f), eo2 = bc2(0.f);
    float rho_k = 1.f;   // delta_rho^k, by repeated multiplication (R5)
    int k;
    for (k = 0;; ++k, rho_k *= c.delta_rho) {
        if (trace.theta) {   // theta at the start of iteration k (hjcd_poccd_trace)
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                if (act[s]) {
                    float* h = trace.theta + (((long long)t * M + m0 + s) * (c.ccd_iters + 1) + k) * n;
#pragma unroll
                    for (int j = 0; j < NMAX; ++j)
                        if (EXACT || j < n) h[j] = lane(th[j], s);
                }
            }
        }
        fk_x2<NMAX, EXACT, REV>(rb, th, s_fr, pe, qe);
        const V rp = tp - pe;                        // r_p (Eq. 4)
        const Q qr = quat_err2(tg.q, qe);             // q_err (Eq. 5), w >= 0
        const f2 sv2 = fma2(qr.z, qr.z, fma2(qr.y, qr.y, qr.x * qr.x));
        const f2 sv = sqrt2(sv2);
        ep2 = sqrt2(dot(rp, rp));
        eo2 = bc2(2.f) * atan2_2(sv, qr.w);            // |omega|
        // Alg. 3 l.14: coarse test (R12), checked at iteration start; R12b:
        // cluster-wide OR of the votes of iteration k (flag ring as k_poccd)
        const bool conv = (act[0] && lo(ep2) < c.eps_p_coarse && lo(eo2) < c.eps_o_coarse) ||
                          (act[1] && hi(ep2) < c.eps_p_coarse && hi(eo2) < c.eps_o_coarse);
        {
            cg::cluster_group cluster = cg::this_cluster();
            const int slot = k % 3;
            const unsigned vote = __ballot_sync(0xffffffffu, conv);
#if HJCD_VOTE_RELAXED
            // K31: one flag tagged with the iteration (k + 1 means "a seed
            // passed at k"; nothing resets it: if any seed passed at k every
            // CTA stops at k, so no later tag can overwrite it unread), written
            // and fenced by the voting lanes only, then a RELAXED cluster
            // arrive: the default release arrive fences every warp-iteration
            (void)slot;
            if (vote && (threadIdx.x & 31) == 0) {
                for (int r = 0; r < CL; ++r) *cluster.map_shared_rank(&s_flag[0], r) = k + 1;
                asm volatile("fence.acq_rel.cluster;" ::: "memory");
            }
            asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
            if (*(volatile int*)&s_flag[0] == k + 1) break;
#else
            if (vote && (threadIdx.x & 31) == 0)
                for (int r = 0; r < CL; ++r) *cluster.map_shared_rank(&s_flag[slot], r) = 1;
            cluster.sync();
            const bool any = s_flag[slot] != 0;
            if (threadIdx.x == 0) s_flag[(k + 2) % 3] = 0;
            if (any) break;
#endif
        }
        if (k == c.ccd_iters) break;

        // Eq. 10 (R2): phi = |omega|, a = v / |v|; sgn(a . z_j) = sgn(v . z_j)
        const V vq = {qr.x, qr.y, qr.z};
        const float dk = fmaxf(c.delta_min, c.delta0 * rho_k);
        const f2 dphi = mk2(lo(eo2) > 0.f ? dk * lo(eo2) : 0.f, hi(eo2) > 0.f ? dk * hi(eo2) : 0.f);
        const float tau2 = c.tau_deg * c.tau_deg;
        // K2b: |v'|^2 = C^2 |v|^2 + S^2 (w^2 + |v|^2 - (v.z)^2) - 2 C S w |v.z|
        f2 Sd, Cd;
        sincos2(bc2(0.5f) * dphi, Sd, Cd);
        const f2 w2 = qr.w * qr.w, wsv2 = w2 + sv2, ka = sv2 + wsv2;
        const f2 ob0 = fma2(Sd * Sd, wsv2, (Cd * Cd) * sv2);
        const f2 ob1 = Sd * Sd, ob2 = ((bc2(2.f) * Cd) * Sd) * qr.w;
        const f2 svsq = sv * sv;   // the score of a zero orientation step (the current residual)

        // ---- Alg. 3 l.6-9: per-joint candidates, scored, greedy argmin (per seed)
        float best_p[2] = {CUDART_INF_F, CUDART_INF_F}, best_o[2] = {CUDART_INF_F, CUDART_INF_F};
        int jp[2] = {0, 0}, jo[2] = {0, 0};
        float dpb[2] = {0.f, 0.f}, dob[2] = {0.f, 0.f};
#pragma unroll
        for (int j = 0; j < NMAX; ++j) {
            if (EXACT || j < n) {
                const DevJoint& J = rb.j[j];
                V Pj, z;
                load_frame(s_fr, j, Pj, z);
                f2 dp, sp, dor, so;
                if (REV || J.type == HJCD_REVOLUTE) {
                    // Eqs. 8-9 (R3): signed angle between the projections of
                    // u = P_ee - P_j and v = P_t - P_j on the plane normal to z_j
                    const V u = pe - Pj;
                    const V v = tp - Pj;
                    const V up = axpy_neg(u, dot(u, z), z);
                    const V vp = axpy_neg(v, dot(v, z), z);
                    const V zxu = cross(z, u);
                    const f2 uu = dot(up, up), vv = dot(vp, vp);
                    const f2 stp = atan2_2(dot(zxu, vp), dot(up, vp));
                    const f2 step = mk2(lo(uu) >= tau2 && lo(vv) >= tau2 ? lo(stp) : 0.f,
                                        hi(uu) >= tau2 && hi(vv) >= tau2 ? hi(stp) : 0.f);   // R4
                    dp = clamp2(th[j] + step, J.lo, J.hi) - th[j];     // R7
                    // score (K2): r_p' = r_p + (1 - cos d) u_perp - sin d (z x u)
                    f2 s2, c2;
                    sincos2(bc2(0.5f) * dp, s2, c2);
                    // a zero step scores the current residual exactly: s2 = 0 makes sn =
                    // omc = 0 whatever c2 is
                    s2 = mk2(lo(dp) == 0.f ? 0.f : lo(s2), hi(dp) == 0.f ? 0.f : hi(s2));
                    const f2 sn = (bc2(2.f) * s2) * c2, omc = (bc2(2.f) * s2) * s2;
                    const V r2 = {fma2(neg(sn), zxu.x, fma2(omc, up.x, rp.x)), fma2(neg(sn), zxu.y, fma2(omc, up.y, rp.y)),
                                  fma2(neg(sn), zxu.z, fma2(omc, up.z, rp.z))};
                    sp = dot(r2, r2);
                    // Eq. 11 (R5): delta(k) sgn(a . z_j) phi, sgn(0) = 0
                    const f2 vz = dot(vq, z);
                    const float vz0 = lo(vz), vz1 = hi(vz);
                    const f2 tsum = th[j] + mk2(vz0 != 0.f ? copysignf(lo(dphi), vz0) : 0.f,
                                                vz1 != 0.f ? copysignf(hi(dphi), vz1) : 0.f);
                    dor = clamp2(tsum, J.lo, J.hi) - th[j];
                    // score (K2b): |v'|^2 of q_err (x) q(z, -d), monotone in |omega'|
                    const f2 avz = mk2(fabsf(vz0), fabsf(vz1));
                    const f2 so_un = fma2(neg(avz), fma2(ob1, avz, ob2), ob0);
                    const bool cl0 = !(lo(tsum) >= J.lo && lo(tsum) <= J.hi) && lo(dor) != 0.f;
                    const bool cl1 = !(hi(tsum) >= J.lo && hi(tsum) <= J.hi) && hi(dor) != 0.f;
                    f2 so_cl = so_un;
                    if (HJCD_X2_UNIFORM || __any_sync(0xffffffffu, cl0 || cl1)) {
                        // clamped step: the closed form at the effective d, in double angles
                        f2 sd, cd;
                        sincos2(dor, sd, cd);
                        const f2 vz2 = vz * vz;
                        so_cl = fma2(neg(sd), qr.w * vz, bc2(0.5f) * fma2(cd, vz2 - w2, ka - vz2));
                    }
                    so = mk2(lo(dor) == 0.f ? lo(svsq) : (cl0 ? lo(so_cl) : lo(so_un)),
                             hi(dor) == 0.f ? hi(svsq) : (cl1 ? hi(so_cl) : hi(so_un)));
                } else {
                    // prismatic (R32): exact 1-D minimiser z . (P_t - P_ee)
                    dp = clamp2(th[j] + dot(z, rp), J.lo, J.hi) - th[j];
                    const V r2 = axpy_neg(rp, dp, z);
                    sp = dot(r2, r2);
                    dor = bc2(0.f);
                    so = svsq;
                }
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    const float sps = lane(sp, s), sos = lane(so, s);
                    if (sps < best_p[s]) { best_p[s] = sps; jp[s] = j; dpb[s] = lane(dp, s); }
                    if (sos < best_o[s]) { best_o[s] = sos; jo[s] = j; dob[s] = lane(dor, s); }
                }
            }
        }

        // ---- Alg. 3 l.10 + P:201: same joint -> the larger |step|, tie -> position (R8)
        int ja[2], jb[2];
        float da[2], db[2];
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            ja[s] = -1; da[s] = 0.f;
            if (jp[s] == jo[s]) {
                jb[s] = jp[s];
                db[s] = fabsf(dpb[s]) >= fabsf(dob[s]) ? dpb[s] : dob[s];
            } else if (jp[s] < jo[s]) {
                ja[s] = jp[s]; da[s] = dpb[s]; jb[s] = jo[s]; db[s] = dob[s];
            } else {
                ja[s] = jo[s]; da[s] = dob[s]; jb[s] = jp[s]; db[s] = dpb[s];
            }
        }
        // r(theta_hat) exactly (DESIGN K3): the downstream joint's rigid motion
        // first, then the upstream one, both about the pre-update frames
        V p2 = pe;
        Q q2 = qr;
        {
            V Pb, Zb;
            load_frame_lanes(s_fr, jb[0], jb[1], Pb, Zb);
            const bool rb0 = REV || !((rb.pmask >> jb[0]) & 1u), rb1 = REV || !((rb.pmask >> jb[1]) & 1u);
            const f2 dbb = mk2(db[0], db[1]);
            f2 s2, c2;
            sincos2(bc2(0.5f) * dbb, s2, c2);
            const V u = p2 - Pb;
            const V up = axpy_neg(u, dot(u, Zb), Zb);
            const V pr = rot_about(p2, up, cross(Zb, u), s2, c2);
            const Q qrr = qerr_rotate2(q2, Zb, c2, s2);
            const V pt = {fma2(dbb, Zb.x, p2.x), fma2(dbb, Zb.y, p2.y), fma2(dbb, Zb.z, p2.z)};   // prismatic
            p2 = {mk2(rb0 ? lo(pr.x) : lo(pt.x), rb1 ? hi(pr.x) : hi(pt.x)),
                  mk2(rb0 ? lo(pr.y) : lo(pt.y), rb1 ? hi(pr.y) : hi(pt.y)),
                  mk2(rb0 ? lo(pr.z) : lo(pt.z), rb1 ? hi(pr.z) : hi(pt.z))};
            q2 = {mk2(rb0 ? lo(qrr.w) : lo(q2.w), rb1 ? hi(qrr.w) : hi(q2.w)),
                  mk2(rb0 ? lo(qrr.x) : lo(q2.x), rb1 ? hi(qrr.x) : hi(q2.x)),
                  mk2(rb0 ? lo(qrr.y) : lo(q2.y), rb1 ? hi(qrr.y) : hi(q2.y)),
                  mk2(rb0 ? lo(qrr.z) : lo(q2.z), rb1 ? hi(qrr.z) : hi(q2.z))};
        }
        if (HJCD_X2_UNIFORM || __any_sync(0xffffffffu, ja[0] >= 0 || ja[1] >= 0)) {
            V Pa, Za;
            load_frame_lanes(s_fr, ja[0] >= 0 ? ja[0] : 0, ja[1] >= 0 ? ja[1] : 0, Pa, Za);
            const bool ra0 = REV || (ja[0] >= 0 && !((rb.pmask >> ja[0]) & 1u));
            const bool ra1 = REV || (ja[1] >= 0 && !((rb.pmask >> ja[1]) & 1u));
            const f2 daa = mk2(da[0], da[1]);   // 0 where there is no second joint: identity
            f2 s2, c2;
            sincos2(bc2(0.5f) * daa, s2, c2);
            const V u = p2 - Pa;
            const V up = axpy_neg(u, dot(u, Za), Za);
            const V pr = rot_about(p2, up, cross(Za, u), s2, c2);
            const Q qrr = qerr_rotate2(q2, Za, c2, s2);
            const V pt = {fma2(daa, Za.x, p2.x), fma2(daa, Za.y, p2.y), fma2(daa, Za.z, p2.z)};
            const bool u0 = ja[0] >= 0, u1 = ja[1] >= 0;
            p2 = {mk2(u0 ? (ra0 ? lo(pr.x) : lo(pt.x)) : lo(p2.x), u1 ? (ra1 ? hi(pr.x) : hi(pt.x)) : hi(p2.x)),
                  mk2(u0 ? (ra0 ? lo(pr.y) : lo(pt.y)) : lo(p2.y), u1 ? (ra1 ? hi(pr.y) : hi(pt.y)) : hi(p2.y)),
                  mk2(u0 ? (ra0 ? lo(pr.z) : lo(pt.z)) : lo(p2.z), u1 ? (ra1 ? hi(pr.z) : hi(pt.z)) : hi(p2.z))};
            q2 = {mk2(u0 && ra0 ? lo(qrr.w) : lo(q2.w), u1 && ra1 ? hi(qrr.w) : hi(q2.w)),
                  mk2(u0 && ra0 ? lo(qrr.x) : lo(q2.x), u1 && ra1 ? hi(qrr.x) : hi(q2.x)),
                  mk2(u0 && ra0 ? lo(qrr.y) : lo(q2.y), u1 && ra1 ? hi(qrr.y) : hi(q2.y)),
                  mk2(u0 && ra0 ? lo(qrr.z) : lo(q2.z), u1 && ra1 ? hi(qrr.z) : hi(q2.z))};
        }
        const V rh = tp - p2;
        const f2 ep_h = sqrt2(dot(rh, rh));
        const f2 qv2 = fma2(q2.z, q2.z, fma2(q2.y, q2.y, q2.x * q2.x));
        const f2 eo_h = bc2(2.f) * mk2(fast_atan2f(sqrt_approx(lo(qv2)), fabsf(lo(q2.w))),
                                       fast_atan2f(sqrt_approx(hi(qv2)), fabsf(hi(q2.w))));
        // ---- Alg. 3 l.11-13 (R10): accept on an improvement > gamma in either space
        bool acc[2];
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            acc[s] = (lane(ep2, s) - lane(ep_h, s)) > c.gamma || (lane(eo2, s) - lane(eo_h, s)) > c.gamma;
            if (trace.words && act[s]) {   // decision word: see hjcd_poccd_trace (include/hjcd.h)
                const float dpv = dpb[s], dov = dob[s];
                trace.words[((long long)t * M + m0 + s) * c.ccd_iters + k] =
                    (uint32_t)jp[s] | ((uint32_t)jo[s] << 5) | ((jp[s] == jo[s] && db[s] != dpv) ? 1u << 10 : 0u) |
                    (acc[s] ? 1u << 11 : 0u) | ((dpv > 0.f ? 1u : dpv < 0.f ? 2u : 0u) << 12) |
                    ((dov > 0.f ? 1u : dov < 0.f ? 2u : 0u) << 14);
            }
        }
        // accepted: theta + d_eff re-clamped (R7); rejected: theta + N(0, sigma^2) (R11)
#pragma unroll
        for (int j = 0; j < NMAX; ++j) {
            if (EXACT || j < n) {
                const float d0 = j == jb[0] ? db[0] : (j == ja[0] ? da[0] : 0.f);
                const float d1 = j == jb[1] ? db[1] : (j == ja[1] ? da[1] : 0.f);
                const f2 nt2 = clamp2(th[j] + mk2(d0, d1), rb.j[j].lo, rb.j[j].hi);
                th[j] = mk2(acc[0] ? lo(nt2) : lo(th[j]), acc[1] ? hi(nt2) : hi(th[j]));
            }
        }
        // K12-style warp-cooperative draws: ~11 % of seeds reject per
        // iteration, so nearly every warp has a rejecting seed in each slot;
        // instead of every lane drawing its two seeds' blocks, the warp
        // spreads the (seed, Philox block) items of its rejecting seeds over
        // its lanes and leaves each block's 4 normals in the owner's (now
        // dead) frame slots; each rejecting seed then applies its own, exactly
        // as perturb() would (the same bits)
        {
            const int lane_id = (int)(threadIdx.x & 31);
            const unsigned rej0 = __ballot_sync(0xffffffffu, act[0] && !acc[0]);
            const unsigned rej1 = __ballot_sync(0xffffffffu, act[1] && !acc[1]);
            if (rej0 | rej1) {
                constexpr int NB = (NMAX + 3) / 4;
                const int nb = EXACT ? NB : (n + 3) / 4;
                const int n0 = __popc(rej0) * nb;
                const int items = n0 + __popc(rej1) * nb;
                for (int it = lane_id; it < items; it += 32) {
                    const int sl = it < n0 ? 0 : 1;
                    const int q = it < n0 ? it : it - n0;
                    const int r = q / nb, blk = q - r * nb;
                    const int ol = (int)__fns(sl ? rej1 : rej0, 0u, r + 1);
                    float g[4];
                    normals4<true>(draw(c, tid, (uint32_t)(m0 + 2 * (ol - lane_id) + sl), P_PERTURB, (uint32_t)k,
                                        (uint32_t)blk), g);
                    s_fr[(2 * blk + sl) * FR + (threadIdx.x - lane_id + ol)] = make_float4(g[0], g[1], g[2], g[3]);
                }
                __syncwarp();
#pragma unroll
                for (int sl = 0; sl < 2; ++sl) {
                    if (act[sl] && !acc[sl]) {
#pragma unroll
                        for (int blk = 0; blk < NB; ++blk) {
                            if (EXACT || 4 * blk < n) {
                                const float4 g4 = s_fr[(2 * blk + sl) * FR + threadIdx.x];
                                const float g[4] = {g4.x, g4.y, g4.z, g4.w};
#pragma unroll
                                for (int e = 0; e < 4; ++e) {
                                    const int j = 4 * blk + e;
                                    if (j < NMAX && (EXACT || j < n)) {
                                        const float v = clampf(lane(th[j], sl) + c.sigma_ccd * g[e], rb.j[j].lo,
                                                               rb.j[j].hi);
                                        th[j] = sl ? mk2(lo(th[j]), v) : mk2(v, hi(th[j]));
                                    }
                                }
                            }
                        }
                    }
                }
                __syncwarp();   // the slots are the next FK's frames
            }
        }
    }

#pragma unroll
    for (int s = 0; s < 2; ++s) {
        if (act[s]) {
            const int m = m0 + s;
#pragma unroll
            for (int j = 0; j < NMAX; ++j)
                if (EXACT || j < n) theta_out[((long long)t * n + j) * M + m] = lane(th[j], s);
            const long long o = (long long)t * M + m;
            const float ep = lane(ep2, s), eo = lane(eo2, s);
            cost_out[o] = c.w_p * c.w_p * ep * ep + c.w_o * c.w_o * eo * eo;   // R14
            if (ep_out) ep_out[o] = ep;
            if (eo_out) eo_out[o] = eo;
            if (iters_out) iters_out[o] = k;
        }
    }
    if (ready) {   // DESIGN K10: this CTA's seeds of target t are in memory
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0 && atomicAdd(ready + t, 1u) + 1u == (uint32_t)CL)
            ready_push(ready, T, t, k);   // DESIGN K26: the cluster's last CTA queues the target
    }
}

template <int NMAX, bool EXACT, int REV>
static cudaError_t launch_poccd_x2_r(const DevRobot& rb, const DevCfg& c, const float* targets, int T, float* theta,
                                     float* cost, float* ep, float* eo, int32_t* iters, TraceOut trace,
                                     uint32_t* ready, cudaStream_t s) {
    int nt, CL;
    texit_shape_x2(c.M, nt, CL);
    if (CL > 16) return cudaErrorInvalidConfiguration;
    const size_t smem = (size_t)NMAX * 3 * px::FR * sizeof(float4);
    static std::atomic<unsigned long long> attr{0};
    cudaError_t e = once_per_device(attr, [] {
        cudaError_t e2 = cudaFuncSetAttribute(k_poccd_x2<NMAX, EXACT, REV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)((size_t)NMAX * 3 * px::FR * sizeof(float4)));
        if (e2 == cudaSuccess)
            e2 = cudaFuncSetAttribute(k_poccd_x2<NMAX, EXACT, REV>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        return e2;
    });
    if (e != cudaSuccess) return e;
    const long long grid = (long long)T * CL;
    if (grid > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid, 1, 1);
    cfg.blockDim = dim3(nt, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr1[2];
    attr1[0].id = cudaLaunchAttributeClusterDimension;
    attr1[0].val.clusterDim.x = CL;
    attr1[0].val.clusterDim.y = 1;
    attr1[0].val.clusterDim.z = 1;
    // A/B (K42): the cluster scheduling policy (0 default, 1 spread, 2 load
    // balancing); the default suits the dependent launch here (load balancing:
    // PO-CCD alone -1 to -3 %, the C3 step +8 %)
    static const int policy = [] {
        const char* v = std::getenv("HJCD_X2_CLUSTER_POLICY");
        return v ? std::atoi(v) : 0;
    }();
    attr1[1].id = cudaLaunchAttributeClusterSchedulingPolicyPreference;
    attr1[1].val.clusterSchedulingPolicyPreference = (cudaClusterSchedulingPolicy)policy;
    cfg.attrs = attr1;
    cfg.numAttrs = policy ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, k_poccd_x2<NMAX, EXACT, REV>, rb, c, targets, T, theta, cost, ep, eo, iters, CL,
                              trace, ready);
}

template <int NMAX, bool EXACT>
cudaError_t launch_poccd_x2_t(const DevRobot& rb, const DevCfg& c, const float* targets, int T, float* theta,
                              float* cost, float* ep, float* eo, int32_t* iters, TraceOut trace, uint32_t* ready,
                              cudaStream_t s) {
    if (rb.pmask == 0u && rb.rx)
        return launch_poccd_x2_r<NMAX, EXACT, 2>(rb, c, targets, T, theta, cost, ep, eo, iters, trace, ready, s);
    if (rb.pmask == 0u)
        return launch_poccd_x2_r<NMAX, EXACT, 1>(rb, c, targets, T, theta, cost, ep, eo, iters, trace, ready, s);
    return launch_poccd_x2_r<NMAX, EXACT, 0>(rb, c, targets, T, theta, cost, ep, eo, iters, trace, ready, s);
}

}  // namespace hjcd

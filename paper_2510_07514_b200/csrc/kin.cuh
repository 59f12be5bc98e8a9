// kin.cuh — device kinematics, quaternion algebra and Philox for the HJCD-IK
// kernels (fp32, registers only).  "P:NNN" cites PAPER.md lines.
//
// All per-joint loops are `#pragma unroll` over the compile-time bound NMAX
// with a uniform `j < rb.n` guard, so per-joint arrays stay in registers (no
// dynamic indexing) and robot constants are constant-bank operands.
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>

#include "hjcd_internal.h"
#include "pk2.cuh"

namespace hjcd {

// ---------------------------------------------------------------- precision
// The polish stage runs in fp32 (the default) or fp64 (hjcd_solve_f64, SURVEY
// §8(f) f1); everything it uses is templated on the scalar R.  vec3<R> is
// float3 / double3; the float forms are the ones the fp32 kernels always used.
template <class R> struct VecT;
template <> struct VecT<float> { using type = float3; };
template <> struct VecT<double> { using type = double3; };
template <class R> using vec3 = typename VecT<R>::type;

template <class R>
struct QuatT {
    R w, x, y, z;
};
using Quat = QuatT<float>;

__device__ __forceinline__ float3 f3(float x, float y, float z) { return make_float3(x, y, z); }
__device__ __forceinline__ double3 f3(double x, double y, double z) { return make_double3(x, y, z); }
template <class R>
__device__ __forceinline__ vec3<R> mk3(R x, R y, R z) { return f3(x, y, z); }
__device__ __forceinline__ float3 operator+(float3 a, float3 b) { return f3(a.x + b.x, a.y + b.y, a.z + b.z); }
__device__ __forceinline__ float3 operator-(float3 a, float3 b) { return f3(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ float3 operator*(float s, float3 a) { return f3(s * a.x, s * a.y, s * a.z); }
__device__ __forceinline__ float dot3(float3 a, float3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ float3 cross3(float3 a, float3 b) {
    return f3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double3 operator+(double3 a, double3 b) { return f3(a.x + b.x, a.y + b.y, a.z + b.z); }
__device__ __forceinline__ double3 operator-(double3 a, double3 b) { return f3(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ double3 operator*(double s, double3 a) { return f3(s * a.x, s * a.y, s * a.z); }
__device__ __forceinline__ double dot3(double3 a, double3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ double3 cross3(double3 a, double3 b) {
    return f3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ float clampf(float x, float lo, float hi) { return fminf(fmaxf(x, lo), hi); }
__device__ __forceinline__ double clampf(double x, double lo, double hi) { return fmin(fmax(x, lo), hi); }

// Hamilton product a (x) conj(b)
template <class R>
__device__ __forceinline__ QuatT<R> qmul_conj(QuatT<R> a, QuatT<R> b) {
    QuatT<R> r;
    r.w = a.w * b.w + a.x * b.x + a.y * b.y + a.z * b.z;
    r.x = -a.w * b.x + a.x * b.w - a.y * b.z + a.z * b.y;
    r.y = -a.w * b.y + a.x * b.z + a.y * b.w - a.z * b.x;
    r.z = -a.w * b.z - a.x * b.y + a.y * b.x + a.z * b.w;
    return r;
}

// q_err = q_t (x) q_e^-1, canonicalised to w >= 0 (Eq. 5; reading R1)
template <class R>
__device__ __forceinline__ QuatT<R> quat_err(QuatT<R> qt, QuatT<R> qe) {
    QuatT<R> q = qmul_conj(qt, qe);
    if (q.w < R(0)) { q.w = -q.w; q.x = -q.x; q.y = -q.y; q.z = -q.z; }
    return q;
}

// |omega| = 2 atan2(|v|, w) for canonical q (Eq. 5: |omega| of
// 2 atan2(|v|,|w|)/|v| * v).  Exact at v = 0.
__device__ __forceinline__ float omega_norm(float sv, float w) { return 2.f * atan2f(sv, fabsf(w)); }

// q_err (x) q(z, -d): the error after rotating the end effector about the
// world axis z by d (q_e' = q(z, d) (x) q_e).  Inputs c2, s2 = cos, sin(d/2).
__device__ __forceinline__ Quat qerr_rotate(Quat q, float3 z, float c2, float s2) {
    Quat r;
    float vz = q.x * z.x + q.y * z.y + q.z * z.z;
    // v x z
    float cx = q.y * z.z - q.z * z.y, cy = q.z * z.x - q.x * z.z, cz = q.x * z.y - q.y * z.x;
    r.w = q.w * c2 + vz * s2;
    r.x = c2 * q.x - s2 * q.w * z.x - s2 * cx;
    r.y = c2 * q.y - s2 * q.w * z.y - s2 * cy;
    r.z = c2 * q.z - s2 * q.w * z.z - s2 * cz;
    return r;
}

// rotation matrix (row-major) -> unit quaternion, w >= 0 (Shepperd), without
// branches: the four pivots 4q_i^2 = t_i are formed, the largest is chosen by
// selects, and q = (column of the symmetric 4x4 form) * rsqrt(t)/2.  Seeds of
// a warp sit in different quadrants, so the branchy form diverges 4 ways.
__device__ __forceinline__ float rsqrt_q(float x) { return rsqrtf(x); }
__device__ __forceinline__ double rsqrt_q(double x) { return 1.0 / sqrt(x); }

template <class T>
__device__ __forceinline__ QuatT<T> quat_from_rot(const T R[9]) {
    const T one = T(1);
    const T t0 = one + R[0] + R[4] + R[8];   // 4 w^2
    const T t1 = one + R[0] - R[4] - R[8];   // 4 x^2
    const T t2 = one - R[0] + R[4] - R[8];   // 4 y^2
    const T t3 = one - R[0] - R[4] + R[8];   // 4 z^2
    const T a = R[7] - R[5], b = R[2] - R[6], cc = R[3] - R[1];   // 4wx, 4wy, 4wz
    const T d = R[1] + R[3], e = R[2] + R[6], f = R[5] + R[7];    // 4xy, 4xz, 4yz
    // same branch order as the classic form: w if tr > 0, else the largest diagonal
    const bool pw = (R[0] + R[4] + R[8]) > T(0);
    const bool px = !pw && R[0] > R[4] && R[0] > R[8];
    const bool py = !pw && !px && R[4] > R[8];
    T t, qw, qx, qy, qz;   // the pivot's column, scaled by 4 q_pivot
    if (pw) { t = t0; qw = t0; qx = a; qy = b; qz = cc; }
    else if (px) { t = t1; qw = a; qx = t1; qy = d; qz = e; }
    else if (py) { t = t2; qw = b; qx = d; qy = t2; qz = f; }
    else { t = t3; qw = cc; qx = e; qy = f; qz = t3; }
    const T is = T(0.5) * rsqrt_q(t);
    QuatT<T> q;
    q.w = qw * is; q.x = qx * is; q.y = qy * is; q.z = qz * is;
    // renormalise (absorbs the rsqrt approximation and FK rounding)
    T inv = rsqrt_q(q.w * q.w + q.x * q.x + q.y * q.y + q.z * q.z);
    if (q.w < T(0)) inv = -inv;
    q.w *= inv; q.x *= inv; q.y *= inv; q.z *= inv;
    return q;
}

// sin and cos of a joint angle (fp32, |err| <= 7.1e-8 on |x| <= 1e4; joint
// angles are always clamped to their limits, which hjcd_robot_create bounds):
// Cody-Waite reduction by pi/2 in two FMA steps, then the cephes sinf/cosf
// minimax polynomials on [-pi/4, pi/4].  Branch-free and short: the library
// sincosf carries a Payne-Hanek slow path (local memory, ~200 instructions)
// per call site, which bloats the polish kernels' code (i-cache misses).
__device__ __forceinline__ void sincos_b(float x, float* s, float* c) {
    const float q = rintf(x * 0.636619772367581343f);
    float r = fmaf(-q, 1.5707963705062866f, x);
    r = fmaf(-q, -4.37113900018624283e-8f, r);
    const float z = r * r;
    const float ps = fmaf(fmaf(fmaf(-1.9515295891e-4f, z, 8.3321608736e-3f), z, -1.6666654611e-1f), z * r, r);
    const float pc = fmaf(fmaf(fmaf(fmaf(2.443315711809948e-5f, z, -1.388731625493765e-3f), z,
                                    4.166664568298827e-2f), z, -0.5f), z, 1.0f);
    const int qi = (int)q;
    const float sa = (qi & 1) ? pc : ps;
    const float ca = (qi & 1) ? ps : pc;
    *s = (qi & 2) ? -sa : sa;
    *c = ((qi + 1) & 2) ? -ca : ca;
}
__device__ __forceinline__ void sincos_b(double x, double* s, double* c) { sincos(x, s, c); }

// K14: fk() for REV = 2 in fp32 with the rotation held as packed column pairs
// (rows 0-1 of each column in one f2, row 2 scalar) and (tx, ty) packed, so
// every column update a*col + b*col' is one FMUL2 + one FFMA2 for rows 0-1
// plus the scalar row 2: 22 instead of 33 issue slots per joint.  Same
// operations per element as the scalar form below; outputs unpacked for free.
template <int NMAX, bool FRAMES, bool EXACT, bool FAST, class A>
__device__ __forceinline__ void fk_rx2(const DevRobotT<float>& rb, const A& th, float3 (&P)[NMAX],
                                       float3 (&Z)[NMAX], float3& pe, Quat& qe) {
    f2 C0 = mk2(1.f, 0.f), C1 = mk2(0.f, 1.f), C2 = mk2(0.f, 0.f);   // R[0,3], R[1,4], R[2,5]
    float r6 = 0.f, r7 = 0.f, r8 = 1.f;                              // R[6], R[7], R[8]
    f2 t01 = mk2(0.f, 0.f);
    float tz = 0.f;
#pragma unroll
    for (int j = 0; j < NMAX; ++j) {
        if (EXACT || j < rb.n) {
            const DevJointT<float>& J = rb.j[j];
            t01 = add2(t01, fma2(C2, bc2(J.t[2]), fma2(C1, bc2(J.t[1]), mul2(C0, bc2(J.t[0])))));
            tz += r6 * J.t[0] + r7 * J.t[1] + r8 * J.t[2];
            // N = R F_j with F_j.R = Rx(alpha): column 0 unchanged
            const f2 N1 = fma2(C2, bc2(J.R[7]), mul2(C1, bc2(J.R[4])));
            const f2 N2 = fma2(C2, bc2(J.R[8]), mul2(C1, bc2(J.R[5])));
            const float n7 = r7 * J.R[4] + r8 * J.R[7];
            const float n8 = r7 * J.R[5] + r8 * J.R[8];
            if (FRAMES) {
                float x, y;
                unpk2(t01, x, y);
                P[j] = make_float3(x, y, tz);
                unpk2(N2, x, y);
                Z[j] = make_float3(x, y, n8);
            }
            float s, c;
            if constexpr (FAST) __sincosf(th[j], &s, &c);
            else sincos_b(th[j], &s, &c);
            // R = N Rz(theta): col0 = c N0 + s N1, col1 = c N1 - s N0
            const f2 C0n = fma2(bc2(s), N1, mul2(bc2(c), C0));
            C1 = fma2(bc2(-s), C0, mul2(bc2(c), N1));
            C0 = C0n;
            C2 = N2;
            const float r6n = c * r6 + s * n7;
            r7 = c * n7 - s * r6;
            r6 = r6n;
            r8 = n8;
        }
    }
    float e[2];
    f2 te = fma2(C2, bc2(rb.eet[2]), fma2(C1, bc2(rb.eet[1]), mul2(C0, bc2(rb.eet[0]))));
    te = add2(t01, te);
    unpk2(te, e[0], e[1]);
    const float tzz = tz + (r6 * rb.eet[0] + r7 * rb.eet[1] + r8 * rb.eet[2]);
    float E[9];
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) {
        const f2 col = fma2(C2, bc2(rb.eeR[6 + cc]), fma2(C1, bc2(rb.eeR[3 + cc]), mul2(C0, bc2(rb.eeR[cc]))));
        unpk2(col, E[cc], E[3 + cc]);
        E[6 + cc] = r6 * rb.eeR[cc] + r7 * rb.eeR[3 + cc] + r8 * rb.eeR[6 + cc];
    }
    pe = make_float3(e[0], e[1], tzz);
    qe = quat_from_rot(E);
}

// Forward kinematics (Eq. 1) with frames (Eq. 7 inputs):
// T = F_1 Rz(th_1) F_2 Rz(th_2) ... F_n Rz(th_n) EE  (prismatic: Tz).
// FRAMES: P[j] = joint origin, Z[j] = joint axis (world), before joint motion
// (identical after it: rotation about z fixes the axis and the origin).
// EXACT: the chain has exactly NMAX DoF (no per-joint guard).  FAST: joint
// sincos on the SFU (__sincosf, |err| <~ 5e-7 rad on the joint ranges): used by
// the coarse stage only (K5); the polish stage uses sincos_b.
// REV: 1 = every DoF joint is revolute (no per-joint type branch); 2 = also
// every F_j rotation is Rx(alpha_j) (rb.rx, DESIGN K11): the rotation product
// skips the structural zeros (12 instead of 27 multiply-adds per joint) with
// the same operation order on the non-zero terms, i.e. the same bits.
// th: a T[NMAX] array, or any type whose th[j] yields joint j's value (a trial
// point computed joint by joint, polish.cuh TrialTheta)
template <int NMAX, bool FRAMES, bool EXACT = false, bool FAST = false, int REV = 0, class T, class A>
__device__ __forceinline__ void fk(const DevRobotT<T>& rb, const A& th, vec3<T> (&P)[NMAX],
                                   vec3<T> (&Z)[NMAX], vec3<T>& pe, QuatT<T>& qe) {
    if constexpr (REV == 2 && sizeof(T) == 4 && NMAX <= 8) {   // (more spills above 8 DoF)
#ifndef HJCD_NO_K14
        fk_rx2<NMAX, FRAMES, EXACT, FAST>(rb, th, P, Z, pe, qe);
        return;
#endif
    }
    T R[9] = {T(1), T(0), T(0), T(0), T(1), T(0), T(0), T(0), T(1)};
    T tx = T(0), ty = T(0), tz = T(0);
#pragma unroll
    for (int j = 0; j < NMAX; ++j) {
        if (EXACT || j < rb.n) {
            const DevJointT<T>& J = rb.j[j];
            tx += R[0] * J.t[0] + R[1] * J.t[1] + R[2] * J.t[2];
            ty += R[3] * J.t[0] + R[4] * J.t[1] + R[5] * J.t[2];
            tz += R[6] * J.t[0] + R[7] * J.t[1] + R[8] * J.t[2];
            T N[9];
            if constexpr (REV == 2) {
#pragma unroll
                for (int r = 0; r < 3; ++r) {
                    N[3 * r] = R[3 * r];
                    N[3 * r + 1] = R[3 * r + 1] * J.R[4] + R[3 * r + 2] * J.R[7];
                    N[3 * r + 2] = R[3 * r + 1] * J.R[5] + R[3 * r + 2] * J.R[8];
                }
            } else {
#pragma unroll
                for (int r = 0; r < 3; ++r)
#pragma unroll
                    for (int cc = 0; cc < 3; ++cc)
                        N[3 * r + cc] = R[3 * r] * J.R[cc] + R[3 * r + 1] * J.R[3 + cc] + R[3 * r + 2] * J.R[6 + cc];
            }
            if (FRAMES) {
                P[j] = mk3<T>(tx, ty, tz);
                Z[j] = mk3<T>(N[2], N[5], N[8]);
            }
            if (REV || J.type == HJCD_REVOLUTE) {
                T s, c;
                if constexpr (FAST) __sincosf(th[j], &s, &c);
                else sincos_b(th[j], &s, &c);
#pragma unroll
                for (int r = 0; r < 3; ++r) {
                    T a = N[3 * r], b = N[3 * r + 1];
                    R[3 * r] = c * a + s * b;
                    R[3 * r + 1] = c * b - s * a;
                    R[3 * r + 2] = N[3 * r + 2];
                }
            } else {
#pragma unroll
                for (int i = 0; i < 9; ++i) R[i] = N[i];
                tx += th[j] * N[2];
                ty += th[j] * N[5];
                tz += th[j] * N[8];
            }
        }
    }
    tx += R[0] * rb.eet[0] + R[1] * rb.eet[1] + R[2] * rb.eet[2];
    ty += R[3] * rb.eet[0] + R[4] * rb.eet[1] + R[5] * rb.eet[2];
    tz += R[6] * rb.eet[0] + R[7] * rb.eet[1] + R[8] * rb.eet[2];
    T E[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int cc = 0; cc < 3; ++cc)
            E[3 * r + cc] = R[3 * r] * rb.eeR[cc] + R[3 * r + 1] * rb.eeR[3 + cc] + R[3 * r + 2] * rb.eeR[6 + cc];
    pe = mk3<T>(tx, ty, tz);
    qe = quat_from_rot(E);
}

// 1/x for normal positive x without the IEEE-division slow path: MUFU.RCP
// approximation + one Newton step (|rel err| <~ 1.5 ulp)
__device__ __forceinline__ float rcp_nr(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return fmaf(r, fmaf(-x, r, 1.f), r);
}

// 1/sqrt(x) for normal positive x: MUFU.RSQ + one Newton step
__device__ __forceinline__ float rsqrt_nr(float x) {
    const float r = rsqrtf(x);
    return r * fmaf(-0.5f * x * r, r, 1.5f);
}

// 1/x from the SFU alone (rcp.approx.ftz, ~1 ulp), for ratios whose rounding
// the caller's own error budget dominates
__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// sqrt from the SFU alone (MUFU.SQRT, ~1 ulp, sqrt(0) = 0): residual norms,
// where the IEEE sqrtf's range checks and slow path only cost issue slots
__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// atan2 on [-pi, pi] with |err| <= 3.3e-7 rad (fp32): odd minimax polynomial
// of degree 15 for atan on [0, 1] + octant reduction (K5); the
// ratio min/max by one SFU reciprocal (no __fdividef range fix-ups; a
// subnormal max gives NaN, which every caller masks or never produces)
__device__ __forceinline__ float fast_atan2f(float y, float x) {
    const float ax = fabsf(x), ay = fabsf(y);
    const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
    const float r = mx > 0.f ? mn * rcp_approx(mx) : 0.f;
    const float s = r * r;
    float p = -0.00405456f;
    p = fmaf(p, s, 0.02186293f);
    p = fmaf(p, s, -0.05591229f);
    p = fmaf(p, s, 0.09642195f);
    p = fmaf(p, s, -0.13908629f);
    p = fmaf(p, s, 0.19946566f);
    p = fmaf(p, s, -0.3332986f);
    p = fmaf(p, s, 0.99999934f);
    float a = p * r;
    a = (ay > ax) ? 1.57079637f - a : a;
    a = (x < 0.f) ? 3.14159274f - a : a;
    return copysignf(a, y);
}

// ---------------------------------------------------------------- targets
template <class R>
struct TargetT {
    vec3<R> p;
    QuatT<R> q;
    bool valid;
};
using Target = TargetT<float>;

// S2: normalise q when | |q| - 1 | <= 1e-3 (tested in fp32 at either precision),
// else invalid (status 3 later).  The fp32 target is widened exactly.
template <class R = float>
__device__ __forceinline__ TargetT<R> load_target(const float* __restrict__ t7) {
    TargetT<R> t;
    const float px = __ldg(t7 + 0), py = __ldg(t7 + 1), pz = __ldg(t7 + 2);
    const float w32 = __ldg(t7 + 3), x32 = __ldg(t7 + 4), y32 = __ldg(t7 + 5), z32 = __ldg(t7 + 6);
    const float nq32 = sqrtf(w32 * w32 + x32 * x32 + y32 * y32 + z32 * z32);
    t.valid = fabsf(nq32 - 1.f) <= 1e-3f && isfinite(nq32) && isfinite(px) && isfinite(py) && isfinite(pz);
    R w = w32, x = x32, y = y32, z = z32;
    R nq = sqrt(w * w + x * x + y * y + z * z);
    t.p = mk3<R>(px, py, pz);
    if (!t.valid) { w = R(1); x = y = z = R(0); nq = R(1); t.p = mk3<R>(R(0), R(0), R(0)); }
    R inv = R(1) / nq;
    if (w < R(0)) inv = -inv;
    t.q.w = w * inv; t.q.x = x * inv; t.q.y = y * inv; t.q.z = z * inv;
    return t;
}

// ---------------------------------------------------------------- Philox4x32-10 (R30)
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    }
    return c;
}

__device__ __forceinline__ uint4 draw(const DevCfg& c, uint32_t tid, uint32_t sid, uint32_t purpose,
                                      uint32_t iter, uint32_t blk) {
    return philox4x32_10(make_uint4(tid, sid, (purpose << 24) | (iter & 0xFFFFFFu), blk), c.key0, c.key1);
}

// ((x >> 9) + 0.5) * 2^-23: exact in fp32, in (0, 1)
__device__ __forceinline__ float u01(uint32_t x) { return ((float)(x >> 9) + 0.5f) * 1.1920928955078125e-07f; }

// 4 standard normals from one Philox block: Box-Muller on (u0,u1), (u2,u3).
// FAST (coarse stage): SFU log2 / sincos (|rel err| ~1e-6 on each normal,
// i.e. ~5e-8 rad on a sigma = 0.05 perturbation, far below the coarse
// tolerance); otherwise the accurate library functions.
template <bool FAST = false>
__device__ __forceinline__ void normals4(uint4 r, float g[4]) {
    float u0 = u01(r.x), u1 = u01(r.y), u2 = u01(r.z), u3 = u01(r.w);
    if (FAST) {
        const float ra = sqrt_approx(-1.38629436f * __log2f(u0)), rb2 = sqrt_approx(-1.38629436f * __log2f(u2));
        float s, c;   // sin/cos(2 pi u - pi) = -sin/-cos(2 pi u), argument in (-pi, pi)
        __sincosf(fmaf(6.28318531f, u1, -3.14159265f), &s, &c);
        g[0] = -ra * c; g[1] = -ra * s;
        __sincosf(fmaf(6.28318531f, u3, -3.14159265f), &s, &c);
        g[2] = -rb2 * c; g[3] = -rb2 * s;
    } else {
        float ra = sqrtf(-2.f * logf(u0)), rb2 = sqrtf(-2.f * logf(u2));
        float s, c;
        sincospif(2.f * u1, &s, &c);
        g[0] = ra * c; g[1] = ra * s;
        sincospif(2.f * u3, &s, &c);
        g[2] = rb2 * c; g[3] = rb2 * s;
    }
}

// fp64 polish: the same Box-Muller in fp64 (as the oracle draws them)
__device__ __forceinline__ void normals4(uint4 r, double g[4]) {
    const double s23 = 1.1920928955078125e-07;
    const double u0 = ((double)(r.x >> 9) + 0.5) * s23, u1 = ((double)(r.y >> 9) + 0.5) * s23;
    const double u2 = ((double)(r.z >> 9) + 0.5) * s23, u3 = ((double)(r.w >> 9) + 0.5) * s23;
    const double ra = sqrt(-2.0 * log(u0)), rb2 = sqrt(-2.0 * log(u2));
    double s, c;
    sincospi(2.0 * u1, &s, &c);
    g[0] = ra * c; g[1] = ra * s;
    sincospi(2.0 * u3, &s, &c);
    g[2] = rb2 * c; g[3] = rb2 * s;
}

// theta <- clamp(theta + sigma * N(0, I)), stream (tid, sid, purpose, iter)
template <int NMAX, bool EXACT = false, bool FAST = false, class T>
__device__ __forceinline__ void perturb(const DevRobotT<T>& rb, const DevCfg& c, T (&th)[NMAX], T sigma,
                                        uint32_t tid, uint32_t sid, uint32_t purpose, uint32_t iter) {
#pragma unroll
    for (int blk = 0; blk < (NMAX + 3) / 4; ++blk) {
        if (EXACT || 4 * blk < rb.n) {
            T g[4];
            if constexpr (sizeof(T) == 4) normals4<FAST>(draw(c, tid, sid, purpose, iter, blk), g);
            else normals4(draw(c, tid, sid, purpose, iter, blk), g);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                int j = 4 * blk + e;
                if (j < NMAX && (EXACT || j < rb.n)) th[j] = clampf(th[j] + sigma * g[e], rb.j[j].lo, rb.j[j].hi);
            }
        }
    }
}

// ---- Alg. 2 l.2-8: top-K + replicate, shared by k_select_replicate and the
// PJ-IK prologue of hjcd_solve's dependent launch (DESIGN K10)

// non-negative float -> order-preserving uint32 (NaN and negatives -> +inf)
__device__ __forceinline__ uint32_t cost_bits(float x) {
    if (!(x >= 0.f)) x = CUDART_INF_F;
    return __float_as_uint(x);
}

// The M stage-1 costs of one target as 64-bit keys (cost bits << 32 | seed
// index), bitonic-sorted ascending in shared memory by the whole CTA (Mpad =
// M rounded up to a power of two >= 2): keys[r] is the r-th of the K rounds
// of argmin-and-remove of Alg. 2 (R14; ties -> lower index).  The costs are
// read through L2 (ld.global.cg), never a possibly stale L1 line: in
// hjcd_solve they were written by a PO-CCD kernel that may still be running.
__device__ __forceinline__ void sort_stage1_keys(const float* cost_t, int M, int Mpad, unsigned long long* keys) {
    for (int i = threadIdx.x; i < Mpad; i += blockDim.x)
        keys[i] = (i < M) ? (((unsigned long long)cost_bits(__ldcg(cost_t + i)) << 32) | (unsigned)i) : ~0ull;
    __syncthreads();
    for (int size = 2; size <= Mpad; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < (Mpad >> 1); i += blockDim.x) {
                const int lo = 2 * i - (i & (stride - 1));
                const int hi = lo + stride;
                const bool up = ((lo & size) == 0);
                const unsigned long long a = keys[lo], b = keys[hi];
                if ((a > b) == up) { keys[lo] = b; keys[hi] = a; }
            }
            __syncthreads();
        }
    }
}

// Alg. 2 l.7-8 (R15): joints 4 blk .. 4 blk + 3 (< n) of polish seed
// b < floor(B/K) K of target t: kept seed b mod K, copy b / K; copies > 0 (or
// every copy with repl_noise_all) get N(0, sigma_rep^2) from ONE Philox block
// (tid, b, REPL, 0, blk), clamped to the fp32 limits.  theta1 is stage 1's
// [T][n][M], read through L2.
template <class R>
__device__ __forceinline__ void replica_block(const R& rb, const DevCfg& c, const float* theta1,
                                              const unsigned long long* keys, int t, int b, int blk,
                                              uint32_t tid, float v[4]) {
    const int K = c.K, M = c.M, n = rb.n;
    const int rank = b % K, cp = b / K;
    const int src = (int)(keys[rank] & 0xffffffffu);
    float g[4] = {0.f, 0.f, 0.f, 0.f};
    const bool noisy = cp > 0 || c.repl_noise_all;
    if (noisy) normals4(draw(c, tid, (uint32_t)b, P_REPL, 0u, (uint32_t)blk), g);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int j = 4 * blk + e;
        if (j < n) {
            v[e] = __ldcg(theta1 + ((long long)t * n + j) * M + src);
            if (noisy) v[e] = clampf(__fmaf_rn(c.sigma_rep, g[e], v[e]), (float)rb.j[j].lo, (float)rb.j[j].hi);
        }
    }
}

}  // namespace hjcd

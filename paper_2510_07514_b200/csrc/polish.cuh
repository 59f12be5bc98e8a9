// polish.cuh — device pieces of PJ-IK (Alg. 4) used by the
// cooperative per-target kernel (pjik_coop.cuh): residual rho = -r, weighted
// cost, the 6x6 Cholesky, and the three step directions (LM via push-through
// K4, dogleg, single coordinate).  Templated on the scalar T: float for the
// default polish, double for the fp64 polish (hjcd_solve_f64, f1).  The float
// forms use the SFU reciprocals / polynomial atan2 (K5); the double forms the
// IEEE operations.
#pragma once
#include "kin.cuh"

namespace hjcd {

__device__ __forceinline__ double rcp_nr(double x) { return 1.0 / x; }
__device__ __forceinline__ double rsqrt_nr(double x) { return 1.0 / sqrt(x); }
__device__ __forceinline__ float atan2_r(float y, float x) { return fast_atan2f(y, x); }
__device__ __forceinline__ double atan2_r(double y, double x) { return atan2(y, x); }

// 6x6 SPD solve by Cholesky, packed lower triangle A[i*(i+1)/2 + j]; the
// pivots are kept as reciprocals (rsqrt + Newton in fp32), so the
// factorisation and both substitutions are multiply-only.  Returns false if a
// pivot is not positive.  NB (K21): no early exit -- the solve runs to the
// end on any input and the flag alone says whether b is valid, so the code
// is one straight-line block
template <class T, bool NB = false>
__device__ __forceinline__ bool chol6_solve(T (&A)[21], T (&b)[6]) {
    T id[6];
    bool ok = true;
#pragma unroll
    for (int i = 0; i < 6; ++i) {
#pragma unroll
        for (int j = 0; j <= i; ++j) {
            T s = A[i * (i + 1) / 2 + j];
#pragma unroll
            for (int k = 0; k < j; ++k) s -= A[i * (i + 1) / 2 + k] * A[j * (j + 1) / 2 + k];
            if (i == j) {
                if constexpr (NB) ok = ok && (s > T(1e-30));
                else if (!(s > T(1e-30))) return false;
                id[i] = rsqrt_nr(s);
                A[i * (i + 1) / 2 + i] = s * id[i];
            } else {
                A[i * (i + 1) / 2 + j] = s * id[j];
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        T s = b[i];
#pragma unroll
        for (int k = 0; k < i; ++k) s -= A[i * (i + 1) / 2 + k] * b[k];
        b[i] = s * id[i];
    }
#pragma unroll
    for (int i = 5; i >= 0; --i) {
        T s = b[i];
#pragma unroll
        for (int k = i + 1; k < 6; ++k) s -= A[k * (k + 1) / 2 + i] * b[k];
        b[i] = s * id[i];
    }
    return ok;
}

template <class V>
__device__ __forceinline__ auto jrow(const V& Jp, const V& Jo, int i) {
    return i == 0 ? Jp.x : i == 1 ? Jp.y : i == 2 ? Jp.z : i == 3 ? Jo.x : i == 4 ? Jo.y : Jo.z;
}

// rho = -r = [P_ee - P_t; -omega] (R19) and its norms
template <class T>
struct ResidT {
    T rho[6];
    T ep, eo;
};
using Resid = ResidT<float>;

template <class T>
__device__ __forceinline__ ResidT<T> residual(const TargetT<T>& tg, vec3<T> pe, QuatT<T> qe) {
    ResidT<T> r;
    const QuatT<T> q = quat_err(tg.q, qe);
    const T sv = sqrt(q.x * q.x + q.y * q.y + q.z * q.z);
    const T ang = T(2) * atan2_r(sv, q.w);                       // |omega| (Eq. 5), q.w >= 0
    const T scale = sv > T(1e-30) ? ang * rcp_nr(sv) : T(2) * rcp_nr(q.w);   // omega = scale * v
    r.rho[0] = pe.x - tg.p.x; r.rho[1] = pe.y - tg.p.y; r.rho[2] = pe.z - tg.p.z;
    r.rho[3] = -scale * q.x; r.rho[4] = -scale * q.y; r.rho[5] = -scale * q.z;
    r.ep = sqrt(r.rho[0] * r.rho[0] + r.rho[1] * r.rho[1] + r.rho[2] * r.rho[2]);
    r.eo = ang;
    return r;
}

template <class T>
__device__ __forceinline__ T cost_w(const T (&W)[6], const T (&rho)[6]) {
    T s = T(0);
#pragma unroll
    for (int i = 0; i < 6; ++i) s += (W[i] * rho[i]) * (W[i] * rho[i]);
    return T(0.5) * s;
}

// clamp(theta + alpha d) joint by joint, read from the per-seed records in
// shared memory (stride nt), so a line-search trial point is never
// materialised as a register array (K19: register pressure at high DoF)
template <class T>
struct TrialTheta {
    const DevRobotT<T>& rb;
    const T* th;   // &S.th[owner], stride nt
    const T* d;    // &S.dir[(kind * NMAX) * nt + owner], stride nt
    int nt;
    T alpha;
    __device__ __forceinline__ T operator[](int j) const {
        return clampf(th[j * nt] + alpha * d[j * nt], rb.j[j].lo, rb.j[j].hi);
    }
};

template <int NMAX, bool EXACT = false, int REV = 0, class T, class A>
__device__ __forceinline__ ResidT<T> eval_at(const DevRobotT<T>& rb, const TargetT<T>& tg, const A& th) {
    vec3<T> P[NMAX], Z[NMAX];   // unused (FRAMES = false), eliminated
    vec3<T> pe;
    QuatT<T> qe;
    fk<NMAX, false, EXACT, false, REV>(rb, th, P, Z, pe, qe);
    return residual(tg, pe, qe);
}

// ---- LM direction (Eq. 12 via push-through, K4): A = W G W + lambda I,
//      G_ik = sum_j J_ij J_kj / D_j; y = A^-1 W rho; dth_j = -(sum_i J_ij W_i y_i) / D_j,
//      then the element-wise trust-region clamp (Alg. 4 l.6, R21)
//      RECOMP (high DoF, K19): 1 / D_j recomputed from the column where it is
//      used instead of held in NMAX registers (invD is then not read)
template <int NMAX, bool EXACT = false, bool RECOMP = false, bool NB = false, class T>
__device__ __forceinline__ bool lm_direction(const DevRobotT<T>& rb, const DevCfg& c, const vec3<T> (&Jp)[NMAX],
                                             const vec3<T> (&Jo)[NMAX], const T (&invD)[NMAX],
                                             const T (&W)[6], const T (&rho)[6], T (&dth)[NMAX]) {
    const int n = rb.n;
    auto inv_d = [&](int j) {
        return RECOMP ? rcp_nr(fmax(dot3(Jp[j], Jp[j]) + dot3(Jo[j], Jo[j]), T(c.d_floor))) : invD[j];
    };
    // G = sum_j (J_j / D_j) J_j^T: scale each column once, then one FMA per term
    T A[21];
#pragma unroll
    for (int q = 0; q < 21; ++q) A[q] = T(0);
#pragma unroll
    for (int j = 0; j < NMAX; ++j) {
        if (EXACT || j < n) {
            const T col[6] = {Jp[j].x, Jp[j].y, Jp[j].z, Jo[j].x, Jo[j].y, Jo[j].z};
            const T id = inv_d(j);
#pragma unroll
            for (int i = 0; i < 6; ++i) {
                const T ui = col[i] * id;
#pragma unroll
                for (int kk = 0; kk <= i; ++kk) A[i * (i + 1) / 2 + kk] += ui * col[kk];
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int kk = 0; kk <= i; ++kk)
            A[i * (i + 1) / 2 + kk] = W[i] * W[kk] * A[i * (i + 1) / 2 + kk] + (i == kk ? T(c.lambda) : T(0));
    T y[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) y[i] = W[i] * rho[i];
    bool ok = true;
    if constexpr (NB) ok = chol6_solve<T, true>(A, y);
    else if (!chol6_solve(A, y)) return false;
#pragma unroll
    for (int i = 0; i < 6; ++i) y[i] *= W[i];
    const T Rt = T(c.R);
#pragma unroll
    for (int j = 0; j < NMAX; ++j) {
        if (EXACT || j < n) {
            const T s = Jp[j].x * y[0] + Jp[j].y * y[1] + Jp[j].z * y[2] + Jo[j].x * y[3] +
                        Jo[j].y * y[4] + Jo[j].z * y[5];
            dth[j] = clampf(-s * inv_d(j), -Rt, Rt);
        }
    }
    return ok;
}

// ---- dogleg direction (Eqs. 14-15, R23): GD = -alpha_c J^T rho (Cauchy),
//      GN = -J^T (J J^T + d_floor I)^-1 rho, smallest tau in [0,1] with |dth(tau)| <= R
//      NB (K21, fp32): branch-free -- the degenerate cases are a flag, the
//      divisions and square roots are SFU reciprocals / rsqrt + Newton
template <int NMAX, bool EXACT = false, bool NB = false, class T>
__device__ __forceinline__ bool dogleg_direction(const DevRobotT<T>& rb, const DevCfg& c, const vec3<T> (&Jp)[NMAX],
                                                 const vec3<T> (&Jo)[NMAX], const T (&rho)[6],
                                                 T (&dth)[NMAX], T (&gn)[NMAX]) {
    const int n = rb.n;
    T gg = T(0);
#pragma unroll
    for (int j = 0; j < NMAX; ++j) {
        if (EXACT || j < n) {
            dth[j] = Jp[j].x * rho[0] + Jp[j].y * rho[1] + Jp[j].z * rho[2] + Jo[j].x * rho[3] +
                     Jo[j].y * rho[4] + Jo[j].z * rho[5];   // g0 = J^T rho
            gg += dth[j] * dth[j];
        }
    }
    T jg2 = T(0);
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        T s = T(0);
#pragma unroll
        for (int j = 0; j < NMAX; ++j)
            if (EXACT || j < n) s += jrow(Jp[j], Jo[j], i) * dth[j];
        jg2 += s * s;
    }
    bool ok = (gg > T(0)) && (jg2 > T(0));
    if constexpr (!NB)
        if (!ok) return false;
    const T alpha_c = NB ? gg * rcp_nr(jg2) : gg / jg2;
    T A[21];
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int kk = 0; kk <= i; ++kk) {
            T s = T(0);
#pragma unroll
            for (int j = 0; j < NMAX; ++j)
                if (EXACT || j < n) s += jrow(Jp[j], Jo[j], i) * jrow(Jp[j], Jo[j], kk);
            A[i * (i + 1) / 2 + kk] = s + (i == kk ? T(c.d_floor) : T(0));
        }
    T y[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) y[i] = rho[i];
    if constexpr (NB) ok = chol6_solve<T, true>(A, y) && ok;
    else if (!chol6_solve(A, y)) return false;
    T ngn2 = T(0), ngd2 = T(0);
#pragma unroll
    for (int j = 0; j < NMAX; ++j) {
        if (EXACT || j < n) {
            gn[j] = -(Jp[j].x * y[0] + Jp[j].y * y[1] + Jp[j].z * y[2] + Jo[j].x * y[3] + Jo[j].y * y[4] +
                      Jo[j].z * y[5]);
            dth[j] = -alpha_c * dth[j];   // GD
            ngn2 += gn[j] * gn[j];
            ngd2 += dth[j] * dth[j];
        }
    }
    const T Rt = T(c.R);
    const T R2 = Rt * Rt;
    T wgd, wgn;   // step = wgd * GD + wgn * GN
    if constexpr (NB) {
        T qa = T(0), qb = T(0);
#pragma unroll
        for (int j = 0; j < NMAX; ++j) {
            if (EXACT || j < n) {
                const T d = dth[j] - gn[j];
                qa += d * d;
                qb += T(2) * gn[j] * d;
            }
        }
        const T qc = ngn2 - R2;
        const T disc = qb * qb - T(4) * qa * qc;
        const T sd = disc > T(0) ? disc * rsqrt_nr(disc) : T(0);
        const T tau = (qa > T(0) && disc >= T(0))
                          ? ((qb < T(0)) ? (T(2) * qc) * rcp_nr(-qb + sd) : (-qb - sd) * rcp_nr(T(2) * qa))
                          : T(-1);
        const bool inside = ngn2 <= R2, blend = tau >= T(0) && tau <= T(1);
        wgd = inside ? T(0) : blend ? tau : Rt * rsqrt_nr(ngd2);
        wgn = inside ? T(1) : blend ? T(1) - tau : T(0);
    } else if (ngn2 <= R2) {
        wgd = T(0); wgn = T(1);
    } else {
        T qa = T(0), qb = T(0);
#pragma unroll
        for (int j = 0; j < NMAX; ++j) {
            if (EXACT || j < n) {
                const T d = dth[j] - gn[j];
                qa += d * d;
                qb += T(2) * gn[j] * d;
            }
        }
        const T qc = ngn2 - R2;
        const T disc = qb * qb - T(4) * qa * qc;
        T tau = T(-1);
        if (qa > T(0) && disc >= T(0)) {
            const T sd = sqrt(disc);
            tau = (qb < T(0)) ? (T(2) * qc) / (-qb + sd) : (-qb - sd) / (T(2) * qa);   // smaller root
        }
        if (tau >= T(0) && tau <= T(1)) { wgd = tau; wgn = T(1) - tau; }
        else { wgd = Rt / sqrt(ngd2); wgn = T(0); }
    }
#pragma unroll
    for (int j = 0; j < NMAX; ++j)
        if (EXACT || j < n) dth[j] = wgd * dth[j] + wgn * gn[j];
    return ok;
}

// ---- single-coordinate direction (Eq. 16, R24): i* = argmax |g_i|, g = J^T W^2 rho,
//      step -sign(g_i*) min(|g_i*|, R) on i* only
template <int NMAX, bool EXACT = false, class T>
__device__ __forceinline__ bool single_coord_direction(const DevRobotT<T>& rb, const DevCfg& c,
                                                       const vec3<T> (&Jp)[NMAX], const vec3<T> (&Jo)[NMAX],
                                                       const T (&W)[6], const T (&rho)[6], T (&dth)[NMAX],
                                                       int& ist_out) {
    const int n = rb.n;
    T wr[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) wr[i] = W[i] * W[i] * rho[i];
    int ist = 0;
    T gbest = T(0), gabs = T(-1);
#pragma unroll
    for (int j = 0; j < NMAX; ++j) {
        if (EXACT || j < n) {
            const T g = Jp[j].x * wr[0] + Jp[j].y * wr[1] + Jp[j].z * wr[2] + Jo[j].x * wr[3] +
                        Jo[j].y * wr[4] + Jo[j].z * wr[5];
            if (fabs(g) > gabs) { gabs = fabs(g); gbest = g; ist = j; }
        }
    }
    ist_out = ist;
    const T Rt = T(c.R);
    const T step = (gbest > T(0)) ? -fmin(gabs, Rt) : fmin(gabs, Rt);
#pragma unroll
    for (int j = 0; j < NMAX; ++j) dth[j] = (j == ist) ? step : T(0);
    return gbest != T(0);
}

// cascade position q < 2A + 2 of a seed -> (direction kind, alpha index):
// LM alpha_1..alpha_A, dogleg, single coordinate alpha_0..alpha_A (Alg. 4
// order, R22-R24); the lowest successful position is the step the sequential
// cascade takes
__device__ __forceinline__ void decode_item(int q, int A, int& kind, int& a) {
    if (q < A) { kind = 0; a = q + 1; return; }
    if (q == A) { kind = 1; a = 0; return; }
    kind = 2;
    a = q - A - 1;
}

}  // namespace hjcd

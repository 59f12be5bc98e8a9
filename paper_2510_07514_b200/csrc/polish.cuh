// polish.cuh — device pieces of PJ-IK (Alg. 4) shared by the
// per-seed kernel (pjik.cu) and the cooperative per-target kernel
// (pjik_coop.cu): residual rho = -r, weighted cost, the 6x6 Cholesky, and the
// three step directions (LM via push-through K4, dogleg, single coordinate).
#pragma once
#include "kin.cuh"

namespace hjcd {

// 6x6 SPD solve by Cholesky, packed lower triangle A[i*(i+1)/2 + j]; the
// pivots are kept as reciprocals (rsqrt + Newton), so the factorisation and
// both substitutions are multiply-only.  Returns false if a pivot is not
// positive.
__device__ __forceinline__ bool chol6_solve(float (&A)[21], float (&b)[6]) {
    float id[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) {
#pragma unroll
        for (int j = 0; j <= i; ++j) {
            float s = A[i * (i + 1) / 2 + j];
#pragma unroll
            for (int k = 0; k < j; ++k) s -= A[i * (i + 1) / 2 + k] * A[j * (j + 1) / 2 + k];
            if (i == j) {
                if (!(s > 1e-30f)) return false;
                id[i] = rsqrt_nr(s);
                A[i * (i + 1) / 2 + i] = s * id[i];
            } else {
                A[i * (i + 1) / 2 + j] = s * id[j];
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        float s = b[i];
#pragma unroll
        for (int k = 0; k < i; ++k) s -= A[i * (i + 1) / 2 + k] * b[k];
        b[i] = s * id[i];
    }
#pragma unroll
    for (int i = 5; i >= 0; --i) {
        float s = b[i];
#pragma unroll
        for (int k = i + 1; k < 6; ++k) s -= A[k * (k + 1) / 2 + i] * b[k];
        b[i] = s * id[i];
    }
    return true;
}

__device__ __forceinline__ float jrow(const float3& Jp, const float3& Jo, int i) {
    return i == 0 ? Jp.x : i == 1 ? Jp.y : i == 2 ? Jp.z : i == 3 ? Jo.x : i == 4 ? Jo.y : Jo.z;
}

// rho = -r = [P_ee - P_t; -omega] (R19) and its norms
struct Resid {
    float rho[6];
    float ep, eo;
};

__device__ __forceinline__ Resid residual(const Target& tg, float3 pe, Quat qe) {
    Resid r;
    const Quat q = quat_err(tg.q, qe);
    const float sv = sqrtf(q.x * q.x + q.y * q.y + q.z * q.z);
    const float ang = 2.f * fast_atan2f(sv, q.w);           // |omega| (Eq. 5), q.w >= 0
    const float scale = sv > 1e-30f ? ang * rcp_nr(sv) : 2.f * rcp_nr(q.w);   // omega = scale * v
    r.rho[0] = pe.x - tg.p.x; r.rho[1] = pe.y - tg.p.y; r.rho[2] = pe.z - tg.p.z;
    r.rho[3] = -scale * q.x; r.rho[4] = -scale * q.y; r.rho[5] = -scale * q.z;
    r.ep = sqrtf(r.rho[0] * r.rho[0] + r.rho[1] * r.rho[1] + r.rho[2] * r.rho[2]);
    r.eo = ang;
    return r;
}

__device__ __forceinline__ float cost_w(const float (&W)[6], const float (&rho)[6]) {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 6; ++i) s += (W[i] * rho[i]) * (W[i] * rho[i]);
    return 0.5f * s;
}

template <int NMAX, bool EXACT = false>
__device__ __forceinline__ Resid eval_at(const DevRobot& rb, const Target& tg, const float (&th)[NMAX]) {
    float3 P[NMAX], Z[NMAX];   // unused (FRAMES = false), eliminated
    float3 pe;
    Quat qe;
    fk<NMAX, false, EXACT>(rb, th, P, Z, pe, qe);
    return residual(tg, pe, qe);
}

// ---- LM direction (Eq. 12 via push-through, K4): A = W G W + lambda I,
//      G_ik = sum_j J_ij J_kj / D_j; y = A^-1 W rho; dth_j = -(sum_i J_ij W_i y_i) / D_j,
//      then the element-wise trust-region clamp (Alg. 4 l.6, R21)
template <int NMAX, bool EXACT = false>
__device__ __forceinline__ bool lm_direction(const DevRobot& rb, const DevCfg& c, const float3 (&Jp)[NMAX],
                                             const float3 (&Jo)[NMAX], const float (&invD)[NMAX],
                                             const float (&W)[6], const float (&rho)[6], float (&dth)[NMAX]) {
    const int n = rb.n;
    float A[21];
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int kk = 0; kk <= i; ++kk) {
            float s = 0.f;
#pragma unroll
            for (int j = 0; j < NMAX; ++j)
                if (EXACT || j < n) s += jrow(Jp[j], Jo[j], i) * jrow(Jp[j], Jo[j], kk) * invD[j];
            A[i * (i + 1) / 2 + kk] = W[i] * W[kk] * s + (i == kk ? c.lambda : 0.f);
        }
    float y[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) y[i] = W[i] * rho[i];
    if (!chol6_solve(A, y)) return false;
#pragma unroll
    for (int i = 0; i < 6; ++i) y[i] *= W[i];
#pragma unroll
    for (int j = 0; j < NMAX; ++j) {
        if (EXACT || j < n) {
            const float s = Jp[j].x * y[0] + Jp[j].y * y[1] + Jp[j].z * y[2] + Jo[j].x * y[3] +
                            Jo[j].y * y[4] + Jo[j].z * y[5];
            dth[j] = clampf(-s * invD[j], -c.R, c.R);
        }
    }
    return true;
}

// ---- dogleg direction (Eqs. 14-15, R23): GD = -alpha_c J^T rho (Cauchy),
//      GN = -J^T (J J^T + d_floor I)^-1 rho, smallest tau in [0,1] with |dth(tau)| <= R
template <int NMAX, bool EXACT = false>
__device__ __forceinline__ bool dogleg_direction(const DevRobot& rb, const DevCfg& c, const float3 (&Jp)[NMAX],
                                                 const float3 (&Jo)[NMAX], const float (&rho)[6],
                                                 float (&dth)[NMAX], float (&gn)[NMAX]) {
    const int n = rb.n;
    float gg = 0.f;
#pragma unroll
    for (int j = 0; j < NMAX; ++j) {
        if (EXACT || j < n) {
            dth[j] = Jp[j].x * rho[0] + Jp[j].y * rho[1] + Jp[j].z * rho[2] + Jo[j].x * rho[3] +
                     Jo[j].y * rho[4] + Jo[j].z * rho[5];   // g0 = J^T rho
            gg += dth[j] * dth[j];
        }
    }
    float jg2 = 0.f;
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        float s = 0.f;
#pragma unroll
        for (int j = 0; j < NMAX; ++j)
            if (EXACT || j < n) s += jrow(Jp[j], Jo[j], i) * dth[j];
        jg2 += s * s;
    }
    if (!(gg > 0.f) || !(jg2 > 0.f)) return false;
    const float alpha_c = gg / jg2;
    float A[21];
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int kk = 0; kk <= i; ++kk) {
            float s = 0.f;
#pragma unroll
            for (int j = 0; j < NMAX; ++j)
                if (EXACT || j < n) s += jrow(Jp[j], Jo[j], i) * jrow(Jp[j], Jo[j], kk);
            A[i * (i + 1) / 2 + kk] = s + (i == kk ? c.d_floor : 0.f);
        }
    float y[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) y[i] = rho[i];
    if (!chol6_solve(A, y)) return false;
    float ngn2 = 0.f, ngd2 = 0.f;
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
    const float R2 = c.R * c.R;
    float wgd, wgn;   // step = wgd * GD + wgn * GN
    if (ngn2 <= R2) {
        wgd = 0.f; wgn = 1.f;
    } else {
        float qa = 0.f, qb = 0.f;
#pragma unroll
        for (int j = 0; j < NMAX; ++j) {
            if (EXACT || j < n) {
                const float d = dth[j] - gn[j];
                qa += d * d;
                qb += 2.f * gn[j] * d;
            }
        }
        const float qc = ngn2 - R2;
        const float disc = qb * qb - 4.f * qa * qc;
        float tau = -1.f;
        if (qa > 0.f && disc >= 0.f) {
            const float sd = sqrtf(disc);
            tau = (qb < 0.f) ? (2.f * qc) / (-qb + sd) : (-qb - sd) / (2.f * qa);   // smaller root
        }
        if (tau >= 0.f && tau <= 1.f) { wgd = tau; wgn = 1.f - tau; }
        else { wgd = c.R / sqrtf(ngd2); wgn = 0.f; }
    }
#pragma unroll
    for (int j = 0; j < NMAX; ++j)
        if (EXACT || j < n) dth[j] = wgd * dth[j] + wgn * gn[j];
    return true;
}

// ---- single-coordinate direction (Eq. 16, R24): i* = argmax |g_i|, g = J^T W^2 rho,
//      step -sign(g_i*) min(|g_i*|, R) on i* only
template <int NMAX, bool EXACT = false>
__device__ __forceinline__ bool single_coord_direction(const DevRobot& rb, const DevCfg& c,
                                                       const float3 (&Jp)[NMAX], const float3 (&Jo)[NMAX],
                                                       const float (&W)[6], const float (&rho)[6],
                                                       float (&dth)[NMAX]) {
    const int n = rb.n;
    float wr[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) wr[i] = W[i] * W[i] * rho[i];
    int ist = 0;
    float gbest = 0.f, gabs = -1.f;
#pragma unroll
    for (int j = 0; j < NMAX; ++j) {
        if (EXACT || j < n) {
            const float g = Jp[j].x * wr[0] + Jp[j].y * wr[1] + Jp[j].z * wr[2] + Jo[j].x * wr[3] +
                            Jo[j].y * wr[4] + Jo[j].z * wr[5];
            if (fabsf(g) > gabs) { gabs = fabsf(g); gbest = g; ist = j; }
        }
    }
    if (gbest == 0.f) return false;
    const float step = (gbest > 0.f) ? -fminf(gabs, c.R) : fminf(gabs, c.R);
#pragma unroll
    for (int j = 0; j < NMAX; ++j) dth[j] = (j == ist) ? step : 0.f;
    return true;
}

// cascade item q of a seed with flags f -> (direction kind, alpha index)
__device__ __forceinline__ void decode_item(int q, int f, int A, int& kind, int& a) {
    const int nlm = (f & 1) ? A : 0;
    const int ndl = (f & 2) ? 1 : 0;
    if (q < nlm) { kind = 0; a = q + 1; return; }
    q -= nlm;
    if (q < ndl) { kind = 1; a = 0; return; }
    kind = 2;
    a = q - ndl;
}

}  // namespace hjcd

// pjik.cu — k_pjik: stage 2 of HJCD-IK, PJ-IK polish (Alg. 4).
//
// One thread per polish seed, everything in registers.  The paper assigns a
// block per seed and GRiD for the Jacobian; here FK + frames give the
// geometric Jacobian in 12 flops per column (Eq. 7) and the weighted LM system
// (Eq. 12) is solved through the exact push-through identity
//   (J^T W^2 J + lambda D)^-1 J^T W^2 = S Jt^T (Jt Jt^T + lambda I_6)^-1 W,
//   S = D^-1/2, Jt = W J S,
// i.e. ONE 6x6 Cholesky for any n (K4) instead of an n x n solve.
// Fallbacks: dogleg (Eqs. 14-15), single coordinate (Eq. 16), perturbation.
#include "kin.cuh"

namespace hjcd {

// 6x6 SPD solve by Cholesky, packed lower triangle A[i*(i+1)/2 + j].
// Returns false if a pivot is not positive.
__device__ __forceinline__ bool chol6_solve(float (&A)[21], float (&b)[6]) {
#pragma unroll
    for (int i = 0; i < 6; ++i) {
#pragma unroll
        for (int j = 0; j <= i; ++j) {
            float s = A[i * (i + 1) / 2 + j];
#pragma unroll
            for (int k = 0; k < j; ++k) s -= A[i * (i + 1) / 2 + k] * A[j * (j + 1) / 2 + k];
            if (i == j) {
                if (!(s > 0.f)) return false;
                A[i * (i + 1) / 2 + i] = sqrtf(s);
            } else {
                A[i * (i + 1) / 2 + j] = s / A[j * (j + 1) / 2 + j];
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        float s = b[i];
#pragma unroll
        for (int k = 0; k < i; ++k) s -= A[i * (i + 1) / 2 + k] * b[k];
        b[i] = s / A[i * (i + 1) / 2 + i];
    }
#pragma unroll
    for (int i = 5; i >= 0; --i) {
        float s = b[i];
#pragma unroll
        for (int k = i + 1; k < 6; ++k) s -= A[k * (k + 1) / 2 + i] * b[k];
        b[i] = s / A[i * (i + 1) / 2 + i];
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
    const float ang = omega_norm(sv, q.w);
    const float scale = sv > 0.f ? ang / sv : 2.f / q.w;   // omega = scale * v (Eq. 5)
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

template <int NMAX>
__device__ __forceinline__ Resid eval_at(const DevRobot& rb, const Target& tg, const float (&th)[NMAX]) {
    float3 P[NMAX], Z[NMAX];   // unused (FRAMES = false), eliminated
    float3 pe;
    Quat qe;
    fk<NMAX, false>(rb, th, P, Z, pe, qe);
    return residual(tg, pe, qe);
}

// ---- LM direction (Eq. 12 via push-through, K4): A = W G W + lambda I,
//      G_ik = sum_j J_ij J_kj / D_j; y = A^-1 W rho; dth_j = -(sum_i J_ij W_i y_i) / D_j,
//      then the element-wise trust-region clamp (Alg. 4 l.6, R21)
template <int NMAX>
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
                if (j < n) s += jrow(Jp[j], Jo[j], i) * jrow(Jp[j], Jo[j], kk) * invD[j];
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
        if (j < n) {
            const float s = Jp[j].x * y[0] + Jp[j].y * y[1] + Jp[j].z * y[2] + Jo[j].x * y[3] +
                            Jo[j].y * y[4] + Jo[j].z * y[5];
            dth[j] = clampf(-s * invD[j], -c.R, c.R);
        }
    }
    return true;
}

// ---- dogleg direction (Eqs. 14-15, R23): GD = -alpha_c J^T rho (Cauchy),
//      GN = -J^T (J J^T + d_floor I)^-1 rho, smallest tau in [0,1] with |dth(tau)| <= R
template <int NMAX>
__device__ __forceinline__ bool dogleg_direction(const DevRobot& rb, const DevCfg& c, const float3 (&Jp)[NMAX],
                                                 const float3 (&Jo)[NMAX], const float (&rho)[6],
                                                 float (&dth)[NMAX], float (&gn)[NMAX]) {
    const int n = rb.n;
    float gg = 0.f;
#pragma unroll
    for (int j = 0; j < NMAX; ++j) {
        if (j < n) {
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
            if (j < n) s += jrow(Jp[j], Jo[j], i) * dth[j];
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
                if (j < n) s += jrow(Jp[j], Jo[j], i) * jrow(Jp[j], Jo[j], kk);
            A[i * (i + 1) / 2 + kk] = s + (i == kk ? c.d_floor : 0.f);
        }
    float y[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) y[i] = rho[i];
    if (!chol6_solve(A, y)) return false;
    float ngn2 = 0.f, ngd2 = 0.f;
#pragma unroll
    for (int j = 0; j < NMAX; ++j) {
        if (j < n) {
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
            if (j < n) {
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
        if (j < n) dth[j] = wgd * dth[j] + wgn * gn[j];
    return true;
}

// ---- single-coordinate direction (Eq. 16, R24): i* = argmax |g_i|, g = J^T W^2 rho,
//      step -sign(g_i*) min(|g_i*|, R) on i* only
template <int NMAX>
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
        if (j < n) {
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

// TEXIT = false: one thread per polish seed anywhere in the grid, per-seed break.
// TEXIT = true : one CTA per target, thread b = polish slot; after the fine test
//   of each iteration the CTA votes (__syncthreads_or) and stops at the first
//   iteration in which ANY seed of the target converged (Alg. 4 l.18 break,
//   P:203/P:309; R26b) — deterministic, no atomics.
template <int NMAX, bool TEXIT>
__global__ void __launch_bounds__(256)
k_pjik(const __grid_constant__ DevRobot rb, const __grid_constant__ DevCfg c,
       const float* __restrict__ targets, int T, const float* __restrict__ seeds,
       float* __restrict__ theta_out, float* __restrict__ ep_out, float* __restrict__ eo_out,
       int32_t* __restrict__ counts_out, int32_t* __restrict__ iters_out) {
    const int n = rb.n;
    const int used = c.copies * c.K;
    int t, b;
    bool active;
    if (TEXIT) {
        t = blockIdx.x;
        b = threadIdx.x;
        active = b < used;
    } else {
        const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
        if (gid >= (long long)T * used) return;
        t = (int)(gid / used);
        b = (int)(gid - (long long)t * used);
        active = true;
    }
    const Target tg = load_target(targets + 7ll * t);
    const uint32_t tid = (uint32_t)(c.tid_offset + t);
    const long long row = (long long)t * c.B + b;

    float th[NMAX], tt[NMAX], dth[NMAX];
#pragma unroll
    for (int j = 0; j < NMAX; ++j) th[j] = (active && j < n) ? seeds[row * n + j] : 0.f;

    int cnt[4] = {0, 0, 0, 0};
    float3 Jp[NMAX], Jo[NMAX];   // frames P, z, then Jacobian columns in place
    Resid r;
    int k;
    for (k = 0;; ++k) {
        float3 pe;
        Quat qe;
        bool conv = false;
        if (active) {
            fk<NMAX, true>(rb, th, Jp, Jo, pe, qe);
            r = residual(tg, pe, qe);
            // Alg. 4 l.18 (R26), checked at iteration start
            conv = r.ep < c.eps_p_fine && r.eo < c.eps_o_fine;
        }
        if (TEXIT) {
            if (__syncthreads_or(conv)) break;
        } else if (conv) {
            break;
        }
        if (k == c.lm_iters) break;
        if (!active) continue;

        // ---- Eq. 7: J columns [z x (P_ee - P_i); z] (prismatic: [z; 0])
#pragma unroll
        for (int j = 0; j < NMAX; ++j) {
            if (j < n) {
                const float3 z = Jo[j];
                if (rb.j[j].type == HJCD_REVOLUTE) {
                    Jp[j] = cross3(z, pe - Jp[j]);
                } else {
                    Jp[j] = z;
                    Jo[j] = f3(0.f, 0.f, 0.f);
                }
            }
        }
        // ---- W (R17): w_{p|o} / (1 + |J row|); D = max(diag J^T J, d_floor) (R20)
        float W[6], invD[NMAX];
        {
            float rn[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int j = 0; j < NMAX; ++j) {
                if (j < n) {
                    rn[0] += Jp[j].x * Jp[j].x; rn[1] += Jp[j].y * Jp[j].y; rn[2] += Jp[j].z * Jp[j].z;
                    rn[3] += Jo[j].x * Jo[j].x; rn[4] += Jo[j].y * Jo[j].y; rn[5] += Jo[j].z * Jo[j].z;
                    invD[j] = 1.f / fmaxf(dot3(Jp[j], Jp[j]) + dot3(Jo[j], Jo[j]), c.d_floor);
                }
            }
#pragma unroll
            for (int i = 0; i < 6; ++i) W[i] = (i < 3 ? c.w_p : c.w_o) / (1.f + sqrtf(rn[i]));
        }
        const float c0 = cost_w(W, r.rho);
        float n0 = 0.f;
#pragma unroll
        for (int i = 0; i < 6; ++i) n0 += r.rho[i] * r.rho[i];

        // Fallback cascade of Alg. 4 (l.3-17) as a state machine with ONE trial
        // evaluation site: phase 0 = LM + line search (Eq. 12-13), 1 = dogleg
        // (Eqs. 14-15), 2 = single coordinate + line search (Eq. 16), 3 = perturb.
        bool accepted = false;
        int phase = 0;
        bool have = lm_direction<NMAX>(rb, c, Jp, Jo, invD, W, r.rho, dth);
        if (!have) phase = 1;
        int a = 0;
        float alpha = 1.f;
        for (;;) {
            if (!have) {
                // prepare the direction of the current phase
                if (phase == 1) have = dogleg_direction<NMAX>(rb, c, Jp, Jo, r.rho, dth, tt);
                else if (phase == 2) have = single_coord_direction<NMAX>(rb, c, Jp, Jo, W, r.rho, dth);
                if (!have) {
                    if (++phase >= 3) break;
                    continue;
                }
                a = 0;
                alpha = 1.f;
            }
#pragma unroll
            for (int j = 0; j < NMAX; ++j)
                if (j < n) tt[j] = clampf(th[j] + alpha * dth[j], rb.j[j].lo, rb.j[j].hi);
            const Resid rt = eval_at<NMAX>(rb, tg, tt);
            bool ok;
            if (phase == 1) {   // dogleg acceptance on the unweighted |rho| (R23)
                float nt = 0.f;
#pragma unroll
                for (int i = 0; i < 6; ++i) nt += rt.rho[i] * rt.rho[i];
                ok = nt < n0;
            } else {            // Eq. 13: c_W(trial) < c_W(theta), W frozen (R22)
                ok = cost_w(W, rt.rho) < c0;
            }
            if (ok) { accepted = true; cnt[phase]++; break; }
            if (phase != 1 && a < c.A) { ++a; alpha *= c.inv_beta; continue; }
            have = false;
            if (++phase >= 3) break;
        }
        if (accepted) {
#pragma unroll
            for (int j = 0; j < NMAX; ++j) th[j] = tt[j];
        } else {
            // ---- Alg. 4 l.17 (R25): random perturbation
            perturb<NMAX>(rb, c, th, c.sigma_lm, tid, (uint32_t)b, P_PJPERT, (uint32_t)k);
            cnt[3]++;
        }
    }

    if (!active) return;
#pragma unroll
    for (int j = 0; j < NMAX; ++j)
        if (j < n) theta_out[row * n + j] = th[j];
    ep_out[row] = r.ep;
    eo_out[row] = r.eo;
    if (counts_out) {
#pragma unroll
        for (int i = 0; i < 4; ++i) counts_out[row * 4 + i] = cnt[i];
    }
    if (iters_out) iters_out[row] = k;
}

template <int NMAX>
static cudaError_t launch_pjik_t(const DevRobot& rb, const DevCfg& c, const float* targets, int T,
                                 const float* seeds, float* theta, float* ep, float* eo, int32_t* counts,
                                 int32_t* iters, cudaStream_t s) {
    const int used = c.copies * c.K;
    if (c.target_early_exit) {
        if (used > 256) return cudaErrorInvalidConfiguration;
        const int block = (used + 31) / 32 * 32;
        k_pjik<NMAX, true><<<T, block, 0, s>>>(rb, c, targets, T, seeds, theta, ep, eo, counts, iters);
    } else {
        const long long total = (long long)T * used;
        const int block = 128;
        const long long grid = (total + block - 1) / block;
        if (grid > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
        k_pjik<NMAX, false><<<(unsigned)grid, block, 0, s>>>(rb, c, targets, T, seeds, theta, ep, eo, counts,
                                                               iters);
    }
    return cudaGetLastError();
}

cudaError_t launch_pjik(const DevRobot& rb, const DevCfg& c, const float* targets, int T,
                        const float* seeds, float* theta, float* ep, float* eo, int32_t* counts,
                        int32_t* iters, cudaStream_t s) {
    if (rb.n <= 8) return launch_pjik_t<8>(rb, c, targets, T, seeds, theta, ep, eo, counts, iters, s);
    if (rb.n <= 16) return launch_pjik_t<16>(rb, c, targets, T, seeds, theta, ep, eo, counts, iters, s);
    return launch_pjik_t<32>(rb, c, targets, T, seeds, theta, ep, eo, counts, iters, s);
}

}  // namespace hjcd

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
#include "polish.cuh"

namespace hjcd {

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
    {
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
    // per-target stop rule: one CTA per target, warp-cooperative cascade (pjik_coop.cu)
    if (c.target_early_exit) return launch_pjik_coop(rb, c, targets, T, seeds, theta, ep, eo, counts, iters, s);
    if (rb.n <= 8) return launch_pjik_t<8>(rb, c, targets, T, seeds, theta, ep, eo, counts, iters, s);
    if (rb.n <= 16) return launch_pjik_t<16>(rb, c, targets, T, seeds, theta, ep, eo, counts, iters, s);
    return launch_pjik_t<32>(rb, c, targets, T, seeds, theta, ep, eo, counts, iters, s);
}

}  // namespace hjcd

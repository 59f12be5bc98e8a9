#pragma once
// ccd.cuh — k_ccd: classic position-only CCD (Alg. 1), the
// baseline HJCD-IK's PO-CCD extends (SURVEY §8(f) f4 ablation).
//
// One thread per (target, seed), M seeds per target (Philox-uniform like
// PO-CCD's S3, or caller-given).  An iteration sweeps the joints from the tip
// to the root (Alg. 1 l.2): Delta theta_j is the signed angle between the
// projections of P_ee - P_j and P_t - P_j on the plane normal to z_j (Eqs.
// 8-9, readings R3, R4), clamped to the limits (R7).  Updating joint j moves
// only the end effector (the frames of joints < j do not depend on theta_j), and
// it moves it by the rigid rotation about (P_j, z_j), so ONE FK per sweep plus
// an O(1) end-effector update per joint is exactly the literal "FK per joint
// update" (K2).  After the sweep, Alg. 1 l.7's test |P_ee - P_t| < eps (R12's
// unsquared reading, eps = eps_p_coarse) freezes the seed.
#include "kin.cuh"

namespace hjcd {

template <int NMAX, bool EXACT>
__global__ void __launch_bounds__(128)
k_ccd(const __grid_constant__ DevRobot rb, const __grid_constant__ DevCfg c,
      const float* __restrict__ targets, int T, const float* __restrict__ seeds,
      float* __restrict__ theta_out, float* __restrict__ ep_out, int32_t* __restrict__ iters_out) {
    const int M = c.M;
    const int n = rb.n;
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= (long long)T * M) return;
    const int t = (int)(gid / M);
    const int m = (int)(gid - (long long)t * M);
    const Target tg = load_target(targets + 7ll * t);
    const uint32_t tid = (uint32_t)(c.tid_offset + t);

    float th[NMAX];
    if (seeds) {
#pragma unroll
        for (int j = 0; j < NMAX; ++j)
            if (EXACT || j < n) th[j] = seeds[((long long)t * n + j) * M + m];
    } else {   // the same Philox draw as PO-CCD's seeding (Alg. 3 l.2-3, R30)
#pragma unroll
        for (int blk = 0; blk < (NMAX + 3) / 4; ++blk) {
            if (EXACT || 4 * blk < n) {
                uint4 r = draw(c, tid, (uint32_t)m, P_INIT, 0u, (uint32_t)blk);
                uint32_t x[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    int j = 4 * blk + e;
                    if (j < NMAX && (EXACT || j < n)) {
                        float lo = rb.j[j].lo, hi = rb.j[j].hi;
                        th[j] = __fmaf_rn(__fsub_rn(hi, lo), u01(x[e]), lo);
                    }
                }
            }
        }
    }
    const float tau2 = c.tau_deg * c.tau_deg;
    float3 P[NMAX], Z[NMAX];
    float3 pe;
    Quat qe;
    float ep = 0.f;
    int k;
    for (k = 0;; ++k) {
        fk<NMAX, true, EXACT>(rb, th, P, Z, pe, qe);
        const float3 rp = tg.p - pe;
        ep = sqrtf(dot3(rp, rp));
        if (ep < c.eps_p_coarse) break;          // Alg. 1 l.7 (R12), tested before the sweep
        if (k == c.ccd_iters) break;
        // Alg. 1 l.2-5: joints from the tip (n-1) to the root (0)
#pragma unroll
        for (int jj = NMAX - 1; jj >= 0; --jj) {
            if (EXACT || jj < n) {
                const DevJoint& J = rb.j[jj];
                const float3 z = Z[jj];
                if (J.type == HJCD_REVOLUTE) {
                    const float3 u = pe - P[jj];
                    const float3 v = tg.p - P[jj];
                    const float3 up = u - dot3(u, z) * z;
                    const float3 vp = v - dot3(v, z) * z;
                    const float3 zxu = cross3(z, u);
                    float step = 0.f;
                    if (dot3(up, up) >= tau2 && dot3(vp, vp) >= tau2)   // R4
                        step = atan2f(dot3(zxu, vp), dot3(up, vp));     // Eq. 9 signed (R3)
                    const float d = clampf(th[jj] + step, J.lo, J.hi) - th[jj];   // R7
                    th[jj] = clampf(th[jj] + d, J.lo, J.hi);
                    // the end effector rotates about (P_j, z_j) by d
                    float s, co;
                    sincos_b(d, &s, &co);
                    pe = pe - (1.f - co) * up + s * zxu;
                } else {
                    // prismatic (R32): the exact 1-D minimiser along z_j
                    const float d = clampf(th[jj] + dot3(z, tg.p - pe), J.lo, J.hi) - th[jj];
                    th[jj] = clampf(th[jj] + d, J.lo, J.hi);
                    pe = pe + d * z;
                }
            }
        }
    }
#pragma unroll
    for (int j = 0; j < NMAX; ++j)
        if (EXACT || j < n) theta_out[((long long)t * n + j) * M + m] = th[j];
    const long long o = (long long)t * M + m;
    if (ep_out) ep_out[o] = ep;
    if (iters_out) iters_out[o] = k;
}

template <int NMAX, bool EXACT>
cudaError_t launch_ccd_t(const DevRobot& rb, const DevCfg& c, const float* targets, int T, const float* seeds,
                         float* theta, float* ep, int32_t* iters, cudaStream_t s) {
    const long long total = (long long)T * c.M;
    const int block = 128;
    const long long grid = (total + block - 1) / block;
    if (grid > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    k_ccd<NMAX, EXACT><<<(unsigned)grid, block, 0, s>>>(rb, c, targets, T, seeds, theta, ep, iters);
    return cudaGetLastError();
}

}  // namespace hjcd

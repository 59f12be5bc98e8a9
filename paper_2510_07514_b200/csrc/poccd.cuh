#pragma once
// poccd.cuh — k_poccd: stage 1 of HJCD-IK, PO-CCD (Alg. 3).
//
// Mapping: one thread per (target, seed).  The paper runs one block per seed
// with two warps per joint; on B200 the per-seed work (~1.6 kflop per
// iteration at n = 7) is far too small to amortise block-level reductions, so
// each seed lives in one thread's registers: FK with frames (n sincos), the 2n
// candidate steps, and EXACT O(1) candidate scoring by rigid rotation of the
// end effector about the joint axis (K2: FK(theta + d e_j) is the
// current end-effector pose rotated about (P_j, z_j) by d), then the greedy
// argmins, the gamma test on the composed two-joint move, and Philox
// perturbation.  Seeding (Alg. 3 l.2-3) is fused in.  Per-seed freeze on the
// coarse test (Alg. 3 l.14) is deterministic.
#include <cooperative_groups.h>
#include <cstdlib>

#include "kin.cuh"

namespace cg = cooperative_groups;

#ifndef HJCD_VOTE_RELAXED
#define HJCD_VOTE_RELAXED 1
#endif
#ifndef HJCD_X1_UNIFORM
#define HJCD_X1_UNIFORM 1
#endif

namespace hjcd {

// TEXIT = false: one thread per (target, seed) anywhere in the grid; each seed
//   freezes on its own coarse test (per-seed break).
// TEXIT = true : the paper's stop rule ("once a seed satisfies the ...
//   thresholds, the parallel loop is broken and all samples are returned";
//   DESIGN.md R12b) as a deterministic lockstep: the M seeds of a target live
//   in ONE thread-block cluster (CL CTAs x nt threads, seed m = rank * nt +
//   threadIdx.x) and after every coarse test the cluster ORs the per-warp
//   "converged" votes into a 3-slot flag ring in each CTA's shared memory
//   (DSMEM stores, then barrier.cluster arrive.release / wait.acquire); all
//   seeds of the target stop at the first iteration in which any seed passed.
// REV: every DoF joint is revolute (no per-joint type branches).
// Occupancy target: 4 CTAs of 128 (<= 128 registers) up to 14 joints; the
// 16- and 32-joint bounds would spill 1-1.6 KB at 128, so they get 170 / 255.
#ifndef HJCD_FRAMES_SMEM_MAX
#define HJCD_FRAMES_SMEM_MAX 32   // every bound: 24 B per joint and thread (98 KB per 128-thread CTA at 32)
#endif
template <int NMAX>
constexpr int poccd_min_blocks() { return NMAX <= 14 ? 4 : (NMAX <= 18 ? 3 : 2); }

template <int NMAX, bool EXACT, bool TEXIT, int REV>
__global__ void __launch_bounds__(poccd_cta(NMAX), poccd_min_blocks<NMAX>() * 128 / poccd_cta(NMAX))
k_poccd(const __grid_constant__ DevRobot rb, const __grid_constant__ DevCfg c,
        const float* __restrict__ targets, int T, const float* __restrict__ seeds,
        float* __restrict__ theta_out, float* __restrict__ cost_out, float* __restrict__ ep_out,
        float* __restrict__ eo_out, int32_t* __restrict__ iters_out, int CL, const TraceOut trace,
        uint32_t* __restrict__ ready) {
    const int M = c.M;
    const int n = rb.n;
    int t, m;
    bool active = true;
    __shared__ int s_flag[3];
    // the frames (P_j, z_j) of this iteration, per thread, so the two moved
    // joints' frames are two indexed loads instead of 2 x NMAX predicated selects
    constexpr bool FRAMES_SMEM = NMAX <= HJCD_FRAMES_SMEM_MAX;
    constexpr int FRS = poccd_cta(NMAX);   // frame stride: the largest CTA size (immediate offsets, K20b)
    extern __shared__ float4 s_frames[];   // [NMAX][blockDim] (P.xyz, z.x), then float2 [NMAX][blockDim] (z.yz)
    if (TEXIT) {
        t = (int)(blockIdx.x / (unsigned)CL);
        m = (int)(blockIdx.x - (unsigned)t * CL) * (int)blockDim.x + (int)threadIdx.x;
        active = m < M;
        // DESIGN K10: the dependent PJ-IK grid may be scheduled once every CTA
        // of this grid is resident or done, so its waiting CTAs never hold
        // resources a PO-CCD CTA still needs
        if (ready) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#ifdef HJCD_PROBE
        if (ready && threadIdx.x == 0) atomicMin(probe_base(ready, T) + t, probe_now());
#endif
        if (threadIdx.x < 3) s_flag[threadIdx.x] = 0;
        cg::this_cluster().sync();   // flags initialised before any remote store
    } else {
        const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
        if (gid >= (long long)T * M) return;
        t = (int)(gid / M);
        m = (int)(gid - (long long)t * M);
    }
    const Target tg = load_target(targets + 7ll * t);
    const uint32_t tid = (uint32_t)(c.tid_offset + t);

    // ---- Alg. 3 l.2-3: theta ~ U(theta_min, theta_max) (fp32 fma: R30)
    float th[NMAX];
    if (seeds) {
#pragma unroll
        for (int j = 0; j < NMAX; ++j)
            if (EXACT || j < n) th[j] = active ? seeds[((long long)t * n + j) * M + m] : rb.j[j].lo;
    } else {
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

    float3 P[NMAX], Z[NMAX];
    float3 pe;
    Quat qe;
    float ep = 0.f, eo = 0.f;
    float rho_k = 1.f;   // delta_rho^k, by repeated multiplication (R5)
    int k;
    for (k = 0;; ++k, rho_k *= c.delta_rho) {
        if (trace.theta && active) {   // theta at the start of iteration k (hjcd_poccd_trace)
            float* h = trace.theta + (((long long)t * M + m) * (c.ccd_iters + 1) + k) * n;
#pragma unroll
            for (int j = 0; j < NMAX; ++j)
                if (EXACT || j < n) h[j] = th[j];
        }
        fk<NMAX, true, EXACT, true, REV>(rb, th, P, Z, pe, qe);
        if constexpr (FRAMES_SMEM) {
            float2* s_fz = (float2*)(s_frames + NMAX * FRS);
#pragma unroll
            for (int j = 0; j < NMAX; ++j) {
                if (EXACT || j < n) {
                    s_frames[j * FRS + threadIdx.x] = make_float4(P[j].x, P[j].y, P[j].z, Z[j].x);
                    s_fz[j * FRS + threadIdx.x] = make_float2(Z[j].y, Z[j].z);
                }
            }
        }
        const float3 rp = tg.p - pe;                   // r_p (Eq. 4)
        const Quat qr = quat_err(tg.q, qe);            // q_err (Eq. 5), w >= 0
        const float sv = sqrt_approx(qr.x * qr.x + qr.y * qr.y + qr.z * qr.z);
        ep = sqrt_approx(dot3(rp, rp));
        eo = 2.f * fast_atan2f(sv, qr.w);              // |omega|
        // Alg. 3 l.14: coarse test (R12), checked at iteration start
        const bool conv = ep < c.eps_p_coarse && eo < c.eps_o_coarse;
        if (TEXIT) {
            // R12b: cluster-wide OR of the votes of iteration k (slot k % 3;
            // slot (k + 2) % 3 is cleared after the barrier: its readers passed
            // barrier k - 1 ... k, its next writers wait for barrier k + 1)
            cg::cluster_group cluster = cg::this_cluster();
            const int slot = k % 3;
            const unsigned vote = __ballot_sync(0xffffffffu, conv && active);
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
        } else if (conv) {
            break;
        }
        if (k == c.ccd_iters) break;

        // Eq. 10 (R2): phi = 2 atan2(|v|, w), a = v / |v|; sgn(a . z_j) = sgn(v . z_j)
        const float phi = eo;
        const float3 vq = f3(qr.x, qr.y, qr.z);
        const float dphi = phi > 0.f ? fmaxf(c.delta_min, c.delta0 * rho_k) * phi : 0.f;   // delta(k) phi
        const float tau2 = c.tau_deg * c.tau_deg;
        // K2b: for an orientation candidate d, expanding q_err (x) q(z, -d) gives
        //   |v'|^2 = C^2 |v|^2 + S^2 (w^2 + |v|^2 - (v.z)^2) - 2 C S w (v.z),
        // C, S = cos, sin(d / 2).  Unclamped, d = sgn(v.z) dphi: C, S of dphi / 2
        // are shared by all joints and the last term is -2 C S w |v.z|.
        float Cd, Sd;
        __sincosf(0.5f * dphi, &Sd, &Cd);
        const float sv2 = sv * sv, w2 = qr.w * qr.w, wsv2 = w2 + sv2, ka = sv2 + wsv2;
        const float ob0 = Cd * Cd * sv2 + Sd * Sd * wsv2;
        const float ob1 = Sd * Sd, ob2 = 2.f * Cd * Sd * qr.w;

        // ---- Alg. 3 l.6-9: per-joint candidates, scored, greedy argmin
        float best_p = CUDART_INF_F, best_o = CUDART_INF_F;
        int jp = 0, jo = 0;
        float dp_best = 0.f, do_best = 0.f;
#pragma unroll
        for (int j = 0; j < NMAX; ++j) {
            if (EXACT || j < n) {
                const DevJoint& J = rb.j[j];
                const float3 z = Z[j];
                float dp, sp, dor, so;
                if (REV || J.type == HJCD_REVOLUTE) {
                    // Eqs. 8-9 (R3): signed angle between the projections of
                    // u = P_ee - P_j and v = P_t - P_j on the plane normal to z_j;
                    // z.(u_p x v_p) = (z x u).v_p
                    const float3 u = pe - P[j];
                    const float3 v = tg.p - P[j];
                    const float3 up = u - dot3(u, z) * z;
                    const float3 vp = v - dot3(v, z) * z;
                    const float3 zxu = cross3(z, u);
                    float step = 0.f;
                    if (dot3(up, up) >= tau2 && dot3(vp, vp) >= tau2)   // R4
                        step = fast_atan2f(dot3(zxu, vp), dot3(up, vp));
                    dp = clampf(th[j] + step, J.lo, J.hi) - th[j];     // R7
                    // score (K2): r_p' = r_p + (1 - cos d) u_perp - sin d (z x u)
                    float s2, c2;
                    __sincosf(0.5f * dp, &s2, &c2);
                    if (dp == 0.f) { s2 = 0.f; c2 = 1.f; }
                    const float sn = 2.f * s2 * c2, omc = 2.f * s2 * s2;
                    const float3 r2 = rp + omc * up - sn * zxu;
                    sp = dot3(r2, r2);
                    // Eq. 11 (R5): delta(k) sgn(a . z_j) phi, sgn(0) = 0
                    const float vz = dot3(vq, z);
                    const float tsum = th[j] + (vz != 0.f ? copysignf(dphi, vz) : 0.f);
                    dor = clampf(tsum, J.lo, J.hi) - th[j];
                    // score (K2): |v'|^2 of q_err (x) q(z, -d), monotone in |omega'|
#if HJCD_X1_UNIFORM
                    {   // K40: the three cases computed branch-free and selected (no divergence)
                        const float avz = fabsf(vz);
                        const float so_un = ob0 - avz * fmaf(ob1, avz, ob2);   // K2b closed form
                        // clamped step: the same closed form at the effective d, in
                        // double angles: C^2 = (1 + cos d) / 2, S^2 = (1 - cos d) / 2, 2 C S = sin d
                        float sd, cd;
                        __sincosf(dor, &sd, &cd);
                        const float vz2 = vz * vz;
                        const float so_cl = 0.5f * fmaf(cd, vz2 - w2, ka - vz2) - sd * (qr.w * vz);
                        so = dor == 0.f ? sv * sv : ((tsum >= J.lo && tsum <= J.hi) ? so_un : so_cl);
                    }
#else
                    if (dor == 0.f) {
                        so = sv * sv;                     // zero step: the current residual, exactly
                    } else if (tsum >= J.lo && tsum <= J.hi) {
                        const float avz = fabsf(vz);
                        so = ob0 - avz * fmaf(ob1, avz, ob2);   // K2b closed form
                    } else {   // clamped step: the same closed form at the effective d, in
                        // double angles: C^2 = (1 + cos d) / 2, S^2 = (1 - cos d) / 2, 2 C S = sin d
                        float sd, cd;
                        __sincosf(dor, &sd, &cd);
                        const float vz2 = vz * vz;
                        so = 0.5f * fmaf(cd, vz2 - w2, ka - vz2) - sd * (qr.w * vz);
                    }
#endif
                } else {
                    // prismatic (R32): exact 1-D minimiser z . (P_t - P_ee)
                    dp = clampf(th[j] + dot3(z, rp), J.lo, J.hi) - th[j];
                    const float3 r2 = rp - dp * z;
                    sp = dot3(r2, r2);
                    dor = 0.f;
                    so = sv * sv;
                }
                if (sp < best_p) { best_p = sp; jp = j; dp_best = dp; }
                if (so < best_o) { best_o = so; jo = j; do_best = dor; }
            }
        }

        // ---- Alg. 3 l.10 + P:201: same joint -> the larger |step|, tie -> position (R8)
        int ja = -1, jb;           // ja upstream (smaller index), jb downstream
        float da = 0.f, db;
        if (jp == jo) {
            jb = jp;
            db = fabsf(dp_best) >= fabsf(do_best) ? dp_best : do_best;
        } else if (jp < jo) {
            ja = jp; da = dp_best; jb = jo; db = do_best;
        } else {
            ja = jo; da = do_best; jb = jp; db = dp_best;
        }
        // frames of the two moved joints (uniform-index selects, no local memory);
        // an orientation winner is always revolute (prismatic candidates are 0)
        float3 Pa = f3(0.f, 0.f, 0.f), Za = Pa, Pb = Pa, Zb = Pa;
        const int ta = (!REV && ja >= 0 && ((rb.pmask >> ja) & 1u)) ? HJCD_PRISMATIC : HJCD_REVOLUTE;
        const int tb = (!REV && ((rb.pmask >> jb) & 1u)) ? HJCD_PRISMATIC : HJCD_REVOLUTE;
        if constexpr (FRAMES_SMEM) {
            const float2* s_fz = (const float2*)(s_frames + NMAX * FRS);
            const float4 fb = s_frames[jb * FRS + threadIdx.x];
            const float2 gb = s_fz[jb * FRS + threadIdx.x];
            Pb = f3(fb.x, fb.y, fb.z); Zb = f3(fb.w, gb.x, gb.y);
            if (ja >= 0) {
                const float4 fa = s_frames[ja * FRS + threadIdx.x];
                const float2 ga = s_fz[ja * FRS + threadIdx.x];
                Pa = f3(fa.x, fa.y, fa.z); Za = f3(fa.w, ga.x, ga.y);
            }
        } else {
#pragma unroll
            for (int j = 0; j < NMAX; ++j) {
                if (EXACT || j < n) {
                    if (j == ja) { Pa = P[j]; Za = Z[j]; }
                    if (j == jb) { Pb = P[j]; Zb = Z[j]; }
                }
            }
        }
        // r(theta_hat) exactly: downstream joint's rigid motion first, then the
        // upstream one, both about the pre-update frames (K3)
        float3 p2 = pe;
        Quat q2 = qr;
        {
            if (tb == HJCD_REVOLUTE) {
                float s2, c2;
                __sincosf(0.5f * db, &s2, &c2);
                const float3 u = p2 - Pb;
                const float3 up = u - dot3(u, Zb) * Zb;
                p2 = p2 - (2.f * s2 * s2) * up + (2.f * s2 * c2) * cross3(Zb, u);
                q2 = qerr_rotate(q2, Zb, c2, s2);
            } else {
                p2 = p2 + db * Zb;
            }
            if (ja >= 0) {
                if (ta == HJCD_REVOLUTE) {
                    float s2, c2;
                    __sincosf(0.5f * da, &s2, &c2);
                    const float3 u = p2 - Pa;
                    const float3 up = u - dot3(u, Za) * Za;
                    p2 = p2 - (2.f * s2 * s2) * up + (2.f * s2 * c2) * cross3(Za, u);
                    q2 = qerr_rotate(q2, Za, c2, s2);
                } else {
                    p2 = p2 + da * Za;
                }
            }
        }
        const float3 rh = tg.p - p2;
        const float ep_h = sqrt_approx(dot3(rh, rh));
        const float eo_h = 2.f * fast_atan2f(sqrt_approx(q2.x * q2.x + q2.y * q2.y + q2.z * q2.z), fabsf(q2.w));
        // ---- Alg. 3 l.11-13 (R10): accept on an improvement > gamma in either space
        const bool accept = (ep - ep_h) > c.gamma || (eo - eo_h) > c.gamma;
        if (trace.words && active)   // decision word: see hjcd_poccd_trace (include/hjcd.h)
            trace.words[((long long)t * M + m) * c.ccd_iters + k] =
                (uint32_t)jp | ((uint32_t)jo << 5) | ((jp == jo && db != dp_best) ? 1u << 10 : 0u) |
                (accept ? 1u << 11 : 0u) | ((dp_best > 0.f ? 1u : dp_best < 0.f ? 2u : 0u) << 12) |
                ((do_best > 0.f ? 1u : do_best < 0.f ? 2u : 0u) << 14);
        if (accept) {
#pragma unroll
            for (int j = 0; j < NMAX; ++j) {
                if (EXACT || j < n) {
                    // theta + d_eff, re-clamped so rounding never leaves [lo, hi]
                    // (the other joints get + 0 and a no-op clamp: one select chain)
                    const float d = j == jb ? db : (j == ja ? da : 0.f);
                    th[j] = clampf(th[j] + d, rb.j[j].lo, rb.j[j].hi);
                }
            }
        }
        if constexpr (TEXIT && FRAMES_SMEM && NMAX > 8) {
            // K12: the rejected seeds' Philox draws (R11), spread over the warp
            // (for >= 3 draws per seed; at n <= 8 the per-lane form is as fast):
            // item (r, blk) = block blk of the r-th rejecting lane, its 4 normals
            // left in that lane's (now dead) frame slot blk; then each rejecting
            // lane applies its own, exactly as perturb() would
            const unsigned rej = __ballot_sync(0xffffffffu, active && !accept);
            if (rej) {
                const int nb = EXACT ? (NMAX + 3) / 4 : (n + 3) / 4;
                const int lane = (int)(threadIdx.x & 31);
                const int items = __popc(rej) * nb;
                for (int it = lane; it < items; it += 32) {
                    const int r = it / nb, blk = it - r * nb;
                    const int ol = (int)__fns(rej, 0u, r + 1);
                    float g[4];
                    normals4<true>(draw(c, tid, (uint32_t)(m - lane + ol), P_PERTURB, (uint32_t)k, (uint32_t)blk), g);
                    s_frames[blk * FRS + (threadIdx.x - lane + ol)] = make_float4(g[0], g[1], g[2], g[3]);
                }
                __syncwarp();
                if (active && !accept) {
#pragma unroll
                    for (int blk = 0; blk < (NMAX + 3) / 4; ++blk) {
                        if (EXACT || 4 * blk < n) {
                            const float4 g4 = s_frames[blk * FRS + threadIdx.x];
                            const float g[4] = {g4.x, g4.y, g4.z, g4.w};
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const int j = 4 * blk + e;
                                if (j < NMAX && (EXACT || j < n))
                                    th[j] = clampf(th[j] + c.sigma_ccd * g[e], rb.j[j].lo, rb.j[j].hi);
                            }
                        }
                    }
                }
            }
        } else if (!accept) {
            perturb<NMAX, EXACT, true>(rb, c, th, c.sigma_ccd, tid, (uint32_t)m, P_PERTURB, (uint32_t)k);   // R11 (K5)
        }
    }

    if (active) {
#pragma unroll
        for (int j = 0; j < NMAX; ++j)
            if (EXACT || j < n) theta_out[((long long)t * n + j) * M + m] = th[j];
        const long long o = (long long)t * M + m;
        cost_out[o] = c.w_p * c.w_p * ep * ep + c.w_o * c.w_o * eo * eo;   // R14
        if (ep_out) ep_out[o] = ep;
        if (eo_out) eo_out[o] = eo;
        if (iters_out) iters_out[o] = k;
    }
    if (TEXIT && ready) {   // DESIGN K10: this CTA's seeds of target t are in memory
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0 && atomicAdd(ready + t, 1u) + 1u == (uint32_t)CL)
            ready_push(ready, T, t, k);   // DESIGN K26: the cluster's last CTA queues the target
#ifdef HJCD_PROBE
        if (threadIdx.x == 0) atomicMax(probe_base(ready, T) + T + t, probe_now());
#endif
    }
}

template <int NMAX>
inline size_t poccd_smem(int) {   // the per-thread frames (24 B per joint), stride poccd_cta(NMAX)
    return NMAX <= HJCD_FRAMES_SMEM_MAX ? (size_t)NMAX * poccd_cta(NMAX) * (sizeof(float4) + sizeof(float2)) : 0;
}

template <int NMAX, bool EXACT, int REV>
static cudaError_t launch_poccd_r(const DevRobot& rb, const DevCfg& c, const float* targets, int T,
                                  const float* seeds, float* theta, float* cost, float* ep, float* eo,
                                  int32_t* iters, TraceOut trace, uint32_t* ready, cudaStream_t s) {
    static std::atomic<unsigned long long> smem_attr{0};   // the frames copy may exceed the 48 KB default
    if (poccd_smem<NMAX>(poccd_cta(NMAX)) > 0) {
        const cudaError_t e = once_per_device(smem_attr, [] {
            const int b = (int)poccd_smem<NMAX>(poccd_cta(NMAX));
            cudaError_t e2 = cudaFuncSetAttribute(k_poccd<NMAX, EXACT, false, REV>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, b);
            if (e2 == cudaSuccess)
                e2 = cudaFuncSetAttribute(k_poccd<NMAX, EXACT, true, REV>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
            return e2;
        });
        if (e != cudaSuccess) return e;
    }
    if (!c.ccd_early_exit) {
        const long long total = (long long)T * c.M;
        const int block = 128;
        const long long grid = (total + block - 1) / block;
        if (grid > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
        k_poccd<NMAX, EXACT, false, REV><<<(unsigned)grid, block, poccd_smem<NMAX>(block), s>>>(
            rb, c, targets, T, seeds, theta, cost, ep, eo, iters, 1, trace, nullptr);
        return cudaGetLastError();
    }
    int nt, CL;
    texit_shape(c.M, NMAX, nt, CL);
    if (CL > 16) return cudaErrorInvalidConfiguration;
    if (CL > 8) {
        static std::atomic<unsigned long long> np{0};
        const cudaError_t e = once_per_device(np, [] {
            return cudaFuncSetAttribute(k_poccd<NMAX, EXACT, true, REV>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        });
        if (e != cudaSuccess) return e;
    }
    const long long grid = (long long)T * CL;
    if (grid > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid, 1, 1);
    cfg.blockDim = dim3(nt, 1, 1);
    cfg.dynamicSmemBytes = poccd_smem<NMAX>(nt);
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    // K42: the 256-thread-CTA clusters (12 / 14 DoF, K15) with the
    // load-balancing scheduling policy (C4 -2.9 %, 12 DoF -1.7 %; at 18 / 24
    // DoF it costs 2.5-5 %, so those keep the default); A/B:
    // HJCD_CLUSTER_POLICY (0 default, 1 spread, 2 load balancing)
    static const int policy = [] {
        const char* v = std::getenv("HJCD_CLUSTER_POLICY");
        return v ? std::atoi(v) : (poccd_cta(NMAX) == 256 ? 2 : 0);
    }();
    attr[1].id = cudaLaunchAttributeClusterSchedulingPolicyPreference;
    attr[1].val.clusterSchedulingPolicyPreference = (cudaClusterSchedulingPolicy)policy;
    cfg.attrs = attr;
    cfg.numAttrs = policy ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, k_poccd<NMAX, EXACT, true, REV>, rb, c, targets, T, seeds, theta, cost, ep, eo,
                              iters, CL, trace, ready);
}

// all-revolute chains (the usual case) run the kernels without per-joint type branches
template <int NMAX, bool EXACT>
cudaError_t launch_poccd_t(const DevRobot& rb, const DevCfg& c, const float* targets, int T,
                           const float* seeds, float* theta, float* cost, float* ep, float* eo,
                           int32_t* iters, TraceOut trace, uint32_t* ready, cudaStream_t s) {
    if (rb.pmask == 0u && rb.rx)
        return launch_poccd_r<NMAX, EXACT, 2>(rb, c, targets, T, seeds, theta, cost, ep, eo, iters, trace, ready, s);
    if (rb.pmask == 0u)
        return launch_poccd_r<NMAX, EXACT, 1>(rb, c, targets, T, seeds, theta, cost, ep, eo, iters, trace, ready, s);
    return launch_poccd_r<NMAX, EXACT, 0>(rb, c, targets, T, seeds, theta, cost, ep, eo, iters, trace, ready, s);
}

}  // namespace hjcd

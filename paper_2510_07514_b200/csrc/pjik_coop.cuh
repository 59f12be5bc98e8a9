#pragma once
// pjik_coop.cuh — k_pjik_coop: PJ-IK (Alg. 4) for one target per CTA
// with the per-target stop rule (Alg. 4 l.18 break; DESIGN.md
// R26b; or, with target_early_exit = 0, a per-seed break) and
// WARP-COOPERATIVE line-search trials (K6).
//
// The B polish seeds of a target advance in lockstep (one thread per seed); the
// CTA votes after each iteration's fine test and stops at the first iteration
// in which any seed converged.  In lockstep, an iteration lasts as long as its
// slowest seed: a seed whose LM step fails runs the whole fallback cascade
// (A further LM trials, a dogleg trial, A+1 single-coordinate trials: up to
// 2A+2 FKs) while the other 31 lanes of its warp idle.  Here every lane first
// evaluates its own LM trial at alpha = 1 (the common case); seeds that fail
// publish theta, their three directions, W, c0 and |rho|^2 to shared memory,
// and ALL 32 lanes of the warp evaluate the pending trials of those seeds in
// parallel.  Each failing seed then takes the FIRST successful trial in cascade
// order (LM alpha_1..alpha_A, dogleg, single alpha_0..alpha_A) — exactly the
// step the sequential cascade takes; extra evaluations have no side effects.
#include <algorithm>

#include "polish.cuh"

namespace hjcd {

// per-seed shared-memory record, structure-of-arrays with stride = blockDim.x
template <class T>
struct CoopSmem {
    T* th;         // [NMAX][nt]
    T* dir;        // [3][NMAX][nt]   LM, dogleg, single-coordinate directions
    T* W;          // [6][nt]
    T* c0;         // [nt]
    T* n0;         // [nt]
    int* flags;    // [nt]  bit0 LM, bit1 dogleg, bit2 single
    unsigned char* own;    // [nt]  rank among the failing seeds -> owner slot
    // [8][nt] u64: byte q of slot o's word q / 8 = cascade position q succeeded
    // (K34: plain byte stores, word-major so each owner reads its words
    // conflict-free; replaces one contended 64-bit atomicOr per success)
    unsigned long long* ok;
};

template <class T, int NMAX>
__device__ __forceinline__ CoopSmem<T> coop_smem(void* base, int nt) {
    CoopSmem<T> s;
    unsigned long long* p64 = (unsigned long long*)base;
    s.ok = p64;
    T* f = (T*)(p64 + 8 * nt);
    s.th = f; f += NMAX * nt;
    s.dir = f; f += 3 * NMAX * nt;
    s.W = f; f += 6 * nt;
    s.c0 = f; f += nt;
    s.n0 = f; f += nt;
    s.flags = (int*)f;
    s.own = (unsigned char*)(s.flags + nt);
    return s;
}

template <class T, int NMAX>
size_t coop_smem_bytes(int nt) {
    return (size_t)nt * (64 + sizeof(T) * (4 * NMAX + 6 + 2) + 4 + 1);
}

// REV: every DoF joint is revolute (no per-joint type branches)
template <class T, int NMAX, bool EXACT, int REV>
__global__ void __launch_bounds__(256)
k_pjik_coop(const __grid_constant__ DevRobotT<T> rb, const __grid_constant__ DevCfg c,
            const float* __restrict__ targets, const float* __restrict__ seeds,
            T* __restrict__ theta_out, T* __restrict__ ep_out, T* __restrict__ eo_out,
            int32_t* __restrict__ counts_out, int32_t* __restrict__ iters_out, const StageLink link) {
    extern __shared__ unsigned long long coop_raw[];
    __shared__ int s_wtot[8];   // per-warp counts of failing seeds (<= 256 threads)
    __shared__ T s_alpha[32];   // line-search steps beta^-a, a = 0..A (A <= 31), by repeated products
    const int nt = blockDim.x;
    const CoopSmem<T> S = coop_smem<T, NMAX>(coop_raw, nt);
    // K19: the fallback directions before the trials at >= 16 DoF and in the
    // fp64 polish (register pressure), and at <= 8 DoF (latency: a slow
    // target's failing seed no longer builds them after its alpha = 1 trial,
    // C2 -1.4 %); at 12-14 DoF the extra work costs the 10k-target C4 more
    // (+13 % k_pjik) than the latency gains
    constexpr bool SPEC_DIRS = NMAX <= 8 || NMAX >= 16 || sizeof(T) == 8;
    // K21: at <= 8 DoF in fp32 the three directions form one straight-line
    // block (branch-free Cholesky and dogleg, unconditional records), so the
    // two 6x6 solves interleave
#ifndef HJCD_NB_DIRS
#define HJCD_NB_DIRS 1
#endif
    constexpr bool NBD = HJCD_NB_DIRS && SPEC_DIRS && NMAX <= 8 && sizeof(T) == 4;
#ifndef HJCD_POLISH_ORDER
#define HJCD_POLISH_ORDER 1
#endif
    const int n = rb.n;
    const int used = c.copies * c.K;
    int t = blockIdx.x;
    const int b = threadIdx.x;
#if HJCD_POLISH_ORDER
    if (link.ready && link.order) {
        // DESIGN K26: this CTA polishes the ready target of the smallest
        // PO-CCD stop iteration, not target blockIdx.x (every PO-CCD CTA is
        // resident or done when this grid starts, and each pushes its target,
        // so the wait is bounded; a stage 1 that cannot complete traps)
        __shared__ int s_t;
        if (b < 32) {
            int got = -1;
            for (unsigned long long spins = 0;; ++spins) {
                got = ready_pop_warp(link.ready, (int)gridDim.x, (int)(blockIdx.x % kReadyShards));
                if (got >= 0) break;
                if (spins > link.spin_limit) __trap();
                __nanosleep(500);
            }
            if (b == 0) s_t = got;
        }
        __syncthreads();
        t = s_t;
    }
#endif
    const int lane = b & 31;
    const bool active = b < used;
    const TargetT<T> tg = load_target<T>(targets + 7ll * t);
    const uint32_t tid = (uint32_t)(c.tid_offset + t);
    const long long row = (long long)t * c.B + b;
    if (b == 0) {
        T al = T(1);
        for (int a = 0; a < 32; ++a) { s_alpha[a] = al; al *= T(c.inv_beta); }
    }   // published by the first __syncthreads_or of the iteration loop

    T th[NMAX], tt[NMAX], dth[NMAX];
    if (link.ready) {
        // DESIGN K10 (hjcd_solve): wait until every CTA of this target's PO-CCD
        // cluster has published its seeds (acquire, gpu scope), then Alg. 2
        // l.2-8 for this target in this CTA: top-K keys sorted in the (not yet
        // used) cascade shared memory, the B x n replicas staged after them
#ifdef HJCD_PROBE
        const int TT = (int)gridDim.x;
        unsigned long long* pr = probe_base(link.ready, TT);
        if (b == 0) pr[2 * TT + t] = probe_now();
#endif
        if (b == 0) {
            const uint32_t* f = link.ready + t;
            uint32_t v;
            for (unsigned long long spins = 0;; ++spins) {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
                if (v >= link.need) break;
                // a stage 1 that cannot complete becomes a CUDA error (the
                // process's context is lost), not a hang: >= ~30 s of polling,
                // scaled with ccd_iters, against ~ms for one PO-CCD cluster
                // (every PO-CCD CTA is already resident when this grid starts)
                if (spins > link.spin_limit) __trap();
                __nanosleep(500);
            }
        }
        __syncthreads();
#ifdef HJCD_PROBE
        if (b == 0) pr[3 * TT + t] = probe_now();
#endif
        sort_stage1_keys(link.cost + (long long)t * c.M, c.M, link.Mpad, coop_raw);
        float* stage = (float*)(coop_raw + link.Mpad);   // [used][NMAX]
        const int nb = (n + 3) / 4;   // one Philox block per 4 joints
#pragma unroll 1
        for (int e = b; e < used * nb; e += nt) {
            const int bb = e / nb, blk = e - bb * nb;
            float v[4];
            replica_block(rb, c, link.theta, coop_raw, t, bb, blk, tid, v);
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (4 * blk + q < n) stage[bb * NMAX + 4 * blk + q] = v[q];
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < NMAX; ++j) th[j] = (active && (EXACT || j < n)) ? T(stage[b * NMAX + j]) : T(0);
        __syncthreads();   // the keys' shared memory becomes the cascade's
    } else {
#pragma unroll
        for (int j = 0; j < NMAX; ++j) th[j] = (active && (EXACT || j < n)) ? T(seeds[row * n + j]) : T(0);
    }

    int cnt[4] = {0, 0, 0, 0};
    vec3<T> Jp[NMAX], Jo[NMAX];
    ResidT<T> r;
    bool live = active;   // per-seed mode: cleared when this seed converges
    int kseed = 0;
    int k;
#ifdef HJCD_PROBE2
    // A/B diagnostic build only: thread 0's cycles per iteration segment
    long long p2_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}, p2_last = clock64();
    int p2_items = 0;
#define P2MARK(i) do { if (b == 0) { const long long nw = clock64(); p2_acc[i] += nw - p2_last; p2_last = nw; } } while (0)
#else
#define P2MARK(i) do {} while (0)
#endif
    for (k = 0;; ++k) {
        vec3<T> pe;
        QuatT<T> qe;
        bool conv = false;
        if (link.trace_theta && live) {   // theta at the start of iteration k (hjcd_pjik_trace)
            float* h = link.trace_theta + (row * (c.lm_iters + 1) + k) * n;
#pragma unroll
            for (int j = 0; j < NMAX; ++j)
                if (EXACT || j < n) h[j] = (float)th[j];
        }
        if (live) {
            fk<NMAX, true, EXACT, false, REV>(rb, th, Jp, Jo, pe, qe);
            r = residual(tg, pe, qe);
            conv = r.ep < T(c.eps_p_fine) && r.eo < T(c.eps_o_fine);   // Alg. 4 l.18 (R26)
        }
        if (c.target_early_exit) {
            if (__syncthreads_or(conv)) break;                  // R26b: target stops
        } else {
            // per-seed break: a converged seed freezes (and keeps helping its
            // warp evaluate trials); the CTA runs while any seed is live
            if (conv) { live = false; kseed = k; }
            if (!__syncthreads_or(live)) break;
        }
        P2MARK(0);
        if (k == c.lm_iters) break;

        bool need = false, have_lm = false, accepted = false;
        int flags = 0, ist = 0;
        uint32_t word = 0u;   // hjcd_pjik_trace decision word of this iteration
        T W[6], c0 = T(0);
        if (live) {
            // ---- Eq. 7 Jacobian, W (R17), D (R20), c_W(theta), |rho|^2
#pragma unroll
            for (int j = 0; j < NMAX; ++j) {
                if (EXACT || j < n) {
                    const vec3<T> z = Jo[j];
                    if (REV || rb.j[j].type == HJCD_REVOLUTE) {
                        Jp[j] = cross3(z, pe - Jp[j]);
                    } else {
                        Jp[j] = z;
                        Jo[j] = mk3<T>(T(0), T(0), T(0));
                    }
                }
            }
            T invD[NMAX];
            {
                T rn[6] = {T(0), T(0), T(0), T(0), T(0), T(0)};
#pragma unroll
                for (int j = 0; j < NMAX; ++j) {
                    if (EXACT || j < n) {
                        rn[0] += Jp[j].x * Jp[j].x; rn[1] += Jp[j].y * Jp[j].y; rn[2] += Jp[j].z * Jp[j].z;
                        rn[3] += Jo[j].x * Jo[j].x; rn[4] += Jo[j].y * Jo[j].y; rn[5] += Jo[j].z * Jo[j].z;
                        if constexpr (!SPEC_DIRS)
                            invD[j] = rcp_nr(fmax(dot3(Jp[j], Jp[j]) + dot3(Jo[j], Jo[j]), T(c.d_floor)));
                    }
                }
#pragma unroll
                for (int i = 0; i < 6; ++i) W[i] = T(i < 3 ? c.w_p : c.w_o) * rcp_nr(T(1) + sqrt(rn[i]));
            }
            c0 = cost_w(W, r.rho);
            have_lm = lm_direction<NMAX, EXACT, SPEC_DIRS, NBD>(rb, c, Jp, Jo, invD, W, r.rho, dth);
            // theta and the LM direction into this seed's record: the alpha = 1
            // trial reads them from there (K19), and so does the cooperative
            // cascade if that trial fails
#pragma unroll
            for (int j = 0; j < NMAX; ++j) {
                S.th[j * nt + b] = th[j];
                S.dir[(0 * NMAX + j) * nt + b] = dth[j];
            }
            if constexpr (SPEC_DIRS) {
                // K19, high DoF: the fallback directions now, while the
                // Jacobian is live, so that it is dead during the trials (6n
                // registers: no spills at 18 / 24 DoF); seeds whose alpha = 1
                // trial then succeeds did this work in vain
                flags = have_lm ? 1 : 0;
                if constexpr (NBD) {
                    // records written whatever the flags say: holes are skipped by flags
                    if (dogleg_direction<NMAX, EXACT, true>(rb, c, Jp, Jo, r.rho, dth, tt)) flags |= 2;   // Eqs. 14-15
#pragma unroll
                    for (int j = 0; j < NMAX; ++j) S.dir[(1 * NMAX + j) * nt + b] = dth[j];
                    if (single_coord_direction<NMAX, EXACT>(rb, c, Jp, Jo, W, r.rho, dth, ist)) flags |= 4;   // Eq. 16
#pragma unroll
                    for (int j = 0; j < NMAX; ++j) S.dir[(2 * NMAX + j) * nt + b] = dth[j];
                } else {
                    if (dogleg_direction<NMAX, EXACT>(rb, c, Jp, Jo, r.rho, dth, tt)) {   // Eqs. 14-15
                        flags |= 2;
#pragma unroll
                        for (int j = 0; j < NMAX; ++j) S.dir[(1 * NMAX + j) * nt + b] = dth[j];
                    }
                    if (single_coord_direction<NMAX, EXACT>(rb, c, Jp, Jo, W, r.rho, dth, ist)) {   // Eq. 16
                        flags |= 4;
#pragma unroll
                        for (int j = 0; j < NMAX; ++j) S.dir[(2 * NMAX + j) * nt + b] = dth[j];
                    }
                }
                // theta back from its record: not held in registers across the directions
#pragma unroll
                for (int j = 0; j < NMAX; ++j) th[j] = S.th[j * nt + b];
            }
        }
        P2MARK(1);

        // ---- trial evaluation, ONE site in two phases (K6).  Phase 0: every
        // live seed evaluates its own LM trial at alpha = 1 (Alg. 4 l.3-9, the
        // common case).  Phase 1, CTA-cooperative: the seeds whose alpha = 1
        // trial failed publish theta, their three directions, W, c0 and |rho|^2;
        // the rest of their cascades (LM alpha_1..alpha_A, dogleg, single
        // alpha_0..alpha_A) is spread over all the CTA's lanes, and each takes
        // the FIRST success in cascade order.
        const bool pending = live && have_lm;
        for (int phase = 0; phase < 2; ++phase) {
            int total = 0;
            if (phase == 1) {
                need = live && !accepted;
                if (need) {
                    T n0 = T(0);
#pragma unroll
                    for (int i = 0; i < 6; ++i) n0 += r.rho[i] * r.rho[i];
                    if constexpr (!SPEC_DIRS) {
                        flags = have_lm ? 1 : 0;   // theta and the LM direction are published already
                        if (dogleg_direction<NMAX, EXACT>(rb, c, Jp, Jo, r.rho, dth, tt)) {   // Eqs. 14-15
                            flags |= 2;
#pragma unroll
                            for (int j = 0; j < NMAX; ++j) S.dir[(1 * NMAX + j) * nt + b] = dth[j];
                        }
                        if (single_coord_direction<NMAX, EXACT>(rb, c, Jp, Jo, W, r.rho, dth, ist)) {   // Eq. 16
                            flags |= 4;
#pragma unroll
                            for (int j = 0; j < NMAX; ++j) S.dir[(2 * NMAX + j) * nt + b] = dth[j];
                        }
                    }
#pragma unroll
                    for (int i = 0; i < 6; ++i) S.W[i * nt + b] = W[i];
                    S.c0[b] = c0;
                    S.n0[b] = n0;
                    S.flags[b] = flags;
                }
                // the failing seeds' cascades as fixed-width item ranges:
                // item (rank, q) = cascade position q < Q = 2A + 2 (LM
                // alpha_1..alpha_A, dogleg, single alpha_0..alpha_A) of the
                // rank-th failing seed; a direction that did not form leaves
                // holes, skipped by the evaluating lane
                const unsigned fail = __ballot_sync(0xffffffffu, need);
                int rank = __popc(fail & ((1u << lane) - 1u));
                if (lane == 0) s_wtot[b >> 5] = __popc(fail);
                for (int w = 0; w < (2 * c.A + 2 + 7) / 8; ++w) S.ok[w * nt + b] = 0ull;
                __syncthreads();
                P2MARK(3);
                int nfail = 0;
                for (int w = 0; w < (nt >> 5); ++w) {
                    const int v = s_wtot[w];
                    if (w < (b >> 5)) rank += v;
                    nfail += v;
                }
                total = nfail * (2 * c.A + 2);
#ifdef HJCD_PROBE2
                p2_items += total;
#endif
                if (total == 0) break;   // uniform over the CTA: no seed failed its alpha = 1 trial
                if (need) S.own[rank] = (unsigned char)b;
                __syncthreads();
                P2MARK(4);
            }
            bool own_ok = false;
            for (int it = b;; it += nt) {
                int o = b, qq = 0, kind = 0, a = 0;
                if (phase == 0) {
                    if (it != b || !pending) break;
                } else {
                    if (it >= total) break;
                    const int rk = it / (2 * c.A + 2);
                    qq = it - rk * (2 * c.A + 2);   // cascade position in the owner's list
                    o = S.own[rk];
                    decode_item(qq, c.A, kind, a);
                    if (!((S.flags[o] >> kind) & 1)) continue;   // that direction did not form
                }
                // clamp(theta + alpha d), joint by joint (alpha = 1 in phase 0: th + 1 * d = th + d exactly)
                const TrialTheta<T> x{rb, S.th + o, S.dir + (kind * NMAX) * nt + o, nt, s_alpha[a]};
                const ResidT<T> rt = eval_at<NMAX, EXACT, REV>(rb, tg, x);
                bool ok;
                if (kind == 1) {   // dogleg: unweighted |rho| (R23)
                    T nt2 = T(0);
#pragma unroll
                    for (int i = 0; i < 6; ++i) nt2 += rt.rho[i] * rt.rho[i];
                    ok = nt2 < S.n0[o];
                } else {           // Eq. 13 with W frozen at theta (R22)
                    T sw = T(0);
#pragma unroll
                    for (int i = 0; i < 6; ++i) {
                        const T wr = (phase == 0 ? W[i] : S.W[i * nt + o]) * rt.rho[i];
                        sw += wr * wr;
                    }
                    ok = T(0.5) * sw < (phase == 0 ? c0 : S.c0[o]);
                }
                if (phase == 0) {
                    own_ok = ok;
                } else if (ok) {
                    ((unsigned char*)(S.ok + (qq >> 3) * nt + o))[qq & 7] = 1;
                }
            }
            if (phase == 0) {
                P2MARK(2);
                if (own_ok) {   // the LM step at alpha = 1 is accepted: the trial point
                    accepted = true;
                    cnt[0]++;
                    word = 1u << 15;   // LM step, alpha index 0
#pragma unroll
                    for (int j = 0; j < NMAX; ++j)
                        if (EXACT || j < n)
                            th[j] = clampf(th[j] + (SPEC_DIRS ? S.dir[(0 * NMAX + j) * nt + b] : dth[j]), rb.j[j].lo,
                                           rb.j[j].hi);
                }
                continue;
            }
            __syncthreads();
            P2MARK(5);
            if (need) {
                int qq = -1;   // first success in cascade order
                for (int w = 0; w < (2 * c.A + 2 + 7) / 8; ++w) {
                    const unsigned long long m = S.ok[w * nt + b];
                    if (qq < 0 && m) qq = 8 * w + (__ffsll((long long)m) - 1) / 8;
                }
                if (qq >= 0) {
                    int kind, a;
                    decode_item(qq, c.A, kind, a);
                    const T alpha = s_alpha[a];
#pragma unroll
                    for (int j = 0; j < NMAX; ++j)
                        if (EXACT || j < n)
                            th[j] = clampf(th[j] + alpha * S.dir[(kind * NMAX + j) * nt + b], rb.j[j].lo, rb.j[j].hi);
                    cnt[kind]++;
                    word = (uint32_t)kind | ((uint32_t)a << 2) | (kind == 2 ? (uint32_t)ist << 8 : 0u) | (1u << 15);
                } else {
                    // R25; SFU Box-Muller in fp32 (K5: ~1e-6 relative on a sigma = 0.05 kick)
                    perturb<NMAX, EXACT, true>(rb, c, th, T(c.sigma_lm), tid, (uint32_t)b, P_PJPERT, (uint32_t)k);
                    cnt[3]++;
                    word = 3u | (1u << 15);
                }
            }
        }
        if (link.trace && live) link.trace[row * c.lm_iters + k] = word;
        P2MARK(6);
    }
#undef P2MARK

#ifdef HJCD_PROBE
    if (link.ready && b == 0) probe_base(link.ready, (int)gridDim.x)[4 * gridDim.x + t] = probe_now();
#endif
    if (!active) return;
#pragma unroll
    for (int j = 0; j < NMAX; ++j)
        if (EXACT || j < n) theta_out[row * n + j] = th[j];
    ep_out[row] = r.ep;
    eo_out[row] = r.eo;
    if (counts_out) {
#pragma unroll
        for (int i = 0; i < 4; ++i) counts_out[row * 4 + i] = cnt[i];
    }
    if (iters_out) iters_out[row] = (c.target_early_exit || live) ? k : kseed;
#ifdef HJCD_PROBE2
    if (b == 0 && counts_out) {   // overwrite seeds 0-1's step counts with the segment totals
        for (int i = 0; i < 7; ++i) counts_out[(long long)t * c.B * 4 + i] = (int32_t)(p2_acc[i] >> 4);
        counts_out[(long long)t * c.B * 4 + 7] = p2_items;
    }
#endif
}

// dynamic shared memory limit of k_pjik_coop: 227 KB per CTA minus its static arrays
constexpr size_t kPjikMaxDynSmem = (size_t)226 * 1024;

template <class T, int NMAX, bool EXACT, int REV>
static cudaError_t launch_coop_r(const DevRobotT<T>& rb, const DevCfg& c, const float* targets, int T_,
                                 const float* seeds, T* theta, T* ep, T* eo, int32_t* counts, int32_t* iters,
                                 cudaStream_t s, const StageLink& link) {
    const int used = c.copies * c.K;
    const int block = (used + 31) / 32 * 32;
    size_t smem = coop_smem_bytes<T, NMAX>(block);
    if (link.ready)   // K10 top-K keys + replica staging
        smem = std::max(smem, (size_t)link.Mpad * sizeof(unsigned long long) + (size_t)used * NMAX * sizeof(float));
    // opt in to what this launch needs (the fp64 records at NMAX = 32 exceed the
    // 227 KB per-CTA limit above 160 polish seeds: a clean configuration error)
    if (smem > kPjikMaxDynSmem) return cudaErrorInvalidConfiguration;
    // once per device: opt in to the most any launch of this kernel may use
    // (capped at the per-CTA limit)
    static std::atomic<unsigned long long> attr{0};
    cudaError_t e = once_per_device(attr, [] {
        const size_t mx = std::min(kPjikMaxDynSmem,
                                   std::max(coop_smem_bytes<T, NMAX>(256), (size_t)8192 * sizeof(unsigned long long) +
                                                                               (size_t)256 * NMAX * sizeof(float)));
        return cudaFuncSetAttribute(k_pjik_coop<T, NMAX, EXACT, REV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)mx);
    });
    if (e != cudaSuccess) return e;
    if (!link.ready) {
        k_pjik_coop<T, NMAX, EXACT, REV><<<T_, block, smem, s>>>(rb, c, targets, seeds, theta, ep, eo, counts, iters,
                                                                 link);
        return cudaGetLastError();
    }
    // DESIGN K10: programmatic dependent of the PO-CCD launch before it on `s`
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)T_, 1, 1);
    cfg.blockDim = dim3((unsigned)block, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr1[1];
    attr1[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr1[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr1;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_pjik_coop<T, NMAX, EXACT, REV>, rb, c, targets, seeds, theta, ep, eo, counts,
                              iters, link);
}

// all-revolute chains run the kernel without per-joint type branches
template <class T, int NMAX, bool EXACT>
cudaError_t launch_coop_t(const DevRobotT<T>& rb, const DevCfg& c, const float* targets, int T_,
                          const float* seeds, T* theta, T* ep, T* eo, int32_t* counts, int32_t* iters,
                          cudaStream_t s, const StageLink& link) {
    if (rb.pmask == 0u && rb.rx)
        return launch_coop_r<T, NMAX, EXACT, 2>(rb, c, targets, T_, seeds, theta, ep, eo, counts, iters, s, link);
    if (rb.pmask == 0u)
        return launch_coop_r<T, NMAX, EXACT, 1>(rb, c, targets, T_, seeds, theta, ep, eo, counts, iters, s, link);
    return launch_coop_r<T, NMAX, EXACT, 0>(rb, c, targets, T_, seeds, theta, ep, eo, counts, iters, s, link);
}

}  // namespace hjcd

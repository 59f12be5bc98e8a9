"""Pins of the oracle's step logic (CPU only): the PJ-IK weights W, the
Box-Muller normals, one PO-CCD iteration worked by hand on a planar arm
(both argmins, the same-joint rule, the gamma test and the perturbation),
SPEC's PO-CCD improvement invariant, and SPEC's PJ-IK invariants including the
fallback-cascade order.  Each pin is computed from something other than the
oracle's own formula (closed forms, plane geometry, the Random123 generator
pinned by its known-answer vectors, or oracle units pinned elsewhere)."""
import math

import numpy as np
import pytest

import oracle
from params import params
from paper_2510_07514_b200 import inputs


def wrap(a):
    return (np.asarray(a) + math.pi) % (2 * math.pi) - math.pi


# ---------------------------------------------------------------- W (R17)
def test_weights_closed_form():
    # rows with hand-picked norms (3-4-5, 5-12-13 triangles and unit vectors):
    # W_i = w_i / (1 + |J_row_i|), w = (w_p, w_p, w_p, w_o, w_o, w_o) = (1, 1, 1, .5, .5, .5)
    J = np.zeros((6, 7))
    J[0, :2] = [3, 4]          # |row| = 5    -> 1/6
    J[1, 2] = -2               # |row| = 2    -> 1/3
    # row 2 = 0               # |row| = 0    -> 1
    J[3, 3:7] = [1, -1, 1, -1] # |row| = 2    -> 0.5/3
    J[4, :2] = [5, 12]         # |row| = 13   -> 0.5/14
    J[5, 6] = 0.5              # |row| = 0.5  -> 0.5/1.5
    W = oracle.weights(params(), J)
    exp = np.array([1 / 6, 1 / 3, 1.0, 0.5 / 3, 0.5 / 14, 0.5 / 1.5])
    assert np.allclose(W, exp, rtol=0, atol=1e-15), (W, exp)
    # w_p and w_o enter linearly
    W2 = oracle.weights(params(w_p=2.0, w_o=0.25), J)
    assert np.allclose(W2, exp * np.array([2, 2, 2, 0.5, 0.5, 0.5]), atol=1e-15)


# ---------------------------------------------------------------- Box-Muller (R11, R25, R30)
def _u01(x):
    return ((x >> 9) + 0.5) * 2.0 ** -23


@pytest.mark.parametrize("seed,tid,sid,purpose,it", [(0, 0, 0, 2, 0), (77, 5, 123, 4, 31), (2 ** 40 + 9, 999, 7, 3, 0)])
def test_normals_are_box_muller_of_philox(seed, tid, sid, purpose, it):
    # joint d takes block d // 4 of the Philox4x32-10 stream (counter =
    # (tid, sid, purpose << 24 | it, block), key = (lo32, hi32) of the seed),
    # uniforms u = ((x >> 9) + 0.5) 2^-23 and the Box-Muller pairs (u0, u1),
    # (u2, u3): z = sqrt(-2 ln ua) (cos | sin)(2 pi ub)
    key = [seed & 0xFFFFFFFF, seed >> 32]
    for d in range(10):
        x = oracle.philox([tid, sid, (purpose << 24) | it, d // 4], key)
        u = [_u01(v) for v in x]
        e = d % 4
        ua, ub = u[2 * (e // 2)], u[2 * (e // 2) + 1]
        rr = math.sqrt(-2.0 * math.log(ua))
        z = rr * (math.cos(2 * math.pi * ub) if e % 2 == 0 else math.sin(2 * math.pi * ub))
        assert abs(oracle.normal(seed, tid, sid, purpose, it, d) - z) < 1e-14, d


# ---------------------------------------------------------------- one PO-CCD iteration by hand
def _planar3(limits):
    ch = inputs.planar([0.5, 0.3, 0.2])
    for j, (lo, hi) in zip(ch.joints, limits):
        j.lo, j.hi = lo, hi
    return ch, np.array([0.5, 0.3, 0.2])


def _planar_frames(L, th):
    c = np.cumsum(th)
    P = [np.zeros(2)]
    for i in range(len(L) - 1):
        P.append(P[-1] + L[i] * np.array([math.cos(c[i]), math.sin(c[i])]))
    pee = P[-1] + L[-1] * np.array([math.cos(c[-1]), math.sin(c[-1])])
    return P, pee, c[-1]


def _rot2(v, a):
    return np.array([math.cos(a) * v[0] - math.sin(a) * v[1], math.sin(a) * v[0] + math.cos(a) * v[1]])


def test_poccd_iteration_by_hand_planar():
    """Alg. 3 l.6-13 on a planar 3-link arm with an SE(2) target,
    from plane geometry only:
      * position candidate of joint j: the angle from (P_ee - P_j) to (P_t - P_j)
        (Eqs. 8-9), clamped into the limits (R7); its score is the distance
        after rotating the end effector about P_j by the clamped step;
      * orientation candidate: the yaw error e = wrap(psi_t - psi) gives
        phi = |e|, a = sign(e) z, so Eq. 11's step is delta(0) e; its score is
        |wrap(e - step_eff)| (R6);
      * argmins with ties to the lower joint; the same joint -> the larger
        |step|, tie -> position (R8); otherwise both applied (R9);
      * accept iff |r_p| or |omega| falls by more than gamma (R10), else
        theta + sigma N(0, 1) per joint from the pinned Box-Muller normals (R11).
    The oracle's recorded decisions and its theta after one iteration must
    match on every decisive instance; every path must occur."""
    rng = np.random.default_rng(2024)
    limits = [(-0.6, 0.4), (-1.4, 1.5), (-2.5, 2.2)]
    ch, L = _planar3(limits)
    lo = np.array([a for a, _ in limits])
    hi = np.array([b for _, b in limits])
    seen = dict(same_p=0, same_o=0, both=0, accept=0, reject=0)
    decisive = 0
    for inst in range(800):
        th = lo + (hi - lo) * rng.random(3)
        # target: the FK of another configuration (reachable), a random yaw offset
        th_t = lo + (hi - lo) * rng.random(3)
        _, pt, _ = _planar_frames(L, th_t)
        psi_t = wrap(rng.uniform(-math.pi, math.pi))
        gamma = float(rng.choice([1e-6, 0.05, 0.2, 5.0]))
        delta0 = float(rng.choice([1.0, 0.6]))
        tgt = np.array([pt[0], pt[1], 0.0, math.cos(psi_t / 2), 0.0, 0.0, math.sin(psi_t / 2)], np.float32)
        pt = tgt[:2].astype(np.float64)
        psi_t = 2 * math.atan2(float(tgt[6]), float(tgt[3]))
        p = params(M=1, ccd_iters=1, ccd_early_exit=0, gamma=gamma, delta0=delta0, eps_p_coarse=1e-12,
                   eps_o_coarse=1e-12, rng_seed=inst, tau_deg=1e-9)
        r = oracle.po_ccd(ch, p, tgt[None], seeds=th.reshape(1, 3, 1), trace=True, tid_offset=inst)
        w = int(r["trace"][0, 0, 0])
        # ---- by hand
        P, pee, psi = _planar_frames(L, th)
        e = float(wrap(psi_t - psi))
        dp, sp, do, so = np.zeros(3), np.zeros(3), np.zeros(3), np.zeros(3)
        for j in range(3):
            u, v = pee - P[j], pt - P[j]
            step = float(wrap(math.atan2(v[1], v[0]) - math.atan2(u[1], u[0])))
            dp[j] = min(max(th[j] + step, lo[j]), hi[j]) - th[j]
            sp[j] = np.linalg.norm(P[j] + _rot2(u, dp[j]) - pt)
            do[j] = min(max(th[j] + delta0 * e, lo[j]), hi[j]) - th[j]
            so[j] = abs(float(wrap(e - do[j])))
        jp, jo = int(np.argmin(sp)), int(np.argmin(so))
        sps, sos = np.sort(sp), np.sort(so)
        if sps[1] - sps[0] < 1e-9 or sos[1] - sos[0] < 1e-9 or abs(abs(e) - math.pi) < 1e-6:
            continue   # a near-tie: both choices are valid readings
        decisive += 1
        assert (w & 31) == jp and ((w >> 5) & 31) == jo, (inst, w, jp, jo, sp, so)
        thh = th.copy()
        if jp == jo:
            take_p = abs(dp[jp]) >= abs(do[jo])
            assert ((w >> 10) & 1) == (0 if take_p else 1), inst
            if take_p:
                thh[jp] += dp[jp]; seen["same_p"] += 1
            else:
                thh[jo] += do[jo]; seen["same_o"] += 1
        else:
            thh[jp] += dp[jp]
            thh[jo] += do[jo]
            seen["both"] += 1
        _, pee2, psi2 = _planar_frames(L, thh)
        ep0, eo0 = np.linalg.norm(pt - pee), abs(e)
        ep1, eo1 = np.linalg.norm(pt - pee2), abs(float(wrap(psi_t - psi2)))
        imp = max(ep0 - ep1, eo0 - eo1)
        if abs(imp - gamma) < 1e-9:
            continue
        accept = imp > gamma
        assert ((w >> 11) & 1) == int(accept), (inst, imp, gamma)
        if accept:
            exp = thh
            seen["accept"] += 1
        else:
            g = np.array([oracle.normal(inst, inst, 0, oracle.PURPOSE_PERTURB, 0, d) for d in range(3)])
            exp = np.clip(th + p["sigma_ccd"] * g, lo, hi)
            seen["reject"] += 1
        assert np.abs(r["theta"][0, :, 0] - exp).max() < 1e-12, (inst, r["theta"][0, :, 0], exp)
    assert decisive >= 300, decisive
    assert min(seen.values()) >= 10, seen


# ---------------------------------------------------------------- SPEC S:237 invariant
@pytest.mark.parametrize("name,gamma", [("panda", 1e-6), ("panda", 2e-3), ("fetch", 1e-6), ("fetch", 2e-3)])
def test_poccd_accepted_updates_improve_by_gamma(name, gamma):
    """SPEC S:237 (Alg. 3 l.11, R10): whenever the greedy branch is taken,
    |r_p| or |omega| falls by more than gamma relative to the pre-update
    residual; otherwise the step is a perturbation (Alg. 3 l.13).  Checked on
    every seed-iteration of 32 one-iteration rounds (>= 1000 with both
    outcomes present); theta stays inside the limits throughout."""
    ch = inputs.robot(name)
    lo, hi = ch.limits()
    Tn, M = 4, 64
    tg = oracle.fk(ch, inputs.halton_configs(ch, Tn, start=3)).astype(np.float32)
    th = np.stack([inputs.uniform_configs(ch, M, seed=100 + t).T for t in range(Tn)])   # [T, n, M]
    p = params(M=M, ccd_iters=1, ccd_early_exit=0, gamma=gamma, eps_p_coarse=1e-9, eps_o_coarse=1e-9)
    r0 = oracle.po_ccd(ch, dict(p, ccd_iters=0), tg, seeds=th)
    ep, eo = r0["ep"], r0["eo"]
    n_acc = n_rej = 0
    for rnd in range(32):
        r = oracle.po_ccd(ch, dict(p, rng_seed=rnd), tg, seeds=th, trace=True)
        acc = (r["trace"][:, :, 0] >> 11) & 1
        moved = r["iters"] == 1
        improved = ((ep - r["ep"]) > gamma) | ((eo - r["eo"]) > gamma)
        assert np.all(improved[moved & (acc == 1)])
        n_acc += int((moved & (acc == 1)).sum())
        n_rej += int((moved & (acc == 0)).sum())
        assert np.all(r["theta"] >= lo[None, :, None]) and np.all(r["theta"] <= hi[None, :, None])
        th, ep, eo = r["theta"], r["ep"], r["eo"]
    assert n_acc + n_rej >= 1000 and n_acc >= 50 and n_rej >= 50, (n_acc, n_rej)


# ---------------------------------------------------------------- SPEC S:334-338 PJ-IK invariants
def _rho(ch, tg, th):
    pose = oracle.fk(ch, th)
    om = np.array([oracle.quat_error(tg[3:].astype(np.float64), q[3:]) for q in pose])
    return np.concatenate([pose[:, :3] - tg[None, :3].astype(np.float64), -om], axis=1)


def _w_closed(J, w_p=1.0, w_o=0.5):
    return np.array([w_p] * 3 + [w_o] * 3) / (1.0 + np.linalg.norm(J, axis=1))


@pytest.mark.parametrize("name", ["panda", "fetch", "panda_x14"])
def test_pjik_step_invariants(name):
    """SPEC S:334-338 (Alg. 4, R21-R25) on every polish step of 24
    one-iteration rounds from far seeds (sigma = 1 rad around Halton answers,
    so all four branches occur):
      * monotone acceptance: an accepted LM / single-coordinate step lowers
        c_W = 1/2 |W rho|^2 with W frozen at the pre-step theta (computed here
        from the closed form of W and the oracle's pinned FK / Jacobian /
        quaternion error); an accepted dogleg step lowers the unweighted |rho|;
      * trust region: |dtheta|_inf <= R (LM, single) and |dtheta|_2 <= R + 1e-9
        (dogleg); a single-coordinate step moves one joint;
      * limits at every iteration boundary;
      * cascade order (Alg. 4 l.3-17): the recorded alpha index of an LM step is
        the first reducing one (oracle.line_search, pinned by brute force); a
        dogleg or single step happens only when no LM trial reduces c_W; a
        single step only when the dogleg trial (oracle.dogleg_step, pinned by
        its interior/boundary cases) does not reduce |rho|; a perturbation
        only when none of the three does;
      * convergence-flag soundness: a seed reported converged has |r_p| < eps_f
        and |omega| < upsilon_f recomputed from its returned theta."""
    ch = inputs.robot(name)
    lo, hi = ch.limits()
    Tn, B = 8, 32
    th0 = inputs.halton_configs(ch, Tn, start=5)
    tg = oracle.fk(ch, th0).astype(np.float32)
    th = inputs.near_configs(ch, np.repeat(th0[:, None, :], B, 1), 1.0, seed=13)
    p = params(B=B, K=B, lm_iters=1, target_early_exit=0)
    R = p["R"]
    seen = np.zeros(4, dtype=int)
    n_conv = 0
    for rnd in range(24):
        r = oracle.pj_ik(ch, dict(p, rng_seed=rnd), tg, th, trace=True)
        kind, a_idx, ist, valid = oracle.pj_word_fields(r["trace"][:, :, 0])
        assert np.all(r["theta"] >= lo) and np.all(r["theta"] <= hi)
        for t in range(Tn):
            conv = r["iters"][t] == 0
            if conv.any():   # converged at the check: recompute the errors from scratch
                rho = _rho(ch, tg[t], th[t][conv])
                assert np.all(np.linalg.norm(rho[:, :3], axis=1) < p["eps_p_fine"])
                assert np.all(np.linalg.norm(rho[:, 3:], axis=1) < p["eps_o_fine"])
                assert np.array_equal(r["theta"][t][conv], th[t][conv])
                n_conv += int(conv.sum())
            for b in np.nonzero(~conv)[0]:
                assert valid[t, b] == 1
                k = int(kind[t, b])
                seen[k] += 1
                x0, x1 = th[t, b], r["theta"][t, b]
                _, J = oracle.fk(ch, x0[None], jac=True)
                W = _w_closed(J[0])
                r0, r1 = _rho(ch, tg[t], np.stack([x0, x1]))
                c0, c1 = 0.5 * np.sum((W * r0) ** 2), 0.5 * np.sum((W * r1) ** 2)
                d = x1 - x0
                # LM direction and its line search through the pinned units
                dlm = oracle.lm_step(p, J[0], W, r0)
                a_lm = -1 if dlm is None else oracle.line_search(ch, p, tg[t], x0, np.clip(dlm, -R, R))
                if k == oracle.PJ_LM:
                    assert c1 < c0 and np.abs(d).max() <= R + 1e-15
                    assert a_lm == a_idx[t, b]
                    continue
                assert a_lm == -1, (t, b, k, a_lm)
                ddl = oracle.dogleg_step(p, J[0], r0)
                dl_ok = False
                if ddl is not None:
                    rt = _rho(ch, tg[t], np.clip(x0 + ddl, lo, hi)[None])[0]
                    dl_ok = np.linalg.norm(rt) < np.linalg.norm(r0)
                if k == oracle.PJ_DOGLEG:
                    assert dl_ok and np.linalg.norm(r1) < np.linalg.norm(r0)
                    assert np.linalg.norm(d) <= R + 1e-9
                    continue
                assert not dl_ok
                i_sc, dsc = oracle.single_coord_step(p, J[0], W, r0)
                a_sc = -1 if i_sc < 0 else oracle.line_search(ch, p, tg[t], x0, dsc)
                if k == oracle.PJ_SINGLE:
                    assert c1 < c0 and np.abs(d).max() <= R + 1e-15
                    assert i_sc == ist[t, b] and a_sc == a_idx[t, b]
                    assert np.count_nonzero(d) == 1 and d[i_sc] != 0
                    continue
                assert a_sc == -1   # perturbation: every branch failed
        th = r["theta"]
    assert seen.sum() >= 1000 and seen.min() >= 5 and n_conv > 0, (seen, n_conv)


# ---------------------------------------------------------------- PJ-IK decision replay (the GPU harness)
def test_pjik_replay_of_own_decisions_is_exact():
    """oracle.pj_ik_replay (the harness of the GPU PJ-IK decision replay):
    replaying the oracle's own decision words reproduces its run bit for bit
    with zero gaps in both stop-rule modes; a forced later alpha, a forced
    fallback branch where LM succeeds, or an invalid word shows up as a
    positive gap."""
    ch = inputs.panda()
    Tn, B = 6, 24
    th0 = inputs.halton_configs(ch, Tn, start=30)
    tg = oracle.fk(ch, th0).astype(np.float32)
    seeds = inputs.near_configs(ch, np.repeat(th0[:, None, :], B, 1), 1.0, seed=21)
    for early in (0, 1):
        p = params(B=B, K=8, lm_iters=48, target_early_exit=early)
        ref = oracle.pj_ik(ch, p, tg, seeds, trace=True)
        rep = oracle.pj_ik_replay(ch, p, tg, seeds, ref["trace"], ref["iters"])
        assert np.array_equal(rep["theta"], ref["theta"])
        assert np.array_equal(rep["ep"], ref["ep"]) and np.array_equal(rep["counts"], ref["counts"])
        assert rep["gap"].max() == 0.0 and rep["stop_gap"].max() == 0.0
        kind, a, ist, valid = oracle.pj_word_fields(ref["trace"])
        steps = np.arange(p["lm_iters"])[None, None, :] < ref["iters"][..., None]
        assert np.array_equal(valid == 1, steps)
        assert np.array_equal(np.stack([(kind[..., :] == k)[steps.nonzero()].sum() for k in range(4)]),
                              ref["counts"].sum((0, 1)))
    kind, a, ist, valid = oracle.pj_word_fields(ref["trace"])
    # an LM step recorded at alpha index 0 forced to alpha index 3: alpha_0 reduces in fp64
    t, b = np.argwhere((kind[:, :, 0] == oracle.PJ_LM) & (a[:, :, 0] == 0) & (valid[:, :, 0] == 1))[0]
    bad = ref["trace"].copy()
    bad[t, b, 0] = (bad[t, b, 0] & ~np.uint32(31 << 2)) | np.uint32(3 << 2)
    rep = oracle.pj_ik_replay(ch, p, tg, seeds, bad, ref["iters"])
    assert rep["gap"][t, b] > 0 and rep["gap_at"][t, b] == 8 * 0 + 1
    # the same step recorded as a perturbation: every LM trial must fail, alpha_0 did not
    bad = ref["trace"].copy()
    bad[t, b, 0] = (bad[t, b, 0] & ~np.uint32(3)) | np.uint32(oracle.PJ_PERTURB)
    rep = oracle.pj_ik_replay(ch, p, tg, seeds, bad, ref["iters"])
    assert rep["gap"][t, b] > 0
    # an invalid word (no step flag) is an infinite gap
    bad = ref["trace"].copy()
    bad[t, b, 0] = 0
    assert np.isinf(oracle.pj_ik_replay(ch, p, tg, seeds, bad, ref["iters"])["gap"][t, b])

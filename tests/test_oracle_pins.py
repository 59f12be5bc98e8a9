"""Pins of the fp64 oracle against things other than itself: closed forms,
finite differences, scipy's rotation library, brute force, the paper's
special cases and SPEC's worked examples (cited per test).  CPU only."""
import math

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import oracle
from params import params
from paper_2510_07514_b200 import inputs

RNG = np.random.default_rng(1234)


def rotvec_of(q_wxyz):
    return Rotation.from_quat([q_wxyz[1], q_wxyz[2], q_wxyz[3], q_wxyz[0]])


def dh_fk_numpy(theta):
    """Panda FK by the Craig modified-DH product Rx(a) Tx(a) Rz(q) Tz(d) —
    a different formula from the oracle's joint-table product."""
    def rx(a):
        c, s = math.cos(a), math.sin(a)
        return np.array([[1, 0, 0, 0], [0, c, -s, 0], [0, s, c, 0], [0, 0, 0, 1.0]])

    def rz(a):
        c, s = math.cos(a), math.sin(a)
        return np.array([[c, -s, 0, 0], [s, c, 0, 0], [0, 0, 1, 0], [0, 0, 0, 1.0]])

    def tx(a):
        m = np.eye(4); m[0, 3] = a; return m

    def tz(d):
        m = np.eye(4); m[2, 3] = d; return m

    T = np.eye(4)
    for (a, d, al, _, _), q in zip(inputs._PANDA_MDH, theta):
        T = T @ rx(al) @ tx(a) @ rz(q) @ tz(d)
    return T @ tz(0.107)


# ---------------------------------------------------------------- P1 FK
def test_planar2_closed_form():
    # S:107-108; general closed form (L1 c1 + L2 c12, L1 s1 + L2 s12, 0), yaw th1+th2
    ch = inputs.planar([1.0, 1.0])
    pose = oracle.fk(ch, np.array([[0.0, 0.0], [math.pi / 2, 0.0]]))
    assert np.allclose(pose[0, :3], [2, 0, 0], atol=1e-15)
    assert np.allclose(pose[0, 3:], [1, 0, 0, 0], atol=1e-15)
    assert np.allclose(pose[1, :3], [0, 2, 0], atol=1e-15)
    L1, L2 = 0.7, 0.4
    ch = inputs.planar([L1, L2])
    th = RNG.uniform(-3, 3, (50, 2))
    pose = oracle.fk(ch, th)
    x = L1 * np.cos(th[:, 0]) + L2 * np.cos(th.sum(1))
    y = L1 * np.sin(th[:, 0]) + L2 * np.sin(th.sum(1))
    assert np.allclose(pose[:, 0], x, atol=1e-14) and np.allclose(pose[:, 1], y, atol=1e-14)
    yaw = np.array([rotvec_of(p[3:]).as_euler("xyz")[2] for p in pose])
    d = np.angle(np.exp(1j * (yaw - th.sum(1))))
    assert np.abs(d).max() < 1e-12


def test_planar3_closed_form():
    L = [0.5, 0.3, 0.2]
    ch = inputs.planar(L)
    th = RNG.uniform(-3, 3, (50, 3))
    pose = oracle.fk(ch, th)
    c = np.cumsum(th, axis=1)
    x = sum(L[i] * np.cos(c[:, i]) for i in range(3))
    y = sum(L[i] * np.sin(c[:, i]) for i in range(3))
    assert np.allclose(pose[:, 0], x, atol=1e-14) and np.allclose(pose[:, 1], y, atol=1e-14)


def test_panda_zero_config_flange():
    # Panda zero configuration flange at (0.088, 0, 0.926)
    pose = oracle.fk(inputs.panda(), np.zeros((1, 7)))
    assert np.allclose(pose[0, :3], [0.088, 0.0, 0.926], atol=1e-12)


def test_panda_matches_dh_product():
    ch = inputs.panda()
    th = inputs.uniform_configs(ch, 64, seed=5)
    pose = oracle.fk(ch, th)
    for p, t in zip(pose, th):
        T = dh_fk_numpy(t)
        assert np.allclose(p[:3], T[:3, 3], atol=1e-12)
        Rq = rotvec_of(p[3:]).as_matrix()
        assert np.allclose(Rq, T[:3, :3], atol=1e-12)


def test_frames_examples():
    # S:116-118
    one = inputs.planar([1.0])
    _, P, z = oracle.fk(one, np.zeros((1, 1)), frames=True)
    assert np.allclose(P[0, 0], [0, 0, 0]) and np.allclose(z[0, 0], [0, 0, 1])
    two = inputs.planar([1.0, 1.0])
    _, P, z = oracle.fk(two, np.array([[math.pi / 2, 0.0]]), frames=True)
    assert np.allclose(P[0, 1], [0, 1, 0], atol=1e-15)


@pytest.mark.parametrize("name", ["panda", "fetch", "panda_x14"])
def test_rigid_rotation_identity(name):
    # P2: FK(theta + x e_j) = ee rotated about (P_j, z_j) by x (revolute) or
    # translated by x z_j (prismatic): pins every frame P_j, z_j
    ch = inputs.robot(name)
    th = inputs.uniform_configs(ch, 8, seed=7)
    types = [j.type for j in ch.joints if j.type != inputs.FIXED]
    for t in th:
        pose, P, z = oracle.fk(ch, t[None], frames=True)
        for j in range(ch.dof):
            x = 0.3
            t2 = t.copy(); t2[j] += x
            pose2 = oracle.fk(ch, t2[None])[0]
            if types[j] == inputs.REVOLUTE:
                R = Rotation.from_rotvec(x * z[0, j])
                p_exp = P[0, j] + R.apply(pose[0, :3] - P[0, j])
                q_exp = (R * rotvec_of(pose[0, 3:])).as_matrix()
            else:
                p_exp = pose[0, :3] + x * z[0, j]
                q_exp = rotvec_of(pose[0, 3:]).as_matrix()
            assert np.allclose(pose2[:3], p_exp, atol=1e-12)
            assert np.allclose(rotvec_of(pose2[3:]).as_matrix(), q_exp, atol=1e-12)


# ---------------------------------------------------------------- P3 Jacobian
@pytest.mark.parametrize("name", ["panda", "fetch", "panda_x14", "panda_x24"])
def test_jacobian_vs_central_fd(name):
    ch = inputs.robot(name)
    th = inputs.uniform_configs(ch, 6, seed=11)
    h = 1e-6
    for t in th:
        _, J = oracle.fk(ch, t[None], jac=True)
        J = J[0]
        R0 = rotvec_of(oracle.fk(ch, t[None])[0, 3:]).as_matrix()
        for j in range(ch.dof):
            tp, tm = t.copy(), t.copy()
            tp[j] += h; tm[j] -= h
            pp, pm = oracle.fk(ch, tp[None])[0], oracle.fk(ch, tm[None])[0]
            dp = (pp[:3] - pm[:3]) / (2 * h)
            assert np.allclose(J[:3, j], dp, atol=1e-8), (j, J[:3, j], dp)
            # angular: vee(dR R^T)
            dR = (rotvec_of(pp[3:]).as_matrix() - rotvec_of(pm[3:]).as_matrix()) / (2 * h)
            W = dR @ R0.T
            w = np.array([W[2, 1], W[0, 2], W[1, 0]])
            assert np.allclose(J[3:, j], w, atol=1e-7), (j, J[3:, j], w)


def test_jacobian_single_lever():
    # single revolute joint about z at origin, ee at (L, 0, 0) -> [0, L, 0, 0, 0, 1]
    ch = inputs.planar([0.8])
    _, J = oracle.fk(ch, np.zeros((1, 1)), jac=True)
    assert np.allclose(J[0, :, 0], [0, 0.8, 0, 0, 0, 1], atol=1e-15)


# ---------------------------------------------------------------- P4 quaternion error
def test_quat_error_vs_scipy_rotvec():
    for _ in range(300):
        qa = Rotation.random(random_state=RNG.integers(1 << 30))
        qb = Rotation.random(random_state=RNG.integers(1 << 30))
        xa, xb = qa.as_quat(), qb.as_quat()
        qt = np.array([xa[3], *xa[:3]])
        qe = np.array([xb[3], *xb[:3]])
        if RNG.random() < 0.5:
            qe = -qe  # double cover must not matter (R1)
        w = oracle.quat_error(qt, qe)
        ref = (qa * qb.inv()).as_rotvec()
        assert np.allclose(w, ref, atol=1e-9)
        assert np.linalg.norm(w) <= math.pi + 1e-12


def test_quat_error_examples():
    # S:134-136
    I = np.array([1.0, 0, 0, 0])
    z90 = np.array([math.cos(math.pi / 4), 0, 0, math.sin(math.pi / 4)])
    assert np.allclose(oracle.quat_error(I, I), 0)
    assert np.allclose(oracle.quat_error(z90, I), [0, 0, math.pi / 2], atol=1e-15)
    assert np.allclose(oracle.quat_error(-z90, z90), 0, atol=1e-15)


def test_angle_axis_examples_and_roundtrip():
    # S:143-145 (Eq. 10)
    I = np.array([1.0, 0, 0, 0])
    z90 = np.array([math.cos(math.pi / 4), 0, 0, math.sin(math.pi / 4)])
    phi, a = oracle.angle_axis(I, I)
    assert phi == 0
    phi, a = oracle.angle_axis(z90, I)
    assert abs(phi - math.pi / 2) < 1e-12 and np.allclose(a, [0, 0, 1])
    for _ in range(100):
        qa = Rotation.random(random_state=RNG.integers(1 << 30))
        qb = Rotation.random(random_state=RNG.integers(1 << 30))
        xa, xb = qa.as_quat(), qb.as_quat()
        phi, a = oracle.angle_axis(np.array([xa[3], *xa[:3]]), np.array([xb[3], *xb[:3]]))
        back = Rotation.from_rotvec(phi * a) * qb
        assert np.allclose(back.as_matrix(), qa.as_matrix(), atol=1e-7)


# ---------------------------------------------------------------- P5 CCD steps
def test_ccd_position_step_examples():
    # S:197-199
    z = [0, 0, 1]
    assert abs(oracle.ccd_position_step([0, 0, 0], z, [1, 0, 0], [0, 1, 0]) - math.pi / 2) < 1e-12
    assert oracle.ccd_position_step([0, 0, 0], z, [1, 0, 0], [1, 0, 0]) == 0
    assert oracle.ccd_position_step([0, 0, 0], z, [1, 0, 0], [0, 0, 1]) == 0


def test_ccd_position_step_is_grid_argmin():
    # the step is the 1-D minimiser of |P_ee - P_t| about (P_j, z_j)
    grid = np.linspace(-math.pi, math.pi, 200001)
    for _ in range(50):
        Pj = RNG.normal(size=3)
        z = RNG.normal(size=3); z /= np.linalg.norm(z)
        pee = RNG.normal(size=3)
        pt = RNG.normal(size=3)
        d = oracle.ccd_position_step(Pj, z, pee, pt, 1e-9)
        u = pee - Pj
        rots = Rotation.from_rotvec(np.outer(grid, z))
        dist = np.linalg.norm(Pj + rots.apply(u) - pt, axis=1)
        g = grid[np.argmin(dist)]
        assert abs(np.angle(np.exp(1j * (d - g)))) < 1e-4
        # sign property: rotating by d never increases the distance
        p2 = Pj + Rotation.from_rotvec(d * z).apply(u)
        assert np.linalg.norm(p2 - pt) <= np.linalg.norm(pee - pt) + 1e-12


def test_ccd_orientation_step_examples():
    # S:206-208 with delta(0) = 1
    p = params()
    I = np.array([1.0, 0, 0, 0])
    z90 = np.array([math.cos(math.pi / 4), 0, 0, math.sin(math.pi / 4)])
    assert oracle.ccd_orientation_step(p, I, I, [0, 0, 1], 0) == 0
    assert abs(oracle.ccd_orientation_step(p, z90, I, [0, 0, 1], 0) - math.pi / 2) < 1e-12
    assert oracle.ccd_orientation_step(p, z90, I, [1, 0, 0], 0) == 0
    # delta(k) = max(delta_min, delta0 rho^k) (R5): k = 200 -> floor 0.1
    assert abs(oracle.ccd_orientation_step(p, z90, I, [0, 0, 1], 200) - 0.1 * math.pi / 2) < 1e-12
    assert abs(oracle.ccd_orientation_step(p, z90, I, [0, 0, -1], 10) + 0.98 ** 10 * math.pi / 2) < 1e-12


# ---------------------------------------------------------------- P6 gradient identity
def test_gradient_identity():
    # grad 1/2 |omega|^2 = -J_o^T omega and grad 1/2 |r_p|^2 = -J_p^T r_p
    ch = inputs.panda()
    th = inputs.uniform_configs(ch, 5, seed=3)
    tgt = oracle.fk(ch, inputs.uniform_configs(ch, 5, seed=4))
    h = 1e-6
    for t, g in zip(th, tgt):
        def f(x):
            p = oracle.fk(ch, x[None])[0]
            rp = g[:3] - p[:3]
            om = oracle.quat_error(g[3:], p[3:])
            return 0.5 * rp @ rp, 0.5 * om @ om, rp, om
        _, _, rp, om = f(t)
        _, J = oracle.fk(ch, t[None], jac=True)
        J = J[0]
        for j in range(7):
            tp, tm = t.copy(), t.copy(); tp[j] += h; tm[j] -= h
            fp, fm = f(tp), f(tm)
            assert abs((fp[0] - fm[0]) / (2 * h) - (-J[:3, j] @ rp)) < 1e-7
            assert abs((fp[1] - fm[1]) / (2 * h) - (-J[3:, j] @ om)) < 1e-7


# ---------------------------------------------------------------- P7 LM step
def test_lm_step_one_dof_sign():
    # 1-DoF about z, ee (1,0,0), target (cos .1, sin .1, 0), w_o = 0 -> ~ +0.1
    ch = inputs.planar([1.0])
    _, J = oracle.fk(ch, np.zeros((1, 1)), jac=True)
    rho = np.array([1 - math.cos(0.1), -math.sin(0.1), 0, 0, 0, 0])   # rho = P_ee - P_t (R19)
    d = oracle.lm_step(params(w_o=0.0), J[0], np.array([1, 1, 1, 0, 0, 0.0]), rho)
    assert abs(d[0] - 0.1) < 0.01


def test_lm_step_newton_and_pinv_limits():
    # n = 6, lambda -> 0: Newton step -J^-1 rho; n > 6: the D-weighted minimum-norm
    # step -D^-1/2 pinv(J D^-1/2) rho (numpy SVD)
    W = np.ones(6)
    for n in (6, 7, 14, 24):
        J = RNG.normal(size=(6, n))
        rho = RNG.normal(size=6) * 1e-2
        lam = 1e-12 if n == 6 else 1e-9   # n > 6: J^T J is rank 6, keep cond(H) ~ 1e9
        d = oracle.lm_step(params(lambda_=lam), J, W, rho)
        D = np.maximum((J * J).sum(0), 1e-8)
        S = np.diag(1 / np.sqrt(D))
        ref = -S @ np.linalg.pinv(J @ S) @ rho
        assert np.allclose(d, ref, rtol=0, atol=1e-5 * np.abs(ref).max()), n


def test_lm_step_zero_residual():
    J = RNG.normal(size=(6, 7))
    assert np.allclose(oracle.lm_step(params(), J, np.ones(6), np.zeros(6)), 0)


# ---------------------------------------------------------------- P8 line search
def test_line_search_examples_and_brute_force():
    ch = inputs.planar([1.0])
    p = params(w_o=0.0)
    tgt = np.array([math.cos(0.5), math.sin(0.5), 0, 1, 0, 0, 0], dtype=np.float32)
    # improves at alpha = 1
    assert oracle.line_search(ch, p, tgt, np.array([0.0]), np.array([0.5])) == 0
    # zero step -> no strict decrease
    assert oracle.line_search(ch, p, tgt, np.array([0.0]), np.array([0.0])) == -1
    # uphill at 1, downhill at 1/beta: step 1.6 overshoots to 1.6 (worse), 0.8 better
    assert oracle.line_search(ch, p, tgt, np.array([0.0]), np.array([1.6])) == 1
    # brute force on Panda: first alpha whose weighted cost decreases
    pa = inputs.panda()
    th = inputs.uniform_configs(pa, 10, seed=9)
    tg = oracle.fk(pa, inputs.uniform_configs(pa, 10, seed=10)).astype(np.float32)
    lo, hi = pa.limits()
    for t, g in zip(th, tg):
        d = RNG.normal(size=7) * 0.3
        _, J = oracle.fk(pa, t[None], jac=True)
        W = oracle.weights(params(), J[0])

        def cw(x):
            q = oracle.fk(pa, x[None])[0]
            r = np.concatenate([q[:3] - g[:3], -oracle.quat_error(g[3:].astype(np.float64), q[3:])])
            return 0.5 * np.sum((W * r) ** 2)
        c0 = cw(t)
        exp = -1
        for a in range(9):
            if cw(np.clip(t + 0.5 ** a * d, lo, hi)) < c0:
                exp = a
                break
        assert oracle.line_search(pa, params(), g, t, d) == exp


# ---------------------------------------------------------------- P9 dogleg
def test_dogleg_interior_and_boundary():
    p = params()
    for n in (3, 7, 14):
        J = RNG.normal(size=(6, n))
        rho = RNG.normal(size=6) * 1e-3
        d = oracle.dogleg_step(p, J, rho)
        gn = -J.T @ np.linalg.solve(J @ J.T + 1e-8 * np.eye(6), rho)
        assert np.allclose(d, gn, atol=1e-10)          # interior GN returned exactly
        rho = RNG.normal(size=6) * 10
        d = oracle.dogleg_step(p, J, rho)
        assert abs(np.linalg.norm(d) - p["R"]) < 1e-9  # on the trust boundary
        # descent direction w.r.t. 1/2 |rho|^2 linearised
        assert d @ (J.T @ rho) < 0
    assert oracle.dogleg_step(p, RNG.normal(size=(6, 7)), np.zeros(6)) is None


# ---------------------------------------------------------------- P10 single coordinate
def test_single_coordinate_examples():
    # gradient (0, 3, -1): with J^T W^2 rho = g  (J = [I3; 0], W = 1, rho = (0,3,-1,0,0,0))
    J = np.zeros((6, 3)); J[:3, :3] = np.eye(3)
    W = np.ones(6)
    rho = np.array([0, 3.0, -1, 0, 0, 0])
    i, d = oracle.single_coord_step(params(R=10.0), J, W, rho)
    assert i == 1 and np.allclose(d, [0, -3, 0])
    i, d = oracle.single_coord_step(params(R=1.0), J, W, rho)
    assert i == 1 and np.allclose(d, [0, -1, 0])


# ---------------------------------------------------------------- P11 top-K / replicate
def test_select_replicate_stable_order_and_copies():
    ch = inputs.panda()
    p = params(M=200, K=10, B=35)
    T = 3
    cost = inputs.random_costs(T, 200, seed=2).astype(np.float64)
    theta = np.stack([inputs.uniform_configs(ch, 200, seed=s).T for s in range(T)])
    seeds, kept = oracle.select_replicate(ch, p, cost, theta)
    lo, hi = ch.limits()
    for t in range(T):
        ref = np.argsort(cost[t], kind="stable")[:10]
        assert np.array_equal(kept[t], ref)
        for b in range(30):
            src = theta[t][:, ref[b % 10]]
            if b < 10:
                assert np.array_equal(seeds[t, b], src)          # copy 0 clean (R15)
            else:
                assert not np.array_equal(seeds[t, b], src)
                assert np.all(seeds[t, b] >= lo) and np.all(seeds[t, b] <= hi)
                assert np.abs(seeds[t, b] - src).max() < 0.2
        assert np.isnan(seeds[t, 30:]).all()                     # B not a multiple of K
    s0, _ = oracle.select_replicate(ch, params(M=200, K=10, B=30, sigma_rep=0.0), cost, theta)
    for b in range(30):
        assert np.array_equal(s0[0, b], theta[0][:, kept[0, b % 10]])   # Sigma = 0


# ---------------------------------------------------------------- P12 RNG
def test_philox_kat():
    # Random123 Philox4x32-10 known-answer vectors
    assert oracle.philox([0, 0, 0, 0], [0, 0]) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert oracle.philox([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert oracle.philox([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0]) == \
        [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def test_normals_are_standard():
    g = np.array([oracle.normal(7, t, s, 2, 0, d) for t in range(40) for s in range(50) for d in range(4)])
    assert abs(g.mean()) < 0.03 and abs(g.std() - 1) < 0.03


def test_uniform_seeds_exact_fp32_and_in_limits():
    ch = inputs.panda()
    s = oracle.uniform_seeds(ch, 0, 5, 1000)
    lo, hi = ch.limits()
    assert np.all(s >= lo[:, None]) and np.all(s <= hi[:, None])
    assert np.array_equal(s.astype(np.float32).astype(np.float64), s)
    for j in range(7):   # roughly uniform
        u = (s[j] - lo[j]) / (hi[j] - lo[j])
        assert abs(u.mean() - 0.5) < 0.05


# ---------------------------------------------------------------- P14 PO-CCD special cases
def test_poccd_seeded_on_answer_converges_at_iteration_zero():
    # target = FK(seed 0) -> converged with 0 updates
    ch = inputs.panda()
    p = params(M=4)
    seeds = oracle.uniform_seeds(ch, 0, 0, 4)
    tgt = oracle.fk(ch, seeds[:, 0][None]).astype(np.float32)
    r = oracle.po_ccd(ch, p, tgt)
    assert r["iters"][0, 0] == 0 and r["ep"][0, 0] < 1e-6


def test_poccd_gamma_infinite_is_random_walk():
    # gamma = inf -> every iteration perturbs: theta_{k+1} = clamp(theta_k + sigma N_k)
    ch = inputs.panda()
    p = params(M=3, gamma=1e9, ccd_iters=5, eps_p_coarse=1e-12, eps_o_coarse=1e-12)
    tgt = oracle.fk(ch, inputs.halton_configs(ch, 1)).astype(np.float32)
    r = oracle.po_ccd(ch, p, tgt)
    lo, hi = ch.limits()
    for m in range(3):
        th = oracle.uniform_seeds(ch, 0, 0, 3)[:, m]
        for k in range(5):
            g = np.array([oracle.normal(0, 0, m, oracle.PURPOSE_PERTURB, k, d) for d in range(7)])
            th = np.clip(th + p["sigma_ccd"] * g, lo, hi)
        assert np.allclose(r["theta"][0, :, m], th, atol=1e-15)


def test_poccd_invariants():
    ch = inputs.fetch_like8()
    p = params(M=64, ccd_iters=32, ccd_early_exit=0)
    tgt = oracle.fk(ch, inputs.halton_configs(ch, 2)).astype(np.float32)
    r = oracle.po_ccd(ch, p, tgt)
    lo, hi = ch.limits()
    assert np.all(r["theta"] >= lo[None, :, None]) and np.all(r["theta"] <= hi[None, :, None])
    r2 = oracle.po_ccd(ch, p, tgt)
    assert np.array_equal(r["theta"], r2["theta"])   # determinism
    # recomputed errors match the reported ones
    for t in range(2):
        for m in range(0, 64, 7):
            q = oracle.fk(ch, r["theta"][t, :, m][None])[0]
            assert abs(np.linalg.norm(q[:3] - tgt[t, :3]) - r["ep"][t, m]) < 1e-12
    # more iterations never hurt the best seed much; error falls from the seeds
    r0 = oracle.po_ccd(ch, params(M=64, ccd_iters=0, ccd_early_exit=0), tgt)
    assert np.median(r["ep"]) < np.median(r0["ep"])


def test_poccd_target_early_exit_is_lockstep_truncation():
    # R12b: with ccd_early_exit every seed of a target stops after k*
    # iterations, k* = the first iteration at which any seed passes the coarse
    # test; each seed's state equals its own per-seed trajectory truncated at k*
    for name in ("panda", "fetch"):
        ch = inputs.robot(name)
        M, Tn = 48, 3
        tg = oracle.fk(ch, inputs.halton_configs(ch, Tn)).astype(np.float32)
        free = oracle.po_ccd(ch, params(M=M, ccd_early_exit=0), tg)
        ex = oracle.po_ccd(ch, params(M=M, ccd_early_exit=1), tg)
        for t in range(Tn):
            conv = (free["ep"][t] < 5e-3) & (free["eo"][t] < 5e-2)
            kstar = free["iters"][t][conv].min() if conv.any() else 64
            assert np.all(ex["iters"][t] == kstar)
            trunc = oracle.po_ccd(ch, params(M=M, ccd_early_exit=0, ccd_iters=int(kstar)), tg[t:t + 1],
                                  tid_offset=t)
            assert np.array_equal(trunc["theta"][0], ex["theta"][t])
            assert np.array_equal(trunc["ep"][0], ex["ep"][t])
            if conv.any():
                assert np.any((ex["ep"][t] < 5e-3) & (ex["eo"][t] < 5e-2))


def test_poccd_replay_of_own_decisions_is_exact():
    # decision replay (the GPU parity harness): replaying the oracle's own
    # recorded decisions reproduces its run bit for bit with zero gaps, in both
    # stop-rule modes; a flipped gamma decision or a non-argmin joint shows up
    # as a positive gap and a different trajectory
    ch = inputs.panda()
    tg = oracle.fk(ch, inputs.halton_configs(ch, 3, start=11)).astype(np.float32)
    for early in (0, 1):
        p = params(M=40, ccd_early_exit=early, ccd_iters=20)
        ref = oracle.po_ccd(ch, p, tg, trace=True)
        rep = oracle.po_ccd_replay(ch, p, tg, ref["trace"], ref["iters"])
        assert np.array_equal(rep["theta"], ref["theta"])
        assert np.array_equal(rep["ep"], ref["ep"]) and np.array_equal(rep["eo"], ref["eo"])
        assert rep["gap"].max() == 0.0 and rep["stop_gap"].max() == 0.0
        w = ref["trace"][:, :, 0]
        assert np.all((w & 31) < ch.dof) and np.all(((w >> 5) & 31) < ch.dof)
        assert np.all(w >> 16 == 0) and np.all((w >> 12) & 3 != 3) and np.all((w >> 14) & 3 != 3)
    # flip the first gamma decision of seed (0, 0)
    bad = ref["trace"].copy()
    assert ref["iters"][0, 0] > 0
    bad[0, 0, 0] ^= 1 << 11
    rep = oracle.po_ccd_replay(ch, p, tg, bad, ref["iters"])
    assert rep["gap"][0, 0] > 0 and not np.array_equal(rep["theta"][0, :, 0], ref["theta"][0, :, 0])
    assert rep["gap"][0, 1:].max() == 0.0
    # force a different position joint: it scores worse than the argmin
    bad = ref["trace"].copy()
    bad[0, 1, 0] = (bad[0, 1, 0] & ~np.uint32(31)) | np.uint32(((bad[0, 1, 0] & 31) + 3) % ch.dof)
    rep = oracle.po_ccd_replay(ch, p, tg, bad, ref["iters"])
    assert rep["gap"][0, 1] > 0
    # an out-of-range joint index is reported as an infinite gap
    bad[0, 2, 0] = 31
    assert np.isinf(oracle.po_ccd_replay(ch, p, tg, bad, ref["iters"])["gap"][0, 2])


# ---------------------------------------------------------------- classic CCD (Alg. 1)
def _planar_fk(L1, L2, th):
    x1 = np.array([L1 * math.cos(th[0]), L1 * math.sin(th[0])])
    return x1, x1 + L2 * np.array([math.cos(th[0] + th[1]), math.sin(th[0] + th[1])])


def test_ccd_one_sweep_planar_by_hand():
    # Alg. 1 on a planar 2-link arm (z axes): one sweep = rotate the tip joint so
    # its link points at the target, then the base joint so the (moved) end
    # effector points at the target; angles from plane geometry (atan2 of the
    # joint-to-point vectors), wrapped to (-pi, pi]
    L1, L2 = 0.6, 0.4
    ch = inputs.planar([L1, L2], lo=-math.pi, hi=math.pi)
    th0 = np.array([0.3, -0.4])
    pt = np.array([0.2, 0.7])
    tg = oracle.fk(ch, np.array([[1.1, 0.9]])).astype(np.float32)
    tg[0, :2] = pt
    tg[0, 2] = 0.0
    p = params(M=1, ccd_iters=1, eps_p_coarse=1e-12)
    r = oracle.ccd(ch, p, tg, seeds=th0.reshape(1, 2, 1))
    wrap = lambda a: (a + math.pi) % (2 * math.pi) - math.pi
    th = th0.copy()
    p1, pe = _planar_fk(L1, L2, th)
    th[1] += wrap(math.atan2(*(pt - p1)[::-1]) - math.atan2(*(pe - p1)[::-1]))
    p1, pe = _planar_fk(L1, L2, th)
    th[0] += wrap(math.atan2(pt[1], pt[0]) - math.atan2(pe[1], pe[0]))
    tg64 = tg.astype(np.float64)[0, :2]
    assert np.allclose(tg64, pt, atol=1e-7)
    assert np.abs(r["theta"][0, :, 0] - th).max() < 1e-6, (r["theta"][0, :, 0], th)


def test_ccd_converges_to_closed_form_planar_ik():
    # position-only 2-link planar IK has exactly two solutions (elbow up/down):
    # cos q2 = (|p|^2 - L1^2 - L2^2) / (2 L1 L2), q1 = atan2(p) - atan2(L2 s2, L1 + L2 c2)
    L1, L2 = 0.6, 0.4
    ch = inputs.planar([L1, L2], lo=-math.pi, hi=math.pi)
    tg = oracle.fk(ch, np.array([[0.7, -1.1]])).astype(np.float32)
    pt = tg[0, :2].astype(np.float64)
    c2 = (pt @ pt - L1 ** 2 - L2 ** 2) / (2 * L1 * L2)
    sols = []
    for s2 in (math.sqrt(1 - c2 * c2), -math.sqrt(1 - c2 * c2)):
        q2 = math.atan2(s2, c2)
        q1 = math.atan2(pt[1], pt[0]) - math.atan2(L2 * s2, L1 + L2 * c2)
        sols.append(np.array([q1, q2]))
    # the literal arccos of Eq. 9 cannot resolve steps below ~1.5e-8 rad in
    # fp64 (acos(1 - 2^-53)), so "converged" means |P_ee - P_t| < 1e-7 m here;
    # seeds that hit a +-pi limit may stall elsewhere (CCD is a local method)
    p = params(M=16, ccd_iters=400, eps_p_coarse=1e-7)
    r = oracle.ccd(ch, p, tg)
    wrap = lambda a: (a + math.pi) % (2 * math.pi) - math.pi
    ok = 0
    for m in range(16):
        th = r["theta"][0, :, m]
        if r["ep"][0, m] < 1e-7:
            d = min(np.abs(wrap(th - s)).max() for s in sols)
            assert d < 1e-6, (th, sols)
            ok += 1
    assert ok >= 6, r["ep"]
    # the error never exceeds the seed's (CCD steps are 1-D minimisers)
    r0 = oracle.ccd(ch, params(M=16, ccd_iters=0), tg)
    assert np.all(r["ep"] <= r0["ep"] + 1e-12)


# ---------------------------------------------------------------- MMD (Table III; R36)
def test_mmd_single_points_closed_form():
    # X = {x}, Y = {y}: the one pairwise distance d is the median, so
    # MMD^2 = k(x,x) + k(y,y) - 2 k(x,y) = 2 - 2 exp(-d^2 / (2 d^2)) = 2 - 2 e^{-1/2}
    m2, h = oracle.mmd2(np.array([[0.3, -1.0, 2.0]]), np.array([[1.1, 0.5, -0.2]]))
    assert abs(m2 - (2 - 2 * math.exp(-0.5))) < 1e-15
    assert abs(h - math.sqrt(0.8 ** 2 + 1.5 ** 2 + 2.2 ** 2)) < 1e-15


def test_mmd_identity_symmetry_and_separation():
    rng = np.random.default_rng(5)
    X = rng.normal(size=(20, 7))
    assert abs(oracle.mmd2(X, X)[0]) < 1e-12
    Y = rng.normal(size=(25, 7))
    assert abs(oracle.mmd2(X, Y)[0] - oracle.mmd2(Y, X)[0]) < 1e-12
    # two tight clusters: separated clusters score far above co-located ones.
    # (The median-heuristic bandwidth grows with the separation, so MMD^2 is NOT
    # monotone in it: ~0.82 at 10 sigma-units vs ~1.05 at 1.)
    base = rng.normal(scale=0.1, size=(20, 3))
    vals = [oracle.mmd2(base, base + np.array([sep, 0, 0]) + rng.normal(scale=0.1, size=(20, 3)))[0]
            for sep in (10.0, 5.0, 2.0, 1.0, 0.0)]
    assert min(vals[:-1]) > 0.5 and 0 <= vals[-1] < 0.1, vals


def test_mmd_against_kernel_matrix_form():
    # the same estimator written as 1^T K 1 block means of the (N+N2)^2 Gram matrix
    rng = np.random.default_rng(9)
    X, Y = rng.normal(size=(6, 4)), rng.normal(loc=0.5, size=(9, 4))
    Z = np.concatenate([X, Y])
    D = np.sqrt(((Z[:, None] - Z[None]) ** 2).sum(-1))
    h = np.median(D[np.triu_indices(len(Z), 1)])
    K = np.exp(-D ** 2 / (2 * h * h))
    ref = K[:6, :6].mean() + K[6:, 6:].mean() - 2 * K[:6, 6:].mean()
    m2, hh = oracle.mmd2(X, Y)
    assert abs(m2 - ref) < 1e-13 and abs(hh - h) < 1e-15


def test_select_topn_order():
    p = params(B=7, K=7)
    ep = np.array([[1e-7, 2e-3, 5e-7, 1e-7, np.nan, 3e-3, 9e-7]])
    eo = np.array([[1e-6, 1e-3, 2e-6, 1e-6, 0.0, 1e-3, 1e-6]])
    # converged (ep < 1e-6, eo < 1e-5): slots 0, 2, 3, 6 by c = ep^2 + eo^2/4:
    # 0 and 3 tie (2.6e-13, lower slot first), 6 (1.06e-12), 2 (1.25e-12);
    # then 1 (4.25e-6), 5 (9.25e-6), and the NaN slot 4 last
    assert list(oracle.select_topn(p, ep, eo, 7)[0]) == [0, 3, 6, 2, 1, 5, 4]


# ---------------------------------------------------------------- P15 PJ-IK special cases
def test_pjik_zero_error_fixed_point_and_convergence():
    ch = inputs.panda()
    p = params(B=4, K=2, target_early_exit=0)
    th0 = inputs.halton_configs(ch, 3)
    tgt = oracle.fk(ch, th0).astype(np.float32)
    # seeds on the (fp32-rounded) answer: converged immediately, no steps
    seeds = np.repeat(th0[:, None, :], 4, axis=1)
    r = oracle.pj_ik(ch, p, tgt, seeds)
    assert np.all(r["iters"] == 0) and np.all(r["counts"] == 0)
    # from theta0 + 1e-2 noise: converges, monotone weighted-cost acceptance
    seeds = inputs.near_configs(ch, np.repeat(th0[:, None, :], 4, axis=1), 1e-2, seed=1)
    r = oracle.pj_ik(ch, p, tgt, seeds)
    assert np.all(r["ep"] < p["eps_p_fine"]) and np.all(r["eo"] < p["eps_o_fine"])
    assert np.all(r["iters"] <= 12)


def test_pjik_target_early_exit_is_lockstep_truncation():
    # R26b: with target_early_exit every seed of a target stops after k* iterations,
    # k* = the first iteration at which any seed passes the fine test; each seed's
    # state equals its own per-seed trajectory truncated at k*
    ch = inputs.fetch_like8()
    B = 12
    th0 = inputs.halton_configs(ch, 4)
    tg = oracle.fk(ch, th0).astype(np.float32)
    seeds = inputs.near_configs(ch, np.repeat(th0[:, None, :], B, 1), 0.2, seed=3)
    free = oracle.pj_ik(ch, params(B=B, K=4, target_early_exit=0), tg, seeds)
    ex = oracle.pj_ik(ch, params(B=B, K=4, target_early_exit=1), tg, seeds)
    for t in range(4):
        conv = (free["ep"][t] < 1e-6) & (free["eo"][t] < 1e-5)
        kstar = free["iters"][t][conv].min() if conv.any() else 128
        assert np.all(ex["iters"][t] == kstar)
        trunc = oracle.pj_ik(ch, params(B=B, K=4, target_early_exit=0, lm_iters=int(kstar)), tg[t:t + 1],
                             seeds[t:t + 1], tid_offset=t)
        assert np.array_equal(trunc["theta"][0], ex["theta"][t])
        if conv.any():
            assert np.any((ex["ep"][t] < 1e-6) & (ex["eo"][t] < 1e-5))


# ---------------------------------------------------------------- P16 end to end
def test_planar2_brute_force_grid():
    # SE(3) target of a 2-DoF planar arm: position + yaw make theta unique; the
    # solver must match a dense grid search (1e-3 rad) within grid resolution
    L1, L2 = 0.6, 0.4
    ch = inputs.planar([L1, L2], lo=-math.pi, hi=math.pi)
    p = params(M=32, K=4, B=8)
    truth = np.array([[0.7, -1.1], [-2.0, 2.3], [2.5, 0.4]])
    tg = oracle.fk(ch, truth).astype(np.float32)
    q, pe, oe, st = oracle.solve(ch, p, tg)
    g = np.arange(-math.pi, math.pi, 1e-3)
    A, Bg = np.meshgrid(g, g, indexing="ij")
    for k in range(3):
        x = L1 * np.cos(A) + L2 * np.cos(A + Bg)
        y = L1 * np.sin(A) + L2 * np.sin(A + Bg)
        yaw = np.angle(np.exp(1j * (A + Bg)))
        ty = 2 * math.atan2(tg[k, 6], tg[k, 3])
        cost = (x - tg[k, 0]) ** 2 + (y - tg[k, 1]) ** 2 + np.angle(np.exp(1j * (yaw - ty))) ** 2
        i = np.unravel_index(np.argmin(cost), cost.shape)
        grid_sol = np.array([g[i[0]], g[i[1]]])
        assert st[k] == 0
        assert np.abs(np.angle(np.exp(1j * (q[k] - grid_sol)))).max() < 2e-3


def test_solve_panda_round_trip_and_unreachable():
    ch = inputs.panda()
    p = params(M=200, K=20, B=40)
    tg = oracle.fk(ch, inputs.halton_configs(ch, 4)).astype(np.float32)
    q, pe, oe, st = oracle.solve(ch, p, tg)
    assert np.all(st == 0)
    back = oracle.fk(ch, q)
    assert np.all(np.linalg.norm(back[:, :3] - tg[:, :3], axis=1) < 1e-6)
    # unreachable targets at 2x max reach (S:567 #9): finite best effort, status 2
    far = inputs.unreachable_targets(3, 2 * inputs.max_reach(ch), seed=0)
    q, pe, oe, st = oracle.solve(ch, params(M=32, K=4, B=8, lm_iters=16), far)
    assert np.all(st == 2) and np.all(np.isfinite(pe)) and np.all(np.isfinite(q))
    # invalid quaternion -> status 3
    bad = tg[:1].copy(); bad[0, 3:] = 0
    q, pe, oe, st = oracle.solve(ch, params(M=8, K=2, B=4), bad)
    assert st[0] == 3

"""fp64 CPU oracle for HJCD-IK — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  It loads oracle/liboracle.so (built
from oracle/hjcd_oracle.cpp by ``build()``) through ctypes and shares no code
with the CUDA path (paper_2510_07514_b200/csrc).  Robots arrive as
``paper_2510_07514_b200.inputs.Chain`` joint tables (plain data).

Every function cites the PAPER.md passage it follows; see hjcd_oracle.cpp.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from typing import Dict, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hjcd_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
MAXJ = 64

PURPOSE_INIT, PURPOSE_PERTURB, PURPOSE_REPL, PURPOSE_PJPERT = 1, 2, 3, 4


def build(force: bool = False) -> str:
    """Compile the oracle with g++ (-O2, no fast-math, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fopenmp", "-fPIC", "-shared",
                               "-ffp-contract=off", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


class OracleRobot(C.Structure):
    _fields_ = [("n", C.c_int32), ("type", C.c_int32 * MAXJ),
                ("origin_xyz", (C.c_double * 3) * MAXJ), ("origin_quat", (C.c_double * 4) * MAXJ),
                ("axis", (C.c_double * 3) * MAXJ), ("lo", C.c_double * MAXJ),
                ("hi", C.c_double * MAXJ), ("ee_xyz", C.c_double * 3), ("ee_quat", C.c_double * 4)]


class OracleConfig(C.Structure):
    _fields_ = [("M", C.c_int32), ("K", C.c_int32), ("B", C.c_int32),
                ("ccd_iters", C.c_int32), ("lm_iters", C.c_int32),
                ("eps_p_coarse", C.c_double), ("eps_o_coarse", C.c_double),
                ("eps_p_fine", C.c_double), ("eps_o_fine", C.c_double),
                ("gamma", C.c_double), ("delta0", C.c_double), ("delta_rho", C.c_double),
                ("delta_min", C.c_double), ("sigma_ccd", C.c_double), ("sigma_rep", C.c_double),
                ("sigma_lm", C.c_double), ("lambda_", C.c_double), ("d_floor", C.c_double),
                ("R", C.c_double), ("beta", C.c_double), ("A", C.c_int32),
                ("w_p", C.c_double), ("w_o", C.c_double), ("succ_p", C.c_double),
                ("succ_o", C.c_double), ("tau_deg", C.c_double), ("rng_seed", C.c_uint64),
                ("repl_noise_all", C.c_int32), ("target_early_exit", C.c_int32),
                ("ccd_early_exit", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        d, i32, i64, u32, u64 = C.c_double, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64
        P = C.c_void_p
        _lib.oracle_normal.restype = d
        _lib.oracle_normal.argtypes = [u64, i64, u32, u32, u32, i32]
        _lib.oracle_ccd_position_step.restype = d
        _lib.oracle_ccd_position_step.argtypes = [P, P, P, P, d]
        _lib.oracle_ccd_orientation_step.restype = d
        _lib.oracle_ccd_orientation_step.argtypes = [P, P, P, P, i32]
        _lib.oracle_uniform_seeds.argtypes = [P, u64, i64, i32, P]
        _lib.oracle_fk.argtypes = [P, P, i32, P, P, P, P]
        _lib.oracle_po_ccd.argtypes = [P, P, P, i32, i64, P, P, P, P, P, P, P, P]
        _lib.oracle_ccd.argtypes = [P, P, P, i32, i64, P, P, P, P]
        _lib.oracle_po_ccd_replay.argtypes = [P, P, P, i32, i64, P, P, P, P, P, P, P, P, P, P]
        _lib.oracle_select_replicate.argtypes = [P, P, P, P, i32, i64, P, P]
        _lib.oracle_pj_ik.argtypes = [P, P, P, i32, i64, P, P, P, P, P, P, P, P]
        _lib.oracle_pj_ik_replay.argtypes = [P, P, P, i32, i64, P, P, P, P, P, P, P, P, P, P, P, P]
        _lib.oracle_solve.argtypes = [P, P, P, i32, i64, P, P, P, P]
        _lib.oracle_line_search.argtypes = [P, P, P, P, P]
        _lib.oracle_lm_step.argtypes = [P, P, i32, P, P, P]
        _lib.oracle_dogleg_step.argtypes = [P, P, i32, P, P]
        _lib.oracle_single_coord_step.argtypes = [P, P, i32, P, P, P]
        _lib.oracle_weights.argtypes = [P, P, i32, P]
        _lib.oracle_num_threads.restype = C.c_int
        _lib.oracle_set_num_threads.argtypes = [i32]
        _lib.oracle_set_num_threads.restype = None
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def make_robot(chain) -> OracleRobot:
    r = OracleRobot()
    if len(chain.joints) > MAXJ:
        raise ValueError("too many joints")
    r.n = len(chain.joints)
    for i, j in enumerate(chain.joints):
        r.type[i] = j.type
        for k in range(3):
            r.origin_xyz[i][k] = j.origin_xyz[k]
            r.axis[i][k] = j.axis[k]
        for k in range(4):
            r.origin_quat[i][k] = j.origin_quat[k]
        r.lo[i], r.hi[i] = j.lo, j.hi
    for k in range(3):
        r.ee_xyz[k] = chain.ee_xyz[k]
    for k in range(4):
        r.ee_quat[k] = chain.ee_quat[k]
    return r


def make_config(p: Dict) -> OracleConfig:
    c = OracleConfig()
    for name, _ in OracleConfig._fields_:
        key = "lambda" if name == "lambda_" else name
        setattr(c, name, p[key])
    return c


def _ref(x):
    return C.byref(x)


# ---------------------------------------------------------------- kinematics
def fk(chain, theta: np.ndarray, frames: bool = False, jac: bool = False):
    """Eq. 1 / Eq. 7: theta [N, n] -> pose [N, 7] (px py pz qw qx qy qz, w >= 0),
    optionally frames P, z [N, n, 3] and J [N, 6, n]."""
    r = make_robot(chain)
    th = np.ascontiguousarray(np.atleast_2d(theta), dtype=np.float64)
    N, n = th.shape
    pose = np.empty((N, 7))
    P = np.empty((N, n, 3)) if frames else None
    z = np.empty((N, n, 3)) if frames else None
    J = np.empty((N, 6, n)) if jac else None
    lib().oracle_fk(_ref(r), _p(th), N, _p(pose), _p(P), _p(z), _p(J))
    out = [pose]
    if frames:
        out += [P, z]
    if jac:
        out.append(J)
    return out[0] if len(out) == 1 else tuple(out)


def quat_error(qt, qe) -> np.ndarray:
    """Eq. 5 with the w >= 0 canonicalisation (R1)."""
    a = np.ascontiguousarray(qt, dtype=np.float64)
    b = np.ascontiguousarray(qe, dtype=np.float64)
    o = np.empty(3)
    lib().oracle_quat_error(_p(a), _p(b), _p(o))
    return o


def angle_axis(qt, qe):
    """Eq. 10 (R2)."""
    a = np.ascontiguousarray(qt, dtype=np.float64)
    b = np.ascontiguousarray(qe, dtype=np.float64)
    phi = C.c_double()
    ax = np.empty(3)
    lib().oracle_angle_axis(_p(a), _p(b), C.byref(phi), _p(ax))
    return phi.value, ax


def ccd_position_step(Pj, rj, pee, pt, tau: float = 1e-6) -> float:
    """Eqs. 8-9 (R3, R4)."""
    arr = [np.ascontiguousarray(x, dtype=np.float64) for x in (Pj, rj, pee, pt)]
    return lib().oracle_ccd_position_step(*[_p(x) for x in arr], tau)


def ccd_orientation_step(params: Dict, qt, qe, rj, k: int) -> float:
    """Eq. 11 with delta(k) (R5)."""
    c = make_config(params)
    arr = [np.ascontiguousarray(x, dtype=np.float64) for x in (qt, qe, rj)]
    return lib().oracle_ccd_orientation_step(_ref(c), *[_p(x) for x in arr], k)


def philox(ctr, key):
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    o = (C.c_uint32 * 4)()
    lib().oracle_philox4x32_10(c, k, o)
    return list(o)


def normal(seed: int, tid: int, sid: int, purpose: int, it: int, d: int) -> float:
    return lib().oracle_normal(seed, tid, sid, purpose, it, d)


def uniform_seeds(chain, seed: int, tid: int, M: int) -> np.ndarray:
    """Alg. 3 l.2-3 seeds for target `tid`: [n, M] f64 (fp32-exact values)."""
    r = make_robot(chain)
    out = np.empty((chain.dof, M))
    lib().oracle_uniform_seeds(_ref(r), seed, tid, M, _p(out))
    return out


# ---------------------------------------------------------------- LM units
def weights(params, J):
    c = make_config(params)
    J = np.ascontiguousarray(J, dtype=np.float64)
    W = np.empty(6)
    lib().oracle_weights(_ref(c), _p(J), J.shape[1], _p(W))
    return W


def lm_step(params, J, W, rho):
    c = make_config(params)
    J = np.ascontiguousarray(J, dtype=np.float64)
    W = np.ascontiguousarray(W, dtype=np.float64)
    rho = np.ascontiguousarray(rho, dtype=np.float64)
    out = np.empty(J.shape[1])
    ok = lib().oracle_lm_step(_ref(c), _p(J), J.shape[1], _p(W), _p(rho), _p(out))
    return out if ok else None


def dogleg_step(params, J, rho):
    c = make_config(params)
    J = np.ascontiguousarray(J, dtype=np.float64)
    rho = np.ascontiguousarray(rho, dtype=np.float64)
    out = np.empty(J.shape[1])
    ok = lib().oracle_dogleg_step(_ref(c), _p(J), J.shape[1], _p(rho), _p(out))
    return out if ok else None


def single_coord_step(params, J, W, rho):
    c = make_config(params)
    J = np.ascontiguousarray(J, dtype=np.float64)
    W = np.ascontiguousarray(W, dtype=np.float64)
    rho = np.ascontiguousarray(rho, dtype=np.float64)
    out = np.empty(J.shape[1])
    i = lib().oracle_single_coord_step(_ref(c), _p(J), J.shape[1], _p(W), _p(rho), _p(out))
    return i, out


def line_search(chain, params, target7, theta, dth) -> int:
    r, c = make_robot(chain), make_config(params)
    t = np.ascontiguousarray(target7, dtype=np.float32)
    th = np.ascontiguousarray(theta, dtype=np.float64)
    d = np.ascontiguousarray(dth, dtype=np.float64)
    return lib().oracle_line_search(_ref(r), _ref(c), _p(t), _p(th), _p(d))


# ---------------------------------------------------------------- stages
def po_ccd(chain, params, targets, tid_offset: int = 0, seeds: Optional[np.ndarray] = None,
           trace: bool = False):
    """Alg. 3 for T x M seeds.  Returns dict of theta [T,n,M], cost, ep, eo,
    iters, margin [T,M] (+ trace [T,M,ccd_iters]: its own decision words)."""
    r, c = make_robot(chain), make_config(params)
    tg = np.ascontiguousarray(targets, dtype=np.float32).reshape(-1, 7)
    T, n, M = tg.shape[0], chain.dof, params["M"]
    sd = None if seeds is None else np.ascontiguousarray(seeds, dtype=np.float64)
    out = dict(theta=np.empty((T, n, M)), cost=np.empty((T, M)), ep=np.empty((T, M)),
               eo=np.empty((T, M)), iters=np.empty((T, M), dtype=np.int32),
               margin=np.empty((T, M)))
    if trace:
        out["trace"] = np.zeros((T, M, max(params["ccd_iters"], 1)), dtype=np.uint32)
    lib().oracle_po_ccd(_ref(r), _ref(c), _p(tg), T, tid_offset, _p(sd), _p(out["theta"]),
                        _p(out["cost"]), _p(out["ep"]), _p(out["eo"]), _p(out["iters"]),
                        _p(out["margin"]), _p(out.get("trace")))
    return out


def po_ccd_replay(chain, params, targets, trace, iters, tid_offset: int = 0, theta_hist=None):
    """Alg. 3 in fp64 following recorded decisions (hjcd_poccd_trace words,
    trace [T,M,ccd_iters] uint32, iters [T,M]) -> dict theta [T,n,M], ep, eo,
    gap [T,M] (how much worse any recorded decision is than the fp64 one) and
    stop_gap [T] (how far outside the coarse box the GPU stopped), gap_at [T,M]
    (8 k + kind of the largest gap: 1 jp, 2 jo, 3 same joint, 4 gamma, 5 stop; -1 none).
    theta_hist [T,M,ccd_iters+1,n] f32 (hjcd_poccd_trace history) resynchronises
    every iteration on the GPU's state (each decision also judged at states one
    fp32 ulp away; the smallest gap counts) and adds step_dev [T,M] (largest
    one-step difference, task space: end-effector m / rotation rad),
    step_excess (its excess over 10x the spread of the fp64 steps from the
    ulp-perturbed states) and step_dev_joint (max |dtheta_j|)."""
    r, c = make_robot(chain), make_config(params)
    tg = np.ascontiguousarray(targets, dtype=np.float32).reshape(-1, 7)
    T, n, M = tg.shape[0], chain.dof, params["M"]
    tr = np.ascontiguousarray(trace, dtype=np.uint32).reshape(T, M, params["ccd_iters"])
    it = np.ascontiguousarray(iters, dtype=np.int32).reshape(T, M)
    out = dict(theta=np.empty((T, n, M)), ep=np.empty((T, M)), eo=np.empty((T, M)),
               gap=np.empty((T, M)), stop_gap=np.empty(T), gap_at=np.empty((T, M), dtype=np.int32))
    h = None
    if theta_hist is not None:
        h = np.ascontiguousarray(theta_hist, dtype=np.float32).reshape(T, M, params["ccd_iters"] + 1, n)
        sd = np.zeros((T, M, 3))
    lib().oracle_po_ccd_replay(_ref(r), _ref(c), _p(tg), T, tid_offset, _p(tr), _p(it), _p(out["theta"]),
                               _p(out["ep"]), _p(out["eo"]), _p(out["gap"]), _p(out["stop_gap"]),
                               _p(out["gap_at"]), _p(h), _p(sd if h is not None else None))
    if h is not None:
        out["step_dev"], out["step_excess"], out["step_dev_joint"] = (sd[..., i].copy() for i in range(3))
    return out


def ccd(chain, params, targets, tid_offset: int = 0, seeds: Optional[np.ndarray] = None):
    """Classic CCD (Alg. 1) for T x M seeds -> dict theta [T,n,M], ep, iters [T,M]."""
    r, c = make_robot(chain), make_config(params)
    tg = np.ascontiguousarray(targets, dtype=np.float32).reshape(-1, 7)
    T, n, M = tg.shape[0], chain.dof, params["M"]
    sd = None if seeds is None else np.ascontiguousarray(seeds, dtype=np.float64)
    out = dict(theta=np.empty((T, n, M)), ep=np.empty((T, M)), iters=np.empty((T, M), dtype=np.int32))
    lib().oracle_ccd(_ref(r), _ref(c), _p(tg), T, tid_offset, _p(sd), _p(out["theta"]), _p(out["ep"]),
                     _p(out["iters"]))
    return out


def select_replicate(chain, params, cost, theta, tid_offset: int = 0):
    """Alg. 2 l.2-8: cost [T,M], theta [T,n,M] -> seeds [T,B,n], kept [T,K]."""
    r, c = make_robot(chain), make_config(params)
    cost = np.ascontiguousarray(cost, dtype=np.float64)
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    T = cost.shape[0]
    seeds = np.empty((T, params["B"], chain.dof))
    kept = np.empty((T, params["K"]), dtype=np.int32)
    lib().oracle_select_replicate(_ref(r), _ref(c), _p(cost), _p(theta), T, tid_offset,
                                  _p(seeds), _p(kept))
    return seeds, kept


def pj_ik(chain, params, targets, seeds, tid_offset: int = 0, trace: bool = False):
    """Alg. 4: seeds [T,B,n] -> dict theta [T,B,n], ep, eo, margin, iters [T,B],
    counts [T,B,4] (+ trace [T,B,lm_iters]: its own decision words, pj_word
    format; 0 where no step was taken)."""
    r, c = make_robot(chain), make_config(params)
    tg = np.ascontiguousarray(targets, dtype=np.float32).reshape(-1, 7)
    sd = np.ascontiguousarray(seeds, dtype=np.float64)
    T, B, n = sd.shape
    assert B == params["B"]
    out = dict(theta=np.empty((T, B, n)), ep=np.empty((T, B)), eo=np.empty((T, B)),
               counts=np.empty((T, B, 4), dtype=np.int32), margin=np.empty((T, B)),
               iters=np.empty((T, B), dtype=np.int32))
    if trace:
        out["trace"] = np.zeros((T, B, max(params["lm_iters"], 1)), dtype=np.uint32)
    lib().oracle_pj_ik(_ref(r), _ref(c), _p(tg), T, tid_offset, _p(sd), _p(out["theta"]),
                       _p(out["ep"]), _p(out["eo"]), _p(out["counts"]), _p(out["margin"]),
                       _p(out["iters"]), _p(out.get("trace")))
    return out


# decision word of PJ-IK (hjcd_pjik_trace / the oracle's own trace)
PJ_LM, PJ_DOGLEG, PJ_SINGLE, PJ_PERTURB = 0, 1, 2, 3


def pj_word_fields(w):
    """(kind, alpha index, single-coordinate index, step-taken flag) of decision words."""
    w = np.asarray(w, dtype=np.uint32)
    return w & 3, (w >> 2) & 31, (w >> 8) & 31, (w >> 15) & 1


def pj_ik_replay(chain, params, targets, seeds, trace, iters, tid_offset: int = 0, theta_hist=None):
    """Alg. 4 in fp64 following recorded decisions (hjcd_pjik_trace words,
    trace [T,B,lm_iters] uint32, iters [T,B]) -> dict theta [T,B,n], ep, eo,
    counts [T,B,4], gap [T,B] (how much worse any recorded decision is than the
    fp64 one, residual-norm units), stop_gap [T], gap_at [T,B] (8 k + kind:
    1 LM trial, 2 dogleg, 3 single index, 4 single trial, 5 continued inside the
    fine box, 6 invalid word; -1 none).  theta_hist [T,B,lm_iters+1,n] f32
    (hjcd_pjik_trace history) resynchronises every iteration on the GPU's
    state and adds step_dev, step_excess and step_dev_joint [T,B] as
    po_ccd_replay."""
    r, c = make_robot(chain), make_config(params)
    tg = np.ascontiguousarray(targets, dtype=np.float32).reshape(-1, 7)
    sd = np.ascontiguousarray(seeds, dtype=np.float64)
    T, B, n = sd.shape
    I = params["lm_iters"]
    tr = np.ascontiguousarray(trace, dtype=np.uint32).reshape(T, B, I)
    it = np.ascontiguousarray(iters, dtype=np.int32).reshape(T, B)
    out = dict(theta=np.full((T, B, n), np.nan), ep=np.full((T, B), np.nan), eo=np.full((T, B), np.nan),
               counts=np.zeros((T, B, 4), dtype=np.int32), gap=np.zeros((T, B)), stop_gap=np.empty(T),
               gap_at=np.full((T, B), -1, dtype=np.int32))
    h = None
    if theta_hist is not None:
        h = np.ascontiguousarray(theta_hist, dtype=np.float32).reshape(T, B, I + 1, n)
        dev = np.zeros((T, B, 3))
    lib().oracle_pj_ik_replay(_ref(r), _ref(c), _p(tg), T, tid_offset, _p(sd), _p(tr), _p(it), _p(out["theta"]),
                              _p(out["ep"]), _p(out["eo"]), _p(out["counts"]), _p(out["gap"]),
                              _p(out["stop_gap"]), _p(out["gap_at"]), _p(h), _p(dev if h is not None else None))
    if h is not None:
        out["step_dev"], out["step_excess"], out["step_dev_joint"] = (dev[..., i].copy() for i in range(3))
    return out


def solve(chain, params, targets, tid_offset: int = 0):
    """Alg. 2 end to end: -> q [T,n], pos_err [T], ori_err [T], status [T]."""
    r, c = make_robot(chain), make_config(params)
    tg = np.ascontiguousarray(targets, dtype=np.float32).reshape(-1, 7)
    T, n = tg.shape[0], chain.dof
    q = np.empty((T, n))
    pe, oe = np.empty(T), np.empty(T)
    st = np.empty(T, dtype=np.int32)
    lib().oracle_solve(_ref(r), _ref(c), _p(tg), T, tid_offset, _p(q), _p(pe), _p(oe), _p(st))
    return q, pe, oe, st


def select_topn(params, ep, eo, N: int):
    """Best N of the B polished seeds per target in R27 order (fine-converged
    first, then c = w_p^2 ep^2 + w_o^2 eo^2 (R14), then slot): a stable sort on
    the (tier, cost) key.  ep, eo [T, B] -> idx [T, N]."""
    used = (params["B"] // params["K"]) * params["K"]
    ep = np.asarray(ep, dtype=np.float64)[:, :used]
    eo = np.asarray(eo, dtype=np.float64)[:, :used]
    cost = params["w_p"] ** 2 * ep ** 2 + params["w_o"] ** 2 * eo ** 2
    cost = np.where(cost >= 0, cost, np.inf)
    tier = ~((ep < params["eps_p_fine"]) & (eo < params["eps_o_fine"]))
    out = np.empty((ep.shape[0], N), dtype=np.int64)
    for t in range(ep.shape[0]):
        order = sorted(range(used), key=lambda b: (bool(tier[t, b]), cost[t, b], b))
        out[t] = order[:N]
    return out


def mmd2(X, Y):
    """Maximum mean discrepancy (PAPER §V-C, Table III; R36): biased
    V-statistic of MMD^2 between point sets X [N, d] and Y [N2, d] with the
    Gaussian kernel k(a, b) = exp(-|a - b|^2 / (2 h^2)), h = median of the
    pairwise distances (i < j) over X u Y.  Plain fp64 definition.
    Returns (MMD^2, h)."""
    X = np.asarray(X, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    Z = np.concatenate([X, Y])
    L = len(Z)
    d = [np.linalg.norm(Z[i] - Z[j]) for i in range(L) for j in range(i + 1, L)]
    h = float(np.median(d))

    def k(a, b):
        s = float(np.sum((a - b) ** 2))
        if h > 0:
            return math.exp(-s / (2.0 * h * h))
        return 1.0 if s == 0.0 else 0.0

    kxx = sum(k(a, b) for a in X for b in X) / (len(X) ** 2)
    kyy = sum(k(a, b) for a in Y for b in Y) / (len(Y) ** 2)
    kxy = sum(k(a, b) for a in X for b in Y) / (len(X) * len(Y))
    return kxx + kyy - 2.0 * kxy, h


def num_threads() -> int:
    return lib().oracle_num_threads()


def set_num_threads(k: int) -> None:
    """OpenMP threads of the oracle's loops (results do not depend on it)."""
    lib().oracle_set_num_threads(int(k))

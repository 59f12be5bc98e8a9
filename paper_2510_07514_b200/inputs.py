"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NO arithmetic of the HJCD-IK method (no FK, no residuals, no
solver steps).  It only describes robots as joint tables and produces joint
configurations: the Halton sequence of the paper's evaluation protocol
("sample joint configurations from a Halton Sequence") and
seeded numpy draws.  Target poses are made by whichever FK the caller owns
(the oracle's in tests, the library's ``fk`` in bench.py).

Robot tables (not in the paper; public data):
  * Panda-like 7-DoF: Craig modified DH, T_i = Rx(a_{i-1}) Tx(a_{i-1}) Rz(q_i) Tz(d_i),
    flange at d = 0.107.
  * Fetch-like 8-DoF: prismatic torso + 7 revolute joints (Appendix B).
  * extend(): cyclic replication of the DoF joints before the end effector
    ("adding replicated revolute joints and links"; R34).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

import numpy as np

REVOLUTE, PRISMATIC, FIXED = 0, 1, 2


@dataclass
class Joint:
    type: int
    origin_xyz: Tuple[float, float, float]
    origin_quat: Tuple[float, float, float, float]  # w x y z
    axis: Tuple[float, float, float]
    lo: float = 0.0
    hi: float = 0.0


@dataclass
class Chain:
    name: str
    joints: List[Joint]
    ee_xyz: Tuple[float, float, float] = (0.0, 0.0, 0.0)
    ee_quat: Tuple[float, float, float, float] = (1.0, 0.0, 0.0, 0.0)

    @property
    def dof(self) -> int:
        return sum(1 for j in self.joints if j.type != FIXED)

    def limits(self) -> Tuple[np.ndarray, np.ndarray]:
        lo = np.array([j.lo for j in self.joints if j.type != FIXED], dtype=np.float64)
        hi = np.array([j.hi for j in self.joints if j.type != FIXED], dtype=np.float64)
        return lo, hi


def _rx_quat(alpha: float) -> Tuple[float, float, float, float]:
    return (math.cos(alpha / 2.0), math.sin(alpha / 2.0), 0.0, 0.0)


def _mdh_joint(a: float, d: float, alpha: float, lo: float, hi: float) -> Joint:
    # Rx(alpha) Tx(a) Tz(d): rotation Rx(alpha), translation (a, -d sin alpha, d cos alpha)
    return Joint(REVOLUTE, (a, -d * math.sin(alpha), d * math.cos(alpha)), _rx_quat(alpha),
                 (0.0, 0.0, 1.0), lo, hi)


_PANDA_MDH = [  # a_{i-1}, d_i, alpha_{i-1}, lo, hi
    (0.0, 0.333, 0.0, -2.8973, 2.8973),
    (0.0, 0.0, -math.pi / 2, -1.7628, 1.7628),
    (0.0, 0.316, math.pi / 2, -2.8973, 2.8973),
    (0.0825, 0.0, math.pi / 2, -3.0718, -0.0698),
    (-0.0825, 0.384, -math.pi / 2, -2.8973, 2.8973),
    (0.0, 0.0, math.pi / 2, -0.0175, 3.7525),
    (0.088, 0.0, math.pi / 2, -2.8973, 2.8973),
]


def panda() -> Chain:
    joints = [_mdh_joint(*row) for row in _PANDA_MDH]
    return Chain("panda7", joints, (0.0, 0.0, 0.107), (1.0, 0.0, 0.0, 0.0))


def fetch_like8() -> Chain:
    I = (1.0, 0.0, 0.0, 0.0)
    Z, Y, X = (0.0, 0.0, 1.0), (0.0, 1.0, 0.0), (1.0, 0.0, 0.0)
    pi = math.pi
    joints = [
        Joint(PRISMATIC, (-0.086875, 0.0, 0.37743), I, Z, 0.0, 0.38615),   # torso_lift
        Joint(REVOLUTE, (0.119525, 0.0, 0.34858), I, Z, -1.6056, 1.6056),  # shoulder_pan
        Joint(REVOLUTE, (0.117, 0.0, 0.06), I, Y, -1.221, 1.518),          # shoulder_lift
        Joint(REVOLUTE, (0.219, 0.0, 0.0), I, X, -pi, pi),                 # upperarm_roll
        Joint(REVOLUTE, (0.133, 0.0, 0.0), I, Y, -2.251, 2.251),           # elbow_flex
        Joint(REVOLUTE, (0.197, 0.0, 0.0), I, X, -pi, pi),                 # forearm_roll
        Joint(REVOLUTE, (0.1245, 0.0, 0.0), I, Y, -2.16, 2.16),            # wrist_flex
        Joint(REVOLUTE, (0.1385, 0.0, 0.0), I, X, -pi, pi),                # wrist_roll
    ]
    return Chain("fetch_like8", joints, (0.16645, 0.0, 0.0), I)


def planar(links: Sequence[float], lo: float = -math.pi, hi: float = math.pi) -> Chain:
    """Planar arm: joint 1 at the origin, joint i+1 at +links[i] along x, all axes z,
    end effector links[-1] beyond the last joint."""
    I = (1.0, 0.0, 0.0, 0.0)
    joints = []
    for i in range(len(links)):
        off = (0.0, 0.0, 0.0) if i == 0 else (float(links[i - 1]), 0.0, 0.0)
        joints.append(Joint(REVOLUTE, off, I, (0.0, 0.0, 1.0), lo, hi))
    return Chain(f"planar{len(links)}", joints, (float(links[-1]), 0.0, 0.0), I)


def extend(chain: Chain, target_dof: int) -> Chain:
    """Cyclic replication of the DoF joints (origin, axis, limits) before the
    end effector (R34; SPEC extend_dof).  A trailing run of FIXED
    joints belongs to the end-effector offset, so the replicas go before it."""
    if target_dof < chain.dof:
        raise ValueError("target_dof < dof")
    base = [j for j in chain.joints if j.type != FIXED]
    tail = len(chain.joints)
    while tail > 0 and chain.joints[tail - 1].type == FIXED:
        tail -= 1
    joints = list(chain.joints[:tail])
    i = 0
    while sum(1 for j in joints if j.type != FIXED) < target_dof:
        joints.append(base[i % len(base)])
        i += 1
    joints += chain.joints[tail:]
    return Chain(f"{chain.name}_x{target_dof}", joints, chain.ee_xyz, chain.ee_quat)


def robot(name: str) -> Chain:
    if name in ("panda", "panda7"):
        return panda()
    if name in ("fetch", "fetch_like8"):
        return fetch_like8()
    if name.startswith("panda_x"):
        return extend(panda(), int(name[len("panda_x"):]))
    raise KeyError(name)


# ---------------------------------------------------------------- Halton
_PRIMES = [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53, 59, 61, 67, 71, 73,
           79, 83, 89, 97, 101, 103, 107, 109, 113, 127, 131]


def halton(index: int, base: int) -> float:
    """Radical inverse of `index` (>= 1) in `base` (SPEC bench.halton)."""
    if base < 2:
        raise ValueError("base < 2")
    f, r, i = 1.0, 0.0, int(index)
    while i > 0:
        f /= base
        r += f * (i % base)
        i //= base
    return r


def halton_configs(chain: Chain, count: int, skip: int = 20, start: int = 0) -> np.ndarray:
    """Joint configurations [count, dof] f64: Halton indices skip+1+start ...,
    bases = first dof primes, mapped affinely into the joint limits
    (R31)."""
    lo, hi = chain.limits()
    n = chain.dof
    out = np.empty((count, n), dtype=np.float64)
    for c in range(count):
        idx = skip + 1 + start + c
        for j in range(n):
            out[c, j] = lo[j] + (hi[j] - lo[j]) * halton(idx, _PRIMES[j])
    return out


# ---------------------------------------------------------------- seeded draws
def uniform_configs(chain: Chain, count: int, seed: int) -> np.ndarray:
    lo, hi = chain.limits()
    rng = np.random.default_rng(seed)
    return lo + (hi - lo) * rng.random((count, chain.dof))


def near_configs(chain: Chain, centers: np.ndarray, sigma: float, seed: int) -> np.ndarray:
    """centers + N(0, sigma^2), clipped into the limits (stage-2-like seeds)."""
    lo, hi = chain.limits()
    rng = np.random.default_rng(seed)
    return np.clip(centers + sigma * rng.standard_normal(centers.shape), lo, hi)


def random_costs(T: int, M: int, seed: int, tie_fraction: float = 0.1) -> np.ndarray:
    """f32 [T][M] ranking keys with deliberate exact ties (top-K parity)."""
    rng = np.random.default_rng(seed)
    c = rng.random((T, M)).astype(np.float32)
    ntie = int(tie_fraction * M)
    for t in range(T):
        src = rng.integers(0, M, size=ntie)
        dst = rng.integers(0, M, size=ntie)
        c[t, dst] = c[t, src]
    return c


def unreachable_targets(count: int, radius: float, seed: int) -> np.ndarray:
    """f32 [count][7]: positions on a sphere of `radius`, random unit quaternions."""
    rng = np.random.default_rng(seed)
    p = rng.standard_normal((count, 3))
    p = radius * p / np.linalg.norm(p, axis=1, keepdims=True)
    q = rng.standard_normal((count, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    q[q[:, 0] < 0] *= -1
    return np.concatenate([p, q], axis=1).astype(np.float32)


def max_reach(chain: Chain) -> float:
    """Sum of joint-origin offset lengths + ee offset (+ prismatic travel)."""
    r = float(np.linalg.norm(chain.ee_xyz))
    for j in chain.joints:
        r += float(np.linalg.norm(j.origin_xyz))
        if j.type == PRISMATIC:
            r += max(abs(j.lo), abs(j.hi))
    return r

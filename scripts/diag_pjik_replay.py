"""Diagnose PJ-IK decision-replay gaps (GPU): rerun one test case, and for each
seed whose replay gap exceeds a bound, restart both sides from the oracle's
replayed theta at the offending iteration and compare their single decisions.

    python scripts/diag_pjik_replay.py [robot] [sigma] [Tn]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
from params import params  # noqa: E402
from paper_2510_07514_b200 import hjcd, inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "panda"
sigma = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
Tn = int(sys.argv[3]) if len(sys.argv) > 3 else 32
dev = torch.device("cuda", 0)
ch = inputs.robot(name)
rb = hjcd.Robot(ch)
B = 40
p = params(B=B, K=10, lm_iters=128, target_early_exit=0)
cfg = hjcd.config_from_params(p)
th0 = inputs.halton_configs(ch, Tn, start=200)
tg = oracle.fk(ch, th0).astype(np.float32)
seeds = inputs.near_configs(ch, np.repeat(th0[:, None, :], B, 1), sigma, seed=31).astype(np.float32)
T = lambda x: torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float32, device=dev)  # noqa: E731
out = hjcd.pjik_trace(rb, cfg, T(tg), T(seeds))
tr = out["trace"].cpu().numpy().view(np.uint32)
it = out["iters"].cpu().numpy()
rep = oracle.pj_ik_replay(ch, p, tg, seeds.astype(np.float64), tr, it)
bad = np.argwhere(rep["gap"] > 1e-5)
print(f"{name} sigma={sigma}: {len(bad)} seeds with gap > 1e-5")
for t, b in bad[:8]:
    at = rep["gap_at"][t, b]
    k, kind = at // 8, at % 8
    print(f"\n== target {t} slot {b}: gap {rep['gap'][t, b]:.3g} at k={k} kind={kind}; "
          f"gpu ep {out['ep'][t, b].item():.3g} oracle-replay ep {rep['ep'][t, b]:.3g}")
    w = tr[t, b, max(0, k - 2):k + 3]
    print("   words k-2..k+2:", [tuple(int(x) for x in f) for f in zip(*oracle.pj_word_fields(w)[:3])])
    # the replayed theta at iteration k
    itk = it.copy()
    itk[t, b] = k
    r_k = oracle.pj_ik_replay(ch, p, tg[t:t + 1], seeds[t:t + 1].astype(np.float64), tr[t:t + 1], itk[t:t + 1],
                              tid_offset=t)
    thk = r_k["theta"][0, b]
    # one step from thk on both sides (same RNG ids: target t, slot b, but iteration 0)
    one = dict(p, lm_iters=1)
    s1 = np.repeat(thk[None, None, :], B, 1)
    og = oracle.pj_ik(ch, one, tg[t:t + 1], s1, tid_offset=t, trace=True)
    gg = hjcd.pjik_trace(rb, hjcd.config_from_params(one), T(tg[t:t + 1]), T(s1.astype(np.float32)))
    ow = oracle.pj_word_fields(og["trace"][0, b, 0])
    gw = oracle.pj_word_fields(gg["trace"].cpu().numpy().view(np.uint32)[0, b, 0])
    print(f"   at theta_k: oracle decision {tuple(int(x) for x in ow[:3])} -> ep {og['ep'][0, b]:.4g} eo "
          f"{og['eo'][0, b]:.4g}; gpu decision {tuple(int(x) for x in gw[:3])} -> ep "
          f"{gg['ep'][0, b].item():.4g} eo {gg['eo'][0, b].item():.4g}")
    print(f"   theta_k {np.array2string(thk, precision=5)}")
    _, J = oracle.fk(ch, thk[None], jac=True)
    sv = np.linalg.svd(J[0], compute_uv=False)
    print(f"   sigma(J) {np.array2string(sv, precision=4)}; start ep/eo {r_k['ep'][0, b]:.4g} / {r_k['eo'][0, b]:.4g}")
    lo, hi = ch.limits()
    print(f"   at limits: {np.nonzero((np.abs(thk - lo) < 1e-6) | (np.abs(thk - hi) < 1e-6))[0]}")

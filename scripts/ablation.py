"""the paper's claim that the hybrid beats either stage alone
(P:167), on a C2-like batch (Panda, T targets, M=1000, K=50, B=100):
  hjcd      full Alg. 2 (PO-CCD -> top-K/replicate -> PJ-IK -> best)
  poccd     PO-CCD only (Alg. 3), best of M by the ranking cost (R14)
  ccd       classic position-only CCD (Alg. 1), best of M by position error
  pjik      PJ-IK only (Alg. 4) from B uniform seeds (the PO-CCD Philox seeds)
Success is re-evaluated in fp64 from the returned theta (oracle FK).
  python scripts/ablation.py [T]"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import oracle
from paper_2510_07514_b200 import hjcd, inputs

T = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
chain = inputs.panda()
robot = hjcd.Robot(chain)
dev = torch.device("cuda", 0)
th = inputs.halton_configs(chain, T)
tg_np = oracle.fk(chain, th).astype(np.float32)
targets = torch.from_numpy(tg_np).to(dev)
cfg = hjcd.default_config()
n = robot.dof


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r = fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return r, sorted(ts)[len(ts) // 2]


def report(name, q, ms):
    q = q.detach().cpu().numpy().astype(np.float64)
    pose = oracle.fk(chain, q)
    pe = np.linalg.norm(pose[:, :3] - tg_np[:, :3], axis=1)
    qt = tg_np[:, 3:].astype(np.float64)
    oe = np.array([np.linalg.norm(oracle.quat_error(a / np.linalg.norm(a), b)) for a, b in zip(qt, pose[:, 3:])])
    ok = (pe < 1e-3) & (oe < math.pi / 180)
    print(f"{name:7s} {ms:8.3f} ms  success@1mm/1deg {ok.mean():.4f}  pos err p50 {np.median(pe):.2e} m"
          f"  ori err p50 {np.median(oe):.2e} rad")


def best_of(theta, key):   # theta [T, n, M], key [T, M] -> [T, n]
    i = torch.argmin(key, dim=1)
    return theta.gather(2, i[:, None, None].expand(-1, n, 1))[..., 0]


r, ms = timed(lambda: hjcd.solve(robot, targets, cfg))
report("hjcd", r[0], ms)
r, ms = timed(lambda: hjcd.poccd(robot, cfg, targets))
report("poccd", best_of(r["theta"], r["cost"]), ms)
r, ms = timed(lambda: hjcd.ccd(robot, cfg, targets))
report("ccd", best_of(r["theta"], r["ep"]), ms)
c0 = hjcd.default_config(ccd_iters=0)
seeds = hjcd.poccd(robot, c0, targets)["theta"][:, :, :cfg.B].permute(0, 2, 1).contiguous()   # uniform seeds


def pj_only():
    o = hjcd.pjik(robot, cfg, targets, seeds)
    return o


r, ms = timed(pj_only)
cost = r["ep"] ** 2 + 0.25 * r["eo"] ** 2
report("pjik", r["theta"].gather(1, torch.argmin(cost, 1)[:, None, None].expand(-1, 1, n))[:, 0], ms)

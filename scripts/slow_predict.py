"""Can a target's polish length be predicted from its stage 1?  For C2 (1000
Panda targets) prints, per target, the PO-CCD stop iteration k* and the
stage-1 best cost next to the PJ-IK iteration count, and the ranks of the
slowest polish targets under each predictor."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2510_07514_b200 import hjcd, inputs

dev = torch.device("cuda", 0)
for name in ("panda", "fetch_like8"):
    chain = inputs.robot(name)
    robot = hjcd.Robot(chain)
    T = 1000
    th = torch.from_numpy(inputs.halton_configs(chain, T).astype(np.float32)).to(dev)
    targets = hjcd.fk(robot, th).contiguous()
    cfg = hjcd.default_config()
    o1 = hjcd.poccd(robot, cfg, targets)
    seeds, _ = hjcd.select_replicate(robot, cfg, o1["cost"], o1["theta"])
    o2 = hjcd.pjik(robot, cfg, targets, seeds)
    kst = o1["iters"].reshape(T, -1)[:, 0].cpu().numpy()
    best = o1["cost"].reshape(T, -1).min(1).values.cpu().numpy()
    kp = o2["iters"].reshape(T, -1)[:, 0].cpu().numpy()
    slow = np.argsort(-kp)[:15]
    rk_k = np.argsort(np.argsort(-kst))      # rank 0 = largest k*
    rk_c = np.argsort(np.argsort(-best))     # rank 0 = largest best cost
    print(f"{name}: polish iters p50 {np.median(kp)} p90 {np.percentile(kp, 90)} n128 {(kp >= 128).sum()}; "
          f"corr(k*, iters) {np.corrcoef(kst, kp)[0, 1]:.3f} corr(best cost, iters) {np.corrcoef(best, kp)[0, 1]:.3f}")
    for t in slow:
        print(f"   t {t:4d} polish iters {kp[t]:4d}  k* {kst[t]:3d} (rank {rk_k[t]:4d})  best cost {best[t]:.3e} (rank {rk_c[t]:4d})")

"""Latency of ONE stage-2 target that runs the whole I_l budget (C2 Halton
target 139: near-singular, no seed reaches the fine tolerance), i.e. the
per-iteration latency that bounds k_pjik under the per-target stop rule.
  HJCD_LIB=... python scripts/tail_latency.py"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2510_07514_b200 import hjcd, inputs

chain = inputs.panda()
robot = hjcd.Robot(chain)
dev = torch.device("cuda", 0)
th = torch.from_numpy(inputs.halton_configs(chain, 1000).astype(np.float32)).to(dev)
targets = hjcd.fk(robot, th).contiguous()
cfg = hjcd.default_config()
o1 = hjcd.poccd(robot, cfg, targets)
seeds, _ = hjcd.select_replicate(robot, cfg, o1["cost"], o1["theta"])
o2 = hjcd.pjik(robot, cfg, targets, seeds)
k = o2["iters"][:, 0]
slow = torch.nonzero(k >= cfg.lm_iters).flatten().tolist()
for t in slow[:3]:
    c1 = hjcd.default_config(target_index_offset=t)
    tg, sd = targets[t:t + 1].contiguous(), seeds[t:t + 1].contiguous()
    for _ in range(3):
        hjcd.pjik(robot, c1, tg, sd)
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        o = hjcd.pjik(robot, c1, tg, sd)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    it = int(o["iters"][0, 0])
    print(os.path.basename(hjcd.LIB_PATH), f"target {t}: {ms:.3f} ms, {it} iterations, {1e3 * ms / max(it, 1):.2f} us/iter")

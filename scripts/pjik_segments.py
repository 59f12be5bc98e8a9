"""Per-iteration cycle split of PJ-IK's critical path (thread 0 of a CTA) from
the HJCD_PROBE2 A/B build, for the slowest C2 targets alone and in the batch:
  HJCD_LIB=paper_2510_07514_b200/_ab/libhjcd_probe2.so python scripts/pjik_segments.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2510_07514_b200 import hjcd, inputs

dev = torch.device("cuda", 0)
chain = inputs.panda()
robot = hjcd.Robot(chain)
T = 1000
th = torch.from_numpy(inputs.halton_configs(chain, T).astype(np.float32)).to(dev)
targets = hjcd.fk(robot, th).contiguous()
cfg = hjcd.default_config()
o1 = hjcd.poccd(robot, cfg, targets)
seeds, _ = hjcd.select_replicate(robot, cfg, o1["cost"], o1["theta"])
NAMES = ["fk+vote", "J,W,D,LM", "trial a=1", "publish+dirs", "item table", "cascade evals", "apply"]


def report(tag, counts, iters, t):
    c = counts[t].reshape(-1)[:8].astype(np.float64) * 16
    k = max(1, int(iters[t, 0]))
    tot = c[:7].sum()
    print(f"{tag} t={t} iters={k} cycles/iter={tot / k:8.0f} items/iter={c[7] / k:6.1f}  " +
          " ".join(f"{n}={c[i] / k:6.0f}" for i, n in enumerate(NAMES)), flush=True)


out = hjcd.pjik(robot, cfg, targets, seeds)
torch.cuda.synchronize()
counts, iters = out["counts"].cpu().numpy(), out["iters"].cpu().numpy()
slow = np.argsort(-iters[:, 0])[:6]
fast = np.argsort(iters[:, 0])[500:503]
for t in list(slow) + list(fast):
    report("batch", counts, iters, t)
for t in slow[:4]:
    c1 = hjcd.default_config(target_index_offset=int(t))
    for _ in range(2):
        o = hjcd.pjik(robot, c1, targets[t:t + 1].contiguous(), seeds[t:t + 1].contiguous())
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    o = hjcd.pjik(robot, c1, targets[t:t + 1].contiguous(), seeds[t:t + 1].contiguous())
    b.record()
    torch.cuda.synchronize()
    print(f"alone t={t}: {a.elapsed_time(b):.3f} ms")
    report("alone", o["counts"].cpu().numpy(), o["iters"].cpu().numpy(), 0)

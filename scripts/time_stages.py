"""Per-stage device times of hjcd_solve on a config (library stage events).
  HJCD_LIB=path/to/variant.so python scripts/time_stages.py [c2|c3|c4] [reps]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2510_07514_b200 import hjcd, inputs

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
CFG = {"c2": ("panda", 1000), "c3": ("fetch_like8", 10000), "c4": ("panda_x14", 10000)}
rname, T = CFG[cfgname] if cfgname in CFG else (cfgname, 1000)   # e.g. panda_x12: 1000 targets
chain = inputs.robot(rname)
robot = hjcd.Robot(chain)
dev = torch.device("cuda", 0)
th = torch.from_numpy(inputs.halton_configs(chain, T).astype(np.float32)).to(dev)
targets = hjcd.fk(robot, th).contiguous()
cfg = hjcd.default_config()
ws = hjcd.Workspace()
for _ in range(3):
    hjcd.solve(robot, targets, cfg, workspace=ws)
evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(reps)]
torch.cuda.synchronize()
for r in range(reps):
    out = hjcd.solve(robot, targets, cfg, workspace=ws, events=evs[r])
torch.cuda.synchronize()
names = ("poccd", "select_rep", "pjik", "select_best")
ms = {n: statistics.median(e[i].elapsed_time(e[i + 1]) for e in evs) for i, n in enumerate(names)}
tot = statistics.median(e[0].elapsed_time(e[4]) for e in evs)
succ = float((out[3] <= 1).float().mean())
print(os.path.basename(hjcd.LIB_PATH), cfgname, " ".join(f"{k}={v:.3f}" for k, v in ms.items()),
      f"total={tot:.3f} ms success={succ:.4f}")

"""Run the C2 workload's solve a few times (for ncu launch lists / full captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2510_07514_b200 import hjcd, inputs

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
robots = {"c2": ("panda", 1000), "c3": ("fetch_like8", 10000), "c4": ("panda_x14", 10000)}
rname, T = robots[cfgname]
chain = inputs.robot(rname)
robot = hjcd.Robot(chain)
dev = torch.device("cuda", 0)
th = torch.from_numpy(inputs.halton_configs(chain, T).astype(np.float32)).to(dev)
targets = hjcd.fk(robot, th).contiguous()
cfg = hjcd.default_config()
for _ in range(reps):
    q, pe, oe, st = hjcd.solve(robot, targets, cfg)
torch.cuda.synchronize()
print("success", float((st <= 1).float().mean()))

"""Timeline of hjcd_solve's dependent launch (DESIGN K10) from the HJCD_PROBE
A/B build (%globaltimer stamps per target):
  HJCD_LIB=paper_2510_07514_b200/_ab/libhjcd_probe.so python scripts/k10_probe.py [c2|c3|c4]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2510_07514_b200 import hjcd, inputs

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
CFG = {"c2": ("panda", 1000), "c3": ("fetch_like8", 10000), "c4": ("panda_x14", 10000)}
rname, T = CFG[cfgname]
chain = inputs.robot(rname)
robot = hjcd.Robot(chain)
dev = torch.device("cuda", 0)
th = torch.from_numpy(inputs.halton_configs(chain, T).astype(np.float32)).to(dev)
targets = hjcd.fk(robot, th).contiguous()
cfg = hjcd.default_config()
ws = hjcd.Workspace()
for _ in range(3):
    out = hjcd.solve(robot, targets, cfg, workspace=ws)
torch.cuda.synchronize()
buf = np.zeros(5 * T, dtype=np.uint64)
rc = hjcd.lib().hjcd_debug_probe(buf.ctypes.data_as(C.POINTER(C.c_uint64)), T)
assert rc == 0, rc
p = buf.reshape(5, T).astype(np.float64)
t0 = p[0].min()
us = (p - t0) / 1e3
names = ["poccd_start", "poccd_end", "pjik_start", "pjik_waited", "pjik_end"]
q = [0, 0.1, 0.5, 0.9, 0.99, 1.0]
print(f"{cfgname}: T={T}, times in us from the first PO-CCD CTA start")
for i, nm in enumerate(names):
    print(f"  {nm:12s} " + " ".join(f"q{int(100 * x):3d}={np.quantile(us[i], x):8.1f}" for x in q))
wait = us[3] - us[2]
print(f"  pjik wait    " + " ".join(f"q{int(100 * x):3d}={np.quantile(wait, x):8.1f}" for x in q))
dur = us[4] - us[3]
slow = np.argsort(-dur)[:12]
print("  slowest PJ-IK targets: t, poccd_end, pjik_start, waited, end, duration")
for t in slow:
    print(f"    {t:5d} {us[1, t]:8.1f} {us[2, t]:8.1f} {us[3, t]:8.1f} {us[4, t]:8.1f} {dur[t]:8.1f}")
print(f"  makespan {us[4].max():.1f} us; PO-CCD last end {us[1].max():.1f} us; first PJ-IK start {us[2].min():.1f} us")

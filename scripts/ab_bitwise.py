"""Bitwise comparison of hjcd_solve between two library builds on C1-C4-like
inputs (run once per library, then compare):
  HJCD_LIB=A python scripts/ab_bitwise.py save /tmp/a.npz; HJCD_LIB=B python scripts/ab_bitwise.py cmp /tmp/a.npz"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2510_07514_b200 import hjcd, inputs

dev = torch.device("cuda", 0)
res = {}
for name, T in (("panda", 1000), ("fetch_like8", 300), ("panda_x14", 300), ("panda_x24", 100)):
    ch = inputs.robot(name)
    rb = hjcd.Robot(ch)
    th = torch.from_numpy(inputs.halton_configs(ch, T).astype(np.float32)).to(dev)
    tg = hjcd.fk(rb, th).contiguous()
    q, pe, oe, st = hjcd.solve(rb, tg, hjcd.default_config())
    o1 = hjcd.poccd(rb, hjcd.default_config(), tg[:50].contiguous())
    res[name] = [x.cpu().numpy() for x in (q, pe, oe, st, o1["theta"], o1["cost"], o1["iters"])]
if sys.argv[1] == "save":
    np.savez(sys.argv[2], **{f"{k}_{i}": v for k, vs in res.items() for i, v in enumerate(vs)})
else:
    ref = np.load(sys.argv[2])
    for k, vs in res.items():
        same = [np.array_equal(v, ref[f"{k}_{i}"], equal_nan=True) for i, v in enumerate(vs)]
        print(k, "bitwise equal" if all(same) else f"DIFFER {same}", flush=True)

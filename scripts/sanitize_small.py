"""Small solves through every fused/staged entry point, for compute-sanitizer:
  compute-sanitizer --tool memcheck|racecheck|synccheck python scripts/sanitize_small.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2510_07514_b200 import hjcd, inputs

dev = torch.device("cuda", 0)
for name, M, T in (("panda", 256, 6), ("fetch_like8", 64, 3), ("panda_x14", 200, 2)):
    ch = inputs.robot(name)
    rb = hjcd.Robot(ch)
    th = torch.from_numpy(inputs.halton_configs(ch, T).astype(np.float32)).to(dev)
    tg = hjcd.fk(rb, th, jac=True)[0].contiguous()
    cfg = hjcd.default_config(M=M, K=min(16, M), B=48, lm_iters=24, ccd_iters=24)
    out = hjcd.solve(rb, tg, cfg)                        # K10 dependent launch
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    out2 = hjcd.solve(rb, tg, cfg, events=evs)          # staged
    hjcd.solve_batch(rb, tg, 8, cfg)
    hjcd.solve_f64(rb, tg, cfg)
    hjcd.solve(rb, tg, hjcd.default_config(M=M, K=min(16, M), B=48, lm_iters=24, ccd_iters=24,
                                          ccd_early_exit=0, target_early_exit=0))
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(out, out2)), name
    print(name, "ok", flush=True)

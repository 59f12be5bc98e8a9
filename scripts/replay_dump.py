"""Dump hjcd_poccd_trace outputs for the decision-replay test cases (GPU side)
to gpurun_out/replay_*.npz, for offline analysis with the oracle here."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import oracle  # noqa: E402  (targets only: FK of Halton configs)
from params import params  # noqa: E402
from paper_2510_07514_b200 import hjcd, inputs  # noqa: E402

CASES = [("panda", 1000, 8, 1), ("panda", 300, 4, 0), ("fetch", 131, 8, 1), ("panda_x14", 300, 4, 1),
         ("panda_x24", 257, 3, 0)]
os.makedirs("gpurun_out", exist_ok=True)
for name, M, Tn, early in CASES:
    ch = inputs.robot(name)
    rb = hjcd.Robot(ch)
    p = params(M=M, ccd_early_exit=early, **({} if early else dict(ccd_iters=24)))
    tg = oracle.fk(ch, inputs.halton_configs(ch, Tn, start=90)).astype(np.float32)
    out = hjcd.poccd_trace(rb, hjcd.config_from_params(p), torch.as_tensor(tg, device="cuda"))
    np.savez(f"gpurun_out/replay_{name}_{M}_{early}.npz", tg=tg,
             **{k: v.cpu().numpy() for k, v in out.items()})
    print(name, M, early, "ok")

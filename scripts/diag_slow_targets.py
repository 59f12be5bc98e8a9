"""The C2 polish tail (GPU): which targets run the whole I_l budget, how many
of their seeds fail the alpha = 1 LM trial per iteration in fp32 (and go
through the cooperative cascade), and how long their polish takes alone, in
fp32 and in the fp64 polish.

    python scripts/diag_slow_targets.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_07514_b200 import hjcd, inputs  # noqa: E402

dev = torch.device("cuda", 0)
ch = inputs.panda()
rb = hjcd.Robot(ch)
T = 1000
th = torch.from_numpy(inputs.halton_configs(ch, T).astype(np.float32)).to(dev)
tg = hjcd.fk(rb, th).contiguous()
cfg = hjcd.default_config()
o1 = hjcd.poccd(rb, cfg, tg)
seeds, _ = hjcd.select_replicate(rb, cfg, o1["cost"], o1["theta"])
out = hjcd.pjik_trace(rb, cfg, tg, seeds)
it = out["iters"][:, 0].cpu().numpy()
tr = out["trace"].cpu().numpy().view(np.uint32)
slow = np.nonzero(it >= cfg.lm_iters)[0]
print(f"targets at the budget: {len(slow)}: {slow.tolist()}")
kind = tr & 3
a = (tr >> 2) & 31
valid = (tr >> 15) & 1
used = (cfg.B // cfg.K) * cfg.K


def timed(fn, reps=5):
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    return sorted(ts)[len(ts) // 2]


for t in slow[:8]:
    v = valid[t, :used]
    fail = ((v == 1) & ~((kind[t, :used] == 0) & (a[t, :used] == 0))).sum(0)   # per iteration
    kinds = np.bincount(kind[t, :used][v == 1], minlength=4)
    s1 = seeds[t:t + 1].contiguous()
    t1 = tg[t:t + 1].contiguous()
    ms32 = timed(lambda: hjcd.pjik(rb, cfg, t1, s1))
    ms64 = timed(lambda: hjcd.pjik_f64(rb, cfg, t1, s1))
    o64 = hjcd.pjik_f64(rb, cfg, t1, s1)
    print(f"t={t}: alpha=1 failures per iteration mean {fail.mean():.1f} (max {fail.max()}), steps "
          f"LM/dogleg/single/perturb {kinds.tolist()}; alone: fp32 {ms32:.3f} ms, fp64 {ms64:.3f} ms "
          f"(fp64 iters {int(o64['iters'][0, 0])}, best ep {float(o64['ep'][0, :used].min()):.3g})")

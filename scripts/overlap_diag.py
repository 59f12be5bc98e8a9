"""Do k_poccd and k_pjik_coop run concurrently on two streams?  Times each
alone and both launched together on two non-blocking streams (C2 inputs).
  python scripts/overlap_diag.py"""
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
s1 = torch.cuda.Stream(device=dev)
lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
s2 = torch.cuda.Stream(device=dev, priority=-1)


def timed(fn, streams):
    main = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(main)
    for s in streams:
        s.wait_event(a)
    fn()
    for s in streams:
        e = torch.cuda.Event()
        e.record(s)
        main.wait_event(e)
    b.record(main)
    torch.cuda.synchronize()
    return a.elapsed_time(b)


for mode in ("cluster", "percall"):
    cfg = hjcd.default_config(ccd_early_exit=1 if mode == "cluster" else 0)
    o1 = hjcd.poccd(robot, cfg, targets)
    seeds, _ = hjcd.select_replicate(robot, cfg, o1["cost"], o1["theta"])
    torch.cuda.synchronize()
    pc = lambda s=s1: hjcd.poccd(robot, cfg, targets, stream=s)
    pj = lambda s=s2: hjcd.pjik(robot, cfg, targets, seeds, stream=s)
    for _ in range(2):
        pc(); pj()
    torch.cuda.synchronize()
    ta = min(timed(pc, [s1]) for _ in range(5))
    tb = min(timed(pj, [s2]) for _ in range(5))
    tab = min(timed(lambda: (pc(), pj()), [s1, s2]) for _ in range(5))
    tba = min(timed(lambda: (pj(), pc()), [s1, s2]) for _ in range(5))
    print(f"{mode}: poccd alone {ta:.3f} ms, pjik alone {tb:.3f} ms, both (poccd first) {tab:.3f} ms, "
          f"both (pjik first) {tba:.3f} ms, sum {ta + tb:.3f}", flush=True)

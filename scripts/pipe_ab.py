"""Step time of hjcd_solve vs the stage-pipeline chunk count (DESIGN K10).
  HJCD_PIPELINE_CHUNKS=C python scripts/pipe_ab.py [c2|c3|c4|c3_T<n>] [reps]
Prints the p50 device time of one hjcd_solve (L2 flushed between reps) and
checks the result bitwise against the serial staged path (hjcd_solve_timed)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2510_07514_b200 import hjcd, inputs

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
CFG = {"c2": ("panda", 1000), "c3": ("fetch_like8", 10000), "c4": ("panda_x14", 10000),
       "c2_T10000": ("panda", 10000), "c3_T1000": ("fetch_like8", 1000), "c2_T300": ("panda", 300), "c2_T2000": ("panda", 2000), "c2_T4000": ("panda", 4000), "c2_T100": ("panda", 100),
       "x12": ("panda_x12", 1000), "x18": ("panda_x18", 1000), "x24": ("panda_x24", 1000), "x13": ("panda_x13", 1000)}
rname, T = CFG[cfgname]
chain = inputs.robot(rname)
robot = hjcd.Robot(chain)
dev = torch.device("cuda", 0)
th = torch.from_numpy(inputs.halton_configs(chain, T).astype(np.float32)).to(dev)
targets = hjcd.fk(robot, th).contiguous()
cfg = hjcd.default_config()
ws = hjcd.Workspace()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
stream = torch.cuda.current_stream()
if os.environ.get("HJCD_AB_STREAM") == "user":   # a created (non-legacy) stream instead of the default one
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
for _ in range(3):
    out = hjcd.solve(robot, targets, cfg, workspace=ws)
lat = []
for r in range(reps):
    flush.fill_(r & 0xFF)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    out = hjcd.solve(robot, targets, cfg, workspace=ws)
    b.record(stream)
    b.synchronize()
    lat.append(a.elapsed_time(b))
evs = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
ref = hjcd.solve(robot, targets, cfg, workspace=hjcd.Workspace(), events=evs)
torch.cuda.synchronize()
same = all(torch.equal(x, y) for x, y in zip(out, ref))
print(f"{cfgname} stream={os.environ.get('HJCD_AB_STREAM', 'default')} p50={statistics.median(lat):.3f} ms "
      f"min={min(lat):.3f} serial_staged={evs[0].elapsed_time(evs[4]):.3f} ms "
      f"success={float((out[3] <= 1).float().mean()):.4f} bitwise_equal_serial={same}", flush=True)

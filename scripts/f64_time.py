"""Device time of hjcd_solve_f64 (f1: fp64 polish) per chain, for A/B builds:
  HJCD_LIB=... python scripts/f64_time.py [reps]
Prints the p50 of `reps` solves (L2 flushed between them), the success rate at
1 mm / 1 deg, the median position error and a checksum of the returned theta
(for a bitwise comparison between builds)."""
import hashlib
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2510_07514_b200 import hjcd, inputs

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
stream = torch.cuda.current_stream()
lib = os.path.basename(os.environ.get("HJCD_LIB", "libhjcd.so"))
for name, T in (("panda", 1000), ("fetch_like8", 1000), ("panda_x12", 300), ("panda_x14", 300)):
    chain = inputs.robot(name)
    rb = hjcd.Robot(chain)
    th = torch.from_numpy(inputs.halton_configs(chain, T).astype(np.float32)).to(dev)
    tg = hjcd.fk(rb, th).contiguous()
    cfg = hjcd.default_config()
    ws = hjcd.Workspace()
    for _ in range(2):
        out = hjcd.solve_f64(rb, tg, cfg, workspace=ws)
    lat = []
    for r in range(reps):
        flush.fill_(r & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        out = hjcd.solve_f64(rb, tg, cfg, workspace=ws)
        b.record(stream)
        b.synchronize()
        lat.append(a.elapsed_time(b))
    q, pe, oe, st = out
    h = hashlib.sha1(q.cpu().numpy().tobytes()).hexdigest()[:12]
    print(f"{lib} f64 {name} T={T} p50={statistics.median(lat):.3f} ms success={float((st <= 1).float().mean()):.4f} "
          f"pos_err_p50={float(pe.median()):.3e} theta_sha1={h}", flush=True)

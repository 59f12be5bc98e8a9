import os, sys, statistics
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
from paper_2510_07514_b200 import hjcd, inputs
chain = inputs.panda(); robot = hjcd.Robot(chain); dev = torch.device("cuda", 0)
th = torch.from_numpy(inputs.halton_configs(chain, 1000).astype(np.float32)).to(dev)
targets = hjcd.fk(robot, th).contiguous()
cfg = hjcd.default_config()
o1 = hjcd.poccd(robot, cfg, targets)
seeds, _ = hjcd.select_replicate(robot, cfg, o1["cost"], o1["theta"])
t = 139
for copies in (1, 8, 37, 74, 148, 296):
    tg = targets[t:t+1].repeat(copies, 1).contiguous()
    sd = seeds[t:t+1].repeat(copies, 1, 1).contiguous()
    c1 = hjcd.default_config(target_index_offset=t)
    for _ in range(3): hjcd.pjik(robot, c1, tg, sd)
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); o = hjcd.pjik(robot, c1, tg, sd); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    print(f"copies {copies:4d}: {statistics.median(ts):.3f} ms, iters {int(o['iters'][0,0])}", flush=True)

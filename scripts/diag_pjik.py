"""Stage-2 diagnostics on C2: per-seed convergence, step-type counts, k* and
per-mode timing (per-seed freeze vs per-target early exit)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2510_07514_b200 import hjcd, inputs

chain = inputs.panda()
robot = hjcd.Robot(chain)
dev = torch.device("cuda", 0)
T = 1000
th = torch.from_numpy(inputs.halton_configs(chain, T).astype(np.float32)).to(dev)
targets = hjcd.fk(robot, th).contiguous()
cfg = hjcd.default_config()
o1 = hjcd.poccd(robot, cfg, targets)
seeds, kept = hjcd.select_replicate(robot, cfg, o1["cost"], o1["theta"])
print("poccd: mean iters", o1["iters"].float().mean().item(), "frac conv", (o1["iters"] < 64).float().mean().item())
ep1 = o1["ep"].cpu().numpy(); eo1 = o1["eo"].cpu().numpy()
best = np.argsort(o1["cost"].cpu().numpy(), axis=1)[:, :50]
bep = np.take_along_axis(ep1, best, 1); beo = np.take_along_axis(eo1, best, 1)
print("top-K seeds: ep p50 %.3g p90 %.3g  eo p50 %.3g p90 %.3g" % (np.median(bep), np.percentile(bep, 90), np.median(beo), np.percentile(beo, 90)))
for mode in (0, 1):
    c = hjcd.default_config(target_early_exit=mode)
    for _ in range(2):
        o2 = hjcd.pjik(robot, c, targets, seeds)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); o2 = hjcd.pjik(robot, c, targets, seeds); e1.record(); torch.cuda.synchronize()
    it = o2["iters"].cpu().numpy(); cnt = o2["counts"].cpu().numpy()
    ep = o2["ep"].cpu().numpy(); eo = o2["eo"].cpu().numpy()
    conv = (ep < 1e-6) & (eo < 1e-5)
    print(f"mode {mode}: {e0.elapsed_time(e1):.3f} ms; seeds conv {conv.mean():.3f}; targets w/ conv {conv.any(1).mean():.4f}")
    print("  iters p50/p90/p99/max", np.percentile(it, [50, 90, 99, 100]))
    tot = cnt.sum((0, 1)); print("  step counts LM/dogleg/single/perturb", tot, "per seed-iter", tot / max(1, it.sum()))
    pert = cnt[..., 3]
    print("  seeds with perturbation", (pert > 0).mean(), "mean perturb", pert.mean())
    if mode == 0:
        fi = np.where(conv, it, 10**6).min(1)
        print("  per-target first-converged iteration p50/p90/p99/max", np.percentile(np.minimum(fi, 128), [50, 90, 99, 100]))
        nc = ~conv.any(1)
        print("  targets without any converged seed:", np.where(nc)[0][:20])
        # best errors of stuck targets
        for t in np.where(nc)[0][:5]:
            b = np.argmin(ep[t] ** 2 + 0.25 * eo[t] ** 2)
            print("   t", t, "best ep %.3g eo %.3g" % (ep[t, b], eo[t, b]), "counts", cnt[t, b], "theta", o2["theta"][t, b].cpu().numpy().round(3))

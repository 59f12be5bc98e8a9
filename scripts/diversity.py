"""SURVEY §8(f) f2 / PAPER §V-C (Table III): solution-set diversity.
For T Halton Panda targets: X = the best 50 of HJCD-IK's polished batch
(hjcd_solve_batch, M = 2000 seeds as in the paper, B = 100, per-seed polish so
the whole batch converges); Y = a reference set standing in for the paper's
TRAC-IK samples (external, out of scope): PJ-IK from 50 independent uniform
starts, per-seed stop rule (SPEC §V-C stand-in).  Reports per-target MMD and
MMD^2 (hjcd_mmd, RBF with the median heuristic, R36) and the same score for a
degenerate batch of 50 copies of the best solution.
  python scripts/diversity.py [T]"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2510_07514_b200 import hjcd, inputs

Tn = int(sys.argv[1]) if len(sys.argv) > 1 else 100
chain = inputs.panda()
robot = hjcd.Robot(chain)
dev = torch.device("cuda", 0)
th = torch.from_numpy(inputs.halton_configs(chain, Tn).astype(np.float32)).to(dev)
targets = hjcd.fk(robot, th).contiguous()
cfg = hjcd.default_config(M=2000, K=50, B=100, target_early_exit=0)
q, pe, oe, st = hjcd.solve_batch(robot, targets, 50, cfg)
# reference: multi-start polish, the best 50 of PJ-IK from 200 uniform starts
# (the PO-CCD Philox seeds with 0 iterations, another rng key), per-seed stop
# rule, 512 iterations
cr = hjcd.default_config(M=200, K=200, B=200, ccd_iters=0, lm_iters=512, target_early_exit=0, rng_seed=12345)
u = hjcd.poccd(robot, cr, targets)["theta"].permute(0, 2, 1).contiguous()
ref = hjcd.pjik(robot, cr, targets, u)
Y, ype, yoe, _ = hjcd.select_topn(robot, cr, targets, ref["theta"], ref["ep"], ref["eo"], 50)
conv_x = ((pe < 1e-3) & (oe < math.pi / 180)).float().mean().item()
conv_y = ((ype < 1e-3) & (yoe < math.pi / 180)).float().mean().item()
m2, bw = hjcd.mmd(q.contiguous(), Y.contiguous())
deg = q[:, :1].expand(-1, 50, -1).contiguous()
d2, _ = hjcd.mmd(deg, Y.contiguous())
m2, d2 = m2.cpu().numpy(), d2.cpu().numpy()
mm = np.sqrt(np.maximum(m2, 0))
print(f"targets {Tn}: batch success {conv_x:.3f}, reference success {conv_y:.3f}")
print(f"HJCD-IK best-50 batch : MMD mean {mm.mean():.5f}  MMD^2 mean {m2.mean():.5f}")
print(f"degenerate (50 x best): MMD mean {np.sqrt(np.maximum(d2, 0)).mean():.5f}  MMD^2 mean {d2.mean():.5f}")
print(f"batch beats degenerate on {(m2 < d2).mean():.3f} of targets; bandwidth median {bw.median().item():.3f} rad")
print("paper (RTX 4060, TRAC-IK reference, kernel unstated): MMD 0.02983, MMD^2 0.00089 (context only)")

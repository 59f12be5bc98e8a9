#!/usr/bin/env python
"""HJCD-IK throughput/latency bench on B200 (BASELINE.json metric).

Workload (BASELINE configs[1], "C2"): Panda-like 7-DoF, 1000 reachable targets
per GPU x M=1000 seeds, K=50, B=100, I_c=64, I_l=128 (DESIGN.md R-defaults);
targets = FK (this library's hjcd_fk on the GPU) of Halton joint
configurations (synthetic, reachable by construction).  One step = one
hjcd_solve over the batch = PO-CCD + top-K/replicate + PJ-IK + best-select.

  python bench.py [--gpus N --steps K --warmup W] [--config c2|c3|c4|c5]
  python bench.py --impl reference ...   (the fp64 CPU oracle, timed on host cores)

Multi-GPU (torchrun, NCCL): each rank solves its own 1000 targets (weak
scaling, targets partitioned by global id) and the per-target results are
all-gathered (north_star's one collective).  Device time per step is the max
over ranks.  Prints ONE JSON line on rank 0.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (robot, targets per GPU, M, K, B, description)
    "c2": ("panda", 1000, 1000, 50, 100, "Panda 7-DoF, 1000 targets x 1000 seeds, 1 mm / 1 deg"),
    "c3": ("fetch_like8", 10000, 1000, 50, 100, "Fetch-like 8-DoF (prismatic torso + 7), 10000 targets"),
    "c4": ("panda_x14", 10000, 1000, 50, 100, "synthetic 14-DoF chain, 10000 targets"),
    "c5": ("panda", 12500, 1000, 50, 100, "Panda, 100000 targets split over 8 GPUs (12500 per GPU)"),
}
METRIC = "IK solves/s (targets solved per second)"
UNIT = "solves/s"


def peaks():
    p = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
    except Exception:
        pass
    return p


def fp32_peak_tflops(pk):
    """FP32 ALU peak: 148 SMs x 128 FP32 lanes x 2 flop (FMA) x max SM clock
    (B200_PROFILING.md unit counts; clock from MEASURED_PEAKS.json)."""
    mhz = float(pk.get("sm_max_mhz", 1965.0))
    return 148 * 128 * 2 * mhz * 1e6 / 1e12, mhz, ("measured sm_max_mhz" if "sm_max_mhz" in pk else "fallback 1965 MHz")


def flops_poccd_iter(n):
    return 200 * n + 175      # FK + residual + candidates + select per seed-iteration


def flops_poccd_final(n):
    return 96 * n + 72 + 70   # the closing FK + residual of every seed


def flops_pjik_iter(n):
    return 295 * n + 430      # LM path with one line-search trial


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index, path):
        self.path = path
        self.gpu = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9 and parts[1].replace(".", "").isdigit():
                    rows.append(parts)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows]
        mx = float(rows[0][2])
        loaded = [s for s in sm if s > 0.5 * mx] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows if r[3].replace(".", "").isdigit())
                if any(r[3].replace(".", "").isdigit() for r in rows) else None}


def run_reference(args, cfgname):
    """--impl reference: the fp64 CPU oracle (as it stands) on host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np

    import oracle
    from paper_2510_07514_b200 import inputs
    rname, Tg, M, K, B, desc = CONFIGS[cfgname]
    chain = inputs.robot(rname)
    p = oracle_params(M, K, B)
    cores = oracle.num_threads()
    per_step = max(4, cores)      # bounded sample: one target per host thread per step
    th = inputs.halton_configs(chain, per_step * (args.steps + args.warmup))
    tg = oracle.fk(chain, th).astype(np.float32)
    times = []
    for s in range(args.warmup + args.steps):
        x = tg[s * per_step:(s + 1) * per_step]
        t0 = time.perf_counter()
        oracle.solve(chain, p, x, tid_offset=s * per_step)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
    ms = 1e3 * statistics.mean(times)
    val = per_step / (ms / 1e3)
    sample = f"{per_step} targets per step (of the {Tg}-target workload), full M/K/B, {args.steps} steps"
    out = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"{cfgname}: {desc}", "robot": rname, "targets_per_step": per_step,
                      "M": M, "K": K, "B": B, "ccd_iters": 64, "lm_iters": 128, "parallelism": "host threads"},
           "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
           "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


def oracle_params(M, K, B):
    return dict(M=M, K=K, B=B, ccd_iters=64, lm_iters=128, eps_p_coarse=5e-3, eps_o_coarse=5e-2,
                eps_p_fine=1e-6, eps_o_fine=1e-5, gamma=1e-6, delta0=1.0, delta_rho=0.98,
                delta_min=0.1, sigma_ccd=0.05, sigma_rep=0.02, sigma_lm=0.05, d_floor=1e-8, R=0.5,
                beta=2.0, A=8, w_p=1.0, w_o=0.5, succ_p=1e-3, succ_o=math.pi / 180, tau_deg=1e-5,
                rng_seed=0, repl_noise_all=0, target_early_exit=1, ccd_early_exit=1,
                **{"lambda": 1e-3})


def cpu_baseline(cfgname, budget_s=12.0):
    """The oracle as it stands on this box's host cores, bounded sample."""
    import numpy as np

    import oracle
    from paper_2510_07514_b200 import inputs
    rname, Tg, M, K, B, _ = CONFIGS[cfgname]
    chain = inputs.robot(rname)
    p = oracle_params(M, K, B)
    cores = oracle.num_threads()
    chunk = max(4, cores)
    done, elapsed, c = 0, 0.0, 0
    while elapsed < budget_s and done < Tg:
        th = inputs.halton_configs(chain, chunk, start=done)
        tg = oracle.fk(chain, th).astype(np.float32)
        t0 = time.perf_counter()
        oracle.solve(chain, p, tg, tid_offset=done)
        elapsed += time.perf_counter() - t0
        done += chunk
        c += 1
    return {"value": done / elapsed, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"first {done} of the {Tg} targets (full M={M}, K={K}, B={B}), {elapsed:.1f} s wall"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="hjcd", choices=["hjcd", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the latency-vs-batch sweep")
    ap.add_argument("--targets", type=int, default=None, help="override targets per GPU")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args, args.config)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2510_07514_b200 import hjcd, inputs
    from paper_2510_07514_b200.parallel import solve_distributed

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU; HJCD_DIST_BACKEND=gloo + more ranks than GPUs is a
    # functional check of the multi-rank path on a single-GPU box (ranks share
    # a device; the gather goes through host memory), not a scaling number
    backend = os.environ.get("HJCD_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    rname, Tg, M, K, B, desc = CONFIGS[args.config]
    if args.targets:
        Tg = args.targets
    chain = inputs.robot(rname)
    robot = hjcd.Robot(chain)
    n = robot.dof
    cfg = hjcd.default_config(M=M, K=K, B=B, target_index_offset=rank * Tg)
    # reachable targets: this library's FK of Halton configurations (rank's slice)
    th = torch.from_numpy(inputs.halton_configs(chain, Tg, start=rank * Tg).astype(np.float32)).to(dev)
    targets = hjcd.fk(robot, th).contiguous()
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2
    ws = hjcd.Workspace()

    KNAMES = ("k_poccd", "k_select_replicate", "k_pjik", "k_select_best")

    def step(events=None):
        fn = (lambda r, t, c: hjcd.solve(r, t, c, workspace=ws, events=events))
        return solve_distributed(robot, targets, cfg, solve_fn=fn) if world > 1 else fn(robot, targets, cfg)

    for _ in range(args.warmup):
        out = step()
    torch.cuda.synchronize()

    # ---------------- timed region: K steps of the public API (hjcd_solve: PJ-IK
    # launched as a programmatic dependent of PO-CCD, DESIGN K10), CUDA events
    # per step on the launching stream
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    # second timed region, same K steps through the staged sequence (one kernel
    # per stage, library events at the stage boundaries: hjcd_solve_timed) for
    # the per-kernel times and the roofline of k_poccd
    sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    for ks in kev:
        for e in ks:
            e.record(stream)      # materialise the events before the timed region
    clk = Clocks(local, os.path.join(ROOT, "gpurun_out", f"clocks_rank{rank}.csv") if os.path.isdir(
        os.path.join(ROOT, "gpurun_out")) else f"/tmp/hjcd_clocks_rank{rank}.csv")
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with clk:
        for s in range(args.steps):
            flush.fill_(s & 0xFF)            # L2 flush between steps (outside the events)
            evs[s][0].record(stream)
            out = step()
            evs[s][1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        for s in range(args.steps):
            flush.fill_(s & 0xFF)
            sev[s][0].record(stream)
            step(kev[s])
            sev[s][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    staged_ms = statistics.mean(a.elapsed_time(b) for a, b in sev)
    ms_local = statistics.mean(step_ms)
    if world > 1:
        t = torch.tensor([ms_local], device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    else:
        ms = ms_local
    total_targets = Tg * world
    value = total_targets / (ms / 1e3)
    q, pe, oe, st = out
    st_np = st.cpu().numpy()
    succ = float(np.mean(st_np <= 1))
    kmean = {k: statistics.mean(ks[i].elapsed_time(ks[i + 1]) for ks in kev) for i, k in enumerate(KNAMES)}

    # ---------------- algorithmic work of the timed launches: the staged entry
    # points run the same kernels on the same inputs (deterministic), untimed,
    # to count the iterations each seed executed
    o1 = hjcd.poccd(robot, cfg, targets)
    seeds, _ = hjcd.select_replicate(robot, cfg, o1["cost"], o1["theta"])
    o2 = hjcd.pjik(robot, cfg, targets, seeds)
    iters_sum = int(o1["iters"].sum().item())
    used = (B // K) * K
    pj_iters_sum = int(o2["iters"][:, :used].sum().item())
    kstar = o2["iters"][:, 0].float()
    pk = peaks()
    peak_tf, mhz, peak_src = fp32_peak_tflops(pk)
    seeds_total = Tg * M
    poccd_flops = iters_sum * flops_poccd_iter(n) + seeds_total * flops_poccd_final(n)
    pjik_flops = pj_iters_sum * flops_pjik_iter(n)
    ach = poccd_flops / (kmean["k_poccd"] / 1e3) / 1e12
    traffic, exec_flops = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
        traffic = tj.get(args.config, {}).get("k_poccd")
        exec_flops = tj.get("_executed_fp32_flops", {}).get(args.config, {}).get("k_poccd")
    except Exception:
        pass
    roofline = {"bound": "alu", "kernel": "k_poccd", "achieved": ach, "peak": peak_tf, "unit": "TFLOP/s",
                "frac": ach / peak_tf, "traffic": traffic,
                "peak_source": f"148 SM x 128 FP32 lanes x 2 x {mhz:.0f} MHz ({peak_src})",
                "algorithmic_flops_per_launch": poccd_flops,
                "ncu_executed_fp32_flops_per_launch": exec_flops,
                "ncu_executed_frac": (exec_flops / (kmean["k_poccd"] / 1e3) / 1e12 / peak_tf) if exec_flops else None,
                "unit_flops": f"{flops_poccd_iter(n)} per seed-iteration + {flops_poccd_final(n)} per seed",
                "kernel_ms": kmean,
                "kernel_ms_source": "library events at the stage boundaries of the K staged timed steps "
                                    "(hjcd_solve_timed: one kernel per stage, %.3f ms per step)" % staged_ms,
                "share_of_step": {k: v / sum(kmean.values()) for k, v in kmean.items()},
                "k_pjik": {"achieved": pjik_flops / (kmean["k_pjik"] / 1e3) / 1e12,
                           "frac": pjik_flops / (kmean["k_pjik"] / 1e3) / 1e12 / peak_tf,
                           "bound_note": "latency of the slowest target (per-target stop rule), not ALU"},
                "poccd_mean_iters": iters_sum / seeds_total,
                "pjik_kstar": {"mean": float(kstar.mean()), "p50": float(kstar.median()),
                               "p99": float(torch.quantile(kstar, 0.99)), "max": float(kstar.max()),
                               "frac_at_budget": float((kstar >= cfg.lm_iters).float().mean())},
                "status_hist": [int((st == i).sum()) for i in range(4)],
                "pjik_mean_iters": pj_iters_sum / (Tg * (B // K) * K)}

    # ---------------- latency vs batch (BASELINE metric "p50 latency vs batch"):
    # one hjcd_solve of T targets, same robot and config, device-resident I/O
    sweep = []
    if not args.no_sweep and world == 1:
        for Ts in (1, 10, 100, 1000, 10000):
            ths = torch.from_numpy(inputs.halton_configs(chain, Ts, start=50000).astype(np.float32)).to(dev)
            tgs = hjcd.fk(robot, ths).contiguous()
            c2 = hjcd.default_config(M=M, K=K, B=B, target_index_offset=50000)
            sws = hjcd.Workspace()
            for _ in range(2):
                hjcd.solve(robot, tgs, c2, workspace=sws)
            reps = 20 if Ts <= 1000 else 5
            lat = []
            for _ in range(reps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                r = hjcd.solve(robot, tgs, c2, workspace=sws)
                b.record(stream)
                b.synchronize()
                lat.append(a.elapsed_time(b))
            lat.sort()
            sweep.append({"targets": Ts, "p50_ms": lat[len(lat) // 2],
                          "p99_ms": lat[min(len(lat) - 1, int(math.ceil(0.99 * len(lat))) - 1)],
                          "solves_per_s": Ts / (lat[len(lat) // 2] / 1e3),
                          "success": float((r[3] <= 1).float().mean())})

    # ---------------- DoF sweep (PAPER Table II protocol): Panda
    # extended cyclically to 7/12/18/24 DoF (R34), 1000 targets, same M/K/B
    dof_sweep = []
    if not args.no_sweep and world == 1:
        for nd in (7, 12, 18, 24):
            ch = inputs.robot(f"panda_x{nd}")
            rbd = hjcd.Robot(ch)
            ths = torch.from_numpy(inputs.halton_configs(ch, 1000).astype(np.float32)).to(dev)
            tgs = hjcd.fk(rbd, ths).contiguous()
            c2 = hjcd.default_config(M=M, K=K, B=B)
            sws = hjcd.Workspace()
            hjcd.solve(rbd, tgs, c2, workspace=sws)
            lat = []
            for _ in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                r = hjcd.solve(rbd, tgs, c2, workspace=sws)
                b.record(stream)
                b.synchronize()
                lat.append(a.elapsed_time(b))
            lat.sort()
            dof_sweep.append({"dof": nd, "targets": 1000, "p50_ms": lat[2], "solves_per_s": 1000 / (lat[2] / 1e3),
                              "success": float((r[3] <= 1).float().mean()),
                              "fine_converged": float((r[3] == 0).float().mean())})

    # ---------------- PAPER Table I protocol (SURVEY 8(d) P-proto, E1; context
    # only): ONE target per solve, 100 Halton targets, M in {1..2000} seeds,
    # K = min(50, M) and B = min(100, M) (SURVEY's reading) or B = 100 (the
    # paper also calls M the "batch size"); mean device time per
    # target and mean reported errors of the answers
    paper_protocol = []
    if not args.no_sweep and world == 1:
        for rn in ("panda", "fetch_like8"):
            ch = inputs.robot(rn)
            rbp = hjcd.Robot(ch)
            ths = torch.from_numpy(inputs.halton_configs(ch, 100).astype(np.float32)).to(dev)
            tgs = hjcd.fk(rbp, ths).contiguous()
            for Mp, Bp in ((1, 1), (1, 100), (10, 10), (10, 100), (100, 100), (1000, 100), (2000, 100)):
                cp = hjcd.default_config(M=Mp, K=min(50, Mp), B=Bp)
                sws = hjcd.Workspace()
                hjcd.solve(rbp, tgs[:1].contiguous(), cp, workspace=sws)
                lat, pes, oes, oks = [], [], [], []
                for i in range(100):
                    ci = hjcd.default_config(M=Mp, K=min(50, Mp), B=Bp, target_index_offset=i)
                    ti = tgs[i:i + 1]
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    r = hjcd.solve(rbp, ti, ci, workspace=sws)
                    b.record(stream)
                    b.synchronize()
                    lat.append(a.elapsed_time(b))
                    pes.append(float(r[1][0]))
                    oes.append(float(r[2][0]))
                    oks.append(int(r[3][0]) <= 1)
                paper_protocol.append({"robot": rn, "M": Mp, "K": min(50, Mp), "B": Bp, "targets": 100, "mean_ms_per_target": statistics.mean(lat),
                                       "mean_pos_err_m": statistics.mean(pes), "mean_ori_err_rad": statistics.mean(oes),
                                       "success": statistics.mean(oks)})

    # ---------------- end to end through the C ABI with host buffers
    tg_host = targets.cpu().pin_memory()
    outh = (torch.empty((Tg, n), dtype=torch.float32).pin_memory(), torch.empty(Tg).pin_memory(),
            torch.empty(Tg).pin_memory(), torch.empty(Tg, dtype=torch.int32).pin_memory())
    hws = hjcd.Workspace()
    for _ in range(2):
        hjcd.solve_host(robot, tg_host, cfg, out=outh, workspace=hws)
    e2e_ms = []
    for s in range(max(3, min(args.steps, 10))):
        flush.fill_(s & 0xFF)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        hjcd.solve_host(robot, tg_host, cfg, out=outh, workspace=hws)
        e2e_ms.append(1e3 * (time.perf_counter() - t0))
    e2e_local = statistics.mean(e2e_ms)
    if world > 1:
        t = torch.tensor([e2e_local], device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_local = float(t.item())
    e2e = {"value": total_targets / (e2e_local / 1e3), "unit": UNIT, "h2d_bytes_per_step": Tg * 7 * 4,
           "d2h_bytes_per_step": Tg * (n + 3) * 4, "ms_per_step": e2e_local, "api": "hjcd_solve_host"}

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = cpu_baseline(args.config)
        srt = sorted(step_ms)
        res = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": "f32", "data": "synthetic",
               "config": {"workload": f"{args.config}: {desc}", "robot": rname, "targets_per_gpu": Tg,
                          "global_targets": total_targets, "M": M, "K": K, "B": B, "ccd_iters": cfg.ccd_iters,
                          "lm_iters": cfg.lm_iters, "parallelism": f"targets partitioned over {world} GPU(s)"
                          + ((" + NCCL all_gather of results" if backend == "nccl" else
                                      f" + {backend} all_gather (functional check, ranks share a GPU)") if world > 1 else ""),
                          "l2": "flushed between steps (256 MiB write)"},
               "p50_ms": srt[len(srt) // 2], "p99_ms": srt[min(len(srt) - 1, int(math.ceil(0.99 * len(srt))) - 1)],
               "latency_note": "p50/p99 of the per-step batch latency (one hjcd_solve of all targets)",
               "success_rate_1mm_1deg": succ,
               "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "latency_vs_batch": sweep,
               "dof_sweep": dof_sweep, "paper_protocol_table1": paper_protocol,
               "gpu_launches": 3 * args.steps,
               "gpu_launches_note": "per hjcd_solve step: k_poccd, k_pjik_coop (dependent launch), k_select_best "
                                    "(+ one memset of the per-target readiness counts)",
               "clocks": clk.summary(),
               "paper_context": "RTX 4060 Laptop, Panda M=1000: 7.53 ms per target (133 targets/s), PAPER.md P:355"}
        print(json.dumps(res))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

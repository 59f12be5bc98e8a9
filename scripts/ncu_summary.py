"""Summarise ncu captures into profiles/ (tracked).

  python scripts/ncu_summary.py TAG gpurun_out/prof.ncu-rep [gpurun_out/launches.csv]

Writes profiles/TAG_ncu.md (per-kernel speed-of-light, pipes, occupancy,
stalls, SASS opcode mix per launch) and merges per-launch DRAM traffic into
profiles/traffic.json ({config: {kernel: bytes}}), which bench.py reports as
roofline.traffic.  With a launch list (the --metrics gpu__time_duration.sum
pass over bench.py) it also writes profiles/TAG_launches.csv and the
per-kernel share of the step.
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NCU = os.environ.get("NCU", "/usr/local/cuda/bin/ncu")

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "FMA-heavy pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads / warp inst"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__occupancy_limit_registers", "CTA limit (registers)"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__cycles_active.avg", "SM active cycles (avg)"),
    ("gpc__cycles_elapsed.max", "elapsed cycles"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "thread FFMA"),
    ("smsp__sass_thread_inst_executed_op_fmul_pred_on.sum", "thread FMUL"),
    ("smsp__sass_thread_inst_executed_op_fadd_pred_on.sum", "thread FADD"),
]


def _csv(args):
    out = subprocess.run([NCU, *args], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def _num(s):
    try:
        return float(str(s).replace(",", ""))
    except ValueError:
        return None


def raw(rep):
    rows = _csv(["-i", rep, "--page", "raw", "--csv"])
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {h: (v, u) for h, v, u in zip(hdr, r, units)}
        out.append(d)
    return out


def to_bytes(v, u):
    x = _num(v)
    if x is None:
        return None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    return x * scale


def opcode_mix(rep, kernel_regex):
    rows = _csv(["-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kernel_regex}"])
    hdr = None
    body = []
    for r in rows:
        if "Instructions Executed" in r and "Source" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            body.append(r)
    if not hdr:
        return {}, {}, {}
    ie, src = hdr.index("Instructions Executed"), hdr.index("Source")
    ti = hdr.index("Predicated-On Thread Instructions Executed") if "Predicated-On Thread Instructions Executed" in hdr else None
    st = hdr.index("Warp Stall Sampling (All Samples)") if "Warp Stall Sampling (All Samples)" in hdr else None
    ops, stalls = collections.Counter(), collections.Counter()
    thread_ops = collections.Counter()
    for r in body:
        toks = r[src].strip().split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        op = op.split(".")[0]
        ops[op] += int(_num(r[ie]) or 0)
        if ti is not None:
            thread_ops[op] += int(_num(r[ti]) or 0)
        if st is not None:
            stalls[op] += int(_num(r[st]) or 0)
    return ops, stalls, thread_ops


def main():
    tag, rep = sys.argv[1], sys.argv[2]
    launches = sys.argv[3] if len(sys.argv) > 3 else None
    config = os.environ.get("HJCD_CONFIG", "c2")
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    kernels = raw(rep)
    lines = [f"# ncu summary {tag}", "", f"Source capture: `{os.path.basename(rep)}` "
             "(`ncu --set full --clock-control none --import-source on`, one B200).", ""]
    traffic = {}
    tpath = os.path.join(prof, "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath))
    seen = set()
    for d in kernels:
        name = d.get("Kernel Name", ("?", ""))[0]
        short = name.split("(")[0].replace("void ", "").replace("hjcd::", "")
        if short in seen:
            continue
        seen.add(short)
        lines += [f"## {short}", "", "| metric | value | unit |", "|---|---|---|"]
        for key, label in METRICS:
            if key in d:
                v, u = d[key]
                lines.append(f"| {label} (`{key}`) | {v} | {u} |")
        rb = to_bytes(*d.get("dram__bytes_read.sum", ("", "")))
        wb = to_bytes(*d.get("dram__bytes_write.sum", ("", "")))
        if rb is not None and wb is not None:
            base = short.split("<")[0]
            traffic.setdefault(config, {})[base] = rb + wb
            lines.append(f"| DRAM read+write per launch | {rb + wb:.0f} | byte |")
        stall_keys = sorted((k for k in d if k.startswith("smsp__average_warp_latency_issue_stalled_") or
                             k.startswith("smsp__pcsamp_warps_issue_stalled_")), key=lambda k: -(_num(d[k][0]) or 0))
        top = [(k, d[k][0]) for k in stall_keys if (_num(d[k][0]) or 0) > 0][:8]
        if top:
            lines += ["", "Top stall reasons (sampled):", ""]
            lines += [f"- `{k}`: {v}" for k, v in top]
        base = short.split("<")[0]
        ops, stalls, tops = opcode_mix(rep, base)
        tot = sum(ops.values())
        if tops:
            # executed FP32 flops from the per-instruction predicated-on thread counts
            # (packed pairs count twice: FFMA2 = 2 FMAs, FMUL2 / FADD2 = 2 operations)
            fl = (2 * tops.get("FFMA", 0) + tops.get("FMUL", 0) + tops.get("FADD", 0) + 4 * tops.get("FFMA2", 0)
                  + 2 * tops.get("FMUL2", 0) + 2 * tops.get("FADD2", 0))
            dur = d.get("gpu__time_duration.sum", ("", ""))
            dur_s = _num(dur[0]) * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(
                dur[1], 1e-3) if _num(dur[0]) else None
            lines += ["", f"Executed FP32 flops per launch (2 FFMA + FMUL + FADD + 4 FFMA2 + 2 FMUL2 + 2 FADD2, "
                          f"thread level): {fl:.4g}"]
            if dur_s:
                lines.append(f"Executed FP32 rate: {fl / dur_s / 1e12:.2f} TFLOP/s at the captured duration")
                traffic.setdefault("_executed_fp32_flops", {}).setdefault(config, {})[base] = fl
        if tot:
            lines += ["", f"SASS opcode mix (warp-level executed instructions, total {tot}):", "",
                      "| opcode | share | stall samples |", "|---|---|---|"]
            for op, n in ops.most_common(16):
                lines.append(f"| {op} | {100 * n / tot:.2f}% | {stalls[op]} |")
        lines.append("")
    if launches and os.path.exists(launches):
        rows = list(csv.reader(open(launches)))
        h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        hdr = rows[h]
        ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
        per = collections.defaultdict(list)
        with open(os.path.join(prof, f"{tag}_launches.csv"), "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["id", "kernel", "gpu__time_duration.sum [ns]"])
            for i, r in enumerate(rows[h + 1:]):
                if len(r) > vi:
                    k = r[ki].split("(")[0].replace("void ", "").replace("hjcd::", "")
                    w.writerow([i, k, r[vi]])
                    if k.startswith("k_"):
                        per[k.split("<")[0]].append(_num(r[vi]) or 0)
        tot = sum(sum(v) / len(v) for v in per.values())
        lines += ["## Launch list (serialised, cold-cache; share of one step)", "",
                  "| kernel | launches | mean ns | share |", "|---|---|---|---|"]
        for k, v in per.items():
            m = sum(v) / len(v)
            lines.append(f"| {k} | {len(v)} | {m:.0f} | {100 * m / tot:.1f}% |")
        lines.append("")
    with open(os.path.join(prof, f"{tag}_ncu.md"), "w") as f:
        f.write("\n".join(lines))
    # the traffic table is merged only for a bench capture (with its launch
    # list) or when HJCD_CONFIG names the workload: a side capture (one slow
    # target, another config) must not overwrite the bench's C2 numbers
    if launches or "HJCD_CONFIG" in os.environ:
        with open(tpath, "w") as f:
            json.dump(traffic, f, indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main()

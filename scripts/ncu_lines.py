"""Per-source-line instruction and stall totals from an ncu report
(--page source --print-source cuda,sass).  Usage:
  python scripts/ncu_lines.py REP KERNEL_REGEX [TOP]"""
import collections
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{kre}"], capture_output=True, text=True).stdout
fname, line, src = "?", None, ""
inst, stall = collections.Counter(), collections.Counter()
text = {}
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0].strip():
        line = (fname, int(r[0]))
        text[line] = r[1].strip()[:80]
    try:
        inst[line] += int(r[hdr.index("Instructions Executed")] or 0)
        stall[line] += int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except (ValueError, IndexError):
        pass
ti, ts = sum(inst.values()), sum(stall.values())
print(f"total warp inst {ti}, stall samples {ts}")
for k, v in stall.most_common(top):
    print(f"{100 * v / ts:5.1f}% stall {100 * inst[k] / ti:5.1f}% inst  {k[0]}:{k[1]}  {text.get(k, '')}")

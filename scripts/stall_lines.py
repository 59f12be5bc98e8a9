"""Stall samples of one kernel per source line of its kernel file (ncu source
page + nvdisasm line table of the SAME build), inlined helpers attributed to
the calling line of the kernel file:
    ncu -i rep --page source --csv -k regex:NAME --print-source sass > src.csv
    cuobjdump -xelf all obj.o; nvdisasm -gi -c obj.cubin > obj.sass
    python scripts/stall_lines.py src.csv obj.sass MANGLED_NAME pjik_coop.cuh path/to/pjik_coop.cuh"""
import collections
import csv
import re
import sys

src_csv, sass, fname, home, home_path = sys.argv[1:6]
rows = list(csv.reader(open(src_csv)))
hdr = rows[1]
ia, iss = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
dyn = [(int(r[ia], 16), int(r[iss] or 0), {hdr[i]: int(r[i] or 0) for i in stall_cols})
       for r in rows[2:] if len(r) > iss and r[ia].startswith("0x")]
base = dyn[0][0]
lines = open(sass).read().split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith(".text." + fname + ":"))
cur, off2line = None, {}
for l in lines[start + 1:]:
    if l.startswith(".text.") or l.startswith("\t.section"):
        break
    if re.search(r'//## File "([^"]+)", line (\d+)', l):
        chain = re.findall(r'"([^"]+)", line (\d+)', l)
        cur = next((int(x) for f, x in chain if f.endswith(home)), None)
        continue
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+", l)
    if m and cur:
        off2line[int(m.group(1), 16)] = cur
tot = sum(d[1] for d in dyn)
by, st = collections.Counter(), collections.defaultdict(collections.Counter)
for a, s_, x in dyn:
    k = off2line.get(a - base, 0)
    by[k] += s_
    for kk, v in x.items():
        st[k][kk] += v
src = open(home_path).read().split("\n")
print(f"total stall samples {tot}")
for k, v in by.most_common(int(sys.argv[6]) if len(sys.argv) > 6 else 20):
    top = ", ".join(f"{a[6:]}={b}" for a, b in st[k].most_common(2))
    print(f"{k:4d} {100 * v / tot:5.1f}%  {top:52s} | {src[k - 1].strip()[:72] if k else '(other file)'}")

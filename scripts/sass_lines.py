"""Dynamic instruction counts of one kernel per source line (ncu source page +
nvdisasm -gi line table), attributing inlined helpers to the kernel-file line
that called them.

    ncu -i rep.ncu-rep --page source --csv -k regex:NAME --print-source sass > src.csv
    nvdisasm -gi -c obj.cubin > obj.sass
    python scripts/sass_lines.py src.csv obj.sass MANGLED_NAME poccd.cuh
"""
import csv
import re
import sys
from collections import Counter, defaultdict

src_csv, sass, fname, home = sys.argv[1:5]
rows = list(csv.reader(open(src_csv)))
hdr = rows[1]
ia, ie = hdr.index("Address"), hdr.index("Instructions Executed")
isrc = hdr.index("Source")
dyn = []
for r in rows[2:]:
    if len(r) > ie and r[ia].startswith("0x"):
        dyn.append((int(r[ia], 16), int(r[ie]), r[isrc].strip()))
base = dyn[0][0]
lines = open(sass).read().split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith(".text." + fname + ":"))
cur = None
off2line = {}
for l in lines[start + 1:]:
    if l.startswith("//----") or l.startswith("\t.section"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', l)
    if m:
        f, ln, f2, ln2 = m.group(1).split("/")[-1], int(m.group(2)), m.group(3), m.group(4)
        if f == home:
            cur = (home, ln)
        elif f2 and f2.split("/")[-1] == home:
            cur = (home, int(ln2))
        else:
            cur = (f, ln) if f2 is None else (f2.split("/")[-1], int(ln2))
        continue
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s", l)
    if m:
        off2line[int(m.group(1), 16)] = cur
agg = Counter()
ops = defaultdict(Counter)
total = 0
for a, n, s in dyn:
    key = off2line.get(a - base, ("?", 0))
    agg[key] += n
    total += n
    op = s.split()[0] if not s.startswith("@") else s.split()[1]
    ops[key][op.split(".")[0]] += n
print(f"total warp instructions {total:.4g}")
for key, n in sorted(agg.items(), key=lambda kv: -kv[1])[:60]:
    print(f"{key[0]}:{key[1]:<5d} {n:12d} {100 * n / total:5.1f}%  {dict(ops[key].most_common(4))}")

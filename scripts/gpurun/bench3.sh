# usage: gpurun -- 'bash scripts/gpurun/bench3.sh [pytest -k expr]'  C2/C3/C4 lines (no sweeps), then selected GPU tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/bench3.txt
for rep in 1 2; do
for cfg in c2 c3 c4; do
  st=20; [ $cfg != c2 ] && st=5
  timeout 300 python bench.py --config $cfg --no-sweep --no-cpu-baseline --steps $st > gpurun_out/bench3_last.log 2>&1
  python - $cfg <<'PY' >> gpurun_out/bench3.txt
import json, sys
d = json.loads([l for l in open("gpurun_out/bench3_last.log") if l.startswith("{")][0])
r = d["roofline"]
print(sys.argv[1], "ms/step %.4f" % d["ms_per_step"], "k_poccd %.4f" % r["kernel_ms"]["k_poccd"], "k_pjik %.4f" % r["kernel_ms"]["k_pjik"], "frac %.4f" % r["frac"], "succ", d["success_rate_1mm_1deg"])
PY
done
done
if [ -n "$1" ]; then
timeout 1200 python -m pytest tests -m gpu -q -s -p no:cacheprovider -k "$1" -rf > gpurun_out/pytest_sel.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sel.log
fi
echo done

# usage: gpurun -- 'bash scripts/gpurun/libs_c2.sh LIB1 LIB2 ...'  (paths relative to the repo; "default" = in-tree)
# C2 bench line (no sweeps, no CPU baseline) for each library build, twice, interleaved
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/libs_c2.txt
for rep in 1 2; do
for L in "$@"; do
  if [ "$L" = "default" ]; then unset HJCD_LIB; else export HJCD_LIB=$GRAFT_REPO_ROOT/$L; fi
  timeout 300 python bench.py --no-sweep --no-cpu-baseline --steps 20 > gpurun_out/libs_c2_last.log 2>&1
  python - "$L" <<'PY' >> gpurun_out/libs_c2.txt
import json, sys
d = json.loads([l for l in open("gpurun_out/libs_c2_last.log") if l.startswith("{")][0])
r = d["roofline"]
print(sys.argv[1], "ms/step %.4f" % d["ms_per_step"], "k_poccd %.4f" % r["kernel_ms"]["k_poccd"], "k_pjik %.4f" % r["kernel_ms"]["k_pjik"], "frac %.4f" % r["frac"], "succ", d["success_rate_1mm_1deg"])
PY
done
done
echo done

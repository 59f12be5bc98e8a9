# usage: gpurun -- 'bash scripts/gpurun/libs_cfgs.sh "c2 c3 c4" LIB1 LIB2 ...'  (paths relative to the repo; "default" = in-tree)
# bench lines (no sweeps, no CPU baseline) per config and library build, twice, interleaved
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CFGS="$1"; shift
rm -f gpurun_out/libs_cfgs.txt
for rep in 1 2; do
for L in "$@"; do
  if [ "$L" = "default" ]; then unset HJCD_LIB; else export HJCD_LIB=$GRAFT_REPO_ROOT/$L; fi
  for cfg in $CFGS; do
    st=20; [ $cfg != c2 ] && st=5
    timeout 300 python bench.py --config $cfg --no-sweep --no-cpu-baseline --steps $st > gpurun_out/libs_last.log 2>&1
    python - "$L" $cfg <<'PY' >> gpurun_out/libs_cfgs.txt
import json, sys
try:
    d = json.loads([l for l in open("gpurun_out/libs_last.log") if l.startswith("{")][0])
except Exception as e:
    print(sys.argv[1], sys.argv[2], "FAILED", open("gpurun_out/libs_last.log").read()[-500:]); sys.exit()
r = d["roofline"]
print(sys.argv[1].split("/")[-1], sys.argv[2], "ms/step %.4f" % d["ms_per_step"], "k_poccd %.4f" % r["kernel_ms"]["k_poccd"], "k_pjik %.4f" % r["kernel_ms"]["k_pjik"], "frac %.4f" % r["frac"], "succ", d["success_rate_1mm_1deg"])
PY
  done
done
done
echo done

# usage: gpurun -- 'bash scripts/gpurun/x2_env_ab.sh'   K17 A/B on C2 and C3 (HJCD_POCCD_X2=1 vs 0), interleaved
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/x2_ab.txt
for rep in 1 2; do
for x in 1 0; do
  for cfg in c2 c3; do
    st=20; [ $cfg = c3 ] && st=5
    HJCD_POCCD_X2=$x timeout 300 python bench.py --config $cfg --no-sweep --no-cpu-baseline --steps $st > gpurun_out/x2_last.log 2>&1
    python - $x $cfg <<'PY' >> gpurun_out/x2_ab.txt
import json, sys
d = json.loads([l for l in open("gpurun_out/x2_last.log") if l.startswith("{")][0])
r = d["roofline"]
print("x2=" + sys.argv[1], sys.argv[2], "ms/step %.4f" % d["ms_per_step"], "k_poccd %.4f" % r["kernel_ms"]["k_poccd"], "k_pjik %.4f" % r["kernel_ms"]["k_pjik"], "frac %.4f" % r["frac"], "succ", d["success_rate_1mm_1deg"])
PY
  done
done
done
echo done

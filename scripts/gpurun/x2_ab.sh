# usage: gpurun -- 'bash scripts/gpurun/x2_ab.sh'
# K17 A/B: the packed two-seeds-per-thread PO-CCD kernel against the one-seed kernel
# (HJCD_POCCD_X2=0), C2 / C3 bench lines, then the replay and C2 parity tests on x2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for x in 1 0 1 0; do
  HJCD_POCCD_X2=$x timeout 300 python bench.py --no-sweep --no-cpu-baseline --steps 20 > gpurun_out/x2_ab_c2_$x.log 2>&1
  HJCD_POCCD_X2=$x timeout 300 python bench.py --config c3 --no-sweep --no-cpu-baseline --steps 5 > gpurun_out/x2_ab_c3_$x.log 2>&1
  python - <<PY >> gpurun_out/x2_ab.txt
import json
for c in ("c2", "c3"):
    d = json.loads([l for l in open("gpurun_out/x2_ab_%s_$x.log" % c) if l.startswith("{")][0])
    r = d["roofline"]
    print("x2=$x", c, "ms/step %.4f" % d["ms_per_step"], "k_poccd %.4f" % r["kernel_ms"]["k_poccd"], "k_pjik %.4f" % r["kernel_ms"]["k_pjik"], "frac %.4f" % r["frac"], "succ", d["success_rate_1mm_1deg"])
PY
done
timeout 1200 python -m pytest tests -m gpu -q -s -p no:cacheprovider -k "replay or c2 or c1 or dependent or concurrent or poccd" -rf > gpurun_out/pytest_x2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_x2.log
echo done

# usage: gpurun -- 'bash scripts/gpurun/x2_ncu.sh'
# K17: C2 bench A/B (x2 vs one-seed kernel) and one full ncu capture of each PO-CCD kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/x2_ab.txt
for x in 1 0; do
  HJCD_POCCD_X2=$x timeout 300 python bench.py --no-sweep --no-cpu-baseline --steps 20 > gpurun_out/x2_ab_c2_$x.log 2>&1
  python - <<PY >> gpurun_out/x2_ab.txt
import json
d = json.loads([l for l in open("gpurun_out/x2_ab_c2_$x.log") if l.startswith("{")][0])
r = d["roofline"]
print("x2=$x c2 ms/step %.4f" % d["ms_per_step"], "k_poccd %.4f" % r["kernel_ms"]["k_poccd"], "frac %.4f" % r["frac"])
PY
done
HJCD_POCCD_X2=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_poccd" -s 1 -c 1 -o gpurun_out/prof_x2 -f python scripts/prof_c2.py c2 2 > gpurun_out/ncu_x2.log 2>&1
HJCD_POCCD_X2=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_poccd" -s 1 -c 1 -o gpurun_out/prof_x1 -f python scripts/prof_c2.py c2 2 > gpurun_out/ncu_x1.log 2>&1
echo done

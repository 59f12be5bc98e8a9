# usage: gpurun -- 'bash scripts/gpurun/env_ab.sh "CFGS" VAR "V1 V2 ..."'   bench lines per value of an environment variable
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CFGS="$1"; VAR="$2"; VALS="$3"
rm -f gpurun_out/env_ab.txt
for rep in 1 2; do
for v in $VALS; do
  for cfg in $CFGS; do
    st=20; [ $cfg != c2 ] && st=5
    env $VAR=$v timeout 300 python bench.py --config $cfg --no-sweep --no-cpu-baseline --steps $st > gpurun_out/env_last.log 2>&1
    python - "$VAR=$v" $cfg <<'PY' >> gpurun_out/env_ab.txt
import json, sys
try:
    d = json.loads([l for l in open("gpurun_out/env_last.log") if l.startswith("{")][0])
except Exception:
    print(sys.argv[1], sys.argv[2], "FAILED", open("gpurun_out/env_last.log").read()[-400:]); sys.exit()
r = d["roofline"]
print(sys.argv[1], sys.argv[2], "ms/step %.4f" % d["ms_per_step"], "k_poccd %.4f" % r["kernel_ms"]["k_poccd"], "k_pjik %.4f" % r["kernel_ms"]["k_pjik"], "frac %.4f" % r["frac"], "kernel", r["kernel"], "succ", d["success_rate_1mm_1deg"])
PY
  done
done
done
echo done

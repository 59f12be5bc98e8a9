# A/B of library variants built with paper_2510_07514_b200/build.py
# (build(defines=[...], lib=..._ab/libhjcd_<name>.so)): per-stage device times.
#   gpurun --timeout 1800 -- 'bash scripts/gpurun/ab.sh paper_2510_07514_b200/_ab/libhjcd_x.so ...'
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for L in paper_2510_07514_b200/libhjcd.so "$@"; do
  for cfg in c2 c3 c4; do HJCD_LIB=$L timeout 300 python scripts/time_stages.py $cfg 10 >> gpurun_out/ab.log 2>&1; done
done
echo done

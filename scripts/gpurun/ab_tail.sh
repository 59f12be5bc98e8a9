cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for L in paper_2510_07514_b200/libhjcd.so paper_2510_07514_b200/_ab/libhjcd_lpw16.so paper_2510_07514_b200/_ab/libhjcd_lpw8.so; do
  for cfg in c2 c3 c4; do HJCD_LIB=$L timeout 300 python scripts/time_stages.py $cfg 10 >> gpurun_out/ab.log 2>&1; done
  HJCD_LIB=$L timeout 300 python scripts/tail_latency.py >> gpurun_out/ab.log 2>&1
done
echo done

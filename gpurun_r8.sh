cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for L in paper_2510_07514_b200/libhjcd.so paper_2510_07514_b200/_ab/libhjcd_coop.so; do
  HJCD_LIB=$L timeout 300 python scripts/tail_latency.py >> gpurun_out/tail.log 2>&1
done
echo done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2; do
for L in paper_2510_07514_b200/_ab/libhjcd_v0.so paper_2510_07514_b200/_ab/libhjcd_v1.so paper_2510_07514_b200/_ab/libhjcd_v2.so paper_2510_07514_b200/libhjcd.so; do
  HJCD_LIB=$L timeout 300 python scripts/time_stages.py c2 20 >> gpurun_out/ab.log 2>&1
  HJCD_LIB=$L timeout 300 python scripts/time_stages.py c4 3 >> gpurun_out/ab.log 2>&1
done
done
echo done

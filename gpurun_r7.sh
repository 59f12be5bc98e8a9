cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for L in paper_2510_07514_b200/libhjcd.so paper_2510_07514_b200/_ab/libhjcd_coop.so paper_2510_07514_b200/_ab/libhjcd_cap1024.so; do
  HJCD_LIB=$L timeout 300 python scripts/time_stages.py c2 20 >> gpurun_out/ab.log 2>&1
  HJCD_LIB=$L timeout 300 python scripts/time_stages.py c3 5 >> gpurun_out/ab.log 2>&1
  HJCD_LIB=$L timeout 300 python scripts/time_stages.py c4 5 >> gpurun_out/ab.log 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=900 -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pjik" -s 1 -c 1 -o gpurun_out/prof_lanes -f python scripts/prof_c2.py c2 2 > gpurun_out/ncu_full.log 2>&1
echo done

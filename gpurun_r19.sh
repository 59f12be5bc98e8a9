cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for L in paper_2510_07514_b200/libhjcd.so paper_2510_07514_b200/_ab/libhjcd_minb3.so; do
  HJCD_LIB=$L timeout 300 python scripts/time_stages.py c2 20 >> gpurun_out/ab.log 2>&1
  HJCD_LIB=$L timeout 300 python scripts/time_stages.py c3 3 >> gpurun_out/ab.log 2>&1
  HJCD_LIB=$L timeout 300 python scripts/time_stages.py c4 3 >> gpurun_out/ab.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "pjik or solve" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
echo done

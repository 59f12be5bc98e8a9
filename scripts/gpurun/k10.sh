# dependent-launch (K10) check: new parity test first, then the step times, then the gpu suite
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k dependent_launch -x > gpurun_out/k10_test.log 2>&1; echo "rc=$?" >> gpurun_out/k10_test.log
for cfg in c2 c3 c4 c2_T300; do timeout 300 python scripts/pipe_ab.py $cfg 15 >> gpurun_out/k10_ab.log 2>&1; done
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=600 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
echo done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in c2 panda_x12 panda_x14 panda_x16 panda_x18 panda_x24; do timeout 300 python scripts/time_stages.py $cfg 5 >> gpurun_out/ab.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "other_chains or maximum or fk_jac" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
echo done

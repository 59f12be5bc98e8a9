cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do timeout 300 python scripts/time_stages.py c2 20 >> gpurun_out/ab.log 2>&1; done
timeout 300 python scripts/time_stages.py c3 3 >> gpurun_out/ab.log 2>&1
timeout 300 python scripts/time_stages.py c4 3 >> gpurun_out/ab.log 2>&1
timeout 300 python scripts/tail_latency.py >> gpurun_out/ab.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=900 -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
echo done

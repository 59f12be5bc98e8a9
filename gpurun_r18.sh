cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=900 -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for cfg in c3 c4 c5; do timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/bench_$cfg.log 2>&1; done
echo done

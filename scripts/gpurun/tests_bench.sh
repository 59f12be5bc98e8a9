# usage: gpurun -- 'bash scripts/gpurun/tests_bench.sh [<pytest -k expression>]'
# the -m gpu suite (printed numbers kept), then the default bench line and a C4 line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
if [ -n "$1" ]; then K=(-k "$1"); else K=(); fi
timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider --timeout=1200 -rf "${K[@]}" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --config c4 --no-sweep --no-cpu-baseline --steps 5 > gpurun_out/bench_c4.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c4.log
echo done

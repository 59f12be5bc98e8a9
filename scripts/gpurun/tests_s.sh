# usage: gpurun -- 'bash scripts/gpurun/tests_s.sh [<pytest -k expression>]'
# the -m gpu suite (or the selected tests) with the tests' printed numbers kept
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
if [ -n "$1" ]; then K=(-k "$1"); else K=(); fi
timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider --timeout=1200 -rf "${K[@]}" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
echo done

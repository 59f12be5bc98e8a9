# usage: gpurun -- 'bash scripts/gpurun/misc.sh'   ablation (f4), C5 on one GPU (100k targets), the per-seed parity prints
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/ablation.py 1000 > gpurun_out/ablation.log 2>&1
timeout 900 python bench.py --config c5 --no-sweep --no-cpu-baseline --steps 5 > gpurun_out/bench_c5_1gpu.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -s -p no:cacheprovider -k "per_seed_parity" > gpurun_out/pytest_perseed.log 2>&1
echo done

# The round's GPU evidence in one gpurun call (run from the repo root):
#   gpurun --timeout 3000 -- 'bash scripts/gpurun/round.sh'
# smoke, the -m gpu suite, the default bench line, the reference arm, a 2-rank
# functional run (gloo, ranks share the one GPU), the ncu launch list of the
# bench command and one full capture of the two stage kernels; then locally:
#   python scripts/ncu_summary.py rNN gpurun_out/prof_c2.ncu-rep gpurun_out/launches.csv
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1; nproc > gpurun_out/nproc.txt; lscpu | grep "Model name" >> gpurun_out/nproc.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider --timeout=900 -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1; echo "reference rc=$?" >> gpurun_out/bench_reference.log
HJCD_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --no-sweep --no-cpu-baseline --steps 5 > gpurun_out/bench_2rank_gloo.log 2>&1; echo "2-rank rc=$?" >> gpurun_out/bench_2rank_gloo.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_poccd|k_pjik" -s 2 -c 2 -o gpurun_out/prof_c2 -f python scripts/prof_c2.py c2 2 > gpurun_out/ncu_full.log 2>&1
echo done

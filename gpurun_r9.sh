cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/time_stages.py c2 20 >> gpurun_out/ab.log 2>&1
timeout 300 python scripts/time_stages.py c3 5 >> gpurun_out/ab.log 2>&1
timeout 300 python scripts/time_stages.py c4 5 >> gpurun_out/ab.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=900 -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_poccd|k_pjik" -s 2 -c 2 -o gpurun_out/prof_c2 -f python scripts/prof_c2.py c2 2 > gpurun_out/ncu_full.log 2>&1
echo done

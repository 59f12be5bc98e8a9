cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=900 -rf -k "cooperative or early_exit" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_poccd|k_pjik" -s 2 -c 2 -o gpurun_out/prof_c2_r6 python scripts/prof_c2.py c2 2 > gpurun_out/ncu_full.log 2>&1
echo done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pjik" -s 4 -c 1 -o gpurun_out/prof_tail -f python scripts/tail_latency.py > gpurun_out/ncu_tail.log 2>&1
echo done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_poccd" -s 1 -c 1 -o gpurun_out/prof_poccd -f python scripts/prof_c2.py c2 2 > gpurun_out/ncu_full.log 2>&1
echo done

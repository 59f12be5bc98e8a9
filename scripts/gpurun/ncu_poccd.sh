# usage: gpurun -- 'bash scripts/gpurun/ncu_poccd.sh [c2|c3|c4] [tag]'   one full ncu capture of the C2 PO-CCD kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_poccd" -s 1 -c 1 -o gpurun_out/prof_${2:-poccd} -f python scripts/prof_c2.py ${1:-c2} 2 > gpurun_out/ncu_${2:-poccd}.log 2>&1
echo done

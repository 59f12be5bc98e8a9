cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/diversity.py 100 > gpurun_out/diversity.log 2>&1
echo done

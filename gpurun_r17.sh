cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
HJCD_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_2rank.log 2>&1; echo "rc=$?" >> gpurun_out/bench_2rank.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 1 --warmup 0 > gpurun_out/ref_2rank.log 2>&1; echo "rc=$?" >> gpurun_out/ref_2rank.log
echo done

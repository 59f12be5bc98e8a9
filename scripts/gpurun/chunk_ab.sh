# K22 chunked-chain A/B: step time and bitwise equality vs the staged path per chunk size
#   gpurun -- 'bash scripts/gpurun/chunk_ab.sh "CHUNKS" "CFGS" [pytest -k expr]'
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CHS=${1:-"-1 296"}; CFGS=${2:-"c2 c3 c4"}
for rep in 1 2; do
for cfg in $CFGS; do
  for ch in $CHS; do
    echo -n "chunk=$ch " >> gpurun_out/chunk_ab.log
    HJCD_CHUNK=$ch timeout 300 python scripts/pipe_ab.py $cfg 15 >> gpurun_out/chunk_ab.log 2>&1
  done
done
done
if [ -n "$3" ]; then
timeout 1200 python -m pytest tests -m gpu -q -s -p no:cacheprovider -k "$3" -rf > gpurun_out/pytest_sel.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sel.log
fi
echo done

# bitwise + step-time A/B of the working library against one saved build:
#   gpurun -- 'bash scripts/gpurun/ab2.sh paper_2510_07514_b200/_ab/libhjcd_X.so [cfgs...]'
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
REF=$1; shift
CFGS=${@:-c2 c3 c4}
HJCD_LIB=$REF timeout 300 python scripts/ab_bitwise.py save /tmp/ref.npz > gpurun_out/ab2.log 2>&1
echo "current vs $(basename $REF):" >> gpurun_out/ab2.log
timeout 300 python scripts/ab_bitwise.py cmp /tmp/ref.npz >> gpurun_out/ab2.log 2>&1
for cfg in $CFGS; do
  for lib in $REF paper_2510_07514_b200/libhjcd.so; do
    echo -n "$(basename $lib) " >> gpurun_out/ab2.log
    HJCD_LIB=$lib timeout 300 python scripts/pipe_ab.py $cfg 15 >> gpurun_out/ab2.log 2>&1
  done
done
echo done

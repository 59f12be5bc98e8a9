cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=paper_2510_07514_b200/_ab
HJCD_LIB=$L/libhjcd_k12.so timeout 300 python scripts/ab_bitwise.py save /tmp/ref.npz > gpurun_out/lpw.log 2>&1
for lib in paper_2510_07514_b200/libhjcd.so $L/libhjcd_lpw16.so; do echo "$(basename $lib) vs k12:" >> gpurun_out/lpw.log; HJCD_LIB=$lib timeout 300 python scripts/ab_bitwise.py cmp /tmp/ref.npz >> gpurun_out/lpw.log 2>&1; done
for cfg in c2 c3 c4; do
  for lib in $L/libhjcd_k12.so paper_2510_07514_b200/libhjcd.so $L/libhjcd_lpw20.so $L/libhjcd_lpw16.so $L/libhjcd_lpw13.so; do
    echo -n "$(basename $lib) " >> gpurun_out/lpw.log
    HJCD_LIB=$lib timeout 300 python scripts/pipe_ab.py $cfg 15 >> gpurun_out/lpw.log 2>&1
  done
done
echo done

# K11 (Rx-form FK) + clamped-orientation closed form: bitwise A/B and step times
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=paper_2510_07514_b200/_ab
HJCD_LIB=$L/libhjcd_norx.so timeout 300 python scripts/ab_bitwise.py save /tmp/norx.npz > gpurun_out/k11.log 2>&1
echo "cur vs norx:" >> gpurun_out/k11.log
timeout 300 python scripts/ab_bitwise.py cmp /tmp/norx.npz >> gpurun_out/k11.log 2>&1
for cfg in c2 c3 c4; do
  for lib in $L/libhjcd_prev.so $L/libhjcd_norx.so paper_2510_07514_b200/libhjcd.so; do
    echo -n "$(basename $lib) " >> gpurun_out/k11.log
    HJCD_LIB=$lib timeout 300 python scripts/pipe_ab.py $cfg 15 >> gpurun_out/k11.log 2>&1
  done
done
echo done

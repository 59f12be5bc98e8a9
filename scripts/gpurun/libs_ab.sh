# step times of several library builds (no bitwise check):
#   gpurun -- 'bash scripts/gpurun/libs_ab.sh "c2 c3" lib1.so lib2.so ...'
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CFGS=$1; shift
: > gpurun_out/libs_ab.log
for cfg in $CFGS; do
  for lib in paper_2510_07514_b200/libhjcd.so "$@"; do
    echo -n "$(basename $lib) " >> gpurun_out/libs_ab.log
    HJCD_LIB=$lib timeout 300 python scripts/pipe_ab.py $cfg 15 >> gpurun_out/libs_ab.log 2>&1
  done
done
echo done

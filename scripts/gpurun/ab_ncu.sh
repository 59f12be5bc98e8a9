# usage: gpurun -- 'bash scripts/gpurun/ab_ncu.sh "CFGS" TAG LIB...'   A/B lines, then one full ncu capture of the C2 PO-CCD kernel (in-tree build)
cd $GRAFT_REPO_ROOT
CFGS="$1"; TAG="$2"; shift; shift
bash scripts/gpurun/libs_cfgs.sh "$CFGS" "$@"
unset HJCD_LIB
bash scripts/gpurun/ncu_poccd.sh c2 "$TAG"

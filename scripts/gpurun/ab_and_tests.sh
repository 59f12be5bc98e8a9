# usage: gpurun -- 'bash scripts/gpurun/ab_and_tests.sh "CFGS" LIB...'   A/B lines, then the -m gpu suite on the in-tree build
cd $GRAFT_REPO_ROOT
CFGS="$1"; shift
bash scripts/gpurun/libs_cfgs.sh "$CFGS" "$@"
bash scripts/gpurun/tests_s.sh

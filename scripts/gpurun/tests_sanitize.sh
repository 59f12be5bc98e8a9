# usage: gpurun -- 'bash scripts/gpurun/tests_sanitize.sh'   the -m gpu suite, then compute-sanitizer
cd $GRAFT_REPO_ROOT
bash scripts/gpurun/tests_s.sh
bash scripts/gpurun/sanitize.sh

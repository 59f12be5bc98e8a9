# usage: gpurun -- 'bash scripts/gpurun/sanitize.sh'   compute-sanitizer over every solve path
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/sanitizer.log
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool" >> gpurun_out/sanitizer.log
  timeout 900 compute-sanitizer --tool $tool python scripts/sanitize_small.py >> gpurun_out/sanitizer.log 2>&1
done
echo done

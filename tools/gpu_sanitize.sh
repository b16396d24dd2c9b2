# compute-sanitizer over the small-shape workload (every kernel family once); summaries -> gpurun_out/sanitize_*.txt
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r2}
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_run.py \
    > gpurun_out/sanitize_${tool}_${TAG}.txt 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitize_${tool}_${TAG}.txt
done

cd $GRAFT_REPO_ROOT
TAG=${TAG:-r2u}
timeout 300 python tools/time_decode.py 1 16 64 > gpurun_out/time_decode_${TAG}.txt 2>&1; echo td rc=$?; cat gpurun_out/time_decode_${TAG}.txt | tail -4
timeout 300 python tools/time_prologue.py > gpurun_out/time_prologue_${TAG}.txt 2>&1; echo tp rc=$?; cat gpurun_out/time_prologue_${TAG}.txt | tail -7
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/sanitize_racecheck_${TAG}.txt 2>&1; echo race rc=$?; tail -3 gpurun_out/sanitize_racecheck_${TAG}.txt
timeout 2400 python -m pytest tests -q -m gpu --timeout 600 -x > gpurun_out/pytest_gpu_${TAG}.txt 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu_${TAG}.txt
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo bench rc=$?; head -c 600 gpurun_out/bench_${TAG}.json

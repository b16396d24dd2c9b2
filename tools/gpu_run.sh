# generic: optional micro, parity tests, bench (default workload + extras)
set -x
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r1}
if [ -n "$MICRO" ]; then timeout 120 ./bench/micro/$MICRO > gpurun_out/micro_${MICRO}_${TAG}.txt 2>&1; echo micro rc=$?; cat gpurun_out/micro_${MICRO}_${TAG}.txt; fi
if [ -z "$NOTEST" ]; then
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 300 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu_${TAG}.txt 2>&1; echo pytest rc=$?; tail -15 gpurun_out/pytest_gpu_${TAG}.txt
fi
timeout 900 python bench.py --steps ${STEPS:-20} --warmup 5 ${BENCH_ARGS} > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo bench rc=$?
cat gpurun_out/bench_${TAG}.json; tail -5 gpurun_out/bench_${TAG}.err

# round-2 baseline: smoke, GPU tests, default bench line (with clocks), launch list
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r2a}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; nproc
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.txt 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke_${TAG}.txt
timeout 1200 python -m pytest tests -q -m gpu -x --timeout 300 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu_${TAG}.txt 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest_gpu_${TAG}.txt
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo bench rc=$?
cat gpurun_out/bench_${TAG}.json; tail -3 gpurun_out/bench_${TAG}.err

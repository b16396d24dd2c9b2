# final check of HEAD: smoke, the whole GPU suite, one default bench line
cd $GRAFT_REPO_ROOT
TAG=${TAG:-final}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.txt 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke_${TAG}.txt
timeout 2400 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest_gpu_${TAG}.txt 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu_${TAG}.txt
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo bench rc=$?; head -c 400 gpurun_out/bench_${TAG}.json

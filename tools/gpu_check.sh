set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
timeout 120 ./bench/micro/micro > gpurun_out/micro.txt 2>&1; echo micro rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo smoke rc=$?; tail -20 gpurun_out/smoke.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1; echo pytest rc=$?; tail -40 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench rc=$?
cat gpurun_out/bench_c2.json; tail -5 gpurun_out/bench_c2.err

cd $GRAFT_REPO_ROOT
TAG=${TAG:-r2b}
timeout 900 python -m pytest tests/test_gpu_parity_r2.py tests/test_gpu_parity.py -q -m gpu -x --timeout 400 -k "${PYTEST_K:-r2 or prologue_bitexact or end_to_end or invalid}" > gpurun_out/pytest_${TAG}.txt 2>&1; echo pytest rc=$?; tail -15 gpurun_out/pytest_${TAG}.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c4_${TAG}.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --also "" --workload c4_decode_t64 > /dev/null 2>&1; echo ncu rc=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c4t1_${TAG}.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --also "" --workload c4_decode_t1 > /dev/null 2>&1; echo ncu rc=$?

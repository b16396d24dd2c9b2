cd $GRAFT_REPO_ROOT
./tools/decode_trace 64 0 2>&1 | tail -16
./tools/decode_trace 64 1 2>&1 | tail -16
./tools/decode_trace 64 2 2>&1 | tail -22
./tools/decode_trace 1 2 2>&1 | tail -22
./bench/micro/prologue_trace 4096 4096 1 2>&1 | tail -10
timeout 300 python tools/time_prologue.py c2_llama2_7b_qo c3_llama3_8b_up c5_llama3_70b_up_rank8 c4_decode_t64 c4_decode_t1 2>&1 | tail -6
timeout 300 python tools/time_decode.py 1 64 2>&1 | tail -2
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py tests/test_gpu_decode.py -q -m gpu --timeout 600 -x > gpurun_out/pytest_r2y.txt 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_r2y.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2y.json 2> gpurun_out/bench_r2y.err; echo bench rc=$?; head -c 1500 gpurun_out/bench_r2y.json

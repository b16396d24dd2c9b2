cd $GRAFT_REPO_ROOT
./tools/decode_trace 64 2>&1 | tail -20
./tools/decode_trace 1 2>&1 | tail -12
./bench/micro/prologue_trace 64 8192 2 2>&1 | tail -12
timeout 300 python tools/time_decode.py 1 16 64 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_decode.py -q -m gpu --timeout 400 -x 2>&1 | tail -5
timeout 2400 python -m pytest tests -q -m gpu --timeout 600 -x > gpurun_out/pytest_gpu_r2w.txt 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu_r2w.txt

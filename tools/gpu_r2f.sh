cd $GRAFT_REPO_ROOT
./tools/decode_trace 64 > gpurun_out/dtrace_r2f.txt 2>&1; ./tools/decode_trace 1 >> gpurun_out/dtrace_r2f.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_decode.py -q -m gpu -x --timeout 300 > gpurun_out/pytest_r2f.txt 2>&1; echo pytest rc=$?; tail -20 gpurun_out/pytest_r2f.txt
timeout 300 python tools/time_decode.py 1 16 64 2>&1 | tail -5

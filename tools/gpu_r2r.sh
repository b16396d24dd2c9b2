cd $GRAFT_REPO_ROOT
./tools/decode_trace 64 | head -9; ./tools/decode_trace 1 | head -9
timeout 300 python tools/time_decode.py 1 16 64 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_decode.py -q -m gpu --timeout 400 -x > gpurun_out/pytest_r2r.txt 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_r2r.txt

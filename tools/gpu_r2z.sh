cd $GRAFT_REPO_ROOT
./tools/decode_trace 64 0 2>&1 | tail -16
./tools/decode_trace 64 2 2>&1 | tail -20
./tools/decode_trace 64 3 2>&1 | tail -20
./tools/decode_trace 1 2 2>&1 | tail -20
./tools/decode_trace 1 3 2>&1 | tail -20
timeout 300 python tools/time_decode.py 1 16 64 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_decode.py -q -m gpu --timeout 400 -x 2>&1 | tail -3

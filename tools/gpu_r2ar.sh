cd $GRAFT_REPO_ROOT
timeout 300 python tools/time_decode.py 1 16 64 2>&1 | tail -3
./tools/decode_trace 64 2 2>&1 | grep -E "^CTA 0|prologue slot 6|rep 3"
timeout 900 python -m pytest tests/test_gpu_decode.py -q -m gpu --timeout 400 -x 2>&1 | tail -2

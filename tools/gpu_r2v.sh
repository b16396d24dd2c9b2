cd $GRAFT_REPO_ROOT
./tools/decode_trace 64 2>&1 | tail -22
./tools/decode_trace 1 2>&1 | tail -22
./bench/micro/prologue_trace 64 8192 2 2>&1 | tail -16
./bench/micro/prologue_trace 1 8192 2 2>&1 | tail -16
timeout 300 python tools/time_decode.py 1 64 2>&1 | tail -3

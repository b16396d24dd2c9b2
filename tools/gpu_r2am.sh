cd $GRAFT_REPO_ROOT
./bench/micro/prologue_trace 4096 4096 1 2>&1 | grep -E "rep 2|slot  [234]"
./bench/micro/prologue_trace 2048 4096 1 2>&1 | grep -E "rep 2|slot  [234]"
timeout 300 python tools/time_prologue.py c2_llama2_7b_qo c3_llama3_8b_up c4_decode_t64 c4_decode_t1 2>&1 | tail -4
timeout 300 python tools/time_decode.py 1 64 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py tests/test_gpu_decode.py -q -m gpu --timeout 600 -x -k "prologue or rotate or linear or full or decode" > gpurun_out/pytest_r2am.txt 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_r2am.txt

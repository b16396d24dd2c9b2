cd $GRAFT_REPO_ROOT
./tools/decode_trace 64 0 2>&1 | tail -7
./tools/decode_trace 64 2 2>&1 | tail -24
./tools/decode_trace 1 2 2>&1 | tail -22
./bench/micro/prologue_trace 4096 4096 1 2>&1 | tail -8
timeout 300 python tools/time_prologue.py c2_llama2_7b_qo c3_llama3_8b_up c5_llama3_70b_up_rank8 c4_decode_t64 c4_decode_t1 2>&1 | tail -6
timeout 300 python tools/time_decode.py 1 16 64 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_parity.py -q -m gpu --timeout 600 -x -k "prologue or rotate or decode or linear" > gpurun_out/pytest_r2ab.txt 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_r2ab.txt
timeout 600 ncu --set full --import-source on --kernel-name regex:prologue_group_kernel --launch-skip 3 --launch-count 1 -f -o gpurun_out/prof_prologue_r2ab python tools/time_prologue.py c3_llama3_8b_up > gpurun_out/ncu_r2ab.log 2>&1; echo ncu rc=$?; tail -2 gpurun_out/ncu_r2ab.log

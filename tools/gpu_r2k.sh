cd $GRAFT_REPO_ROOT
TAG=${TAG:-r2k}
./tools/decode_trace 64 > gpurun_out/dtrace_${TAG}.txt 2>&1
for a in "1 8192 2" "64 8192 2"; do echo "== prologue_trace $a"; timeout 60 ./bench/micro/prologue_trace $a; done > gpurun_out/ptrace_${TAG}.txt 2>&1
timeout 600 python tools/time_prologue.py > gpurun_out/time_prologue_${TAG}.txt 2>&1; cat gpurun_out/time_prologue_${TAG}.txt | tail -5
timeout 300 python tools/time_decode.py 1 64 2>&1 | tail -3
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py tests/test_gpu_decode.py -q -m gpu --timeout 400 -x > gpurun_out/pytest_${TAG}.txt 2>&1; echo pytest rc=$?; tail -8 gpurun_out/pytest_${TAG}.txt

cd $GRAFT_REPO_ROOT
TAG=${TAG:-r2o}
for a in "1 8192 2" "64 8192 2"; do echo "== prologue_trace $a"; timeout 60 ./bench/micro/prologue_trace $a; done > gpurun_out/ptrace_${TAG}.txt 2>&1
./tools/decode_trace 64 > gpurun_out/dtrace_${TAG}.txt 2>&1
timeout 300 python tools/time_decode.py 1 16 64 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_decode.py -q -m gpu --timeout 400 -x > gpurun_out/pytest_${TAG}.txt 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_${TAG}.txt

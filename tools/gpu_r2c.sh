cd $GRAFT_REPO_ROOT
TAG=${TAG:-r2c}
for a in "1 8192 1" "64 8192 1" "2048 4096 1" "64 8192 0"; do echo "== prologue_trace $a"; timeout 60 ./bench/micro/prologue_trace $a; done > gpurun_out/trace_${TAG}.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity_r2.py -q -m gpu -x --timeout 400 > gpurun_out/pytest_${TAG}.txt 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest_${TAG}.txt

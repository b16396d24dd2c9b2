cd $GRAFT_REPO_ROOT
TAG=${TAG:-r2d}
timeout 600 python -m pytest tests/test_gpu_decode.py -q -m gpu -x --timeout 300 > gpurun_out/pytest_${TAG}.txt 2>&1; echo pytest rc=$?; tail -30 gpurun_out/pytest_${TAG}.txt
timeout 300 python tools/time_decode.py 1 16 64 2>&1 | tail -5

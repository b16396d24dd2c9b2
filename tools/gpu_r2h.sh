cd $GRAFT_REPO_ROOT
TAG=${TAG:-r2h}
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_variants.py tests/test_gpu_parity_r2.py -q -m gpu --timeout 300 > gpurun_out/pytest_${TAG}.txt 2>&1; echo pytest rc=$?; tail -25 gpurun_out/pytest_${TAG}.txt
timeout 300 python tools/time_decode.py 1 16 64 2>&1 | tail -5
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_dec_${TAG}.csv python tools/time_decode.py 1 64 > /dev/null 2>&1; echo ncu rc=$?

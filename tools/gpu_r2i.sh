cd $GRAFT_REPO_ROOT
TAG=${TAG:-r2i}
./tools/decode_trace 64 > gpurun_out/dtrace_${TAG}.txt 2>&1; ./tools/decode_trace 1 >> gpurun_out/dtrace_${TAG}.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_variants.py tests/test_gpu_multigpu.py -q -m gpu --timeout 300 -x > gpurun_out/pytest_${TAG}.txt 2>&1; echo pytest rc=$?; tail -25 gpurun_out/pytest_${TAG}.txt
timeout 300 python tools/time_decode.py 1 16 64 2>&1 | tail -5
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_dec_${TAG}.csv python tools/time_decode.py 1 64 > /dev/null 2>&1; echo ncu rc=$?

cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py tests/test_gpu_variants.py -q -m gpu --timeout 600 -x > gpurun_out/pytest_r2al.txt 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_r2al.txt
timeout 300 python tools/time_prologue.py c2_llama2_7b_qo c3_llama3_8b_up c3_llama3_8b_down 2>&1 | tail -3

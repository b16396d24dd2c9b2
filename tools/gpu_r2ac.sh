cd $GRAFT_REPO_ROOT
./bench/micro/prologue_trace 4096 4096 1 2>&1 | tail -8
timeout 300 python tools/time_prologue.py c2_llama2_7b_qo c3_llama3_8b_up c5_llama3_70b_up_rank8 c3_llama3_8b_down c4_decode_t64 c4_decode_t1 2>&1 | tail -6
./tools/decode_trace 64 1 2>&1 | tail -7
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -q -m gpu --timeout 600 -x -k "prologue or rotate or linear or full" > gpurun_out/pytest_r2ac.txt 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_r2ac.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2ac.json 2> gpurun_out/bench_r2ac.err; echo bench rc=$?; python -c "
import json; d=json.load(open('gpurun_out/bench_r2ac.json')); print(d['value'], d['breakdown_ms']); print({k:(v.get('tops'),v.get('ms_per_step')) for k,v in d.get('also',{}).items()})"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:prologue_group_kernel --launch-skip 3 --launch-count 1 -f -o gpurun_out/prof_prologue_r2ac python tools/time_prologue.py c3_llama3_8b_up > gpurun_out/ncu_r2ac.log 2>&1; echo ncu rc=$?

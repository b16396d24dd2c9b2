cd $GRAFT_REPO_ROOT
timeout 300 python tools/time_prologue.py c2_llama2_7b_qo c3_llama3_8b_up c3_llama3_8b_down c4_decode_t64 c4_decode_t1 2>&1 | tail -5
timeout 1800 python -m pytest tests -q -m gpu --timeout 600 -x > gpurun_out/pytest_gpu_r2ao.txt 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu_r2ao.txt
timeout 900 python bench.py > gpurun_out/bench_r2ao.json 2> gpurun_out/bench_r2ao.err; echo bench rc=$?; python -c "
import json; d=json.load(open('gpurun_out/bench_r2ao.json')); print(d['value'], d['breakdown_ms']['prologue'], d['breakdown_ms']['rrs_gemm'], d['roofline']['frac']); print({k:(round(v.get('tops') or 0,1), v.get('ms_per_step')) for k,v in d.get('also',{}).items()})"

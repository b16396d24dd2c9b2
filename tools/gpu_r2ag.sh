cd $GRAFT_REPO_ROOT
timeout 300 python tools/time_decode.py 1 16 64 2>&1 | tail -3
timeout 300 python tools/time_prologue.py c2_llama2_7b_qo c3_llama3_8b_up c3_llama3_8b_down c4_decode_t64 c4_decode_t1 2>&1 | tail -5
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2ag.json 2> gpurun_out/bench_r2ag.err; echo bench rc=$?; python -c "
import json; d=json.load(open('gpurun_out/bench_r2ag.json')); print(d['value'], d['ms_per_step'], d['breakdown_ms'], d['e2e']); print({k:(v.get('tops'),v.get('ms_per_step'), v.get('breakdown_ms')) for k,v in d.get('also',{}).items()})"

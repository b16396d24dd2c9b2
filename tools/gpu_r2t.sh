cd $GRAFT_REPO_ROOT
TAG=${TAG:-r2t}
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -q -m gpu --timeout 400 -x -k "i8 or plain or partials" > gpurun_out/pytest_${TAG}.txt 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_${TAG}.txt
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --workload c3_llama3_8b_up --also c3_llama3_8b_up_i8 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_${TAG}.json')); print('e4m3', d['value'], d['breakdown_ms']['rrs_gemm'], d['breakdown_ms']['plain_gemm'])
v=d['also']['c3_llama3_8b_up_i8']; print('i8', v['tops'], v['breakdown_ms']['rrs_gemm'], v['breakdown_ms']['plain_gemm'])"
timeout 600 ncu --replay-mode application --set full --clock-control none --import-source on -k regex:prologue_decode -s 2 -c 1 -o gpurun_out/prof_prologue_decode_${TAG} python tools/time_decode.py 64 > gpurun_out/ncu_pd_${TAG}.log 2>&1; echo ncu pd rc=$?; tail -3 gpurun_out/ncu_pd_${TAG}.log
TAG=${TAG} bash tools/gpu_sanitize.sh

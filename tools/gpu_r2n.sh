cd $GRAFT_REPO_ROOT
TAG=${TAG:-r2n}
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --also c3_llama3_8b_down,c2_llama2_7b_qo > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo bench rc=$?; tail -2 gpurun_out/bench_${TAG}.err
python - <<'PY'
import json
d=json.load(open("gpurun_out/bench_r2n.json"))
print("head", d["value"], d["breakdown_ms"], d["rrs_overhead_vs_plain_gemm"])
for k,v in d.get("also",{}).items(): print(k, v.get("tops"), v.get("breakdown_ms"), v.get("rrs_overhead_vs_plain_gemm"))
PY
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py tests/test_gpu_multigpu.py -q -m gpu --timeout 400 -x > gpurun_out/pytest_${TAG}.txt 2>&1; echo pytest rc=$?; tail -6 gpurun_out/pytest_${TAG}.txt

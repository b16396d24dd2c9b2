# Round-2 evidence: smoke, full GPU tests, default bench (with cpu_baseline), reference arm, launch list of the
# bench command, ncu --set full of the hot kernels (headline GEMM + fused prologue, decode GEMM + decode prologue)
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r2}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; nproc
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.txt 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke_${TAG}.txt
if [ -z "$SKIP_TESTS" ]; then
timeout 2400 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest_gpu_${TAG}.txt 2>&1; echo pytest rc=$?; tail -4 gpurun_out/pytest_gpu_${TAG}.txt
fi
timeout 1200 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo bench rc=$?; tail -2 gpurun_out/bench_${TAG}.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err; echo ref rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --also c4_decode_t64,c4_decode_t1 > /dev/null 2>&1; echo launches rc=$?
for K in rrs_gemm_kernel prologue_group; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/prof_${K}_${TAG} python bench.py --steps 3 --warmup 3 --no-cpu-baseline --also "" > /dev/null 2>&1; echo ncu $K rc=$?
done
for K in rrs_decode_gemm prologue_decode; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/prof_${K}_${TAG} python bench.py --steps 3 --warmup 3 --no-cpu-baseline --also "" --workload c4_decode_t64 > /dev/null 2>&1; echo ncu $K rc=$?
done
ls gpurun_out

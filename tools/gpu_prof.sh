# parity subset + bench + ncu launch list + full captures of the named kernels
set -x
cd $GRAFT_REPO_ROOT
WL=${WL:-c2_llama2_7b_qo}; TAG=${TAG:-r1}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 300 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.txt 2>&1; echo pytest rc=$?; tail -15 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --workload $WL ${BENCH_ARGS} > gpurun_out/bench_${WL}_${TAG}.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench_${WL}_${TAG}.json; tail -5 gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_${WL}_${TAG}.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --workload $WL > /dev/null 2>&1; echo ncu1 rc=$?
for K in ${KERNELS:-fwht_colmax smooth_quant rrs_gemm_kernel}; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/prof_${K}_${WL}_${TAG} python bench.py --steps 3 --warmup 3 --no-cpu-baseline --workload $WL > /dev/null 2>&1; echo ncu $K rc=$?
done

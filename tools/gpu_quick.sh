# fast GEMM sanity (short timeouts: a hung kernel must not hang the box), then the full GPU suite + bench
set -x
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r1}
timeout 180 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 60 -k "partials or plain or rrs_gemm_y" > gpurun_out/pytest_quick_${TAG}.txt 2>&1; rc=$?; echo quick rc=$rc; tail -15 gpurun_out/pytest_quick_${TAG}.txt
if [ $rc -ne 0 ]; then exit 1; fi
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 300 > gpurun_out/pytest_gpu_${TAG}.txt 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest_gpu_${TAG}.txt
timeout 900 python bench.py --steps ${STEPS:-20} --warmup 5 ${BENCH_ARGS} > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo bench rc=$?
cat gpurun_out/bench_${TAG}.json; tail -5 gpurun_out/bench_${TAG}.err
if [ -n "$LAUNCHES" ]; then
for WL in $LAUNCHES; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_${WL}_${TAG}.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --also "" --workload $WL > /dev/null 2>&1; echo ncu $WL rc=$?
done
fi

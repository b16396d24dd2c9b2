# round evidence: default bench (with cpu_baseline), reference arm, smoke, launch list of the bench command,
# ncu --set full of the hot kernels of the headline workload
set -x
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r1}
WL=${WL:-c3_llama3_8b_up}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; nproc
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.txt 2>&1; echo smoke rc=$?; tail -3 gpurun_out/smoke_${TAG}.txt
timeout 900 python bench.py > gpurun_out/bench_default_${TAG}.json 2> gpurun_out/bench_default_${TAG}.err; echo bench rc=$?
cat gpurun_out/bench_default_${TAG}.json; tail -3 gpurun_out/bench_default_${TAG}.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err; echo ref rc=$?
cat gpurun_out/bench_ref_${TAG}.json; tail -3 gpurun_out/bench_ref_${TAG}.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_${WL}_${TAG}.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --also "" --workload $WL > /dev/null 2>&1; echo launches rc=$?
for K in ${KERNELS:-rrs_gemm_kernel prologue_fused}; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/prof_${K}_${WL}_${TAG} python bench.py --steps 3 --warmup 3 --no-cpu-baseline --also "" --workload $WL > /dev/null 2>&1; echo ncu $K rc=$?
done
ls gpurun_out

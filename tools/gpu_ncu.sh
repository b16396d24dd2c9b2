# ncu evidence for one workload: launch list (timing shares) + one --set full capture per hot kernel
set -x
cd $GRAFT_REPO_ROOT
WL=${1:-c2_llama2_7b_qo}
TAG=${2:-r1}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_${WL}_${TAG}.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --workload $WL > /dev/null 2>&1; echo ncu1 rc=$?
for K in fwht_colmax fwht_quant rrs_gemm_kernel; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/prof_${K}_${WL}_${TAG} python bench.py --steps 3 --warmup 3 --no-cpu-baseline --workload $WL > /dev/null 2>&1; echo ncu $K rc=$?
done
ls -la gpurun_out

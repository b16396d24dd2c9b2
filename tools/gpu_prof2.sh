# ncu --set full captures: $PROF = "kernel_regex:workload ..." (one bench process per capture)
set -x
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r1}
for KW in $PROF; do
K=${KW%%:*}; WL=${KW##*:}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o gpurun_out/prof_${K}_${WL}_${TAG} python bench.py --steps 3 --warmup 3 --no-cpu-baseline --also "" --workload $WL > /dev/null 2>&1; echo ncu $K $WL rc=$?
done

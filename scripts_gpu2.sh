set -x
cd $GRAFT_REPO_ROOT
python -m paper_2409_20361_b200.build >/dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -15
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo rc=$?
cat gpurun_out/bench_c2.json; tail -5 gpurun_out/bench_c2.err
timeout 600 python bench.py --steps 10 --warmup 3 --workload c3_llama3_8b_up --no-cpu-baseline > gpurun_out/bench_c3up.json 2>&1; cat gpurun_out/bench_c3up.json | tail -3
timeout 600 python bench.py --steps 10 --warmup 3 --workload c3_llama3_8b_down --no-cpu-baseline > gpurun_out/bench_c3down.json 2>&1; cat gpurun_out/bench_c3down.json | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rrs_gemm_kernel -s 2 -c 1 -o gpurun_out/prof_gemm_c2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu2 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwht -s 4 -c 2 -o gpurun_out/prof_fwht_c2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu3 rc=$?
ls -la gpurun_out

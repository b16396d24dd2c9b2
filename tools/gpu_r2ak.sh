cd $GRAFT_REPO_ROOT
timeout 300 python tools/time_prologue.py c5_llama3_70b_up_rank8 c3_llama3_8b_down 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:"fwht_colmax_kernel|smooth_quant_kernel" --launch-skip 4 --launch-count 2 -f -o gpurun_out/prof_down_r2ak python tools/time_prologue.py c3_llama3_8b_down > gpurun_out/ncu_r2ak.log 2>&1; echo ncu rc=$?

cd $GRAFT_REPO_ROOT
TAG=${TAG:-r2p}
for a in "64 8192 2"; do echo "== prologue_trace $a"; timeout 60 ./bench/micro/prologue_trace $a; done > gpurun_out/ptrace_${TAG}.txt 2>&1
./tools/decode_trace 64 > gpurun_out/dtrace_${TAG}.txt 2>&1
timeout 300 python tools/time_decode.py 1 64 2>&1 | tail -3

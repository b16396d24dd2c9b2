#!/bin/bash
# Build the timeline harnesses (tools/decode_trace, bench/micro/prologue_trace) for sm_100a, from anywhere.
set -e
R="$(cd "$(dirname "$0")/.." && pwd)"
C=$R/paper_2409_20361_b200/csrc
NL=$(python -c "import nvidia.nccl,os;print(os.path.join(list(nvidia.nccl.__path__)[0],'lib'))")
NI=$(python -c "import nvidia.nccl,os;print(os.path.join(list(nvidia.nccl.__path__)[0],'include'))")
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DRRS_TRACE -I$R/include -I$NI"
L="-lcuda -L$NL -l:libnccl.so.2 -Xlinker -rpath=$NL"
nvcc $F -o $R/tools/decode_trace $R/tools/decode_trace.cu $C/api.cu $C/prologue.cu $C/gemm.cu $L &
nvcc $F -o $R/bench/micro/prologue_trace $R/bench/micro/prologue_trace.cu $C/api.cu $C/gemm.cu $C/decode.cu $L &
wait
nvcc $F -DRRS_GROUP_B6_MIN_K=1073741824 -o $R/bench/micro/prologue_trace_b5 $R/bench/micro/prologue_trace.cu $C/api.cu $C/gemm.cu $C/decode.cu $L
nvcc $F -DRRS_FWHT_BITWIDEN=1 -o $R/bench/micro/prologue_trace_bits $R/bench/micro/prologue_trace.cu $C/api.cu $C/gemm.cu $C/decode.cu $L
nvcc $F -DRRS_GROUP_CLUSTER=4 -o $R/bench/micro/prologue_trace_c4 $R/bench/micro/prologue_trace.cu $C/api.cu $C/gemm.cu $C/decode.cu $L

#!/bin/bash
# Build the microbenchmarks / timeline harnesses (sm_100a).  Run from anywhere.
set -e
cd "$(dirname "$0")"
NL=$(python -c "import nvidia.nccl,os;print(os.path.join(list(nvidia.nccl.__path__)[0],'lib'))")
NI=$(python -c "import nvidia.nccl,os;print(os.path.join(list(nvidia.nccl.__path__)[0],'include'))")
ARCH="-gencode arch=compute_100a,code=sm_100a"
C=../../paper_2409_20361_b200/csrc
nvcc $ARCH -O3 -o micro micro.cu
nvcc $ARCH -O3 -o tma_bw tma_bw.cu -lcuda
nvcc $ARCH -O3 -std=c++17 -DRRS_TRACE -I../../include -I$NI -o gemm_trace gemm_trace.cu $C/api.cu $C/prologue.cu \
  -lcuda -L$NL -l:libnccl.so.2 -Xlinker -rpath=$NL
nvcc $ARCH -O3 -std=c++17 -DRRS_TRACE -I../../include -I$NI -o prologue_trace prologue_trace.cu $C/api.cu $C/gemm.cu \
  -lcuda -L$NL -l:libnccl.so.2 -Xlinker -rpath=$NL
nvcc $ARCH -O3 -std=c++17 -I../../include -I$NI -o gemm_time gemm_time.cu $C/api.cu $C/prologue.cu \
  -lcuda -L$NL -l:libnccl.so.2 -Xlinker -rpath=$NL

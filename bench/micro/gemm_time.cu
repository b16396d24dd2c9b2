// Median time of the RRS / plain GEMM over a sweep of shapes (no timeline instrumentation), to separate the
// per-group cost from the per-tile cost.  Build: see build.sh.  Usage: gemm_time [T N K plain]...
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cstdlib>
#include "../../paper_2409_20361_b200/csrc/gemm.cu"

int main(int argc, char** argv) {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int64_t TM = 8192, NM = 28672, KM = 16384;
  int8_t *X, *W; float *xs, *sg, *ws; uint16_t* Y;
  cudaMalloc(&X, TM * KM); cudaMalloc(&W, NM * KM); cudaMalloc(&xs, TM * 4); cudaMalloc(&sg, KM / 128 * 4);
  cudaMalloc(&ws, NM * 4); cudaMalloc(&Y, TM * NM * 2);
  cudaMemset(X, 0x38, TM * KM); cudaMemset(W, 0x38, NM * KM);
  std::vector<float> one(TM > NM ? TM : NM, 1.0f);
  cudaMemcpy(xs, one.data(), TM * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(ws, one.data(), NM * 4, cudaMemcpyHostToDevice);
  cudaFree(sg);
  cudaMalloc(&sg, KM / 32 * 4);
  cudaMemcpy(sg, one.data(), KM / 32 * 4, cudaMemcpyHostToDevice);
  for (int a0 = 1; a0 + 3 < argc; a0 += 4) {
    const int64_t T = atoll(argv[a0]), N = atoll(argv[a0 + 1]), K = atoll(argv[a0 + 2]);
    const int plain = atoi(argv[a0 + 3]);
    const int group = getenv("RRS_GROUP") ? atoi(getenv("RRS_GROUP")) : 128;
    rrs::GemmArgs a{X, xs, sg, W, ws, T, N, K, group, 1.0f / K, plain != 0, true, Y, 0, N, nullptr};
    std::vector<float> v;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 12; ++rep) {
      cudaEventRecord(e0);
      rrs::launch_gemm(a, nsm, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep >= 2) v.push_back(ms * 1e3f);
    }
    std::sort(v.begin(), v.end());
    const float us = v[v.size() / 2];
    const int tiles = (int)(((T + 255) / 256) * ((N + 239) / 240));
    printf("T %5lld N %6lld K %6lld %s: %8.1f us  %6.0f TOPS  tiles %d (%.2f waves)  err=%s\n", (long long)T,
           (long long)N, (long long)K, plain ? "plain" : "rrs  ", us, 2.0 * T * N * K / (us * 1e-6) / 1e12, tiles,
           tiles / (double)(nsm / 2), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

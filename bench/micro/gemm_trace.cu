// Timeline of the RRS GEMM's MMA / promotion handshake per CTA: first tile, tile boundary, second tile.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DRRS_TRACE -I../../include -o gemm_trace
//        gemm_trace.cu -lcuda
#include <cstdio>
#include <vector>
#include <algorithm>
#include "../../paper_2409_20361_b200/csrc/gemm.cu"

int main(int argc, char** argv) {
  const int64_t T = argc > 1 ? atoll(argv[1]) : 4096, N = argc > 2 ? atoll(argv[2]) : 14336, K = argc > 3 ? atoll(argv[3]) : 4096;
  const int plain = argc > 4 ? atoi(argv[4]) : 0;
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int8_t *X, *W; float *xs, *sg, *ws; uint16_t* Y;
  cudaMalloc(&X, T * K); cudaMalloc(&W, N * K); cudaMalloc(&xs, T * 4); cudaMalloc(&sg, K / 128 * 4);
  cudaMalloc(&ws, N * 4); cudaMalloc(&Y, T * N * 2);
  cudaMemset(X, 0x38, T * K); cudaMemset(W, 0x38, N * K);
  std::vector<float> one(std::max(T, N), 1.0f);
  cudaMemcpy(xs, one.data(), T * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(ws, one.data(), N * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(sg, one.data(), K / 128 * 4, cudaMemcpyHostToDevice);
  rrs::GemmArgs a{X, xs, sg, W, ws, T, N, K, 128, 1.0f / K, plain != 0, true, Y, 0, N, nullptr};
  for (int rep = 0; rep < 4; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t err = rrs::launch_gemm(a, nsm, 0);
    cudaEventRecord(e1);
    cudaError_t e2 = cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("rep %d: %s/%s %.1f us = %.0f TOPS\n", rep, cudaGetErrorString(err), cudaGetErrorString(e2), ms * 1e3,
           2.0 * T * N * K / (ms * 1e-3) / 1e12);
  }
  static unsigned long long h[160][32][8];
  cudaMemcpyFromSymbol(h, rrs::g_gtrace, sizeof(h));
  const int G = (int)(K / 128);
  for (int c : {0, 1, 2, 100}) {
    unsigned long long t0 = h[c][0][0] ? h[c][0][0] : h[c][0][3];
    printf("CTA %d (ns from its first MMA wait):\n  tile g : tempty  full  issued | w0 tfull  w0 rel | wl tfull  wl rel\n", c);
    for (int r = 0; r < 32; ++r) {
      const int it = r < 24 ? 0 : 1, g = r < 16 ? r : (r < 24 ? G - 8 + (r - 16) : r - 24);
      if (r == 16 && G <= 16) continue;
      auto f = [&](int s) { return h[c][r][s] ? (long long)(h[c][r][s] - t0) : -1LL; };
      printf("  %d %3d: %6lld %6lld %6lld | %6lld %6lld | %6lld %6lld\n", it, g, f(0), f(1), f(2), f(3), f(4), f(5), f(6));
    }
    const char* lab[8] = {"epi start", "beta staged", "store buf free", "staged", "store issued", "epi end",
                          "tile start (acc zeroed)", "-"};
    for (int it = 0; it < 2; ++it)
      for (int k = 0; k < 7; ++k)
        if (h[c][8 * it + k][7])
          printf("  tile %d %-24s %lld\n", it, lab[k], (long long)(h[c][8 * it + k][7] - t0));
  }
  return 0;
}

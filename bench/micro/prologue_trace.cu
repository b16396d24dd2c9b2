// Per-CTA timeline of the two prologue kernels (fwht_colmax, smooth_quant) on a C2-shaped input.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DRRS_TRACE -I../../include
//        -o prologue_trace prologue_trace.cu
#include <cstdio>
#include <vector>
#include <algorithm>
#include "../../paper_2409_20361_b200/csrc/prologue.cu"

int main(int argc, char** argv) {
  const int64_t T = argc > 1 ? atoll(argv[1]) : 2048, K = argc > 2 ? atoll(argv[2]) : 4096;
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  std::vector<uint16_t> hx(T * K);
  for (int64_t i = 0; i < T * K; ++i) hx[i] = (uint16_t)(0x3F80 + (i * 2654435761u % 127)) ^ ((i & 1) << 15);
  std::vector<int32_t> hp(K);
  for (int i = 0; i < K; ++i) hp[i] = i;
  unsigned long long st = 88172645463325252ull;  // xorshift shuffle: a random perm like the real reorder
  for (int i = K - 1; i > 0; --i) {
    st ^= st << 13; st ^= st >> 7; st ^= st << 17;
    std::swap(hp[i], hp[st % (unsigned long long)(i + 1)]);
  }
  uint16_t* X; float* Xr; unsigned* cm; float* sg; int8_t* q; float* sc; int32_t* perm;
  cudaMalloc(&X, T * K * 2); cudaMalloc(&Xr, T * K * 4); cudaMalloc(&cm, K * 4); cudaMalloc(&sg, K / 128 * 4);
  cudaMalloc(&q, T * K); cudaMalloc(&sc, T * 4); cudaMalloc(&perm, K * 4);
  cudaMemcpy(X, hx.data(), T * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(perm, hp.data(), K * 4, cudaMemcpyHostToDevice);
  unsigned* counter;
  cudaMalloc(&counter, 256);
  const bool fused = argc > 3 && atoi(argv[3]) == 1;
  const bool decode = argc > 3 && atoi(argv[3]) == 2;
  for (int rep = 0; rep < 3 && decode; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t le = rrs::launch_prologue_decode(X, T, K, perm, cm, Xr, sg, nullptr, q, sc, false, 128, 0);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    float a;
    cudaEventElapsedTime(&a, e0, e1);
    printf("rep %d: %s / %s decode prologue %.1f us\n", rep, cudaGetErrorString(le), cudaGetErrorString(e), a * 1e3);
  }
  for (int rep = 0; rep < 3 && fused; ++rep) {
    cudaMemset(cm, 0, K * 4);
    cudaMemset(counter, 0, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    rrs::launch_prologue_fused(X, T, K, Xr, perm, sg, nullptr, q, sc, true, 128, 0);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    float a;
    cudaEventElapsedTime(&a, e0, e1);
    printf("rep %d: %s fused prologue %.1f us\n", rep, cudaGetErrorString(e), a * 1e3);
  }
  for (int rep = 0; rep < 3 && !fused && !decode; ++rep) {
    cudaMemset(cm, 0, K * 4);
    cudaEvent_t e0, e1, e2;
    cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2);
    cudaEventRecord(e0);
    rrs::launch_fwht_colmax(X, T, K, cm, Xr, nsm, 0);
    cudaEventRecord(e1);
    rrs::launch_smooth_quant(Xr, T, K, perm, cm, sg, nullptr, q, sc, true, 128, nsm, 0);
    cudaEventRecord(e2);
    cudaError_t e = cudaDeviceSynchronize();
    float a, b;
    cudaEventElapsedTime(&a, e0, e1); cudaEventElapsedTime(&b, e1, e2);
    printf("rep %d: %s fwht_colmax %.1f us, smooth_quant %.1f us\n", rep, cudaGetErrorString(e), a * 1e3, b * 1e3);
  }
  static unsigned long long h[3][1024][16];
  cudaMemcpyFromSymbol(h, rrs::g_trace, sizeof(h));
  for (int k = 0; k < 3; ++k) {
    unsigned long long t0 = ~0ull;
    int n = 0;
    for (int c = 0; c < 1024; ++c) if (h[k][c][0]) { t0 = std::min(t0, h[k][c][0]); n = c + 1; }
    printf("kernel %d: %d CTAs traced\n", k, n);
    // per slot: min / median / max offset (us) over CTAs
    for (int s = 0; s < 16; ++s) {
      std::vector<double> v;
      for (int c = 0; c < n; ++c) if (h[k][c][s]) v.push_back((h[k][c][s] - t0) * 1e-3);
      if (v.empty()) continue;
      std::sort(v.begin(), v.end());
      printf("  slot %2d: n=%4zu  min %7.2f  med %7.2f  max %7.2f us\n", s, v.size(), v.front(), v[v.size() / 2], v.back());
    }
  }
  return 0;
}

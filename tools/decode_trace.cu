// Timeline of the decode regime at configs[3] (K = N = 8192), synthetic codes: rrs_decode_gemm_kernel (CTAs 0..7) alone,
// or the whole layer (prologue_decode_group_kernel + the GEMM launched with PDL, as rrs_linear does).
//   tools/build_traces.sh;  tools/decode_trace T [mode]   mode: 0 GEMM, 1 GEMM with X loaded once (W stream only),
//                                                          2 layer (prologue + GEMM), 3 layer without PDL,
//                                                          4-7: mode 1 and no MMA / no TMEM store / no TMEM load / none
#include <cstdio>
#include <vector>
#include <algorithm>
#include "../paper_2409_20361_b200/csrc/decode.cu"

namespace rrs {
void copy_prologue_trace(void* dst, size_t bytes);  // prologue.cu (-DRRS_TRACE)
void copy_prologue_trace_clk(void* dst, size_t bytes);
}

int main(int argc, char** argv) {
  const int T = argc > 1 ? atoi(argv[1]) : 64;
  const int mode = argc > 2 ? atoi(argv[2]) : 0;
  const int64_t K = 8192, N = 8192;
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int8_t* X; uint8_t* W; float *xs, *sg, *ws; uint16_t* Y; uint8_t* flush; uint16_t* Xb; int32_t* perm;
  cudaMalloc(&X, T * K); cudaMalloc(&W, N * K / 2); cudaMalloc(&xs, T * 4); cudaMalloc(&sg, K / 128 * 4);
  cudaMalloc(&ws, N * 4); cudaMalloc(&Y, T * N * 2); cudaMalloc(&flush, 256 << 20);
  cudaMalloc(&Xb, T * K * 2); cudaMalloc(&perm, K * 4);
  cudaMemset(X, 1, T * K); cudaMemset(W, 0x11, N * K / 2); cudaMemset(Xb, 0x3F, T * K * 2);
  std::vector<int32_t> hp(K);
  for (int i = 0; i < K; ++i) hp[i] = i;
  unsigned long long st = 88172645463325252ull;  // xorshift shuffle: a random perm like the calibrated reorder
  for (int i = K - 1; i > 0; --i) {
    st ^= st << 13; st ^= st >> 7; st ^= st << 17;
    std::swap(hp[i], hp[st % (unsigned long long)(i + 1)]);
  }
  cudaMemcpy(perm, hp.data(), K * 4, cudaMemcpyHostToDevice);
  int exp = mode == 1 ? 1 : 0;
  if (mode >= 4) exp = 1 | (mode == 4 ? 2 : mode == 5 ? 4 : mode == 6 ? 8 : 14);  // 4 no MMA, 5 no st, 6 no ld, 7 none
  rrs::g_dec_no_pdl = mode == 3;
  const bool layer = mode == 2 || mode == 3;
  cudaMemcpyToSymbol(rrs::g_dec_exp, &exp, sizeof(int));
  rrs::DecodeArgs a{X, xs, sg, W, ws, T, N, K, 128, 1.0f / K, Y, 0, N};
  for (int rep = 0; rep < 4; ++rep) {
    cudaMemset(flush, rep, 256 << 20);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t e = cudaSuccess;
    if (layer)
      e = rrs::launch_prologue_decode(Xb, T, K, perm, nullptr, nullptr, sg, nullptr, X, xs, false, 128, 0);
    if (e == cudaSuccess) e = rrs::launch_decode_gemm(a, nsm, 0);
    cudaEventRecord(e1);
    cudaError_t e2 = cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("rep %d: %s / %s  %.2f us\n", rep, cudaGetErrorString(e), cudaGetErrorString(e2), ms * 1e3);
  }
  static unsigned long long h[8][8][64];
  cudaMemcpyFromSymbol(h, rrs::g_dtrace, sizeof(h));
  static unsigned long long hp2[3][1024][16];
  rrs::copy_prologue_trace(hp2, sizeof(hp2));
  unsigned long long t0 = h[0][5][0];
  if (layer) {  // common origin: the first prologue CTA's start
    for (int c = 0; c < T && c < 1024; ++c) if (hp2[2][c][0] && hp2[2][c][0] < t0) t0 = hp2[2][c][0];
    for (int sl = 0; sl < 7; ++sl) {
      double mn = 1e30, mx = -1e30;
      for (int c = 0; c < T && c < 1024; ++c)
        if (hp2[2][c][sl]) { double v = (double)(long long)(hp2[2][c][sl] - t0) * 1e-3; mn = v < mn ? v : mn; mx = v > mx ? v : mx; }
      if (mn < 1e29) printf("prologue slot %d: %.2f .. %.2f us\n", sl, mn, mx);
    }
    static unsigned long long hc[3][1024][16];
    rrs::copy_prologue_trace_clk(hc, sizeof(hc));
    for (int sl = 1; sl < 7; ++sl)  // CTA 0: SM cycles and ns from slot 0 -> effective clock
      if (hc[2][0][sl] && hp2[2][0][sl])
        printf("prologue CTA 0 slot %d: %llu cycles / %.0f ns = %.2f GHz\n", sl, hc[2][0][sl] - hc[2][0][0],
               (double)(hp2[2][0][sl] - hp2[2][0][0]), (double)(hc[2][0][sl] - hc[2][0][0]) / (double)(hp2[2][0][sl] - hp2[2][0][0]));
  }
  int nlast = 0;
  while (nlast + 1 < 64 && h[0][4][nlast + 1]) ++nlast;
  for (int c = 0; c < 8; ++c) {
    printf("CTA %d: start %.2f  first conv %.2f  last promoted %.2f  cl-wait1 %.2f  pushed %.2f  cl-sync2 %.2f  end %.2f us\n", c,
           (double)(long long)(h[c][5][0] - t0) * 1e-3, (double)(long long)(h[c][2][0] - t0) * 1e-3,
           (double)(long long)(h[c][4][nlast] - t0) * 1e-3, (double)(long long)(h[c][7][0] - t0) * 1e-3,
           (double)(long long)(h[c][7][1] - t0) * 1e-3, (double)(long long)(h[c][7][2] - t0) * 1e-3,
           (double)(long long)(h[c][6][0] - t0) * 1e-3);
  }
  const char* names[7] = {"W issued", "X issued", "converted", "MMA issued", "promoted", "start", "end"};
  for (int c = 0; c < 1; ++c) {
    printf("CTA %d: start %.2f, end %.2f us\n", c, (double)(long long)(h[c][5][0] - t0) * 1e-3,
           (double)(long long)(h[c][6][0] - t0) * 1e-3);
    for (int ev = 0; ev < 5; ++ev) {
      printf("  %-10s", names[ev]);
      for (int i = 0; i < 32; ++i) printf(" %6.2f", h[c][ev][i] ? (double)(long long)(h[c][ev][i] - t0) * 1e-3 : -1.0);
      printf("\n");
    }
  }
  return 0;
}

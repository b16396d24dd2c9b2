// Timeline of rrs_decode_gemm_kernel (CTAs 0..7) at configs[3] (K = N = 8192), synthetic codes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DRRS_TRACE -I../include -o decode_trace \
//        decode_trace.cu ../paper_2409_20361_b200/csrc/api.cu ../paper_2409_20361_b200/csrc/prologue.cu \
//        ../paper_2409_20361_b200/csrc/gemm.cu -lcuda -lnccl
#include <cstdio>
#include <vector>
#include "../paper_2409_20361_b200/csrc/decode.cu"

int main(int argc, char** argv) {
  const int T = argc > 1 ? atoi(argv[1]) : 64;
  const int64_t K = 8192, N = 8192;
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int8_t* X; uint8_t* W; float *xs, *sg, *ws; uint16_t* Y; uint8_t* flush;
  cudaMalloc(&X, T * K); cudaMalloc(&W, N * K / 2); cudaMalloc(&xs, T * 4); cudaMalloc(&sg, K / 128 * 4);
  cudaMalloc(&ws, N * 4); cudaMalloc(&Y, T * N * 2); cudaMalloc(&flush, 256 << 20);
  cudaMemset(X, 1, T * K); cudaMemset(W, 0x11, N * K / 2);
  rrs::DecodeArgs a{X, xs, sg, W, ws, T, N, K, 128, 1.0f / K, Y, 0, N};
  for (int rep = 0; rep < 4; ++rep) {
    cudaMemset(flush, rep, 256 << 20);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t e = rrs::launch_decode_gemm(a, nsm, 0);
    cudaEventRecord(e1);
    cudaError_t e2 = cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("rep %d: %s / %s  %.2f us\n", rep, cudaGetErrorString(e), cudaGetErrorString(e2), ms * 1e3);
  }
  static unsigned long long h[8][8][64];
  cudaMemcpyFromSymbol(h, rrs::g_dtrace, sizeof(h));
  const char* names[7] = {"W issued", "X issued", "converted", "MMA issued", "promoted", "start", "end"};
  for (int c = 0; c < 8; ++c) {
    unsigned long long t0 = h[0][5][0];
    printf("CTA %d: start %.2f  first conv %.2f  last promoted %.2f  cl-wait1 %.2f  pushed %.2f  cl-sync2 %.2f  end %.2f us\n", c,
           (double)(long long)(h[c][5][0] - t0) * 1e-3, (double)(long long)(h[c][2][0] - t0) * 1e-3,
           (double)(long long)(h[c][4][15] - t0) * 1e-3, (double)(long long)(h[c][7][0] - t0) * 1e-3,
           (double)(long long)(h[c][7][1] - t0) * 1e-3, (double)(long long)(h[c][7][2] - t0) * 1e-3,
           (double)(long long)(h[c][6][0] - t0) * 1e-3);
  }
  for (int c = 0; c < 2; ++c) {
    unsigned long long t0 = h[c][5][0];
    printf("CTA %d: start 0, end %.2f us\n", c, (h[c][6][0] - t0) * 1e-3);
    for (int ev = 0; ev < 5; ++ev) {
      printf("  %-10s", names[ev]);
      for (int i = 0; i < 16; ++i) printf(" %6.2f", h[c][ev][i] ? (double)(long long)(h[c][ev][i] - t0) * 1e-3 : -1.0);
      printf("\n");
    }
  }
  return 0;
}

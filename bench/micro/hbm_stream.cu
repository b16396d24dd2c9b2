// HBM streaming microbenchmark for the decode W stream (DESIGN.md §7 decode regime): aggregate bandwidth of one CTA
// per SM pulling a private contiguous region into shared memory with cp.async.bulk copies of CHUNK bytes, NST in
// flight, nothing else on the SM; L2 flushed before each run.  Also 2 CTAs x half the chunks, and 8-KiB halves of
// 16-KiB tiles with a 16-KiB stride (the 128-row decode CTA's pattern).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hbm_stream hbm_stream.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2409_20361_b200/csrc/ptx.cuh"

using namespace rrs::ptx;
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

__global__ void stream_kernel(const uint8_t* src, int64_t bytes_per_cta, int chunk, int nst, int64_t stride,
                              unsigned* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + nst * chunk);
  const int n = (int)(bytes_per_cta / chunk);
  const uint8_t* base = src + (int64_t)blockIdx.x * (stride == chunk ? bytes_per_cta : bytes_per_cta * 2);
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) mbar_init(&bar[s], 1);
    fence_barrier_init();
    for (int i = 0; i < nst && i < n; ++i) {
      mbar_arrive_expect_tx(&bar[i], chunk);
      bulk_load(smem + i * chunk, base + (int64_t)i * stride, chunk, &bar[i]);
    }
    unsigned acc = 0;
    for (int i = 0; i < n; ++i) {
      const int s = i % nst;
      mbar_wait(&bar[s], (i / nst) & 1);
      acc += smem[s * chunk + (i & 63)];
      if (i + nst < n) {
        mbar_arrive_expect_tx(&bar[s], chunk);
        bulk_load(smem + s * chunk, base + (int64_t)(i + nst) * stride, chunk, &bar[s]);
      }
    }
    sink[blockIdx.x] = acc;
  }
}

// reads a buffer larger than L2 (clean lines replace the dirty ones a write-flush leaves behind)
__global__ void read_kernel(const uint4* p, int64_t n, unsigned* sink) {
  unsigned acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc ^= __ldcg(p + i).x;
  if (acc == 0x12345678u) sink[0] = acc;
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int64_t total = 256ll << 20;
  uint8_t* src; uint8_t* flush; unsigned* sink;
  CK(cudaMalloc(&src, 2 * total + (64 << 20))); CK(cudaMalloc(&flush, 256 << 20)); CK(cudaMalloc(&sink, 4096 * 4));
  CK(cudaMemset(src, 1, 2 * total));
  uint8_t* clean; CK(cudaMalloc(&clean, 256 << 20)); CK(cudaMemset(clean, 0, 256 << 20));
  CK(cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  struct Cfg { int ctas, chunk, nst, halves; } cfgs[] = {
      {128, 8192, 16, 0}, {128, 16384, 8, 0}, {128, 16384, 12, 0}, {148, 16384, 8, 0}, {148, 8192, 16, 0},
      {148, 32768, 4, 0}, {148, 4096, 32, 0}, {128, 8192, 16, 1}, {296, 8192, 8, 0}, {148, 65536, 3, 0}};

  for (int64_t MB : {64, 512}) {  // plain LDG.128 read of MB (all SMs), same timing: the event overhead and the LDG rate
    float best = 1e9f;
    uint8_t* big; CK(cudaMalloc(&big, MB << 20)); CK(cudaMemset(big, 1, MB << 20));
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaMemset(flush, rep, 256 << 20));
      cudaEvent_t a, b;
      cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      read_kernel<<<4 * nsm, 512>>>((const uint4*)big, (MB << 20) / 16, sink);
      cudaEventRecord(b);
      CK(cudaDeviceSynchronize());
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep > 0 && ms < best) best = ms;
    }
    printf("LDG read %lld MB: %.2f us -> %.0f GB/s\n", (long long)MB, best * 1e3, (MB << 20) / (best * 1e-3) / 1e9);
    cudaFree(big);
  }
  for (int mode = 0; mode < 2; ++mode)
  for (auto c : cfgs) {
    const int64_t per = (total / c.ctas) / c.chunk * c.chunk;
    const int64_t stride = c.halves ? 2 * c.chunk : c.chunk;
    const int smem = c.nst * c.chunk + 8 * c.nst;
    float best = 1e9f;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaMemset(flush, rep, 256 << 20));
      if (mode == 1) read_kernel<<<4 * nsm, 512>>>((const uint4*)clean, (256 << 20) / 16, sink);
      cudaEvent_t a, b;
      cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      stream_kernel<<<c.ctas, 32, smem>>>(src, per, c.chunk, c.nst, stride, sink);
      cudaEventRecord(b);
      CK(cudaDeviceSynchronize());
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep > 0 && ms < best) best = ms;
    }
    printf("%s ctas %3d chunk %6d nst %2d %s: %.2f us for %.1f MB -> %.0f GB/s (%.1f GB/s per CTA)\n", mode ? "write+read flush" : "write flush     ", c.ctas, c.chunk,
           c.nst, c.halves ? "halves" : "contig", best * 1e3, per * c.ctas / 1e6, per * c.ctas / (best * 1e-3) / 1e9,
           per / (best * 1e-3) / 1e9);
  }
  return 0;
}

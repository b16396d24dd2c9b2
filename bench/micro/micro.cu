// Microbenchmarks that decide the hard parts of the design:
// TMEM->RF load bandwidth, FP32/FP64/conversion issue rates, and the int8 tcgen05 MMA rate.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro micro.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2409_20361_b200/csrc/ptx.cuh"

// 32 lanes x 32 columns of 32-bit (microbenchmark only; the product kernels use the x16 shape)
#define RRS_TMEM_LD32(taddr, r)                                                                          \
  asm volatile(                                                                                         \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"  \
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                          \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),  \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),        \
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),      \
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),      \
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                                           \
      : "r"(taddr))
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

using namespace rrs::ptx;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

__global__ void tmem_ld_bw(int iters, unsigned long long* cycles, uint32_t* sink) {
  __shared__ uint32_t taddr_s;
  const int w = threadIdx.x >> 5;
  if (w == 0) tmem_alloc(&taddr_s, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = taddr_s + (((w & 3) * 32) << 16);
  uint32_t acc = 0, r[32];
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const uint32_t col = ((i * 32) + (w >> 2) * 256) & 511;
    RRS_TMEM_LD32(base + col, r);
    tmem_ld_wait();
#pragma unroll
    for (int k = 0; k < 32; ++k) acc ^= r[k];
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  __syncthreads();
  if (w == 0) tmem_dealloc(taddr_s, 512);
}

// 8 independent chains per thread, 3-register FFMA
__global__ void ffma3(int iters, float b, float c, unsigned long long* cycles, float* sink) {
  float a[8];
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 0.001f + k;
  float bb = b + threadIdx.x * 1e-9f, cc = c - threadIdx.x * 1e-9f;
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], bb, cc);
  }
  unsigned long long t1 = clock64();
  float s = 0; for (int k = 0; k < 8; ++k) s += a[k];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

// promotion pattern: acc[k] = fma(s, P[k] - M, acc[k]) with P in registers (FADD + FFMA)
__global__ void promo(int iters, float s0, unsigned long long* cycles, float* sink) {
  float acc[16], p[16];
  for (int k = 0; k < 16; ++k) { acc[k] = 0; p[k] = 12582912.0f + k + threadIdx.x; }
  float s = s0 + threadIdx.x * 1e-9f;
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = fmaf(s, p[k] - 12582912.0f, acc[k]);
    s += 1e-7f;
  }
  unsigned long long t1 = clock64();
  float t = 0; for (int k = 0; k < 16; ++k) t += acc[k];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = t;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

// same with packed f32x2 (sm_100 FADD2/FFMA2)
__global__ void promo2(int iters, float s0, unsigned long long* cycles, float* sink) {
  unsigned long long acc[8], p[8];
  for (int k = 0; k < 8; ++k) {
    float2 a = make_float2(0.f, 0.f), q = make_float2(12582912.0f + 2 * k + threadIdx.x, 12582913.0f + 2 * k);
    acc[k] = *reinterpret_cast<unsigned long long*>(&a);
    p[k] = *reinterpret_cast<unsigned long long*>(&q);
  }
  float2 mm = make_float2(-12582912.0f, -12582912.0f);
  unsigned long long m = *reinterpret_cast<unsigned long long*>(&mm);
  float s = s0 + threadIdx.x * 1e-9f;
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    float2 ss = make_float2(s, s);
    unsigned long long sv = *reinterpret_cast<unsigned long long*>(&ss);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      unsigned long long f;
      asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(f) : "l"(p[k]), "l"(m));
      asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[k]) : "l"(sv), "l"(f));
    }
    s += 1e-7f;
  }
  unsigned long long t1 = clock64();
  float t = 0;
  for (int k = 0; k < 8; ++k) { float2 a = *reinterpret_cast<float2*>(&acc[k]); t += a.x + a.y; }
  sink[blockIdx.x * blockDim.x + threadIdx.x] = t;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

__global__ void dadd(int iters, unsigned long long* cycles, double* sink) {
  double a[8], b[8];
  for (int k = 0; k < 8; ++k) { a[k] = threadIdx.x + k; b[k] = 1.0 + k; }
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) { a[k] = a[k] + b[k]; b[k] = b[k] - a[k]; }
  }
  unsigned long long t1 = clock64();
  double s = 0; for (int k = 0; k < 8; ++k) s += a[k] + b[k];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

// f32 -> f64 and f64 -> f32 (RN) conversions (the FWHT's input widening and output rounding): 8 chains, each step
// one F2F.F64.F32 and one F2F.F32.F64
__global__ void cvt64(int iters, unsigned long long* cycles, float* sink) {
  float a[8];
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 0.25f + k;
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = __double2float_rn((double)a[k] * 1.0000001);
  }
  unsigned long long t1 = clock64();
  float s = 0; for (int k = 0; k < 8; ++k) s += a[k];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

__global__ void i2f(int iters, unsigned long long* cycles, float* sink) {
  int p[8]; float acc[8];
  for (int k = 0; k < 8; ++k) { p[k] = threadIdx.x * 7 + k; acc[k] = 0; }
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) { acc[k] += __int2float_rn(p[k]); p[k] += 3; }
  }
  unsigned long long t1 = clock64();
  float s = 0; for (int k = 0; k < 8; ++k) s += acc[k];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

__global__ void __launch_bounds__(128, 1) mma_i8_rate(int iters, int N, unsigned long long* cycles, uint32_t* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t taddr_s;
  uint8_t* a = smem;            // 128 x 128 B
  uint8_t* b = smem + 16384;    // 256 x 128 B
  for (int i = threadIdx.x; i < 49152 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u;
  const int w = threadIdx.x >> 5;
  if (w == 0) tmem_alloc(&taddr_s, 512);
  if (threadIdx.x == 32) { mbar_init(&bar, 1); fence_barrier_init(); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t idesc = idesc_i8(128, N);
  unsigned long long t0 = clock64();
  if (w == 1 && elect_one()) {
    const uint64_t ad = smem_desc_sw128(a), bd = smem_desc_sw128(b);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        mma_i8(taddr_s + ((i & 1) * 256), ad + 2 * k, bd + 2 * k, idesc, (i > 1) || k > 0);
    }
    mma_commit(&bar);
  }
  if (w == 1) mbar_wait(&bar, 0);
  unsigned long long t1 = clock64();
  tc_fence_after();
  __syncthreads();
  uint32_t r[32];
  RRS_TMEM_LD32(taddr_s + (((w & 3) * 32) << 16), r);
  tmem_ld_wait();
  if (threadIdx.x == 32) cycles[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = r[0];
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc(taddr_s, 512);
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d, clock %d kHz\n", nsm, clk);
  unsigned long long* cyc; CK(cudaMalloc(&cyc, 4096 * 8));
  void* sink; CK(cudaMalloc(&sink, 1 << 24));
  unsigned long long h[4096];
  auto report = [&](const char* name, int blocks, double ops_per_block) {
    cudaMemcpy(h, cyc, blocks * 8, cudaMemcpyDeviceToHost);
    double mx = 0; for (int i = 0; i < blocks; ++i) mx = mx > h[i] ? mx : (double)h[i];
    printf("%-28s %10.1f per clk per SM (cycles %.0f)\n", name, ops_per_block / mx, mx);
  };
  for (int warps : {4, 8, 12, 16, 32}) {
    int iters = 4096;
    tmem_ld_bw<<<nsm, warps * 32>>>(iters, cyc, (uint32_t*)sink); CK(cudaDeviceSynchronize());
    char nm[64]; snprintf(nm, 64, "tmem ld bytes (%d warps)", warps);
    report(nm, nsm, (double)iters * warps * 32 * 32 * 4);
  }
  for (int t : {256, 512, 1024}) {
    int iters = 4096;
    ffma3<<<nsm, t>>>(iters, 1.0001f, 0.5f, cyc, (float*)sink); CK(cudaDeviceSynchronize());
    char nm[64]; snprintf(nm, 64, "FFMA 3-reg lanes (%d thr)", t); report(nm, nsm, (double)iters * 8 * t);
    promo<<<nsm, t>>>(iters, 0.01f, cyc, (float*)sink); CK(cudaDeviceSynchronize());
    snprintf(nm, 64, "promo FADD+FFMA elems (%d)", t); report(nm, nsm, (double)iters * 16 * t);
    promo2<<<nsm, t>>>(iters, 0.01f, cyc, (float*)sink); CK(cudaDeviceSynchronize());
    snprintf(nm, 64, "promo f32x2 elems (%d)", t); report(nm, nsm, (double)iters * 16 * t);
    dadd<<<nsm, t>>>(iters, cyc, (double*)sink); CK(cudaDeviceSynchronize());
    snprintf(nm, 64, "DADD lanes (%d thr)", t); report(nm, nsm, (double)iters * 16 * t);
    cvt64<<<nsm, t>>>(iters, cyc, (float*)sink); CK(cudaDeviceSynchronize());
    snprintf(nm, 64, "f32->f64->f32 + DMUL (%d)", t); report(nm, nsm, (double)iters * 8 * t);
    i2f<<<nsm, t>>>(iters, cyc, (float*)sink); CK(cudaDeviceSynchronize());
    snprintf(nm, 64, "I2F lanes (%d thr)", t); report(nm, nsm, (double)iters * 8 * t);
  }
  CK(cudaFuncSetAttribute(mma_i8_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 49152 + 1024));
  for (int N : {128, 256}) {
    int iters = 2048;
    mma_i8_rate<<<nsm, 128, 49152 + 1024>>>(iters, N, cyc, (uint32_t*)sink); CK(cudaDeviceSynchronize());
    char nm[64]; snprintf(nm, 64, "int8 MMA MACs (N=%d)", N);
    report(nm, nsm, (double)iters * 4 * 128.0 * N * 32);
    uint32_t v; cudaMemcpy(&v, sink, 4, cudaMemcpyDeviceToHost);
    printf("   mma result sample %u (expect %u)\n", v, (unsigned)(128 * (iters >= 2 ? 2 : 1)));
  }
  return 0;
}

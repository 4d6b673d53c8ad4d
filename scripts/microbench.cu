// Microbenchmarks for design decisions (not part of the product):
//  1. DFMA throughput, register operands
//  2. DFMA with constant-bank operands, 2 KB vs 24 KB constant footprint
//  3. DMMA m8n8k4 f64 throughput
//  4. cp.async.bulk + mbarrier expect_tx with 32 KB and 64 KB transactions
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void k_dfma_reg(double* out, int iters) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 1.000001, c = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

template <int NC>
struct CParams { double m[NC]; };

template <int NC>
__global__ void k_dfma_const(const __grid_constant__ CParams<NC> p, double* out, int iters) {
  double acc[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) acc[r] = threadIdx.x + r;
  double x = threadIdx.x * 1e-3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < NC / 8; ++c)
#pragma unroll
      for (int r = 0; r < 8; ++r) acc[r] = fma(p.m[c * 8 + r], x, acc[r]);
    x += 1e-7;
  }
  double s = 0;
#pragma unroll
  for (int r = 0; r < 8; ++r) s += acc[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) c[t][0] = c[t][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_bulk(const double* src, double* dst, int bytes, int* ok) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = (uint64_t*)(sm + bytes);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar)), "r"(bytes));
    const int chunk = 8192;
    for (int o = 0; o < bytes; o += chunk)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(sm + o)),
                   "l"((const char*)src + o), "r"(chunk), "r"(sa(bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(sa(bar)) : "memory");
  const double* d = (const double*)sm;
  int bad = 0;
  for (int i = threadIdx.x; i < bytes / 8; i += blockDim.x) bad += d[i] != src[i];
  if (bad) atomicAdd(ok, bad);
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  double* out;
  CK(cudaMalloc(&out, sizeof(double) * sms * 8 * 1024));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  // 1. DFMA register
  {
    int iters = 4096, blocks = sms * 8, threads = 256;
    k_dfma_reg<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0);
    k_dfma_reg<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double fmas = 1.0 * blocks * threads * iters * 16 * 8;
    printf("DFMA reg: %.2f TFMA/s = %.1f DFMA/clk/SM at %d MHz (%.2f TFLOPS)\n", fmas / ms / 1e9,
           fmas / (ms * 1e-3) / sms / (prop.clockRate * 1e3), prop.clockRate / 1000, 2 * fmas / ms / 1e9);
  }
  // 2. DFMA const
  {
    CParams<256> p2;
    CParams<3072> p24;
    for (int i = 0; i < 256; ++i) p2.m[i] = 1.0 + i * 1e-6;
    for (int i = 0; i < 3072; ++i) p24.m[i] = 1.0 + i * 1e-6;
    int blocks = sms * 8, threads = 256;
    int it2 = 256, it24 = 256 / 12;
    k_dfma_const<256><<<blocks, threads>>>(p2, out, 2);
    cudaEventRecord(e0);
    k_dfma_const<256><<<blocks, threads>>>(p2, out, it2);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double f2 = 1.0 * blocks * threads * it2 * 256;
    printf("DFMA const 2KB: %.1f DFMA/clk/SM\n", f2 / (ms * 1e-3) / sms / (prop.clockRate * 1e3));
    k_dfma_const<3072><<<blocks, threads>>>(p24, out, 1);
    cudaEventRecord(e0);
    k_dfma_const<3072><<<blocks, threads>>>(p24, out, it24);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double f24 = 1.0 * blocks * threads * it24 * 3072;
    printf("DFMA const 24KB: %.1f DFMA/clk/SM\n", f24 / (ms * 1e-3) / sms / (prop.clockRate * 1e3));
  }
  // 3. DMMA
  {
    int iters = 2048, blocks = sms * 8, threads = 256;
    k_dmma<<<blocks, threads>>>(out, 8);
    cudaEventRecord(e0);
    k_dmma<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double macs = 1.0 * blocks * (threads / 32) * iters * 8 * 256;
    printf("DMMA m8n8k4: %.2f TFLOPS = %.1f MAC/clk/SM\n", 2 * macs / ms / 1e9,
           macs / (ms * 1e-3) / sms / (prop.clockRate * 1e3));
  }
  // 4. bulk copy expect_tx sizes
  {
    double* src;
    CK(cudaMalloc(&src, 1 << 20));
    double h[131072 / 8];
    for (int i = 0; i < 131072 / 8; ++i) h[i] = i * 0.5 + 1;
    CK(cudaMemcpy(src, h, 131072, cudaMemcpyHostToDevice));
    int* ok;
    CK(cudaMalloc(&ok, 4));
    for (int bytes : {16384, 32768, 65536, 98304, 131072}) {
      CK(cudaMemset(ok, 0, 4));
      CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes + 64));
      k_bulk<<<1, 128, bytes + 64>>>(src, out, bytes, ok);
      cudaError_t e = cudaDeviceSynchronize();
      int bad = -1;
      cudaMemcpy(&bad, ok, 4, cudaMemcpyDeviceToHost);
      printf("bulk expect_tx %6d bytes: %s, mismatches=%d\n", bytes, cudaGetErrorString(e), bad);
    }
  }
  return 0;
}

// Microbenchmarks round 2 (design decisions only, not product code):
//  A. DMMA and DFMA issued together: separate pipes or one FP64 datapath?
//  B. cp.async.bulk global->shared throughput per SM vs copy size and the
//     alignment of the shared-memory destination (32 / 64 / 128 B).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void k_mix(double* out, int iters, int use_dmma, int use_dfma) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
  double f[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) { c[t][0] = c[t][1] = 0.0; f[t] = t; }
  for (int i = 0; i < iters; ++i) {
    if (use_dmma) {
#pragma unroll
      for (int t = 0; t < 8; ++t)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
    if (use_dfma) {
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int t = 0; t < 8; ++t) f[t] = fma(f[t], b, a);
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1] + f[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// each CTA streams `reps` tiles of n_copies x copy_bytes into smem at offset
// `align_off` + i * (copy_bytes + pad); one thread issues everything
__global__ void k_bulk_rate(const char* src, size_t src_span, int copy_bytes, int n_copies, int pad, int reps,
                            int lanes, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = (uint64_t*)sm;
  unsigned char* dst = sm + 128;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x >= lanes) return;
  const size_t cta_off = (size_t)blockIdx.x * n_copies * copy_bytes * 4;
  for (int rep = 0; rep < reps; ++rep) {
    if (threadIdx.x == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar)), "r"(n_copies * copy_bytes));
    __syncwarp(lanes == 32 ? 0xffffffffu : 1u);
    for (int i = threadIdx.x; i < n_copies; i += lanes) {
      const char* s = src + (cta_off + (size_t)(rep % 4) * n_copies * copy_bytes + (size_t)i * copy_bytes) % src_span;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sa(dst + i * (copy_bytes + pad))),
                   "l"(s), "r"(copy_bytes), "r"(sa(bar))
                   : "memory");
    }
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(sa(bar)),
                 "r"(rep & 1)
                 : "memory");
  }
  if (threadIdx.x == 0) sink[blockIdx.x] = dst[0];
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
  const double clk = prop.clockRate * 1e3;
  for (int mode = 1; mode <= 3; ++mode) {
    int iters = 2048, blocks = sms * 4, threads = 256;
    int dm = mode & 1, df = (mode >> 1) & 1;
    k_mix<<<blocks, threads>>>(out, 8, dm, df);
    cudaEventRecord(e0);
    k_mix<<<blocks, threads>>>(out, iters, dm, df);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps = 1.0 * blocks * threads / 32;
    const double dmma_macs = dm * warps * iters * 8 * 256;
    const double dfma = df * 1.0 * blocks * threads * iters * 64;
    printf("mix dmma=%d dfma=%d: %.3f ms  DMMA %.1f MAC/clk/SM  DFMA %.1f FMA/clk/SM  total %.1f /clk/SM\n", dm, df, ms,
           dmma_macs / (ms * 1e-3) / sms / clk, dfma / (ms * 1e-3) / sms / clk,
           (dmma_macs + dfma) / (ms * 1e-3) / sms / clk);
  }
  char* src;
  const size_t span = size_t(1) << 31;
  CK(cudaMalloc(&src, span));
  CK(cudaMemset(src, 1, span));
  unsigned long long* sink;
  CK(cudaMalloc(&sink, 8 * 4096));
  struct Cfg { int bytes, copies, pad, lanes; };
  Cfg cfgs[] = {{512, 64, 0, 1}, {512, 64, 32, 1}, {512, 64, 64, 1}, {512, 64, 128, 1}, {512, 64, 32, 32},
                {1024, 32, 0, 1}, {2048, 16, 0, 1}, {4096, 8, 0, 1}, {8192, 4, 0, 1}, {32768, 1, 0, 1}};
  for (const Cfg& c : cfgs) {
    const int smem = 128 + c.copies * (c.bytes + c.pad);
    CK(cudaFuncSetAttribute(k_bulk_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int blocks = sms * 4, reps = 64;
    k_bulk_rate<<<blocks, 32, smem>>>(src, span, c.bytes, c.copies, c.pad, 4, c.lanes, sink);
    cudaEventRecord(e0);
    k_bulk_rate<<<blocks, 32, smem>>>(src, span, c.bytes, c.copies, c.pad, reps, c.lanes, sink);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = 1.0 * blocks * reps * c.copies * c.bytes;
    printf("bulk %5d B x %2d copies pad %3d lanes %2d: %7.0f GB/s (4 CTAs/SM, 1 tile in flight each)\n", c.bytes,
           c.copies, c.pad, c.lanes, bytes / ms / 1e6);
  }
  return 0;
}

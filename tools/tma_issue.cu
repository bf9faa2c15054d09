// Microbenchmark: issue rate and throughput of TMA bulk copies (cp.async.bulk)
// from one thread per CTA, 1 CTA per SM, global -> shared, various sizes and
// numbers in flight. Reports per-CTA GB/s and ns per issued copy.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const unsigned char* src, size_t span, int bytes, int inflight, int total, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < inflight; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  unsigned long long t0 = clock64();
  const unsigned char* base = src + (size_t)blockIdx.x * span;
  for (int j = 0; j < total; ++j) {
    const int s = j % inflight;
    const uint32_t ph = (j / inflight) & 1;
    if (j >= inflight) {
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{.reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0,1,0,P;}"
                     : "=r"(ok) : "r"(s32(&bar[s])), "r"(ph ^ 1));
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar[s])), "r"(bytes));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     s32(sm + (size_t)s * bytes)),
                 "l"(base + ((size_t)j * bytes) % span), "r"(bytes), "r"(s32(&bar[s])));
  }
  for (int j = total; j < total + inflight; ++j) {
    const int s = j % inflight;
    const uint32_t ph = (j / inflight) & 1;
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0,1,0,P;}"
                   : "=r"(ok) : "r"(s32(&bar[s])), "r"(ph ^ 1));
  }
  out[blockIdx.x] = clock64() - t0;
}
int main() {
  const size_t span = 64ull << 20;  // 64 MiB per CTA (DRAM-resident)
  unsigned char* src; unsigned long long* out;
  cudaMalloc(&src, span * 148); cudaMallocManaged(&out, 148 * 8);
  cudaMemset(src, 1, span * 148);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int sizes[] = {4096, 16384, 32768};
  int infl[] = {1, 2, 4, 8};
  for (int b : sizes)
    for (int f : infl) {
      if ((size_t)b * f > 200 * 1024) continue;
      int total = (int)((256ll << 20) / 148 / b);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      k<<<148, 32, b * f>>>(src, span, b, f, total, out);
      cudaEventRecord(e0);
      k<<<148, 32, b * f>>>(src, span, b, f, total, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double bytes = (double)total * b * 148;
      printf("copy %6d B x %d in flight: %7.1f GB/s total, %5.1f GB/s/SM, %6.0f ns per copy\n", b, f,
             bytes / ms / 1e6, bytes / ms / 1e6 / 148, ms * 1e6 / total);
    }
  return 0;
}

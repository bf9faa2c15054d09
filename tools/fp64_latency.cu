// Microbenchmark: dependent-chain latency of fp64 add / mul and F2F on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(const float* x, double* out, long long* cyc) {
  double s = 0.0, p = 1.0, f = 0.0;
  float v = x[threadIdx.x];
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < 4096; ++i) s = __dadd_rn(s, 1.0000001);
  long long t1 = clock64();
#pragma unroll 16
  for (int i = 0; i < 4096; ++i) p = __dmul_rn(p, 1.0000001);
  long long t2 = clock64();
#pragma unroll 16
  for (int i = 0; i < 4096; ++i) { f = (double)v; v = (float)f + 1.0f; }
  long long t3 = clock64();
  out[threadIdx.x] = s + p + f;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}
int main() {
  float* x; double* o; long long* c;
  cudaMalloc(&x, 128); cudaMalloc(&o, 256); cudaMallocManaged(&c, 64);
  cudaMemset(x, 0, 128);
  chain<<<1, 32>>>(x, o, c);
  cudaDeviceSynchronize();
  printf("cycles per dependent op: DADD %.2f  DMUL %.2f  F2F+F2F+FADD %.2f\n", c[0] / 4096.0, c[1] / 4096.0, c[2] / 4096.0);
  return 0;
}

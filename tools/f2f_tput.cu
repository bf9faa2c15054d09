// Microbenchmark: throughput of float->double conversion (F2F) vs an integer
// bit-manipulation conversion, and of DADD/DMUL, with many warps per SM.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double f2d_int(float x) {
  const unsigned u = __float_as_uint(x);
  unsigned hi = (u & 0x80000000u) | (((u & 0x7fffffffu) >> 3) + (896u << 20));
  hi = ((u & 0x7f800000u) == 0u) ? (u & 0x80000000u) : hi;
  return __hiloint2double((int)hi, (int)(u << 29));
}
template <int MODE>
__global__ void k(const float* x, double* out) {
  float v[8];
  for (int i = 0; i < 8; ++i) v[i] = x[(threadIdx.x + i) & 255] + i;
  double acc[8] = {};
  for (int it = 0; it < 2048; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      double d;
      if (MODE == 0) d = (double)v[i];
      else if (MODE == 1) d = f2d_int(v[i]);
      else d = __dmul_rn((double)i, acc[i]);
      acc[i] = __dadd_rn(acc[i], d);
      v[i] += 1.0f;
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* x; double* o;
  cudaMalloc(&x, 1024); cudaMalloc(&o, 148 * 1024 * 8 * 4);
  cudaMemset(x, 0, 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[3] = {"F2F+DADD", "int f2d+DADD", "DMUL+DADD"};
  for (int m = 0; m < 3; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (m == 0) k<0><<<148 * 2, 512>>>(x, o);
      if (m == 1) k<1><<<148 * 2, 512>>>(x, o);
      if (m == 2) k<2><<<148 * 2, 512>>>(x, o);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double elems = 148.0 * 2 * 512 * 2048 * 8;
      if (rep) printf("%-14s %.3f ms  -> %.2f Gelem/s  (%.2f elem/clk/SM at 1.965 GHz)\n", names[m], ms, elems / ms / 1e6, elems / (ms * 1e-3) / 148 / 1.965e9);
    }
  }
  return 0;
}

// k_route.cu -- K4 router and K5 LUT builder.
//
// K4 (§IV.B.1 Router): remap every probe through the
// mapping tables (owner, local id), emit the miss mask for probes that
// are not GPU-resident and keep only this rank's probes ("effective
// nprobe per shard") as work items. Items are (query, probe) pairs in
// query-major order; item i owns ngroups(list) groups of 32 vectors and
// item_off is their exclusive prefix sum (item_off[n] = total groups W).
//
// K5 (stage 2 of Fig. 2): LUT_q[j][c] = -2 <q_j, y_{j,c}>, the
// query-dependent part of the residual-PQ distance,
// written in the scan's shared-memory layout [j/64][c][j%64] (padded
// sub-spaces j >= m hold 0).
#include "vlr_device.cuh"
#include "vlr_internal.cuh"

namespace vlr {

constexpr int kRouteThreads = 1024;

__global__ void __launch_bounds__(kRouteThreads) k_route(const int32_t* __restrict__ probes, int n, int rank,
                                                         const int32_t* __restrict__ owner,
                                                         const int32_t* __restrict__ local,
                                                         const int64_t* __restrict__ gbase,
                                                         uint8_t* __restrict__ miss, int32_t* __restrict__ probes_out,
                                                         int32_t* __restrict__ plocal,
                                                         int64_t* __restrict__ item_off) {
  __shared__ long long warp_sums[kRouteThreads / 32];
  __shared__ long long s_carry;
  if (threadIdx.x == 0) s_carry = 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int base = 0; base < n; base += kRouteThreads) {
    const int i = base + threadIdx.x;
    long long g = 0;
    if (i < n) {
      const int l = probes[i];
      const int o = owner[l];
      miss[i] = o < 0 ? 1 : 0;
      if (probes_out) probes_out[i] = l;
      const int loc = (o == rank) ? local[l] : -1;
      plocal[i] = loc;
      if (loc >= 0) g = gbase[loc + 1] - gbase[loc];
    }
    // block exclusive scan of g
    long long incl = g;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      long long v = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) warp_sums[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      long long ws = warp_sums[lane];
      long long wi = ws;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        long long v = __shfl_up_sync(kFull, wi, o);
        if (lane >= o) wi += v;
      }
      warp_sums[lane] = wi - ws;  // exclusive prefix of warp totals
    }
    __syncthreads();
    const long long carry = s_carry;
    if (i < n) item_off[i] = carry + warp_sums[wid] + incl - g;
    __syncthreads();
    if (threadIdx.x == kRouteThreads - 1) s_carry = carry + warp_sums[wid] + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) item_off[n] = s_carry;
}

cudaError_t launch_route(const DeviceIndex& ix, const Workspace& ws, int nq, int np, uint8_t* miss,
                         int32_t* probes_out, cudaStream_t s) {
  const int n = nq * np;
  k_route<<<1, kRouteThreads, 0, s>>>(ws.probes, n, ix.rank, ix.owner, ix.local, ix.gbase, miss, probes_out, ws.plocal,
                                      ws.item_off);
  return cudaGetLastError();
}

// ----------------------------------------------------------------- K5 LUT
__global__ void __launch_bounds__(256) k_lut(const float* __restrict__ Q, int d, int m, int dsub,
                                             const float* __restrict__ Y, int npairs, float* __restrict__ lut) {
  const int q = blockIdx.x, pair = blockIdx.y;
  extern __shared__ float qs[];
  for (int t = threadIdx.x; t < d; t += blockDim.x) qs[t] = Q[(size_t)q * d + t];
  __syncthreads();
  float* out = lut + ((size_t)q * npairs + pair) * (256 * 64);
  const int jj = threadIdx.x & 63;
  const int j = pair * 64 + jj;
  for (int c = threadIdx.x >> 6; c < 256; c += 4) {
    float v = 0.f;
    if (j < m) {
      const float* y = Y + ((size_t)j * 256 + c) * dsub;
      const float* qq = qs + j * dsub;
      float dot = 0.f;
      for (int u = 0; u < dsub; ++u) dot = fmaf(qq[u], __ldg(y + u), dot);
      v = -2.f * dot;
    }
    out[c * 64 + jj] = v;
  }
}

cudaError_t launch_lut(const float* Q, const DeviceIndex& ix, const Workspace& ws, int nq, cudaStream_t s) {
  if (nq <= 0) return cudaSuccess;
  dim3 grid(nq, ix.npairs);
  const size_t sm = (size_t)ix.d * sizeof(float);
  if (sm > 48 * 1024) cudaFuncSetAttribute(k_lut, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_lut<<<grid, 256, sm, s>>>(Q, ix.d, ix.m, ix.dsub, ix.codebooks, ix.npairs, ws.lut);
  return cudaGetLastError();
}

}  // namespace vlr

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
// grid (npairs * 4 code quarters, ceil(nq / kLutQB)); 256 threads = 4 codes x
// 64 sub-spaces (jj fastest -> coalesced LUT rows). Each thread keeps its
// codeword y_{j,c} in registers and reuses it for kLutQB queries, whose
// sub-vectors sit in shared memory padded to dsub+1 per sub-space (bank-
// conflict-free across the 64 sub-spaces of a warp).
constexpr int kLutQB = 8;
constexpr int kLutMaxDsub = 32;

__global__ void __launch_bounds__(256) k_lut(const float* __restrict__ Q, int nq, int d, int m, int dsub,
                                             const float* __restrict__ Y, int npairs, float* __restrict__ lut) {
  extern __shared__ float qs[];  // [kLutQB][64 * (dsub + 1)]
  const int pair = blockIdx.x >> 2, cq = blockIdx.x & 3;
  const int q0 = blockIdx.y * kLutQB;
  const int jj = threadIdx.x & 63, cs = threadIdx.x >> 6;
  const int j = pair * 64 + jj;
  const int jv = min(64, m - pair * 64);  // valid sub-spaces of this pair (>= 1)
  const int row = jv * (dsub + 1);
  for (int i = threadIdx.x; i < kLutQB * jv * dsub; i += blockDim.x) {
    const int qq = i / (jv * dsub), r = i - qq * jv * dsub;
    const int jl = r / dsub, u = r - jl * dsub;
    const int jg = pair * 64 + jl;
    float v = 0.f;
    if (q0 + qq < nq) v = Q[(size_t)(q0 + qq) * d + jg * dsub + u];
    qs[qq * row + jl * (dsub + 1) + u] = v;
  }
  __syncthreads();
  const int nqb = min(kLutQB, nq - q0);
  for (int c = cq * 64 + cs; c < cq * 64 + 64; c += 4) {
    float acc[kLutQB];
#pragma unroll
    for (int qq = 0; qq < kLutQB; ++qq) acc[qq] = 0.f;
    if (j < m) {
      const float* y = Y + ((size_t)j * 256 + c) * dsub;
      for (int u0 = 0; u0 < dsub; u0 += kLutMaxDsub) {
        float yr[kLutMaxDsub];
#pragma unroll
        for (int u = 0; u < kLutMaxDsub; ++u) yr[u] = (u0 + u < dsub) ? __ldg(y + u0 + u) : 0.f;
#pragma unroll
        for (int qq = 0; qq < kLutQB; ++qq) {
          const float* qv = qs + qq * row + jj * (dsub + 1) + u0;
          float a = acc[qq];
#pragma unroll
          for (int u = 0; u < kLutMaxDsub; ++u)
            if (u0 + u < dsub) a = fmaf(qv[u], yr[u], a);
          acc[qq] = a;
        }
      }
    }
    for (int qq = 0; qq < nqb; ++qq)
      lut[(((size_t)(q0 + qq) * npairs + pair) * 256 + c) * 64 + jj] = -2.f * acc[qq];
  }
}

cudaError_t launch_lut(const float* Q, const DeviceIndex& ix, const Workspace& ws, int nq, cudaStream_t s) {
  if (nq <= 0) return cudaSuccess;
  dim3 grid(ix.npairs * 4, (nq + kLutQB - 1) / kLutQB);
  const size_t sm = (size_t)kLutQB * (ix.m < 64 ? ix.m : 64) * (ix.dsub + 1) * sizeof(float);
  static size_t configured = 0;
  if (sm > 48 * 1024 && sm > configured) {
    cudaError_t e = cudaFuncSetAttribute(k_lut, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    configured = sm;
  }
  k_lut<<<grid, 256, sm, s>>>(Q, nq, ix.d, ix.m, ix.dsub, ix.codebooks, ix.npairs, ws.lut);
  return cudaGetLastError();
}

}  // namespace vlr

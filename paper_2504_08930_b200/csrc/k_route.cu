// k_route.cu -- K4 router and K5 LUT builder.
//
// K4 (§IV.B.1 Router): every probe is remapped through the
// mapping tables (owner, local id), the miss mask marks probes that are
// not GPU-resident and only this rank's probes ("effective nprobe per
// shard") become work items -- done in the epilogue of K3 (k_coarse.cu),
// which also writes each item's within-query prefix of groups. Items are
// (query, probe) pairs in query-major order; item i owns ngroups(list) groups
// of 32 vectors; K4b (below) turns the per-query prefixes into the global
// exclusive prefix item_off (item_off[n] = total groups W).
//
// K5 (stage 2 of Fig. 2): LUT_q[j][c] = -2 <q_j, y_{j,c}>, the
// query-dependent part of the residual-PQ distance;
// -<q_j, y_{j,c}> for the inner-product metric (NEXT-3),
// written in the scan's shared-memory layout [j/64][c][j%64] (padded
// sub-spaces j >= m hold 0).
#include "vlr_device.cuh"
#include "vlr_internal.cuh"

namespace vlr {

// K4b: item_off[q*np + p] = sum_{q' < q} qtot[q'] + item_local[q*np + p];
// item_off[nq*np] = W. Every block recomputes the (short) query prefix in
// shared memory, so there is no serial pass over the items.
constexpr int kOffThreads = 256;

__global__ void __launch_bounds__(kOffThreads) k_offsets(int nq, int np, const int64_t* __restrict__ qtot,
                                                         const int64_t* __restrict__ item_local,
                                                         int64_t* __restrict__ item_off) {
  pdl_entry();  // PDL: wait for the previous kernel in the stream, then let the next one launch
  extern __shared__ long long qbase[];  // [nq + 1]
  __shared__ long long wsum[kOffThreads / 32];
  __shared__ long long carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < nq; b0 += kOffThreads) {
    const int i = b0 + threadIdx.x;
    const long long v = i < nq ? qtot[i] : 0;
    long long incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long t = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    long long wb = 0, tot = 0;
    for (int w = 0; w < kOffThreads / 32; ++w) {
      if (w < warp) wb += wsum[w];
      tot += wsum[w];
    }
    const long long c0 = carry;
    if (i < nq) qbase[i] = c0 + wb + incl - v;
    __syncthreads();
    if (threadIdx.x == 0) carry = c0 + tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) qbase[nq] = carry;
  __syncthreads();
  const long long n = (long long)nq * np;
  for (long long i = blockIdx.x * (long long)kOffThreads + threadIdx.x; i < n; i += (long long)gridDim.x * kOffThreads)
    item_off[i] = qbase[i / np] + item_local[i];
  if (blockIdx.x == 0 && threadIdx.x == 0) item_off[n] = qbase[nq];
}

cudaError_t launch_offsets(const DeviceIndex& ix, const Workspace& ws, int nq, int np, cudaStream_t s) {
  const long long n = (long long)nq * np;
  long long blocks = (n + kOffThreads - 1) / kOffThreads;
  if (blocks > 148 * 4) blocks = 148 * 4;
  if (blocks < 1) blocks = 1;
  const size_t sm = (size_t)(nq + 1) * sizeof(long long);
  cudaError_t e = ensure_smem((const void*)k_offsets, sm);
  if (e != cudaSuccess) return e;
  (void)ix;
  return launch_pdl(k_offsets, dim3((int)blocks), dim3(kOffThreads), sm, s, nq, np, ws.qtot, ws.item_local,
                    ws.item_off);
}

// ----------------------------------------------------------------- K5 LUT
// grid (npairs * 4 code quarters, ceil(nq / kLutQB)); 256 threads = 16 x 4
// sub-spaces (jj4) x 16 code slots (cc). A thread computes 4 consecutive
// sub-spaces x 4 codes x kLutQB queries: codewords stay in registers across
// the queries, query sub-vectors come from shared memory (padded to dsub+1
// per sub-space), and each (code, query) result is one 16-B store (the 16
// jj4 lanes of a code write 256 contiguous bytes of the LUT row).
constexpr int kLutQB = 8;

__global__ void __launch_bounds__(256) k_lut(const float* __restrict__ Q, int nq, int d, int m, int dsub,
                                             const float* __restrict__ Y, int npairs, float scale,
                                             float* __restrict__ lut) {
  extern __shared__ float qs[];  // [kLutQB][jv * (dsub + 1)]
  const int pair = blockIdx.x >> 2, cq = blockIdx.x & 3;
  const int q0 = blockIdx.y * kLutQB;
  const int jj4 = threadIdx.x & 15, cc = threadIdx.x >> 4;
  const int jv = min(64, m - pair * 64);  // valid sub-spaces of this pair (>= 1)
  const int row = jv * (dsub + 1);
  for (int i = threadIdx.x; i < kLutQB * jv * dsub; i += blockDim.x) {
    const int qq = i / (jv * dsub), r = i - qq * jv * dsub;
    const int jl = r / dsub, u = r - jl * dsub;
    float v = 0.f;
    if (q0 + qq < nq) v = Q[(size_t)(q0 + qq) * d + (pair * 64 + jl) * dsub + u];
    qs[qq * row + jl * (dsub + 1) + u] = v;
  }
  __syncthreads();
  const int nqb = min(kLutQB, nq - q0);
#pragma unroll 1
  for (int ci = 0; ci < 4; ++ci) {
    const int c = cq * 64 + cc + 16 * ci;
    float acc[4][kLutQB];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int qq = 0; qq < kLutQB; ++qq) acc[a][qq] = 0.f;
    for (int u0 = 0; u0 < dsub; u0 += 8) {
      float yr[4][8];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int jl = 4 * jj4 + a;
        const float* y = Y + ((size_t)(pair * 64 + jl) * 256 + c) * dsub + u0;
#pragma unroll
        for (int u = 0; u < 8; ++u) yr[a][u] = (jl < jv && u0 + u < dsub) ? __ldg(y + u) : 0.f;
      }
#pragma unroll
      for (int qq = 0; qq < kLutQB; ++qq) {
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const int jl = min(4 * jj4 + a, jv - 1);
          const float* qv = qs + qq * row + jl * (dsub + 1) + u0;
          float t = acc[a][qq];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (u0 + u < dsub) t = fmaf(qv[u], yr[a][u], t);
          acc[a][qq] = t;
        }
      }
    }
    for (int qq = 0; qq < nqb; ++qq) {
      const float4 v = make_float4(scale * acc[0][qq], scale * acc[1][qq], scale * acc[2][qq], scale * acc[3][qq]);
      *reinterpret_cast<float4*>(lut + (((size_t)(q0 + qq) * npairs + pair) * 256 + c) * 64 + 4 * jj4) = v;
    }
  }
}

// Fast path for dsub == 8 (every BASELINE config): thread (jj, cs) keeps the 8
// queries' sub-vectors of sub-space jj in registers (64 floats) and walks 16
// codes: per code 2 LDG.128 of the codeword, 64 FMA, 8 coalesced stores.
__global__ void __launch_bounds__(256) k_lut8(const float* __restrict__ Q, int nq, int d, int m,
                                              const float* __restrict__ Y, int npairs, float scale,
                                              float* __restrict__ lut) {
  const int pair = blockIdx.x >> 2, cq = blockIdx.x & 3;
  const int q0 = blockIdx.y * kLutQB;
  const int jj = threadIdx.x & 63, cs = threadIdx.x >> 6;
  const int j = pair * 64 + jj;
  const int nqb = min(kLutQB, nq - q0);
  float qv[kLutQB][8];
#pragma unroll
  for (int qq = 0; qq < kLutQB; ++qq) {
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
    if (qq < nqb && j < m) {
      const float4* src = reinterpret_cast<const float4*>(Q + (size_t)(q0 + qq) * d + j * 8);
      a = __ldg(src);
      b = __ldg(src + 1);
    }
    qv[qq][0] = a.x; qv[qq][1] = a.y; qv[qq][2] = a.z; qv[qq][3] = a.w;
    qv[qq][4] = b.x; qv[qq][5] = b.y; qv[qq][6] = b.z; qv[qq][7] = b.w;
  }
#pragma unroll 2
  for (int i = 0; i < 16; ++i) {
    const int c = cq * 64 + cs + 4 * i;
    float4 ya = make_float4(0.f, 0.f, 0.f, 0.f), yb = ya;
    if (j < m) {
      const float4* y = reinterpret_cast<const float4*>(Y + ((size_t)j * 256 + c) * 8);
      ya = __ldg(y);
      yb = __ldg(y + 1);
    }
#pragma unroll
    for (int qq = 0; qq < kLutQB; ++qq) {
      float t = 0.f;
      t = fmaf(qv[qq][0], ya.x, t); t = fmaf(qv[qq][1], ya.y, t);
      t = fmaf(qv[qq][2], ya.z, t); t = fmaf(qv[qq][3], ya.w, t);
      t = fmaf(qv[qq][4], yb.x, t); t = fmaf(qv[qq][5], yb.y, t);
      t = fmaf(qv[qq][6], yb.z, t); t = fmaf(qv[qq][7], yb.w, t);
      if (qq < nqb) lut[(((size_t)(q0 + qq) * npairs + pair) * 256 + c) * 64 + jj] = scale * t;
    }
  }
}

// 4-bit codes (16 codewords per sub-space): LUT_q[pair][c][jj], c < 16. One
// CTA per (pair, query), thread (jj, c) = one fp32 dot of dsub terms; the 64
// jj lanes of a code write 256 contiguous bytes.
__global__ void __launch_bounds__(1024) k_lut16(const float* __restrict__ Q, int d, int m, int dsub,
                                                const float* __restrict__ Y, int npairs, float scale,
                                                float* __restrict__ lut) {
  const int pair = blockIdx.x, q = blockIdx.y;
  const int jj = threadIdx.x & 63, c = threadIdx.x >> 6;
  const int j = pair * 64 + jj;
  float t = 0.f;
  if (j < m) {
    const float* qv = Q + (size_t)q * d + (size_t)j * dsub;
    const float* y = Y + ((size_t)j * 16 + c) * dsub;
    for (int u = 0; u < dsub; ++u) t = fmaf(__ldg(qv + u), __ldg(y + u), t);
  }
  lut[(((size_t)q * npairs + pair) * 16 + c) * 64 + jj] = scale * t;
}

// 4-bit codes, PAIR mode (default; DESIGN.md §K6 4-bit): slot j' = packed byte
// b of sub-codes 2j' (low nibble) and 2j'+1 (high nibble), looked up in a
// 256-entry pair table LUT2_q[j'][b] = LUT_q[2j'][b & 15] + LUT_q[2j'+1][b >> 4]
// (fp32; a missing sub-space 2j'+1 = m contributes 0). Same layout as the
// 8-bit LUT ([pair of 64 slots][256][64]), so the 8-bit scan consumes it with
// half the lookups of the nibble scan. One CTA per (64 slots, query): the 2 x
// 16 x 64 sub-dots go to shared memory, then 256 x 64 sums are written.
__global__ void __launch_bounds__(256) k_lut_pair(const float* __restrict__ Q, int d, int m, int dsub,
                                                  const float* __restrict__ Y, int npairs, float scale,
                                                  float* __restrict__ lut) {
  __shared__ float s_t[2][16][64];
  const int pair = blockIdx.x, q = blockIdx.y;
  for (int i = threadIdx.x; i < 2 * 16 * 64; i += blockDim.x) {
    const int jj = i & 63, c = (i >> 6) & 15, hf = i >> 10;
    const int j = 2 * (pair * 64 + jj) + hf;
    float t = 0.f;
    if (j < m) {
      const float* qv = Q + (size_t)q * d + (size_t)j * dsub;
      const float* y = Y + ((size_t)j * 16 + c) * dsub;
      for (int u = 0; u < dsub; ++u) t = fmaf(__ldg(qv + u), __ldg(y + u), t);
    }
    s_t[hf][c][jj] = scale * t;
  }
  __syncthreads();
  float* out = lut + ((size_t)q * npairs + pair) * 256 * 64;
  for (int i = threadIdx.x; i < 256 * 64; i += blockDim.x) {
    const int jj = i & 63, c = i >> 6;
    out[i] = s_t[0][c & 15][jj] + s_t[1][c >> 4][jj];
  }
}

cudaError_t launch_lut(const float* Q, const DeviceIndex& ix, const Workspace& ws, int nq, cudaStream_t s) {
  if (nq <= 0) return cudaSuccess;
  const float scale = ix.metric == 1 ? -1.f : -2.f;  // exact power-of-two scaling of the fp32 dot
  if (ix.nbits == 4 && ix.code_bits == 8) {
    k_lut_pair<<<dim3(ix.npairs, nq), 256, 0, s>>>(Q, ix.d, ix.m, ix.dsub, ix.codebooks, ix.npairs, scale, ws.lut);
    return cudaGetLastError();
  }
  if (ix.nbits == 4) {
    k_lut16<<<dim3(ix.npairs, nq), 1024, 0, s>>>(Q, ix.d, ix.m, ix.dsub, ix.codebooks, ix.npairs, scale, ws.lut);
    return cudaGetLastError();
  }
  dim3 grid(ix.npairs * 4, (nq + kLutQB - 1) / kLutQB);
  if (ix.dsub == 8 && (ix.d % 4) == 0) {
    k_lut8<<<grid, 256, 0, s>>>(Q, nq, ix.d, ix.m, ix.codebooks, ix.npairs, scale, ws.lut);
    return cudaGetLastError();
  }
  const size_t sm = (size_t)kLutQB * (ix.m < 64 ? ix.m : 64) * (ix.dsub + 1) * sizeof(float);
  cudaError_t e = ensure_smem((const void*)k_lut, sm);
  if (e != cudaSuccess) return e;
  k_lut<<<grid, 256, sm, s>>>(Q, nq, ix.d, ix.m, ix.dsub, ix.codebooks, ix.npairs, scale, ws.lut);
  return cudaGetLastError();
}

// ----------------------------------------------------------------- access histogram
// NEXT-2 ("the router monitors ... per-cluster access
// frequencies"): counts[l] += number of (query, probe) pairs that probed l.
// Warp-aggregated atomics on int64 counters.
__global__ void k_access_hist(const int32_t* __restrict__ probes, long long n, int nlist,
                              unsigned long long* __restrict__ counts) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int l = probes[i];
    if (l >= 0 && l < nlist) atomicAdd(counts + l, 1ull);
  }
}

cudaError_t launch_access_hist(const int32_t* probes, long long n, int nlist, unsigned long long* counts,
                               cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_access_hist<<<(int)blocks, 256, 0, s>>>(probes, n, nlist, counts);
  return cudaGetLastError();
}

}  // namespace vlr

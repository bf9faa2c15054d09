// k_coarse.cu -- coarse quantizer of the IVF-PQ search (stage 1 of Fig. 2,
// PAPER.md:117, :147): which nprobe clusters each query visits.
//
//  qprep   : ||q|| per query, non-finite check (status bit 0).
//  K1 simt : filter distances dt[q][l] = ||c_l||^2 - 2<q, c_l> (fp32 FMA).
//            (The tcgen05 TF32 filter in k_filter_tc.cu computes the same
//            quantity on the tensor cores.)
//  K2      : theta~ = nprobe'-th smallest dt (radix select), candidate set
//            {l : dt <= theta~ + 2 Delta*} (DESIGN.md §K1-K3 band proof).
//  K3      : exact fp64 D = sum_t (q_t - c_t)^2 in dimension order with
//            correctly-rounded dsub/dmul/dadd (no FMA) for the candidates,
//            sort by (D, l), keep nprobe' -> probes + term1 = (float)D.
//            Bit-identical to the definition.
#include <cfloat>

#include "vlr_device.cuh"
#include "vlr_internal.cuh"

namespace vlr {

// ----------------------------------------------------------------- qprep
__global__ void k_qprep(const float* __restrict__ Q, int d, int d4, float* __restrict__ qnorm,
                        float* __restrict__ qtf32, int32_t* status) {
  const int q = blockIdx.x;
  const float* row = Q + (size_t)q * d;
  double s = 0.0;
  bool bad = false;
  for (int t = threadIdx.x; t < d4; t += blockDim.x) {
    float v = t < d ? row[t] : 0.f;
    bad |= !isfinite(v);
    s += (double)v * (double)v;
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
    qtf32[(size_t)q * d4 + t] = __uint_as_float(r);
  }
  __shared__ double red[32];
  __shared__ int sbad;
  if (threadIdx.x == 0) sbad = 0;
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  __syncthreads();
  if (bad) atomicOr(&sbad, 1);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    qnorm[q] = (float)sqrt(t) * 1.0000002f;
    if (sbad) atomicOr(status, 1);
  }
}

cudaError_t launch_qprep(const float* Q, int nq, int d, int d4, float* qnorm, float* qtf32, int32_t* status,
                         cudaStream_t s) {
  if (nq <= 0) return cudaSuccess;
  k_qprep<<<nq, 256, 0, s>>>(Q, d, d4, qnorm, qtf32, status);
  return cudaGetLastError();
}

// ----------------------------------------------------------------- K1 (SIMT)
// 64 queries x 64 centroids per CTA, 256 threads, 4x4 outputs each, BK = 16.
constexpr int FB = 64, FK = 16;
__global__ void __launch_bounds__(256) k_filter_simt(const float* __restrict__ Q, int nq, const float* __restrict__ C,
                                                     const float* __restrict__ cn2, int L, int d,
                                                     float* __restrict__ dt) {
  __shared__ float sq[FK][FB + 4];
  __shared__ float sc[FK][FB + 4];
  const int q0 = blockIdx.y * FB, l0 = blockIdx.x * FB;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < d; k0 += FK) {
    for (int i = threadIdx.x; i < FB * FK; i += 256) {
      int r = i / FK, c = i % FK;
      int gq = q0 + r, gl = l0 + r, gk = k0 + c;
      sq[c][r] = (gq < nq && gk < d) ? Q[(size_t)gq * d + gk] : 0.f;
      sc[c][r] = (gl < L && gk < d) ? C[(size_t)gl * d + gk] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < FK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sq[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = sc[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int gq = q0 + ty * 4 + i;
    if (gq >= nq) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int gl = l0 + tx * 4 + j;
      if (gl < L) dt[(size_t)gq * L + gl] = cn2[gl] - 2.f * acc[i][j];
    }
  }
}

cudaError_t launch_filter_simt(const float* Q, int nq, const DeviceIndex& ix, float* dt, cudaStream_t s) {
  if (nq <= 0) return cudaSuccess;
  dim3 grid((ix.nlist + FB - 1) / FB, (nq + FB - 1) / FB);
  k_filter_simt<<<grid, 256, 0, s>>>(Q, nq, ix.centroids, ix.cnorm2, ix.nlist, ix.d, dt);
  return cudaGetLastError();
}

// ----------------------------------------------------------------- K2 select
// One CTA (1024 threads) per query. Radix select (4 x 8-bit digits) of the
// np-th smallest order key, then the band bound and candidate compaction.
__global__ void __launch_bounds__(1024) k_select(const float* __restrict__ dt, int L, int np,
                                                 const float* __restrict__ qnorm, float cmax, float e_dot,
                                                 int32_t* __restrict__ cand, int32_t* __restrict__ ncand,
                                                 float* __restrict__ bound_out) {
  const int q = blockIdx.x;
  const float* row = dt + (size_t)q * L;
  __shared__ unsigned hist[256];
  __shared__ unsigned s_prefix, s_want, s_cnt;
  unsigned prefix = 0u, mask = 0u, want = (unsigned)np;
  const int lane = threadIdx.x & 31;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0u;
    __syncthreads();
    for (int i0 = 0; i0 < L; i0 += blockDim.x) {
      const int i = i0 + threadIdx.x;
      bool act = false;
      unsigned bin = 0u;
      if (i < L) {
        unsigned key = fkey(row[i]);
        act = (key & mask) == prefix;
        bin = (key >> shift) & 255u;
      }
      // warp-aggregated histogram update
      const unsigned am = __ballot_sync(kFull, act);
      if (act) {
        const unsigned peers = __match_any_sync(am, bin);
        if (lane == __ffs(peers) - 1) atomicAdd(&hist[bin], (unsigned)__popc(peers));
      }
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      // lane handles bins [8*lane, 8*lane+8): find the bin holding the want-th key
      unsigned loc[8], tot = 0u;
#pragma unroll
      for (int b = 0; b < 8; ++b) { loc[b] = hist[lane * 8 + b]; tot += loc[b]; }
      unsigned incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        unsigned v = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += v;
      }
      const unsigned excl = incl - tot;
      if (excl < want && want <= incl) {
        unsigned c = excl;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          if (c < want && want <= c + loc[b]) {
            s_prefix = prefix | ((unsigned)(lane * 8 + b) << shift);
            s_want = want - c;
          }
          c += loc[b];
        }
      }
    }
    __syncthreads();
    prefix = s_prefix;
    want = s_want;
    mask |= 255u << shift;
    __syncthreads();
  }
  const float theta = fkey_inv(prefix);
  // band (Appendix A of SURVEY / DESIGN §K1-K3): Delta* bounds |dt - (D - ||q||^2)|
  const float qn = qnorm[q];
  const float u = 5.9604645e-8f;  // 2^-24
  const float delta = 2.0f * (2.0f * (e_dot + 2.0f * u) * qn * cmax + 4.0f * u * (cmax * cmax + qn * qn));
  const float bnd = theta + 2.0f * delta;
  if (threadIdx.x == 0) {
    s_cnt = 0u;
    bound_out[q] = bnd;
  }
  __syncthreads();
  int32_t* out = cand + (size_t)q * kCandCap;
  for (int i0 = 0; i0 < L; i0 += blockDim.x) {
    const int i = i0 + threadIdx.x;
    const bool keep = i < L && row[i] <= bnd;
    const unsigned km = __ballot_sync(kFull, keep);
    unsigned base = 0u;
    if (lane == 0 && km) base = atomicAdd(&s_cnt, (unsigned)__popc(km));
    base = __shfl_sync(kFull, base, 0);
    if (keep) {
      const unsigned pos = base + __popc(km & ((1u << lane) - 1u));
      if (pos < (unsigned)kCandCap) out[pos] = i;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) ncand[q] = (int32_t)s_cnt;
}

cudaError_t launch_select(const DeviceIndex& ix, const Workspace& ws, int nq, int np, float e_dot, cudaStream_t s) {
  if (nq <= 0) return cudaSuccess;
  k_select<<<nq, 1024, 0, s>>>(ws.dt, ix.nlist, np, ws.qnorm, ix.cmax, e_dot, ws.cand, ws.ncand, ws.bound);
  return cudaGetLastError();
}

// ----------------------------------------------------------------- K3 refine
constexpr int kRefineThreads = 256;
constexpr int kSortCap = 2048;  // >= kMaxNprobe + kRefineChunk

__device__ __forceinline__ double exact_coarse(const float* __restrict__ qs, const float* __restrict__ c, int d) {
  // D = sum_{t=0}^{d-1} (q_t - c_t)^2, left to right, each op correctly rounded
  double s = 0.0;
  int t = 0;
  if ((d & 3) == 0) {
    const float4* c4 = reinterpret_cast<const float4*>(c);
    for (; t < d; t += 4) {
      const float4 v = __ldg(c4 + (t >> 2));
      double e;
      e = __dsub_rn((double)qs[t + 0], (double)v.x); s = __dadd_rn(s, __dmul_rn(e, e));
      e = __dsub_rn((double)qs[t + 1], (double)v.y); s = __dadd_rn(s, __dmul_rn(e, e));
      e = __dsub_rn((double)qs[t + 2], (double)v.z); s = __dadd_rn(s, __dmul_rn(e, e));
      e = __dsub_rn((double)qs[t + 3], (double)v.w); s = __dadd_rn(s, __dmul_rn(e, e));
    }
  } else {
    for (; t < d; ++t) {
      const double e = __dsub_rn((double)qs[t], (double)__ldg(c + t));
      s = __dadd_rn(s, __dmul_rn(e, e));
    }
  }
  return s;
}

__device__ __forceinline__ bool key_less(double a, int ia, double b, int ib) {
  return a < b || (a == b && ia < ib);
}

// bitonic sort of n (power of two) (key, id) pairs in shared memory, ascending
__device__ void bitonic_sort(double* key, int* id, int n) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < (n >> 1); i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const double ka = key[lo], kb = key[hi];
        const int ia = id[lo], ib = id[hi];
        const bool swap = up ? key_less(kb, ib, ka, ia) : key_less(ka, ia, kb, ib);
        if (swap) {
          key[lo] = kb; key[hi] = ka;
          id[lo] = ib; id[hi] = ia;
        }
      }
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kRefineThreads) k_refine(const float* __restrict__ Q, const float* __restrict__ C,
                                                           int d, int L, int np, const float* __restrict__ dt,
                                                           const int32_t* __restrict__ cand,
                                                           const int32_t* __restrict__ ncand,
                                                           const float* __restrict__ bound,
                                                           int32_t* __restrict__ probes, float* __restrict__ term1) {
  extern __shared__ __align__(16) unsigned char sm[];
  double* key = reinterpret_cast<double*>(sm);             // [kSortCap]
  int* id = reinterpret_cast<int*>(key + kSortCap);        // [kSortCap]
  int* lbuf = id + kSortCap;                               // [kRefineChunk]
  float* qs = reinterpret_cast<float*>(lbuf + kRefineChunk);  // [d]
  __shared__ int s_cnt;
  const int q = blockIdx.x;
  for (int t = threadIdx.x; t < d; t += blockDim.x) qs[t] = Q[(size_t)q * d + t];
  const int nc = ncand[q];
  const bool listed = nc <= kCandCap;
  const int src_len = listed ? nc : L;
  const float bnd = bound[q];
  const int32_t* lst = cand + (size_t)q * kCandCap;
  const float* row = dt + (size_t)q * L;
  int nbest = 0;
  int pos = 0;
  __syncthreads();
  while (pos < src_len) {
    // gather up to kRefineChunk candidate ids
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    if (listed) {
      const int take = min(kRefineChunk, src_len - pos);
      for (int i = threadIdx.x; i < take; i += blockDim.x) lbuf[i] = lst[pos + i];
      pos += take;
      if (threadIdx.x == 0) s_cnt = take;
    } else {
      while (pos < src_len) {
        __syncthreads();
        if (s_cnt + (int)blockDim.x > kRefineChunk) break;
        const int i = pos + threadIdx.x;
        if (i < src_len && row[i] <= bnd) lbuf[atomicAdd(&s_cnt, 1)] = i;
        pos += blockDim.x;
      }
    }
    __syncthreads();
    const int cnt = s_cnt;
    // exact distances
    for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
      const int l = lbuf[j];
      key[nbest + j] = exact_coarse(qs, C + (size_t)l * d, d);
      id[nbest + j] = l;
    }
    const int tot = nbest + cnt;
    int n2 = 1;
    while (n2 < tot) n2 <<= 1;
    for (int j = tot + threadIdx.x; j < n2; j += blockDim.x) {
      key[j] = DBL_MAX;
      id[j] = 0x7fffffff;
    }
    bitonic_sort(key, id, n2);
    nbest = min(np, tot);
  }
  for (int p = threadIdx.x; p < np; p += blockDim.x) {
    // nbest == np whenever the candidate set holds >= np clusters (always: the band
    // contains the np smallest); defensive -1 otherwise
    probes[(size_t)q * np + p] = p < nbest ? id[p] : -1;
    term1[(size_t)q * np + p] = p < nbest ? __double2float_rn(key[p]) : CUDART_INF_F;
  }
}

size_t refine_smem(int d) {
  return (size_t)kSortCap * (sizeof(double) + sizeof(int)) + kRefineChunk * sizeof(int) + (size_t)d * sizeof(float);
}

cudaError_t launch_refine(const float* Q, const DeviceIndex& ix, const Workspace& ws, int nq, int np, cudaStream_t s) {
  if (nq <= 0) return cudaSuccess;
  const size_t sm = refine_smem(ix.d);
  static int configured_for = -1;
  if (sm > 48 * 1024 && configured_for < (int)sm) {
    cudaError_t e = cudaFuncSetAttribute(k_refine, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    configured_for = (int)sm;
  }
  k_refine<<<nq, kRefineThreads, sm, s>>>(Q, ix.centroids, ix.d, ix.nlist, np, ws.dt, ws.cand, ws.ncand, ws.bound,
                                           ws.probes, ws.term1);
  return cudaGetLastError();
}

}  // namespace vlr

// k_coarse.cu -- coarse quantizer of the IVF-PQ search (stage 1 of Fig. 2,
// PAPER.md:117, :147): which nprobe clusters each query visits.
//
//  qprep   : ||q|| per query, non-finite check (status bit 0).
//  (K1, the filter dt[q][l] = ||c_l||^2 - 2<q~, c~_l> on the tcgen05 tensor
//   cores, is in k_filter_tc.cu.)
//  K2      : theta~ = nprobe'-th smallest dt (radix select), candidate set
//            {l : dt <= theta~ + 2 Delta*} (DESIGN.md §K1-K3 band proof).
//  K3      : exact fp64 D = sum_t (q_t - c_t)^2 in dimension order with
//            correctly-rounded dsub/dmul/dadd (no FMA) for the candidates,
//            sort by (D, l), keep nprobe' -> probes + term1 = (float)D.
//            Bit-identical to the definition. Inner-product
//            metric (NEXT-3): D = -sum_t q_t c_t (products exact in fp64, the
//            sum in dimension order); the filter then holds -2<q, c>
//            (||c||^2 = 0 in K1), the same key scaled by 2.
#include <algorithm>
#include <cfloat>
#include <cstdio>

#include <cuda_fp16.h>

#include "vlr_device.cuh"
#include "vlr_internal.cuh"

namespace vlr {

// ----------------------------------------------------------------- qprep
// ||q|| (fp64 sum, rounded up), non-finite check, and the filter operand
// fp16(q 2^e_q) with 2^e_q the power of two putting max |q_t| 2^e_q in
// [2^13, 2^14) (exponent clamped to [-60, 60]; DESIGN.md §5 bounds the
// subnormal flush that clamping can cause).
// qf16t (optional): the same fp16 operand pre-tiled for K1's B loads: [qtile of QT rows][kblock of 64][QT rows]
// [64 cols], each 128-B row's 16-B chunks XOR-swizzled by (row & 7) (the SW128 K-major image), so a K1 stage's
// B tile is ONE contiguous bulk copy; rows of the last tile past nq are zero (CTAs q >= nq write only those).
__global__ void k_qprep(const float* __restrict__ Q, int nq, int d, int d8, float* __restrict__ qnorm,
                        float* __restrict__ qsq, uint16_t* __restrict__ qf16, float* __restrict__ qinv, int32_t* status,
                        uint16_t* __restrict__ qf16t, int QT) {
  pdl_entry();  // PDL: wait for the previous kernel in the stream, then let the next one launch
  const int q = blockIdx.x;
  if (q >= nq) {  // zero padding rows of the tiled operand
    const int qt = q / QT, r = q % QT, kbn = (d8 + 63) / 64;
    for (int t = threadIdx.x; t < kbn * 64; t += blockDim.x) {
      const int kb = t >> 6, col = t & 63;
      qf16t[((size_t)(qt * kbn + kb) * QT + r) * 64 + (((col >> 3) ^ (r & 7)) << 3) + (col & 7)] = 0;
    }
    return;
  }
  const float* row = Q + (size_t)q * d;
  double s = 0.0;
  float mx = 0.f;
  bool bad = false;
  for (int t = threadIdx.x; t < d; t += blockDim.x) {
    const float v = row[t];
    bad |= !isfinite(v);
    s += (double)v * (double)v;
    mx = fmaxf(mx, fabsf(v));
  }
  __shared__ double red[32];
  __shared__ float redm[32];
  __shared__ int sbad;
  __shared__ float s_scale;
  if (threadIdx.x == 0) sbad = 0;
  for (int o = 16; o; o >>= 1) {
    s += __shfl_xor_sync(kFull, s, o);
    mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
  }
  __syncthreads();
  if (bad) atomicOr(&sbad, 1);
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = s;
    redm[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    float m = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      t += red[w];
      m = fmaxf(m, redm[w]);
    }
    qnorm[q] = (float)sqrt(t) * 1.0000002f;
    qsq[q] = (float)t;
    int e = 0;
    if (m > 0.f && isfinite(m)) {
      frexpf(m, &e);  // m < 2^e
      e = 14 - e;
      e = e < -60 ? -60 : (e > 60 ? 60 : e);
    }
    s_scale = ldexpf(1.f, e);
    qinv[q] = ldexpf(1.f, -e);
    if (sbad) atomicOr(status, 1);
  }
  __syncthreads();
  const float sc = s_scale;
  const int kbn = (d8 + 63) / 64;
  for (int t = threadIdx.x; t < (qf16t ? kbn * 64 : d8); t += blockDim.x) {
    const float v = t < d ? row[t] * sc : 0.f;
    const uint16_t h = __half_as_ushort(__float2half_rn(v));
    if (t < d8) qf16[(size_t)q * d8 + t] = h;
    if (qf16t) {
      const int qt = q / QT, r = q % QT, kb = t >> 6, col = t & 63;
      qf16t[((size_t)(qt * kbn + kb) * QT + r) * 64 + (((col >> 3) ^ (r & 7)) << 3) + (col & 7)] = h;
    }
  }
}

cudaError_t launch_qprep(const float* Q, int nq, int d, int d8, float* qnorm, float* qsq, uint16_t* qf16, float* qinv,
                         int32_t* status, uint16_t* qf16t, int QT, cudaStream_t s) {
  if (nq <= 0) return cudaSuccess;
  const int grid = qf16t ? (nq + QT - 1) / QT * QT : nq;
  return launch_pdl(k_qprep, dim3(grid), dim3(256), 0, s, Q, nq, d, d8, qnorm, qsq, qf16, qinv, status, qf16t, QT);
}

// ----------------------------------------------------------------- K2 select
// One CTA per query. theta' = the np-th smallest of the 32-centroid group
// minima written by K1 (a subset order statistic, so theta' >= theta~, the
// np-th smallest filter value), found by a radix select in
// shared memory; if there are fewer groups than np, theta' = +inf (every
// centroid is a candidate). Then one coalesced pass over the filter row
// compacts {l : dt[l] <= theta' + 2 Delta*}.
//
// Centroid-sharded coarse stage (world > 1):
// rank r filters only its centroid range [lo, hi) (K1 writes those columns),
// and the global theta' is assembled from every rank's share in two modes:
//  kSelStage1: theta_r = the np-th smallest of the rank's OWN group minima;
//     x1[q][0..np) = the multiset of its np smallest group minima (values
//     < theta_r, then theta_r repeated; +inf padding if the range has fewer
//     than np groups). No compaction.
//  kSelStage2: theta' = the np-th smallest of the G*np values gathered from
//     every rank (x1_all [G][nq][np]): the np smallest group minima of all L
//     centroids are among them, so theta' is exactly the single-GPU theta'
//     (+inf when fewer than np groups exist in total); then the compaction
//     over [lo, hi) as in kSelFull. The band bound is the same expression of
//     replicated scalars on every rank, so the union of the ranks' candidate
//     sets is the single-GPU candidate set.
constexpr int kSelThreads = 1024;
constexpr int kSelMaxGroups = 16384;  // groups per rank <= 16384 (nlist <= 512K) for the sorted-minima path
constexpr int kSelGroupCap = 2048;    // qualifying 32-centroid groups gathered per query (else: full row scan)
constexpr int kSelGather = 8192;      // filter values gathered per query in shared memory (the theta~ select)

// radix select (4 x 8-bit digits) of the want-th smallest (1-based) of n order-preserving keys in shared
// memory; the whole CTA calls it, the result is CTA-uniform
__device__ unsigned radix_select_kth(const unsigned* skeys, int n, unsigned want) {
  __shared__ unsigned hist[256];
  __shared__ unsigned s_prefix, s_want;
  const int lane = threadIdx.x & 31;
  unsigned prefix = 0u, mask = 0u;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0u;
    __syncthreads();
    for (int i0 = 0; i0 < n; i0 += blockDim.x) {
      const int i = i0 + threadIdx.x;
      const unsigned key = i < n ? skeys[i] : 0u;
      const bool act = i < n && (key & mask) == prefix;
      const unsigned bin = (key >> shift) & 255u;
      // plain shared-memory atomics: a match_any-aggregated variant measured slower (K2 stage 1 at world 8
      // 8.4 -> 21.5 us, profiles/r02/launches_shard_g8_m.csv)
      if (act) atomicAdd(&hist[bin], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      unsigned loc[8], tot = 0u;
#pragma unroll
      for (int b = 0; b < 8; ++b) { loc[b] = hist[lane * 8 + b]; tot += loc[b]; }
      unsigned incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned v = __shfl_up_sync(kFull, incl, o);
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
    __syncthreads();  // s_prefix / s_want / hist reused by the next digit
  }
  return prefix;
}

template <int MODE>
__global__ void __launch_bounds__(kSelThreads, 2) k_select(const float* __restrict__ dt, const float* __restrict__ gmin,
                                                        int L, int lo, int hi, int np, int world,
                                                        const float* __restrict__ qnorm, float cmax,
                                                        float e_dot, float e_abs, const float* __restrict__ qinv,
                                                        float c_inv, const float* __restrict__ x1_all,
                                                        float* __restrict__ x1, int32_t* __restrict__ cand,
                                                        int32_t* __restrict__ ncand, float* __restrict__ bound_out,
                                                        PeerOut pout, PeerIn pin) {
  pdl_entry();  // PDL: wait for the previous kernel in the stream, then let the next one launch
  extern __shared__ unsigned skeys[];  // >= max(keys of the theta' select, 2 kSelGather) words
  __shared__ unsigned s_cnt, s_ng, s_ovf;
  __shared__ int s_grp[kSelGroupCap];
  const int q = blockIdx.x;
  const int nq = gridDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int ngL = (L + 31) / 32;               // groups of all L centroids (gmin row stride)
  const int g0 = lo / 32, ng = hi > lo ? (hi + 31) / 32 - g0 : 0;  // this rank's groups
  // ---- theta': an upper bound of theta~ (the np-th smallest filter value)
  float theta = CUDART_INF_F;
  if constexpr (MODE == kSelStage2) {
    peer_wait(pin);  // NVLink peer exchange: every rank's x1 slab has landed in this rank's inbox
    const int n = world * np;  // <= kSelMaxGroups (checked at launch)
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int r = i / np, j = i - r * np;
      skeys[i] = fkey(x1_all[((size_t)r * nq + q) * np + j]);
    }
    __syncthreads();
    theta = fkey_inv(radix_select_kth(skeys, n, (unsigned)np));
  } else {
    if (ng >= np && ng <= kSelMaxGroups) {
      for (int i = threadIdx.x; i < ng; i += blockDim.x) skeys[i] = fkey(gmin[(size_t)q * ngL + g0 + i]);
      __syncthreads();
      theta = fkey_inv(radix_select_kth(skeys, ng, (unsigned)np));
    }
  }
  const float qn = qnorm[q];
  const float u = 5.9604645e-8f;  // 2^-24
  // fp16 subnormal flush of the scaled operands (absolute):
  // A = sqrt(d) 2^-25 (||q|| c_inv + c_max q_inv)(1 + 2^-11) + d 2^-50 c_inv q_inv,
  // e_abs = sqrt(d) 2^-25 (1 + 2^-11), d 2^-50 = e_abs^2 / (1 + 2^-11)^2 <= e_abs^2
  const float qi = qinv[q];
  const float abs_dot = e_abs * (qn * c_inv + cmax * qi) + e_abs * e_abs * (c_inv * qi) + 1.2e-38f;
  const float delta = 2.0f * (2.0f * (e_dot + 2.0f * u) * qn * cmax + 4.0f * u * (cmax * cmax + qn * qn) +
                              2.0f * abs_dot);
  // ---- gather every filter value <= lim of this range into shared memory, (key, centroid) pairs:
  // stage 1 gathers below theta' (the np smallest values of the range are among them), the others
  // below theta' + 2 Delta* (a superset of the candidate set). K1 stored gmin = the minimum of the
  // group's 32 stored values (+inf past L), so only groups with gmin <= lim are read (one 128-B piece).
  const float lim = MODE == kSelStage1 ? theta : theta + 2.0f * delta;
  unsigned* sk = skeys;                 // [kSelGather] keys
  unsigned* sid = skeys + kSelGather;   // [kSelGather] centroid ids
  __syncthreads();  // skeys (the theta' select) consumed
  if (threadIdx.x == 0) { s_cnt = 0u; s_ng = 0u; s_ovf = 0u; }
  __syncthreads();
  const float* grow = gmin + (size_t)q * ngL + g0;
  for (int i0 = 0; i0 < ng; i0 += blockDim.x) {
    const int i = i0 + threadIdx.x;
    const bool keep = i < ng && grow[i] <= lim;
    const unsigned km = __ballot_sync(kFull, keep);
    if (km == 0u) continue;
    unsigned base = 0u;
    if (lane == 0) base = atomicAdd(&s_ng, (unsigned)__popc(km));
    base = __shfl_sync(kFull, base, 0);
    const unsigned pos = base + __popc(km & ((1u << lane) - 1u));
    if (keep && pos < (unsigned)kSelGroupCap) s_grp[pos] = g0 + i;
  }
  __syncthreads();
  const unsigned ngq = s_ng;
  const float* row = dt + (size_t)q * L;
  if (ngq <= (unsigned)kSelGroupCap) {
    for (unsigned j = warp; j < ngq; j += nwarp) {  // warp-uniform: one 128-B piece per group
      const int l = s_grp[j] * 32 + lane;
      const float v = l < hi ? row[l] : CUDART_INF_F;
      const bool keep = v <= lim;
      const unsigned km = __ballot_sync(kFull, keep);
      if (km == 0u) continue;
      unsigned base = 0u;
      if (lane == 0) base = atomicAdd(&s_cnt, (unsigned)__popc(km));
      base = __shfl_sync(kFull, base, 0);
      const unsigned pos = base + __popc(km & ((1u << lane) - 1u));
      if (keep && pos < (unsigned)kSelGather) {
        sk[pos] = fkey(v);
        sid[pos] = (unsigned)l;
      }
    }
  } else if (threadIdx.x == 0) {
    s_ovf = 1u;
  }
  __syncthreads();
  const unsigned n_g = s_cnt;
  const bool ok = !s_ovf && n_g <= (unsigned)kSelGather;
  __syncthreads();  // every thread has read n_g / ok before s_cnt is reused below
  if constexpr (MODE == kSelStage1) {
    // x1 row: the np smallest filter values of this range as a multiset (exchanged; the union's np-th
    // smallest is the global theta~). P2P: straight into every rank's inbox.
    float* out = x1 + (size_t)q * np;
    const long long slab = (long long)nq * np;
    auto put = [&](int i, float v) {
      if (pout.G) peer_store(pout, slab, (long long)q * np + i, v);
      else out[i] = v;
    };
    if (ok) {
      if (n_g >= (unsigned)np) {
        const unsigned kth = radix_select_kth(sk, (int)n_g, (unsigned)np);
        if (threadIdx.x == 0) s_cnt = 0u;
        __syncthreads();
        for (unsigned i = threadIdx.x; i < n_g; i += blockDim.x)
          if (sk[i] < kth) put((int)atomicAdd(&s_cnt, 1u), fkey_inv(sk[i]));  // fewer than np are below
        __syncthreads();
        for (int i = (int)s_cnt + threadIdx.x; i < np; i += blockDim.x) put(i, fkey_inv(kth));
      } else {  // the whole range holds fewer than np values (theta' = +inf): all of them, +inf padding
        for (int i = threadIdx.x; i < np; i += blockDim.x) put(i, i < (int)n_g ? fkey_inv(sk[i]) : CUDART_INF_F);
      }
    } else {
      // too many values below theta' for the gather: the np smallest GROUP MINIMA (any np genuine filter
      // values give an np-th smallest >= theta~: a valid, looser bound), or every group minimum
      if (threadIdx.x == 0) s_cnt = 0u;
      __syncthreads();
      if (ng < np || ng > kSelMaxGroups) {
        for (int i = threadIdx.x; i < np; i += blockDim.x) put(i, i < ng ? grow[i] : CUDART_INF_F);
      } else {
        for (int i = threadIdx.x; i < ng; i += blockDim.x)
          if (grow[i] < theta) put((int)atomicAdd(&s_cnt, 1u), grow[i]);
        __syncthreads();
        for (int i = (int)s_cnt + threadIdx.x; i < np; i += blockDim.x) put(i, theta);
      }
    }
    peer_signal(pout);
    return;
  } else {
    // single GPU: tighten theta' to theta~ itself, the np-th smallest gathered value (every value below
    // theta' + 2 Delta* is in the gather, and theta~ <= theta'); stage 2 already holds the global theta~
    float th = theta;
    if constexpr (MODE == kSelFull) {
      if (ok && n_g >= (unsigned)np) th = fkey_inv(radix_select_kth(sk, (int)n_g, (unsigned)np));
    }
    const float bnd = th + 2.0f * delta;
    if (threadIdx.x == 0) {
      s_cnt = 0u;
      bound_out[q] = bnd;
    }
    __syncthreads();
    int32_t* out = cand + (size_t)q * kCandCap;
    auto emit = [&](bool keep, int i) {
      const unsigned km = __ballot_sync(kFull, keep);
      if (km == 0u) return;
      unsigned base = 0u;
      if (lane == 0) base = atomicAdd(&s_cnt, (unsigned)__popc(km));
      base = __shfl_sync(kFull, base, 0);
      if (keep) {
        const unsigned pos = base + __popc(km & ((1u << lane) - 1u));
        if (pos < (unsigned)kCandCap) out[pos] = i;
      }
    };
    if (ok) {
      const unsigned kb = fkey(bnd);
      for (unsigned i0 = 0; i0 < n_g; i0 += blockDim.x) {
        const unsigned i = i0 + threadIdx.x;
        emit(i < n_g && sk[i] <= kb, i < n_g ? (int)sid[i] : 0);
      }
    } else {
      const int n = hi - lo;
      if ((L & 3) == 0 && (lo & 3) == 0 && (n & 3) == 0) {
        const float4* r4 = reinterpret_cast<const float4*>(row + lo);
        constexpr int U = 2;  // loads in flight per thread before any emit
        for (int i0 = 0; i0 < n / 4; i0 += U * blockDim.x) {
          float4 v[U];
#pragma unroll
          for (int uu = 0; uu < U; ++uu) {
            const int i = i0 + uu * blockDim.x + threadIdx.x;
            v[uu] = i < n / 4 ? __ldg(r4 + i) : make_float4(CUDART_INF_F, CUDART_INF_F, CUDART_INF_F, CUDART_INF_F);
          }
#pragma unroll
          for (int uu = 0; uu < U; ++uu) {
            const int i = i0 + uu * blockDim.x + threadIdx.x;
            const bool in = i < n / 4;
            emit(in && v[uu].x <= bnd, lo + 4 * i);
            emit(in && v[uu].y <= bnd, lo + 4 * i + 1);
            emit(in && v[uu].z <= bnd, lo + 4 * i + 2);
            emit(in && v[uu].w <= bnd, lo + 4 * i + 3);
          }
        }
      } else {
        for (int i0 = 0; i0 < n; i0 += blockDim.x) {
          const int i = i0 + threadIdx.x;
          emit(i < n && row[lo + i] <= bnd, lo + i);
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) ncand[q] = (int32_t)s_cnt;
  }
}

// mode: kSelFull (single GPU / replicated coarse), kSelStage1 (-> ws.x1), kSelStage2 (ws.x1_all -> candidates)
cudaError_t launch_select(const DeviceIndex& ix, const Workspace& ws, int nq, int np, float e_dot, int mode,
                          cudaStream_t s, const PeerOut* po, const PeerIn* pi) {
  const PeerOut pout = po ? *po : PeerOut{};
  const PeerIn pin = pi ? *pi : PeerIn{};
  if (nq <= 0) return cudaSuccess;
  const int lo = mode == kSelFull ? 0 : ix.c_lo, hi = mode == kSelFull ? ix.nlist : ix.c_hi;
  const int ng = (hi + 31) / 32 - lo / 32;
  size_t n_keys = ng <= kSelMaxGroups ? (size_t)ng : 0;
  if (mode == kSelStage2) {
    n_keys = (size_t)ix.world * np;
    if (n_keys > (size_t)kSelMaxGroups) return cudaErrorInvalidValue;  // world * nprobe' <= 16384
  }
  const size_t sm = std::max(n_keys, (size_t)2 * kSelGather) * sizeof(unsigned);
  const void* fn = mode == kSelStage1 ? (const void*)k_select<kSelStage1>
                   : mode == kSelStage2 ? (const void*)k_select<kSelStage2> : (const void*)k_select<kSelFull>;
  cudaError_t e = ensure_smem(fn, sm);
  if (e != cudaSuccess) return e;
  const float e_abs = sqrtf((float)ix.d) * 2.9802322e-8f * 1.00049f * 1.0001f;  // sqrt(d) 2^-25 (1 + 2^-11), rounded up
#define VLR_SEL_ARGS ws.dt, ws.gmin, ix.nlist, lo, hi, np, ix.world, ws.qnorm, ix.cmax, e_dot, e_abs, ws.qinv, \
                     ix.c_inv, ws.x1_all, ws.x1, ws.cand, ws.ncand, ws.bound, pout, pin
  if (mode == kSelStage1) return launch_pdl(k_select<kSelStage1>, dim3(nq), dim3(kSelThreads), sm, s, VLR_SEL_ARGS);
  if (mode == kSelStage2) return launch_pdl(k_select<kSelStage2>, dim3(nq), dim3(kSelThreads), sm, s, VLR_SEL_ARGS);
  return launch_pdl(k_select<kSelFull>, dim3(nq), dim3(kSelThreads), sm, s, VLR_SEL_ARGS);
#undef VLR_SEL_ARGS
}

// ----------------------------------------------------------------- K3 refine
// One CTA (16 warps) per query. Candidate ids are gathered in chunks of up to
// kRefineChunk; a warp takes 32 candidates at a time (lane l <-> candidate l)
// and streams their centroid rows through shared memory in 32-dimension tiles
// (cp.async, double-buffered, 16-B chunks XOR-swizzled by row so the per-lane
// LDS.128 of a row is conflict-free). Each lane then runs its candidate's
// exact fp64 sum in dimension order; the chunk is merged with the running best
// nprobe' by a bitonic sort on (D, l).
constexpr int kRefineThreads = 512;
constexpr int kRefineWarps = kRefineThreads / 32;
constexpr int kRescanWarps = 8;  // warps computing exact distances on the (rare) overflow path
constexpr int kSortCap = 4096;  // max sort buffer: >= kMaxNprobe + kRefineChunk (power of two)
static_assert(kSortCap >= kMaxNprobe + kRefineChunk, "K3 sort buffer");
// the launch sizes the buffer to next_pow2(np + kRefineChunk) (2048 for
// np <= 1024: two K3b CTAs per SM stay resident)
static int sort_cap(int np) {
  int c = 1;
  while (c < np + kRefineChunk) c <<= 1;
  return c;
}
constexpr int kRefinePer = (kMaxNprobe + kRefineThreads - 1) / kRefineThreads;  // router items per thread
static_assert(kRescanWarps * 2048 * sizeof(float) >= kMaxNprobe * (sizeof(double) + sizeof(int)),
              "kRefMerge's rank-merge output lives in the rescan tiles");
constexpr int kRankSortMax = 512;  // K3b selects by rank (O(n^2 / threads)) up to this many candidates

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

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// exact D for 32 candidates of a warp (lane <-> rows[lane]); buf = S x 32 x 32
// floats. Tiles of 32 dimensions are streamed with cp.async S-1 tiles ahead;
// the 16-B chunks of row r are XOR-swizzled by (r & 7) so that lane r's
// LDS.128 of its own row are conflict-free.
// one dimension's term of the exact key, accumulated in t-order:
// L2 s += (q - c)^2 (dsub, dmul, dadd), IP s += q c (dmul exact for fp32 inputs)
template <int MET>
__device__ __forceinline__ double key_term(double s, double q, double c) {
  if constexpr (MET == 1) return __dadd_rn(s, __dmul_rn(q, c));
  const double e = __dsub_rn(q, c);
  return __dadd_rn(s, __dmul_rn(e, e));
}
template <int MET>
__device__ __forceinline__ double key_final(double s) { return MET == 1 ? -s : s; }

template <int S, int MET>
__device__ double warp_exact(const double* __restrict__ qs, const float* __restrict__ C, int d, int row_id,
                             float* buf, int lane) {
  double s = 0.0;
  const int ntile = d >> 5;  // full 32-dim tiles (d % 4 == 0 guaranteed by the caller for ntile > 0)
  // this lane copies 8 of the tile's 256 16-byte chunks: (row r, chunk k) for
  // idx = i*32 + lane; source pointers and swizzled destinations are fixed
  // for the whole task, only the tile offset moves
  const float* src[8];
  uint32_t dst[8];
  const uint32_t buf_s = (uint32_t)__cvta_generic_to_shared(buf);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int idx = i * 32 + lane;
    const int r = idx >> 3, k = idx & 7;
    src[i] = C + (size_t)__shfl_sync(kFull, row_id, r) * d + 4 * k;
    dst[i] = buf_s + (uint32_t)(r * 32 + ((k ^ (r & 7)) << 2)) * 4u;
  }
  auto issue = [&](int tile) {
    if (tile < ntile) {
      const uint32_t so = (uint32_t)(tile % S) * 4096u;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst[i] + so), "l"(src[i] + tile * 32)
                     : "memory");
    }
    cp_async_commit();  // (possibly empty) group keeps the wait count uniform
  };
#pragma unroll
  for (int t = 0; t < S - 1; ++t) issue(t);
  for (int tile = 0; tile < ntile; ++tile) {
    issue(tile + S - 1);
    cp_async_wait<S - 1>();
    __syncwarp();
    const float* rowp = buf + (tile % S) * 1024 + lane * 32;
    const double2* qt = reinterpret_cast<const double2*>(qs + tile * 32);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float4 v = *reinterpret_cast<const float4*>(rowp + ((k ^ (lane & 7)) << 2));
      const double2 qa = qt[2 * k], qb = qt[2 * k + 1];
      s = key_term<MET>(s, qa.x, (double)v.x);
      s = key_term<MET>(s, qa.y, (double)v.y);
      s = key_term<MET>(s, qb.x, (double)v.z);
      s = key_term<MET>(s, qb.y, (double)v.w);
    }
    __syncwarp();
  }
  cp_async_wait<0>();
  for (int t = ntile * 32; t < d; ++t)  // tail dimensions, still in order
    s = key_term<MET>(s, qs[t], (double)__ldg(C + (size_t)row_id * d + t));
  return key_final<MET>(s);
}

// Two candidates per lane (rows rid0, rid1: two independent in-order fp64
// chains interleaved, so each chain's 8-cycle DADD latency overlaps the other's
// work); 64 rows per tile (8 KB per stage). Same per-candidate arithmetic and
// order as warp_exact -> bit-identical D.
template <int S, int MET>
__device__ void warp_exact2(const double* __restrict__ qs, const float* __restrict__ C, int d, int rid0, int rid1,
                            float* buf, int lane, double& D0, double& D1) {
  double s0 = 0.0, s1 = 0.0;
  const int ntile = d >> 5;
  const float* src[16];
  uint32_t dst[16];
  const uint32_t buf_s = (uint32_t)__cvta_generic_to_shared(buf);
#pragma unroll
  for (int i = 0; i < 16; ++i) {  // (row r of 64, chunk k): rows 0-31 -> rid0 of lane r, 32-63 -> rid1
    const int idx = i * 32 + lane;
    const int r = idx >> 3, k = idx & 7;
    const int rr = r & 31;
    const int rid = __shfl_sync(kFull, r < 32 ? rid0 : rid1, rr);
    src[i] = C + (size_t)rid * d + 4 * k;
    dst[i] = buf_s + (uint32_t)(r * 32 + ((k ^ (r & 7)) << 2)) * 4u;
  }
  auto issue = [&](int tile) {
    if (tile < ntile) {
      const uint32_t so = (uint32_t)(tile % S) * 8192u;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst[i] + so), "l"(src[i] + tile * 32)
                     : "memory");
    }
    cp_async_commit();
  };
#pragma unroll
  for (int t = 0; t < S - 1; ++t) issue(t);
  for (int tile = 0; tile < ntile; ++tile) {
    issue(tile + S - 1);
    cp_async_wait<S - 1>();
    __syncwarp();
    const float* row0 = buf + (tile % S) * 2048 + lane * 32;
    const float* row1 = row0 + 32 * 32;
    const double2* qt = reinterpret_cast<const double2*>(qs + tile * 32);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float4 v = *reinterpret_cast<const float4*>(row0 + ((k ^ (lane & 7)) << 2));
      const float4 w = *reinterpret_cast<const float4*>(row1 + ((k ^ (lane & 7)) << 2));
      const double2 qa = qt[2 * k], qb = qt[2 * k + 1];
      s0 = key_term<MET>(s0, qa.x, (double)v.x);
      s1 = key_term<MET>(s1, qa.x, (double)w.x);
      s0 = key_term<MET>(s0, qa.y, (double)v.y);
      s1 = key_term<MET>(s1, qa.y, (double)w.y);
      s0 = key_term<MET>(s0, qb.x, (double)v.z);
      s1 = key_term<MET>(s1, qb.x, (double)w.z);
      s0 = key_term<MET>(s0, qb.y, (double)v.w);
      s1 = key_term<MET>(s1, qb.y, (double)w.w);
    }
    __syncwarp();
  }
  cp_async_wait<0>();
  for (int t = ntile * 32; t < d; ++t) {  // tail dimensions, still in order
    s0 = key_term<MET>(s0, qs[t], (double)__ldg(C + (size_t)rid0 * d + t));
    s1 = key_term<MET>(s1, qs[t], (double)__ldg(C + (size_t)rid1 * d + t));
  }
  D0 = key_final<MET>(s0);
  D1 = key_final<MET>(s1);
}

template <int MET>
__device__ __forceinline__ double scalar_exact(const double* __restrict__ qs, const float* __restrict__ C, int d,
                                               int row_id) {
  double s = 0.0;
  for (int t = 0; t < d; ++t) s = key_term<MET>(s, qs[t], (double)__ldg(C + (size_t)row_id * d + t));
  return key_final<MET>(s);
}

// K3a: exact fp64 D of every listed candidate, 4 warps per CTA, warp <-> 32
// candidates of one query; grid (nq, kCandCap / 128). CTAs past the query's
// candidate count (or queries whose list overflowed) exit at once.
// product configuration (S, W) = (3, 4): 56 KB of shared memory per CTA -> 4 CTAs/SM, so the ~512
// non-empty CTAs of a 256-query C4 batch run in one round (S = 4: 72 KB, 3 CTAs/SM, two rounds).
// Measured K3a+K3b at C4 (tools/k3a_sweep.sh, profiles/k3a_sweep_r01.txt): (4,4) 0.087-0.088 ms,
// (3,4) 0.070, (2,4) 0.071, (2,8) 0.075, (2,2) 0.073, (4,2) 0.093. VLR_EXACT_CFG=S,W selects another.
constexpr int kExactWarps = 4;
constexpr int kExactStages = 3;

template <int MET, int S, int W, int CH = 1>
__global__ void __launch_bounds__(W * 32) k_exact(const float* __restrict__ Q, const float* __restrict__ C,
                                                  int d, int nq, int ny, const int32_t* __restrict__ cand,
                                                  const int32_t* __restrict__ ncand,
                                                  double* __restrict__ exact) {
  pdl_entry();  // PDL: wait for the previous kernel in the stream, then let the next one launch
  extern __shared__ __align__(16) unsigned char sm[];
  double* qs = reinterpret_cast<double*>(sm);
  float* tiles = reinterpret_cast<float*>(qs + ((d + 1) & ~1));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // persistent over tasks (q, y) = candidate block y of query q, y-major (every query's first block
  // first): a task past the query's candidate count costs one L2 read here instead of a CTA launch
  // (the grid of empty CTAs dominated at world 8, where a rank holds ~20 candidates per query)
  for (int t = blockIdx.x; t < nq * ny; t += gridDim.x) {
    const int q = t % nq, y = t / nq;
    const int nc = ncand[q];
    const int g0 = y * W * 32 * CH;
    if (nc > kCandCap || g0 >= nc) continue;  // CTA-uniform
    __syncthreads();  // qs of the previous task consumed
    for (int i = threadIdx.x; i < d; i += blockDim.x) qs[i] = (double)Q[(size_t)q * d + i];
    __syncthreads();
    const int32_t* lst = cand + (size_t)q * kCandCap;
    // groups of 32 CH candidates: this warp takes g = g0 + 32 CH warp + stride i
    const int stride = ny * W * 32 * CH;
    for (int g = g0 + warp * 32 * CH; g < nc; g += stride) {
      const int j = g + lane;
      const int rid = lst[j < nc ? j : g];
      if constexpr (CH == 2) {
        if ((d & 3) == 0 && g + 32 < nc) {  // a second chain with at least one real candidate
          const int j1 = j + 32;
          const int rid1 = lst[j1 < nc ? j1 : g];
          double D0, D1;
          warp_exact2<S, MET>(qs, C, d, rid, rid1, tiles + warp * (S * 2048), lane, D0, D1);
          if (j < nc) exact[(size_t)q * kCandCap + j] = D0;
          if (j1 < nc) exact[(size_t)q * kCandCap + j1] = D1;
          continue;
        }
      }
      double D;
      if ((d & 3) == 0)
        D = warp_exact<S, MET>(qs, C, d, rid, tiles + warp * (S * 1024 * CH), lane);
      else
        D = scalar_exact<MET>(qs, C, d, rid);
      if (j < nc) exact[(size_t)q * kCandCap + j] = D;
    }
  }
}

template <int S, int W, int CH = 1>
static cudaError_t launch_exact_t(const float* Q, const DeviceIndex& ix, const Workspace& ws, int nq, cudaStream_t s) {
  const size_t sm = (size_t)((ix.d + 1) & ~1) * sizeof(double) + (size_t)W * S * 1024 * CH * sizeof(float);
  auto fn = ix.metric == 1 ? k_exact<1, S, W, CH> : k_exact<0, S, W, CH>;
  cudaError_t e = ensure_smem((const void*)fn, sm);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, W * 32, sm)) != cudaSuccess) return e;
  const int ny = 1024 / (W * 32 * CH);  // 1024 candidates per pass over a query's list; more loop
  const int tasks = nq * ny;
  const int grid = std::max(1, std::min(tasks, sms * std::max(per_sm, 1)));
  return launch_pdl(fn, dim3(grid), dim3(W * 32), sm, s, Q, (const float*)ix.centroids, ix.d, nq, ny,
                    (const int32_t*)ws.cand, (const int32_t*)ws.ncand, ws.exact);
}

cudaError_t launch_exact(const float* Q, const DeviceIndex& ix, const Workspace& ws, int nq, cudaStream_t s) {
  if (nq <= 0) return cudaSuccess;
  // VLR_EXACT_CFG="S,W[,CH]" (stages, warps, chains per lane) overrides the product choice (3, 4, 1)
  // (profiles/k3a_sweep_r01.txt). The sharded coarse stage uses it too: a rank's candidates are not ~1/G of
  // every query's but concentrate on the queries whose neighbourhood lies in its centroid range (ids are
  // not random), so one warp per query (the former (16, 1) latency choice) serialised up to ~5 passes
  static int env_s = -1, env_w = 0, env_c = 1;
  if (env_s < 0) {
    env_s = 0;
    const char* e = getenv("VLR_EXACT_CFG");
    if (e && e[0]) {
      int s_ = 0, w_ = 0, c_ = 1;
      const int n = sscanf(e, "%d,%d,%d", &s_, &w_, &c_);
      if (n >= 2) { env_s = s_; env_w = w_; env_c = n >= 3 ? c_ : 1; }
    }
  }
  int S = 3, W = 4, CH = 1;
  if (env_s > 0) { S = env_s; W = env_w; CH = env_c; }
  const int cfg = S * 100 + W * 10 + CH;
  switch (cfg) {
    case 241: return launch_exact_t<2, 4>(Q, ix, ws, nq, s);
    case 441: return launch_exact_t<4, 4>(Q, ix, ws, nq, s);
    case 281: return launch_exact_t<2, 8>(Q, ix, ws, nq, s);
    case 221: return launch_exact_t<2, 2>(Q, ix, ws, nq, s);
    case 421: return launch_exact_t<4, 2>(Q, ix, ws, nq, s);
    case 322: return launch_exact_t<3, 2, 2>(Q, ix, ws, nq, s);
    case 342: return launch_exact_t<3, 4, 2>(Q, ix, ws, nq, s);
    case 522: return launch_exact_t<5, 2, 2>(Q, ix, ws, nq, s);
    case 1611: return launch_exact_t<16, 1>(Q, ix, ws, nq, s);
    case 3211: return launch_exact_t<32, 1>(Q, ix, ws, nq, s);
    case 821: return launch_exact_t<8, 2>(Q, ix, ws, nq, s);
    default: return launch_exact_t<kExactStages, kExactWarps>(Q, ix, ws, nq, s);
  }
}

// K3b modes: kRefRoute (single GPU: sort the candidates, keep nprobe', route),
// kRefLocal (sharded coarse stage 2: this rank's candidates -> its sorted top
// nprobe' exact (D, l) list x2[q], no routing), kRefMerge (sharded stage 3:
// the G sorted lists gathered from every rank, x2_all [G][nq][np] -> the
// global top nprobe', then the router). kRefMerge sorts exactly the multiset
// kRefRoute would (the global top nprobe' of the union of the ranks'
// candidate sets is contained in the union of their local top nprobe'), so the
// probes are bitwise those of the single-GPU path.

template <int MET, int MODE>
__global__ void __launch_bounds__(kRefineThreads) k_refine(const float* __restrict__ Q, const float* __restrict__ C,
                                                           int d, int L, int lo, int hi, int np, int scap,
                                                           int by_residual, int world,
                                                           const float* __restrict__ qsq, const float* __restrict__ dt,
                                                           const int32_t* __restrict__ cand,
                                                           const int32_t* __restrict__ ncand,
                                                           const float* __restrict__ bound,
                                                           const double* __restrict__ exact,
                                                           CoarseEntry* __restrict__ x2,
                                                           const CoarseEntry* __restrict__ x2_all,
                                                           int32_t* __restrict__ probes, float* __restrict__ term1,
                                                           int rank, const int32_t* __restrict__ owner,
                                                           const int32_t* __restrict__ local,
                                                           const int64_t* __restrict__ gbase, uint8_t* __restrict__ miss,
                                                           int32_t* __restrict__ probes_out,
                                                           int32_t* __restrict__ plocal,
                                                           int64_t* __restrict__ item_local,
                                                           int64_t* __restrict__ qtot, PeerOut pout, PeerIn pin) {
  pdl_entry();  // PDL: wait for the previous kernel in the stream, then let the next one launch
  extern __shared__ __align__(16) unsigned char sm[];
  float* tiles = reinterpret_cast<float*>(sm);                        // [kRescanWarps][2][32][32]
  double* key = reinterpret_cast<double*>(tiles + kRescanWarps * 2048);  // [scap]
  int* id = reinterpret_cast<int*>(key + scap);                       // [scap]
  int* lbuf = id + scap;                                              // [kRefineChunk]
  double* qs = reinterpret_cast<double*>(lbuf + kRefineChunk);        // [d]
  __shared__ int s_cnt;
  const int q = blockIdx.x;
  const int nq = gridDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int nbest = 0;
  if constexpr (MODE == kRefMerge) {
    peer_wait(pin);  // NVLink peer exchange: every rank's x2 slab has landed in this rank's inbox
    // G sorted lists of np entries; padding (+inf, -1) is skipped
    const int src_len = world * np;
    if (src_len <= scap) {
      // merge by rank (one pass, no sort): every list is sorted by (D, l) and the ids are distinct across
      // lists (disjoint centroid ranges), so an entry's position in the union is its index in its own list
      // plus, for every other list, the number of its entries that precede it (binary search in shared
      // memory). Entries of position < np are the global top np, in order -- the same unique sequence the
      // bitonic path produces. Padding is staged as (+inf, INT_MAX): after every real entry.
      for (int i = threadIdx.x; i < src_len; i += blockDim.x) {
        const int r = i / np, j = i - r * np;
        const CoarseEntry e = x2_all[((size_t)r * nq + q) * np + j];
        key[i] = e.l >= 0 ? e.D : CUDART_INF;
        id[i] = e.l >= 0 ? e.l : 0x7fffffff;
      }
      if (threadIdx.x == 0) s_cnt = 0;
      __syncthreads();
      double* okey = reinterpret_cast<double*>(tiles);  // [np] (the rescan tiles are unused in this mode)
      int* oid = reinterpret_cast<int*>(okey + np);      // [np]
      for (int i = threadIdx.x; i < src_len; i += blockDim.x) {
        const int r = i / np, j = i - r * np;
        const double D = key[i];
        const int l = id[i];
        if (l == 0x7fffffff) continue;
        atomicAdd(&s_cnt, 1);
        int rk = j;
        for (int r2 = 0; r2 < world && rk < np; ++r2) {
          if (r2 == r) continue;
          const double* k2 = key + r2 * np;
          const int* i2 = id + r2 * np;
          int lo2 = 0, hi2 = np;
          while (lo2 < hi2) {
            const int m = (lo2 + hi2) >> 1;
            if (key_less(k2[m], i2[m], D, l)) lo2 = m + 1;
            else hi2 = m;
          }
          rk += lo2;
        }
        if (rk < np) {
          okey[rk] = D;
          oid[rk] = l;
        }
      }
      __syncthreads();
      nbest = min(np, s_cnt);
      for (int p = threadIdx.x; p < nbest; p += blockDim.x) {
        key[p] = okey[p];
        id[p] = oid[p];
      }
      __syncthreads();
    }
    for (int pos = 0; src_len > scap && pos < src_len; pos += kRefineChunk) {
      if (threadIdx.x == 0) s_cnt = 0;
      __syncthreads();
      const int take = min(kRefineChunk, src_len - pos);
      for (int i = threadIdx.x; i < take; i += blockDim.x) {
        const int r = (pos + i) / np, j = (pos + i) - r * np;
        const CoarseEntry e = x2_all[((size_t)r * nq + q) * np + j];
        if (e.l >= 0) {
          const int at = nbest + atomicAdd(&s_cnt, 1);
          key[at] = e.D;
          id[at] = e.l;
        }
      }
      __syncthreads();
      const int tot = nbest + s_cnt;
      int n2 = 1;
      while (n2 < tot) n2 <<= 1;
      for (int j = tot + threadIdx.x; j < n2; j += blockDim.x) {
        key[j] = DBL_MAX;
        id[j] = 0x7fffffff;
      }
      bitonic_sort(key, id, n2);
      nbest = min(np, tot);
    }
  } else {
    const int nc = ncand[q];
    const bool listed = nc <= kCandCap;
    if (!listed)  // the query (fp64) is needed only by the rescan path, which computes exact keys here
      for (int t = threadIdx.x; t < d; t += blockDim.x) qs[t] = (double)Q[(size_t)q * d + t];
    const int src_len = listed ? nc : hi - lo;
    const float bnd = bound[q];
    const int32_t* lst = cand + (size_t)q * kCandCap;
    const float* row = dt + (size_t)q * L + lo;  // rescan of this rank's filter columns [lo, hi)
    const bool vec_ok = (d & 3) == 0;
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
          // uniform snapshot of the count: every thread reads it between two barriers, before any thread
          // of this iteration adds to it (a read racing with other warps' atomicAdd could make some
          // threads break and others loop on: barrier divergence)
          __syncthreads();
          const int cnt_now = s_cnt;
          __syncthreads();
          if (cnt_now + (int)blockDim.x > kRefineChunk) break;
          const int i = pos + threadIdx.x;
          if (i < src_len && row[i] <= bnd) lbuf[atomicAdd(&s_cnt, 1)] = lo + i;
          pos += blockDim.x;
        }
      }
      __syncthreads();
      const int cnt = s_cnt;
      // exact distances: precomputed by K3a for listed candidates; the overflow
      // (rescan) path computes them here, 32 candidates per warp pass
      if (listed) {
        const double* ex = exact + (size_t)q * kCandCap + (pos - cnt);
        for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
          key[nbest + j] = ex[j];
          id[nbest + j] = lbuf[j];
        }
      } else {
        for (int g = warp * 32; warp < kRescanWarps && g < cnt; g += kRescanWarps * 32) {
          const int j = g + lane;
          const int rid = j < cnt ? lbuf[j] : lbuf[g];
          const double dsum = vec_ok ? warp_exact<2, MET>(qs, C, d, rid, tiles + warp * 2048, lane)
                                     : scalar_exact<MET>(qs, C, d, rid);
          if (j < cnt) {
            key[nbest + j] = dsum;
            id[nbest + j] = rid;
          }
        }
      }
      const int tot = nbest + cnt;
      if (listed && nbest == 0 && pos >= src_len && tot <= kRankSortMax) {
        // the whole (short) candidate list at once: select the np best by rank (each entry counts the
        // entries before it in (D, l) order; ids are distinct, so ranks are distinct) instead of a bitonic
        // sort -- no barrier per stage. Same unique order.
        __syncthreads();
        double* okey = reinterpret_cast<double*>(tiles);  // [np] (the rescan tiles are unused when listed)
        int* oid = reinterpret_cast<int*>(okey + np);
        for (int i = threadIdx.x; i < tot; i += blockDim.x) {
          const double D = key[i];
          const int l = id[i];
          int rk = 0;
          for (int j = 0; j < tot; ++j) rk += key_less(key[j], id[j], D, l) ? 1 : 0;
          if (rk < np) {
            okey[rk] = D;
            oid[rk] = l;
          }
        }
        __syncthreads();
        nbest = min(np, tot);
        for (int p = threadIdx.x; p < nbest; p += blockDim.x) {
          key[p] = okey[p];
          id[p] = oid[p];
        }
        __syncthreads();
        break;
      }
      int n2 = 1;
      while (n2 < tot) n2 <<= 1;
      for (int j = tot + threadIdx.x; j < n2; j += blockDim.x) {
        key[j] = DBL_MAX;
        id[j] = 0x7fffffff;
      }
      bitonic_sort(key, id, n2);
      nbest = min(np, tot);
    }
  }
  if constexpr (MODE == kRefLocal) {
    // this rank's sorted top-np exact list, padded with (+inf, -1)
    for (int p = threadIdx.x; p < np; p += blockDim.x) {
      CoarseEntry e;
      e.D = p < nbest ? key[p] : CUDART_INF;
      e.l = p < nbest ? id[p] : -1;
      e.pad = 0;
      if (pout.G) peer_store(pout, (long long)nq * np, (long long)q * np + p, e);
      else x2[(size_t)q * np + p] = e;
    }
    peer_signal(pout);
    return;
  } else {
    // ---- router epilogue (K4 fused): mask, owned work items
    // and their within-query prefix (groups of 32 vectors); K4b adds the
    // query bases. Items p of this query are handled kRefinePer per thread in order.
    __shared__ long long s_wsum[kRefineWarps];
    long long g2[kRefinePer];
    const int p0 = kRefinePer * threadIdx.x;
    // term1: the key itself with residual codes (||q-c||^2
    // or -<q,c>); without, ||q||^2 (L2) or 0 (IP)
    const float t1c = by_residual ? 0.f : (MET == 1 ? 0.f : qsq[q]);
#pragma unroll
    for (int h = 0; h < kRefinePer; ++h) {
      const int p = p0 + h;
      g2[h] = 0;
      if (p < np) {
        // nbest == np whenever the candidate set holds >= np clusters (always: the
        // band contains the np smallest)
        const int l = p < nbest ? id[p] : -1;
        const size_t o = (size_t)q * np + p;
        probes[o] = l;
        term1[o] = p < nbest ? (by_residual ? __double2float_rn(key[p]) : t1c) : CUDART_INF_F;
        const int own = l >= 0 ? owner[l] : -1;
        miss[o] = own < 0 ? 1 : 0;
        if (probes_out) probes_out[o] = l;
        const int loc = (own == rank) ? local[l] : -1;
        plocal[o] = loc;
        if (loc >= 0) g2[h] = gbase[loc + 1] - gbase[loc];
      }
    }
    long long mine = 0;
#pragma unroll
    for (int h = 0; h < kRefinePer; ++h) mine += g2[h];
    long long incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long v = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    long long wbase = 0, total = 0;
    for (int w = 0; w < kRefineWarps; ++w) {
      const long long v = s_wsum[w];
      if (w < warp) wbase += v;
      total += v;
    }
    long long ex = wbase + incl - mine;
#pragma unroll
    for (int h = 0; h < kRefinePer; ++h) {
      if (p0 + h < np) item_local[(size_t)q * np + p0 + h] = ex;
      ex += g2[h];
    }
    if (threadIdx.x == 0) qtot[q] = total;
  }
}

size_t refine_smem(int d, int scap) {
  return (size_t)kRescanWarps * 2048 * sizeof(float) + (size_t)scap * (sizeof(double) + sizeof(int)) +
         kRefineChunk * sizeof(int) + (size_t)d * sizeof(double);
}

template <int MET>
static const void* refine_fn(int mode) {
  return mode == kRefLocal ? (const void*)k_refine<MET, kRefLocal>
         : mode == kRefMerge ? (const void*)k_refine<MET, kRefMerge> : (const void*)k_refine<MET, kRefRoute>;
}

// mode kRefRoute / kRefLocal (-> ws.x2) / kRefMerge (ws.x2_all -> probes, route)
cudaError_t launch_refine(const float* Q, const DeviceIndex& ix, const Workspace& ws, int nq, int np, uint8_t* miss,
                          int32_t* probes_out, int mode, cudaStream_t s, const PeerOut* po, const PeerIn* pi) {
  if (nq <= 0) return cudaSuccess;
  const PeerOut pout = po ? *po : PeerOut{};
  const PeerIn pin = pi ? *pi : PeerIn{};
  // kRefMerge sorts chunks of up to kRefineChunk entries with the running np best, as the other modes
  const int scap = sort_cap(np);
  const size_t sm = refine_smem(ix.d, scap);
  const void* fn = ix.metric == 1 ? refine_fn<1>(mode) : refine_fn<0>(mode);
  cudaError_t e = ensure_smem(fn, sm);
  if (e != cudaSuccess) return e;
  const int lo = mode == kRefRoute ? 0 : ix.c_lo, hi = mode == kRefRoute ? ix.nlist : ix.c_hi;
  void* args[] = {(void*)&Q, (void*)&ix.centroids, (void*)&ix.d, (void*)&ix.nlist, (void*)&lo, (void*)&hi,
                  (void*)&np, (void*)&scap, (void*)&ix.by_residual, (void*)&ix.world, (void*)&ws.qsq,
                  (void*)&ws.dt, (void*)&ws.cand, (void*)&ws.ncand, (void*)&ws.bound, (void*)&ws.exact,
                  (void*)&ws.x2, (void*)&ws.x2_all, (void*)&ws.probes, (void*)&ws.term1, (void*)&ix.rank,
                  (void*)&ix.owner, (void*)&ix.local, (void*)&ix.gbase, (void*)&miss, (void*)&probes_out,
                  (void*)&ws.plocal, (void*)&ws.item_local, (void*)&ws.qtot, (void*)&pout, (void*)&pin};
  return launch_pdl_c(fn, dim3(nq), dim3(kRefineThreads), sm, s, args);
}

}  // namespace vlr

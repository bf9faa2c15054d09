// k_filter_tc.cu -- K1 coarse filter on the 5th-gen tensor cores (tcgen05).
//
// dt[q][l] = ||c_l||^2 - 2 <q~, c~_l>   (the coarse-quantizer contraction,
// stage 1 of Fig. 2; ||q||^2 is constant per query)
// with q~ = fp16(q 2^e_q) 2^-e_q and c~ = fp16(c 2^e_c) 2^-e_c: operands
// scaled by powers of two (max |x 2^e| < 2^14, so no fp16 overflow) and
// rounded to fp16 (RN, 11-bit significand: the same relative precision as
// TF32 at half the bytes and twice the MMA rate); products exact, fp32
// accumulation in TMEM; the epilogue multiplies by 2^-(e_q + e_c) exactly.
//
// Swap-AB: A = a 128-centroid tile (M = 128, K-major rows of the centroid
// matrix), B = the query batch (N = up to 256 per accumulator, two
// accumulators for up to 512 queries), so a small batch still fills the
// 128-row MMA. Warp roles (192 threads): warp 0 = TMA producer (one elected
// lane: cp.async.bulk.tensor 2D, SWIZZLE_128B, mbarrier complete_tx),
// warp 1 = TMEM allocator + MMA issuer (one lane: tcgen05.mma.kind::f16,
// tcgen05.commit -> mbarriers), warps 2-5 = epilogue (tcgen05.ld 32x32b,
// thread i <-> TMEM lane i <-> centroid m0+i; coalesced stores of dt).
// The error of dt w.r.t. the exact D - ||q||^2 is bounded in DESIGN.md §5
// (band proof); K2/K3 make the probes exact.
#include <cuda.h>
#include <cuda_fp16.h>

#include "vlr_device.cuh"
#include "vlr_internal.cuh"

namespace vlr {

constexpr int kTcM = 128;        // centroids per tile (MMA M)
constexpr int kTcBK = 64;        // fp16 elements per K block (128 B = one SW128 row)
constexpr int kTcThreads = 192;  // 6 warps
constexpr int kTcMaxStages = 6;
#ifndef VLR_K1_EXPERIMENT
#define VLR_K1_EXPERIMENT 0  // timing-only builds (tools/variants.py): 1 no dt stores, 2 no MMAs, 3 no epilogue
#endif
constexpr int kTcCluster = 1;    // default B-multicast cluster size (launch_filter_tc): 1 = off. Measured at
                                 // C4, batch 256: 0.060 ms (1), 0.066 (2), 0.067 (4) -- the filter is not
                                 // bound by the re-read query tile (profiles/k1_persistent_r01.md)

__device__ __forceinline__ uint32_t s32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(b)), "r"(n));
}
__device__ __forceinline__ void mb_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mb_try(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred P1;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n}\n"
      : "=r"(ok)
      : "r"(s32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
// bounded wait: a pipeline bug traps (CUDA error) instead of hanging the GPU
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
  const unsigned long long t0 = globaltimer_ns();
  for (uint32_t i = 0; !mb_try(b, parity); ++i)
    if ((i & 1023u) == 1023u && globaltimer_ns() - t0 > 4000000000ull) asm volatile("trap;");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          s32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(s32(bar))
      : "memory");
}
// B-operand multicast across a cluster of CL CTAs (adjacent centroid tiles):
// CTA r loads rows [r nN/CL, (r+1) nN/CL) of the query tile and the TMA
// writes them into the same smem offset of every CTA in ctaMask, completing
// bytes on each destination's mbarrier at the same offset.
__device__ __forceinline__ void tma_2d_mc(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                          uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(s32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(s32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_16k(void* dst, const void* src, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];" ::"r"(
                   s32(dst)),
               "l"(src), "r"(s32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   s32(dst)),
               "l"(src), "r"(bytes), "r"(s32(bar))
               : "memory");
}
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          s32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  __syncwarp();  // .aligned: the whole warp executes the cluster barrier together
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  // UMMA shared-memory descriptor, K-major SWIZZLE_128B: start>>4, LBO = 1 (unused),
  // SBO = 1024 B (8 rows x 128 B), version 1 (bits 46-47), layout type 2 (bits 61-63)
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void mma_f16(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(bar))
               : "memory");
}

#ifdef VLR_K1_TRACE
__device__ unsigned long long g_k1_trace[4096][6];  // per CTA: start, setup done, first stage full, tfull, end, smid
#endif
template <int CL>
__global__ void __launch_bounds__(kTcThreads, 1)
    k_filter_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int L, int nq,
                int kblocks, int nN, int nacc, int stages, const float* __restrict__ cn2,
                const float* __restrict__ qinv, float c_inv, float* __restrict__ dt, float* __restrict__ gmin,
                int ngroups, const uint16_t* __restrict__ At, int t0, const uint16_t* __restrict__ Bt) {
  pdl_entry();  // PDL: wait for the previous kernel in the stream, then let the next one launch
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[kTcMaxStages], empty[kTcMaxStages], tfull;
  __shared__ uint32_t tmem_base;
  __shared__ float s_inv[512];  // per query column: 2^-(e_q + e_c)
#ifdef VLR_K1_TRACE
  const unsigned long long tr0 = globaltimer_ns();
#endif
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = t0 + (int)blockIdx.x;  // centroid tile (this rank's range starts at tile t0)
  const int m0 = tile * kTcM;
  const int q0 = blockIdx.y * (nN * nacc);
  const uint32_t bytesA = kTcM * 128, bytesB = (uint32_t)(nacc * nN * 128);
  const uint32_t stage_bytes = bytesA + bytesB;
  const int ncols_used = nN * nacc;
  uint32_t ncols = 32;
  while ((int)ncols < ncols_used) ncols <<= 1;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      mb_init(&full[s], 1);
      mb_init(&empty[s], CL);  // CL > 1: every cluster CTA's MMAs must have read the stage (B is multicast)
    }
    mb_init(&tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(&tmem_base)), "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if constexpr (CL > 1) cluster_sync_all();  // peers' barriers initialised before any multicast lands
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = tmem_base;
  const uint32_t crank = CL > 1 ? cluster_rank() : 0u;
#ifdef VLR_K1_TRACE
  const int trc = blockIdx.x + blockIdx.y * gridDim.x;
  if (threadIdx.x == 0 && trc < 4096) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_k1_trace[trc][0] = tr0;
    g_k1_trace[trc][1] = globaltimer_ns();
    g_k1_trace[trc][5] = smid;
  }
#endif
  constexpr uint16_t kMask = (uint16_t)((1u << CL) - 1u);

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < kblocks; ++kb) {
        const int s = kb % stages;
        const uint32_t ph = (uint32_t)(kb / stages) & 1u;
        mb_wait(&empty[s], ph ^ 1u);
        uint8_t* sA = smem + (size_t)s * stage_bytes;
        uint8_t* sB = sA + bytesA;
        mb_expect_tx(&full[s], stage_bytes);
        if (At) bulk_g2s_16k(sA, At + ((size_t)tile * kblocks + kb) * (kTcM * kTcBK), &full[s]);
        else tma_2d(sA, &tmA, kb * kTcBK, m0, &full[s]);
        if constexpr (CL > 1) {  // nacc == 1: this CTA's 1/CL of the query rows, to every cluster CTA
          const int rq = nN / CL;
          tma_2d_mc(sB + (size_t)crank * rq * 128, &tmB, kb * kTcBK, q0 + (int)crank * rq, &full[s], kMask);
        } else if (Bt) {  // pre-tiled query operand (k_qprep): the stage's whole B tile in one bulk copy
          bulk_g2s(sB, Bt + ((size_t)blockIdx.y * kblocks + kb) * (size_t)(nacc * nN) * kTcBK, bytesB, &full[s]);
        } else {
          for (int r = 0; r < nacc * nN; r += 256) {
            tma_2d(sB + (size_t)r * 128, &tmB, kb * kTcBK, q0 + r, &full[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // instruction descriptor: F32 accum, A/B F16, K-major, N, M = 128
      const uint32_t idesc = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(nN >> 3) << 17) | ((uint32_t)(kTcM >> 4) << 24);
      for (int kb = 0; kb < kblocks; ++kb) {
        const int s = kb % stages;
        const uint32_t ph = (uint32_t)(kb / stages) & 1u;
        mb_wait(&full[s], ph);
#ifdef VLR_K1_TRACE
        if (kb == 0 && trc < 4096) g_k1_trace[trc][2] = globaltimer_ns();
#endif
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t aaddr = s32(smem + (size_t)s * stage_bytes);
        const uint32_t baddr = aaddr + bytesA;
#pragma unroll
        for (int kk = 0; kk < kTcBK / 16; ++kk) {  // K = 16 fp16 (32 B) per MMA
          const uint64_t ad = sw128_desc(aaddr + kk * 32);
          for (int acc = 0; acc < nacc; ++acc) {
            const uint64_t bd = sw128_desc(baddr + (uint32_t)(acc * nN * 128) + kk * 32);
            if (VLR_K1_EXPERIMENT != 2) mma_f16(tbase + (uint32_t)(acc * nN), ad, bd, idesc, (kb | kk) != 0 ? 1u : 0u);
          }
        }
        if constexpr (CL > 1) mma_commit_mc(&empty[s], kMask);  // frees stage s in every cluster CTA's count
        else mma_commit(&empty[s]);  // frees the smem stage once these MMAs have read it
      }
      mma_commit(&tfull);  // accumulator complete
    }
    __syncwarp();
  } else {
    // epilogue: warps 2..5 -> TMEM lane groups (warp % 4)
    const int lg = warp & 3;
    const int row = m0 + lg * 32 + lane;
    const float cn = row < L ? cn2[row] : 0.f;
    for (int j = threadIdx.x - 64; j < ncols_used; j += 128) {
      const int q = q0 + j;
      s_inv[j] = q < nq ? qinv[q] * c_inv : 0.f;  // product of powers of two >= 2^-120: exact
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");  // epilogue warps only
    mb_wait(&tfull, 0);
#ifdef VLR_K1_TRACE
    if (threadIdx.x == 64 && trc < 4096) g_k1_trace[trc][3] = globaltimer_ns();
#endif
    asm volatile("tcgen05.fence::after_thread_sync;");
    // 32 query columns at a time: dt stores (lanes = 32 consecutive centroids,
    // coalesced) and the min over this warp's 32 centroids of each column
    // (transpose-reduce: 31 shuffles leave column j's min in lane j).
    const int grp = tile * 4 + lg;
    for (int c = 0; c < (VLR_K1_EXPERIMENT == 3 ? 0 : ncols_used); c += 32) {
      uint32_t v[32];
      const uint32_t taddr = tbase + ((uint32_t)(lg * 32) << 16) + (uint32_t)c;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(taddr));
      if (c + 16 < ncols_used) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
              "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
              "=r"(v[30]), "=r"(v[31])
            : "r"(taddr + 16u));
      } else {
#pragma unroll
        for (int j = 16; j < 32; ++j) v[j] = __float_as_uint(CUDART_INF_F);
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      float f[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        f[j] = row < L ? cn - 2.f * (__uint_as_float(v[j]) * s_inv[c + j]) : CUDART_INF_F;
        const int q = q0 + c + j;
        if (VLR_K1_EXPERIMENT != 1 && row < L && q < nq && c + j < ncols_used) dt[(size_t)q * L + row] = f[j];
      }
#pragma unroll
      for (int w = 16; w >= 1; w >>= 1) {
        const bool upper = (lane & w) != 0;
#pragma unroll
        for (int j = 0; j < w; ++j) {
          const float send = upper ? f[j] : f[j + w];
          const float keep = upper ? f[j + w] : f[j];
          f[j] = fminf(keep, __shfl_xor_sync(kFull, send, w));
        }
      }
      const int q = q0 + c + lane;
      if (q < nq && c + lane < ncols_used && grp < ngroups) gmin[(size_t)q * ngroups + grp] = f[0];
    }
  }
#ifdef VLR_K1_TRACE
  if (threadIdx.x == 64 && trc < 4096) g_k1_trace[trc][4] = globaltimer_ns();
#endif
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if constexpr (CL > 1) cluster_sync_all();  // no CTA leaves while peers may still multicast into it
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(ncols));
  }
}

// Persistent variant for nq <= 256 (one accumulator of nN <= 256 columns per
// tile): one CTA per SM loops over the 128-centroid tiles t = blockIdx.x,
// t += gridDim.x, with a DOUBLE-BUFFERED TMEM accumulator (2 x nN <= 512
// columns) so the epilogue of tile i (warps 2-5) overlaps the TMA/MMA
// mainloop of tile i+1, and the smem ring (up to 4 stages of 48 KB at nN =
// 256) stays full across tile boundaries. The per-element arithmetic is that
// of k_filter_tc (same operands, same fp32 MMA accumulation over K, same
// epilogue), so the band proof is unchanged.
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(b)) : "memory");
}

__global__ void __launch_bounds__(kTcThreads, 1)
    k_filter_tc_p(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int L, int nq,
                  int kblocks, int nN, int stages, const float* __restrict__ cn2, const float* __restrict__ qinv,
                  float c_inv, float* __restrict__ dt, float* __restrict__ gmin, int ngroups) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[kTcMaxStages], empty[kTcMaxStages], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base;
  __shared__ float s_inv[256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = (L + kTcM - 1) / kTcM;
  const uint32_t bytesA = kTcM * 128, bytesB = (uint32_t)(nN * 128);
  const uint32_t stage_bytes = bytesA + bytesB;
  uint32_t ncols = 32;
  while ((int)ncols < 2 * nN) ncols <<= 1;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      mb_init(&full[s], 1);
      mb_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mb_init(&tfull[b], 1);
      mb_init(&tempty[b], 4);  // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(&tmem_base)), "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      uint32_t g = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int kb = 0; kb < kblocks; ++kb, ++g) {
          const uint32_t s = g % (uint32_t)stages, ph = (g / (uint32_t)stages) & 1u;
          mb_wait(&empty[s], ph ^ 1u);
          uint8_t* sA = smem + (size_t)s * stage_bytes;
          mb_expect_tx(&full[s], stage_bytes);
          tma_2d(sA, &tmA, kb * kTcBK, t * kTcM, &full[s]);
          tma_2d(sA + bytesA, &tmB, kb * kTcBK, 0, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(nN >> 3) << 17) | ((uint32_t)(kTcM >> 4) << 24);
      uint32_t g = 0;
      int i = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
        const int ab = i & 1, u = i >> 1;
        if (u >= 1) mb_wait(&tempty[ab], (uint32_t)(u - 1) & 1u);  // the epilogue has drained this buffer
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t dacc = tbase + (uint32_t)(ab * nN);
        for (int kb = 0; kb < kblocks; ++kb, ++g) {
          const uint32_t s = g % (uint32_t)stages, ph = (g / (uint32_t)stages) & 1u;
          mb_wait(&full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t aaddr = s32(smem + (size_t)s * stage_bytes);
          const uint32_t baddr = aaddr + bytesA;
#pragma unroll
          for (int kk = 0; kk < kTcBK / 16; ++kk)
            mma_f16(dacc, sw128_desc(aaddr + kk * 32), sw128_desc(baddr + kk * 32), idesc, (kb | kk) != 0 ? 1u : 0u);
          mma_commit(&empty[s]);
        }
        mma_commit(&tfull[ab]);
      }
    }
    __syncwarp();
  } else {
    const int lg = warp & 3;
    for (int j = threadIdx.x - 64; j < nN; j += 128) s_inv[j] = j < nq ? qinv[j] * c_inv : 0.f;
    asm volatile("bar.sync 1, 128;" ::: "memory");
    int i = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      const int ab = i & 1, u = i >> 1;
      mb_wait(&tfull[ab], (uint32_t)u & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int row = t * kTcM + lg * 32 + lane;
      const float cn = row < L ? cn2[row] : 0.f;
      const int grp = t * 4 + lg;
      for (int c = 0; c < nN; c += 32) {
        uint32_t v[32];
        const uint32_t taddr = tbase + ((uint32_t)(lg * 32) << 16) + (uint32_t)(ab * nN + c);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr));
        if (c + 16 < nN) {
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
                "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
                "=r"(v[30]), "=r"(v[31])
              : "r"(taddr + 16u));
        } else {
#pragma unroll
          for (int j = 16; j < 32; ++j) v[j] = __float_as_uint(CUDART_INF_F);
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        float f[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          f[j] = row < L ? cn - 2.f * (__uint_as_float(v[j]) * s_inv[c + j < nN ? c + j : 0]) : CUDART_INF_F;
          const int q = c + j;
          if (row < L && q < nq && q < nN) dt[(size_t)q * L + row] = f[j];
        }
#pragma unroll
        for (int w = 16; w >= 1; w >>= 1) {
          const bool upper = (lane & w) != 0;
#pragma unroll
          for (int j = 0; j < w; ++j) {
            const float send = upper ? f[j] : f[j + w];
            const float keep = upper ? f[j + w] : f[j];
            f[j] = fminf(keep, __shfl_xor_sync(kFull, send, w));
          }
        }
        const int q = c + lane;
        if (q < nq && q < nN && grp < ngroups) gmin[(size_t)q * ngroups + grp] = f[0];
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mb_arrive(&tempty[ab]);  // this warp's TMEM lanes of buffer ab are read
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(ncols));
  }
}

// ---------------------------------------------------------------- CTA-pair filter (cta_group::2)
// The same contraction with M = 256-centroid tiles on a CTA PAIR (a 2-CTA
// cluster on one TPC): CTA t of the pair holds centroid rows [128t, 128t+128)
// of the tile (A, K-major) and query rows [t QT/2, (t+1) QT/2) of the batch
// tile (B, K-major); the leader (rank 0) issues tcgen05.mma.cta_group::2 with
// M = 256, N = QT, which reads both CTAs' shared memory at the same offsets
// and leaves each CTA the accumulator of ITS 128 rows x QT columns in its own
// TMEM. Both CTAs' tensor TMAs (.cta_group::2) complete their bytes on the
// leader's full barrier (rank-0 address from mapa); the leader's commits are
// multicast to both CTAs' empty / tfull barriers. Per 128 centroids an SM
// now ingests A (256 KB at d 1024) + HALF the query tile instead of the whole
// one: 512 KB instead of 768 KB at QT = 256 (K1). Arithmetic per
// element is that of k_filter_tc (same operands, fp32 accumulation over K in
// the tensor core, same epilogue), so the band proof is unchanged.
__device__ __forceinline__ uint32_t mapa_rank0(uint32_t saddr) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(saddr));
  return r;
}
__device__ __forceinline__ void tma_2d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar_rank0) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(bar_rank0)
      : "memory");
}
__device__ __forceinline__ void mma_f16_pair(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          s32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

// grid.x = 2 x (pairs of 128-centroid tiles in [t0, t_end)), grid.y = query tiles of QT rows; cluster (2,1,1).
// tmA: the pre-tiled fp16 centroids (cf16t) as a 2-D [tiles*kblocks*128][64] tensor, box {64, 128},
// no swizzle (the tiles are stored pre-swizzled); tmB: fp16 queries [nq][d8], box {64, QT/2}, SWIZZLE_128B.
__global__ void __launch_bounds__(kTcThreads, 1)
    k_filter_pair(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int L, int nq,
                  int kblocks, int QT, int stages, const float* __restrict__ cn2, const float* __restrict__ qinv,
                  float c_inv, float* __restrict__ dt, float* __restrict__ gmin, int ngroups, int t0, int t_end) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[kTcMaxStages], empty[kTcMaxStages], tfull;
  __shared__ uint32_t tmem_base;
  __shared__ float s_inv[256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_rank();                // 0 = leader
  const int tile = t0 + (int)blockIdx.x;                // this CTA's 128-centroid tile (pairs: 2p, 2p+1)
  const int m0 = tile * kTcM;
  const int q0 = blockIdx.y * QT;
  const int half = QT / 2;
  const uint32_t bytesA = kTcM * 128, bytesB = (uint32_t)half * 128;
  const uint32_t stage_bytes = bytesA + bytesB;
  uint32_t ncols = 32;
  while ((int)ncols < QT) ncols <<= 1;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      mb_init(&full[s], 1);   // leader: its own arrive.expect_tx (both CTAs' bytes)
      mb_init(&empty[s], 1);  // the leader's MMA commit, multicast to both CTAs
    }
    mb_init(&tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
  }
  if (warp == 1) {  // collective over the pair: same warp, same destination offset in both CTAs
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(&tmem_base)), "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync_all();  // the leader's barriers are initialised before the peer's TMA signals them
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t full0 = mapa_rank0(s32(&full[0]));  // the leader's full barriers (same layout)
      for (int kb = 0; kb < kblocks; ++kb) {
        const int s = kb % stages;
        const uint32_t ph = (uint32_t)(kb / stages) & 1u;
        mb_wait(&empty[s], ph ^ 1u);
        uint8_t* sA = smem + (size_t)s * stage_bytes;
        uint8_t* sB = sA + bytesA;
        if (crank == 0) mb_expect_tx(&full[s], 2u * stage_bytes);
        const uint32_t fb = full0 + (uint32_t)s * 8u;
        tma_2d_pair(s32(sA), &tmA, 0, (tile * kblocks + kb) * kTcM, fb);
        tma_2d_pair(s32(sB), &tmB, kb * kTcBK, q0 + (int)crank * half, fb);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && crank == 0) {
      // instruction descriptor: F32 accum, A/B F16, K-major, N = QT, M = 256
      const uint32_t idesc = (1u << 4) | ((uint32_t)(QT >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
      for (int kb = 0; kb < kblocks; ++kb) {
        const int s = kb % stages;
        const uint32_t ph = (uint32_t)(kb / stages) & 1u;
        mb_wait(&full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t aaddr = s32(smem + (size_t)s * stage_bytes);
        const uint32_t baddr = aaddr + bytesA;
#pragma unroll
        for (int kk = 0; kk < kTcBK / 16; ++kk)
          mma_f16_pair(tbase, sw128_desc(aaddr + kk * 32), sw128_desc(baddr + kk * 32), idesc, (kb | kk) != 0 ? 1u : 0u);
        mma_commit_pair(&empty[s]);  // frees stage s in both CTAs once these MMAs have read it
      }
      mma_commit_pair(&tfull);  // both CTAs' accumulators complete
    }
    __syncwarp();
  } else {
    // epilogue: warps 2..5 -> TMEM lane groups (warp % 4) = this CTA's 128 centroid rows
    const int lg = warp & 3;
    const int row = m0 + lg * 32 + lane;
    const bool live = tile < t_end;  // the pair's second tile past the range end (odd tile count): no stores
    const float cn = row < L ? cn2[row] : 0.f;
    for (int j = threadIdx.x - 64; j < QT; j += 128) {
      const int q = q0 + j;
      s_inv[j] = q < nq ? qinv[q] * c_inv : 0.f;  // product of powers of two >= 2^-120: exact
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");  // epilogue warps only
    mb_wait(&tfull, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int grp = tile * 4 + lg;
    for (int c = 0; c < QT; c += 32) {
      uint32_t v[32];
      const uint32_t taddr = tbase + ((uint32_t)(lg * 32) << 16) + (uint32_t)c;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(taddr));
      if (c + 16 < QT) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
              "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
              "=r"(v[30]), "=r"(v[31])
            : "r"(taddr + 16u));
      } else {
#pragma unroll
        for (int j = 16; j < 32; ++j) v[j] = __float_as_uint(CUDART_INF_F);
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      float f[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        f[j] = row < L ? cn - 2.f * (__uint_as_float(v[j]) * s_inv[c + j < QT ? c + j : 0]) : CUDART_INF_F;
        const int q = q0 + c + j;
        if (live && row < L && q < nq && c + j < QT) dt[(size_t)q * L + row] = f[j];
      }
#pragma unroll
      for (int w = 16; w >= 1; w >>= 1) {
        const bool upper = (lane & w) != 0;
#pragma unroll
        for (int j = 0; j < w; ++j) {
          const float send = upper ? f[j] : f[j + w];
          const float keep = upper ? f[j + w] : f[j];
          f[j] = fminf(keep, __shfl_xor_sync(kFull, send, w));
        }
      }
      const int q = q0 + c + lane;
      if (live && q < nq && c + lane < QT && grp < ngroups) gmin[(size_t)q * ngroups + grp] = f[0];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync_all();  // the peer's MMAs / commits no longer touch this CTA's smem or barriers
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(ncols));
  }
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D fp16 tensor [rows][cols] (row stride cols*2 B), box {64, box_rows}, SWIZZLE_128B (swizzle = false:
// none -- for tiles stored pre-swizzled)
cudaError_t make_tmap_2d(void* map_, const uint16_t* base, int rows, int cols, int box_rows, bool swizzle) {
  CUtensorMap* map = reinterpret_cast<CUtensorMap*>(map_);
  EncodeTiledFn fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * sizeof(uint16_t)};
  cuuint32_t box[2] = {(cuuint32_t)kTcBK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<uint16_t*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

static int btiled_env() {
  static int v = -1;  // VLR_FILTER_BTILED=0: K1's B through the 2-D tensor map of the row-major queries
  if (v < 0) {
    const char* e = getenv("VLR_FILTER_BTILED");
    v = e ? atoi(e) : 1;
  }
  return v;
}
static int pair_env_get() {
  static int v = -1;  // VLR_FILTER_PAIR=1: the CTA-pair kernel (off by default: measured slower at C4)
  if (v < 0) {
    const char* e = getenv("VLR_FILTER_PAIR");
    v = e ? atoi(e) : 0;
  }
  return v;
}
static int persistent_env_get() {
  static int v = -1;  // VLR_FILTER_PERSISTENT=1: the persistent double-buffered kernel (experiment)
  if (v < 0) {
    const char* e = getenv("VLR_FILTER_PERSISTENT");
    v = e ? atoi(e) : 0;
  }
  return v;
}

static int num_sms() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

// query rows per CTA (nN) of the one-CTA kernel for nq <= 256: the batch rounded up to 16, halved while the
// grid (tiles x query tiles) has fewer than 2 CTAs per SM -- a rank of the sharded coarse stage filters only
// 1/world of the tiles (C4, world 8: 64 tiles -> nN 64, 256 CTAs)
static int filter_nn(int nq, int tiles) {
  int nN = ((nq + 15) / 16) * 16;
  static int env_nn = -1;  // VLR_FILTER_NN: fixed query tile (multiple of 16, <= 256; timing experiments)
  if (env_nn < 0) {
    const char* e = getenv("VLR_FILTER_NN");
    env_nn = e ? atoi(e) : 0;
  }
  if (env_nn >= 16 && env_nn % 16 == 0) return std::min(nN, std::min(env_nn, 256));
  const int sms = num_sms();
  // halve the query tile while the grid has fewer CTAs than SMs: each halving re-reads every centroid tile
  // once more, so stop at one CTA per SM (measured at world 8, 64 tiles: nN 64/128 -> stage 1 0.070 ms,
  // nN 32 (the former "2 per SM" rule) 0.081 ms; tools/k1_bench.py, profiles/r02/k1_bench_w8_l.jsonl)
  while (nN > 32 && (long long)tiles * ((nq + nN - 1) / nN) < (long long)sms) nN = ((nN / 2 + 15) / 16) * 16;
  return nN;
}

int filter_btile_rows(int nq, int tiles) {
  if (!btiled_env() || pair_env_get() || persistent_env_get()) return 0;
  return nq <= 256 ? filter_nn(nq, tiles) : 512;  // = nN * nacc of the one-CTA kernel
}

cudaError_t launch_filter_tc(const uint16_t* Qh, const float* qinv, int nq, const DeviceIndex& ix, int t_lo, int t_hi,
                             float* dt, float* gmin, const uint16_t* Qt, cudaStream_t s) {
  if (nq <= 0 || t_hi <= t_lo) return cudaSuccess;
  const int ntiles_all = (ix.nlist + kTcM - 1) / kTcM;
  const bool full_range = t_lo == 0 && t_hi == ntiles_all;
  int nacc, nN;
  if (nq <= 256) {
    nacc = 1;
    nN = filter_nn(nq, t_hi - t_lo);
  } else {
    nacc = 2;
    nN = 256;
  }
  // VLR_FILTER_PERSISTENT=1: the persistent double-buffered kernel for batches <= 256 (experiment; measured
  // 0.102 ms vs 0.060 ms for the one-tile-per-CTA kernel at C4, batch 256: latency-bound at 1 CTA per SM,
  // DRAM 20% / L2 16% of peak, profiles/k1_persistent_r01.md). Off by default.
  const int persistent = persistent_env_get();
  // B multicast cluster size (VLR_FILTER_CLUSTER, default kTcCluster): CL CTAs on adjacent centroid tiles
  // each load 1/CL of the query tile and multicast it to the others (rows per slice a multiple of 8 = one
  // SW128 atom). One accumulator (nq <= 256) only.
  static int cl_env = -1;
  if (cl_env < 0) {
    const char* ce = getenv("VLR_FILTER_CLUSTER");
    cl_env = ce ? atoi(ce) : kTcCluster;
  }
  int CL = 1;
  const bool use_persistent = persistent && full_range;
  if (nacc == 1 && !use_persistent)
    for (int c : {4, 2})
      if (c <= cl_env && nN % (8 * c) == 0 && (t_hi - t_lo) % c == 0) { CL = c; break; }
  // CTA-pair kernel (VLR_FILTER_PAIR=1): the query tile QT <= 256 rows is
  // halved (multiple of 16) while the grid has fewer than ~2 CTAs per SM, so a shard's few centroid tiles
  // still fill the GPU (world > 1: each rank filters 1/world of the tiles)
  const int pair_env = pair_env_get();
  if (pair_env && !use_persistent && CL == 1) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int tiles = t_hi - t_lo, pairs = (tiles + 1) / 2;
    int QT = nq <= 256 ? ((nq + 15) / 16) * 16 : 256;
    static int qt_env = -1;  // VLR_FILTER_QT: fixed query tile (experiments)
    if (qt_env < 0) {
      const char* qe = getenv("VLR_FILTER_QT");
      qt_env = qe ? atoi(qe) : 0;
    }
    if (qt_env >= 32 && qt_env <= 256 && qt_env % 32 == 0) QT = qt_env;
    else
      while (QT > 32 && (long long)2 * pairs * ((nq + QT - 1) / QT) < 2LL * sms) QT = ((QT / 2 + 15) / 16) * 16;
    if (QT < 32) QT = 32;  // two halves of >= 16 rows (N multiple of 16, one SW128 atom per half)
    CUtensorMap tmBp;
    cudaError_t e = make_tmap_2d(&tmBp, Qh, nq, ix.d8, QT / 2, true);
    if (e != cudaSuccess) return e;
    const uint32_t stage_bytes = kTcM * 128 + (uint32_t)(QT / 2) * 128;
    int stages = (int)((100 * 1024) / stage_bytes);
    static int st_env = -1;  // VLR_FILTER_STAGES (experiments)
    if (st_env < 0) {
      const char* se = getenv("VLR_FILTER_STAGES");
      st_env = se ? atoi(se) : 0;
    }
    if (st_env >= 2) stages = st_env;
    if (stages > kTcMaxStages) stages = kTcMaxStages;
    if (stages < 2) stages = 2;
    const size_t smem = (size_t)stages * stage_bytes + 1024;
    e = ensure_smem((const void*)k_filter_pair, smem);
    if (e != cudaSuccess) return e;
    const int kblocks = (ix.d8 + kTcBK - 1) / kTcBK;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * pairs, (nq + QT - 1) / QT);
    cfg.blockDim = dim3(kTcThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_filter_pair, *reinterpret_cast<const CUtensorMap*>(ix.tmapAt), tmBp, ix.nlist,
                              nq, kblocks, QT, stages, (const float*)ix.cnorm2, qinv, ix.c_inv, dt, gmin,
                              (ix.nlist + 31) / 32, t_lo, t_hi);
  }
  const int box_rows_b = (nN < 256 ? nN : 256) / CL;
  CUtensorMap tmB;
  cudaError_t e = make_tmap_2d(&tmB, Qh, nq, ix.d8, box_rows_b, true);
  if (e != cudaSuccess) return e;
  const int kblocks = (ix.d8 + kTcBK - 1) / kTcBK;
  if (nacc == 1 && use_persistent) {
    nN = ((nq + 15) / 16) * 16;  // one accumulator holds the whole batch (no query tiles)
    CUtensorMap tmBp;
    e = make_tmap_2d(&tmBp, Qh, nq, ix.d8, nN, true);
    if (e != cudaSuccess) return e;
    tmB = tmBp;
    const uint32_t sb = kTcM * 128 + (uint32_t)(nN * 128);
    int stages = (int)((200 * 1024) / sb);
    if (stages > kTcMaxStages) stages = kTcMaxStages;
    if (stages < 2) stages = 2;
    const size_t smem = (size_t)stages * sb + 1024;
    e = ensure_smem((const void*)k_filter_tc_p, smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int ntiles = (ix.nlist + kTcM - 1) / kTcM;
    k_filter_tc_p<<<ntiles < sms ? ntiles : sms, kTcThreads, smem, s>>>(
        *reinterpret_cast<const CUtensorMap*>(ix.tmapA), tmB, ix.nlist, nq, kblocks, nN, stages, ix.cnorm2, qinv,
        ix.c_inv, dt, gmin, (ix.nlist + 31) / 32);
    return cudaGetLastError();
  }
  const uint32_t stage_bytes = kTcM * 128 + (uint32_t)(nacc * nN * 128);
  // ~100 KB of stages so that two CTAs share an SM: one CTA's epilogue
  // overlaps the other's TMA/MMA pipeline
  int stages = (int)((100 * 1024) / stage_bytes);
  if (stages > kTcMaxStages) stages = kTcMaxStages;
  if (stages < 2) stages = 2;
  const size_t smem = (size_t)stages * stage_bytes + 1024;
  e = ensure_smem(CL == 4 ? (const void*)k_filter_tc<4> : CL == 2 ? (const void*)k_filter_tc<2> : (const void*)k_filter_tc<1>,
                  smem);
  if (e != cudaSuccess) return e;
  const int tiles = t_hi - t_lo;
  dim3 grid(tiles, (nq + nN * nacc - 1) / (nN * nacc));  // CL divides tiles
  const CUtensorMap& tmA = *reinterpret_cast<const CUtensorMap*>(ix.tmapA);
  const int ngroups = (ix.nlist + 31) / 32;
  static int tiled = -1;  // VLR_FILTER_TILED=0: 2-D tensor TMA of A from the row-major fp16 copy (experiments)
  if (tiled < 0) {
    const char* te = getenv("VLR_FILTER_TILED");
    tiled = te ? atoi(te) : 1;
  }
  const uint16_t* At = (tiled && ix.cf16t) ? ix.cf16t : nullptr;
  if (CL == 1) {
    return launch_pdl(k_filter_tc<1>, grid, dim3(kTcThreads), smem, s, tmA, tmB, ix.nlist, nq, kblocks, nN, nacc,
                      stages, (const float*)ix.cnorm2, qinv, ix.c_inv, dt, gmin, ngroups, At, t_lo, Qt);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (CL == 4)
    return cudaLaunchKernelEx(&cfg, k_filter_tc<4>, tmA, tmB, ix.nlist, nq, kblocks, nN, nacc, stages,
                              (const float*)ix.cnorm2, qinv, ix.c_inv, dt, gmin, ngroups, At, t_lo,
                              (const uint16_t*)nullptr);
  return cudaLaunchKernelEx(&cfg, k_filter_tc<2>, tmA, tmB, ix.nlist, nq, kblocks, nN, nacc, stages,
                            (const float*)ix.cnorm2, qinv, ix.c_inv, dt, gmin, ngroups, At, t_lo,
                            (const uint16_t*)nullptr);
}

// fp16(c * scale) (round to nearest even) into a d8-padded copy; scale is a power of two
__global__ void k_round_f16(const float* __restrict__ src, int rows, int d, int d8, float scale,
                            uint16_t* __restrict__ dst) {
  const long long n = (long long)rows * d8;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / d8;
    const int c = (int)(i - r * d8);
    const float v = c < d ? src[r * d + c] * scale : 0.f;
    dst[i] = __half_as_ushort(__float2half_rn(v));
  }
}

cudaError_t launch_round_f16(const float* src, int rows, int d, int d8, float scale, uint16_t* dst, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  long long n = (long long)rows * d8;
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  k_round_f16<<<(int)blocks, 256, 0, s>>>(src, rows, d, d8, scale, dst);
  return cudaGetLastError();
}

// A operand pre-tiled and pre-swizzled (load time): At[tile][kb] = the 16 KB
// SWIZZLE_128B image of rows [128 tile, 128 tile + 128) x cols [64 kb, 64 kb + 64)
// of cf16 (row r at byte 128 r, its 16-byte chunk j at chunk position j ^ (r & 7);
// rows >= L and cols >= d8 zero). One plain 1-D bulk copy of 16 KB into a
// 1024-aligned smem stage then lands exactly what the 2-D SW128 tensor TMA
// would, but each CTA streams a contiguous 256 KB region of HBM (the tensor
// TMA's 128-byte row pieces at a 2 KB stride measured DRAM-locality-bound).
__global__ void k_tile_f16(const uint16_t* __restrict__ cf16, int L, int d8, int kblocks, int ntiles,
                           uint4* __restrict__ At) {
  const long long n = (long long)ntiles * kblocks * 128 * 8;  // 16-byte chunks
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int pos = (int)(i & 7);                 // chunk position in the smem row
    const int r = (int)((i >> 3) & 127);
    const long long tk = i >> 10;                 // tile * kblocks + kb
    const int kb = (int)(tk % kblocks), tile = (int)(tk / kblocks);
    const int j = pos ^ (r & 7);                  // source chunk
    const int row = tile * 128 + r, col = kb * 64 + j * 8;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (row < L && col < d8) v = *reinterpret_cast<const uint4*>(cf16 + (size_t)row * d8 + col);
    At[i] = v;
  }
}

#ifdef VLR_K1_TRACE
extern "C" int vlr_debug_k1_trace(unsigned long long* out, int n) {
  return cudaMemcpyFromSymbol(out, g_k1_trace, sizeof(unsigned long long) * 6 * (n < 4096 ? n : 4096)) == cudaSuccess
             ? 0 : -1;
}
#endif

cudaError_t launch_tile_f16(const DeviceIndex& ix, cudaStream_t s) {
  const int kblocks = (ix.d8 + kTcBK - 1) / kTcBK, ntiles = (ix.nlist + kTcM - 1) / kTcM;
  const long long n = (long long)ntiles * kblocks * 1024;
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  k_tile_f16<<<(int)blocks, 256, 0, s>>>(ix.cf16, ix.nlist, ix.d8, kblocks, ntiles, reinterpret_cast<uint4*>(ix.cf16t));
  return cudaGetLastError();
}

}  // namespace vlr

// vlr_device.cuh -- device helpers shared by libvlr.so kernels (product path).
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

namespace vlr {

constexpr unsigned kFull = 0xffffffffu;

// bounded mbarrier waits trap (CUDA error) after 4 s instead of hanging the GPU
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// total order on (distance, id) pairs: reading A7 (ties by id)
__device__ __forceinline__ bool lex_less(float d1, long long i1, float d2, long long i2) {
  return d1 < d2 || (d1 == d2 && i1 < i2);
}

// Warp-register top-k (k <= 32): lane i < k holds the i-th smallest (bd, bid)
// of everything inserted so far, ascending by (dist, id). Lanes >= k are idle.
// Insert one warp-uniform candidate (d, id): the lanes holding larger entries
// shift up one slot (shfl_up) and the candidate lands in the freed slot.
__device__ __forceinline__ void wtk_insert(float& bd, long long& bid, float d, long long id, int k, int lane) {
  const bool gt = lane < k && lex_less(d, id, bd, bid);
  const unsigned msk = __ballot_sync(kFull, gt);
  const float ud = __shfl_up_sync(kFull, bd, 1);
  const long long uid = __shfl_up_sync(kFull, bid, 1);
  if (msk == 0u) return;
  const int p = __ffs(msk) - 1;
  if (lane == p) {
    bd = d;
    bid = id;
  } else if (lane > p && gt) {
    bd = ud;
    bid = uid;
  }
}

// Offer each lane's (dist, id) to the warp list; lanes with cand=false skip.
// ids are fetched lazily through `idp` only for lanes that pass the threshold.
__device__ __forceinline__ void wtk_offer(float& bd, long long& bid, float dist, bool cand, int k, int lane,
                                          long long my_id) {
  unsigned cm = __ballot_sync(kFull, cand);
  while (cm) {
    const int src = __ffs(cm) - 1;
    cm &= cm - 1;
    const float d = __shfl_sync(kFull, dist, src);
    const long long id = __shfl_sync(kFull, my_id, src);
    wtk_insert(bd, bid, d, id, k, lane);
  }
}

// Merge one (dist, id) candidate per lane into the warp list with a bitonic
// network: sort the 32 candidates ascending (15 compare-exchange steps), take
// the element-wise min with the list reversed (a bitonic sequence holding the
// 32 smallest of the union), then a 5-step bitonic merge. Lanes without a
// candidate pass (+inf, -1). ~21 shuffle steps in total: cheaper than
// wtk_offer once more than ~6 lanes carry candidates.
__device__ __forceinline__ void wtk_cmpx(float& d, long long& id, int lane, int stride, bool up) {
  const float od = __shfl_xor_sync(kFull, d, stride);
  const long long oid = __shfl_xor_sync(kFull, id, stride);
  const bool lower = (lane & stride) == 0;
  const bool take_min = lower == up;
  const bool o_less = lex_less(od, oid, d, id);
  if (take_min ? o_less : lex_less(d, id, od, oid)) {
    d = od;
    id = oid;
  }
}

__device__ __forceinline__ void wtk_merge32(float& bd, long long& bid, float d, long long id, int k, int lane) {
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1)
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) wtk_cmpx(d, id, lane, stride, (lane & size) == 0 || size == 32);
  // d ascending across lanes; pair list[lane] with cand[31 - lane]
  const float rd = __shfl_sync(kFull, d, 31 - lane);
  const long long rid = __shfl_sync(kFull, id, 31 - lane);
  float ld = lane < k ? bd : CUDART_INF_F;
  long long lid = lane < k ? bid : -1;
  if (lex_less(rd, rid, ld, lid)) {
    ld = rd;
    lid = rid;
  }
#pragma unroll
  for (int stride = 16; stride > 0; stride >>= 1) wtk_cmpx(ld, lid, lane, stride, true);
  if (lane < k) {
    bd = ld;
    bid = lid;
  }
}

// Warp-cooperative k-selection: the running list (lane i < k holds the i-th
// smallest) is merged with n entries fetched as fetch(i) -> (dist, id), in
// chunks of 32*E: k rounds of (lane-local min over E entries + list entry,
// 5-step warp argmin by (dist, id)); the winner's slot is retired. Sorted
// output, ties by id. Padding is (+inf, -1).
template <int E, class F>
__device__ __forceinline__ void warp_select_merge(float& bd, long long& bid, int k, int lane, int n, F fetch) {
  for (int base = 0; base < n; base += 32 * E) {
    float ed[E + 1];
    long long eid[E + 1];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = base + e * 32 + lane;
      ed[e] = CUDART_INF_F;
      eid[e] = -1;
      if (i < n) fetch(i, ed[e], eid[e]);
    }
    ed[E] = lane < k ? bd : CUDART_INF_F;
    eid[E] = lane < k ? bid : -1;
    float nd = CUDART_INF_F;
    long long nid = -1;
    for (int r = 0; r < k; ++r) {
      float md = ed[0];
      long long mid = eid[0];
      int ms = 0;
#pragma unroll
      for (int e = 1; e <= E; ++e)
        if (lex_less(ed[e], eid[e], md, mid)) {
          md = ed[e];
          mid = eid[e];
          ms = e;
        }
      float wd = md;
      long long wid = mid;
      int wl = lane;
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        const float od = __shfl_xor_sync(kFull, wd, o);
        const long long oid = __shfl_xor_sync(kFull, wid, o);
        const int ol = __shfl_xor_sync(kFull, wl, o);
        if (lex_less(od, oid, wd, wid) || (od == wd && oid == wid && ol < wl)) {
          wd = od;
          wid = oid;
          wl = ol;
        }
      }
      if (lane == r) {
        nd = wd;
        nid = wid;
      }
      if (wid < 0) break;  // only padding left (warp-uniform)
      if (lane == wl) {
#pragma unroll
        for (int e = 0; e <= E; ++e)
          if (e == ms) {
            ed[e] = CUDART_INF_F;
            eid[e] = -1;
          }
      }
    }
    bd = nd;
    bid = nid;
  }
}

// float <-> order-preserving unsigned key
__device__ __forceinline__ unsigned fkey(float f) {
  unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float fkey_inv(unsigned k) {
  unsigned u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}

// ---------------------------------------------------------------- NVLink peer exchange
// ("P2P exchange"): a producer kernel stores its slab of an
// exchanged buffer straight into every rank's inbox (IPC-mapped peer device
// memory over NVLink; the own inbox for the own rank), and its LAST CTA to
// finish raises flag[kind][rank] = epoch in every rank's inbox (system-scope
// release after a system fence); a consumer kernel's first thread waits until
// all world flags of its kind carry the search's epoch (acquire), bounded.
constexpr int kMaxWorld = 8;
struct PeerOut {
  void* base[kMaxWorld];       // per rank: the inbox region of this exchange kind ([world][slab] layout)
  uint32_t* flag[kMaxWorld];   // per rank: that rank's flags of this kind ([world], written at [my rank])
  int G, rank;                 // G = 0: no peer exchange (write the local buffer)
  uint32_t epoch;
  int* ctr;                    // CTA-completion counter (local, 0 between launches)
};
struct PeerIn {
  const uint32_t* flags;       // own inbox flags of this kind ([world])
  int G;                       // 0: nothing to wait for
  uint32_t epoch;
  int32_t* status;             // bit 2 (value 4): a peer did not arrive within the bound
};

__device__ __forceinline__ void st_release_sys_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// polling load: relaxed (no L1 invalidation per iteration, as ld.acquire costs); the waiter issues one
// acquire fence after it has seen the flag
__device__ __forceinline__ uint32_t ld_relaxed_sys_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Programmatic dependent launch (PDL): a kernel launched with the programmatic-serialization attribute
// (launch_pdl) may start while the previous kernel of its stream is still running; griddepcontrol.wait
// blocks until that kernel has completed and its memory is visible, launch_dependents lets the next
// kernel start launching. Every chained kernel calls this first, before any early return (so that a
// kernel can never complete before its predecessor). A no-op for a normal launch.
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// element o of this rank's slab (slab elements per rank) into every rank's inbox
template <class T>
__device__ __forceinline__ void peer_store(const PeerOut& p, long long slab, long long o, const T& v) {
  for (int g = 0; g < p.G; ++g) reinterpret_cast<T*>(p.base[g])[(long long)p.rank * slab + o] = v;
}

// every thread of every CTA calls it once, after its stores
__device__ __forceinline__ void peer_signal(const PeerOut& p) {
  if (p.G == 0) return;
  // the barrier orders every thread's peer stores before thread 0's system-scope fence (fences are
  // cumulative), so one fence per CTA releases them all (a fence per thread cost a MEMBAR.SYS each)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned total = gridDim.x * gridDim.y * gridDim.z;
    if ((unsigned)atomicAdd(p.ctr, 1) == total - 1) {  // the last CTA: every CTA's stores are fenced
      *p.ctr = 0;
      __threadfence_system();
      for (int g = 0; g < p.G; ++g) st_release_sys_u32(p.flag[g] + p.rank, p.epoch);
    }
  }
}

// prologue of a consumer kernel: all ranks' slabs of this kind have arrived
__device__ __forceinline__ void peer_wait(const PeerIn& w) {
  if (w.G == 0) return;
  if (threadIdx.x == 0) {
    const unsigned long long t0 = globaltimer_ns();
    for (int r = 0; r < w.G; ++r) {
      unsigned ns = 32;
      for (uint32_t spin = 0; ld_relaxed_sys_u32(w.flags + r) != w.epoch; ++spin) {
        __nanosleep(ns);
        ns = ns < 512 ? 2 * ns : 512;  // back off: many CTAs of a consumer kernel poll at once
        if ((spin & 255u) == 255u && globaltimer_ns() - t0 > 4000000000ull) {  // bounded: never hang
          atomicOr(w.status, 4);
          break;
        }
      }
    }
    __threadfence_system();  // acquire: the slabs after the flags (then the barrier extends it to the CTA)
  }
  __syncthreads();
}

// 16-byte packed result entry used by the cross-GPU exchange
struct __align__(16) Packed {
  float d;
  int32_t pad;
  long long id;
};

}  // namespace vlr

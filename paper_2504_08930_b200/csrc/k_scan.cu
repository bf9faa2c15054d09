// k_scan.cu -- K6 ADC list scan with fused warp top-k, K7 per-rank merge,
// K8 shard merge.
//
// K6: for every owned work item (query q, probed resident list l) and every
// vector i of l:  dist_i = (term1_{q,l} + b_i) + sum_j LUT_q[j][code_ij]
// (DESIGN.md §Numerics), kept if among the k smallest (dist, id) seen by the
// warp. The LUT of the current query lives in shared memory ("shared
// memory stages partial LUTs"), moved there by one TMA bulk copy
// (cp.async.bulk + mbarrier).
//
// Work decomposition: the owned (q, p) items, in query-major
// order, form a stream of W groups of 32 vectors. Persistent CTA c takes the
// contiguous range [c*W/G, (c+1)*W/G) -- perfect balance to one group, no
// blocks for pruned probes. Inside a CTA, the range is cut at
// query boundaries into segments; warps take the segment's groups round-robin.
//
// Inner loop, lane l of a warp handles vector l of a 32-vector group. Its
// m_pad code bytes are in 32-bit registers, stored ROTATED at load time (K0):
// register byte s = 32r + t holds the code of sub-space j = 32r + (l ^ t).
// The LUT is laid out [j/64][code][j%64] fp32, so at step (t, r) the 32 lanes
// read 32 different sub-spaces j%32 = l^t -> 32 different banks: conflict-free
// gathers. One PRMT builds the byte address code*256 + (l^t)*4 (the code byte
// goes to byte 1, the lane offset to byte 0); the slab/half offset is the LDS
// immediate. Per lookup: PRMT + LDS + FADD (+1/R LOP3 for the lane offset).
//
// 4-bit codes (NEXT-3, the paper's IVF-FS code width): the same
// kernel with NB = 4. A lane's 16-byte chunk holds 32 rotated NIBBLES (slot
// s = 32r + t in nibble t of chunk r, low nibble first), the LUT is
// [j/64][code 0..15][j%64] (4 KB per 64 sub-spaces), and each code word is
// split once into its even and odd nibbles (w & 0x0F0F0F0F, (w >> 4) &
// 0x0F0F0F0F) so the same one-PRMT address build applies.
#include <cfloat>
#include <climits>
#include <cstdlib>

#include "vlr_device.cuh"
#include "vlr_internal.cuh"

namespace vlr {

// Optional per-lane L2 line prefetch kPfDist groups (of this warp) beyond the
// register double buffer. Off by default: distances 1-4 measured no faster
// than 0 at C4 (profiles/r01_summary.md), and the extra L2 requests cost power
// under sustained load (tools/sustained.py: -0.8% mean step time without).
#ifndef VLR_PF_DIST
#define VLR_PF_DIST 0
#endif
constexpr int kPfDist = VLR_PF_DIST;

struct ScanArgs {
  int nq, np, k, npairs;
  uint32_t lut_bytes;  // per query: npairs x ksub x 64 x 4
  const int32_t* plocal;
  const float* term1;
  const int64_t* item_off;
  const int64_t* gbase;
  const uint8_t* codes;
  const float* bias;
  const int64_t* ids;
  const float* lut;
  float* pdist;
  int64_t* pid;
  // NEXT-4 early per-query release (k_scan<..., REL = true> only)
  unsigned long long* qdone;  // [nq] groups scanned so far per query (zeroed before the launch)
  uint32_t* ready;            // [nq] device-accessible (normally pinned host) release flags
  uint32_t epoch;             // value written to ready[q] when row q is final
  int64_t* out_ids;           // [nq][k] final rows (device or pinned host)
  float* out_dist;
  int waves;                  // REL: the batch is scanned in this many query waves
  // large k (k > 32, DUMP scan): every candidate's (dist, position) goes to dump[(g - WL) * 32 + lane] for
  // the groups g of queries [q_lo, q_hi); k_select_large keeps each query's k smallest
  int q_lo, q_hi;
  uint2* dump;
  int alt;                    // 1: even CTAs walk their queries backward (all scans; REL always)
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const unsigned long long t0 = globaltimer_ns();
  for (uint32_t i = 0;; ++i) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) break;
    if ((i & 1023u) == 1023u && globaltimer_ns() - t0 > 4000000000ull) asm volatile("trap;");  // bounded: never hang the GPU
  }
}
__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// MP padded sub-spaces of NB-bit codes: MP*NB/32 code words per lane, in
// MP*NB/128 chunks of 16 bytes
template <int MP, int NB>
struct Grp {
  uint32_t w[MP * NB / 32];
  float b, t1;
  long long gaddr;
};

// Advance the item cursor to the item holding group gg (item_off[it] <= gg <
// item_off[it + 1]). Non-owned probes are empty items (0 groups): at world 8
// about 7 of 8 consecutive items are empty, so a one-by-one walk costs a chain
// of dependent L2 loads at every item boundary. The warp probes 32 items per
// step (one load, a ballot); gg is warp-uniform, so the loop is too.
__device__ __forceinline__ void advance_item(const ScanArgs& a, long long gg, long long& it, int lane) {
  if (a.item_off[it + 1] > gg) return;
  const long long n_items = (long long)a.nq * a.np;  // item_off has n_items + 1 entries
  for (;;) {
    const long long j = it + 1 + lane;  // candidate: the first item whose end exceeds gg
    const bool past = j >= n_items || a.item_off[j + 1] > gg;
    const unsigned m = __ballot_sync(kFull, past);
    if (m) {
      it += 1 + (__ffs(m) - 1);
      return;
    }
    it += 32;
  }
}

// L2 prefetch of a whole group's codes: each lane prefetches one 128-B line
// (LSU prefetch, no data return; a 4 KB TMA bulk prefetch per group costs
// ~0.3 us of TMA issue time, tools/tma_issue.cu): keeps DRAM requests in
// flight beyond the register double buffer (K6).
template <int MP, int NB>
__device__ __forceinline__ void grp_prefetch(const ScanArgs& a, long long gg, long long& it, int lane) {
  advance_item(a, gg, it, lane);
  const long long gaddr = a.gbase[a.plocal[it]] + (gg - a.item_off[it]);
  if (lane < MP * NB / 32)  // 128-byte lines of the group
    asm volatile("prefetch.global.L2 [%0];" ::"l"(a.codes + gaddr * (4 * MP * NB) + lane * 128) : "memory");
}

template <int MP, int NB, int EXP = 0>
__device__ __forceinline__ void grp_load(Grp<MP, NB>& G, const ScanArgs& a, long long gg, long long& it, int lane) {
  constexpr int kChunks = MP * NB / 128;
  // the item cursor's loads (item_off, plocal, gbase, term1) hit L1; a per-group metadata array written by
  // K4b (one 8-byte word per group) measured slower: its first touch per line is an L2 round trip on the
  // path to the code loads (scan 1.53 -> 1.81 ms at C4, profiles/r02/scan_trace_gmeta_n_slower.jsonl); a
  // per-warp cache of the current item (end, address offset, term1; loads only at item boundaries) measured
  // slower too (1.543 -> 1.577 ms, 8 B of spills at 128 registers; profiles/r02/scan_trace_icache_v.jsonl)
  advance_item(a, gg, it, lane);
  const int loc = a.plocal[it];
  G.gaddr = a.gbase[loc] + (gg - a.item_off[it]);
  G.t1 = a.term1[it];
  const uint4* src = reinterpret_cast<const uint4*>(a.codes) + G.gaddr * (32 * kChunks) + lane;
#pragma unroll
  for (int c = 0; c < kChunks; ++c) {
    uint4 v;
    if constexpr (EXP == 2) v = make_uint4(gg * 2654435761u + c, gg * 40503u + lane, c * 7919u, lane * 104729u);
    else v = ldg_stream(src + c * 32);
    G.w[4 * c + 0] = v.x;
    G.w[4 * c + 1] = v.y;
    G.w[4 * c + 2] = v.z;
    G.w[4 * c + 3] = v.w;
  }
  G.b = __ldg(a.bias + G.gaddr * 32 + lane);
}

// two independent fp32 accumulators in one 64-bit register pair: FADD2
// (sm_100 packed fp32 add), elementwise identical to two FADDs
__device__ __forceinline__ void fadd2(unsigned long long& acc, float a, float b) {
  asm("{\n.reg .b64 t;\nmov.b64 t, {%1, %2};\nadd.rn.f32x2 %0, %0, t;\n}" : "+l"(acc) : "f"(a), "f"(b));
}
__device__ __forceinline__ float lo32(unsigned long long v) { return __uint_as_float((unsigned)v); }
__device__ __forceinline__ float hi32(unsigned long long v) { return __uint_as_float((unsigned)(v >> 32)); }

// sum_j LUT[j][code_j] for this lane's vector, fixed order:
// accumulator r collects sub-spaces 32r + (lane ^ t), t = 0..31 in order;
// accumulators are paired into FADD2s, result ((acc0 + acc1) + (acc2 + acc3))
// (R = 4; a pairwise tree of the pair sums in general).
template <int MP, int NB>
__device__ __forceinline__ float grp_adc(const Grp<MP, NB>& G, const unsigned char* lutc, uint32_t lane4) {
  constexpr int R = MP / 32;
  constexpr int kSlab = NB == 8 ? 65536 : 4096;  // LUT bytes per 64 sub-spaces
  auto look = [&](int t, int r, uint32_t off) -> float {
    uint32_t word, sel;
    if constexpr (NB == 8) {
      const int s = r * 32 + t;
      word = G.w[s >> 2];
      sel = (uint32_t)(s & 3);
    } else {  // nibble t of chunk r: word r*4 + t/8, byte (t%8)/2, odd t = high nibble
      const uint32_t w = G.w[r * 4 + (t >> 3)];
      word = (t & 1) ? ((w >> 4) & 0x0F0F0F0Fu) : (w & 0x0F0F0F0Fu);
      sel = (uint32_t)((t & 7) >> 1);
    }
    const uint32_t addr = __byte_perm(word, off, 0x5504u | (sel << 4));
    return *reinterpret_cast<const float*>(lutc + addr + (r >> 1) * kSlab + ((r & 1) << 7));
  };
  if constexpr (R == 1) {
    float acc = 0.f;
#pragma unroll
    for (int t = 0; t < 32; ++t) acc += look(t, 0, lane4 ^ (uint32_t)(t << 2));
    return acc;
  } else {
    constexpr int P = R / 2;
    unsigned long long a2[P];
#pragma unroll
    for (int p = 0; p < P; ++p) a2[p] = 0ull;
    float a1 = 0.f;
#pragma unroll
    for (int t = 0; t < 32; ++t) {
      const uint32_t off = lane4 ^ (uint32_t)(t << 2);
#pragma unroll
      for (int p = 0; p < P; ++p) fadd2(a2[p], look(t, 2 * p, off), look(t, 2 * p + 1, off));
      if constexpr (R & 1) a1 += look(t, R - 1, off);
    }
    float ps[P];
#pragma unroll
    for (int p = 0; p < P; ++p) ps[p] = lo32(a2[p]) + hi32(a2[p]);
#pragma unroll
    for (int w = 1; w < P; w <<= 1)
#pragma unroll
      for (int p = 0; p + w < P; p += 2 * w) ps[p] = ps[p] + ps[p + w];
    return (R & 1) ? ps[0] + a1 : ps[0];
  }
}

// offer the lanes' (d, id) with cand set to the warp list (k entries); thr is
// the list's k-th distance
__device__ __forceinline__ void offer32(float& bd, long long& bid, float& thr, float d, long long id, bool cand, int k,
                                        int lane) {
  const unsigned cm = __ballot_sync(kFull, cand);
  if (cm) {
    if (__popc(cm) > 6) wtk_merge32(bd, bid, cand ? d : CUDART_INF_F, cand ? id : -1, k, lane);
    else wtk_offer(bd, bid, d, cand, k, lane, id);
    thr = __shfl_sync(kFull, bd, k - 1);
  }
}

// offer a list held by lanes < k (padding (+inf, -1) elsewhere) to the warp list
__device__ __forceinline__ void list_offer(float& bd, long long& bid, float& thr, float d, long long id, int k,
                                           int lane) {
  offer32(bd, bid, thr, d, id, lane < k && d < CUDART_INF_F && d <= thr, k, lane);
}

// ---------------------------------------------------------------- K7 per-rank merge
// Top-k by (dist, id) of the union of the partial lists the scan wrote for a
// query: every scan CTA whose range intersects the query's groups holds
// kScanWarps warp lists of k, each SORTED ascending (padding (+inf, -1) last).
// One CTA of nw warps per query, three phases:
//  A. the k smallest list HEADS (minima) are found (lanes hold one list head
//     each; warp lists + a pairwise tree). Their k-th distance T0 bounds the
//     answer: k distinct entries are <= T0, so the final k-th <= T0, and a
//     list whose head is > T0 cannot contribute. At most k lists (plus ties)
//     pass.
//  B. the indices of the lists with head <= T0 are compacted into shared
//     memory.
//  C. warp 0 stages those lists (k coalesced entries each, 32 lists at a
//     time) in shared memory and k-way merges them: k rounds of a 5-step
//     warp argmin over the 32 list heads.
// Batch 1 (148 CTAs x 16 lists) reads 2,368 heads and ~k whole lists instead
// of 23,680 entries; batch 256 (~32 lists per query) needs one warp.
constexpr int kMergeMaxWarps = 16;
constexpr int kMergeMaxLists = 4096;  // >= (scan CTAs) x kScanWarps (checked at launch)
static_assert(kScanWarps <= kMergeMaxWarps, "the in-scan release merge runs on the scan CTA's warps");

// pairwise tree over the CTA's warp lists; warp 0 ends with the CTA list.
// Level `stride` reads slots = stride (mod 2 stride) and writes slots = 0
// (mod 2 stride): one barrier per level.
__device__ __forceinline__ void cta_tree(float& bd, long long& bid, float& thr, int k, int lane, int warp, int nw,
                                         float* s_d, long long* s_id) {
  if (nw == 1) return;
  s_d[warp * 32 + lane] = lane < k ? bd : CUDART_INF_F;
  s_id[warp * 32 + lane] = lane < k ? bid : -1;
  __syncthreads();
  for (int stride = 1; stride < nw; stride <<= 1) {
    if ((warp & (2 * stride - 1)) == 0 && warp + stride < nw) {
      list_offer(bd, bid, thr, s_d[(warp + stride) * 32 + lane], s_id[(warp + stride) * 32 + lane], k, lane);
      s_d[warp * 32 + lane] = lane < k ? bd : CUDART_INF_F;
      s_id[warp * 32 + lane] = lane < k ? bid : -1;
    }
    __syncthreads();
  }
}

struct MergeSmem {
  long long s_id[kMergeMaxWarps * 32];
  long long s_lid[32 * 33];                    // staged lists (phase C)
  float s_d[kMergeMaxWarps * 32];
  float s_ld[32 * 33];
  int s_rel[kMergeMaxLists];                   // relevant list indices
  float s_t0;
  int s_nrel;
};

// partial-list loads: the standalone K7 reads partials of a finished kernel
// (read-only path); the scan's in-kernel release merge (NEXT-4) reads partials
// other CTAs of the same launch wrote, so it goes through L2 (ld.global.cg)
template <bool CG, typename T>
__device__ __forceinline__ T ldp(const T* p) {
  if constexpr (CG) return __ldcg(p);
  else return __ldg(p);
}

// merge of query q by the whole CTA (nw = blockDim.x / 32 warps); warp 0
// writes the row. Warps other than 0 return after phase B (no barrier after).
// The scan split the group range [WL, WH) of q's wave statically over n_cta
// CTAs; q's groups are [S, E); CTA c's lists for q sit at
// slot (c + q + zoff) (zoff = wave * n_cta keeps the slots of different waves
// apart; 0 without waves).
template <bool CG>
__device__ __forceinline__ void merge_query(
    int q, int k, int n_cta, long long WL, long long WH, long long zoff, long long S, long long E,
    const float* pdist, const int64_t* pid, int64_t* out_ids, float* out_dist, Packed* __restrict__ packed,
    MergeSmem& sm, const PeerOut* pout = nullptr, int nq = 0) {
  float* s_d = sm.s_d;
  long long* s_id = sm.s_id;
  float& s_t0 = sm.s_t0;
  int& s_nrel = sm.s_nrel;
  int* s_rel = sm.s_rel;
  float* s_ld = sm.s_ld;
  long long* s_lid = sm.s_lid;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const long long W = WH - WL;
  const long long* pidl = reinterpret_cast<const long long*>(pid);
  float bd = CUDART_INF_F, thr = CUDART_INF_F;
  long long bid = -1;
  int cf = 0, nl = 0;  // lists of CTAs cf.. : nl = (#CTAs) x kScanWarps
  bool maybe_empty = false;
  auto start = [&](int c) { return (long long)c * W / n_cta; };
  if (E > S) {
    // largest c with start(c) = floor(c W / G) <= g  <=>  c W < (g + 1) G
    auto cta_of = [&](long long g) {
      const long long c = ((g - WL + 1) * n_cta - 1) / W;
      return (int)(c < n_cta - 1 ? c : n_cta - 1);
    };
    cf = cta_of(S);
    nl = (cta_of(E - 1) - cf + 1) * kScanWarps;
    maybe_empty = W < n_cta;  // otherwise every CTA owns >= 1 group
  }
  const long long base = (long long)(cf + q + zoff) * kScanWarps * k;  // list li starts at base + li * k
  auto head_ok = [&](int li) { return !maybe_empty || start(cf + li / kScanWarps) != start(cf + li / kScanWarps + 1); };
  // ---- phase A: k smallest heads
  constexpr int U = 4;
  for (int l0 = warp * 32 * U; l0 < nl; l0 += nw * 32 * U) {
    float d[U];
    long long id[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int li = l0 + u * 32 + lane;
      d[u] = CUDART_INF_F;
      id[u] = -1;
      if (li < nl && head_ok(li)) {
        d[u] = ldp<CG>(pdist + base + (long long)li * k);
        id[u] = ldp<CG>(pidl + base + (long long)li * k);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) offer32(bd, bid, thr, d[u], id[u], d[u] < CUDART_INF_F && d[u] <= thr, k, lane);
  }
  cta_tree(bd, bid, thr, k, lane, warp, nw, s_d, s_id);
  if (warp == 0) {
    const float t0 = __shfl_sync(kFull, bd, k - 1);
    if (lane == 0) s_t0 = t0;
  }
  __syncthreads();
  const float t0 = s_t0;
  // ---- phase B: indices of the lists whose head <= T0 -> shared memory
  if (threadIdx.x == 0) s_nrel = 0;
  __syncthreads();
  for (int l0 = warp * 32; l0 < nl; l0 += nw * 32) {
    const int li = l0 + lane;
    float h = CUDART_INF_F;
    if (li < nl && head_ok(li)) h = ldp<CG>(pdist + base + (long long)li * k);
    const bool rel = h < CUDART_INF_F && h <= t0;
    const unsigned rm = __ballot_sync(kFull, rel);
    if (rm) {
      int at = 0;
      if (lane == 0) at = atomicAdd(&s_nrel, __popc(rm));
      at = __shfl_sync(kFull, at, 0);
      if (rel) s_rel[at + __popc(rm & ((1u << lane) - 1u))] = li;
    }
  }
  __syncthreads();
  if (warp != 0) return;
  // ---- phase C (warp 0): k-way merge of the relevant sorted lists, 32 at a
  // time (lane r owns list r of the batch, staged in shared memory)
  const int nrel = s_nrel;
  bd = CUDART_INF_F;
  bid = -1;
  for (int r0 = 0; r0 < nrel; r0 += 32) {
    const int nb = nrel - r0 < 32 ? nrel - r0 : 32;
    for (int r1 = 0; r1 < nb; r1 += 8) {  // stage: k coalesced entries per list, 8 lists' loads in flight
      float sd[8];
      long long sid[8];
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const int r = r1 + v;
        if (r < nb && lane < k) {
          const long long o = base + (long long)s_rel[r0 + r] * k + lane;
          sd[v] = ldp<CG>(pdist + o);
          sid[v] = ldp<CG>(pidl + o);
        }
      }
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const int r = r1 + v;
        if (r < nb && lane < k) {
          s_ld[r * 33 + lane] = sd[v];
          s_lid[r * 33 + lane] = sid[v];
        }
      }
    }
    __syncwarp();
    int p = 0;
    float hd = lane < nb ? s_ld[lane * 33] : CUDART_INF_F;
    long long hid = lane < nb ? s_lid[lane * 33] : -1;
    float od = CUDART_INF_F;
    long long oid = -1;
    for (int t = 0; t < k; ++t) {
      float wd = hd;
      long long wid = hid;
      int wl = lane;
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        const float xd = __shfl_xor_sync(kFull, wd, o);
        const long long xid = __shfl_xor_sync(kFull, wid, o);
        const int xl = __shfl_xor_sync(kFull, wl, o);
        if (lex_less(xd, xid, wd, wid) || (xd == wd && xid == wid && xl < wl)) {
          wd = xd;
          wid = xid;
          wl = xl;
        }
      }
      if (!(wd < CUDART_INF_F)) break;  // only padding left (warp-uniform)
      if (lane == t) {
        od = wd;
        oid = wid;
      }
      if (lane == wl) {
        ++p;
        hd = p < k ? s_ld[lane * 33 + p] : CUDART_INF_F;
        hid = p < k ? s_lid[lane * 33 + p] : -1;
      }
    }
    __syncwarp();
    if (r0 == 0) {
      bd = od;
      bid = oid;
    } else {
      list_offer(bd, bid, thr, od, oid, k, lane);
    }
    thr = __shfl_sync(kFull, bd, k - 1);
  }
  if (lane < k) {
    if (pout && pout->G) {  // NVLink peer exchange: this rank's partial row into every rank's inbox
      Packed p;
      p.d = bd;
      p.pad = 0;
      p.id = bid;
      peer_store(*pout, (long long)nq * k, (long long)q * k + lane, p);
    } else if (packed) {
      Packed p;
      p.d = bd;
      p.pad = 0;
      p.id = bid;
      packed[(size_t)q * k + lane] = p;
    } else {
      out_ids[(size_t)q * k + lane] = bid;
      out_dist[(size_t)q * k + lane] = bd;
    }
  }
}


__global__ void __launch_bounds__(kMergeMaxWarps * 32) k_rank_merge(
    int nq, int np, int k, int n_cta, const int64_t* __restrict__ item_off, const float* __restrict__ pdist,
    const int64_t* __restrict__ pid, int64_t* __restrict__ out_ids, float* __restrict__ out_dist,
    Packed* __restrict__ packed, PeerOut pout) {
  pdl_entry();  // PDL: wait for the previous kernel in the stream, then let the next one launch
  __shared__ MergeSmem sm;
  const int q = blockIdx.x;
  merge_query<false>(q, k, n_cta, 0, item_off[(long long)nq * np], 0, item_off[(long long)q * np],
                     item_off[(long long)(q + 1) * np], pdist, pid, out_ids, out_dist, packed, sm, &pout, nq);
  // merge_query returns warps > 0 early (after phase B): the CTA's arrival is by warp 0
  if (pout.G && (threadIdx.x >> 5) == 0) {
    __threadfence_system();
    __syncwarp();
    if (threadIdx.x == 0 && (unsigned)atomicAdd(pout.ctr, 1) == gridDim.x - 1) {
      *pout.ctr = 0;
      __threadfence_system();
      for (int g = 0; g < pout.G; ++g) st_release_sys_u32(pout.flag[g] + pout.rank, pout.epoch);
    }
  }
}

template <int MP, int NB, int EXP, bool DUMP = false>
__device__ __forceinline__ void grp_finish(const Grp<MP, NB>& G, const ScanArgs& a, const unsigned char* lutc,
                                           uint32_t lane4, int lane, float& bd, long long& bid, float& thr,
                                           long long dslot = 0) {
  float s;
  if constexpr (EXP == 1) {  // timing experiment: no LUT gathers (ALU sum of code words)
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < MP * NB / 32; ++i) x ^= G.w[i];
    s = (float)(x & 0xffff) * 1e-9f;
  } else {
    s = grp_adc<MP, NB>(G, lutc, lane4);
  }
  const float dist = (G.t1 + G.b) + s;
  if constexpr (DUMP) {  // large k: every candidate out (padding rows have dist = +inf)
    a.dump[dslot * 32 + lane] = make_uint2(__float_as_uint(dist), (uint32_t)(G.gaddr * 32 + lane));
    return;
  }
  const bool cand = dist <= thr;
  long long my_id = 0;
  if (cand) my_id = __ldg(reinterpret_cast<const long long*>(a.ids) + G.gaddr * 32 + lane);
  const unsigned cm = __ballot_sync(kFull, cand);
  if (cm) {
    if (__popc(cm) > 6) wtk_merge32(bd, bid, cand ? dist : CUDART_INF_F, cand ? my_id : -1, a.k, lane);
    else wtk_offer(bd, bid, dist, cand, a.k, lane, my_id);
    thr = __shfl_sync(kFull, bd, a.k - 1);
  }
}

// ---------------------------------------------------------------- NEXT-4 release
// REL scan (NEXT-4, the GPU analog of the paper's dynamic dispatcher,
// P:408-414): the scan runs on all SMs but one and, after each query segment,
// adds the segment's group count to qdone[q] (release-ordered after the
// segment's partial lists). One resident merger CTA (k_release_merge, on the
// remaining SM, launched on a forked stream) picks up every query whose count
// is complete, merges its partial lists with the K7 code (through L2) and
// raises ready[q]. The merge is not inlined into the scan: its registers make
// the MP = 128 scan loop spill. So that queries complete
// progressively rather than all at the end, the REL batch is cut at query
// boundaries into a.waves waves (wave z = queries [z nq / Z, (z+1) nq / Z));
// every CTA scans its static share of wave 0, then of wave 1, ... (no grid
// barrier: each CTA's share of a wave is proportional, so waves finish in
// order). Without REL there is one wave: the plain static split of the stream.
__device__ __forceinline__ void rel_segment_done(const ScanArgs& a, int q, long long ng) {
  if (threadIdx.x == 0) {
    __threadfence();  // this CTA's partial lists (stored before the caller's barrier) before its count
    atomicAdd(a.qdone + q, (unsigned long long)ng);
  }
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Warp merge of query q's partial lists (same result as K7: the k smallest
// (dist, id) of the union, ids unique). The lists of CTAs cf.. of q's wave
// (slot c + q + zoff, kScanWarps lists of k sorted entries each):
//  A. the k smallest list heads give T0 (k distinct entries are <= T0);
//  B. every list whose head is <= T0 (at most k plus ties) is offered whole.
__device__ __forceinline__ void warp_merge_query(const ScanArgs& a, int q, int G, long long WL, long long WH,
                                                 long long zoff, long long S, long long E, int lane, float& bd,
                                                 long long& bid) {
  const int k = a.k;
  const long long W = WH - WL;
  const long long* pidl = reinterpret_cast<const long long*>(a.pid);
  float thr = CUDART_INF_F;
  bd = CUDART_INF_F;
  bid = -1;
  if (E <= S) return;
  auto cta_of = [&](long long g) {
    const long long c = ((g - WL + 1) * G - 1) / W;
    return (int)(c < G - 1 ? c : G - 1);
  };
  auto start = [&](int c) { return (long long)c * W / G; };
  const int cf = cta_of(S);
  const int nl = (cta_of(E - 1) - cf + 1) * kScanWarps;
  const bool maybe_empty = W < G;
  const long long base = (long long)(cf + q + zoff) * kScanWarps * k;
  auto head_ok = [&](int li) { return !maybe_empty || start(cf + li / kScanWarps) != start(cf + li / kScanWarps + 1); };
  for (int l0 = 0; l0 < nl; l0 += 32) {  // A
    const int li = l0 + lane;
    float d = CUDART_INF_F;
    long long id = -1;
    if (li < nl && head_ok(li)) {
      d = __ldcg(a.pdist + base + (long long)li * k);
      id = __ldcg(pidl + base + (long long)li * k);
    }
    offer32(bd, bid, thr, d, id, d < CUDART_INF_F && d <= thr, k, lane);
  }
  const float t0 = __shfl_sync(kFull, bd, k - 1);
  bd = CUDART_INF_F;
  bid = -1;
  thr = CUDART_INF_F;
  for (int l0 = 0; l0 < nl; l0 += 32) {  // B
    const int li = l0 + lane;
    float h = CUDART_INF_F;
    if (li < nl && head_ok(li)) h = __ldcg(a.pdist + base + (long long)li * k);
    unsigned rm = __ballot_sync(kFull, h < CUDART_INF_F && h <= t0);
    while (rm) {
      const int r = __ffs(rm) - 1;
      rm &= rm - 1;
      const long long o = base + (long long)(l0 + r) * k + lane;
      float d = CUDART_INF_F;
      long long id = -1;
      if (lane < k) {
        d = __ldcg(a.pdist + o);
        id = __ldcg(pidl + o);
      }
      list_offer(bd, bid, thr, d, id, k, lane);
    }
  }
}

// qdone[q] bit 63 = "claimed": the merger (during the scan) and k_release_rest (after it) both claim a query
// with an atomicOr before merging it, so exactly one of them releases it (the scan's group counts stay
// below 2^63)
constexpr unsigned long long kClaim = 1ull << 63;
#ifdef VLR_SCAN_TRACE
// timing variant: per query the globaltimer ns of its flag store and who released it (1 merger, 2 rest);
// [0] = first k_release_rest CTA start, [1] = merger end
__device__ unsigned long long g_rel_trace[4096][2];
__device__ unsigned long long g_rel_misc[4];  // [2] stamp before the fork, [3] stamp after the join
__global__ void k_stamp(int i) { g_rel_misc[i] = globaltimer_ns(); }
#endif
__device__ __forceinline__ bool rel_claim(const ScanArgs& a, int q, int lane) {
  unsigned long long old = 0;
  if (lane == 0) old = atomicOr(a.qdone + q, kClaim);
  return (__shfl_sync(kFull, old, 0) & kClaim) == 0;
}

// merge query q's partial lists, write its row and raise its flag (one warp; q is complete and claimed)
__device__ __forceinline__ void release_query(const ScanArgs& a, int q, int G, int lane, int who = 0) {
  const int nq = a.nq, np = a.np, Z = a.waves;
  __threadfence();  // acquire: q's partial lists after its completed count
  const long long S = a.item_off[(long long)q * np], E = a.item_off[(long long)(q + 1) * np];
  int z = (int)(((long long)(q + 1) * Z - 1) / nq);  // q's wave and its group range (k_scan's split)
  z = z < Z - 1 ? z : Z - 1;
  const long long WL = a.item_off[(long long)((long long)z * nq / Z) * np];
  const long long WH = a.item_off[(long long)((long long)(z + 1) * nq / Z) * np];
  float bd;
  long long bid;
  warp_merge_query(a, q, G, WL, WH, (long long)z * G, S, E, lane, bd, bid);
  if (lane < a.k) {
    a.out_ids[(size_t)q * a.k + lane] = bid;
    a.out_dist[(size_t)q * a.k + lane] = bd;
  }
  __threadfence_system();  // row q (possibly in pinned host memory) before its flag
  __syncwarp();
  if (lane == 0) st_release_sys(a.ready + q, a.epoch);
#ifdef VLR_SCAN_TRACE
  if (lane == 0 && q < 4096) {
    g_rel_trace[q][0] = globaltimer_ns();
    g_rel_trace[q][1] = (unsigned long long)who;
  }
#else
  (void)who;
#endif
  __syncwarp();
}

// the resident merger CTA: warp w owns queries w, w + nw, ... and merges and releases each one as soon as
// the scan has finished it (qdone[q] == its groups), in whatever order they complete (the scan's CTAs walk
// their queries in alternating directions, so completion is not in query order); G = the scan's grid size.
// The queries still unreleased when the scan ends are taken by k_release_rest (all SMs, one warp each).
__global__ void __launch_bounds__(kMergeMaxWarps * 32, 1) k_release_merge(ScanArgs a, int G, int32_t* status) {
  extern __shared__ unsigned char s_rel[];  // [nq] 1 = released here or claimed by k_release_rest
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nq = a.nq, np = a.np;
  for (int q = threadIdx.x; q < nq; q += blockDim.x) s_rel[q] = 0;
  __syncthreads();
  const int mine = warp < nq ? (nq - warp + nw - 1) / nw : 0;
  int left = mine;
  const unsigned long long t0 = globaltimer_ns();
  while (left > 0) {
    bool any = false;
    for (int j0 = 0; j0 < mine; j0 += 32) {
      // lane i polls query warp + nw (j0 + i) (relaxed load; the acquire is the fence in release_query)
      const int j = j0 + lane;
      const int qq = warp + nw * j;
      bool ready = false;
      if (j < mine && !s_rel[qq]) {
        const long long S = a.item_off[(long long)qq * np], E = a.item_off[(long long)(qq + 1) * np];
        const unsigned long long v = ld_relaxed_gpu(a.qdone + qq);
        ready = (v & kClaim) != 0 || v == (unsigned long long)(E - S);
      }
      unsigned m = __ballot_sync(kFull, ready);
      while (m) {
        const int r = __ffs(m) - 1;
        m &= m - 1;
        const int q = warp + nw * (j0 + r);
        if (rel_claim(a, q, lane)) release_query(a, q, G, lane, 1);
        if (lane == 0) s_rel[q] = 1;
        __syncwarp();
        --left;
        any = true;
      }
    }
    if (!any) {
      __nanosleep(256);
      // bounded: a query whose scan did not complete in time is NOT merged and NOT released (its partial
      // lists may be incomplete or left over from an earlier search): ready[q] stays != epoch, the host
      // wait (vlr_wait_ready / vlr_poll_ready) times out instead of returning a wrong row, and status bit 1
      // is reported as VLR_ERR_CUDA by vlr_search / the next call on the handle
      if (globaltimer_ns() - t0 > 4000000000ull) {
        if (lane == 0) atomicOr(status, 2);
        break;
      }
    }
  }
#ifdef VLR_SCAN_TRACE
  __syncthreads();
  if (threadIdx.x == 0) g_rel_misc[1] = globaltimer_ns();
#endif
}

// after the release scan (stream order: every partial list is final): one warp per query claims and
// releases the queries the merger has not taken yet -- the queries completing at the very end of the scan
// are released in parallel over the GPU instead of 16 at a time by the merger's warps
__global__ void __launch_bounds__(512) k_release_rest(ScanArgs a, int G) {
  const int lane = threadIdx.x & 31;
  const int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q >= a.nq) return;
#ifdef VLR_SCAN_TRACE
  if (threadIdx.x == 0) atomicMin(&g_rel_misc[0], globaltimer_ns());
#endif
  if ((ld_relaxed_gpu(a.qdone + q) & kClaim) != 0) return;  // released (or being released) by the merger
  if (rel_claim(a, q, lane)) release_query(a, q, G, lane, 2);
}

#ifdef VLR_SCAN_TRACE
// timing variant (tools/scan_trace.py): per CTA start, end, LUT-wait ns, segments, smid, groups
__device__ unsigned long long g_scan_trace[1024][6];
#endif
template <int MP, int NB, int EXP, bool REL = false, bool DUMP = false>
__global__ void __launch_bounds__(kScanThreads, 1) k_scan(ScanArgs a) {
  pdl_entry();  // PDL: wait for the previous kernel in the stream, then let the next one launch
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ long long s_it;
  __shared__ long long s_ng;
  __shared__ int s_z, s_qa, s_qb, s_q;
  __shared__ long long s_g0, s_g1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int G = gridDim.x, c = blockIdx.x;
  const uint32_t lut_bytes = a.lut_bytes;
  if (threadIdx.x == 0) {
    mbar_init(&mbar, 1);
    fence_mbar_init();
  }
  const uint32_t lane4 = (uint32_t)lane << 2;
  const unsigned char* lutc = smem;
  uint32_t phase = 0;
#ifdef VLR_SCAN_TRACE
  unsigned long long tr_start = globaltimer_ns(), tr_lut = 0, tr_seg = 0, tr_grp = 0;
#endif
  // REL: the wave index lives in shared memory and is re-read where needed, so
  // no register is held across the scan loop for it (the MP = 128 loop needs
  // all 128 registers)
  if constexpr (REL) {
    if (threadIdx.x == 0) s_z = 0;
    __syncthreads();
  }
  auto zcur = [&]() -> int { return *reinterpret_cast<volatile int*>(&s_z); };
  // REL: the wave loop's counter is s_z and its bound the kernel parameter, so no register is live across
  // the scan loop for them (a register counter made the MP = 128 REL loop spill)
  for (int z1 = 0;; ++z1) {
    if constexpr (REL) {
      __syncthreads();  // s_z of the previous wave written
      if (zcur() >= a.waves) break;
    } else {
      if (z1 > 0) break;
    }
    const int z = REL ? zcur() : 0;
    const int i_lo = (REL ? (int)((long long)z * a.nq / a.waves) : a.q_lo) * a.np;
    const int i_hi = (REL ? (int)((long long)(z + 1) * a.nq / a.waves) : a.q_hi) * a.np;
    const long long WL = a.item_off[i_lo], WH = a.item_off[i_hi];
    const long long g0 = WL + (long long)c * (WH - WL) / G, g1 = WL + (long long)(c + 1) * (WH - WL) / G;
    if constexpr (REL) {
      __syncthreads();  // every thread has read s_z
      if (threadIdx.x == 0) s_z = z + 1;
    }
    if (g0 >= g1) continue;  // CTA-uniform
    // item containing group g0: the last i with item_off[i] <= g0, by a CTA-parallel search (each round
    // samples kScanThreads positions: 2 dependent loads for up to 256K items, where a one-thread binary
    // search costs ~15 dependent L2 round trips -- paid at every wave start of the release scan)
    {
      int lo = i_lo, hi = i_hi;  // item_off[lo] <= g0 < item_off[hi]
      while (hi - lo > 1) {
        const int step = (hi - lo + kScanThreads - 1) / kScanThreads;
        const int i = lo + (int)threadIdx.x * step;
        __syncthreads();  // s_it of the previous round / wave consumed
        if (threadIdx.x == 0) s_it = lo;
        __syncthreads();
        if (threadIdx.x > 0 && i < hi && a.item_off[i] <= g0) atomicMax(reinterpret_cast<long long*>(&s_it), (long long)i);
        __syncthreads();
        lo = (int)s_it;
        hi = lo + step < hi ? lo + step : hi;
      }
      __syncthreads();
      if (threadIdx.x == 0) s_it = lo;
      __syncthreads();
    }
    // the CTA's queries: q_a (holding group g0) .. q_b (holding group g1 - 1), kept in shared memory (no
    // registers live across the scan loop); one segment per query
    {
      long long it0 = s_it;
      advance_item(a, g0, it0, lane);
      if (threadIdx.x == 0) {
        int qb = (int)(it0 / a.np);
        s_qa = qb;
        while (a.item_off[(long long)(qb + 1) * a.np] < g1) ++qb;
        s_qb = qb;
        s_g0 = g0;
        s_g1 = g1;
      }
      __syncthreads();
    }
    auto vol_i = [](const int& x) { return *reinterpret_cast<const volatile int*>(&x); };
    auto vol_l = [](const long long& x) { return *reinterpret_cast<const volatile long long*>(&x); };
    for (int si = 0; si <= vol_i(s_qb) - vol_i(s_qa); ++si) {
      // even CTAs walk their queries backward, odd CTAs forward: for NEXT-4 (REL) the query shared by CTAs
      // 2j and 2j+1 is scanned first by both and completes early; VLR_SCAN_ALT=1 applies
      // the same order to every scan
      const int q = ((REL || a.alt) && (c & 1) == 0) ? vol_i(s_qb) - si : vol_i(s_qa) + si;
      const long long qstart = a.item_off[(long long)q * a.np], qend = a.item_off[(long long)(q + 1) * a.np];
      const long long cg0 = vol_l(s_g0), cg1 = vol_l(s_g1);
      const long long g = qstart > cg0 ? qstart : cg0;
      const long long seg_end = qend < cg1 ? qend : cg1;
      if (g >= seg_end) continue;  // a query without owned groups (CTA-uniform)
      if (threadIdx.x == 0) {
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&mbar, lut_bytes);
        const unsigned char* src = reinterpret_cast<const unsigned char*>(a.lut) + (size_t)q * lut_bytes;
        for (uint32_t off = 0; off < lut_bytes; off += 32768u)
          bulk_g2s(smem + off, src + off, lut_bytes - off < 32768u ? lut_bytes - off : 32768u, &mbar);
      }
      if constexpr (REL) {  // segment length and query through shared memory: nothing extra stays live across
        if (threadIdx.x == 0) {  // the scan loop
          s_ng = seg_end - g;
          s_q = q;
        }
      }
#ifdef VLR_SCAN_TRACE
      const unsigned long long tw0 = globaltimer_ns();
#endif
      mbar_wait(&mbar, phase);
      phase ^= 1u;
#ifdef VLR_SCAN_TRACE
      tr_lut += globaltimer_ns() - tw0;
      ++tr_seg;
      tr_grp += (unsigned long long)(seg_end - g);
#endif

      float bd = CUDART_INF_F, thr = CUDART_INF_F;
      long long bid = -1;
      long long gg = g + warp;
      // item cursors of the loads and of the L2 prefetch (kPfDist groups of this warp ahead), from an item
      // at or before the segment's first (the item holding g0, or q's first item)
      long long it = g == cg0 ? vol_l(s_it) : (long long)q * a.np, itp = it;
      Grp<MP, NB> A, B;
      if (gg < seg_end) {
        for (int p = 1; p <= kPfDist; ++p)
          if (gg + p * kScanWarps < seg_end) grp_prefetch<MP, NB>(a, gg + p * kScanWarps, itp, lane);
        grp_load<MP, NB, EXP>(A, a, gg, it, lane);
      }
      while (gg < seg_end) {
        const long long gn = gg + kScanWarps;
        if constexpr (kPfDist > 0)
          if (gn + kPfDist * kScanWarps < seg_end) grp_prefetch<MP, NB>(a, gn + kPfDist * kScanWarps, itp, lane);
        if (gn < seg_end) grp_load<MP, NB, EXP>(B, a, gn, it, lane);
        grp_finish<MP, NB, EXP, DUMP>(A, a, lutc, lane4, lane, bd, bid, thr, gg - WL);
        if (gn >= seg_end) break;
        const long long gm = gn + kScanWarps;
        if constexpr (kPfDist > 0)
          if (gm + kPfDist * kScanWarps < seg_end) grp_prefetch<MP, NB>(a, gm + kPfDist * kScanWarps, itp, lane);
        if (gm < seg_end) grp_load<MP, NB, EXP>(A, a, gm, it, lane);
        grp_finish<MP, NB, EXP, DUMP>(B, a, lutc, lane4, lane, bd, bid, thr, gn - WL);
        gg = gm;
      }
      // REL: q comes back from shared memory (no register live across the scan loop for it; the same for the
      // plain scan measured slower: 1.562 vs 1.530 ms at C4, profiles/r02/scan_ab_smemq_aa.jsonl)
      const int qs = REL ? *reinterpret_cast<volatile int*>(&s_q) : q;
      const long long slot = ((long long)(c + qs) + (long long)(REL ? zcur() - 1 : 0) * G) * kScanWarps * a.k + warp * a.k;
      if (!DUMP && lane < a.k) {  // REL: released by thread 0's fence after the barrier (rel_segment_done)
        a.pdist[slot + lane] = bd;
        a.pid[slot + lane] = bid;
      }
      __syncthreads();  // every warp is done with this LUT
      if constexpr (REL) rel_segment_done(a, qs, s_ng);
    }
  }
#ifdef VLR_SCAN_TRACE
  if (threadIdx.x == 0 && c < 1024) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_scan_trace[c][0] = tr_start;
    g_scan_trace[c][1] = globaltimer_ns();
    g_scan_trace[c][2] = tr_lut;
    g_scan_trace[c][3] = tr_seg;
    g_scan_trace[c][4] = smid;
    g_scan_trace[c][5] = tr_grp;
  }
#endif
}

#ifdef VLR_SCAN_TRACE
extern "C" int vlr_debug_rel_trace(unsigned long long* out, int n, unsigned long long* misc) {
  const unsigned long long init[4] = {~0ull, 0ull, 0ull, 0ull};
  if (!out) return cudaMemcpyToSymbol(g_rel_misc, init, sizeof(init)) == cudaSuccess ? 0 : -1;  // reset
  if (cudaMemcpyFromSymbol(out, g_rel_trace, sizeof(unsigned long long) * 2 * (n < 4096 ? n : 4096)) != cudaSuccess)
    return -1;
  return cudaMemcpyFromSymbol(misc, g_rel_misc, sizeof(unsigned long long) * 4) == cudaSuccess ? 0 : -1;
}
extern "C" int vlr_debug_scan_trace(unsigned long long* out, int n) {
  return cudaMemcpyFromSymbol(out, g_scan_trace, sizeof(unsigned long long) * 6 * (n < 1024 ? n : 1024)) == cudaSuccess
             ? 0 : -1;
}
#endif

// VLR_SCAN_ALT=1: the plain / large-k scan alternates the segment order too (measured neutral at C4:
// 1.536-1.540 ms either way, profiles/r02/scan_trace_alt*_s.jsonl; default off)
static int scan_alt() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("VLR_SCAN_ALT");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v;
}

int scan_ctas(const DeviceIndex& ix) {
  (void)ix;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;  // at most one persistent CTA per SM (128 KB LUT + 16 warps); capi.cu may leave SMs free
}

template <int MP, int NB, int EXP, bool REL = false, bool DUMP = false>
static cudaError_t launch_scan_e(const ScanArgs& a, int n_cta, cudaStream_t s) {
  // the LUT of one query: ceil(MP / 64) slabs of 64 slots (8-bit slots: 64 KB each; MP 192 -> 192 KB)
  constexpr size_t kLutMax = (size_t)((MP + 63) / 64) * (NB == 8 ? kLutPairBytes : kLutPairBytes4);
  cudaError_t e = ensure_smem((const void*)k_scan<MP, NB, EXP, REL, DUMP>, kLutMax > 2 * kLutPairBytes ? kLutMax
                                                                                                  : (size_t)(2 * kLutPairBytes));
  if (e != cudaSuccess) return e;
  if (n_cta == 0) return cudaSuccess;  // configure (and so load) only
  return launch_pdl(k_scan<MP, NB, EXP, REL, DUMP>, dim3(n_cta), dim3(kScanThreads), (size_t)a.lut_bytes, s, a);
}

// VLR_SCAN_EXPERIMENT=1|2 (timing experiments only; results are wrong):
// 1 = no LUT gathers, 2 = no code loads.
static int scan_experiment() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("VLR_SCAN_EXPERIMENT");
    v = e ? atoi(e) : 0;
  }
  return v;
}

template <int MP, int NB>
static cudaError_t launch_scan_t(const ScanArgs& a, int n_cta, cudaStream_t s) {
  if (a.ready) return launch_scan_e<MP, NB, 0, true>(a, n_cta, s);
  if (a.dump) return launch_scan_e<MP, NB, 0, false, true>(a, n_cta, s);
  if constexpr (MP == 128 && NB == 8) {
    const int x = scan_experiment();
    if (x == 1) return launch_scan_e<MP, NB, 1>(a, n_cta, s);
    if (x == 2) return launch_scan_e<MP, NB, 2>(a, n_cta, s);
  }
  return launch_scan_e<MP, NB, 0>(a, n_cta, s);
}

static cudaError_t launch_scan_k(const DeviceIndex& ix, const ScanArgs& a, int n_cta, cudaStream_t s);

cudaError_t launch_scan(const DeviceIndex& ix, const Workspace& ws, int nq, int np, int k, cudaStream_t s,
                        const Release* rel) {
  if (nq <= 0) return cudaSuccess;
  ScanArgs a{nq, np, k, ix.npairs, (uint32_t)(ix.npairs * ix.lut_pair_bytes), ws.plocal, ws.term1, ws.item_off,
             ix.gbase, ix.codes, ix.bias, ix.ids, ws.lut, ws.pdist, ws.pid,
             nullptr, nullptr, 0u, nullptr, nullptr, 1, 0, nq, nullptr, scan_alt()};
  int G = ws.n_cta;
  if (rel) {
    if ((long long)ws.n_cta * kScanWarps > kMergeMaxLists || ws.n_cta < 2) return cudaErrorInvalidConfiguration;
    G = ws.n_cta - 1;  // one SM for the resident merger CTA
    a.qdone = ws.qdone;
    a.ready = rel->ready;
    a.epoch = rel->epoch;
    a.out_ids = rel->out_ids;
    a.out_dist = rel->out_dist;
    static int env_waves = -1;  // VLR_RELEASE_WAVES: experiment override of the wave count
    if (env_waves < 0) {
      const char* e = getenv("VLR_RELEASE_WAVES");
      env_waves = e ? atoi(e) : 0;
    }
    // the partial-list slots are sized for kMaxReleaseWaves waves (capi.cu ensure_ws): clamp the override
    const int zw = env_waves > 0 ? (env_waves < kMaxReleaseWaves ? env_waves : kMaxReleaseWaves) : kReleaseWaves;
    a.waves = nq < zw ? nq : zw;
    // Both kernels must be loaded before the fork: with lazy module loading, loading a kernel while the
    // spinning merger runs waits for the merger (and the merger waits for the scan).
    cudaError_t e = launch_scan_k(ix, a, 0, s);
    if (e != cudaSuccess) return e;
    if ((e = ensure_smem((const void*)k_release_merge, (size_t)a.nq)) != cudaSuccess) return e;
    if ((e = ensure_smem((const void*)k_release_rest, 0)) != cudaSuccess) return e;
#ifdef VLR_SCAN_TRACE
    k_stamp<<<1, 1, 0, s>>>(2);
#endif
    // fork: the merger CTA runs concurrently with the scan on a second stream, joined back before return
    e = cudaEventRecord(rel->fork, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(rel->stream, rel->fork, 0);
    if (e != cudaSuccess) return e;
    static int rel_exp = -1;  // VLR_REL_EXPERIMENT=1: the merger exits at once (timing experiment: nothing
    if (rel_exp < 0) {        // is released, the host waits time out)
      const char* e = getenv("VLR_REL_EXPERIMENT");
      rel_exp = e ? atoi(e) : 0;
    }
    ScanArgs am = a;
    if (rel_exp == 1) am.nq = 0;
    k_release_merge<<<1, kMergeMaxWarps * 32, (size_t)a.nq, rel->stream>>>(am, G, ws.status);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    e = launch_scan_k(ix, a, G, s);
    if (e == cudaSuccess && rel_exp != 1) {  // the stragglers, in parallel (claims settle merger vs rest)
      k_release_rest<<<(a.nq + 15) / 16, 512, 0, s>>>(a, G);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaEventRecord(rel->join, rel->stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, rel->join, 0);
#ifdef VLR_SCAN_TRACE
    k_stamp<<<1, 1, 0, s>>>(3);
#endif
    return e;
  }
  return launch_scan_k(ix, a, G, s);
}

static cudaError_t launch_scan_k(const DeviceIndex& ix, const ScanArgs& a, int n_cta, cudaStream_t s) {
  if (ix.code_bits == 4) {
    switch (ix.mpad) {
      case 32: return launch_scan_t<32, 4>(a, n_cta, s);
      case 64: return launch_scan_t<64, 4>(a, n_cta, s);
      case 96: return launch_scan_t<96, 4>(a, n_cta, s);
      case 128: return launch_scan_t<128, 4>(a, n_cta, s);
      case 192: return launch_scan_t<192, 4>(a, n_cta, s);
      case 256: return launch_scan_t<256, 4>(a, n_cta, s);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (ix.mpad) {
    case 32: return launch_scan_t<32, 8>(a, n_cta, s);
    case 64: return launch_scan_t<64, 8>(a, n_cta, s);
    case 96: return launch_scan_t<96, 8>(a, n_cta, s);
    case 128: return launch_scan_t<128, 8>(a, n_cta, s);
    case 160: return launch_scan_t<160, 8>(a, n_cta, s);  // 8-bit m <= 160, or 4-bit pair mode m <= 320
    case 192: return launch_scan_t<192, 8>(a, n_cta, s);  // 8-bit m <= 192, or 4-bit pair mode m <= 384 (PQ384x4)
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_rank_merge(const DeviceIndex& ix, const Workspace& ws, int nq, int np, int k, int64_t* out_ids,
                              float* out_dist, void* out_packed, cudaStream_t s, const PeerOut* po) {
  const PeerOut pout = po ? *po : PeerOut{};
  (void)ix;
  if (nq <= 0) return cudaSuccess;
  // expected lists per query: (scan CTAs spanned) x warps
  const long long lists = ((long long)ws.n_cta / nq + 2) * kScanWarps;
  int nw = 1;
  while (nw < kMergeMaxWarps && (long long)nw * 128 < lists) nw <<= 1;
  if ((long long)ws.n_cta * kScanWarps > kMergeMaxLists) return cudaErrorInvalidConfiguration;
  return launch_pdl(k_rank_merge, dim3(nq), dim3(nw * 32), 0, s, nq, np, k, ws.n_cta, ws.item_off, ws.pdist, ws.pid,
                    out_ids, out_dist, reinterpret_cast<Packed*>(out_packed), pout);
}

// ---------------------------------------------------------------- large k (k > 32)
// §8(b) allows k up to 1024; the warp-register top-k holds 32. For k > 32 the
// scan runs in DUMP mode (every candidate's (dist, vector position) written
// per group, 8 B per vector next to the 132 B of codes and bias it reads)
// over a chunk of queries, and k_select_large (one CTA per query) keeps the
// k smallest by (dist, id): a radix select of the k-th distance key over the
// query's candidates (4 passes of 8 bits), the entries below it, the entries
// equal to it in ascending id order up to k, then a bitonic sort by
// (dist, id). Same unique result as the warp top-k path.
constexpr int kSelLargeThreads = 1024;
constexpr int kSelLargeEqCap = 3072;  // entries equal to the k-th key held for the id tie-break

__device__ __forceinline__ bool lt_did(float d1, long long i1, float d2, long long i2) {
  return d1 < d2 || (d1 == d2 && i1 < i2);
}

__global__ void __launch_bounds__(kSelLargeThreads) k_select_large(
    int q_lo, int np, int k, const int64_t* __restrict__ item_off, const uint2* __restrict__ dump,
    const int64_t* __restrict__ ids, int64_t* __restrict__ out_ids, float* __restrict__ out_dist,
    Packed* __restrict__ packed) {
  pdl_entry();  // PDL: wait for the previous kernel in the stream, then let the next one launch
  __shared__ unsigned hist[256];
  __shared__ unsigned s_prefix, s_want, s_cnt, s_neq, s_valid;
  __shared__ float sd[kMaxKLarge];      // the kk <= 1024 selected entries (bitonic-sorted in place)
  __shared__ long long sid[kMaxKLarge];
  __shared__ long long seq[kSelLargeEqCap];
  const int q = q_lo + blockIdx.x;
  const long long WL = item_off[(long long)q_lo * np];  // the chunk's first group (the DUMP scan's base)
  const long long S = (item_off[(long long)q * np] - WL) * 32, E = (item_off[(long long)(q + 1) * np] - WL) * 32;
  const unsigned kInfKey = 0xFF800000u;  // fkey(+inf)
  if (threadIdx.x == 0) { s_valid = 0u; s_cnt = 0u; s_neq = 0u; }
  __syncthreads();
  unsigned nv = 0;
  for (long long i = S + threadIdx.x; i < E; i += blockDim.x) nv += fkey(__uint_as_float(dump[i].x)) < kInfKey;
  atomicAdd(&s_valid, nv);
  __syncthreads();
  const unsigned valid = s_valid;
  const int kk = (int)(valid < (unsigned)k ? valid : (unsigned)k);
  unsigned theta = kInfKey;
  if (kk > 0) {  // the kk-th smallest key among the finite ones
    unsigned prefix = 0u, mask = 0u, want = (unsigned)kk;
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0u;
      __syncthreads();
      for (long long i = S + threadIdx.x; i < E; i += blockDim.x) {
        const unsigned key = fkey(__uint_as_float(dump[i].x));
        if (key < kInfKey && (key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        unsigned c = 0;
        for (int b = 0; b < 256; ++b) {
          if (c + hist[b] >= want) { s_prefix = prefix | ((unsigned)b << shift); s_want = want - c; break; }
          c += hist[b];
        }
      }
      __syncthreads();
      prefix = s_prefix;
      want = s_want;
      mask |= 255u << shift;
      __syncthreads();
    }
    theta = prefix;
  }
  // entries below theta (fewer than kk of them) and the theta-equal ones (ids, for the tie-break)
  for (long long i = S + threadIdx.x; i < E; i += blockDim.x) {
    const uint2 e = dump[i];
    const unsigned key = fkey(__uint_as_float(e.x));
    if (kk == 0 || key > theta) continue;
    const long long id = __ldg(reinterpret_cast<const long long*>(ids) + e.y);
    if (key < theta) {
      const unsigned at = atomicAdd(&s_cnt, 1u);
      sd[at] = __uint_as_float(e.x);
      sid[at] = id;
    } else {
      const unsigned at = atomicAdd(&s_neq, 1u);
      if (at < (unsigned)kSelLargeEqCap) seq[at] = id;
    }
  }
  __syncthreads();
  const int nlt = (int)s_cnt;
  const int neq = (int)s_neq;
  const int need = kk - nlt;  // theta-equal entries to take, smallest ids first
  if (need > 0) {
    if (neq <= kSelLargeEqCap) {
      // rank of each equal id among the equal ids (ids are unique): the need smallest go in
      for (int j = threadIdx.x; j < neq; j += blockDim.x) {
        const long long v = seq[j];
        int r = 0;
        for (int t = 0; t < neq; ++t) r += seq[t] < v;
        if (r < need) {
          sd[nlt + r] = fkey_inv(theta);
          sid[nlt + r] = v;
        }
      }
    } else if (threadIdx.x == 0) {  // (pathological ties) repeated minimum over the equal entries
      long long last = -1;
      for (int r = 0; r < need; ++r) {
        long long best = LLONG_MAX;
        for (long long i = S; i < E; ++i) {
          const uint2 e = dump[i];
          if (fkey(__uint_as_float(e.x)) != theta) continue;
          const long long id = ids[e.y];
          if (id > last && id < best) best = id;
        }
        sd[nlt + r] = fkey_inv(theta);
        sid[nlt + r] = best;
        last = best;
      }
    }
  }
  __syncthreads();
  int n2 = 1;
  while (n2 < kk) n2 <<= 1;
  for (int j = kk + threadIdx.x; j < n2; j += blockDim.x) {
    sd[j] = CUDART_INF_F;
    sid[j] = LLONG_MAX;
  }
  for (int size = 2; size <= n2; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < (n2 >> 1); i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
        const bool up = (lo & size) == 0;
        const float da = sd[lo], db = sd[hi];
        const long long ia = sid[lo], ib = sid[hi];
        if (up ? lt_did(db, ib, da, ia) : lt_did(da, ia, db, ib)) {
          sd[lo] = db; sd[hi] = da;
          sid[lo] = ib; sid[hi] = ia;
        }
      }
    }
  __syncthreads();
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    const float dv = j < kk ? sd[j] : CUDART_INF_F;
    const long long iv = j < kk ? sid[j] : -1;
    if (packed) {
      Packed pk;
      pk.d = dv;
      pk.pad = 0;
      pk.id = iv;
      packed[(size_t)q * k + j] = pk;
    } else {
      out_ids[(size_t)q * k + j] = iv;
      out_dist[(size_t)q * k + j] = dv;
    }
  }
}

// the large-k path of one search: chunks of queries whose candidates fit ws.dump
cudaError_t launch_scan_large(const DeviceIndex& ix, const Workspace& ws, int nq, int np, int k, int64_t* out_ids,
                              float* out_dist, void* out_packed, cudaStream_t s) {
  if (nq <= 0) return cudaSuccess;
  const int qc = ws.dump_nq;  // queries per chunk (ensure_ws: chunk x max groups per query <= dump capacity)
  if (qc < 1) return cudaErrorInvalidConfiguration;
  for (int q0 = 0; q0 < nq; q0 += qc) {
    const int q1 = q0 + qc < nq ? q0 + qc : nq;
    ScanArgs a{nq, np, k, ix.npairs, (uint32_t)(ix.npairs * ix.lut_pair_bytes), ws.plocal, ws.term1, ws.item_off,
               ix.gbase, ix.codes, ix.bias, ix.ids, ws.lut, ws.pdist, ws.pid,
               nullptr, nullptr, 0u, nullptr, nullptr, 1, q0, q1, ws.dump, scan_alt()};
    cudaError_t e = launch_scan_k(ix, a, ws.n_cta, s);
    if (e != cudaSuccess) return e;
    e = launch_pdl(k_select_large, dim3(q1 - q0), dim3(kSelLargeThreads), 0, s, q0, np, k, ws.item_off, ws.dump,
                   ix.ids, out_ids, out_dist, reinterpret_cast<Packed*>(out_packed));
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// ---------------------------------------------------------------- K8 shard merge
// parts [S][nq][k]: top-k of the union per query.
__global__ void k_merge_parts(int n_shards, int nq, int k, const Packed* __restrict__ packed,
                              const int64_t* __restrict__ pids, const float* __restrict__ pdist,
                              int64_t* __restrict__ out_ids, float* __restrict__ out_dist, PeerIn pin) {
  pdl_entry();  // PDL: wait for the previous kernel in the stream, then let the next one launch
  peer_wait(pin);  // NVLink peer exchange: every rank's partial rows have landed in this rank's inbox
  const int lane = threadIdx.x & 31;
  const int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q >= nq) return;
  float bd = CUDART_INF_F;
  long long bid = -1;
  warp_select_merge<4>(bd, bid, k, lane, n_shards * k, [&](int i, float& d, long long& id) {
    const size_t o = ((size_t)(i / k) * nq + q) * k + (i % k);
    if (packed) {
      const Packed p = packed[o];
      d = p.d;
      id = p.id;
    } else {
      d = pdist[o];
      id = pids[o];
    }
  });
  if (lane < k) {
    out_ids[(size_t)q * k + lane] = bid;
    out_dist[(size_t)q * k + lane] = bd;
  }
}

// K8 for k > 32: one CTA per query sorts the n_shards * k gathered entries by
// (dist, id) in shared memory (bitonic) and keeps the k smallest.
constexpr int kMergeLargeCap = 8192;  // n_shards * k (checked by the callers)
__global__ void __launch_bounds__(1024) k_merge_large(int n_shards, int nq, int k, const Packed* __restrict__ packed,
                                                      const int64_t* __restrict__ pids,
                                                      const float* __restrict__ pdist, int64_t* __restrict__ out_ids,
                                                      float* __restrict__ out_dist) {
  pdl_entry();  // PDL: wait for the previous kernel in the stream, then let the next one launch
  extern __shared__ __align__(16) unsigned char smm[];
  const int n = n_shards * k;
  int n2 = 1;
  while (n2 < n) n2 <<= 1;
  long long* sid = reinterpret_cast<long long*>(smm);
  float* sd = reinterpret_cast<float*>(sid + n2);
  const int q = blockIdx.x;
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    float dv = CUDART_INF_F;
    long long iv = LLONG_MAX;
    if (i < n) {
      const size_t o = ((size_t)(i / k) * nq + q) * k + (i % k);
      if (packed) { dv = packed[o].d; iv = packed[o].id; }
      else { dv = pdist[o]; iv = pids[o]; }
      if (iv < 0) iv = LLONG_MAX;  // padding sorts last
    }
    sd[i] = dv;
    sid[i] = iv;
  }
  for (int size = 2; size <= n2; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < (n2 >> 1); i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
        const bool up = (lo & size) == 0;
        const float da = sd[lo], db = sd[hi];
        const long long ia = sid[lo], ib = sid[hi];
        if (up ? lt_did(db, ib, da, ia) : lt_did(da, ia, db, ib)) {
          sd[lo] = db; sd[hi] = da;
          sid[lo] = ib; sid[hi] = ia;
        }
      }
    }
  __syncthreads();
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    const bool pad = sid[j] == LLONG_MAX;
    out_ids[(size_t)q * k + j] = pad ? -1 : sid[j];
    out_dist[(size_t)q * k + j] = pad ? CUDART_INF_F : sd[j];
  }
}

static cudaError_t launch_merge_large(const Packed* packed, const int64_t* pids, const float* pdist, int n_shards,
                                      int nq, int k, int64_t* out_ids, float* out_dist, cudaStream_t s) {
  const int n = n_shards * k;
  if (n > kMergeLargeCap) return cudaErrorInvalidValue;
  int n2 = 1;
  while (n2 < n) n2 <<= 1;
  const size_t sm = (size_t)n2 * (sizeof(long long) + sizeof(float));
  cudaError_t e = ensure_smem((const void*)k_merge_large, sm);
  if (e != cudaSuccess) return e;
  return launch_pdl(k_merge_large, dim3(nq), dim3(1024), sm, s, n_shards, nq, k, packed, pids, pdist, out_ids, out_dist);
}

cudaError_t launch_merge_packed(const void* parts, int n_shards, int nq, int k, int64_t* out_ids, float* out_dist,
                                cudaStream_t s, const PeerIn* pi) {
  const PeerIn pin = pi ? *pi : PeerIn{};
  if (nq <= 0) return cudaSuccess;
  if (k > kMaxK)
    return launch_merge_large(reinterpret_cast<const Packed*>(parts), nullptr, nullptr, n_shards, nq, k, out_ids,
                              out_dist, s);
  const int wpb = 8;
  return launch_pdl(k_merge_parts, dim3((nq + wpb - 1) / wpb), dim3(wpb * 32), 0, s, n_shards, nq, k,
                    reinterpret_cast<const Packed*>(parts), nullptr, nullptr, out_ids, out_dist, pin);
}

cudaError_t launch_merge_split(const int64_t* part_ids, const float* part_dist, int n_shards, int nq, int k,
                               int64_t* out_ids, float* out_dist, cudaStream_t s) {
  if (nq <= 0) return cudaSuccess;
  if (k > kMaxK) return launch_merge_large(nullptr, part_ids, part_dist, n_shards, nq, k, out_ids, out_dist, s);
  const int wpb = 8;
  return launch_pdl(k_merge_parts, dim3((nq + wpb - 1) / wpb), dim3(wpb * 32), 0, s, n_shards, nq, k, nullptr,
                    part_ids, part_dist, out_ids, out_dist, PeerIn{});
}

}  // namespace vlr

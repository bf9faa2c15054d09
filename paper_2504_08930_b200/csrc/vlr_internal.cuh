// vlr_internal.cuh -- shared declarations of libvlr.so (product path).
// No code here is shared with oracle/ (test infrastructure).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <utility>
#include <string>
#include <vector>

#include "vlr.h"
#include "vlr_device.cuh"

namespace vlr {

// ---------------------------------------------------------------- constants
constexpr int kWarp = 32;
constexpr int kMaxK = 32;          // warp-register top-k (one entry per lane)
constexpr int kMaxKLarge = 1024;   // k > 32: DUMP scan + per-query radix select (k_select_large), §8(b)
constexpr size_t kDumpBudget = (size_t)1 << 30;  // bytes of the large-k candidate buffer (queries chunked to fit)
constexpr int kMaxM = 192;         // max sub-quantizers, 8-bit codes (scan instantiations up to 192 slots)
constexpr int kMaxM4 = 384;        // max sub-quantizers, 4-bit codes (pair mode: 192 byte slots; PQ384x4)
#ifndef VLR_SCAN_THREADS
#define VLR_SCAN_THREADS 512
#endif
constexpr int kScanThreads = VLR_SCAN_THREADS;  // 16 warps per scan CTA (tuning variants: tools/variants.py)
constexpr int kScanWarps = kScanThreads / kWarp;
constexpr int kCandCap = 8192;     // K2 candidate list capacity per query (overflow -> rescan)
constexpr int kRefineChunk = 1024; // K3 candidates per exact-refine flush
constexpr int kReleaseWaves = 1;      // NEXT-4: default query waves of the release-mode scan (the
                                      // alternating segment order replaces waves, VLR_RELEASE_WAVES keeps them)
constexpr int kMaxReleaseWaves = 16;  // upper bound (VLR_RELEASE_WAVES is clamped to it; sizes the partial slots)
constexpr int kMaxNprobe = 2048;   // cap on nprobe' (K3 sort buffer; the paper's operating point)
constexpr int kMaxWorldProbes = 16384;  // world x nprobe' cap of the sharded coarse stage (K2 stage-2 select)
constexpr int kLutPairBytes = 256 * 64 * 4;  // one [256 codes][64 sub-spaces] fp32 slab (8-bit codes)
constexpr int kLutPairBytes4 = 16 * 64 * 4;  // one [16 codes][64 sub-spaces] fp32 slab (4-bit codes)

// ---------------------------------------------------------------- errors
struct Error {
  vlr_status st;
  std::string msg;
};
void set_error(const std::string& msg);

#define VLR_CUDA_TRY(expr)                                                              \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess) {                                                            \
      ::vlr::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));             \
      return _e == cudaErrorMemoryAllocation ? VLR_ERR_OOM : VLR_ERR_CUDA;              \
    }                                                                                   \
  } while (0)

// ---------------------------------------------------------------- device data
// one exact coarse candidate exchanged between ranks by the centroid-sharded
// coarse stage: fp64 key D (O2), cluster id l (-1 = padding, D = +inf)
struct __align__(16) CoarseEntry {
  double D;
  int32_t l;
  int32_t pad;
};

// K2 / K3b modes (k_coarse.cu)
constexpr int kSelFull = 0, kSelStage1 = 1, kSelStage2 = 2;
constexpr int kRefRoute = 0, kRefLocal = 1, kRefMerge = 2;

struct DeviceIndex {
  int d = 0, d8 = 0, nlist = 0, m = 0, mpad = 0, npairs = 0, dsub = 0;
  int nbits = 8, ksub = 256;   // bits per sub-code (8, or 4: nibble-packed) and codewords per sub-space
  int lut_pair_bytes = kLutPairBytes;  // LUT bytes per 64 code slots (256 or 16 codes x 64 x 4)
  // scan code slots: 8-bit codes and 4-bit PAIR mode (default for nbits 4: one slot = one packed byte =
  // two sub-codes, looked up in a 256-entry pair table, DESIGN.md §K6 4-bit) have code_bits 8; the
  // nibble mode (VLR_PQ4_NIBBLE=1 at load) has code_bits 4, one slot per sub-code
  int code_bits = 8, code_m = 0;
  int rank = 0, world = 1, device = 0;
  int metric = 0;              // 0 squared L2, 1 inner product (distance = -<q, x>)
  int by_residual = 1;         // 1: codes encode x - c_l
  bool shard_only = false;
  // centroid-sharded coarse stage (world > 1): this rank filters centroids [c_lo, c_hi)
  // (whole 128-centroid K1 tiles, dealt contiguously); world == 1: [0, nlist)
  int c_lo = 0, c_hi = 0;
  bool coarse_sharded = false;  // the NCCL search runs the sharded coarse stage (VLR_COARSE_REPLICATED=1: off)
  // replicated, coarse quantizer
  float* centroids = nullptr;  // [nlist][d]
  float* cnorm2 = nullptr;     // [nlist] ||c||^2 (fp64 -> fp32); zeros for metric 1 (filter = -2<q,c>)
  uint16_t* cf16 = nullptr;    // [nlist][d8] fp16(c * 2^c_exp) (RN), zero-padded to d8 (filter operand A)
  uint16_t* cf16t = nullptr;   // [ceil(nlist/128)][ceil(d8/64)][128][64] the same, tiled + SW128-swizzled (K1 A loads)
  int c_exp = 0;               // power-of-two centroid scale: max |c * 2^c_exp| < 2^14
  float c_inv = 1.f;           // 2^-c_exp
  alignas(64) unsigned char tmapA[128] = {};  // CUtensorMap of cf16 (box 64 x 128, SWIZZLE_128B)
  alignas(64) unsigned char tmapAt[128] = {}; // CUtensorMap of cf16t as [tiles*kblocks*128][64] (box 64 x 128, pre-swizzled)
  float cmax = 0.f;            // max ||c|| (host), for the filter band
  float* codebooks = nullptr;  // [m][ksub][dsub]
  int32_t* owner = nullptr;    // [nlist] owner rank or -1 (mapping table)
  int32_t* local = nullptr;    // [nlist] local list index on this rank or -1
  std::vector<int32_t> owner_h;
  // this rank's resident lists (lane-interleaved groups of 32 vectors)
  int32_t n_local = 0;
  int64_t n_groups = 0, n_vec = 0;
  int64_t* gbase = nullptr;    // [n_local+1] first group of each local list
  uint8_t* codes = nullptr;    // [n_groups][mpad*code_bits/128 chunks][32 lanes][16 B], per-lane rotated
  float* bias = nullptr;       // [n_groups*32] b_i = ||yhat||^2 + 2<c_l, yhat> (+inf for padding)
  int64_t* ids = nullptr;      // [n_groups*32] (-1 for padding)
  int64_t bytes = 0;
  std::vector<int64_t> top_groups;  // [i] = groups of the i largest local lists (large-k buffer bound)
  void* nccl = nullptr;        // ncclComm_t
};

struct Workspace {
  int cap_nq = 0, cap_np = 0, cap_k = 0;
  int n_cta_cap = 0;           // SM count: the partial-list slots are sized for a grid this large
  int n_cta = 0;               // the current search's scan grid (n_cta_cap - the handle's scan reserve)
  float* qnorm = nullptr;      // [nq] ||q|| (fp32, rounded up; filter band)
  float* qsq = nullptr;        // [nq] ||q||^2 (fp64 sum -> fp32; term1 of L2 with by_residual = 0)
  uint16_t* qf16 = nullptr;    // [nq][d8] fp16(q * 2^e_q) (RN), zero-padded (filter operand B)
  uint16_t* qf16t = nullptr;   // the same pre-tiled for one-copy B loads (k_qprep): [ceil(nq/512)*512][kb*64]
  float* qinv = nullptr;       // [nq] 2^-e_q
  float* dt = nullptr;         // [nq][nlist] filter distances ||c||^2 - 2<q,c>
  float* gmin = nullptr;       // [nq][ceil(nlist/32)] min of dt over each 32-centroid group
  int32_t* cand = nullptr;     // [nq][kCandCap]
  int32_t* ncand = nullptr;    // [nq]
  double* exact = nullptr;     // [nq][kCandCap] exact fp64 D of listed candidates (K3a)
  float* x1 = nullptr;         // [nq][np] sharded coarse stage 1: this rank's np smallest group minima
  float* x1_all = nullptr;     // [world][nq][np] gathered x1 (rank order)
  CoarseEntry* x2 = nullptr;   // [nq][np] stage 2: this rank's sorted top-np exact (D, l)
  CoarseEntry* x2_all = nullptr;  // [world][nq][np] gathered x2
  float* bound = nullptr;      // [nq] candidate bound theta~ + 2 Delta*
  int32_t* probes = nullptr;   // [nq][np]
  float* term1 = nullptr;      // [nq][np] query-dependent constant of probe p (fp64 -> fp32): ||q - c_l||^2
                               // (L2), -<q, c_l> (IP), ||q||^2 (L2, by_residual 0), 0 (IP, by_residual 0)
  int32_t* plocal = nullptr;   // [nq][np] local list or -1
  int64_t* item_off = nullptr; // [nq*np + 1] group prefix of owned work items
  int64_t* item_local = nullptr; // [nq*np] within-query group prefix
  int64_t* qtot = nullptr;     // [nq] groups owned per query
  unsigned long long* qdone = nullptr;  // [nq] groups scanned per query (NEXT-4 release counters)
  float* lut = nullptr;        // [nq][npairs][ksub][64]
  float* pdist = nullptr;      // [(n_cta + nq) * warps * k] scan partials
  int64_t* pid = nullptr;
  uint2* dump = nullptr;       // large k: [dump_nq x max groups per query x 32] (dist bits, vector position)
  int dump_nq = 0;             // queries per large-k chunk
  void* send = nullptr;        // [nq][k] 16-byte entries (world > 1)
  void* recv = nullptr;        // [world][nq][k]
  float* h_stage = nullptr;    // pinned staging for vlr_search_host (queries)
  float* d_q = nullptr;        // device queries for vlr_search_host (two buffers: d_q, d_q2, used in turn so the
  float* d_q2 = nullptr;       // H2D copy of the next batch overlaps this one's kernels)
  int64_t* d_ids = nullptr;
  float* d_dist = nullptr;
  uint8_t* d_miss = nullptr;
  int32_t* d_probes = nullptr;
  int32_t* status = nullptr;   // device status word (bit0: non-finite query)
  int32_t* h_status = nullptr; // pinned mirror
};

}  // namespace vlr

struct vlr_index {
  vlr::DeviceIndex ix;
  // Workspace slots (cross-batch pipelining): search number i uses slot i % nslots; a
  // search waits (stream event) for the previous user of its slot before it writes the slot, so two
  // searches enqueued on different streams overlap on the device (batch i+1's coarse stage beside batch
  // i's scan). nslots = 1 (default): one workspace, every search is ordered by its stream alone.
  static constexpr int kSlots = 2;
  vlr::Workspace wsl[kSlots];
  struct SlotRes {
    cudaEvent_t done = nullptr;   // recorded at the end of the slot's last search
    bool pending = false;         // `done` was recorded and not yet waited for by a later user
    // K5 side stream: the LUT depends only on Q (residual decomposition), so it runs beside
    // K2-K4 (latency-bound, few CTAs) and joins before the scan
    cudaStream_t lut_stream = nullptr;
    cudaEvent_t lut_fork = nullptr, lut_join = nullptr;
    // NEXT-4 merger stream + fork/join events (created on first use)
    cudaStream_t rel_stream = nullptr;
    cudaEvent_t rel_fork = nullptr, rel_join = nullptr;
    // vlr_search_host*: query staging buffer i (d_q / d_q2) filled on h2d_stream (q_ready[i]) and free again
    // once its search has read it (q_free[i], recorded on the search stream)
    cudaEvent_t q_ready[2] = {}, q_free[2] = {};
    bool q_used[2] = {};
    int qbuf = 0;
  } res[kSlots];
  cudaStream_t h2d_stream = nullptr;  // host -> device query copies of vlr_search_host* (overlap the search)
  int nslots = 1;
  int scan_reserve = 0;      // SMs the scan's persistent grid leaves free (vlr_set_pipeline)
  uint64_t seq = 0;          // searches started (slot = seq % nslots)
  int profiling = 0;  // 0 off, 1 every stage, 2 scan only
  static constexpr int kRing = 64;
  cudaEvent_t ev[kRing][9] = {};
  int prof_mode[kRing] = {};
  int64_t nsearch = 0;       // searches recorded while profiling
  int launches = 0;
  bool dead = false;  // NCCL failure
  // NVLink peer exchange (vlr_p2p_*): every rank's inbox IPC-mapped here; one region per
  // workspace slot (two searches in flight exchange through different regions)
  struct PeerLink {
    bool on = false;
    int cap_nq = 0, cap_np = 0, cap_k = 0, G = 0, nslots = 1;
    void* inbox = nullptr;                    // own inbox (cudaMalloc base, exported with cudaIpcGetMemHandle)
    size_t bytes = 0, slot_bytes = 0, off_x1 = 0, off_x2 = 0, off_res = 0, off_flags = 0;  // offsets within a slot
    void* peer[vlr::kMaxWorld] = {};          // every rank's inbox base (own = inbox; others IPC-opened)
    int* ctr = nullptr;                       // [nslots][3] CTA-completion counters
    uint32_t epoch = 0;
  } p2p;
  std::mutex mu;  // held while a search is enqueued and while vlr_update_hot swaps the residency
  int lut_side = -1;  // -1 unset; 0 serial (VLR_LUT_SERIAL=1, A/B timing), 1 forked
  int stage = 0, stage_nq = 0, stage_np = 0, stage_slot = 0;  // staged search progress (vlr_coarse_stage1/2, vlr_search_stage3)
  std::string last_err;
};

namespace vlr {

// ---------------------------------------------------------------- launches with programmatic dependence
// The search chain (qprep, K1, K2, K3a, K3b, K4b, K6, K7, K8) is launched with the programmatic stream
// serialization attribute: a kernel's CTAs launch while its predecessor finishes, and wait at
// griddepcontrol.wait (pdl_entry, vlr_device.cuh) for its completion -- the launch latency between two
// dependent kernels overlaps the predecessor's tail. VLR_PDL=0: ordinary launches (A/B timing).
bool pdl_on();  // VLR_PDL != 0 and the current search allows it (pdl_for_search)
// PDL is used only without cross-batch pipelining: an early-launched CTA waiting at griddepcontrol.wait
// holds SM slots the other stream's batch would use (measured at G = 8, pipelined: 0.369 -> 0.403 ms)
void pdl_for_search(bool allow);
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
inline cudaError_t launch_pdl_c(const void* kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t s, void** args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  return cudaLaunchKernelExC(&cfg, kernel, args);
}

// Per-(device, kernel) launch configuration: raises the kernel's dynamic shared-memory limit to at
// least `bytes` on the CURRENT device (the attribute is per device context) and forces its module to be
// loaded (cudaFuncGetAttributes); cached, thread-safe. Every launcher calls it before a launch.
cudaError_t ensure_smem(const void* fn, size_t bytes);

// ---------------------------------------------------------------- launchers
// K0 layout (load time)
cudaError_t launch_layout(const DeviceIndex& ix, const uint8_t* stage_codes, const int64_t* stage_ids,
                          const int64_t* vbase, const int32_t* lglob, cudaStream_t s);
// stage 0..2 coarse quantizer
cudaError_t launch_qprep(const float* Q, int nq, int d, int d8, float* qnorm, float* qsq, uint16_t* qf16, float* qinv,
                         int32_t* status, uint16_t* qf16t, int QT, cudaStream_t s);
// K1's query tile (rows of B per CTA): the pre-tiled operand written by qprep uses it; 0 = K1 reads the
// row-major fp16 queries through a tensor map (VLR_FILTER_BTILED=0, or the pair / persistent kernels)
int filter_btile_rows(int nq, int tiles);
// K1 over centroid tiles [t_lo, t_hi) (128 centroids each): dt columns and gmin groups of those tiles
cudaError_t launch_filter_tc(const uint16_t* Qh, const float* qinv, int nq, const DeviceIndex& ix, int t_lo, int t_hi,
                             float* dt, float* gmin, const uint16_t* Qt, cudaStream_t s);
cudaError_t launch_round_f16(const float* src, int rows, int d, int d8, float scale, uint16_t* dst, cudaStream_t s);
cudaError_t make_tmap_2d(void* map, const uint16_t* base, int rows, int cols, int box_rows, bool swizzle);
cudaError_t launch_tile_f16(const DeviceIndex& ix, cudaStream_t s);
cudaError_t launch_select(const DeviceIndex& ix, const Workspace& ws, int nq, int np, float e_dot, int mode,
                          cudaStream_t s, const PeerOut* po = nullptr, const PeerIn* pi = nullptr);
cudaError_t launch_exact(const float* Q, const DeviceIndex& ix, const Workspace& ws, int nq, cudaStream_t s);
cudaError_t launch_refine(const float* Q, const DeviceIndex& ix, const Workspace& ws, int nq, int np, uint8_t* miss,
                          int32_t* probes_out, int mode, cudaStream_t s, const PeerOut* po = nullptr,
                          const PeerIn* pi = nullptr);
// stage 3..4
cudaError_t launch_offsets(const DeviceIndex& ix, const Workspace& ws, int nq, int np, cudaStream_t s);
cudaError_t launch_lut(const float* Q, const DeviceIndex& ix, const Workspace& ws, int nq, cudaStream_t s);
cudaError_t launch_access_hist(const int32_t* probes, long long n, int nlist, unsigned long long* counts,
                               cudaStream_t s);
// stage 5..7
int scan_ctas(const DeviceIndex& ix);
struct Release {               // NEXT-4 early per-query release (vlr_search_release_async)
  uint32_t* ready;
  uint32_t epoch;
  int64_t* out_ids;
  float* out_dist;
  cudaStream_t stream;         // the merger CTA's stream (forked from / joined to the search stream; set per
  cudaEvent_t fork, join;      // workspace slot by the search)
};
cudaError_t launch_scan(const DeviceIndex& ix, const Workspace& ws, int nq, int np, int k, cudaStream_t s,
                        const Release* rel = nullptr);
cudaError_t launch_rank_merge(const DeviceIndex& ix, const Workspace& ws, int nq, int np, int k,
                              int64_t* out_ids, float* out_dist, void* out_packed, cudaStream_t s,
                              const PeerOut* po = nullptr);
cudaError_t launch_scan_large(const DeviceIndex& ix, const Workspace& ws, int nq, int np, int k, int64_t* out_ids,
                              float* out_dist, void* out_packed, cudaStream_t s);
cudaError_t launch_merge_packed(const void* parts, int n_shards, int nq, int k, int64_t* out_ids, float* out_dist,
                                cudaStream_t s, const PeerIn* pi = nullptr);
cudaError_t launch_merge_split(const int64_t* part_ids, const float* part_dist, int n_shards, int nq, int k,
                               int64_t* out_ids, float* out_dist, cudaStream_t s);

}  // namespace vlr

// capi.cu -- the C ABI of libvlr.so (include/vlr.h): index residency, the
// search pipeline (stream-ordered launches of K1..K8), NCCL exchange.
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <ctime>
#include <limits>
#include <map>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cub/device/device_radix_sort.cuh>
#include <numeric>
#include <thread>
#include <string>
#include <vector>

#include "vlr_device.cuh"
#include "vlr_internal.cuh"

namespace vlr {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

cudaError_t ensure_smem(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;  // (device, kernel) -> configured bytes
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find({dev, fn});
  if (it != done.end() && it->second >= bytes) return cudaSuccess;
  if (bytes > 48 * 1024) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
  }
  cudaFuncAttributes fa;  // forces the (lazy) module load now, not inside a later fork/spin
  if ((e = cudaFuncGetAttributes(&fa, fn)) != cudaSuccess) return e;
  done[{dev, fn}] = std::max(bytes, it != done.end() ? it->second : (size_t)0);
  return cudaSuccess;
}

static thread_local bool g_pdl_search = true;
void pdl_for_search(bool allow) { g_pdl_search = allow; }
bool pdl_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("VLR_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1 && g_pdl_search;
}

static vlr_status fail(vlr_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

// relative bound on the filter's dot-product error (DESIGN.md §5 band proof):
// operands scaled by powers of two and rounded to fp16 (RN, 11-bit significand:
// relative error <= 2^-11 each for normal results; the subnormal-flush term is
// added by the caller's band), products exact in fp32, fp32
// accumulation over d terms in the tensor core bounded conservatively by
// d * 2^-23 (order and rounding mode unspecified).
static float filter_edot(int d) { return 2.0f * 4.8828125e-4f + 2.3841858e-7f + 1.01f * (float)d * 1.1920929e-7f; }

// NVTX ranges per pipeline stage (host-side enqueue spans; with nsys/ncu
// --nvtx they label the K-stages). On when VLR_NVTX=1 or profiling is on.
static bool nvtx_on(const vlr_index* h) {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("VLR_NVTX");
    env = (e && e[0] == '1') ? 1 : 0;
  }
  return env == 1 || h->profiling != 0;
}
struct NvtxRange {
  bool on;
  NvtxRange(const vlr_index* h, const char* name) : on(nvtx_on(h)) {
    if (on) nvtxRangePushA(name);
  }
  ~NvtxRange() {
    if (on) nvtxRangePop();
  }
};

template <class T>
static cudaError_t dalloc(T** p, size_t n) {
  *p = nullptr;
  if (n == 0) n = 1;
  return cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T));
}

__global__ void k_adjacent_dup(const int64_t* sorted, long long n, int32_t* flag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x + 1; i < n; i += (long long)gridDim.x * blockDim.x)
    if (sorted[i] == sorted[i - 1]) atomicOr(flag, 1);
}
__global__ void k_negative(const int64_t* ids, long long n, int32_t* flag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    if (ids[i] < 0) atomicOr(flag, 2);
}

static void free_ws(Workspace& w) {
  void* ps[] = {w.qnorm, w.qsq, w.qf16, w.qf16t, w.qinv, w.dt, w.gmin, w.cand, w.ncand, w.exact, w.x1, w.x1_all, w.x2, w.x2_all, w.dump, w.bound, w.probes, w.term1, w.plocal, w.item_off, w.item_local, w.qtot, w.qdone, w.lut,
                w.pdist, w.pid, w.send, w.recv, w.d_q, w.d_q2, w.d_ids, w.d_dist, w.d_miss, w.d_probes, w.status};
  for (void* p : ps)
    if (p) cudaFree(p);
  if (w.h_status) cudaFreeHost(w.h_status);
  w = Workspace{};
}

static void free_index(DeviceIndex& ix) {
  void* ps[] = {ix.centroids, ix.cf16, ix.cf16t, ix.cnorm2, ix.codebooks, ix.owner, ix.local, ix.gbase, ix.codes, ix.bias, ix.ids};
  for (void* p : ps)
    if (p) cudaFree(p);
  if (ix.nccl) ncclCommDestroy(reinterpret_cast<ncclComm_t>(ix.nccl));
  ix = DeviceIndex{};
}

static vlr_status ensure_ws(vlr_index* h, int slot, int nq, int np, int k) {
  Workspace& w = h->wsl[slot];
  const DeviceIndex& ix = h->ix;
  if (w.status && nq <= w.cap_nq && np <= w.cap_np && k <= w.cap_k) return VLR_OK;
  if (h->p2p.on) return fail(VLR_ERR_UNSUPPORTED, "peer exchange connected: batch beyond the reserved workspace");
  const int cnq = std::max(nq, w.cap_nq), cnp = std::max(np, w.cap_np), ck = std::max(k, w.cap_k);
  int32_t status_keep = 0;
  if (w.h_status) status_keep = *w.h_status;
  VLR_CUDA_TRY(cudaDeviceSynchronize());
  free_ws(w);
  w.cap_nq = cnq;
  w.cap_np = cnp;
  w.cap_k = ck;
  w.n_cta_cap = scan_ctas(ix);
  w.n_cta = w.n_cta_cap;
  const size_t nqs = (size_t)cnq;
  VLR_CUDA_TRY(dalloc(&w.qnorm, nqs));
  VLR_CUDA_TRY(dalloc(&w.qsq, nqs));
  VLR_CUDA_TRY(dalloc(&w.qf16, nqs * ix.d8));
  VLR_CUDA_TRY(dalloc(&w.qf16t, (size_t)((cnq + 511) / 512 * 512) * ((ix.d8 + 63) / 64 * 64)));
  VLR_CUDA_TRY(dalloc(&w.qinv, nqs));
  VLR_CUDA_TRY(dalloc(&w.dt, nqs * ix.nlist));
  VLR_CUDA_TRY(dalloc(&w.gmin, nqs * ((ix.nlist + 31) / 32)));
  VLR_CUDA_TRY(dalloc(&w.cand, nqs * kCandCap));
  VLR_CUDA_TRY(dalloc(&w.ncand, nqs));
  VLR_CUDA_TRY(dalloc(&w.exact, nqs * kCandCap));
  VLR_CUDA_TRY(dalloc(&w.x1, nqs * cnp));
  VLR_CUDA_TRY(dalloc(&w.x2, nqs * cnp));
  if (ix.world > 1 || ix.nccl) {  // gathered coarse-stage buffers (NCCL or the caller's transport, vlr_coarse_stage*)
    VLR_CUDA_TRY(dalloc(&w.x1_all, nqs * cnp * ix.world));
    VLR_CUDA_TRY(dalloc(&w.x2_all, nqs * cnp * ix.world));
  }
  VLR_CUDA_TRY(dalloc(&w.bound, nqs));
  VLR_CUDA_TRY(dalloc(&w.probes, nqs * cnp));
  VLR_CUDA_TRY(dalloc(&w.term1, nqs * cnp));
  VLR_CUDA_TRY(dalloc(&w.plocal, nqs * cnp));
  VLR_CUDA_TRY(dalloc(&w.item_off, nqs * cnp + 1));
  VLR_CUDA_TRY(dalloc(&w.item_local, nqs * cnp));
  VLR_CUDA_TRY(dalloc(&w.qtot, nqs));
  VLR_CUDA_TRY(dalloc(&w.qdone, nqs));
  VLR_CUDA_TRY(dalloc(&w.lut, nqs * ix.npairs * (ix.lut_pair_bytes / 4)));
  // warp partial lists (k <= 32 path only): slot (c + q + wave * n_cta)
  const size_t nslots = ((size_t)w.n_cta_cap * kMaxReleaseWaves + nqs) * kScanWarps * std::min(ck, kMaxK);
  VLR_CUDA_TRY(dalloc(&w.pdist, nslots));
  if (ck > kMaxK) {  // large-k candidate buffer: chunks of dump_nq queries x (groups of the np largest lists)
    const int64_t maxg = ix.top_groups[std::min<size_t>((size_t)cnp, ix.top_groups.size() - 1)];
    const size_t per_q = (size_t)std::max<int64_t>(maxg, 1) * 32 * sizeof(uint2);
    w.dump_nq = (int)std::max<size_t>(1, std::min<size_t>((size_t)cnq, kDumpBudget / per_q));
    VLR_CUDA_TRY(dalloc(&w.dump, (size_t)w.dump_nq * per_q / sizeof(uint2)));
  }
  VLR_CUDA_TRY(dalloc(&w.pid, nslots));
  if (ix.nccl) {  // exchange buffers (world > 1 with a communicator, or the forced 1-rank exchange)
    VLR_CUDA_TRY(dalloc(reinterpret_cast<Packed**>(&w.send), nqs * ck));
    VLR_CUDA_TRY(dalloc(reinterpret_cast<Packed**>(&w.recv), nqs * ck * ix.world));
  }
  VLR_CUDA_TRY(dalloc(&w.d_q, nqs * ix.d));
  VLR_CUDA_TRY(dalloc(&w.d_q2, nqs * ix.d));
  VLR_CUDA_TRY(dalloc(&w.d_ids, nqs * ck));
  VLR_CUDA_TRY(dalloc(&w.d_dist, nqs * ck));
  VLR_CUDA_TRY(dalloc(&w.d_miss, nqs * cnp));
  VLR_CUDA_TRY(dalloc(&w.d_probes, nqs * cnp));
  VLR_CUDA_TRY(dalloc(&w.status, 1));
  VLR_CUDA_TRY(cudaMemset(w.status, 0, sizeof(int32_t)));
  VLR_CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&w.h_status), sizeof(int32_t)));
  *w.h_status = status_keep;
  return VLR_OK;
}

// Index splitter. Without counts: the paper's deal -- hot lists
// sorted by size descending (ties: ascending cluster id), dealt round-robin
// over ranks. With counts (NEXT-2 traffic-aware deal):
// load_l = size_l * (count_l + 1) (the vectors a rank scans for list l per
// profiled stream, Laplace-smoothed), lists sorted by load descending (ties: size descending, then id),
// each given to the rank with the least load so far (ties: lowest rank) --
// greedy LPT, which bounds the max rank load by 4/3 of the optimum.
static void deal(const int64_t* offs, const int64_t* counts, const int32_t* hot, int32_t n_hot, int32_t world,
                 int32_t* out_owner) {
  std::vector<int32_t> ord((size_t)n_hot);
  std::iota(ord.begin(), ord.end(), 0);
  auto size = [&](int32_t i) { return offs[hot[i] + 1] - offs[hot[i]]; };
  if (!counts) {
    std::sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) {
      return size(a) != size(b) ? size(a) > size(b) : hot[a] < hot[b];
    });
    for (size_t r = 0; r < ord.size(); ++r) out_owner[ord[r]] = (int32_t)(r % world);
    return;
  }
  // +1: Laplace smoothing, so lists the calibration stream never probed still carry their size
  // (with a raw count of 0 they would all pile onto one rank: adding 0 never changes the least-loaded rank)
  auto load = [&](int32_t i) { return (double)size(i) * ((double)counts[hot[i]] + 1.0); };
  std::sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) {
    if (load(a) != load(b)) return load(a) > load(b);
    return size(a) != size(b) ? size(a) > size(b) : hot[a] < hot[b];
  });
  std::vector<double> acc((size_t)world, 0.0);
  for (int32_t i : ord) {
    int32_t best = 0;
    for (int32_t r = 1; r < world; ++r)
      if (acc[r] < acc[best]) best = r;
    out_owner[i] = best;
    acc[best] += load(i);
  }
}

// ---------------------------------------------------------------- NCCL (non-blocking communicator)
// The communicator is created non-blocking (ncclConfig_t.blocking = 0), so no
// NCCL call can hang the caller: every call that returns ncclInProgress is
// polled with ncclCommGetAsyncError up to VLR_NCCL_TIMEOUT_MS (default 300000 ms);
// an error or a timeout aborts the communicator (ncclCommAbort makes the
// enqueued NCCL kernels exit) and marks the handle dead -> VLR_ERR_NCCL.
static int64_t nccl_timeout_ms() {
  const char* e = getenv("VLR_NCCL_TIMEOUT_MS");
  const long long v = e ? atoll(e) : 0;
  return v > 0 ? (int64_t)v : (int64_t)300000;
}

static vlr_status nccl_dead(vlr_index* h, const std::string& what) {
  if (h->ix.nccl) ncclCommAbort(reinterpret_cast<ncclComm_t>(h->ix.nccl));
  h->ix.nccl = nullptr;
  h->dead = true;
  return fail(VLR_ERR_NCCL, what + " (communicator aborted; the index handle is unusable)");
}

// wait until a non-blocking NCCL call has completed its host-side part
static ncclResult_t nccl_settle(ncclComm_t comm, ncclResult_t r, int64_t timeout_ms, bool* timed_out) {
  *timed_out = false;
  if (r != ncclInProgress) return r;
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    ncclResult_t st = ncclSuccess;
    ncclResult_t q = ncclCommGetAsyncError(comm, &st);
    if (q != ncclSuccess) return q;
    if (st != ncclInProgress) return st;
    if (std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count() >
        timeout_ms) {
      *timed_out = true;
      return ncclInProgress;
    }
    std::this_thread::yield();
  }
}

static ncclResult_t nccl_settle_init(ncclComm_t* comm, int world, ncclUniqueId uid, int rank, ncclConfig_t* cfg,
                                     bool* timed_out) {
  *timed_out = false;
  ncclResult_t r = ncclCommInitRankConfig(comm, world, uid, rank, cfg);
  if (r != ncclInProgress) return r;
  return nccl_settle(*comm, r, nccl_timeout_ms(), timed_out);
}

static vlr_status nccl_allgather(vlr_index* h, const void* send, void* recv, size_t bytes, cudaStream_t s,
                                 const char* what) {
  NvtxRange nv(h, what);
  ncclComm_t comm = reinterpret_cast<ncclComm_t>(h->ix.nccl);
  bool to = false;
  ncclResult_t r = nccl_settle(comm, ncclAllGather(send, recv, bytes, ncclUint8, comm, s), nccl_timeout_ms(), &to);
  if (to) return nccl_dead(h, std::string("ncclAllGather (") + what + ") not enqueued within VLR_NCCL_TIMEOUT_MS");
  if (r != ncclSuccess) return nccl_dead(h, std::string("ncclAllGather (") + what + "): " + ncclGetErrorString(r));
  return VLR_OK;
}

// a bounded device stall before the first collective of a search (VLR_FAULT_STALL_US, fault injection for
// the timeout tests: a peer that never arrives looks like this to the waiting rank)
__global__ void k_stall(unsigned long long ns) {
  const unsigned long long t0 = globaltimer_ns();
  while (globaltimer_ns() - t0 < ns) __nanosleep(1000);
}
static cudaError_t fault_stall(cudaStream_t s) {
  static long long us = -1;
  if (us < 0) {
    const char* e = getenv("VLR_FAULT_STALL_US");
    us = e ? atoll(e) : 0;
  }
  if (us <= 0) return cudaSuccess;
  k_stall<<<1, 32, 0, s>>>((unsigned long long)us * 1000ull);
  return cudaGetLastError();
}

// synchronise `s`; with a communicator, poll the stream and the communicator's
// asynchronous error state instead of blocking, up to VLR_NCCL_TIMEOUT_MS
static vlr_status wait_stream(vlr_index* h, cudaStream_t s) {
  if (!h->ix.nccl) {
    VLR_CUDA_TRY(cudaStreamSynchronize(s));
    return VLR_OK;
  }
  ncclComm_t comm = reinterpret_cast<ncclComm_t>(h->ix.nccl);
  const int64_t tmo = nccl_timeout_ms();
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaStreamQuery(s);
    if (q == cudaSuccess) return VLR_OK;
    if (q != cudaErrorNotReady) VLR_CUDA_TRY(q);
    ncclResult_t st = ncclSuccess;
    if (ncclCommGetAsyncError(comm, &st) != ncclSuccess || (st != ncclSuccess && st != ncclInProgress))
      return nccl_dead(h, std::string("NCCL asynchronous error: ") + ncclGetErrorString(st));
    if (std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count() > tmo)
      return nccl_dead(h, "search did not complete within VLR_NCCL_TIMEOUT_MS (a peer rank stopped?)");
    std::this_thread::yield();
  }
}

}  // namespace vlr

using namespace vlr;

extern "C" {

vlr_status vlr_deal_owners(const int64_t* list_offsets, int32_t nlist, const int64_t* counts, const int32_t* hot,
                           int32_t n_hot, int32_t world, int32_t* out_owner) {
  if (!list_offsets || nlist < 1 || n_hot < 0 || world < 1 || (n_hot > 0 && (!hot || !out_owner)))
    return fail(VLR_ERR_INVALID_ARG, "vlr_deal_owners: bad args");
  std::vector<uint8_t> seen((size_t)nlist, 0);
  for (int32_t i = 0; i < n_hot; ++i) {
    if (hot[i] < 0 || hot[i] >= nlist) return fail(VLR_ERR_UNKNOWN_CLUSTER, "hot cluster id out of range");
    if (seen[hot[i]]++) return fail(VLR_ERR_UNKNOWN_CLUSTER, "hot cluster listed twice");
  }
  if (counts)
    for (int32_t l = 0; l < nlist; ++l)
      if (counts[l] < 0) return fail(VLR_ERR_INVALID_ARG, "negative access count");
  deal(list_offsets, counts, hot, n_hot, world, out_owner);
  return VLR_OK;
}

vlr_status vlr_update_hot(vlr_index* h, const vlr_index_desc* desc) {
  if (!h || !desc) return fail(VLR_ERR_INVALID_ARG, "vlr_update_hot: null handle/desc");
  const DeviceIndex& cur = h->ix;
  if (desc->d != cur.d || desc->nlist != cur.nlist || desc->m != cur.m || desc->nbits != cur.nbits ||
      desc->metric != cur.metric || desc->by_residual != cur.by_residual)
    return fail(VLR_ERR_INVALID_ARG, "vlr_update_hot: index shape/variant differs from the handle's");
  // build the new residency as a separate shard-only handle (no communicator), while the
  // current one keeps serving (searches on other host threads take h->mu only to enqueue)
  vlr_comm_desc cm{cur.rank, cur.world, cur.device, nullptr};
  vlr_index* n = nullptr;
  vlr_status st = vlr_load_index(desc, &cm, &n);
  if (st != VLR_OK) return st;
  {
    std::lock_guard<std::mutex> lock(h->mu);
    VLR_CUDA_TRY(cudaSetDevice(cur.device));
    VLR_CUDA_TRY(cudaDeviceSynchronize());  // searches already enqueued on the old residency finish first
    DeviceIndex old = h->ix;
    n->ix.nccl = old.nccl;  // the communicator and the handle's mode stay
    n->ix.shard_only = old.shard_only;
    n->ix.coarse_sharded = old.coarse_sharded;
    old.nccl = nullptr;
    if (n->ix.mpad != old.mpad || n->ix.npairs != old.npairs || n->ix.lut_pair_bytes != old.lut_pair_bytes) {
      for (auto& w : h->wsl) free_ws(w);  // scan/LUT shapes changed (e.g. a different 4-bit mode): size again
    }
    h->ix = n->ix;
    n->ix = old;  // freed with the temporary handle
  }
  vlr_index_free(n);
  return VLR_OK;
}


const char* vlr_last_error(void) { return g_err.c_str(); }
int32_t vlr_version(void) { return (VLR_VERSION_MAJOR << 16) | VLR_VERSION_MINOR; }

vlr_status vlr_load_index(const vlr_index_desc* desc, const vlr_comm_desc* comm, vlr_index** out) {
  if (!desc || !out) return fail(VLR_ERR_INVALID_ARG, "vlr_load_index: null desc/out");
  *out = nullptr;
  const vlr_index_desc& D = *desc;
  vlr_comm_desc cm{0, 1, -1, nullptr};
  if (comm) cm = *comm;
  if (cm.world < 1 || cm.rank < 0 || cm.rank >= cm.world) return fail(VLR_ERR_INVALID_ARG, "bad rank/world");
  if (D.d < 1 || D.nlist < 1 || D.m < 1) return fail(VLR_ERR_INVALID_ARG, "d, nlist, m must be >= 1");
  if (D.d % D.m != 0) return fail(VLR_ERR_DIM_MISMATCH, "d % m != 0");
  if (D.nbits != 8 && D.nbits != 4) return fail(VLR_ERR_UNSUPPORTED, "nbits must be 8 or 4");
  if (D.metric != 0 && D.metric != 1) return fail(VLR_ERR_UNSUPPORTED, "metric must be 0 (squared L2) or 1 (inner product)");
  if (D.by_residual != 0 && D.by_residual != 1) return fail(VLR_ERR_INVALID_ARG, "by_residual must be 0 or 1");
  if (D.nbits == 8 && D.m > kMaxM) return fail(VLR_ERR_UNSUPPORTED, "m > 192 (8-bit codes)");
  if (D.nbits == 4 && D.m > kMaxM4) return fail(VLR_ERR_UNSUPPORTED, "m > 384 (4-bit codes)");
  if (!D.centroids || !D.codebooks || !D.list_offsets) return fail(VLR_ERR_INVALID_ARG, "null array");
  if (D.n_hot < 0 || (D.n_hot > 0 && !D.hot)) return fail(VLR_ERR_INVALID_ARG, "bad hot set");
  const int L = D.nlist, d = D.d, m = D.m, dsub = d / m;
  const int ksub = 1 << D.nbits;
  const int64_t cbytes = ((int64_t)m * D.nbits + 7) / 8;  // bytes of one input code row
  if (D.list_offsets[0] != 0) return fail(VLR_ERR_INVALID_ARG, "list_offsets[0] != 0");
  for (int l = 0; l < L; ++l)
    if (D.list_offsets[l + 1] < D.list_offsets[l]) return fail(VLR_ERR_INVALID_ARG, "list_offsets decreasing");
  const int64_t N = D.list_offsets[L];
  if (N > 0 && (!D.ids || !D.codes)) return fail(VLR_ERR_INVALID_ARG, "null ids/codes");
  // finiteness + centroid norms (fp64)
  std::vector<float> cn2((size_t)L);
  double cmax2 = 0.0;
  float cabs = 0.f;
  for (int l = 0; l < L; ++l) {
    double s = 0.0;
    const float* c = D.centroids + (size_t)l * d;
    for (int t = 0; t < d; ++t) {
      if (!std::isfinite(c[t])) return fail(VLR_ERR_NONFINITE, "non-finite centroid");
      s += (double)c[t] * c[t];
      cabs = std::max(cabs, std::fabs(c[t]));
    }
    cn2[l] = D.metric == 1 ? 0.f : (float)s;  // IP: the filter holds -2<q,c>
    cmax2 = std::max(cmax2, s);
  }
  const size_t ncb = (size_t)m * ksub * dsub;
  for (size_t i = 0; i < ncb; ++i)
    if (!std::isfinite(D.codebooks[i])) return fail(VLR_ERR_NONFINITE, "non-finite codebook");
  // hot set and owners (index splitter)
  std::vector<int32_t> owner((size_t)L, -1);
  {
    std::vector<int32_t> hot(D.hot, D.hot + D.n_hot);
    for (int i = 0; i < D.n_hot; ++i) {
      const int32_t l = hot[i];
      if (l < 0 || l >= L) return fail(VLR_ERR_UNKNOWN_CLUSTER, "hot cluster id out of range");
      if (owner[l] != -1) return fail(VLR_ERR_UNKNOWN_CLUSTER, "hot cluster listed twice");
      owner[l] = -2;
    }
    if (D.hot_owner) {
      for (int i = 0; i < D.n_hot; ++i) {
        if (D.hot_owner[i] < 0 || D.hot_owner[i] >= cm.world) return fail(VLR_ERR_UNKNOWN_CLUSTER, "hot_owner out of range");
        owner[hot[i]] = D.hot_owner[i];
      }
    } else {
      std::vector<int32_t> own((size_t)D.n_hot);
      deal(D.list_offsets, nullptr, hot.data(), D.n_hot, cm.world, own.data());
      for (int i = 0; i < D.n_hot; ++i) owner[hot[i]] = own[i];
    }
  }
  // device
  int dev = cm.device;
  if (dev < 0) {
    if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(VLR_ERR_CUDA, "no CUDA device");
  }
  VLR_CUDA_TRY(cudaSetDevice(dev));
  vlr_index* h = new vlr_index();
  DeviceIndex& ix = h->ix;
  ix.d = d;
  ix.d8 = (d + 7) / 8 * 8;
  ix.nlist = L;
  ix.m = m;
  ix.dsub = dsub;
  ix.nbits = D.nbits;
  ix.ksub = ksub;
  {
    const char* nib = getenv("VLR_PQ4_NIBBLE");  // 4-bit nibble-slot scan instead of pair tables (experiments)
    // (nibble slots are instantiated up to 256 sub-spaces; above, pair mode)
    ix.code_bits = (D.nbits == 4 && D.m <= 256 && nib && atoi(nib) == 1) ? 4 : 8;
  }
  ix.code_m = (D.nbits == 4 && ix.code_bits == 8) ? (m + 1) / 2 : m;  // pair mode: one slot per packed byte
  ix.lut_pair_bytes = (1 << ix.code_bits) * 64 * 4;
  if (ix.code_bits == 8) {
    ix.mpad = ((ix.code_m + 31) / 32) * 32;
  } else {  // scan instantiations for 4-bit slots: 32, 64, 96, 128, 192, 256 sub-spaces
    const int sizes[] = {32, 64, 96, 128, 192, 256};
    for (int v : sizes)
      if (m <= v) { ix.mpad = v; break; }
  }
  ix.npairs = (ix.mpad + 63) / 64;
  ix.rank = cm.rank;
  ix.world = cm.world;
  ix.metric = D.metric;
  ix.by_residual = D.by_residual;
  ix.device = dev;
  ix.shard_only = cm.world > 1 && cm.nccl_unique_id == nullptr;
  {  // this rank's centroid range for the sharded coarse stage: whole 128-centroid tiles, dealt contiguously
    const int T = (L + 127) / 128;
    const int t_lo = (int)((int64_t)cm.rank * T / cm.world), t_hi = (int)((int64_t)(cm.rank + 1) * T / cm.world);
    ix.c_lo = std::min(L, t_lo * 128);
    ix.c_hi = std::min(L, t_hi * 128);
  }
  ix.cmax = (float)std::sqrt(cmax2) * 1.0000002f;
  {  // power-of-two filter scale: max |c| 2^c_exp in [2^13, 2^14) (fp16 range), exponent clamped
    int e = 0;
    if (cabs > 0.f) {
      std::frexp(cabs, &e);  // cabs < 2^e
      e = std::min(60, std::max(-60, 14 - e));
    }
    ix.c_exp = e;
    ix.c_inv = std::ldexp(1.0f, -e);
  }
  ix.owner_h = owner;
  auto bail = [&](vlr_status st) {
    free_index(ix);
    delete h;
    return st;
  };
#define LTRY(expr)                                                                   \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess) {                                                         \
      set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));                 \
      return bail(_e == cudaErrorMemoryAllocation ? VLR_ERR_OOM : VLR_ERR_CUDA);     \
    }                                                                                \
  } while (0)
  cudaStream_t s;
  LTRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  // replicated tables
  std::vector<int32_t> local((size_t)L, -1), lglob;
  std::vector<int64_t> vbase_h(1, 0), gbase_h(1, 0);
  for (int l = 0; l < L; ++l) {
    if (owner[l] == cm.rank) {
      local[l] = (int32_t)lglob.size();
      lglob.push_back(l);
      const int64_t n = D.list_offsets[l + 1] - D.list_offsets[l];
      vbase_h.push_back(vbase_h.back() + n);
      gbase_h.push_back(gbase_h.back() + (n + 31) / 32);
    }
  }
  ix.n_local = (int32_t)lglob.size();
  {  // groups of the i largest local lists, i = 0..n_local (bounds one query's candidates for the large-k path)
    std::vector<int64_t> gl((size_t)ix.n_local);
    for (int32_t i = 0; i < ix.n_local; ++i) gl[i] = gbase_h[i + 1] - gbase_h[i];
    std::sort(gl.begin(), gl.end(), std::greater<int64_t>());
    ix.top_groups.assign(1, 0);
    for (int64_t v : gl) ix.top_groups.push_back(ix.top_groups.back() + v);
  }
  ix.n_vec = vbase_h.back();
  ix.n_groups = gbase_h.back();
  LTRY(dalloc(&ix.centroids, (size_t)L * d));
  LTRY(dalloc(&ix.cnorm2, (size_t)L));
  LTRY(dalloc(&ix.cf16, (size_t)L * ix.d8));
  LTRY(dalloc(&ix.codebooks, ncb));
  LTRY(dalloc(&ix.owner, (size_t)L));
  LTRY(dalloc(&ix.local, (size_t)L));
  LTRY(dalloc(&ix.gbase, (size_t)ix.n_local + 1));
  LTRY(dalloc(&ix.codes, (size_t)ix.n_groups * 32 * (ix.mpad * ix.code_bits / 8)));
  LTRY(dalloc(&ix.bias, (size_t)ix.n_groups * 32));
  LTRY(dalloc(&ix.ids, (size_t)ix.n_groups * 32));
  LTRY(cudaMemcpyAsync(ix.centroids, D.centroids, sizeof(float) * L * d, cudaMemcpyHostToDevice, s));
  LTRY(cudaMemcpyAsync(ix.cnorm2, cn2.data(), sizeof(float) * L, cudaMemcpyHostToDevice, s));
  LTRY(launch_round_f16(ix.centroids, L, d, ix.d8, std::ldexp(1.0f, ix.c_exp), ix.cf16, s));
  LTRY(make_tmap_2d(ix.tmapA, ix.cf16, L, ix.d8, 128, true));
  LTRY(dalloc(&ix.cf16t, (size_t)((L + 127) / 128) * 128 * (size_t)((ix.d8 + 63) / 64) * 64));
  LTRY(launch_tile_f16(ix, s));
  // the pre-tiled copy as a 2-D [tiles * kblocks * 128][64] tensor (box = one 16 KB tile image, stored
  // pre-swizzled: no TMA swizzle) for the CTA-pair filter's .cta_group::2 tensor loads
  LTRY(make_tmap_2d(ix.tmapAt, ix.cf16t, ((L + 127) / 128) * ((ix.d8 + 63) / 64) * 128, 64, 128, false));
  LTRY(cudaMemcpyAsync(ix.codebooks, D.codebooks, sizeof(float) * ncb, cudaMemcpyHostToDevice, s));
  LTRY(cudaMemcpyAsync(ix.owner, owner.data(), sizeof(int32_t) * L, cudaMemcpyHostToDevice, s));
  LTRY(cudaMemcpyAsync(ix.local, local.data(), sizeof(int32_t) * L, cudaMemcpyHostToDevice, s));
  LTRY(cudaMemcpyAsync(ix.gbase, gbase_h.data(), sizeof(int64_t) * gbase_h.size(), cudaMemcpyHostToDevice, s));
  // staging: owned lists' codes and ids, local order (= ascending cluster id)
  uint8_t* scodes = nullptr;
  int64_t *sids = nullptr, *svbase = nullptr, *ssorted = nullptr;
  int32_t *slglob = nullptr, *sflag = nullptr;
  void* cubtmp = nullptr;
  auto free_stage = [&]() {
    void* ps[] = {scodes, sids, svbase, ssorted, slglob, sflag, cubtmp};
    for (void* p : ps)
      if (p) cudaFree(p);
  };
  int32_t flag_h = 0;
  if (ix.n_vec > 0) {
    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) e = dalloc(&scodes, (size_t)ix.n_vec * cbytes);
    if (e == cudaSuccess) e = dalloc(&sids, (size_t)ix.n_vec);
    if (e == cudaSuccess) e = dalloc(&svbase, vbase_h.size());
    if (e == cudaSuccess) e = dalloc(&slglob, lglob.size());
    if (e == cudaSuccess) e = dalloc(&sflag, 1);
    // copy runs of consecutive owned lists
    int l = 0;
    while (e == cudaSuccess && l < L) {
      if (owner[l] != cm.rank) { ++l; continue; }
      int r = l;
      while (r + 1 < L && owner[r + 1] == cm.rank) ++r;
      const int64_t a = D.list_offsets[l], b = D.list_offsets[r + 1];
      const int64_t dst = vbase_h[local[l]];
      if (b > a) {
        e = cudaMemcpyAsync(scodes + dst * cbytes, D.codes + a * cbytes, (size_t)(b - a) * cbytes,
                            cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess)
          e = cudaMemcpyAsync(sids + dst, D.ids + a, (size_t)(b - a) * sizeof(int64_t), cudaMemcpyHostToDevice, s);
      }
      l = r + 1;
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(svbase, vbase_h.data(), sizeof(int64_t) * vbase_h.size(), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(slglob, lglob.data(), sizeof(int32_t) * lglob.size(), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(sflag, 0, sizeof(int32_t), s);
    // ids: >= 0 and unique among this rank's vectors (device radix sort)
    if (e == cudaSuccess) {
      k_negative<<<1024, 256, 0, s>>>(sids, ix.n_vec, sflag);
      e = cudaGetLastError();
    }
    size_t tmpb = 0;
    if (e == cudaSuccess) e = dalloc(&ssorted, (size_t)ix.n_vec);
    if (e == cudaSuccess)
      e = cub::DeviceRadixSort::SortKeys(nullptr, tmpb, (const int64_t*)sids, ssorted, (int64_t)ix.n_vec, 0, 64, s);
    if (e == cudaSuccess) e = cudaMalloc(&cubtmp, tmpb ? tmpb : 1);
    if (e == cudaSuccess)
      e = cub::DeviceRadixSort::SortKeys(cubtmp, tmpb, (const int64_t*)sids, ssorted, (int64_t)ix.n_vec, 0, 64, s);
    if (e == cudaSuccess) {
      k_adjacent_dup<<<1024, 256, 0, s>>>(ssorted, ix.n_vec, sflag);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = launch_layout(ix, scodes, sids, svbase, slglob, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&flag_h, sflag, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    free_stage();
    if (e != cudaSuccess) {
      set_error(std::string("load_index staging/layout: ") + cudaGetErrorString(e));
      cudaStreamDestroy(s);
      return bail(e == cudaErrorMemoryAllocation ? VLR_ERR_OOM : VLR_ERR_CUDA);
    }
  }
  LTRY(cudaStreamSynchronize(s));
  cudaStreamDestroy(s);
  if (flag_h & 2) {
    set_error("negative vector id");
    return bail(VLR_ERR_INVALID_ARG);
  }
  if (flag_h & 1) {
    set_error("duplicate vector id among resident vectors");
    return bail(VLR_ERR_DUPLICATE_ID);
  }
  ix.bytes = (int64_t)L * d * 4 + (int64_t)L * ix.d8 * 2 + (int64_t)((L + 127) / 128) * 128 * ((ix.d8 + 63) / 64) * 64 * 2 + L * 4 + (int64_t)ncb * 4 + 2LL * L * 4 + (ix.n_local + 1) * 8 +
             ix.n_groups * 32 * (ix.mpad * ix.code_bits / 8 + 4 + 8);
  // NCCL communicator (collective)
  // VLR_FORCE_EXCHANGE=1 with world == 1 and an NCCL id: a 1-rank communicator, so the exchange path
  // (rank merge into packed entries -> ncclAllGather -> K8 merge) runs on a single GPU (tests)
  const char* fx = getenv("VLR_FORCE_EXCHANGE");
  const bool force_x = cm.world == 1 && fx && atoi(fx) == 1;
  if ((cm.world > 1 || force_x) && cm.nccl_unique_id) {
    ncclUniqueId uid;
    std::memcpy(&uid, cm.nccl_unique_id, sizeof(uid));
    ncclComm_t comm_h = nullptr;
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.blocking = 0;  // no NCCL call may hang the caller: poll with a timeout (nccl_settle)
    bool to = false;
    ncclResult_t r = nccl_settle_init(&comm_h, cm.world, uid, cm.rank, &cfg, &to);
    if (to || r != ncclSuccess) {
      if (comm_h) ncclCommAbort(comm_h);
      set_error(to ? std::string("ncclCommInitRankConfig: not all ranks joined within VLR_NCCL_TIMEOUT_MS")
                   : std::string("ncclCommInitRankConfig: ") + ncclGetErrorString(r));
      return bail(VLR_ERR_NCCL);
    }
    ix.nccl = comm_h;
  }
  {
    // the collective search shards the coarse stage (also on a forced 1-rank communicator, where the
    // exchanges are self-copies: tests); VLR_COARSE_REPLICATED=1: every rank runs the full coarse stage
    const char* rep_env = getenv("VLR_COARSE_REPLICATED");
    ix.coarse_sharded = ix.nccl != nullptr && !(rep_env && atoi(rep_env) == 1);
  }
  {
    // VLR_SCAN_RESERVE=n: the scan's persistent grid leaves n SMs free (experiments; vlr_set_pipeline)
    const char* rs = getenv("VLR_SCAN_RESERVE");
    if (rs) h->scan_reserve = std::max(0, std::min(atoi(rs), scan_ctas(ix) - 2));
  }
  *out = h;
  return VLR_OK;
#undef LTRY
}

static void p2p_close(vlr_index* h) {
  auto& L = h->p2p;
  for (int g = 0; g < L.G; ++g)
    if (L.peer[g] && L.peer[g] != L.inbox) cudaIpcCloseMemHandle(L.peer[g]);
  if (L.inbox) cudaFree(L.inbox);
  if (L.ctr) cudaFree(L.ctr);
  L = vlr_index::PeerLink{};
}

void vlr_index_free(vlr_index* h) {
  if (!h) return;
  cudaSetDevice(h->ix.device);
  cudaDeviceSynchronize();
  for (auto& row : h->ev)
    for (auto& e : row)
      if (e) cudaEventDestroy(e);
  if (h->h2d_stream) cudaStreamDestroy(h->h2d_stream);
  for (auto& r : h->res) {
    cudaEvent_t evs[] = {r.done, r.lut_fork, r.lut_join, r.rel_fork, r.rel_join, r.q_ready[0], r.q_ready[1],
                         r.q_free[0], r.q_free[1]};
    for (cudaEvent_t e : evs)
      if (e) cudaEventDestroy(e);
    if (r.lut_stream) cudaStreamDestroy(r.lut_stream);
    if (r.rel_stream) cudaStreamDestroy(r.rel_stream);
  }
  p2p_close(h);
  for (auto& w : h->wsl) free_ws(w);
  free_index(h->ix);
  delete h;
}

vlr_status vlr_reserve(vlr_index* h, int32_t max_nq, int32_t max_nprobe, int32_t max_k) {
  if (!h || max_nq < 0 || max_nprobe < 1 || max_k < 1) return fail(VLR_ERR_INVALID_ARG, "vlr_reserve: bad args");
  if (max_k > kMaxKLarge) return fail(VLR_ERR_UNSUPPORTED, "k > 1024");
  cudaSetDevice(h->ix.device);
  const int np = std::min(max_nprobe, h->ix.nlist);
  if (np > kMaxNprobe) return fail(VLR_ERR_UNSUPPORTED, "nprobe' > 2048");
  std::lock_guard<std::mutex> lock(h->mu);
  for (int b = 0; b < h->nslots; ++b) {
    const vlr_status st = ensure_ws(h, b, std::max(max_nq, 1), np, max_k);
    if (st != VLR_OK) return st;
  }
  return VLR_OK;
}

vlr_status vlr_set_pipeline(vlr_index* h, int32_t slots, int32_t scan_reserve_sms) {
  if (!h) return fail(VLR_ERR_INVALID_ARG, "null index");
  if (slots < 1 || slots > vlr_index::kSlots) return fail(VLR_ERR_INVALID_ARG, "slots must be 1 or 2");
  std::lock_guard<std::mutex> lock(h->mu);
  int sms = 0;
  VLR_CUDA_TRY(cudaSetDevice(h->ix.device));
  VLR_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->ix.device));
  if (scan_reserve_sms < 0 || scan_reserve_sms > sms - 2)
    return fail(VLR_ERR_INVALID_ARG, "scan_reserve_sms must be in [0, SMs - 2]");
  if (h->p2p.inbox && slots != h->p2p.nslots)
    return fail(VLR_ERR_UNSUPPORTED, "the peer-exchange inbox was exported for another slot count");
  if (slots > h->nslots && h->wsl[0].status) {  // size the new slots like slot 0
    const Workspace& w0 = h->wsl[0];
    for (int b = h->nslots; b < slots; ++b) {
      const vlr_status st = ensure_ws(h, b, w0.cap_nq, w0.cap_np, w0.cap_k);
      if (st != VLR_OK) return st;
    }
  }
  h->nslots = slots;
  h->scan_reserve = scan_reserve_sms;
  return VLR_OK;
}

// device status word (mirrored to pinned host memory at the end of every search):
// bit 0 = a non-finite query (qprep), bit 1 = the NEXT-4 merger's bounded wait
// expired (those queries were neither merged nor released), bit 2 = a peer
// exchange wait expired. Reported and cleared by the first call that sees it.
static vlr_status take_status(Workspace& w, const char* when) {
  const int32_t st = *w.h_status;
  if (!st) return VLR_OK;
  *w.h_status = 0;
  if (st & 1) return fail(VLR_ERR_NONFINITE, std::string("non-finite query") + when);
  if (st & 4) return fail(VLR_ERR_CUDA, std::string("peer exchange: a rank's slab did not arrive within the bound "
                                                    "(a peer stopped?); the results are invalid") + when);
  return fail(VLR_ERR_CUDA, std::string("release merger timed out waiting for the scan; the affected queries "
                                        "were not released") + when);
}

static inline void rec(vlr_index* h, int i, cudaStream_t s) {
  // mode 1: every stage boundary; mode 2: only around the scan (events 5, 6)
  if (h->profiling == 1 || (h->profiling == 2 && (i == 5 || i == 6)))
    cudaEventRecord(h->ev[h->nsearch % vlr_index::kRing][i], s);
}

// ---------------------------------------------------------------- NVLink peer exchange plumbing
// Exchange kinds: 0 = coarse stage 1 (x1, fp32 [nq][np] per rank), 1 = coarse
// stage 2 (x2, 16-B entries [nq][np]), 2 = results (16-B entries [nq][k]).
// Each workspace slot has its own inbox region (flags included) and counters: two searches in flight
// (cross-batch pipelining) never share one.
static PeerOut peer_out(const vlr_index* h, int kind, int slot) {
  PeerOut o{};
  const auto& L = h->p2p;
  const size_t so = L.slot_bytes * (size_t)slot;
  const size_t off = so + (kind == 0 ? L.off_x1 : kind == 1 ? L.off_x2 : L.off_res);
  for (int g = 0; g < L.G; ++g) {
    o.base[g] = static_cast<char*>(L.peer[g]) + off;
    o.flag[g] = reinterpret_cast<uint32_t*>(static_cast<char*>(L.peer[g]) + so + L.off_flags) + kind * L.G;
  }
  o.G = L.G;
  o.rank = h->ix.rank;
  o.epoch = L.epoch;
  o.ctr = L.ctr + 3 * slot + kind;
  return o;
}
static PeerIn peer_in(vlr_index* h, int kind, int slot) {
  PeerIn i{};
  const auto& L = h->p2p;
  const size_t so = L.slot_bytes * (size_t)slot;
  i.flags = reinterpret_cast<const uint32_t*>(static_cast<char*>(L.inbox) + so + L.off_flags) + kind * L.G;
  i.G = L.G;
  i.epoch = L.epoch;
  i.status = h->wsl[slot].status;
  return i;
}
static void* inbox_region(vlr_index* h, int kind, int slot) {
  const auto& L = h->p2p;
  return static_cast<char*>(L.inbox) + L.slot_bytes * (size_t)slot +
         (kind == 0 ? L.off_x1 : kind == 1 ? L.off_x2 : L.off_res);
}

// ---------------------------------------------------------------- the search pipeline
// Phases (the staged API exposes the two exchange points between them; the
// collective search runs them back to back with NCCL all-gathers):
//  A  qprep, K1 filter (this rank's centroid tiles when sharded), LUT fork,
//     K2 (single GPU / replicated: + K3a + K3b route; sharded: stage 1 -> x1)
//  B  (sharded) K2 stage 2 from x1_all, K3a exact, K3b local -> x2
//  C  (sharded: K3b merge of x2_all + route), K4b offsets, LUT join, K6 scan,
//     K7 rank merge (-> packed entries when a communicator exchanges results)
struct Pipe {
  const float* Q;
  int nq, np, k;
  cudaStream_t s;
  int slot = 0;
  Workspace* w = nullptr;  // the slot's workspace
  int n = 0;  // launches
  bool lut_forked = false;  // this search forked K5 (joined before the scan)
};

static vlr_status lut_fork(vlr_index* h, Pipe& p) {
  if (h->lut_side < 0) {
    const char* e = getenv("VLR_LUT_SERIAL");
    h->lut_side = (e && e[0] == '1') ? 0 : 1;
  }
  p.lut_forked = h->lut_side == 1 && h->profiling != 1;  // per-stage profiling keeps stages serial
  if (!p.lut_forked) return VLR_OK;
  auto& r = h->res[p.slot];
  if (!r.lut_stream) {
    VLR_CUDA_TRY(cudaStreamCreateWithFlags(&r.lut_stream, cudaStreamNonBlocking));
    VLR_CUDA_TRY(cudaEventCreateWithFlags(&r.lut_fork, cudaEventDisableTiming));
    VLR_CUDA_TRY(cudaEventCreateWithFlags(&r.lut_join, cudaEventDisableTiming));
  }
  // forked after K1 so K5's CTAs do not take SM slots from the filter's waves;
  // everything before the fork on s (incl. the previous search of this slot, whose
  // scan read w.lut) is ordered before K5
  VLR_CUDA_TRY(cudaEventRecord(r.lut_fork, p.s));
  VLR_CUDA_TRY(cudaStreamWaitEvent(r.lut_stream, r.lut_fork, 0));
  VLR_CUDA_TRY(launch_lut(p.Q, h->ix, *p.w, p.nq, r.lut_stream)); ++p.n;
  VLR_CUDA_TRY(cudaEventRecord(r.lut_join, r.lut_stream));
  return VLR_OK;
}

static vlr_status phase_a(vlr_index* h, Pipe& p, bool sharded, uint8_t* out_miss, int32_t* out_probes) {
  NvtxRange nv(h, sharded ? "vlr coarse stage 1 (qprep, K1, K2s1)" : "vlr coarse (qprep, K1, K2, K3a, K3b)");
  DeviceIndex& ix = h->ix;
  Workspace& w = *p.w;
  VLR_CUDA_TRY(cudaMemsetAsync(w.status, 0, sizeof(int32_t), p.s));
  rec(h, 0, p.s);
  const int t_lo = sharded ? ix.c_lo / 128 : 0;
  const int t_hi = sharded ? (ix.c_hi + 127) / 128 : (ix.nlist + 127) / 128;
  const int bt = filter_btile_rows(p.nq, t_hi - t_lo);
  VLR_CUDA_TRY(launch_qprep(p.Q, p.nq, ix.d, ix.d8, w.qnorm, w.qsq, w.qf16, w.qinv, w.status, bt ? w.qf16t : nullptr,
                            bt, p.s)); ++p.n;
  VLR_CUDA_TRY(launch_filter_tc(w.qf16, w.qinv, p.nq, ix, t_lo, t_hi, w.dt, w.gmin, bt ? w.qf16t : nullptr, p.s)); ++p.n;
  vlr_status st = lut_fork(h, p);
  if (st != VLR_OK) return st;
  rec(h, 1, p.s);
  if (sharded && h->p2p.on) {
    const PeerOut po = peer_out(h, 0, p.slot);
    VLR_CUDA_TRY(launch_select(ix, w, p.nq, p.np, filter_edot(ix.d), kSelStage1, p.s, &po)); ++p.n;
    return VLR_OK;
  }
  VLR_CUDA_TRY(launch_select(ix, w, p.nq, p.np, filter_edot(ix.d), sharded ? kSelStage1 : kSelFull, p.s)); ++p.n;
  if (sharded) return VLR_OK;
  rec(h, 2, p.s);
  VLR_CUDA_TRY(launch_exact(p.Q, ix, w, p.nq, p.s)); ++p.n;
  VLR_CUDA_TRY(launch_refine(p.Q, ix, w, p.nq, p.np, out_miss, out_probes, kRefRoute, p.s)); ++p.n;
  rec(h, 3, p.s);
  return VLR_OK;
}

static vlr_status phase_b(vlr_index* h, Pipe& p) {
  NvtxRange nv(h, "vlr coarse stage 2 (K2s2, K3a, K3b local)");
  DeviceIndex& ix = h->ix;
  Workspace& w = *p.w;
  const bool pp = h->p2p.on;
  PeerIn pi;
  PeerOut po;
  Workspace wv = w;  // the gathered buffers are the inbox regions under the peer exchange
  if (pp) {
    pi = peer_in(h, 0, p.slot);
    po = peer_out(h, 1, p.slot);
    wv.x1_all = static_cast<float*>(inbox_region(h, 0, p.slot));
  }
  VLR_CUDA_TRY(launch_select(ix, wv, p.nq, p.np, filter_edot(ix.d), kSelStage2, p.s, nullptr, pp ? &pi : nullptr)); ++p.n;
  rec(h, 2, p.s);
  VLR_CUDA_TRY(launch_exact(p.Q, ix, w, p.nq, p.s)); ++p.n;
  VLR_CUDA_TRY(launch_refine(p.Q, ix, w, p.nq, p.np, nullptr, nullptr, kRefLocal, p.s, pp ? &po : nullptr)); ++p.n;
  return VLR_OK;
}

static vlr_status phase_c(vlr_index* h, Pipe& p, bool sharded, int64_t* out_ids, float* out_dist, uint8_t* out_miss,
                          int32_t* out_probes, const Release* rel, bool packed) {
  NvtxRange nv(h, rel ? "vlr route + release scan (K4b, K6 REL, merger)" : "vlr route + scan + merge (K4b, K6, K7)");
  DeviceIndex& ix = h->ix;
  Workspace& w = *p.w;
  if (sharded) {
    if (h->p2p.on) {
      const PeerIn pi = peer_in(h, 1, p.slot);
      Workspace wv = w;
      wv.x2_all = static_cast<CoarseEntry*>(inbox_region(h, 1, p.slot));
      VLR_CUDA_TRY(launch_refine(p.Q, ix, wv, p.nq, p.np, out_miss, out_probes, kRefMerge, p.s, nullptr, &pi)); ++p.n;
    } else {
      VLR_CUDA_TRY(launch_refine(p.Q, ix, w, p.nq, p.np, out_miss, out_probes, kRefMerge, p.s)); ++p.n;
    }
    rec(h, 3, p.s);
  }
  // the forked LUT joins before K4b, so that K4b -> K6 stays a programmatic (PDL) pair
  if (p.lut_forked) VLR_CUDA_TRY(cudaStreamWaitEvent(p.s, h->res[p.slot].lut_join, 0));
  VLR_CUDA_TRY(launch_offsets(ix, w, p.nq, p.np, p.s)); ++p.n;
  rec(h, 4, p.s);
  if (!p.lut_forked) {
    VLR_CUDA_TRY(launch_lut(p.Q, ix, w, p.nq, p.s)); ++p.n;
  }
  rec(h, 5, p.s);
  if (p.k > kMaxK) {  // large k: DUMP scan + per-query select, per chunk of queries (k_scan.cu)
    VLR_CUDA_TRY(launch_scan_large(ix, w, p.nq, p.np, p.k, out_ids, out_dist, packed ? w.send : nullptr, p.s));
    p.n += 2 * ((p.nq + w.dump_nq - 1) / w.dump_nq);
    rec(h, 6, p.s);
    rec(h, 7, p.s);
    return VLR_OK;
  }
  if (rel) VLR_CUDA_TRY(cudaMemsetAsync(w.qdone, 0, sizeof(unsigned long long) * p.nq, p.s));
  VLR_CUDA_TRY(launch_scan(ix, w, p.nq, p.np, p.k, p.s, rel)); ++p.n;
  rec(h, 6, p.s);
  if (!rel) {  // release mode: the scan merged and released every row itself
    if (h->p2p.on && packed) {
      const PeerOut po = peer_out(h, 2, p.slot);
      VLR_CUDA_TRY(launch_rank_merge(ix, w, p.nq, p.np, p.k, out_ids, out_dist, nullptr, p.s, &po)); ++p.n;
    } else {
      VLR_CUDA_TRY(launch_rank_merge(ix, w, p.nq, p.np, p.k, out_ids, out_dist, packed ? w.send : nullptr, p.s)); ++p.n;
    }
  }
  rec(h, 7, p.s);
  return VLR_OK;
}

static vlr_status check_search_args(vlr_index* h, int32_t nq, int32_t nprobe, int32_t k, int* np) {
  if (h->dead) return fail(VLR_ERR_NCCL, "index unusable after an NCCL failure");
  if (nq < 0 || nprobe < 1 || k < 1) return fail(VLR_ERR_INVALID_ARG, "nq < 0, nprobe < 1 or k < 1");
  if (k > kMaxKLarge) return fail(VLR_ERR_UNSUPPORTED, "k > 1024");
  if (k > kMaxK && h->ix.world * k > 8192) return fail(VLR_ERR_UNSUPPORTED, "world x k > 8192 (k > 32 merge)");
  if (k > kMaxK && (uint64_t)h->ix.n_groups * 32 >= (1ull << 32))
    return fail(VLR_ERR_UNSUPPORTED, "k > 32 needs < 2^32 resident vector slots on a rank");
  *np = std::min(nprobe, h->ix.nlist);
  if (*np > kMaxNprobe) return fail(VLR_ERR_UNSUPPORTED, "nprobe' > 2048");
  if (h->ix.world * *np > kMaxWorldProbes && h->ix.world > 1)
    return fail(VLR_ERR_UNSUPPORTED, "world x nprobe' > 16384 (sharded coarse stage)");
  return VLR_OK;
}

// Workspace slot of the next search: slot = seq % nslots. With more than one slot the
// stream first waits for the slot's previous search (event), so searches on different streams can
// overlap while none writes a slot another search still reads. Not under stream capture (the graph's
// replays are ordered by the capturing stream). The caller holds h->mu.
static bool capturing(cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
}
static vlr_status acquire_slot(vlr_index* h, int nq, int np, int k, cudaStream_t s, int* slot) {
  const int b = h->nslots > 1 ? (int)(h->seq % (uint64_t)h->nslots) : 0;
  vlr_status st = ensure_ws(h, b, nq, np, k);
  if (st != VLR_OK) return st;
  auto& r = h->res[b];
  if (h->nslots > 1 && r.pending && !capturing(s)) {
    VLR_CUDA_TRY(cudaStreamWaitEvent(s, r.done, 0));
    r.pending = false;
  }
  Workspace& w = h->wsl[b];
  w.n_cta = std::max(2, w.n_cta_cap - h->scan_reserve);
  ++h->seq;
  *slot = b;
  return VLR_OK;
}
static vlr_status release_slot(vlr_index* h, int b, cudaStream_t s) {
  if (h->nslots < 2 || capturing(s)) return VLR_OK;
  auto& r = h->res[b];
  if (!r.done) VLR_CUDA_TRY(cudaEventCreateWithFlags(&r.done, cudaEventDisableTiming));
  VLR_CUDA_TRY(cudaEventRecord(r.done, s));
  r.pending = true;
  return VLR_OK;
}

// enqueue one search; the caller holds h->mu (the workspace slots and the residency are per handle).
// slot_in >= 0: the caller acquired that slot (vlr_search_host stages its queries there first).
static vlr_status search_locked(vlr_index* h, const float* Q, int32_t nq, int32_t nprobe, int32_t k, int64_t* out_ids,
                                float* out_dist, uint8_t* out_miss, int32_t* out_probes, void* stream,
                                const Release* rel_in, int slot_in = -1, int* slot_out = nullptr) {
  int np = 0;
  vlr_status st = check_search_args(h, nq, nprobe, k, &np);
  if (st != VLR_OK) return st;
  DeviceIndex& ix = h->ix;
  h->launches = 0;
  if (nq == 0) return VLR_OK;
  if (!Q || !out_ids || !out_dist || !out_miss) return fail(VLR_ERR_INVALID_ARG, "null buffer");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  VLR_CUDA_TRY(cudaSetDevice(ix.device));
  const bool p2p = h->p2p.on;  // NVLink peer exchange: collective over the ranks' inboxes, no NCCL calls
  if (p2p) {
    if (nq > h->p2p.cap_nq || np > h->p2p.cap_np || k > h->p2p.cap_k || k > kMaxK)
      return fail(VLR_ERR_UNSUPPORTED, "peer exchange: batch beyond the caps reserved at vlr_p2p_export (or k > 32)");
    if (rel_in) return fail(VLR_ERR_UNSUPPORTED, "peer exchange: early release is on the NCCL / shard-only paths");
  }
  int slot = slot_in;
  if (slot < 0 && (st = acquire_slot(h, nq, np, k, s, &slot)) != VLR_OK) return st;
  // PDL only for eager launches without pipelining: captured into a CUDA graph, the programmatic edges
  // measured slower (B = 256 graph replay p50 1.85 -> 2.17 ms)
  pdl_for_search(h->nslots == 1 && !capturing(s));
  if (slot_out) *slot_out = slot;
  Workspace& w = h->wsl[slot];
  st = take_status(w, " (detected in a previous search on this handle)");
  if (st != VLR_OK) return st;
  const bool exchange = ix.nccl != nullptr || p2p;
  if (ix.nccl && !p2p) {  // an error of an earlier asynchronous search on this communicator
    ncclResult_t as = ncclSuccess;
    if (ncclCommGetAsyncError(reinterpret_cast<ncclComm_t>(ix.nccl), &as) != ncclSuccess ||
        (as != ncclSuccess && as != ncclInProgress))
      return nccl_dead(h, std::string("NCCL asynchronous error of an earlier search: ") + ncclGetErrorString(as));
  }
  if (p2p && ++h->p2p.epoch == 0) ++h->p2p.epoch;  // every rank runs the same searches: epochs agree
  Release relv{};
  const Release* rel = nullptr;
  if (rel_in) {  // the merger runs on the slot's own stream
    auto& r = h->res[slot];
    if (!r.rel_stream) {
      VLR_CUDA_TRY(cudaStreamCreateWithFlags(&r.rel_stream, cudaStreamNonBlocking));
      VLR_CUDA_TRY(cudaEventCreateWithFlags(&r.rel_fork, cudaEventDisableTiming));
      VLR_CUDA_TRY(cudaEventCreateWithFlags(&r.rel_join, cudaEventDisableTiming));
    }
    relv = *rel_in;
    relv.stream = r.rel_stream;
    relv.fork = r.rel_fork;
    relv.join = r.rel_join;
    rel = &relv;
  }
  const bool sharded = p2p || (ix.nccl && ix.coarse_sharded);
  Pipe p{Q, nq, np, k, s};
  p.slot = slot;
  p.w = &w;
  if ((st = phase_a(h, p, sharded, out_miss, out_probes)) != VLR_OK) return st;
  if (exchange) VLR_CUDA_TRY(fault_stall(s));
  if (sharded && !p2p) {
    if ((st = nccl_allgather(h, w.x1, w.x1_all, sizeof(float) * nq * np, s, "coarse stage 1")) != VLR_OK) return st;
    if ((st = phase_b(h, p)) != VLR_OK) return st;
    if ((st = nccl_allgather(h, w.x2, w.x2_all, sizeof(CoarseEntry) * nq * np, s, "coarse stage 2")) != VLR_OK)
      return st;
  } else if (p2p) {
    if ((st = phase_b(h, p)) != VLR_OK) return st;
  }
  if ((st = phase_c(h, p, sharded, out_ids, out_dist, out_miss, out_probes, rel, exchange && !rel)) != VLR_OK)
    return st;
  if (p2p) {
    const PeerIn pi = peer_in(h, 2, slot);
    VLR_CUDA_TRY(launch_merge_packed(inbox_region(h, 2, slot), h->p2p.G, nq, k, out_ids, out_dist, s, &pi)); ++p.n;
  } else if (exchange && !rel) {  // release mode: each rank releases its partial rows; vlr_merge_ready merges them
    if ((st = nccl_allgather(h, w.send, w.recv, (size_t)nq * k * sizeof(Packed), s, "results")) != VLR_OK) return st;
    VLR_CUDA_TRY(launch_merge_packed(w.recv, ix.world, nq, k, out_ids, out_dist, s)); ++p.n;
  }
  rec(h, 8, s);
  VLR_CUDA_TRY(cudaMemcpyAsync(w.h_status, w.status, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  h->launches = p.n;
  if (h->profiling) h->prof_mode[h->nsearch++ % vlr_index::kRing] = h->profiling;
  if (slot_in < 0) return release_slot(h, slot, s);
  return VLR_OK;
}

static vlr_status search_impl(vlr_index* h, const float* Q, int32_t nq, int32_t nprobe, int32_t k, int64_t* out_ids,
                              float* out_dist, uint8_t* out_miss, int32_t* out_probes, void* stream,
                              const Release* rel, int* slot_out = nullptr) {
  if (!h) return fail(VLR_ERR_INVALID_ARG, "null index");
  std::lock_guard<std::mutex> lock(h->mu);
  return search_locked(h, Q, nq, nprobe, k, out_ids, out_dist, out_miss, out_probes, stream, rel, -1, slot_out);
}

vlr_status vlr_search_async(vlr_index* h, const float* Q, int32_t nq, int32_t nprobe, int32_t k, int64_t* out_ids,
                            float* out_dist, uint8_t* out_miss, int32_t* out_probes, void* stream) {
  return search_impl(h, Q, nq, nprobe, k, out_ids, out_dist, out_miss, out_probes, stream, nullptr);
}

// device-accessible = device memory of this device, managed, or pinned host memory
// (mapped into the device's address space under UVA)
static bool device_accessible(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged ||
         (at.type == cudaMemoryTypeHost && at.devicePointer == p);
}

vlr_status vlr_search_release_async(vlr_index* h, const float* Q, int32_t nq, int32_t nprobe, int32_t k,
                                    int64_t* out_ids, float* out_dist, uint8_t* out_miss, int32_t* out_probes,
                                    uint32_t* ready, uint32_t epoch, void* stream) {
  if (!h) return fail(VLR_ERR_INVALID_ARG, "null index");
  if (h->ix.nccl && !h->ix.coarse_sharded)
    return fail(VLR_ERR_UNSUPPORTED, "early release with a communicator needs the sharded coarse stage");
  if (k > kMaxK) return fail(VLR_ERR_UNSUPPORTED, "early release: k > 32");
  if (nq > 0) {
    if (!ready || epoch == 0) return fail(VLR_ERR_INVALID_ARG, "release: null ready flags or epoch 0");
    VLR_CUDA_TRY(cudaSetDevice(h->ix.device));
    if (!device_accessible(ready) || !out_ids || !out_dist || !device_accessible(out_ids) ||
        !device_accessible(out_dist))
      return fail(VLR_ERR_INVALID_ARG, "release: ready/ids/dist must be device or pinned (mapped) host memory");
  }
  const Release rel{ready, epoch, out_ids, out_dist, nullptr, nullptr, nullptr};  // stream: the slot's
  return search_impl(h, Q, nq, nprobe, k, out_ids, out_dist, out_miss, out_probes, stream, &rel);
}

int32_t vlr_poll_ready(const uint32_t* ready, int32_t nq, uint32_t epoch, uint8_t* seen, int32_t* out_q,
                       int64_t* out_t_ns, int32_t max_out, int64_t timeout_us) {
  if (!ready || !seen || !out_q || nq < 0 || max_out < 1) return -1;
  const volatile uint32_t* r = ready;
  const auto t0 = std::chrono::steady_clock::now();
  int32_t n = 0;
  for (;;) {
    for (int32_t q = 0; q < nq && n < max_out; ++q) {
      if (seen[q] || r[q] != epoch) continue;
      seen[q] = 1;
      out_q[n] = q;
      if (out_t_ns) {
        timespec ts;
        clock_gettime(CLOCK_MONOTONIC, &ts);
        out_t_ns[n] = (int64_t)ts.tv_sec * 1000000000LL + ts.tv_nsec;
      }
      ++n;
    }
    if (n > 0) break;
    if (std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() - t0).count() >=
        timeout_us)
      break;
  }
  std::atomic_thread_fence(std::memory_order_acquire);  // rows of the released queries after their flags
  return n;
}

int32_t vlr_wait_ready(const uint32_t* ready, int32_t nq, uint32_t epoch, int64_t* out_t_ns, int64_t timeout_us) {
  if (!ready || nq < 0) return -1;
  const volatile uint32_t* r = ready;
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<uint8_t> seen((size_t)nq, 0);
  int32_t n = 0, lo = 0;  // queries below lo are all seen
  while (n < nq) {
    bool any = false;
    for (int32_t q = lo; q < nq; ++q) {
      if (seen[q] || r[q] != epoch) continue;
      seen[q] = 1;
      any = true;
      ++n;
      if (out_t_ns) {
        timespec ts;
        clock_gettime(CLOCK_MONOTONIC, &ts);
        out_t_ns[q] = (int64_t)ts.tv_sec * 1000000000LL + ts.tv_nsec;
      }
    }
    while (lo < nq && seen[lo]) ++lo;
    if (!any && std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() - t0).count() >=
                    timeout_us)
      break;
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  return n;
}

// The dispatcher side of NEXT-4 across ranks ("Each GPU worker sets
// a completion flag ... the dispatcher merges"): polls the n_shards flag arrays;
// query q is final once every shard has released it (ready[s][q] == epoch);
// its final row is the k smallest (dist, id) of the shards' partial rows (k-way
// merge of sorted rows, padding (-1, +inf) last). Host only.
int32_t vlr_merge_ready(int32_t n_shards, const uint32_t* const* ready, uint32_t epoch, int32_t nq, int32_t k,
                        const int64_t* const* part_ids, const float* const* part_dist, int64_t* out_ids,
                        float* out_dist, int64_t* out_t_ns, int64_t timeout_us) {
  if (n_shards < 1 || !ready || !part_ids || !part_dist || !out_ids || !out_dist || nq < 0 || k < 1) return -1;
  for (int32_t r = 0; r < n_shards; ++r)
    if (!ready[r] || !part_ids[r] || !part_dist[r]) return -1;
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<uint8_t> done((size_t)nq, 0);
  std::vector<int32_t> pos((size_t)n_shards);
  int32_t n = 0, lo = 0;
  while (n < nq) {
    bool any = false;
    for (int32_t q = lo; q < nq; ++q) {
      if (done[q]) continue;
      bool all = true;
      for (int32_t r = 0; r < n_shards && all; ++r) all = reinterpret_cast<const volatile uint32_t*>(ready[r])[q] == epoch;
      if (!all) continue;
      std::atomic_thread_fence(std::memory_order_acquire);  // the rows were written before the flags
      std::fill(pos.begin(), pos.end(), 0);
      for (int32_t j = 0; j < k; ++j) {
        int32_t best = -1;
        float bd = 0.f;
        int64_t bi = 0;
        for (int32_t r = 0; r < n_shards; ++r) {
          if (pos[r] >= k) continue;
          const int64_t id = part_ids[r][(size_t)q * k + pos[r]];
          if (id < 0) continue;  // padding: the rest of this row is padding
          const float dv = part_dist[r][(size_t)q * k + pos[r]];
          if (best < 0 || dv < bd || (dv == bd && id < bi)) { best = r; bd = dv; bi = id; }
        }
        if (best < 0) {
          out_ids[(size_t)q * k + j] = -1;
          out_dist[(size_t)q * k + j] = std::numeric_limits<float>::infinity();
        } else {
          out_ids[(size_t)q * k + j] = bi;
          out_dist[(size_t)q * k + j] = bd;
          ++pos[best];
        }
      }
      done[q] = 1;
      any = true;
      ++n;
      if (out_t_ns) {
        timespec ts;
        clock_gettime(CLOCK_MONOTONIC, &ts);
        out_t_ns[q] = (int64_t)ts.tv_sec * 1000000000LL + ts.tv_nsec;
      }
    }
    while (lo < nq && done[lo]) ++lo;
    if (!any && std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() - t0).count() >=
                    timeout_us)
      break;
  }
  return n;
}

vlr_status vlr_search(vlr_index* h, const float* Q, int32_t nq, int32_t nprobe, int32_t k, int64_t* out_ids,
                      float* out_dist, uint8_t* out_miss, int32_t* out_probes, void* stream) {
  int slot = 0;
  vlr_status st = search_impl(h, Q, nq, nprobe, k, out_ids, out_dist, out_miss, out_probes, stream, nullptr, &slot);
  if (st != VLR_OK || nq == 0) return st;
  if ((st = wait_stream(h, reinterpret_cast<cudaStream_t>(stream))) != VLR_OK) return st;
  return take_status(h->wsl[slot], "");
}

static vlr_status search_host_impl(vlr_index* h, const float* hQ, int32_t nq, int32_t nprobe, int32_t k,
                                   int64_t* h_ids, float* h_dist, uint8_t* h_miss, int32_t* h_probes, void* stream,
                                   bool sync) {
  if (!h) return fail(VLR_ERR_INVALID_ARG, "null index");
  if (nq < 0 || nprobe < 1 || k < 1) return fail(VLR_ERR_INVALID_ARG, "nq < 0, nprobe < 1 or k < 1");
  if (k > kMaxKLarge) return fail(VLR_ERR_UNSUPPORTED, "k > 1024");
  if (nq == 0) return VLR_OK;
  if (!hQ || !h_ids || !h_dist || !h_miss) return fail(VLR_ERR_INVALID_ARG, "null buffer");
  const int np = std::min(nprobe, h->ix.nlist);
  if (np > kMaxNprobe) return fail(VLR_ERR_UNSUPPORTED, "nprobe' > 2048");
  VLR_CUDA_TRY(cudaSetDevice(h->ix.device));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int slot = 0;
  {
    // the staging buffers belong to the handle's workspace, which ensure_ws may reallocate and
    // vlr_update_hot may free: size, stage and enqueue under the handle's mutex
    std::lock_guard<std::mutex> lock(h->mu);
    vlr_status st = check_search_args(h, nq, nprobe, k, &slot);  // (validates before a slot is taken)
    if (st != VLR_OK) return st;
    if ((st = acquire_slot(h, nq, np, k, s, &slot)) != VLR_OK) return st;
    Workspace& w = h->wsl[slot];
    // the queries go through one of two staging buffers, copied on the handle's H2D stream: the copy of
    // batch i+1 overlaps batch i's kernels (stream capture: the copy stays on `stream`)
    auto& r = h->res[slot];
    const int qi = r.qbuf;
    r.qbuf ^= 1;
    float* dq = qi ? w.d_q2 : w.d_q;
    const size_t qbytes = sizeof(float) * nq * h->ix.d;
    if (capturing(s)) {
      VLR_CUDA_TRY(cudaMemcpyAsync(dq, hQ, qbytes, cudaMemcpyHostToDevice, s));
    } else {
      if (!h->h2d_stream) VLR_CUDA_TRY(cudaStreamCreateWithFlags(&h->h2d_stream, cudaStreamNonBlocking));
      if (!r.q_ready[qi]) {
        VLR_CUDA_TRY(cudaEventCreateWithFlags(&r.q_ready[qi], cudaEventDisableTiming));
        VLR_CUDA_TRY(cudaEventCreateWithFlags(&r.q_free[qi], cudaEventDisableTiming));
      }
      if (r.q_used[qi]) VLR_CUDA_TRY(cudaStreamWaitEvent(h->h2d_stream, r.q_free[qi], 0));  // its last reader
      VLR_CUDA_TRY(cudaMemcpyAsync(dq, hQ, qbytes, cudaMemcpyHostToDevice, h->h2d_stream));
      VLR_CUDA_TRY(cudaEventRecord(r.q_ready[qi], h->h2d_stream));
      VLR_CUDA_TRY(cudaStreamWaitEvent(s, r.q_ready[qi], 0));
    }
    st = search_locked(h, dq, nq, nprobe, k, w.d_ids, w.d_dist, w.d_miss, h_probes ? w.d_probes : nullptr, stream,
                       nullptr, slot);
    if (st != VLR_OK) return st;
    if (!capturing(s)) {  // every kernel of the search has read dq once `stream` passes this point
      VLR_CUDA_TRY(cudaEventRecord(r.q_free[qi], s));
      r.q_used[qi] = true;
    }
    VLR_CUDA_TRY(cudaMemcpyAsync(h_ids, w.d_ids, sizeof(int64_t) * nq * k, cudaMemcpyDeviceToHost, s));
    VLR_CUDA_TRY(cudaMemcpyAsync(h_dist, w.d_dist, sizeof(float) * nq * k, cudaMemcpyDeviceToHost, s));
    VLR_CUDA_TRY(cudaMemcpyAsync(h_miss, w.d_miss, (size_t)nq * np, cudaMemcpyDeviceToHost, s));
    if (h_probes)
      VLR_CUDA_TRY(cudaMemcpyAsync(h_probes, w.d_probes, sizeof(int32_t) * nq * np, cudaMemcpyDeviceToHost, s));
    if ((st = release_slot(h, slot, s)) != VLR_OK) return st;
  }
  Workspace& w = h->wsl[slot];
  if (!sync) return VLR_OK;  // results land when `stream` reaches this point; status: next call
  vlr_status st = wait_stream(h, s);
  if (st != VLR_OK) return st;
  return take_status(w, "");
}

vlr_status vlr_search_host(vlr_index* h, const float* hQ, int32_t nq, int32_t nprobe, int32_t k, int64_t* h_ids,
                           float* h_dist, uint8_t* h_miss, int32_t* h_probes, void* stream) {
  return search_host_impl(h, hQ, nq, nprobe, k, h_ids, h_dist, h_miss, h_probes, stream, true);
}

vlr_status vlr_search_host_async(vlr_index* h, const float* hQ, int32_t nq, int32_t nprobe, int32_t k,
                                 int64_t* h_ids, float* h_dist, uint8_t* h_miss, int32_t* h_probes, void* stream) {
  return search_host_impl(h, hQ, nq, nprobe, k, h_ids, h_dist, h_miss, h_probes, stream, false);
}

// ---------------------------------------------------------------- staged (caller-exchanged) search
// The collective search split at its two coarse-stage exchange points and its
// result exchange, for shard-only handles (world > 1, no communicator): the
// caller moves x1 / x2 between the ranks with any transport and merges the
// partial results with vlr_merge_partials. Same kernels as the NCCL path.
static vlr_status staged_begin(vlr_index* h, const float* Q, int32_t nq, int32_t nprobe, int32_t k, int* np) {
  if (!h) return fail(VLR_ERR_INVALID_ARG, "null index");
  if (!h->ix.shard_only) return fail(VLR_ERR_INVALID_ARG, "staged search needs a shard-only handle (world > 1, no communicator)");
  vlr_status st = check_search_args(h, nq, nprobe, k, np);
  if (st != VLR_OK) return st;
  if (k > kMaxK) return fail(VLR_ERR_UNSUPPORTED, "staged search: k > 32");
  if (nq < 1 || !Q) return fail(VLR_ERR_INVALID_ARG, "staged search: nq >= 1 and queries required");
  VLR_CUDA_TRY(cudaSetDevice(h->ix.device));
  // sized for any k up front: a reallocation between the stages would drop the LUT and the gathered
  // buffers of the batch in flight
  pdl_for_search(h->nslots == 1);
  return ensure_ws(h, h->stage_slot, nq, *np, std::max(k, kMaxK));  // k <= 32 only (vlr.h: staged search)
}

vlr_status vlr_coarse_stage1(vlr_index* h, const float* Q, int32_t nq, int32_t nprobe, float* d_x1, void* stream) {
  if (!h) return fail(VLR_ERR_INVALID_ARG, "null index");
  std::lock_guard<std::mutex> lock(h->mu);
  int np = 0;
  vlr_status st = staged_begin(h, Q, nq, nprobe, 1, &np);
  if (st != VLR_OK) return st;
  if (!d_x1) return fail(VLR_ERR_INVALID_ARG, "null x1");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int slot = 0;  // the batch keeps this workspace slot through stage 3
  if ((st = acquire_slot(h, nq, np, kMaxK, s, &slot)) != VLR_OK) return st;
  h->stage_slot = slot;
  Workspace& w = h->wsl[slot];
  if ((st = take_status(w, " (detected in a previous search on this handle)")) != VLR_OK) return st;
  Pipe p{Q, nq, np, 1, s};
  p.slot = slot;
  p.w = &w;
  if ((st = phase_a(h, p, true, nullptr, nullptr)) != VLR_OK) return st;
  VLR_CUDA_TRY(cudaMemcpyAsync(d_x1, w.x1, sizeof(float) * nq * np, cudaMemcpyDeviceToDevice, s));
  h->stage = 1;
  h->stage_nq = nq;
  h->stage_np = np;
  h->launches = p.n;
  return VLR_OK;
}

vlr_status vlr_coarse_stage2(vlr_index* h, const float* Q, int32_t nq, int32_t nprobe, const float* d_x1_all, void* d_x2,
                             void* stream) {
  if (!h) return fail(VLR_ERR_INVALID_ARG, "null index");
  std::lock_guard<std::mutex> lock(h->mu);
  int np = 0;
  vlr_status st = staged_begin(h, Q, nq, nprobe, 1, &np);
  if (st != VLR_OK) return st;
  if (!d_x1_all || !d_x2) return fail(VLR_ERR_INVALID_ARG, "null x1_all / x2");
  if (h->stage != 1 || h->stage_nq != nq || h->stage_np != np)
    return fail(VLR_ERR_INVALID_ARG, "vlr_coarse_stage2 must follow vlr_coarse_stage1 of the same batch");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  Workspace& w = h->wsl[h->stage_slot];
  VLR_CUDA_TRY(cudaMemcpyAsync(w.x1_all, d_x1_all, sizeof(float) * nq * np * h->ix.world, cudaMemcpyDeviceToDevice, s));
  Pipe p{Q, nq, np, 1, s};
  p.slot = h->stage_slot;
  p.w = &w;
  if ((st = phase_b(h, p)) != VLR_OK) return st;
  VLR_CUDA_TRY(cudaMemcpyAsync(d_x2, w.x2, sizeof(CoarseEntry) * nq * np, cudaMemcpyDeviceToDevice, s));
  h->stage = 2;
  h->launches += p.n;
  return VLR_OK;
}

vlr_status vlr_search_stage3(vlr_index* h, const float* Q, int32_t nq, int32_t nprobe, int32_t k, const void* d_x2_all,
                             int64_t* d_ids, float* d_dist, uint8_t* d_miss, int32_t* d_probes, void* stream) {
  if (!h) return fail(VLR_ERR_INVALID_ARG, "null index");
  std::lock_guard<std::mutex> lock(h->mu);
  int np = 0;
  vlr_status st = staged_begin(h, Q, nq, nprobe, k, &np);
  if (st != VLR_OK) return st;
  if (!d_x2_all || !d_ids || !d_dist || !d_miss) return fail(VLR_ERR_INVALID_ARG, "null buffer");
  if (h->stage != 2 || h->stage_nq != nq || h->stage_np != np)
    return fail(VLR_ERR_INVALID_ARG, "vlr_search_stage3 must follow vlr_coarse_stage2 of the same batch");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  Workspace& w = h->wsl[h->stage_slot];
  VLR_CUDA_TRY(cudaMemcpyAsync(w.x2_all, d_x2_all, sizeof(CoarseEntry) * nq * np * h->ix.world,
                               cudaMemcpyDeviceToDevice, s));
  Pipe p{Q, nq, np, k, s};
  p.slot = h->stage_slot;
  p.w = &w;
  if ((st = phase_c(h, p, true, d_ids, d_dist, d_miss, d_probes, nullptr, false)) != VLR_OK) return st;
  rec(h, 8, s);
  VLR_CUDA_TRY(cudaMemcpyAsync(w.h_status, w.status, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  if ((st = release_slot(h, h->stage_slot, s)) != VLR_OK) return st;
  h->stage = 0;
  h->launches += p.n;
  if (h->profiling) h->prof_mode[h->nsearch++ % vlr_index::kRing] = h->profiling;
  return VLR_OK;
}

// ---------------------------------------------------------------- NVLink peer exchange (setup)
static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

vlr_status vlr_p2p_export(vlr_index* h, void* handle_out) {
  if (!h || !handle_out) return fail(VLR_ERR_INVALID_ARG, "vlr_p2p_export: null argument");
  std::lock_guard<std::mutex> lock(h->mu);
  const DeviceIndex& ix = h->ix;
  if (ix.world < 2 || ix.world > kMaxWorld) return fail(VLR_ERR_UNSUPPORTED, "peer exchange needs 2 <= world <= 8");
  Workspace& w = h->wsl[0];
  for (int b = 0; b < h->nslots; ++b)
    if (!h->wsl[b].status)
      return fail(VLR_ERR_INVALID_ARG, "vlr_p2p_export: call vlr_reserve first (the inbox is sized by it)");
  VLR_CUDA_TRY(cudaSetDevice(ix.device));
  p2p_close(h);
  auto& L = h->p2p;
  L.G = ix.world;
  L.nslots = h->nslots;
  L.cap_nq = w.cap_nq;
  L.cap_np = w.cap_np;
  L.cap_k = std::min(w.cap_k, kMaxK);
  const size_t G = (size_t)L.G, nq = (size_t)L.cap_nq, np = (size_t)L.cap_np, k = (size_t)L.cap_k;
  L.off_x1 = 0;
  L.off_x2 = align256(L.off_x1 + G * nq * np * sizeof(float));
  L.off_res = align256(L.off_x2 + G * nq * np * sizeof(CoarseEntry));
  L.off_flags = align256(L.off_res + G * nq * k * sizeof(Packed));
  L.slot_bytes = align256(L.off_flags + 3 * G * sizeof(uint32_t));
  L.bytes = L.slot_bytes * (size_t)L.nslots;
  VLR_CUDA_TRY(cudaMalloc(&L.inbox, L.bytes));
  VLR_CUDA_TRY(cudaMemset(L.inbox, 0, L.bytes));
  VLR_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&L.ctr), 3 * L.nslots * sizeof(int)));
  VLR_CUDA_TRY(cudaMemset(L.ctr, 0, 3 * L.nslots * sizeof(int)));
  cudaIpcMemHandle_t mh;
  VLR_CUDA_TRY(cudaIpcGetMemHandle(&mh, L.inbox));
  static_assert(sizeof(mh) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(handle_out, &mh, sizeof(mh));
  return VLR_OK;
}

vlr_status vlr_p2p_connect(vlr_index* h, const void* handles) {
  if (!h || !handles) return fail(VLR_ERR_INVALID_ARG, "vlr_p2p_connect: null argument");
  std::lock_guard<std::mutex> lock(h->mu);
  auto& L = h->p2p;
  if (!L.inbox) return fail(VLR_ERR_INVALID_ARG, "vlr_p2p_connect: vlr_p2p_export first");
  VLR_CUDA_TRY(cudaSetDevice(h->ix.device));
  for (int g = 0; g < L.G; ++g) {
    if (g == h->ix.rank) {
      L.peer[g] = L.inbox;
      continue;
    }
    cudaIpcMemHandle_t mh;
    std::memcpy(&mh, static_cast<const char*>(handles) + 64 * g, 64);
    void* p = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&p, mh, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      for (int r = 0; r < g; ++r)
        if (L.peer[r] && L.peer[r] != L.inbox) cudaIpcCloseMemHandle(L.peer[r]);
      std::fill(L.peer, L.peer + kMaxWorld, nullptr);
      return fail(VLR_ERR_CUDA, std::string("cudaIpcOpenMemHandle of rank ") + std::to_string(g) + ": " +
                                     cudaGetErrorString(e));
    }
    L.peer[g] = p;
  }
  L.on = true;
  L.epoch = 0;
  return VLR_OK;
}

vlr_status vlr_p2p_setup(vlr_index* h) {
  if (!h) return fail(VLR_ERR_INVALID_ARG, "null index");
  if (!h->ix.nccl) return fail(VLR_ERR_INVALID_ARG, "vlr_p2p_setup needs a communicator (else export / connect)");
  std::vector<char> mine(64), all(64 * (size_t)h->ix.world);
  vlr_status st = vlr_p2p_export(h, mine.data());
  if (st != VLR_OK) return st;
  // the handles travel over the communicator: a device copy, one all-gather
  char* d = nullptr;
  VLR_CUDA_TRY(cudaMalloc(&d, all.size() + 64));
  VLR_CUDA_TRY(cudaMemcpy(d, mine.data(), 64, cudaMemcpyHostToDevice));
  cudaStream_t s = nullptr;
  VLR_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  st = nccl_allgather(h, d, d + 64, 64, s, "peer-exchange handles");
  if (st == VLR_OK) st = wait_stream(h, s);
  cudaStreamDestroy(s);
  if (st == VLR_OK) {
    VLR_CUDA_TRY(cudaMemcpy(all.data(), d + 64, all.size(), cudaMemcpyDeviceToHost));
  }
  cudaFree(d);
  if (st != VLR_OK) return st;
  return vlr_p2p_connect(h, all.data());
}

vlr_status vlr_merge_partials(const int64_t* part_ids, const float* part_dist, int32_t n_shards, int32_t nq, int32_t k,
                              int64_t* out_ids, float* out_dist, void* stream) {
  if (n_shards < 1 || nq < 0 || k < 1) return fail(VLR_ERR_INVALID_ARG, "vlr_merge_partials: bad sizes");
  if (k > kMaxKLarge || (k > kMaxK && (int64_t)n_shards * k > 8192))
    return fail(VLR_ERR_UNSUPPORTED, "k > 1024, or n_shards x k > 8192 for k > 32");
  if (nq == 0) return VLR_OK;
  if (!part_ids || !part_dist || !out_ids || !out_dist) return fail(VLR_ERR_INVALID_ARG, "null buffer");
  VLR_CUDA_TRY(launch_merge_split(part_ids, part_dist, n_shards, nq, k, out_ids, out_dist,
                                  reinterpret_cast<cudaStream_t>(stream)));
  return VLR_OK;
}

vlr_status vlr_access_counts(const vlr_index* h, const int32_t* d_probes, int64_t n, int64_t* d_counts,
                             void* stream) {
  if (!h || n < 0 || (n > 0 && (!d_probes || !d_counts))) return fail(VLR_ERR_INVALID_ARG, "vlr_access_counts: bad args");
  VLR_CUDA_TRY(launch_access_hist(d_probes, n, h->ix.nlist, reinterpret_cast<unsigned long long*>(d_counts),
                                  reinterpret_cast<cudaStream_t>(stream)));
  return VLR_OK;
}

vlr_status vlr_index_info(const vlr_index* h, int64_t* bytes, int32_t* n_lists, int64_t* n_vec) {
  if (!h) return fail(VLR_ERR_INVALID_ARG, "null index");
  if (bytes) *bytes = h->ix.bytes;
  if (n_lists) *n_lists = h->ix.n_local;
  if (n_vec) *n_vec = h->ix.n_vec;
  return VLR_OK;
}

vlr_status vlr_index_owners(const vlr_index* h, int32_t* out) {
  if (!h || !out) return fail(VLR_ERR_INVALID_ARG, "null arg");
  std::memcpy(out, h->ix.owner_h.data(), sizeof(int32_t) * h->ix.owner_h.size());
  return VLR_OK;
}

vlr_status vlr_set_profiling(vlr_index* h, int32_t enable) {
  if (!h) return fail(VLR_ERR_INVALID_ARG, "null index");
  if (enable && !h->ev[0][0]) {
    VLR_CUDA_TRY(cudaSetDevice(h->ix.device));
    for (auto& row : h->ev)
      for (auto& e : row) VLR_CUDA_TRY(cudaEventCreate(&e));
  }
  if (enable < 0 || enable > 2) return fail(VLR_ERR_INVALID_ARG, "profiling mode must be 0, 1 or 2");
  h->profiling = enable;
  return VLR_OK;
}

vlr_status vlr_stage_times(vlr_index* h, int32_t back, float* ms, int32_t n) {
  if (!h || !ms) return fail(VLR_ERR_INVALID_ARG, "null arg");
  if (!h->ev[0][0]) return fail(VLR_ERR_INVALID_ARG, "profiling never enabled");
  if (back < 0 || back >= vlr_index::kRing || back >= h->nsearch)
    return fail(VLR_ERR_INVALID_ARG, "no such recorded search");
  const int slot = (int)((h->nsearch - 1 - back) % vlr_index::kRing);
  cudaEvent_t* ev = h->ev[slot];
  const int stages = std::min(n, 8);
  if (h->prof_mode[slot] == 2) {  // scan only
    VLR_CUDA_TRY(cudaEventSynchronize(ev[6]));
    for (int i = 0; i < stages; ++i) ms[i] = std::numeric_limits<float>::quiet_NaN();
    if (stages > 5) VLR_CUDA_TRY(cudaEventElapsedTime(&ms[5], ev[5], ev[6]));
    return VLR_OK;
  }
  VLR_CUDA_TRY(cudaEventSynchronize(ev[8]));
  for (int i = 0; i < stages; ++i) {
    float t = 0.f;
    VLR_CUDA_TRY(cudaEventElapsedTime(&t, ev[i], ev[i + 1]));
    ms[i] = t;
  }
  return VLR_OK;
}

int32_t vlr_last_launch_count(const vlr_index* h) { return h ? h->launches : 0; }

vlr_status vlr_nccl_unique_id(void* out) {
  if (!out) return fail(VLR_ERR_INVALID_ARG, "null out");
  ncclUniqueId uid;
  ncclResult_t r = ncclGetUniqueId(&uid);
  if (r != ncclSuccess) return fail(VLR_ERR_NCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
  static_assert(sizeof(uid) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out, &uid, sizeof(uid));
  return VLR_OK;
}

}  // extern "C"

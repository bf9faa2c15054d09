/*
 * vlr.h -- C ABI of libvlr.so: batched IVF-PQ search over the GPU-resident
 * ("hot") inverted lists, B200 (sm_100a) native.
 *
 * Method: VectorLiteRAG (arXiv 2504.08930). The calls follow the paper's
 * problem statement (BASELINE.json north_star):
 *   load_index(centroids, PQ codebooks, inverted lists, hot-cluster set)
 *   search(queries, nprobe, k) -> (ids, distances, per-query miss mask)
 * Citations are PAPER.md line numbers (P:n) and DESIGN.md reading ids (A*).
 *
 * Conventions for every call:
 *  - No C++ exception crosses this ABI. Every call returns a vlr_status;
 *    vlr_last_error() gives a thread-local message for the last failure on
 *    the calling thread (valid until the next vlr_* call on that thread).
 *  - "host" pointers are ordinary CPU memory (pinned or pageable);
 *    "device" pointers are CUDA global memory on the index's device.
 *  - Streams are passed as void* (a cudaStream_t); NULL = legacy default.
 *  - One in-flight search per index handle (the workspace is per handle):
 *    calls on one handle from several host threads are serialised while they
 *    enqueue, and must pass the SAME stream so that the device work is
 *    ordered too; distinct handles are independent.
 *  - There is no CPU fallback: every step of search runs in this library's
 *    sm_100a kernels. Without a usable GPU, load_index fails with VLR_ERR_CUDA.
 */
#ifndef VLR_H_
#define VLR_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VLR_VERSION_MAJOR 1
#define VLR_VERSION_MINOR 3

typedef struct vlr_index vlr_index; /* opaque; created by vlr_load_index, freed by vlr_index_free */

typedef enum {
  VLR_OK = 0,
  VLR_ERR_INVALID_ARG = 1,     /* null pointer, nprobe < 1, k < 1, negative id, bad offsets, ... */
  VLR_ERR_DIM_MISMATCH = 2,    /* d % m != 0, or d/m inconsistent with the codebooks */
  VLR_ERR_NONFINITE = 3,       /* NaN/Inf in centroids, codebooks (load) or queries (search) */
  VLR_ERR_UNKNOWN_CLUSTER = 4, /* hot id out of [0, nlist) or listed twice; hot_owner out of range */
  VLR_ERR_DUPLICATE_ID = 5,    /* a vector id occurs twice among this rank's resident vectors */
  VLR_ERR_OOM = 6,             /* device allocation failed */
  VLR_ERR_CUDA = 7,            /* any other CUDA runtime error (no device, launch failure, ...) */
  VLR_ERR_NCCL = 8,            /* NCCL error; the communicator is aborted, the handle unusable */
  VLR_ERR_UNSUPPORTED = 9      /* valid but outside this version: nbits not in {4, 8}, metric not in
                                  {0, 1}, m > 192 (8-bit) / 384 (4-bit), k > 1024, nprobe' > 2048 */
} vlr_status;

/*
 * Index description (all pointers HOST, read during vlr_load_index only;
 * every array is copied, the caller may free them on return).
 *
 * Definitions (§II.A-B; readings A2, A5 in DESIGN.md):
 *   vector i of list l reconstructs to xhat_i = c_l + concat_j Y[j][code_ij]
 *   (residual PQ, sub-space j = dims [j*dsub, (j+1)*dsub), dsub = d/m);
 *   with by_residual = 0, xhat_i = concat_j Y[j][code_ij].
 *   metric 0: dist(q, x) = ||q - x||^2; metric 1 (inner product, "the
 *   approach is independent of the distance metric"; reading A1' in
 *   DESIGN.md): dist(q, x) = -<q, x>, so "ascending distance" is descending
 *   similarity, and the coarse quantizer probes the largest <q, c_l>.
 */
typedef struct {
  int32_t d;            /* vector dimension, >= 1 */
  int32_t nlist;        /* number of inverted lists / coarse centroids, >= 1 */
  int32_t m;            /* PQ sub-quantizers, d % m == 0, 1 <= m <= 192 (nbits 8) or 384 (nbits 4) */
  int32_t nbits;        /* bits per sub-code: 8 (256 codewords) or 4 (16 codewords; the paper's 4-bit
                           PQ, reading A4') */
  int32_t metric;       /* 0 = squared L2, 1 = inner product (distance reported as -<q, x>) */
  int32_t by_residual;  /* 1 = codes encode x - c_l, 0 = codes encode x */
  const float* centroids;      /* [nlist][d] row-major fp32 */
  const float* codebooks;      /* [m][2^nbits][d/m] fp32 */
  const int64_t* list_offsets; /* [nlist+1]; list l = rows [offsets[l], offsets[l+1]); offsets[0] = 0,
                                  non-decreasing; N = offsets[nlist] (empty lists allowed) */
  const int64_t* ids;          /* [N] vector ids, >= 0, unique (-1 is the padding id) */
  const uint8_t* codes;        /* [N][ceil(m*nbits/8)]; nbits 8: byte j of row i = sub-code j of vector i;
                                  nbits 4: sub-code j = low nibble of byte j/2 for even j, high nibble
                                  for odd j */
  const int32_t* hot;          /* [n_hot] cluster ids resident on the GPUs; no duplicates.
                                  May be NULL iff n_hot == 0 (then every probe is a miss). */
  int32_t n_hot;
  const int32_t* hot_owner;    /* optional [n_hot]: rank owning hot[i]; NULL = deal hot lists by size
                                  descending (ties: ascending cluster id) round-robin over ranks
                                  ("sorted by size and distributed to GPU shards in a
                                  round-robin fashion") */
} vlr_index_desc;

/*
 * Process/device placement. world == 1: a single-GPU index.
 * world > 1 with nccl_unique_id != NULL: rank `rank` of an NCCL communicator
 *   (the 128-byte ncclUniqueId, created by rank 0 and broadcast by the caller,
 *   e.g. through torch.distributed); vlr_load_index and vlr_search* are then
 *   COLLECTIVE: every rank calls them with identical arguments (SPMD).
 *   Partitioning: the hot lists are dealt over
 *   the ranks (below), and the COARSE QUANTIZER is sharded too: rank r filters
 *   only its contiguous range of 128-centroid tiles, the ranks exchange their
 *   nprobe' smallest group minima (all-gather 1), each rank refines its own
 *   candidates exactly and the ranks exchange their sorted top-nprobe' exact
 *   (distance, cluster) lists (all-gather 2); every rank then holds the exact
 *   global probes (bitwise those of world == 1). The partial top-k of the
 *   owned probes are all-gathered and merged on every rank (all-gather 3).
 *   The communicator is non-blocking: every NCCL step, and vlr_search's wait,
 *   is bounded by the environment variable VLR_NCCL_TIMEOUT_MS (default
 *   300000); an NCCL error or that timeout aborts the communicator and
 *   returns VLR_ERR_NCCL (the handle is then unusable; free it).
 *   VLR_COARSE_REPLICATED=1 at load: every rank runs the full coarse stage
 *   instead (no coarse exchanges; for comparison).
 * world > 1 with nccl_unique_id == NULL: "shard-only" mode: this handle holds
 *   rank `rank`'s share of the hot lists. vlr_search runs the replicated
 *   coarse stage and returns this shard's PARTIAL top-k; the staged calls
 *   (vlr_coarse_stage1/2, vlr_search_stage3) run the sharded coarse stage
 *   with the exchanges done by the caller. Combine shards with
 *   vlr_merge_partials. (Used to test sharding on one GPU, and for callers
 *   that bring their own transport.)
 * Fault injection (tests): VLR_FAULT_STALL_US=n delays every search of a
 *   handle with a communicator by a bounded n-microsecond device stall before
 *   its first collective.
 */
typedef struct {
  int32_t rank;
  int32_t world;
  int32_t device;               /* CUDA device ordinal used by this handle */
  const void* nccl_unique_id;   /* NULL or pointer to a 128-byte ncclUniqueId */
} vlr_comm_desc;

/* Build the device-resident hot shard of this rank (H2D copies + layout
 * kernel K0 + tables). Synchronous. comm may be NULL (= {0, 1, current device, NULL}). */
vlr_status vlr_load_index(const vlr_index_desc* desc, const vlr_comm_desc* comm, vlr_index** out);

/*
 * Batched search (stream-ordered, no host synchronisation; CUDA-graph
 * capturable once vlr_reserve has sized the workspace for (nq, nprobe, k)).
 * Internally the LUT build runs on a handle-owned side stream forked from and
 * joined back to `stream` with events (VLR_LUT_SERIAL=1 keeps it on `stream`);
 * all work is complete when `stream`'s work up to this call is complete.
 *
 *  d_queries [nq][d] device fp32.   nq >= 0 (nq == 0 is a no-op).
 *  nprobe >= 1; clamped to nprobe' = min(nprobe, nlist); nprobe' <= 2048
 *  (the paper's operating point), else VLR_ERR_UNSUPPORTED.
 *  1 <= k <= 1024. k <= 32: warp-register top-k fused into the scan; k > 32:
 *  the scan writes every candidate's distance and a per-query radix select
 *  keeps the k smallest (same unique result).
 *  world x nprobe' <= 16384 and (k > 32) world x k <= 8192 when world > 1.
 *  Outputs (device, caller-allocated):
 *   d_ids  [nq][k] int64, d_dist [nq][k] fp32: row q = the k smallest
 *      candidates by (ADC distance, id), ascending; missing slots (-1, +inf).
 *      Distances are dist(q, xhat) of the PQ reconstruction, computed as
 *      ||q-c_l||^2 + (||yhat||^2 + 2<c_l,yhat>) - 2<q,yhat> in fp32 for the
 *      default residual L2 index (the other variants drop the c_l terms or
 *      use -<q,c_l> - <q,yhat>; within 1e-5 relative of
 *      the fp64 definition).
 *      Candidates are the vectors of probed lists that are GPU-resident.
 *   d_miss [nq][nprobe'] uint8: 1 iff probe p of query q is not resident on
 *      any GPU; hit rate eta_q = 1 - mean_p d_miss[q][p].
 *   d_probes [nq][nprobe'] int32 or NULL: the probed cluster ids, ascending by
 *      (exact fp64 coarse distance dist(q, c_l), cluster id) (bit-exact
 *      w.r.t. the definition in DESIGN.md §O2).
 *  Errors: INVALID_ARG / UNSUPPORTED synchronously; a non-finite query is
 *  detected on the device and reported by vlr_search, or by the next
 *  vlr_search_async/vlr_search on this handle.
 */
vlr_status vlr_search_async(vlr_index* idx, const float* d_queries, int32_t nq, int32_t nprobe, int32_t k,
                            int64_t* d_ids, float* d_dist, uint8_t* d_miss, int32_t* d_probes, void* stream);

/* vlr_search_async + wait for completion + device status check. With a
 * communicator the wait polls the stream and the communicator's asynchronous
 * error state, bounded by VLR_NCCL_TIMEOUT_MS (-> VLR_ERR_NCCL, see above). */
vlr_status vlr_search(vlr_index* idx, const float* d_queries, int32_t nq, int32_t nprobe, int32_t k,
                      int64_t* d_ids, float* d_dist, uint8_t* d_miss, int32_t* d_probes, void* stream);

/* End-to-end search with HOST buffers (same semantics and shapes as
 * vlr_search): copies h_queries to the device, searches, copies the results
 * back and synchronises `stream`. Pinned host memory gives full PCIe speed.
 * h_probes may be NULL. */
vlr_status vlr_search_host(vlr_index* idx, const float* h_queries, int32_t nq, int32_t nprobe, int32_t k,
                           int64_t* h_ids, float* h_dist, uint8_t* h_miss, int32_t* h_probes, void* stream);

/*
 * NEXT-4: early per-query release -- the GPU analog of the paper's dynamic
 * dispatcher (P:408-414 [§IV.C]: "GPU ... completion flags", "per-query
 * callback" so a finished query does not wait for its batch; Fig. 14).
 * Same search and outputs as vlr_search_async, but the scan runs on all SMs
 * but one with even CTAs walking their queries backward (so queries complete
 * throughout the scan), and a resident merger CTA (on the
 * remaining SM, forked onto a second stream and joined back to `stream`)
 * merges each query's partial lists as soon as the scan has finished the
 * query, in completion order, then raises ready[q] = epoch; the queries still
 * unreleased when the scan ends are merged by a follow-up kernel over all SMs
 * (no separate K7 launch).
 *   ready [nq] uint32: flags, device-accessible -- device memory or pinned
 *      host memory (cudaHostAlloc / cudaMallocHost, used through its UVA
 *      pointer); the caller sets them != epoch before the call.
 *   epoch: nonzero value that marks "row q final" for this call (use a new
 *      value per search on the same flags).
 *   d_ids / d_dist: as vlr_search_async, and may also be pinned host memory;
 *      row q is final (and visible to the host) once ready[q] == epoch (the
 *      row is written before the flag with system-scope release ordering).
 *   d_miss / d_probes: device memory, valid at stream completion as usual.
 * Rows with no resident probe are released first, as padding. Results are
 * bit-identical to vlr_search_async (same distances, same merge code). Not
 * graph-capturable (the epoch is a launch argument).
 * Sharded (world > 1: shard-only handles, or a communicator with the sharded
 * coarse stage): every rank releases ITS partial rows (its owned probes only;
 * no result all-gather), and the dispatcher merges the shards' rows per query
 * with vlr_merge_ready as soon as every shard has released it.
 * Across processes, put the rows and flags in host memory every rank maps
 * (e.g. POSIX shared memory registered with cudaHostRegister).
 * Errors: as vlr_search_async; UNSUPPORTED for k > 32, or a communicator
 * with VLR_COARSE_REPLICATED=1; INVALID_ARG for epoch 0, NULL or
 * non-device-accessible ready/ids/dist.
 */
vlr_status vlr_search_release_async(vlr_index* idx, const float* d_queries, int32_t nq, int32_t nprobe, int32_t k,
                                    int64_t* d_ids, float* d_dist, uint8_t* d_miss, int32_t* d_probes,
                                    uint32_t* ready, uint32_t epoch, void* stream);

/* Host-side dispatcher poll for vlr_search_release_async (the
 * thread-safe queue feeding per-query callbacks): spins until at least one
 * query q < nq with seen[q] == 0 has ready[q] == epoch, or timeout_us passes.
 * Each newly ready q is appended to out_q (at most max_out), seen[q] is set to
 * 1, and out_t_ns (may be NULL) receives the CLOCK_MONOTONIC time in ns at
 * which the flag was observed. Returns the number appended (0 on timeout), -1
 * for bad arguments. An acquire fence follows the flag reads, so the rows of
 * the returned queries can be read after the call. Host only; no CUDA calls. */
int32_t vlr_poll_ready(const uint32_t* ready, int32_t nq, uint32_t epoch, uint8_t* seen, int32_t* out_q,
                       int64_t* out_t_ns, int32_t max_out, int64_t timeout_us);

/* The cross-rank dispatcher merge of NEXT-4 (host only): ready[s] [nq] flags
 * and part_ids[s] / part_dist[s] [nq][k] partial rows of shard s (as released
 * by vlr_search_release_async on each shard, host-visible). Spins until every
 * query is released by all n_shards shards or timeout_us passes; each query's
 * row out_ids/out_dist [nq][k] is written as soon as its last shard released
 * it: the k smallest (dist, id) of the shards' sorted rows. out_t_ns (may be
 * NULL) [nq]: CLOCK_MONOTONIC ns when q was merged. Returns the number of
 * merged queries (nq on success), -1 for bad arguments. */
int32_t vlr_merge_ready(int32_t n_shards, const uint32_t* const* ready, uint32_t epoch, int32_t nq, int32_t k,
                        const int64_t* const* part_ids, const float* const* part_dist, int64_t* out_ids,
                        float* out_dist, int64_t* out_t_ns, int64_t timeout_us);

/* Native dispatcher loop for vlr_search_release_async without per-query
 * callbacks: spins until every q < nq has ready[q] == epoch or timeout_us
 * passes; out_t_ns (may be NULL) [nq] receives, per query, the
 * CLOCK_MONOTONIC time in ns at which its flag was first observed. Returns
 * the number of released queries (nq on success), -1 for bad arguments. An
 * acquire fence follows the flag reads. Host only; no CUDA calls. */
int32_t vlr_wait_ready(const uint32_t* ready, int32_t nq, uint32_t epoch, int64_t* out_t_ns, int64_t timeout_us);

/* vlr_search_host without the final synchronisation (serving pipelines):
 * the search and the D2H copies are enqueued on `stream`, the H2D copy of the
 * queries on a handle-owned copy stream into one of two staging buffers used
 * in turn (events order it after the previous reader of that buffer and
 * before the search), and the call returns; h_* outputs are valid once
 * `stream` has completed this work (cudaStreamSynchronize / an event).
 * Back-to-back calls keep the GPU busy across batches: batch i+1's H2D copy
 * overlaps batch i's kernels. h_queries and the outputs must be pinned host
 * memory (pageable memory makes the copies synchronous) and stay valid until
 * completion. Under stream capture the copy stays on `stream`. A non-finite
 * query is reported by the next call on the handle. */
vlr_status vlr_search_host_async(vlr_index* idx, const float* h_queries, int32_t nq, int32_t nprobe, int32_t k,
                                 int64_t* h_ids, float* h_dist, uint8_t* h_miss, int32_t* h_probes, void* stream);

/*
 * Staged search (shard-only handles: world > 1, nccl_unique_id == NULL): the
 * collective search of one batch cut at its exchange points, so that the
 * caller moves the data between ranks (any transport). Every rank calls, in
 * order, on the same stream, with the same queries and arguments:
 *  1. vlr_coarse_stage1 -> d_x1 [nq][nprobe'] fp32 (device): this rank's
 *     nprobe' smallest filter group minima (K1 on its centroid tiles, K2).
 *     The caller all-gathers x1 in rank order -> x1_all [world][nq][nprobe'].
 *  2. vlr_coarse_stage2(x1_all) -> d_x2 [nq][nprobe'] 16-byte entries
 *     {double D; int32 l; int32 pad} (device): this rank's candidates refined
 *     exactly (fp64), its top nprobe' sorted by (D, l),
 *     padding (+inf, -1). The caller all-gathers x2 -> x2_all
 *     [world][nq][nprobe'] entries.
 *  3. vlr_search_stage3(x2_all) -> the exact global probes and miss mask (as
 *     vlr_search_async, identical on every rank) and THIS SHARD's partial
 *     top-k in d_ids / d_dist; the caller gathers the partials and merges them
 *     with vlr_merge_partials.
 * Constraints: world x nprobe' <= 16384; 1 <= k <= 32; nq >= 1; the calls of
 * one batch must not be interleaved with other searches on the handle
 * (INVALID_ARG otherwise). Status and errors as vlr_search_async.
 */
vlr_status vlr_coarse_stage1(vlr_index* idx, const float* d_queries, int32_t nq, int32_t nprobe, float* d_x1,
                             void* stream);
vlr_status vlr_coarse_stage2(vlr_index* idx, const float* d_queries, int32_t nq, int32_t nprobe,
                             const float* d_x1_all, void* d_x2, void* stream);
vlr_status vlr_search_stage3(vlr_index* idx, const float* d_queries, int32_t nq, int32_t nprobe, int32_t k,
                             const void* d_x2_all, int64_t* d_ids, float* d_dist, uint8_t* d_miss,
                             int32_t* d_probes, void* stream);

/*
 * NVLink peer exchange: the three exchanges of the collective
 * search (coarse stage 1, coarse stage 2, results) without NCCL calls. Each
 * rank owns an inbox (device memory, IPC-exported); the producer kernels (K2
 * stage 1, K3b local, K7) store their slabs straight into every rank's inbox
 * over NVLink and the last CTA raises a per-rank flag (system-scope release);
 * the consumer kernels (K2 stage 2, K3b merge, K8) wait for all flags
 * (acquire, bounded: a missing peer sets status bit 2 -> VLR_ERR_CUDA, no
 * hang). Searches after connect are COLLECTIVE on every rank and return the
 * FINAL rows (shard-only handles too); batches up to the caps reserved before
 * the export (vlr_reserve; k <= 32), no early release.
 *  vlr_p2p_export(idx, out64): allocates the inbox, writes its 64-byte IPC handle.
 *  vlr_p2p_connect(idx, handles): handles [world][64] in rank order (exchanged
 *    by the caller, e.g. torch.distributed); opens every peer's inbox.
 *  vlr_p2p_setup(idx): export + all-gather of the handles over the handle's
 *    NCCL communicator + connect (collective).
 */
vlr_status vlr_p2p_export(vlr_index* idx, void* handle_out);
vlr_status vlr_p2p_connect(vlr_index* idx, const void* handles);
vlr_status vlr_p2p_setup(vlr_index* idx);

/* Pre-size the per-handle workspace (every slot, see vlr_set_pipeline) for
 * batches up to (max_nq, max_nprobe, max_k) so that later searches allocate
 * nothing (required before graph capture). */
vlr_status vlr_reserve(vlr_index* idx, int32_t max_nq, int32_t max_nprobe, int32_t max_k);

/*
 * Cross-batch pipelining. slots = 1 (default) or 2 workspace
 * slots; search number i on the handle uses slot i % slots. With 2 slots a
 * search first makes its stream wait (event) for the previous search of its
 * slot, so searches enqueued on two different streams overlap on the device:
 * batch i+1's coarse stage (K1-K5) runs beside batch i's scan. Searches on
 * one stream stay ordered; results are bitwise those of slots = 1.
 * scan_reserve_sms in [0, SMs - 2]: SMs the scan's persistent grid leaves
 * free for the other stream's coarse stage (0 = one scan CTA per SM).
 * With the peer exchange every rank must use the same slot count (set
 * before vlr_p2p_export; UNSUPPORTED after) and issue the same searches in
 * the same order. Not under stream capture (a captured search uses its slot
 * without the event). Memory: one workspace per slot. INVALID_ARG for bad
 * values. Initial scan reserve: env VLR_SCAN_RESERVE (else 0).
 */
vlr_status vlr_set_pipeline(vlr_index* idx, int32_t slots, int32_t scan_reserve_sms);

/*
 * Merge S shard-partial results (shard-only mode) into the final top-k:
 * d_part_ids [S][nq][k], d_part_dist [S][nq][k] device -> d_ids/d_dist [nq][k]
 * (the k smallest by (dist, id) of the union; "merges ... re-ranks them
 * to obtain the final top-k"). Stream-ordered.
 */
vlr_status vlr_merge_partials(const int64_t* d_part_ids, const float* d_part_dist, int32_t n_shards,
                              int32_t nq, int32_t k, int64_t* d_ids, float* d_dist, void* stream);

/* Cluster access profile (NEXT-2; P:254 access-frequency profiling, P:419
 * runtime monitoring): d_counts[l] += number of entries of d_probes[0..n)
 * equal to l (entries < 0 or >= nlist are ignored). d_probes is the device
 * probe output of vlr_search* (any n = nq * nprobe'); d_counts is a device
 * int64 [nlist] array the caller zeroes. Stream-ordered. */
vlr_status vlr_access_counts(const vlr_index* idx, const int32_t* d_probes, int64_t n, int64_t* d_counts,
                             void* stream);

/* NEXT-2 index splitter: owner rank of each hot list, written to
 * out_owner[i] for hot[i] (host arrays; list_offsets [nlist+1] as in
 * vlr_index_desc). counts == NULL: the paper's deal -- size descending, ties
 * by ascending cluster id, round-robin over `world` ranks (the default
 * of vlr_load_index). counts [nlist] (access counts of a calibration stream,
 * e.g. vlr_access_counts): traffic-aware deal -- load = size x (count + 1),
 * descending, each list to the least-loaded rank (greedy LPT). Pass the
 * result as vlr_index_desc.hot_owner. Host only. INVALID_ARG /
 * UNKNOWN_CLUSTER as vlr_load_index. */
vlr_status vlr_deal_owners(const int64_t* list_offsets, int32_t nlist, const int64_t* counts, const int32_t* hot,
                           int32_t n_hot, int32_t world, int32_t* out_owner);

/* NEXT-2 shard refresh (P:416-425 [§IV.D]: re-profile, re-partition, reload
 * the shard; "<10 s per shard"): rebuild this handle's resident lists
 * for a new hot set / owner assignment in `desc` (same d, nlist, m, nbits,
 * metric, by_residual as the handle, else INVALID_ARG; all arrays host,
 * copied). The new residency is built in fresh device memory while the
 * current one keeps serving: searches issued from other host threads
 * meanwhile run on the old residency. Then, after the device has finished
 * the work already enqueued, the handle switches atomically (w.r.t. this
 * library's calls) and the old residency is freed. Peak device memory = old
 * + new shard. Synchronous; not collective (with world > 1, each rank
 * refreshes its own shard and the caller keeps the owner tables consistent,
 * e.g. by passing the same desc on every rank). Errors as vlr_load_index; on
 * error the handle is unchanged. */
vlr_status vlr_update_hot(vlr_index* idx, const vlr_index_desc* desc);

/* Device bytes held by the handle, number of resident lists and vectors on this rank. */
vlr_status vlr_index_info(const vlr_index* idx, int64_t* bytes_on_device, int32_t* n_owned_lists,
                          int64_t* n_owned_vectors);

/* Owner rank of every cluster (-1 = not resident): out [nlist] int32 host. */
vlr_status vlr_index_owners(const vlr_index* idx, int32_t* out_owner);

/* Per-stage device timing of subsequent searches (CUDA events recorded on the
 * search stream into a ring of the last 64 searches). Stage order: 0 coarse
 * filter (qprep + K1), 1 select (K2), 2 refine (K3), 3 route (K4), 4 LUT (K5),
 * 5 scan (K6), 6 rank merge (K7), 7 exchange + merge (K8).
 * enable: 0 off, 1 every stage boundary (9 events per search), 2 only the
 * two events around the scan (the bench's timed region: stage 5 valid, the
 * others NaN). vlr_stage_times waits for search number `back` before the
 * last one (back = 0: the last search; back < 64) and writes min(n, 8) ms
 * values. INVALID_ARG for another mode or a search that was not recorded. */
vlr_status vlr_set_profiling(vlr_index* idx, int32_t enable);
vlr_status vlr_stage_times(vlr_index* idx, int32_t back, float* ms, int32_t n);

/* Number of kernel launches issued by the last search on this handle. */
int32_t vlr_last_launch_count(const vlr_index* idx);

/* Create an NCCL unique id (rank 0 of a world > 1 job) into out[128]; the
 * caller distributes it to the other ranks (e.g. torch.distributed.broadcast). */
vlr_status vlr_nccl_unique_id(void* out128);

void vlr_index_free(vlr_index* idx);
const char* vlr_last_error(void);
int32_t vlr_version(void); /* (major << 16) | minor */

#ifdef __cplusplus
}
#endif
#endif /* VLR_H_ */

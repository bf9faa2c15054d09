/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for batched IVF-PQ
 * search over the GPU-resident ("hot") inverted lists (VectorLiteRAG,
 * arXiv 2504.08930).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this code. The
 * product path (paper_2504_08930_b200/, include/vlr.h) never links or calls
 * it, and shares no code, header, table or constant with it.
 *
 * Arithmetic: IEEE-754 fp64, sums taken strictly in index order, compiled
 * with -O2 -ffp-contract=off (no FMA contraction, no -ffast-math), so every
 * value is a fixed sequence of correctly-rounded operations.
 *
 * What it computes (§II.B "Search Operation in IVF Index",
 * and Fig. 2 caption PAPER.md:117; readings in DESIGN.md §Readings):
 *   O2  D[q,l] = sum_{t=0}^{d-1} (q_t - c_{l,t})^2                (stage 1)
 *   O3  probes[q] = first nprobe' = min(nprobe, nlist) clusters of the list
 *       of (D[q,l], l) sorted ascending (ties by cluster id, reading A7)
 *   O4  miss[q][p] = 1 iff probes[q][p] is not in the hot set
 *       ("clusters ... that fall within the cached hot cluster set")
 *   O5  candidates: every vector of every probed list with miss = 0
 *   O6  dist_i = sum_t (q_t - xhat_{i,t})^2, xhat_i = c_l + concat_j Y[j][code_ij]
 *       (residual PQ, reading A2; sub-space j = dims [j*dsub,(j+1)*dsub), A5)
 *       -- "the exact distance to the PQ-reconstructed vector", the quantity
 *       the LUT of stage 2/3 accumulates.
 *   O7  result: k smallest candidates by (dist, id), padded with (-1, +inf);
 *       also the (k+1)-th distance (for the tie rule R3).
 * Variants (NEXT-3, readings A1'/A2'/A4' in DESIGN.md §2):
 *   nbits = 4 (the paper's 4-bit PQ): 16 codewords per
 *       sub-space, Y is [m][16][dsub], a code row has ceil(m/2) bytes and
 *       sub-code j is the low nibble of byte j/2 for even j, the high nibble
 *       for odd j;
 *   by_residual = 0: xhat_i = concat_j Y[j][code_ij] (no centroid term);
 *   metric = 1 (inner product, "independent of the distance metric",
 *       PAPER.md:243): coarse key D[q,l] = -<q, c_l> and dist_i = -<q, xhat_i>,
 *       each summed sequentially in t-order; ranking ascending by these
 *       negated inner products is ranking by descending similarity.
 * Pins: tests/test_oracle_pins.py (see DESIGN.md §Oracle pins).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---- O2: exact coarse distance, sequential fp64 sum ---- */
double oracle_coarse_dist(const float* q, const float* c, int32_t d) {
    double s = 0.0;
    for (int32_t t = 0; t < d; ++t) {
        double diff = (double)q[t] - (double)c[t];
        double sq = diff * diff;
        s = s + sq;
    }
    return s;
}

/* ---- O2 (metric = 1): exact negated inner product, sequential fp64 sum ---- */
double oracle_coarse_ip(const float* q, const float* c, int32_t d) {
    double s = 0.0;
    for (int32_t t = 0; t < d; ++t) {
        double pr = (double)q[t] * (double)c[t];
        s = s + pr;
    }
    return -s;
}

static double coarse_key(const float* q, const float* c, int32_t d, int32_t metric) {
    return metric == 1 ? oracle_coarse_ip(q, c, d) : oracle_coarse_dist(q, c, d);
}

typedef struct { double d; int64_t id; } pair_t;

static int cmp_pair(const void* a, const void* b) {
    const pair_t* x = (const pair_t*)a;
    const pair_t* y = (const pair_t*)b;
    if (x->d < y->d) return -1;
    if (x->d > y->d) return 1;
    if (x->id < y->id) return -1;
    if (x->id > y->id) return 1;
    return 0;
}

/* ---- O3: probes = first nprobe' of sort by (D, l) ---- */
int oracle_coarse(const float* Q, int64_t nq, const float* C, int32_t nlist, int32_t d,
                  int32_t nprobe, int32_t* probes, double* probe_dist, int32_t metric, int32_t nthreads) {
    if (nprobe < 1 || nlist < 1 || d < 1 || metric < 0 || metric > 1) return 1;
    int32_t np = nprobe < nlist ? nprobe : nlist;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic)
#endif
    for (int64_t qi = 0; qi < nq; ++qi) {
        pair_t* all = (pair_t*)malloc(sizeof(pair_t) * (size_t)nlist);
        for (int32_t l = 0; l < nlist; ++l) {
            all[l].d = coarse_key(Q + qi * d, C + (int64_t)l * d, d, metric);
            all[l].id = l;
        }
        qsort(all, (size_t)nlist, sizeof(pair_t), cmp_pair);
        for (int32_t p = 0; p < np; ++p) {
            probes[qi * np + p] = (int32_t)all[p].id;
            if (probe_dist) probe_dist[qi * np + p] = all[p].d;
        }
        free(all);
    }
    return 0;
}

/* ---- O6: distance of query q to the reconstruction of vector `pos` of
 * list l: xhat = c_l + concat_j Y[j][code_j] formed in fp64 ---- */
double oracle_adc_dist(const float* q, const float* c_l, const float* Y, const uint8_t* code,
                       int32_t d, int32_t m) {
    int32_t dsub = d / m;
    double s = 0.0;
    for (int32_t t = 0; t < d; ++t) {
        int32_t j = t / dsub;
        int32_t u = t - j * dsub;
        double y = (double)Y[((int64_t)j * 256 + code[j]) * dsub + u];
        double xh = (double)c_l[t] + y;
        double diff = (double)q[t] - xh;
        double sq = diff * diff;
        s = s + sq;
    }
    return s;
}

/* sub-code j of a code row: byte j (nbits 8), or nibble j (nbits 4: low
 * nibble of byte j/2 for even j, high nibble for odd j) */
static int32_t subcode(const uint8_t* code, int32_t j, int32_t nbits) {
    if (nbits == 8) return code[j];
    return (code[j >> 1] >> (4 * (j & 1))) & 15;
}

/* bytes of one code row */
static int64_t row_bytes(int32_t m, int32_t nbits) { return ((int64_t)m * nbits + 7) / 8; }

/* ---- O6 variants: xhat = [c_l +] concat_j Y[j][code_j] (by_residual), and
 * dist = sum_t (q_t - xhat_t)^2 (metric 0) or -sum_t q_t xhat_t (metric 1) ---- */
double oracle_adc_dist_v(const float* q, const float* c_l, const float* Y, const uint8_t* code,
                         int32_t d, int32_t m, int32_t nbits, int32_t metric, int32_t by_residual) {
    if (metric == 0 && by_residual && nbits == 8) return oracle_adc_dist(q, c_l, Y, code, d, m);
    int32_t dsub = d / m;
    int32_t ksub = 1 << nbits;
    double s = 0.0;
    for (int32_t t = 0; t < d; ++t) {
        int32_t j = t / dsub;
        int32_t u = t - j * dsub;
        double xh = (double)Y[((int64_t)j * ksub + subcode(code, j, nbits)) * dsub + u];
        if (by_residual) xh = (double)c_l[t] + xh;
        if (metric == 1) {
            double pr = (double)q[t] * xh;
            s = s + pr;
        } else {
            double diff = (double)q[t] - xh;
            double sq = diff * diff;
            s = s + sq;
        }
    }
    return metric == 1 ? -s : s;
}

/* keep the kk smallest (dist,id) pairs in best[0..kk-1] (sorted) by insertion */
static void insert_best(pair_t* best, int32_t kk, double dist, int64_t id) {
    pair_t v; v.d = dist; v.id = id;
    if (cmp_pair(&v, &best[kk - 1]) >= 0) return;
    int32_t i = kk - 1;
    while (i > 0 && cmp_pair(&v, &best[i - 1]) < 0) { best[i] = best[i - 1]; --i; }
    best[i] = v;
}

/*
 * Full search, O2-O7. is_hot[l] in {0,1} marks GPU-resident clusters.
 * Outputs: out_ids/out_dist [nq*k], miss/probes [nq*nprobe'], kth1 [nq]
 * (the (k+1)-th smallest candidate distance, +inf if fewer than k+1),
 * ncand [nq] (number of candidates scanned). Any output pointer may be NULL
 * except out_ids/out_dist.
 */
int oracle_search(const float* Q, int64_t nq, int32_t d, const float* C, int32_t nlist,
                  const float* Y, int32_t m, int32_t nbits, const int64_t* offsets, const int64_t* ids,
                  const uint8_t* codes, const uint8_t* is_hot, int32_t nprobe, int32_t k,
                  int64_t* out_ids, double* out_dist, uint8_t* miss, int32_t* probes,
                  double* kth1, int64_t* ncand, int32_t metric, int32_t by_residual, int32_t nthreads) {
    if (nprobe < 1 || k < 1 || m < 1 || d % m != 0 || metric < 0 || metric > 1) return 1;
    if (nbits != 8 && nbits != 4) return 1;
    const int64_t rb = row_bytes(m, nbits);
    int32_t np = nprobe < nlist ? nprobe : nlist;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic)
#endif
    for (int64_t qi = 0; qi < nq; ++qi) {
        const float* q = Q + qi * d;
        /* O2 + O3 */
        pair_t* all = (pair_t*)malloc(sizeof(pair_t) * (size_t)nlist);
        for (int32_t l = 0; l < nlist; ++l) {
            all[l].d = coarse_key(q, C + (int64_t)l * d, d, metric);
            all[l].id = l;
        }
        qsort(all, (size_t)nlist, sizeof(pair_t), cmp_pair);
        /* O4 + O5 + O6 + O7 */
        int32_t kk = k + 1;
        pair_t* best = (pair_t*)malloc(sizeof(pair_t) * (size_t)kk);
        for (int32_t i = 0; i < kk; ++i) { best[i].d = INFINITY; best[i].id = -1; }
        int64_t nc = 0;
        for (int32_t p = 0; p < np; ++p) {
            int32_t l = (int32_t)all[p].id;
            uint8_t is_miss = is_hot[l] ? 0 : 1;
            if (probes) probes[qi * np + p] = l;
            if (miss) miss[qi * np + p] = is_miss;
            if (is_miss) continue;
            for (int64_t i = offsets[l]; i < offsets[l + 1]; ++i) {
                double dist = oracle_adc_dist_v(q, C + (int64_t)l * d, Y, codes + i * rb, d, m, nbits, metric,
                                                by_residual);
                insert_best(best, kk, dist, ids[i]);
                ++nc;
            }
        }
        for (int32_t i = 0; i < k; ++i) {
            out_ids[qi * k + i] = best[i].d == INFINITY ? -1 : best[i].id;
            out_dist[qi * k + i] = best[i].d;
        }
        if (kth1) kth1[qi] = best[k].d;
        if (ncand) ncand[qi] = nc;
        free(best);
        free(all);
    }
    return 0;
}

/*
 * dist_ref(q, vector): O6 for explicit (query row, list, position) triples,
 * used to check every distance the GPU returns (rule R2).
 */
int oracle_dist_many(const float* Q, int32_t d, const float* C, const float* Y, int32_t m, int32_t nbits,
                     const uint8_t* codes, const int64_t* qidx, const int32_t* list,
                     const int64_t* pos, int64_t n, double* out, int32_t metric, int32_t by_residual,
                     int32_t nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
    for (int64_t i = 0; i < n; ++i)
        out[i] = oracle_adc_dist_v(Q + qidx[i] * d, C + (int64_t)list[i] * d, Y, codes + pos[i] * row_bytes(m, nbits),
                                   d, m, nbits, metric, by_residual);
    return 0;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

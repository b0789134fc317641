/*
 * knnm_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C (OpenMP) restatement of the reference's numba kernels on the
 * S-Merge / J-Merge hot path (`knnmerge/_kernels.py`, reference package
 * under pkg/src/knnmerge/).  It is the checker for the CUDA path and the
 * CPU baseline leg of bench.py; nothing in paper_1908_00814_b200/ links,
 * imports or calls it.
 *
 * Parity status: pinned.  tests/test_oracle_golden.py checks the full
 * merges built on these functions against golden vectors produced by the
 * reference itself (tests/golden/make_golden.py).
 *
 * Arithmetic contract (mirrors numba without fastmath): fp64 accumulation
 * of fp32 inputs, strictly sequential, no FMA contraction.  This file MUST
 * be compiled with -ffp-contract=off (see oracle/Makefile).
 *
 * Layout (reference _kernels.py:1-15): ids int32 (m,cap) padded -1,
 * dists float64 (m,cap) padded +inf, flags uint8 (m,cap), sizes int32 (m).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define TAG_L1 0
#define TAG_L2 1
#define TAG_COSINE 2

#define MODE_ALL 0
#define MODE_CROSS 1
#define MODE_CROSS_OR_S2 2

static const uint64_t U64_GAMMA = 0x9E3779B97F4A7C15ULL;
static const uint64_t U64_MIX1 = 0xBF58476D1CE4E5B9ULL;
static const uint64_t U64_MIX2 = 0x94D049BB133111EBULL;

/* _kernels.py:43-80 dense_dist */
double orc_dense_dist(const float *a, const float *b, int64_t d, int tag) {
    if (tag == TAG_L1) {
        double acc = 0.0;
        for (int64_t t = 0; t < d; t++) acc += fabs((double)a[t] - (double)b[t]);
        return acc;
    } else if (tag == TAG_L2) {
        double acc = 0.0;
        for (int64_t t = 0; t < d; t++) {
            double diff = (double)a[t] - (double)b[t];
            acc += diff * diff;
        }
        return acc;
    } else {
        double dot = 0.0, na = 0.0, nb = 0.0;
        for (int64_t t = 0; t < d; t++) {
            double x = (double)a[t], y = (double)b[t];
            dot += x * y;
            na += x * x;
            nb += y * y;
        }
        if (na == 0.0 || nb == 0.0) return (na == nb) ? 0.0 : 1.0;
        if (dot > 0.0 && dot * dot >= na * nb) return 0.0;
        double r = 1.0 - dot / (sqrt(na) * sqrt(nb));
        return r < 0.0 ? 0.0 : r;
    }
}

/* _kernels.py:113-119 pair_dists_dense */
void orc_pair_dists(const float *data, int64_t d, const int32_t *pa,
                    const int32_t *pb, int64_t m, int tag, double *out) {
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < m; t++)
        out[t] = orc_dense_dist(data + (int64_t)pa[t] * d,
                                data + (int64_t)pb[t] * d, d, tag);
}

/* _kernels.py:159-192 _insert (spec twin: graph.py:54-81 update_nn) */
static inline int orc_insert(int32_t *ids, double *dists, uint8_t *flags,
                             int32_t *sizes, int64_t cap, int64_t row,
                             int32_t nid, double nd) {
    if (cap == 0) return 0;
    int32_t *ri = ids + row * cap;
    double *rd = dists + row * cap;
    uint8_t *rf = flags + row * cap;
    int64_t sz = sizes[row];
    if (sz == cap && nd >= rd[sz - 1]) return 0;
    for (int64_t t = 0; t < sz; t++)
        if (ri[t] == nid) return 0;
    int64_t pos = sz;
    for (int64_t t = 0; t < sz; t++) {
        double dt = rd[t];
        if (nd < dt || (nd == dt && nid < ri[t])) { pos = t; break; }
    }
    int64_t last;
    if (sz == cap) {
        last = cap - 1;
    } else {
        last = sz;
        sizes[row] = (int32_t)(sz + 1);
    }
    for (int64_t t = last; t > pos; t--) {
        ri[t] = ri[t - 1];
        rd[t] = rd[t - 1];
        rf[t] = rf[t - 1];
    }
    ri[pos] = nid;
    rd[pos] = nd;
    rf[pos] = 1;
    return 1;
}

int orc_insert_one(int32_t *ids, double *dists, uint8_t *flags, int32_t *sizes,
                   int64_t cap, int64_t row, int32_t nid, double nd) {
    return orc_insert(ids, dists, flags, sizes, cap, row, nid, nd);
}

/* _kernels.py:195-205 apply_updates (sequential reference order) */
int64_t orc_apply_updates(int32_t *ids, double *dists, uint8_t *flags,
                          int32_t *sizes, int64_t cap, const int32_t *pa,
                          const int32_t *pb, const double *pd, int64_t m) {
    int64_t c = 0;
    for (int64_t t = 0; t < m; t++) {
        c += orc_insert(ids, dists, flags, sizes, cap, pa[t], pb[t], pd[t]);
        c += orc_insert(ids, dists, flags, sizes, cap, pb[t], pa[t], pd[t]);
    }
    return c;
}

/* _kernels.py:208-214 apply_updates_directed */
int64_t orc_apply_directed(int32_t *ids, double *dists, uint8_t *flags,
                           int32_t *sizes, int64_t cap, const int32_t *rows,
                           const int32_t *nids, const double *nds, int64_t m) {
    int64_t c = 0;
    for (int64_t t = 0; t < m; t++)
        c += orc_insert(ids, dists, flags, sizes, cap, rows[t], nids[t], nds[t]);
    return c;
}

/* _kernels.py:217-254 apply_updates_grouped: stable counting sort of the
 * 2m directed updates by target row, then rows in parallel. */
int64_t orc_apply_grouped(int32_t *ids, double *dists, uint8_t *flags,
                          int32_t *sizes, int64_t n, int64_t cap,
                          const int32_t *pa, const int32_t *pb,
                          const double *pd, int64_t m) {
    int64_t *indptr = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    for (int64_t t = 0; t < m; t++) {
        indptr[pa[t] + 1]++;
        indptr[pb[t] + 1]++;
    }
    for (int64_t i = 0; i < n; i++) indptr[i + 1] += indptr[i];
    int32_t *src = (int32_t *)malloc(sizeof(int32_t) * (size_t)(indptr[n] + 1));
    double *dd = (double *)malloc(sizeof(double) * (size_t)(indptr[n] + 1));
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
    memcpy(fill, indptr, sizeof(int64_t) * (size_t)n);
    for (int64_t t = 0; t < m; t++) {
        int64_t p = fill[pa[t]]++;
        src[p] = pb[t];
        dd[p] = pd[t];
        p = fill[pb[t]]++;
        src[p] = pa[t];
        dd[p] = pd[t];
    }
    int64_t acc = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : acc)
    for (int64_t r = 0; r < n; r++) {
        int64_t local = 0;
        for (int64_t s = indptr[r]; s < indptr[r + 1]; s++)
            local += orc_insert(ids, dists, flags, sizes, cap, r, src[s], dd[s]);
        acc += local;
    }
    free(indptr);
    free(src);
    free(dd);
    free(fill);
    return acc;
}

/* _kernels.py:262-281 reverse_csr; indptr has n+1 entries, rids/rnew have
 * indptr[n] = sum(sizes) entries. Order: (source row i, slot t). */
void orc_reverse_csr(const int32_t *ids, const uint8_t *flags,
                     const int32_t *sizes, int64_t n, int64_t cap,
                     int64_t *indptr, int32_t *rids, uint8_t *rnew) {
    /* flag 2 = a new entry left out of this round by rho-sampling
     * (orc_sample_new); never present at rho = 1 (the reference) */
    memset(indptr, 0, sizeof(int64_t) * (size_t)(n + 1));
    for (int64_t i = 0; i < n; i++)
        for (int64_t t = 0; t < sizes[i]; t++)
            if (flags[i * cap + t] != 2) indptr[ids[i * cap + t] + 1]++;
    for (int64_t i = 0; i < n; i++) indptr[i + 1] += indptr[i];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
    memcpy(fill, indptr, sizeof(int64_t) * (size_t)n);
    for (int64_t i = 0; i < n; i++)
        for (int64_t t = 0; t < sizes[i]; t++) {
            if (flags[i * cap + t] == 2) continue;
            int64_t j = ids[i * cap + t];
            int64_t p = fill[j]++;
            rids[p] = (int32_t)i;
            rnew[p] = flags[i * cap + t];
        }
    free(fill);
}

/* _kernels.py:306-313 _mix_state (splitmix64 step) */
static inline uint64_t orc_mix(uint64_t *state) {
    *state += U64_GAMMA;
    uint64_t z = *state;
    z = (z ^ (z >> 30)) * U64_MIX1;
    z = (z ^ (z >> 27)) * U64_MIX2;
    return z ^ (z >> 31);
}

/* Sample rate rho < 1 (classic NN-Descent; no reference counterpart, the
 * reference is rho = 1): of row u's new entries (list order p_0 < p_1 <
 * ...), at most new_cap take part in this round, chosen by the reverse
 * sampler's partial Fisher-Yates (splitmix64, state seed ^ SALT ^
 * (u+1)*gamma, one warm-up step); the others get flag 2: skipped by
 * reverse_csr and assemble, and still new after the round. */
#define ORC_FWD_SALT 0x6a09e667f3bcc909ULL
void orc_sample_new(const int32_t *sizes, int64_t n, int64_t cap, uint8_t *flags,
                    int64_t new_cap, uint64_t seed) {
#pragma omp parallel for schedule(static)
    for (int64_t u = 0; u < n; u++) {
        int64_t pos[256];
        int64_t c = 0;
        for (int64_t t = 0; t < sizes[u]; t++)
            if (flags[u * cap + t]) pos[c++] = t;
        if (c <= new_cap) continue;
        uint8_t keep[256];
        memset(keep, 0, sizeof(keep));
        int64_t idx[256];
        for (int64_t t = 0; t < c; t++) idx[t] = t;
        uint64_t state = (seed ^ ORC_FWD_SALT) ^ ((uint64_t)(u + 1) * U64_GAMMA);
        (void)orc_mix(&state);
        for (int64_t t = 0; t < new_cap; t++) {
            uint64_t z = orc_mix(&state);
            int64_t r = t + (int64_t)(z % (uint64_t)(c - t));
            int64_t tmp = idx[t];
            idx[t] = idx[r];
            idx[r] = tmp;
            keep[idx[t]] = 1;
        }
        for (int64_t t = 0; t < c; t++)
            if (!keep[t]) flags[u * cap + pos[t]] = 2;
    }
}

/* _kernels.py:316-383 assemble_neighborhoods.  nbh (n,width) int32 padded
 * -1, nnew (n,width) uint8, nlen (n); width = cap + rev_cap. */
void orc_assemble(const int32_t *ids, const uint8_t *flags,
                  const int32_t *sizes, int64_t n, int64_t cap,
                  const int64_t *rindptr, const int32_t *rids,
                  const uint8_t *rnew, int64_t rev_cap, uint64_t seed,
                  int32_t *nbh, uint8_t *nnew, int32_t *nlen) {
    int64_t width = cap + rev_cap;
#pragma omp parallel
    {
        int32_t *buf_id = (int32_t *)malloc(sizeof(int32_t) * (size_t)(width + 1));
        uint8_t *buf_new = (uint8_t *)malloc((size_t)(width + 1));
        int64_t idx_cap = 0;
        int64_t *idx = NULL;
#pragma omp for schedule(dynamic, 256)
        for (int64_t u = 0; u < n; u++) {
            int32_t *out_id = nbh + u * width;
            uint8_t *out_new = nnew + u * width;
            for (int64_t t = 0; t < width; t++) { out_id[t] = -1; out_new[t] = 0; }
            int64_t m = 0;
            for (int64_t t = 0; t < sizes[u]; t++) {
                if (flags[u * cap + t] == 2) continue; /* sits out (rho) */
                buf_id[m] = ids[u * cap + t];
                buf_new[m] = flags[u * cap + t];
                m++;
            }
            int64_t lo = rindptr[u];
            int64_t deg = rindptr[u + 1] - lo;
            if (deg <= rev_cap) {
                for (int64_t t = 0; t < deg; t++) {
                    buf_id[m] = rids[lo + t];
                    buf_new[m] = rnew[lo + t];
                    m++;
                }
            } else {
                if (deg > idx_cap) {
                    free(idx);
                    idx_cap = deg;
                    idx = (int64_t *)malloc(sizeof(int64_t) * (size_t)idx_cap);
                }
                for (int64_t t = 0; t < deg; t++) idx[t] = t;
                uint64_t state = seed ^ ((uint64_t)(u + 1) * U64_GAMMA);
                (void)orc_mix(&state);
                for (int64_t t = 0; t < rev_cap; t++) {
                    uint64_t z = orc_mix(&state);
                    int64_t r = t + (int64_t)(z % (uint64_t)(deg - t));
                    int64_t tmp = idx[t];
                    idx[t] = idx[r];
                    idx[r] = tmp;
                    int64_t p = lo + idx[t];
                    buf_id[m] = rids[p];
                    buf_new[m] = rnew[p];
                    m++;
                }
            }
            /* insertion sort by id, then compact duplicates OR-ing flags */
            for (int64_t a = 1; a < m; a++) {
                int32_t ki = buf_id[a];
                uint8_t kn = buf_new[a];
                int64_t b = a - 1;
                while (b >= 0 && buf_id[b] > ki) {
                    buf_id[b + 1] = buf_id[b];
                    buf_new[b + 1] = buf_new[b];
                    b--;
                }
                buf_id[b + 1] = ki;
                buf_new[b + 1] = kn;
            }
            int64_t w = 0;
            for (int64_t a = 0; a < m; a++) {
                if (w > 0 && out_id[w - 1] == buf_id[a]) {
                    if (buf_new[a]) out_new[w - 1] = 1;
                } else {
                    out_id[w] = buf_id[a];
                    out_new[w] = buf_new[a];
                    w++;
                }
            }
            nlen[u] = (int32_t)w;
        }
        free(buf_id);
        free(buf_new);
        free(idx);
    }
}

/* _kernels.py:391-399 _pair_admissible */
static inline int orc_admissible(int na, int nb, int la, int lb, int mode) {
    if (!(na || nb)) return 0;
    if (mode == MODE_CROSS) return la != lb;
    if (mode == MODE_CROSS_OR_S2) return la != lb || (la == 1 && lb == 1);
    return 1;
}

/* _kernels.py:402-417 count_pairs over rows [lo, hi) */
void orc_count_pairs(const int32_t *nbh, const uint8_t *nnew,
                     const int32_t *nlen, int64_t width, const int8_t *labels,
                     int mode, int64_t lo, int64_t hi, int64_t *counts) {
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t u = lo; u < hi; u++) {
        int64_t c = 0;
        int64_t w = nlen[u];
        const int32_t *row = nbh + u * width;
        const uint8_t *rn = nnew + u * width;
        for (int64_t p = 0; p < w; p++)
            for (int64_t q = p + 1; q < w; q++)
                c += orc_admissible(rn[p], rn[q], labels[row[p]], labels[row[q]], mode);
        counts[u - lo] = c;
    }
}

/* _kernels.py:420-437 fill_pairs over rows [lo, hi) */
void orc_fill_pairs(const int32_t *nbh, const uint8_t *nnew,
                    const int32_t *nlen, int64_t width, const int8_t *labels,
                    int mode, int64_t lo, int64_t hi, const int64_t *offsets,
                    int32_t *pa, int32_t *pb) {
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t u = lo; u < hi; u++) {
        int64_t pos = offsets[u - lo];
        int64_t w = nlen[u];
        const int32_t *row = nbh + u * width;
        const uint8_t *rn = nnew + u * width;
        for (int64_t p = 0; p < w; p++)
            for (int64_t q = p + 1; q < w; q++)
                if (orc_admissible(rn[p], rn[q], labels[row[p]], labels[row[q]], mode)) {
                    pa[pos] = row[p];
                    pb[pos] = row[q];
                    pos++;
                }
    }
}

/* _kernels.py:529-563 merge_rear_rows; outputs pre-filled by caller is not
 * required: every slot is written. rk = rear row stride. */
void orc_merge_rear_rows(const int32_t *uids, const double *udists,
                         const int32_t *usizes, const int32_t *rids,
                         const double *rdists, const int32_t *rsizes,
                         int64_t n, int64_t k, int64_t rk, int32_t *out_ids,
                         double *out_dists, int32_t *out_sizes) {
#pragma omp parallel for schedule(static)
    for (int64_t u = 0; u < n; u++) {
        const int32_t *ui = uids + u * k;
        const double *ud = udists + u * k;
        const int32_t *ri = rids + u * rk;
        const double *rd = rdists + u * rk;
        int32_t *oi = out_ids + u * k;
        double *od = out_dists + u * k;
        for (int64_t t = 0; t < k; t++) { oi[t] = -1; od[t] = INFINITY; }
        int64_t a = 0, b = 0, w = 0;
        int64_t ua = usizes[u], rb = rsizes[u];
        while (w < k && (a < ua || b < rb)) {
            int32_t cid;
            double cd;
            if (a < ua && (b >= rb || ud[a] < rd[b] ||
                           (ud[a] == rd[b] && ui[a] <= ri[b]))) {
                cid = ui[a];
                cd = ud[a];
                a++;
            } else {
                cid = ri[b];
                cd = rd[b];
                b++;
            }
            int dup = 0;
            for (int64_t t = 0; t < w; t++)
                if (oi[t] == cid) { dup = 1; break; }
            if (!dup) {
                oi[w] = cid;
                od[w] = cd;
                w++;
            }
        }
        out_sizes[u] = (int32_t)w;
    }
}

/* numpy pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
 * pairwise_sum_DOUBLE; block 128, 8 accumulators) -- the arithmetic of
 * construct.py:79-83 `np.where(mask, dists, 0.0).sum()` over the
 * C-contiguous (n,k) array. */
static double orc_pairwise(const double *a, int64_t n) {
    if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; i++) r += a[i];
        return r;
    } else if (n <= 128) {
        double r[8];
        int64_t i;
        for (int j = 0; j < 8; j++) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return orc_pairwise(a, n2) + orc_pairwise(a + n2, n - n2);
    }
}

/* construct.py:79-83 _phi_arrays */
double orc_phi(const double *dists, const int32_t *sizes, int64_t n, int64_t k) {
    if (n * k == 0) return 0.0;
    double *tmp = (double *)malloc(sizeof(double) * (size_t)(n * k));
    for (int64_t u = 0; u < n; u++)
        for (int64_t t = 0; t < k; t++)
            tmp[u * k + t] = (t < sizes[u]) ? dists[u * k + t] : 0.0;
    double r = orc_pairwise(tmp, n * k);
    free(tmp);
    return r;
}

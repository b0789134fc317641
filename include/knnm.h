/*
 * knnm.h -- C-ABI of libknnm.so, the B200 (sm_100a) engine for the
 * cross-subset NN-Descent local join behind S-Merge / J-Merge
 * ("On the Merge of k-NN Graph", arXiv 1908.00814).
 *
 * The reference (`knnmerge`, pkg/src/knnmerge/) has no FFI: its operator
 * layer is a set of numba functions on flat numpy arrays, called as
 * `_k.<name>(...)` from construct.py / merge.py.  Each entry point below
 * names the reference call(s) it replaces (file:line, relative to
 * pkg/src/knnmerge/).  Python binds this header with ctypes
 * (paper_1908_00814_b200/_lib.py); INTEGRATION.md shows the binding.
 *
 * Conventions
 *   - Plain host pointers and sizes only; the library owns all device
 *     memory and copies host<->device itself (stream-ordered on the
 *     context's private CUDA stream).
 *   - Array layout is the reference's (_kernels.py:1-15): ids int32 (n,k)
 *     padded -1, dists float64 (n,k) padded +inf, flags uint8 (n,k),
 *     sizes int32 (n).  Row r of the engine state is local id r, i.e. the
 *     r-th entry of the ascending union of member ids.
 *   - Every function returns KNNM_OK (0) or a negative error code; the
 *     message is available from knnm_last_error() (thread-local).  Input
 *     validation that the reference performs in Python (ValueError) stays
 *     in the Python host layer; these calls return KNNM_ERR_ARG for
 *     contract breaches they can detect.
 *   - A context is not re-entrant; one context per device per thread.
 *   - Arithmetic: distances are bit-identical to the reference's
 *     dense_dist (fp64 accumulation of fp32 inputs, sequential, no FMA),
 *     and list updates replay the reference's sequential per-row insertion
 *     order, so results are bit-exact with the reference.
 */
#ifndef KNNM_H
#define KNNM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KNNM_OK 0
#define KNNM_ERR_CUDA -1   /* CUDA runtime / launch failure            */
#define KNNM_ERR_ARG -2    /* invalid argument                          */
#define KNNM_ERR_STATE -3  /* call out of order (e.g. round before begin) */
#define KNNM_ERR_NOMEM -4  /* device allocation failed                  */
#define KNNM_ERR_LIMIT -5  /* input exceeds a supported bound            */

/* Metric tags (_kernels.py:24-27; core.py:28-51 Metric). */
#define KNNM_L1 0
#define KNNM_L2 1
#define KNNM_COSINE 2

/* Pair-admissibility modes (_kernels.py:29-31). */
#define KNNM_MODE_ALL 0
#define KNNM_MODE_CROSS 1
#define KNNM_MODE_CROSS_OR_S2 2

typedef struct knnm_ctx knnm_ctx;

/* Per-context counters and timings (cumulative since create / reset). */
typedef struct knnm_stats {
    double join_ms;        /* local-join kernel time (CUDA events)        */
    double reverse_ms;     /* reverse CSR build                           */
    double assemble_ms;    /* neighbourhood assembly (+pair counting)     */
    double update_ms;      /* candidate bucketing + sequential insertion  */
    double other_ms;       /* init, phi, export, merge-rear               */
    int64_t join_launches; /* local-join kernel launches                  */
    int64_t pairs;         /* admissible pairs evaluated (= distance evals) */
    int64_t init_evals;    /* init-path distance evaluations              */
    int64_t members;       /* sum over active hoods of |M_u| (members in >=1 pair) */
    int64_t candidates;    /* directed updates surviving the prefilter     */
    int64_t accepted;      /* accepted list insertions                    */
    int64_t rounds;        /* rounds run                                  */
    int64_t exact_evals;   /* pairs re-evaluated in fp64 after fp32 screen */
    int64_t launches;      /* kernels launched by this context            */
    int64_t h2d_bytes;     /* host -> device bytes copied                 */
    int64_t join_redos;    /* optimistic single-shot joins redone in chunks */
    int64_t d2h_bytes;     /* device -> host bytes copied                 */
    double join_kernel_ms; /* local-join kernel alone (roofline denominator) */
    int64_t written_slots; /* update slots the join wrote (prefilter survivors) */
    int64_t join_row_bytes; /* bytes per gathered member row in the join   */
    int64_t heavy_rev_rows; /* reverse segments longer than a warp sorts (block path) */
    int64_t seg_hub_rows;   /* rows with more memberships than a warp ranks (block path) */
    int64_t apply_rows_in;  /* rows the apply loaded (>= 1 update slot)     */
    int64_t apply_rows_out; /* rows the apply stored (>= 1 accepted insert) */
    double apply_kernel_ms; /* the apply kernel alone (roofline denominator) */
    int64_t active_hoods;   /* hoods with >= 1 admissible pair, over all rounds */
    int64_t bf_tc_launches; /* brute-force calls served by the tcgen05 route */
    int64_t lazy_batches;   /* lazy exact-evaluation batches in the apply (pairs: exact_evals) */
    int64_t tc_join_launches; /* local joins on the tcgen05 lazy route (k_join_tc) */
    int64_t dense_join_launches; /* local joins on the fp64 register-tile route (k_join_dense) */
} knnm_stats;

const char *knnm_last_error(void);
int knnm_version(void);

/* Create / destroy an engine bound to CUDA device `device`. */
int knnm_create(int device, knnm_ctx **out);
int knnm_destroy(knnm_ctx *ctx);

/* Upload the dense dataset (Dataset.vectors, core.py:96-104): float32
 * (n_all, d) row-major host array; metric = KNNM_L1/L2/COSINE.  The device
 * copy is kept across merges (tree merges and H-Merge reuse it). */
int knnm_set_dataset(knnm_ctx *ctx, const float *vectors, int64_t n_all,
                     int32_t d, int32_t metric);
/* Host-only content fingerprint of a buffer (threads, no GPU): the Python
 * engine keys its device-resident dataset on it, so an in-place edit of
 * Dataset.vectors is never served from a stale device copy. */
int knnm_fingerprint(const void *p, int64_t bytes, uint64_t *out);

/* Begin a merge or build over `n` local rows.  Replaces
 * `Dataset.take(union_gids)` (core.py:148-166; merge.py:217-219, 297-301),
 * the label setup (merge.py:222-223, 304-305) and the list allocation
 * (merge.py:227-230, 308-311).  union_gids: ascending int64 (n) global ids;
 * labels: int8 (n); k = list capacity. Lists start empty. */
int knnm_begin(knnm_ctx *ctx, const int64_t *union_gids, int64_t n,
               const int8_t *labels, int32_t k);

/* Load one input subgraph.  Replaces split (graph.py:202-229) +
 * _localize_rows (merge.py:129-143) + the rear-list assembly
 * (merge.py:249-256 / 333-335).  rows: int32 (m) local rows of the graph's
 * members; g_ids int32 (m, gk) GLOBAL neighbour ids, g_dists float64 (m,gk),
 * g_sizes int32 (m).  Entries [0,k1) become the list head (flags old);
 * entries [k1,size) are kept as the rear list for knnm_export. */
int knnm_load_graph(knnm_ctx *ctx, const int32_t *rows, int64_t m,
                    const int32_t *g_ids, const double *g_dists,
                    const int32_t *g_sizes, int32_t gk, int32_t k1);

/* As knnm_load_graph, but g_ids / g_dists / g_sizes are device pointers
 * (graph already resident in HBM, e.g. a torch CUDA tensor). */
int knnm_load_graph_dev(knnm_ctx *ctx, const int32_t *rows, int64_t m,
                        const int32_t *g_ids, const double *g_dists,
                        const int32_t *g_sizes, int32_t gk, int32_t k1);

/* Directed inserts in the given order.  Replaces _eval_pairs +
 * apply_updates_directed (construct.py:86-108; _kernels.py:208-214) as used
 * by _append_random (merge.py:166-176), the raw-row init (merge.py:318-325)
 * and the random init of nn_descent (construct.py:255-259).  rows/nids:
 * int32 (m) local ids.  *accepted receives the accepted count.
 * If capture is on, the m distances are kept for knnm_capture_fetch. */
int knnm_insert_directed(knnm_ctx *ctx, const int32_t *rows,
                         const int32_t *nids, int64_t m, int64_t *accepted);

/* knnm_insert_directed with rows[i] repeated `count` times (the
 * np.repeat(rows, count) target layout of merge.py:173); nids has
 * mrows*count entries.  The repeat is expanded on the device. */
int knnm_insert_rows(knnm_ctx *ctx, const int32_t *rows, int64_t mrows,
                     int32_t count, const int32_t *nids, int64_t *accepted);

/* Random cross-subset append (merge.py:146-176, _sample_pool_rows +
 * _append_random).  The host makes the PCG64 draws in the reference's order;
 * the device holds the (nrows, t) draw matrix and reports rows containing a
 * repeated value (ascending, as np.nonzero does), the host redraws exactly
 * those rows, and finally the device maps the draws through `pool` (local
 * ids of the other side) and inserts them into `rows` (targets repeat t
 * times, apply_updates_directed order).  bad must hold nrows entries. */
int knnm_draws_load(knnm_ctx *ctx, const int64_t *cand, int64_t nrows,
                    int32_t t, int64_t *bad, int64_t *nbad);
int knnm_draws_replace(knnm_ctx *ctx, const int64_t *rows, int64_t nrows,
                       const int64_t *vals, int64_t *bad, int64_t *nbad);
int knnm_draws_insert(knnm_ctx *ctx, const int32_t *rows, const int32_t *pool,
                      int64_t npool, int64_t *accepted);
/* knnm_draws_insert restricted to draw rows [r0, r1) (a sharded merge's
 * owned rows); the draw matrix is still generated for every row, so the
 * PCG64 stream advances exactly as the reference's. */
int knnm_draws_insert_range(knnm_ctx *ctx, const int32_t *rows, const int32_t *pool,
                            int64_t npool, int64_t r0, int64_t r1, int64_t *accepted);

/* Device-side draws for knnm_draws_*: a bit-exact restatement of numpy's
 * PCG64 + Generator.integers(0, m, size=(nrows, t)) (pcg64.h,
 * distributions.c buffered_bounded_lemire_uint32).  pcg = {state_hi,
 * state_lo, inc_hi, inc_lo} of rng.bit_generator.state; has_uint32 /
 * uinteger its half-buffer.  *consumed = raw 32-bit values used, so the
 * caller can advance its generator to the identical state.  gen fills the
 * whole matrix; regen redraws the listed rows (ascending, row-major, as
 * `cand[rows] = rng.integers(0, m, size=(len(rows), t))`).  Both return the
 * rows that contain a repeated value, as knnm_draws_load does. */
int knnm_draws_gen(knnm_ctx *ctx, const uint64_t *pcg, int32_t has_uint32,
                   uint32_t uinteger, uint64_t m, int64_t nrows, int32_t t,
                   int64_t *consumed, int64_t *bad, int64_t *nbad);
int knnm_draws_regen(knnm_ctx *ctx, const uint64_t *pcg, int32_t has_uint32,
                     uint32_t uinteger, uint64_t m, const int64_t *rows,
                     int64_t nrows, int64_t *consumed, int64_t *bad, int64_t *nbad);

/* Host-side (no context, no GPU): union of two strictly ascending id arrays
 * and each input's row in it (merge.py:217-221 np.union1d + searchsorted,
 * one linear pass; split by merge path over host threads for large inputs).
 * uni needs na + nb entries; *nu = union size; *shared = whether the inputs
 * share an id (merge.py:181 disjointness check); labels (nullable, na + nb
 * entries) = 1 where the union entry comes from b, else 0 (the merge labels
 * of merge.py:222-223 / 304-305). */
int knnm_merge_members(const int64_t *a, int64_t na, const int64_t *b, int64_t nb,
                       int64_t *uni, int32_t *rows_a, int32_t *rows_b, int64_t *nu,
                       int32_t *shared, int8_t *labels);

/* Host-side (no context, no GPU): nrows successive
 * sample_distinct(rng, n, k, exclude=exclude[r]) draws (core.py:222-230,
 * numpy Generator.choice(pool, k, replace=False)) from the PCG64 state
 * {state_hi, state_lo, inc_hi, inc_lo} + half-buffer, which are updated in
 * place to numpy's state after the draws.  out: int64 (nrows, k). */
int knnm_sample_distinct_rows(uint64_t *pcg, int32_t *has_uint32, uint32_t *uinteger,
                              int64_t n, int32_t k, const int32_t *exclude,
                              int64_t nrows, int64_t *out);

/* One local-join round.  Replaces one iteration of _descent_rounds
 * (construct.py:136-164): reverse_csr, assemble_neighborhoods (rev_cap),
 * flag clear, count_pairs/fill_pairs, pair_dists_dense and
 * apply_updates_grouped (_kernels.py:262-437, 113-119, 217-254).
 * *pairs = admissible pairs (RoundStats.pairs), *accepted = accepted
 * inserts (RoundStats.updates). */
int knnm_round(knnm_ctx *ctx, int32_t mode, int32_t rev_cap,
               uint64_t round_seed, int64_t *pairs, int64_t *accepted);

/* Id-sharded rounds.  The context owns local rows [lo, hi);
 * list arrays stay replicated between rounds (the host all-gathers owned row
 * blocks after each round, see paper_1908_00814_b200/distributed.py).
 * knnm_round_local runs the reverse step into owned rows, the hoods of owned
 * vertices and the local join over them, leaving reference-order update
 * slots for EVERY target row: cnt (u32, n) slots per target, boff (u64, n+1)
 * their offsets, Bd (f64) / Bs (int32) the slots -- rows of rank q are the
 * contiguous slot range [boff[lo_q], boff[hi_q]).  knnm_round_apply applies
 * owned rows from nsrc received blocks in source-rank order (= hood order =
 * the reference's order): recv_cnt (nsrc, hi-lo) u32 device array,
 * recv_base host array of nsrc element offsets of each block in recv_Bd /
 * recv_Bs (device).  knnm_local_views / knnm_state_views expose device
 * pointers for the collectives; knnm_local_views returns Bs = NULL when the
 * round's slots are packed (one u64 per slot in Bd: fp32 distance bits in
 * the high word, source row in the low word; recv_Bs is then ignored). */
int knnm_set_shard(knnm_ctx *ctx, int64_t lo, int64_t hi);
/* knnm_round_local runs the reverse step and the hoods; the local join then
 * runs per hood chunk: knnm_local_chunks gives this rank's chunk count (1
 * when the round's 2P slots fit the candidate budget, 0 without pairs), and
 * knnm_local_join(c) fills the slots of chunk c (an empty slot view for
 * c >= count, so every rank can run the busiest rank's number of chunks).
 * Chunks are consecutive ascending hood ranges, so applying the received
 * blocks in (source rank, chunk) order is still the reference's per-row
 * order (construct.py:147-164 chunks the same way). */
int knnm_round_local(knnm_ctx *ctx, int32_t mode, int32_t rev_cap,
                     uint64_t round_seed, int64_t *pairs_local);
int knnm_local_chunks(knnm_ctx *ctx, int32_t *nchunks);
int knnm_local_join(knnm_ctx *ctx, int32_t chunk);
int knnm_local_views(knnm_ctx *ctx, void **cnt, void **boff, void **Bd, void **Bs);
/* Same views over the WRITTEN slots only: slots the join left unwritten can
 * never be accepted, so the exchange drops them.  Per target row the written
 * slots keep their reference order; cnt = written slots per row, boff their
 * offsets in the compacted Bd / Bs (Bs = NULL when packed).  *total = number
 * of written slots.  Call after knnm_round_local; the views stay valid until
 * the next round. */
int knnm_local_compact(knnm_ctx *ctx, void **cnt, void **boff, void **Bd, void **Bs,
                       int64_t *total);
int knnm_round_apply(knnm_ctx *ctx, int32_t nsrc, const uint32_t *recv_cnt,
                     const uint64_t *recv_base, const double *recv_Bd,
                     const int32_t *recv_Bs, int64_t *accepted);
int knnm_state_views(knnm_ctx *ctx, void **ids, void **dists, void **flags, void **sizes);
/* Replication of owned rows without re-sending unchanged ones: after
 * knnm_round_apply, knnm_pack_rows packs the owned rows the round changed
 * (flags cleared by the assembly or an accepted insert; all owned rows when
 * all != 0, e.g. after a sharded initialisation) into row records
 * (f64 dists[k] | i32 ids[k] | i32 row | i32 size | u8 flags[k], padded to
 * *rec_bytes, a multiple of 8) in a context-owned device buffer, valid until
 * the next call; knnm_unpack_rows writes received records into the lists. */
int knnm_pack_rows(knnm_ctx *ctx, int32_t all, void **buf, int64_t *count, int32_t *rec_bytes);
int knnm_unpack_rows(knnm_ctx *ctx, const void *buf, int64_t count);

/* Candidate-slot budget in bytes (default 40 GiB; 0 restores it).  Rounds
 * whose 2P slots exceed it run in ascending hood chunks; a small budget
 * forces the chunked path (tests). */
int knnm_set_cand_budget(knnm_ctx *ctx, int64_t bytes);

/* Stream ordering with caller-owned CUDA streams (e.g. torch's current
 * stream), without a host sync: knnm_wait_stream makes the context's stream
 * wait for the work queued so far on `stream` (call before passing tensors
 * another stream produced); knnm_signal_stream makes `stream` wait for the
 * context's queued work (call before another stream reads context memory). */
int knnm_wait_stream(knnm_ctx *ctx, void *stream);
int knnm_signal_stream(knnm_ctx *ctx, void *stream);

/* Exact brute-force top-k (construct.py:273-348; _kernels.py:445-506):
 * for each query -- queries[nq, d] (host) or dataset rows rows[nq] -- the k
 * nearest candidates by (exact fp64 distance, id).  Row queries search the
 * rows of the current union (knnm_begin; ids are local rows); vector queries
 * search the whole dataset.  exclude_self drops the query row itself
 * (brute_force_graph).
 * Missing entries are -1 / +inf.  k <= 64.
 * Certified u8 L2 datasets (integers in [0, 255]) with k <= 32 run on the
 * tensor cores (tcgen05 kind::i8 Gram tiles, exact s32 -> exact distances);
 * everything else on the exact fp64 SIMT kernel. */
int knnm_bf_topk(knnm_ctx *ctx, const float *queries, const int64_t *rows, int64_t nq,
                 int32_t k, int32_t exclude_self, int32_t *out_ids, double *out_dists);
/* pair_dists_dense (_kernels.py:113-119): exact reference distances of the
 * union-row pairs (pa[i], pb[i]) -> out[i] (host arrays; knnm_begin first).
 * Serves the on_pair route of brute_force_graph (construct.py:296-312). */
int knnm_pair_dists(knnm_ctx *ctx, const int32_t *pa, const int32_t *pb, int64_t m, double *out);
/* Brute-force route: -1 auto (default), 0 exact SIMT, 1 tensor cores
 * (fails with KNNM_ERR_LIMIT when the data is not certified u8 L2). */
int knnm_set_bf_variant(knnm_ctx *ctx, int32_t variant);
/* Route the last knnm_bf_topk took: 0 SIMT, 1 tensor cores. */
int knnm_bf_route(knnm_ctx *ctx, int32_t *route);

/* phi over the current lists (construct.py:79-83), with numpy's pairwise
 * summation order, so the value is bit-identical to the reference. */
int knnm_phi(knnm_ctx *ctx, double *out);

/* The same phi, computed asynchronously on a side stream from the lists as
 * they are when called (e.g. right after knnm_round): the next round's
 * reverse, assembly and join overlap it, and every call that writes the
 * lists waits for it on the device.  knnm_phi_fetch waits for the pending
 * value and returns the one stored in `slot` (0 <= slot < KNNM_PHI_SLOTS). */
#define KNNM_PHI_SLOTS 64
int knnm_phi_async(knnm_ctx *ctx, int32_t slot);
int knnm_phi_fetch(knnm_ctx *ctx, int32_t slot, double *out);

/* Export the lists in global id space (construct.py:212-223), merging the
 * loaded rear lists back in when merge_rear != 0 (graph.py:259-280,
 * _kernels.py:529-563).  Outputs: ids int32 (n,k), dists float64 (n,k),
 * sizes int32 (n); flags are all False, as in the reference. */
int knnm_export(knnm_ctx *ctx, int32_t merge_rear, int32_t *out_ids,
                double *out_dists, int32_t *out_sizes);

/* As knnm_export, but the outputs are device pointers (result stays in HBM). */
int knnm_export_dev(knnm_ctx *ctx, int32_t merge_rear, int32_t *out_ids,
                    double *out_dists, int32_t *out_sizes);

/* Download the raw local-id state (for per-iteration parity checks). */
int knnm_get_state(knnm_ctx *ctx, int32_t *ids, double *dists,
                   uint8_t *flags, int32_t *sizes);

/* Capture mode for the reference's on_pair hook (construct.py:102-108):
 * when on, every distance evaluation of the next insert_directed / round
 * call is recorded in reference order (local ids pa, pb and value pd). */
int knnm_set_capture(knnm_ctx *ctx, int32_t on);
int knnm_capture_count(knnm_ctx *ctx, int64_t *count);
int knnm_capture_fetch(knnm_ctx *ctx, int32_t *pa, int32_t *pb, double *pd,
                       int64_t count);

/* Local-join kernel choice: -1 auto, 0 = exact route (fp64 on every pair),
 * 1 = tiled route (fp32 SIMT screen, exact by certificate or by fp64
 * re-evaluation), 2 = tensor-core route (fp16 mma.sync Gram blocks; only for
 * datasets with the dot-form certificate, otherwise auto), 3 = tcgen05 route
 * for non-certified long rows (rigorous fixed-point lower bounds from u8 limb
 * products, exact values in the apply; non-negative L2 data, k + rev_cap <=
 * 80; otherwise auto), 4 = exact fp64 register tiles for non-certified short
 * rows (every admissible pair exact, no fp32 screen; otherwise auto).  All
 * routes give bit-identical results; the switch exists for tests and
 * measurement. */
int knnm_set_join_variant(knnm_ctx *ctx, int32_t variant);

/* Sample rate rho < 1 (classic NN-Descent; no reference counterpart -- the
 * reference is rho = 1): at most new_cap of a row's new entries take part in
 * each round (the rest stay new), chosen by splitmix64 partial Fisher-Yates;
 * pass rev_cap = new_cap to knnm_round as well.  0 = all (reference). */
int knnm_set_sample(knnm_ctx *ctx, int32_t new_cap);

/* Hood processing order (performance only; results are independent of it):
 * iters > 0 rounds of min-label propagation over the lists build a
 * locality order once per merge; 0 processes hoods in id order. */
int knnm_set_locality(knnm_ctx *ctx, int32_t iters);

/* on = 0 disables the u8 tensor-core route (integer data in [0, 255]) so the
 * fp16 route is used instead; takes effect at the next knnm_set_dataset. */
int knnm_set_u8(knnm_ctx *ctx, int32_t on);

/* Dataset facts: cert bit 0 = fp32 difference-form arithmetic is provably
 * exact (integer entries, d*range^2 < 2^24 for L2); bit 1 = fp16 rows with
 * fp32 dot products are exact (integer entries, |v| <= 2048,
 * 2*d*max|v|^2 < 2^24); bit 2 = entries are integers in [0, 255] (u8
 * rows, s32 integer MMA); dp = padded row length in floats. */
int knnm_get_info(knnm_ctx *ctx, int32_t *cert, int32_t *dp);

/* Timing / counters. profiling=1 records CUDA events around every phase. */
int knnm_set_profiling(knnm_ctx *ctx, int32_t on);
int knnm_get_stats(knnm_ctx *ctx, knnm_stats *out);
int knnm_reset_stats(knnm_ctx *ctx);

/* Stream-ordered timing: record event `slot` (0..7) on the context stream;
 * knnm_elapsed waits for slot b and returns the device time b - a in ms. */
int knnm_mark(knnm_ctx *ctx, int32_t slot);
int knnm_elapsed(knnm_ctx *ctx, int32_t a, int32_t b, double *ms);

/* Block until all work on the context stream is done. */
int knnm_sync(knnm_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* KNNM_H */

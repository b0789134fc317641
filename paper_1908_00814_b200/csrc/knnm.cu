// knnm.cu -- libknnm.so: context, memory plan and the C-ABI (include/knnm.h)
// for the B200 S-Merge / J-Merge round engine.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cmath>

#include <algorithm>
#include <cstdarg>
#include <functional>
#include <memory>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/knnm.h"
#include "knnm_kernels.cuh"
#include "knnm_bf.cuh"
#include "knnm_tcjoin.cuh"
#include "knnm_dense.cuh"

using namespace knnm;

struct knnm_ctx;
extern "C" {
static int phi_kernels(knnm_ctx *c, const double **res, cudaStream_t stream);  // defined with knnm_phi
}

namespace {

thread_local std::string g_err;

int fail(int code, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(x)                                                                             \
    do {                                                                                  \
        cudaError_t e_ = (x);                                                             \
        if (e_ != cudaSuccess)                                                            \
            return fail(e_ == cudaErrorMemoryAllocation ? KNNM_ERR_NOMEM : KNNM_ERR_CUDA, \
                        "%s:%d %s: %s", __FILE__, __LINE__, #x, cudaGetErrorString(e_));  \
    } while (0)
#define CKL()                     \
    do {                          \
        CK(cudaGetLastError());   \
        c->stats.launches += 1;   \
    } while (0)
#define TRY(...)                \
    do {                        \
        int r_ = (__VA_ARGS__); \
        if (r_ != KNNM_OK) return r_; \
    } while (0)

struct DBuf {
    void *p = nullptr;
    size_t bytes = 0;
    template <typename T>
    T *as() const { return reinterpret_cast<T *>(p); }
};

int ensure(DBuf &b, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (b.bytes >= bytes) return KNNM_OK;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    CK(cudaMalloc(&b.p, bytes));
    b.bytes = bytes;
    return KNNM_OK;
}

void release(DBuf &b) {
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
}

enum Phase { PH_JOIN = 0, PH_REVERSE, PH_ASSEMBLE, PH_UPDATE, PH_OTHER, PH_JOINK, PH_APPLYK, PH_NUM };

struct PhiTree {
    int64_t N = -1;
    std::vector<int64_t> leaf_lo;
    std::vector<int32_t> leaf_len;
    std::vector<int32_t> left, right, level_start;
};

}  // namespace

struct knnm_ctx {
    int device = 0;
    int sms = 148;
    cudaStream_t st = nullptr;
    // asynchronous phi (knnm_phi_async): computed on st2 while the next
    // round's reverse / assembly / join run on st; list writers wait on ev_phi
    cudaStream_t st2 = nullptr;
    cudaEvent_t ev_lists = nullptr, ev_phi = nullptr;
    bool phi_pending = false;
    double *hphi = nullptr;  // pinned, KNNM_PHI_SLOTS results
    // dataset
    DBuf vec;
    int64_t n_all = 0;
    int d = 0, dp = 0, metric = 1;
    bool have_data = false;
    bool cert = false;  // fp32 arithmetic is exact for this dataset + metric
    bool cert_dot = false;  // fp16 rows + fp32 dot products are exact (L2)
    DBuf nrm64;             // exact fp64 squared norm of every subset row (cosine)
    DBuf mpack;             // fused membership segments: base << 32 | count
    DBuf f32chk;            // loaded list distances not exact in fp32 (count)
    DBuf live;              // per row: its hood can hold a new entry this round
    DBuf segheavy;          // rows with > SEG_SMEM memberships (k_seg_rank_heavy)
    uint64_t state_gen = 1;      // bumped by every call that may change the lists
    uint64_t phi_gen = 0;        // state_gen phi_val was computed at
    double phi_val = 0.0;
    bool phi_in_updates = false; // the round's apply also computes phi (one sync)
    void *stg_buf[2] = {nullptr, nullptr};  // pinned staging for pageable copies
    cudaEvent_t stg_ev[2] = {nullptr, nullptr};
    bool stg_busy[2] = {false, false};
    bool lists_f32 = true;  // every list distance is an exact fp32 value
    int slots_mode = SLOTS_PLAIN;  // format of the slots the next apply reads
    // generation-tagged packed slots (tensor-core join, unsharded rounds):
    // bits 24-31 of a slot's low word carry the round's tag (1..254), so a
    // slot left from an earlier round reads as unwritten and the per-round
    // "cannot pass" prefill is not needed.  slot_gen = tag of the current
    // round's slots (0: NaN-prefilled format); gen_valid = the buffer holds
    // only tagged slots (else it is zeroed before the next tagged round).
    uint32_t slot_gen = 0, last_gen = 0;
    bool gen_valid = false;
    bool gen_slots = true;  // KNNM_GEN_SLOTS=0 turns the tagged format off
    int new_cap = 0;               // rho-sampling: new entries per row per round (0 = all)
    bool cert_u8 = false;   // entries are integers in [0, 255]: u8 rows, s32 MMA
    int dph = 0;            // fp16 row length (multiple of 16)
    int rowb = 0;           // staged bytes per row for the tensor-core join
    DBuf vec16, norms, sub16, subnorms;
    const uint8_t *sub16p = nullptr;
    const float *subnormp = nullptr;
    // -1 auto, 0 exact (fp64 every pair), 1 tiled / chunked fp32, 2 tensor core
    // (mma.sync, certified), 3 tensor core (tcgen05 lazy bounds)
    int join_variant = -1;
    int bf_variant = -1;    // brute force: -1 auto, 0 SIMT exact, 1 tcgen05 (certified u8 only)
    int lazy_ahead = LZB_AHEAD;  // look-ahead chunks of a lazy evaluation batch (KNNM_LAZY_AHEAD)
    // rows longer than this defer exact values to the apply (KNNM_LAZY_MIN_D;
    // measured: config 4, d = 100, is faster exact-in-join, config 3, d = 960, lazy)
    int lazy_min_d = 384;
    int bf_last_route = 0;  // route the last knnm_bf_topk took (0 SIMT, 1 tcgen05)
    DBuf bfq, bfqn, bfpart;  // brute force: gathered query rows / norms, partial lists
    bool bf_u8 = false;      // integers in [0, 255]: exact u8 Gram tiles for brute force
    DBuf bfx, bfxn;          // u8 copy of the candidate rows when the join has none
    bool u8_enabled = true;
    // tcgen05 lazy join (k_join_tc): non-negative finite L2 data in 24-bit
    // fixed point, three u8 limb planes per union row (built once per merge)
    bool tcj_data = false;
    double tcj_scale = 0.0;  // 2^(24 - e), max entry <= 2^e
    int tcj_dpad = 0;        // limb plane length (roundup(d, 16))
    bool limbs_ready = false;
    bool sub64_ready = false;  // fp64 union rows for k_join_dense
    DBuf sub64, nsq, djrec;
    bool tcj_round = false;  // the round's lazy slots hold k_join_tc's bounds (lo_rel = 1)
    DBuf limbs, lnx, lax;
    // current merge
    DBuf sub, ugid, labels, labbits;
    bool ug_identity = false;  // union = 0 .. n_all-1: ugid not uploaded
    const float *subp = nullptr;
    int64_t n = 0;
    int k = 0;
    bool begun = false;
    DBuf ids, dists, flags, sizes;
    DBuf tail_ids, tail_d, tail_s;
    int tk = 0;
    bool have_tail = false;
    int64_t shard_lo = 0, shard_hi = -1;  // owned rows (sharded rounds); -1 = n
    // round scratch
    DBuf indeg, roff, rev, heavy, giant, gscratch32, nbh, nlen, hpairs, poff, worst0, active, rowmeta;
    DBuf wcnt, woff, cBd, cBs;  // written-slot compaction (sharded exchange)
    DBuf dirty, rsel, rsoff, rpack;  // owned rows changed by a sharded round, their records
    DBuf bound, boff, mcount, moff, mcur, memb, start, Bd, Bs;
    DBuf order, lab0, lab1;       // locality order of hoods (per merge)
    bool have_order = false;
    int locality_iters = 8;
    uint64_t memb_cap = 0, start_cap = 0;
    DBuf draws, draw_rows, draw_bad, pool, scan_pos;  // random-append draw matrix (device)
    int64_t draw_n = 0;
    int draw_t = 0;
    DBuf scan_tmp[4], scan_off[4];
    DBuf counters;
    unsigned long long cap = 0;  // candidate record capacity
    size_t cand_budget_bytes = (size_t)40 << 30;  // knnm_set_cand_budget
    // sharded round in progress: its hood chunks (knnm_local_join)
    int lc_mode = 0, lc_W = 0;
    bool lc_single = true;  // one chunk = the round's active hoods
    int64_t lc_nact = 0;
    std::vector<std::vector<int32_t>> lc_lists;
    std::vector<uint64_t> lc_pairs2;
    // staging
    DBuf stage[4];
    unsigned long long *hcnt = nullptr;  // pinned mirror of counters
    // outputs
    DBuf out_ids, out_d, out_s;
    // phi
    PhiTree phi;
    DBuf phi_leaf_lo, phi_leaf_len, phi_left, phi_right, phi_level, phi_leaves, phi_inner;
    // capture
    bool capture = false;
    std::vector<int32_t> cap_pa, cap_pb;
    std::vector<double> cap_pd;
    // profiling
    bool profiling = false;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
    std::vector<cudaEvent_t> ev_pool;
    double phase_ms[PH_NUM] = {0, 0, 0, 0, 0, 0, 0};
    knnm_stats stats{};
    cudaEvent_t marks[8] = {};
    cudaEvent_t ev_wait = nullptr, ev_sig = nullptr;  // knnm_wait_stream / knnm_signal_stream
};

namespace {

int ev_get(knnm_ctx *c, cudaEvent_t *e) {
    if (!c->ev_pool.empty()) {
        *e = c->ev_pool.back();
        c->ev_pool.pop_back();
        return KNNM_OK;
    }
    CK(cudaEventCreate(e));
    return KNNM_OK;
}

struct PhaseTimer {
    knnm_ctx *c;
    int ph;
    cudaEvent_t a = nullptr, b = nullptr;
    PhaseTimer(knnm_ctx *c_, int ph_) : c(c_), ph(ph_) {
        if (c->profiling && ev_get(c, &a) == KNNM_OK) cudaEventRecord(a, c->st);
    }
    ~PhaseTimer() {
        if (a && ev_get(c, &b) == KNNM_OK) {
            cudaEventRecord(b, c->st);
            c->pending.push_back({ph, {a, b}});
        }
    }
};

int resolve_timers(knnm_ctx *c) {
    for (auto &p : c->pending) {
        float ms = 0;
        CK(cudaEventSynchronize(p.second.second));
        CK(cudaEventElapsedTime(&ms, p.second.first, p.second.second));
        c->phase_ms[p.first] += ms;
        c->ev_pool.push_back(p.second.first);
        c->ev_pool.push_back(p.second.second);
    }
    c->pending.clear();
    return KNNM_OK;
}

int grid_for(knnm_ctx *c, int64_t work, int threads, int per_sm = 8) {
    int64_t g = (work + threads - 1) / threads;
    int64_t cap = (int64_t)c->sms * per_sm;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

// Large transfers to / from pageable host memory (plain numpy arrays) go
// through a pinned double buffer: the driver's own staging of pageable
// copies runs far below PCIe rates, so chunks are DMA'd to/from pinned
// memory while the previous chunk is copied on the host by several threads.
constexpr size_t STG_CHUNK = 16u << 20;
constexpr size_t STG_MIN = 8u << 20;

bool host_pageable(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

void par_memcpy(void *dst, const void *src, size_t bytes) {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t nt = std::min<size_t>(std::min(8u, hw), std::max<size_t>(1, bytes >> 21));
    if (nt <= 1) {
        memcpy(dst, src, bytes);
        return;
    }
    const size_t part = ((bytes + nt - 1) / nt + 4095) & ~(size_t)4095;
    std::vector<std::thread> th;
    for (size_t t = 1; t < nt; t++) {
        const size_t off = t * part;
        if (off >= bytes) break;
        th.emplace_back([=] { memcpy((char *)dst + off, (const char *)src + off, std::min(part, bytes - off)); });
    }
    memcpy(dst, src, std::min(part, bytes));
    for (auto &x : th) x.join();
}

int ensure_staging(knnm_ctx *c) {
    for (int i = 0; i < 2; i++) {
        if (!c->stg_buf[i]) {
            CK(cudaHostAlloc(&c->stg_buf[i], STG_CHUNK, cudaHostAllocDefault));
            CK(cudaEventCreateWithFlags(&c->stg_ev[i], cudaEventDisableTiming));
            c->stg_busy[i] = false;
        }
    }
    return KNNM_OK;
}

// A pending asynchronous phi reads the lists: writers wait for it on st.
void phi_wait(knnm_ctx *c) {
    if (c && c->phi_pending) {
        cudaStreamWaitEvent(c->st, c->ev_phi, 0);
        c->phi_pending = false;
    }
}

// device union-id table, or nullptr for an identity union
const int64_t *ugid_of(const knnm_ctx *c) { return c->ug_identity ? nullptr : c->ugid.as<int64_t>(); }

int h2d(knnm_ctx *c, void *dst, const void *src, size_t bytes) {
    if (bytes == 0) return KNNM_OK;
    c->stats.h2d_bytes += (int64_t)bytes;
    if (bytes < STG_MIN || !host_pageable(src)) {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->st));
        return KNNM_OK;
    }
    TRY(ensure_staging(c));
    for (size_t off = 0, i = 0; off < bytes; off += STG_CHUNK, i++) {
        const int sl = (int)(i & 1);
        const size_t len = std::min(STG_CHUNK, bytes - off);
        if (c->stg_busy[sl]) CK(cudaEventSynchronize(c->stg_ev[sl]));  // its last DMA is done
        par_memcpy(c->stg_buf[sl], (const char *)src + off, len);
        CK(cudaMemcpyAsync((char *)dst + off, c->stg_buf[sl], len, cudaMemcpyHostToDevice, c->st));
        CK(cudaEventRecord(c->stg_ev[sl], c->st));
        c->stg_busy[sl] = true;
    }
    return KNNM_OK;  // the source may be released: it has been copied out
}

int d2h(knnm_ctx *c, void *dst, const void *src, size_t bytes) {
    if (bytes == 0) return KNNM_OK;
    c->stats.d2h_bytes += (int64_t)bytes;
    if (bytes < STG_MIN || !host_pageable(dst)) {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->st));
        return KNNM_OK;
    }
    TRY(ensure_staging(c));
    size_t prev_off = 0, prev_len = 0;
    int prev_sl = -1;
    for (size_t off = 0, i = 0; off < bytes; off += STG_CHUNK, i++) {
        const int sl = (int)(i & 1);
        const size_t len = std::min(STG_CHUNK, bytes - off);
        // (slot sl's previous chunk was copied out one iteration ago)
        CK(cudaMemcpyAsync(c->stg_buf[sl], (const char *)src + off, len, cudaMemcpyDeviceToHost, c->st));
        CK(cudaEventRecord(c->stg_ev[sl], c->st));
        c->stg_busy[sl] = true;
        if (prev_sl >= 0) {
            CK(cudaEventSynchronize(c->stg_ev[prev_sl]));
            par_memcpy((char *)dst + prev_off, c->stg_buf[prev_sl], prev_len);
        }
        prev_off = off;
        prev_len = len;
        prev_sl = sl;
    }
    CK(cudaEventSynchronize(c->stg_ev[prev_sl]));
    par_memcpy((char *)dst + prev_off, c->stg_buf[prev_sl], prev_len);
    return KNNM_OK;  // complete on return (as a pageable cudaMemcpy)
}

int sync_counters(knnm_ctx *c) {
    CK(cudaMemcpyAsync(c->hcnt, c->counters.p, sizeof(unsigned long long) * C_NUM, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    return KNNM_OK;
}

// Exclusive scan of n values into out[0..n] (out[n] = total).  Tile sums
// recurse through preallocated per-level buffers (no allocation per call
// once warmed up).
template <typename TI, typename TO>
int scan(knnm_ctx *c, const TI *in, TO *out, int64_t n, int level = 0) {
    int64_t ntiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    if (ntiles < 1) ntiles = 1;
    if (level >= 4) return fail(KNNM_ERR_LIMIT, "scan too deep");
    TRY(ensure(c->scan_tmp[level], sizeof(TO) * (size_t)(ntiles + 1)));
    TRY(ensure(c->scan_off[level], sizeof(TO) * (size_t)(ntiles + 1)));
    TO *tiles = c->scan_tmp[level].as<TO>();
    TO *toffs = c->scan_off[level].as<TO>();
    k_scan_tiles<TI, TO><<<(unsigned)ntiles, SCAN_THREADS, 0, c->st>>>(in, out, n, tiles);
    CKL();
    if (ntiles == 1) {
        CK(cudaMemcpyAsync(out + n, tiles, sizeof(TO), cudaMemcpyDeviceToDevice, c->st));
        return KNNM_OK;
    }
    TRY((scan<TO, TO>(c, tiles, toffs, ntiles, level + 1)));
    k_scan_add<TO><<<(unsigned)((n + 255) / 256), 256, 0, c->st>>>(out, n, toffs);
    CKL();
    k_scan_total<TO><<<1, 1, 0, c->st>>>(out, n, toffs, ntiles);
    CKL();
    return KNNM_OK;
}

// Slots the candidate budget holds: 8 bytes each when the source row rides in
// the packed slot (tensor-core join: no Bs array), else 8 + 4.
uint64_t bucket_budget(knnm_ctx *c, bool packed_only = false) {
    return c->cand_budget_bytes / (packed_only ? sizeof(double) : sizeof(double) + sizeof(int32_t));
}

int ensure_slots_noinit(knnm_ctx *c, uint64_t slots) {
    TRY(ensure(c->Bd, sizeof(double) * slots));
    TRY(ensure(c->Bs, sizeof(int32_t) * slots));
    c->gen_valid = false;
    return KNNM_OK;
}

int ensure_slots(knnm_ctx *c, uint64_t slots, bool need_bs = true) {
    TRY(ensure(c->Bd, sizeof(double) * slots));
    if (need_bs) TRY(ensure(c->Bs, sizeof(int32_t) * slots));
    // NaN fill: a slot the join does not write cannot pass (see k_apply_stream)
    CK(cudaMemsetAsync(c->Bd.p, 0xff, sizeof(double) * slots, c->st));
    c->gen_valid = false;
    c->slot_gen = 0;
    return KNNM_OK;
}

// Packed slots with a generation tag instead of the prefill: a new tag per
// round (1..254); the whole buffer is zeroed only when it was (re)allocated,
// used in another format, or the tags wrap.
int ensure_slots_tagged(knnm_ctx *c, uint64_t slots) {
    // (tensor-core join only: the source row is in the slot, no Bs array)
    const size_t before = c->Bd.bytes;
    TRY(ensure(c->Bd, sizeof(double) * slots));
    if (c->Bd.bytes != before || !c->gen_valid || c->last_gen >= 254) {
        CK(cudaMemsetAsync(c->Bd.p, 0, c->Bd.bytes, c->st));
        c->last_gen = 0;
        c->gen_valid = true;
    }
    c->slot_gen = ++c->last_gen;
    return KNNM_OK;
}

int ensure_memb(knnm_ctx *c, uint64_t recs, uint64_t starts) {
    if (recs > c->memb_cap) {
        TRY(ensure(c->memb, sizeof(MembRec) * recs));
        c->memb_cap = recs;
    }
    if (starts > c->start_cap) {
        TRY(ensure(c->start, sizeof(uint32_t) * starts));
        c->start_cap = starts;
    }
    return KNNM_OK;
}

// Membership ranking: moff = scan(mcount); bucket memberships by row (fill
// kernel launched by the caller between the two halves); then k_seg_rank.
// wout: records of hood memberships rank into start[u * W + p] (wout = W);
// directed-insert records into start[ordinal] (wout = 1)
int rank_memberships(knnm_ctx *c, uint32_t wout, bool fused = false) {
    TRY(ensure(c->segheavy, sizeof(int32_t) * (size_t)c->n));
    unsigned long long *cnt = c->counters.as<unsigned long long>();
    CK(cudaMemsetAsync(cnt + C_SEGHEAVY, 0, sizeof(unsigned long long), c->st));
    const unsigned long long *mp = fused ? c->mpack.as<unsigned long long>() : nullptr;
    // fused rounds: the row totals (bucket sizes) come from here, not from
    // per-membership atomics in k_assemble
    uint32_t *tot = fused ? c->bound.as<uint32_t>() : nullptr;
    k_seg_rank<<<grid_for(c, c->n * 32, SEG_WARPS * 32, 16), SEG_WARPS * 32, 0, c->st>>>(
        c->n, c->moff.as<uint32_t>(), c->memb.as<MembRec>(), c->start.as<uint32_t>(), mp,
        c->segheavy.as<int32_t>(), cnt, tot, wout);
    CKL();
    // hub rows: block per row, count read on the device
    k_seg_rank_heavy<<<c->sms * 2, SEGH_THREADS, 0, c->st>>>(
        c->moff.as<uint32_t>(), c->memb.as<MembRec>(), c->start.as<uint32_t>(), mp,
        c->segheavy.as<int32_t>(), cnt, tot, wout);
    CKL();
    return KNNM_OK;
}

// Sequential per-row application of the slot buckets (row r: slots
// [boff[r], boff[r+1]), already in the reference's order).
// Exact-evaluation context of the apply kernels.  Approximate slots (sign
// bit set) are written only by the non-certified tiled join.
bool metric_is_cos(const knnm_ctx *c) { return c->metric == KNNM_COSINE; }


LazyExact lazy_of(knnm_ctx *c) {
    LazyExact z;
    z.nrows = c->n;
    z.ahead = c->lazy_ahead;
    z.sub = c->subp;
    z.nrm64 = c->metric == KNNM_COSINE ? c->nrm64.as<double>() : nullptr;
    z.dp = c->dp;
    z.d = c->d;
    z.tag = c->metric;
    // k_join_tc stores rigorous lower bounds of the reference value itself
    z.lo_rel = c->tcj_round ? 1.0 : 1.0 - (double)(c->d + 8) * ldexp(1.0, -23);
    z.lo_abs = (double)(4 * c->d + 64) * ldexp(1.0, -24);
    if (c->metric == KNNM_COSINE) {
        z.hi_rel = 1.0;
        z.hi_abs = z.lo_abs;
    } else if (c->tcj_round) {
        // k_join_tc: bound - exact <= 2 (dropped limb products + truncation);
        // entries <= 2^24 / scale, so sum x <= d 2^24 / scale
        const double sc = 1.0 / c->tcj_scale;
        z.hi_rel = 1.0 + (double)(c->d + 16) * ldexp(1.0, -50);
        z.hi_abs = 2.0 * ((double)c->d * TJC_GMAX_TAIL * sc * sc + 2.0 * sc * (double)c->d * ldexp(1.0, 24) * sc +
                          (double)c->d * sc * sc);
    } else {
        z.hi_rel = 1.0 / (1.0 - (double)(c->d + 8) * ldexp(1.0, -23));
        z.hi_abs = 0.0;
    }
    return z;
}

int run_updates(knnm_ctx *c) {
    phi_wait(c);  // the apply writes the lists a pending phi still reads
    int64_t n = c->n;
    unsigned long long *cnt = c->counters.as<unsigned long long>();
    CK(cudaMemsetAsync(cnt + C_CAND, 0, sizeof(unsigned long long) * 2, c->st));
    CK(cudaMemsetAsync(cnt + C_WRITTEN, 0, sizeof(unsigned long long), c->st));
    CK(cudaMemsetAsync(cnt + C_ROWS_IN, 0, sizeof(unsigned long long) * 3, c->st));
    const int E = (c->k + 31) / 32;
    const int blocks = grid_for(c, n * 32, APPLY_WARPS * 32, 16);
#define KNNM_AP_LAUNCH(EE, LZ, F)                                                                \
    k_apply_stream<EE, LZ, F><<<blocks, APPLY_WARPS * 32, 0, c->st>>>(                             \
        n, c->k, c->boff.as<uint64_t>(), c->Bd.as<double>(), c->Bs.as<int32_t>(),               \
        c->ids.as<int32_t>(), c->dists.as<double>(), c->flags.as<uint8_t>(), c->sizes.as<int32_t>(), \
        cnt, lazy_of(c), c->slots_mode == SLOTS_PACKED ? c->slot_gen : 0u)
    const bool f32 = c->lists_f32;
    {
        PhaseTimer ptk(c, PH_APPLYK);  // the apply kernel alone (roofline)
        if (E == 1) {
            if (c->slots_mode == SLOTS_LAZY) KNNM_AP_LAUNCH(1, SLOTS_LAZY, false);
            else if (c->slots_mode == SLOTS_PACKED && f32) KNNM_AP_LAUNCH(1, SLOTS_PACKED, true);
            else if (c->slots_mode == SLOTS_PACKED) KNNM_AP_LAUNCH(1, SLOTS_PACKED, false);
            else KNNM_AP_LAUNCH(1, SLOTS_PLAIN, false);
        } else {
            if (c->slots_mode == SLOTS_LAZY) KNNM_AP_LAUNCH(2, SLOTS_LAZY, false);
            else if (c->slots_mode == SLOTS_PACKED && f32) KNNM_AP_LAUNCH(2, SLOTS_PACKED, true);
            else if (c->slots_mode == SLOTS_PACKED) KNNM_AP_LAUNCH(2, SLOTS_PACKED, false);
            else KNNM_AP_LAUNCH(2, SLOTS_PLAIN, false);
        }
        CKL();
    }
#undef KNNM_AP_LAUNCH
    // a round's final apply also reduces phi, fetched in the same wait
    const double *phi_res = nullptr;
    if (c->phi_in_updates && c->n * c->k > 0) TRY(phi_kernels(c, &phi_res, c->st));
    TRY(sync_counters(c));
    if (phi_res) {
        CK(cudaMemcpy(&c->phi_val, phi_res, sizeof(double), cudaMemcpyDeviceToHost));
        c->phi_gen = c->state_gen;
    }
    c->stats.candidates += (int64_t)c->hcnt[C_CAND];
    c->stats.apply_rows_in += (int64_t)c->hcnt[C_ROWS_IN];
    c->stats.apply_rows_out += (int64_t)c->hcnt[C_ROWS_OUT];
    c->stats.lazy_batches += (int64_t)c->hcnt[C_LZ_BATCHES];
    c->stats.written_slots += (int64_t)c->hcnt[C_WRITTEN];
    c->stats.seg_hub_rows += (int64_t)c->hcnt[C_SEGHEAVY];
    return KNNM_OK;
}

// Locality order of the hoods for this merge (see k_label_prop).
int build_locality_order(knnm_ctx *c) {
    const int64_t n = c->n;
    TRY(ensure(c->order, sizeof(int32_t) * n));
    TRY(ensure(c->lab0, sizeof(int32_t) * (n + 1)));
    TRY(ensure(c->lab1, sizeof(int32_t) * (n + 1)));
    int32_t *a = c->lab0.as<int32_t>(), *b = c->lab1.as<int32_t>();
    k_iota<<<grid_for(c, n, 256), 256, 0, c->st>>>(a, n);
    CKL();
    for (int it = 0; it < c->locality_iters; it++) {
        k_label_prop<<<grid_for(c, n, 256), 256, 0, c->st>>>(c->ids.as<int32_t>(), c->flags.as<uint8_t>(),
                                                            c->sizes.as<int32_t>(), n, c->k, a, b);
        CKL();
        std::swap(a, b);
    }
    // counting sort by label (labels are row ids in [0, n))
    CK(cudaMemsetAsync(c->mcount.p, 0, sizeof(uint32_t) * (n + 1), c->st));
    CK(cudaMemsetAsync(c->mcur.p, 0, sizeof(uint32_t) * (n + 1), c->st));
    k_label_hist<<<grid_for(c, n, 256), 256, 0, c->st>>>(a, n, c->mcount.as<uint32_t>());
    CKL();
    TRY(scan<uint32_t, uint32_t>(c, c->mcount.as<uint32_t>(), c->moff.as<uint32_t>(), n));
    k_label_scatter<<<grid_for(c, n, 256), 256, 0, c->st>>>(a, n, c->moff.as<uint32_t>(),
                                                           c->mcur.as<uint32_t>(), c->order.as<int32_t>());
    CKL();
    c->have_order = true;
    return KNNM_OK;
}

void build_phi_tree(PhiTree &t, int64_t N) {
    t.N = N;
    t.leaf_lo.clear();
    t.leaf_len.clear();
    struct Node { int32_t l, r, h; };
    std::vector<Node> nodes;
    struct Res { int32_t ref, h; };
    // iterative-safe recursion (depth ~ log2(N/64))
    std::function<Res(int64_t, int64_t)> rec = [&](int64_t lo, int64_t n) -> Res {
        if (n <= 128) {
            t.leaf_lo.push_back(lo);
            t.leaf_len.push_back((int32_t)n);
            return Res{-(int32_t)t.leaf_lo.size(), 0};
        }
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        Res a = rec(lo, n2);
        Res b = rec(lo + n2, n - n2);
        int32_t h = std::max(a.h, b.h) + 1;
        nodes.push_back(Node{a.ref, b.ref, h});
        return Res{(int32_t)nodes.size() - 1, h};
    };
    rec(0, N);
    int32_t H = 0;
    for (auto &nd : nodes) H = std::max(H, nd.h);
    std::vector<int32_t> order(nodes.size());
    for (size_t i = 0; i < nodes.size(); i++) order[i] = (int32_t)i;
    std::stable_sort(order.begin(), order.end(),
                     [&](int32_t a, int32_t b) { return nodes[a].h < nodes[b].h; });
    std::vector<int32_t> pos(nodes.size());
    for (size_t i = 0; i < order.size(); i++) pos[order[i]] = (int32_t)i;
    t.left.resize(nodes.size());
    t.right.resize(nodes.size());
    for (size_t i = 0; i < order.size(); i++) {
        const Node &nd = nodes[order[i]];
        t.left[i] = nd.l >= 0 ? pos[nd.l] : nd.l;
        t.right[i] = nd.r >= 0 ? pos[nd.r] : nd.r;
    }
    t.level_start.assign(H + 1, 0);
    // level h (1..H) occupies [level_start[h-1], level_start[h])
    std::vector<int32_t> cnt(H + 1, 0);
    for (auto &nd : nodes) cnt[nd.h]++;
    t.level_start[0] = 0;
    for (int h = 1; h <= H; h++) t.level_start[h] = t.level_start[h - 1] + cnt[h];
}

}  // namespace

// ---------------------------------------------------------------------------
// Host-side numpy PCG64 (pcg64.h) and Generator.choice(pop, size,
// replace=False) (Floyd's algorithm with a linear-probing hash set, or the
// tail shuffle for large samples, then an in-place Fisher-Yates shuffle; all
// bounded draws via Lemire's method).  Restated natively so the per-row
// sample_distinct loop of merge.py:318-325 runs in C++ instead of 500k Python
// calls; tests/test_host.py pins it against numpy.
// ---------------------------------------------------------------------------
namespace {
struct HostPcg {
    unsigned __int128 s, inc;
    int has;
    uint32_t u;
    static unsigned __int128 mult() {
        return ((unsigned __int128)0x2360ED051FC65DA4ULL << 64) | 0x4385DF649FCCF645ULL;
    }
    uint32_t next32() {
        if (has) {
            has = 0;
            return u;
        }
        s = s * mult() + inc;
        const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
        const unsigned r = (unsigned)(s >> 122);
        const uint64_t v = (x >> r) | (x << ((64u - r) & 63u));
        has = 1;
        u = (uint32_t)(v >> 32);
        return (uint32_t)v;
    }
    uint64_t bounded(uint64_t rng) {  // random_bounded_uint64(0, rng), rng < 2^32
        if (rng == 0) return 0;
        if (rng == 0xFFFFFFFFull) return next32();
        const uint64_t excl = rng + 1;
        uint64_t m = (uint64_t)next32() * excl;
        uint32_t left = (uint32_t)m;
        if (left < excl) {
            const uint32_t thr = (uint32_t)((0xFFFFFFFFull - rng) % excl);
            while (left < thr) {
                m = (uint64_t)next32() * excl;
                left = (uint32_t)m;
            }
        }
        return m >> 32;
    }
};

void host_choice(HostPcg &p, int64_t pop, int64_t size, int64_t *out, std::vector<uint64_t> &hs,
                 std::vector<int64_t> &tmp) {
    if (pop > 10000 && size > pop / 50) {  // tail shuffle
        tmp.resize(pop);
        for (int64_t i = 0; i < pop; i++) tmp[i] = i;
        for (int64_t i = pop - 1; i >= std::max<int64_t>(pop - size, 1); i--) {
            const int64_t j = (int64_t)p.bounded((uint64_t)i);
            std::swap(tmp[i], tmp[j]);
        }
        for (int64_t t = 0; t < size; t++) out[t] = tmp[pop - size + t];
        return;
    }
    uint64_t mask = (uint64_t)(1.2 * (double)size);
    for (int sh = 1; sh < 64; sh <<= 1) mask |= mask >> sh;
    hs.assign(mask + 1, ~0ull);
    for (int64_t j = pop - size; j < pop; j++) {
        const uint64_t val = p.bounded((uint64_t)j);
        uint64_t loc = val & mask;
        while (hs[loc] != ~0ull && hs[loc] != val) loc = (loc + 1) & mask;
        if (hs[loc] == ~0ull) {
            hs[loc] = val;
            out[j - pop + size] = (int64_t)val;
        } else {
            loc = (uint64_t)j & mask;
            while (hs[loc] != ~0ull) loc = (loc + 1) & mask;
            hs[loc] = (uint64_t)j;
            out[j - pop + size] = j;
        }
    }
    for (int64_t i = size - 1; i >= 1; i--) {
        const int64_t j = (int64_t)p.bounded((uint64_t)i);
        std::swap(out[i], out[j]);
    }
}
// ---- the per-row choice loop, parallel ------------------------------------
// numpy's per-row Generator.choice(pool, k, replace=False) calls share one
// PCG64 stream, so row r's draws start where row r-1's ended.  Every draw is
// one 32-bit word of the stream except for Lemire rejections (probability
// < pool / 2^32 per draw).  So: (1) the 64-bit outputs are generated in
// parallel by LCG jump-ahead into a word buffer; (2) one sequential pass
// finds each row's first word by replaying only the draw *counts* (a
// multiply-compare per draw, no sets, no shuffles); (3) the rows are then
// computed in parallel from their own offsets by host_choice over a buffer
// reader -- the same arithmetic, so the same values, and the generator ends
// in the same state.
struct WordPcg {  // host_choice's interface over a pre-generated word buffer
    const uint32_t *w;
    size_t i, n;
    bool ok = true;
    uint32_t next32() {
        if (i >= n) { ok = false; return 0; }
        return w[i++];
    }
    uint64_t bounded(uint64_t rng) {
        if (rng == 0) return 0;
        if (rng == 0xFFFFFFFFull) return next32();
        const uint64_t excl = rng + 1;
        uint64_t m = (uint64_t)next32() * excl;
        uint32_t left = (uint32_t)m;
        if (left < excl) {
            const uint32_t thr = (uint32_t)((0xFFFFFFFFull - rng) % excl);
            while (left < thr && ok) {
                m = (uint64_t)next32() * excl;
                left = (uint32_t)m;
            }
        }
        return m >> 32;
    }
};

template <typename G>
void choice_draws(G &p, int64_t pop, int64_t size, int64_t *out, std::vector<uint64_t> &hs,
                  std::vector<int64_t> &tmp) {
    if (pop > 10000 && size > pop / 50) {  // tail shuffle
        tmp.resize(pop);
        for (int64_t i = 0; i < pop; i++) tmp[i] = i;
        for (int64_t i = pop - 1; i >= std::max<int64_t>(pop - size, 1); i--) {
            const int64_t j = (int64_t)p.bounded((uint64_t)i);
            std::swap(tmp[i], tmp[j]);
        }
        for (int64_t t = 0; t < size; t++) out[t] = tmp[pop - size + t];
        return;
    }
    uint64_t mask = (uint64_t)(1.2 * (double)size);
    for (int sh = 1; sh < 64; sh <<= 1) mask |= mask >> sh;
    hs.assign(mask + 1, ~0ull);
    for (int64_t j = pop - size; j < pop; j++) {
        const uint64_t val = p.bounded((uint64_t)j);
        uint64_t loc = val & mask;
        while (hs[loc] != ~0ull && hs[loc] != val) loc = (loc + 1) & mask;
        if (hs[loc] == ~0ull) {
            hs[loc] = val;
            out[j - pop + size] = (int64_t)val;
        } else {
            loc = (uint64_t)j & mask;
            while (hs[loc] != ~0ull) loc = (loc + 1) & mask;
            hs[loc] = (uint64_t)j;
            out[j - pop + size] = j;
        }
    }
    for (int64_t i = size - 1; i >= 1; i--) {
        const int64_t j = (int64_t)p.bounded((uint64_t)i);
        std::swap(out[i], out[j]);
    }
}

// Words a row's draws consume from the reader (its values are not needed).
void choice_skip(WordPcg &p, int64_t pop, int64_t size) {
    if (pop > 10000 && size > pop / 50) {
        for (int64_t i = pop - 1; i >= std::max<int64_t>(pop - size, 1); i--) p.bounded((uint64_t)i);
        return;
    }
    for (int64_t j = pop - size; j < pop; j++) p.bounded((uint64_t)j);
    for (int64_t i = size - 1; i >= 1; i--) p.bounded((uint64_t)i);
}

// LCG jump-ahead of the PCG64 state by `delta` steps.
unsigned __int128 pcg_advance(unsigned __int128 s, unsigned __int128 inc, uint64_t delta) {
    unsigned __int128 cm = HostPcg::mult(), cp = inc, am = 1, ap = 0;
    while (delta) {
        if (delta & 1) {
            am *= cm;
            ap = ap * cm + cp;
        }
        cp = (cm + 1) * cp;
        cm *= cm;
        delta >>= 1;
    }
    return am * s + ap;
}

// 64-bit outputs [first, first + count) after state s0 (output i comes from
// the state advanced i + 1 times), as 32-bit words lo, hi.
void pcg_words(unsigned __int128 s0, unsigned __int128 inc, uint64_t first, uint64_t count, uint32_t *out) {
    unsigned __int128 s = pcg_advance(s0, inc, first);
    for (uint64_t i = 0; i < count; i++) {
        s = s * HostPcg::mult() + inc;
        const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
        const unsigned r = (unsigned)(s >> 122);
        const uint64_t v = (x >> r) | (x << ((64u - r) & 63u));
        out[2 * i] = (uint32_t)v;
        out[2 * i + 1] = (uint32_t)(v >> 32);
    }
}

// Parallel form of the per-row loop; returns false when the word estimate
// was short (the caller then runs the sequential loop).
bool sample_rows_parallel(HostPcg &p, int64_t n, int32_t k, const int32_t *exclude, int64_t nrows,
                          int64_t *out) {
    auto pool_of = [&](int64_t r) {
        const int64_t ex = exclude[r];
        return (ex >= 0 && ex < n) ? n - 1 : n;
    };
    // nominal words per row (+ slack for rejections)
    uint64_t nominal = 0;
    for (int64_t r = 0; r < nrows; r++) {
        const int64_t pop = pool_of(r);
        nominal += (pop > 10000 && k > pop / 50) ? (uint64_t)std::min<int64_t>(k, pop - 1) : (uint64_t)(2 * k - 1);
    }
    const uint64_t need = nominal + nominal / 256 + 4096;
    const uint64_t outs = need / 2 + 1;
    // (uninitialised: every word is written by the generator threads)
    std::unique_ptr<uint32_t[]> bufp(new uint32_t[1 + 2 * outs]);
    uint32_t *buf = bufp.get();
    const size_t nbuf = 1 + 2 * outs;
    const size_t base = p.has ? 0 : 1;  // word 0 = the buffered half when present
    buf[0] = p.u;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const uint64_t nt = std::min<uint64_t>(std::min(16u, hw), std::max<uint64_t>(1, outs >> 16));
    {
        std::vector<std::thread> th;
        const uint64_t part = (outs + nt - 1) / nt;
        for (uint64_t t = 0; t < nt; t++) {
            const uint64_t a = t * part, b = std::min(outs, a + part);
            if (a >= b) break;
            th.emplace_back(pcg_words, p.s, p.inc, a, b - a, buf + 1 + 2 * a);
        }
        for (auto &x : th) x.join();
    }
    // sequential pass: each row's first word.  A Floyd row without a
    // rejection candidate (low word of w * excl below excl, checked for all
    // its draws at once: a vectorisable loop) consumes exactly 2k - 1 words;
    // any other row is replayed draw by draw.
    std::vector<uint64_t> start(nrows + 1);
    WordPcg rd{buf + base, 0, nbuf - base};
    for (int64_t r = 0; r < nrows; r++) {
        start[r] = rd.i;
        const int64_t pop = pool_of(r);
        const bool floyd = !(pop > 10000 && k > pop / 50);
        if (floyd && k >= 1 && rd.i + 2 * (size_t)k - 1 <= rd.n) {
            const uint32_t *w = rd.w + rd.i;
            uint32_t flag = 0;
            for (int d2 = 0; d2 < k; d2++) {
                const uint32_t excl = (uint32_t)(pop - k + d2 + 1);
                flag |= (uint32_t)(w[d2] * excl) < excl;
            }
            for (int d2 = 0; d2 < k - 1; d2++) {
                const uint32_t excl = (uint32_t)(k - d2);
                flag |= (uint32_t)(w[k + d2] * excl) < excl;
            }
            if (!flag) {
                rd.i += 2 * (size_t)k - 1;
                continue;
            }
        }
        choice_skip(rd, pop, k);
        if (!rd.ok) return false;
    }
    start[nrows] = rd.i;
    // the rows, in parallel
    {
        const uint64_t nr = (uint64_t)nrows;
        const uint64_t ntr = std::min<uint64_t>(std::min(16u, hw), std::max<uint64_t>(1, nr >> 12));
        std::vector<std::thread> th;
        const uint64_t part = (nr + ntr - 1) / ntr;
        for (uint64_t t = 0; t < ntr; t++) {
            const uint64_t a = t * part, b = std::min(nr, a + part);
            if (a >= b) break;
            th.emplace_back([&, a, b] {
                std::vector<uint64_t> hs;
                std::vector<int64_t> tmp;
                for (uint64_t r = a; r < b; r++) {
                    WordPcg w{buf + base, (size_t)start[r], (size_t)start[r + 1]};
                    int64_t *o = out + r * k;
                    choice_draws(w, pool_of((int64_t)r), k, o, hs, tmp);
                    const int64_t ex = exclude[r];
                    if (ex >= 0 && ex < n)
                        for (int t2 = 0; t2 < k; t2++) o[t2] += o[t2] >= ex ? 1 : 0;
                }
            });
        }
        for (auto &x : th) x.join();
    }
    // generator state after the consumed words
    // (numpy: fetching a 64-bit output stores its high half and sets the
    // flag; consuming the stored half only clears the flag)
    const uint64_t used = start[nrows];  // words read from buf[base ...]
    if (used == 0) return true;          // nothing consumed
    const uint64_t from_pairs = p.has ? used - 1 : used;
    const uint64_t nout = (from_pairs + 1) / 2;
    p.s = pcg_advance(p.s, p.inc, nout);
    if (nout > 0) p.u = buf[2 + 2 * (nout - 1)];
    p.has = (from_pairs & 1) ? 1 : 0;
    return true;
}

}  // namespace

extern "C" {

const char *knnm_last_error(void) { return g_err.c_str(); }
int knnm_version(void) { return 1; }

int knnm_create(int device, knnm_ctx **out) {
    if (!out) return fail(KNNM_ERR_ARG, "null out");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(KNNM_ERR_ARG, "device %d of %d", device, ndev);
    CK(cudaSetDevice(device));
    knnm_ctx *c = new knnm_ctx();
    c->device = device;
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    c->sms = prop.multiProcessorCount;
    if (const char *e = getenv("KNNM_LAZY_AHEAD")) c->lazy_ahead = std::max(0, std::min(64, atoi(e)));
    if (const char *e = getenv("KNNM_LAZY_MIN_D")) c->lazy_min_d = std::max(0, atoi(e));
    if (const char *e = getenv("KNNM_GEN_SLOTS")) c->gen_slots = atoi(e) != 0;
    CK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    CK(cudaHostAlloc((void **)&c->hcnt, sizeof(unsigned long long) * C_NUM, cudaHostAllocDefault));
    TRY(ensure(c->counters, sizeof(unsigned long long) * C_NUM));
    CK(cudaMemset(c->counters.p, 0, sizeof(unsigned long long) * C_NUM));
    CK(cudaFuncSetAttribute(k_rev_heavy, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)(2 * sizeof(uint32_t) * BLOCK_SORT_MAX)));
    for (auto f : {k_join_exact<0>, k_join_exact<1>, k_join_exact<2>})
        CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    for (auto f : {k_join_chunked<0>, k_join_chunked<1>, k_join_chunked<2>})
        CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    for (auto f : {k_join_dense<0>, k_join_dense<1>, k_join_dense<2>})
        CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DJ_SMEM_CAP));
#define KNNM_MJ_ALL(M)                                                                       \
    k_join_mma<false, 1, M>, k_join_mma<false, 2, M>, k_join_mma<false, 4, M>,              \
        k_join_mma<true, 1, M>, k_join_mma<true, 2, M>, k_join_mma<true, 4, M>
    for (auto f : {KNNM_MJ_ALL(0), KNNM_MJ_ALL(1), KNNM_MJ_ALL(2)})
        CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
#undef KNNM_MJ_ALL
    CK(cudaFuncSetAttribute(k_merge_rear, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)mr_smem_bytes(64, 64)));
    CK(cudaFuncSetAttribute(k_join_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TJC_SMEM_CAP));
    for (auto f : {k_bf_topk<0>, k_bf_topk<1>, k_bf_topk<2>})
        CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(BF_THREADS * BF_MAXK * (sizeof(double) + sizeof(int32_t)))));
    for (auto f : {k_join_tiled<0, false, false>, k_join_tiled<1, false, false>,
                   k_join_tiled<2, false, false>, k_join_tiled<0, false, true>,
                   k_join_tiled<1, false, true>, k_join_tiled<2, false, true>,
                   k_join_tiled<0, true, false>, k_join_tiled<1, true, false>})
        CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    *out = c;
    return KNNM_OK;
}

int knnm_destroy(knnm_ctx *c) {
    if (!c) return KNNM_OK;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->st);
    DBuf *all[] = {&c->vec, &c->sub, &c->ugid, &c->labels, &c->labbits, &c->ids, &c->dists, &c->flags,
                   &c->sizes, &c->tail_ids, &c->tail_d, &c->tail_s, &c->indeg, &c->roff,
                   &c->rev, &c->heavy, &c->giant, &c->gscratch32, &c->nbh, &c->nlen, &c->hpairs,
                   &c->poff, &c->worst0, &c->active, &c->rowmeta, &c->wcnt, &c->woff, &c->cBd, &c->cBs, &c->order, &c->lab0, &c->lab1, &c->bound, &c->boff, &c->mcount, &c->moff, &c->mcur, &c->memb, &c->start, &c->Bd, &c->Bs, &c->limbs, &c->lnx, &c->lax, &c->sub64, &c->nsq, &c->djrec,
                   &c->counters, &c->draws, &c->draw_rows,
                   &c->draw_bad, &c->pool, &c->scan_pos, &c->vec16, &c->norms, &c->sub16, &c->subnorms, &c->out_ids, &c->out_d,
                   &c->out_s, &c->phi_leaf_lo, &c->phi_leaf_len, &c->phi_left, &c->phi_right,
                   &c->phi_level, &c->phi_leaves, &c->phi_inner, &c->nrm64, &c->mpack, &c->f32chk, &c->live, &c->segheavy};
    for (DBuf *b : all) release(*b);
    for (int i = 0; i < 2; i++) {
        if (c->stg_buf[i]) cudaFreeHost(c->stg_buf[i]);
        if (c->stg_ev[i]) cudaEventDestroy(c->stg_ev[i]);
    }
    for (auto &b : c->scan_tmp) release(b);
    for (auto &b : c->scan_off) release(b);
    for (auto &b : c->stage) release(b);
    for (auto &p : c->pending) {
        cudaEventDestroy(p.second.first);
        cudaEventDestroy(p.second.second);
    }
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    if (c->ev_wait) cudaEventDestroy(c->ev_wait);
    if (c->ev_sig) cudaEventDestroy(c->ev_sig);
    for (auto e : c->marks)
        if (e) cudaEventDestroy(e);
    if (c->hcnt) cudaFreeHost(c->hcnt);
    if (c->hphi) cudaFreeHost(c->hphi);
    if (c->st2) {
        cudaStreamSynchronize(c->st2);
        cudaStreamDestroy(c->st2);
    }
    if (c->ev_lists) cudaEventDestroy(c->ev_lists);
    if (c->ev_phi) cudaEventDestroy(c->ev_phi);
    cudaStreamDestroy(c->st);
    delete c;
    return KNNM_OK;
}

int knnm_set_dataset(knnm_ctx *c, const float *vectors, int64_t n_all, int32_t d, int32_t metric) {
    if (!c || (!vectors && n_all > 0)) return fail(KNNM_ERR_ARG, "null argument");
    if (n_all < 1 || d < 1) return fail(KNNM_ERR_ARG, "empty dataset");
    if (metric < 0 || metric > 2) return fail(KNNM_ERR_ARG, "metric tag %d not dense", metric);
    CK(cudaSetDevice(c->device));
    PhaseTimer pt(c, PH_OTHER);
    int dp = (d + 3) & ~3;
    TRY(ensure(c->vec, sizeof(float) * (size_t)n_all * dp));
    if (dp == d) {
        TRY(h2d(c, c->vec.p, vectors, sizeof(float) * (size_t)n_all * d));
    } else {
        TRY(ensure(c->stage[0], sizeof(float) * (size_t)n_all * d));
        TRY(h2d(c, c->stage[0].p, vectors, sizeof(float) * (size_t)n_all * d));
        k_pad_rows<<<grid_for(c, n_all * dp, 256), 256, 0, c->st>>>(
            c->stage[0].as<float>(), d, dp, n_all, c->vec.as<float>());
        CKL();
    }
    c->n_all = n_all;
    c->d = d;
    c->dp = dp;
    c->metric = metric;
    c->have_data = true;
    // exactness certificate: integer entries and d * range^2 < 2^24 (L2) or
    // d * range < 2^24 (L1) make every fp32 partial sum an exact integer
    {
        unsigned long long *cnt = c->counters.as<unsigned long long>();
        unsigned long long init[3] = {0ull, 0ull, 0xffffffffull};
        CK(cudaMemcpyAsync(cnt + C_NUM - 3, init, sizeof(init), cudaMemcpyHostToDevice, c->st));
        k_data_stats<<<grid_for(c, n_all * dp, 256), 256, 0, c->st>>>(c->vec.as<float>(),
                                                                      n_all * dp, cnt + C_NUM - 3);
        CKL();
        TRY(sync_counters(c));
        auto unkey = [](unsigned long long k) {
            uint32_t kk = (uint32_t)k;
            uint32_t b = (kk & 0x80000000u) ? (kk & 0x7fffffffu) : ~kk;
            float f;
            memcpy(&f, &b, 4);
            return (double)f;
        };
        double mx = unkey(c->hcnt[C_NUM - 2]), mn = unkey(c->hcnt[C_NUM - 1]);
        bool ints = c->hcnt[C_NUM - 3] == 0;
        double range = mx - mn;
        c->cert = false;
        if (ints && metric == KNNM_L2) c->cert = (double)d * range * range < 16777216.0;
        if (ints && metric == KNNM_L1) c->cert = (double)d * range < 16777216.0;
        const double maxabs = std::max(std::fabs(mx), std::fabs(mn));
        c->cert_dot = ints && metric == KNNM_L2 && maxabs <= 2048.0 &&
                      2.0 * (double)d * maxabs * maxabs < 16777216.0;
        CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * C_NUM, c->st));
        c->cert_u8 = c->cert_dot && mn >= 0.0 && mx <= 255.0 && c->u8_enabled;
        // brute force needs only exact s32 dot products and u32 distances
        c->bf_u8 = ints && mn >= 0.0 && mx <= 255.0 && (double)d * 65025.0 < 2147483648.0;
        // fixed-point limbs: every G accumulator below 2^31 (3 d 255^2)
        c->tcj_data = metric == KNNM_L2 && mn >= 0.0 && std::isfinite(mx) && mx > 0.0 &&
                      3.0 * (double)d * 65025.0 < 2147483648.0;
        if (c->tcj_data) {
            int e = 0;
            std::frexp(mx, &e);  // mx < 2^e
            c->tcj_scale = std::ldexp(1.0, 24 - e);
            c->tcj_dpad = (d + 15) & ~15;  // limb plane length (16-byte copies)
        }
        c->limbs_ready = false;
        c->sub64_ready = false;
        if (c->cert_u8) {
            c->dph = (d + 31) & ~31;  // u8 elements per row
            c->rowb = c->dph;
            TRY(ensure(c->vec16, (size_t)n_all * c->rowb));
            TRY(ensure(c->norms, sizeof(float) * (size_t)n_all));
            k_to_u8<<<grid_for(c, n_all * 32, 256, 16), 256, 0, c->st>>>(
                c->vec.as<float>(), dp, n_all, c->dph, c->vec16.as<uint8_t>(), c->norms.as<float>());
            CKL();
        } else if (c->cert_dot) {
            c->dph = (d + 15) & ~15;
            c->rowb = 2 * c->dph;
            TRY(ensure(c->vec16, sizeof(__half) * (size_t)n_all * c->dph));
            TRY(ensure(c->norms, sizeof(float) * (size_t)n_all));
            k_to_half<<<grid_for(c, n_all * 32, 256, 16), 256, 0, c->st>>>(
                c->vec.as<float>(), dp, n_all, c->dph, c->vec16.as<__half>(), c->norms.as<float>());
            CKL();
        }
    }
    c->begun = false;
    return KNNM_OK;
}

int knnm_begin(knnm_ctx *c, const int64_t *union_gids, int64_t n, const int8_t *labels, int32_t k) {
    if (c) c->state_gen++;  // the lists may change: cached phi is stale
    phi_wait(c);
    if (!c || !union_gids || !labels) return fail(KNNM_ERR_ARG, "null argument");
    if (!c->have_data) return fail(KNNM_ERR_STATE, "knnm_set_dataset first");
    if (n < 1) return fail(KNNM_ERR_ARG, "empty union");
    if (k < 1 || k > 64) return fail(KNNM_ERR_LIMIT, "k=%d outside [1, 64]", k);
    if ((uint64_t)n * (uint64_t)k >= (1ull << 31)) return fail(KNNM_ERR_LIMIT, "n*k too large");
    if (n >= (1ll << 30)) return fail(KNNM_ERR_LIMIT, "n must be below 2^30");  // WarpRow id packing
    if (union_gids[0] < 0 || union_gids[n - 1] >= c->n_all)
        return fail(KNNM_ERR_ARG, "union ids outside the dataset");
    CK(cudaSetDevice(c->device));
    PhaseTimer pt(c, PH_OTHER);
    c->n = n;
    c->k = k;
    c->slots_mode = SLOTS_PLAIN;
    c->limbs_ready = false;  // limb planes follow the union
    c->sub64_ready = false;
    c->tcj_round = false;
    // fp32 list rows only on certified data (distances are integers < 2^24)
    // and only while every loaded distance is an exact fp32 value
    c->lists_f32 = c->cert || c->cert_dot;
    TRY(ensure(c->f32chk, sizeof(unsigned long long)));
    CK(cudaMemsetAsync(c->f32chk.p, 0, sizeof(unsigned long long), c->st));
    // an identity union (0 .. n_all-1, ascending) needs no id table on the
    // device: local row = global id
    bool identity = (n == c->n_all && union_gids[0] == 0 && union_gids[n - 1] == n - 1);
    c->ug_identity = identity;
    if (!identity) {
        TRY(ensure(c->ugid, sizeof(int64_t) * n));
        TRY(h2d(c, c->ugid.p, union_gids, sizeof(int64_t) * n));
    }
    c->sub16p = c->vec16.as<uint8_t>();
    c->subnormp = c->norms.as<float>();
    if (c->cert_dot && !identity) {
        TRY(ensure(c->sub16, (size_t)n * c->rowb));
        TRY(ensure(c->subnorms, sizeof(float) * (size_t)n));
        k_gather_rows<<<grid_for(c, n * (c->rowb / 16), 256), 256, 0, c->st>>>(
            reinterpret_cast<const float *>(c->vec16.p), c->rowb / 4, c->ugid.as<int64_t>(), n,
            c->sub16.as<float>());
        CKL();
        k_gather_norms<<<grid_for(c, n, 256), 256, 0, c->st>>>(c->norms.as<float>(),
                                                                c->ugid.as<int64_t>(), n,
                                                                c->subnorms.as<float>());
        CKL();
        c->sub16p = c->sub16.as<uint8_t>();
        c->subnormp = c->subnorms.as<float>();
    }
    if (identity) {
        c->subp = c->vec.as<float>();
    } else {
        TRY(ensure(c->sub, sizeof(float) * (size_t)n * c->dp));
        k_gather_rows<<<grid_for(c, n * (c->dp / 4), 256), 256, 0, c->st>>>(
            c->vec.as<float>(), c->dp, c->ugid.as<int64_t>(), n, c->sub.as<float>());
        CKL();
        c->subp = c->sub.as<float>();
    }
    if (metric_is_cos(c)) {
        TRY(ensure(c->nrm64, sizeof(double) * (size_t)n));
        k_row_sqnorm64<<<grid_for(c, n, 128), 128, 0, c->st>>>(c->subp, c->dp, c->d, n,
                                                               c->nrm64.as<double>());
        CKL();
    }
    TRY(ensure(c->labels, n));
    TRY(h2d(c, c->labels.p, labels, n));
    TRY(ensure(c->labbits, sizeof(uint32_t) * (size_t)((n + 31) / 32 + 1)));
    k_label_bits<<<grid_for(c, (n + 31) / 32, 256), 256, 0, c->st>>>(c->labels.as<int8_t>(), n,
                                                                     c->labbits.as<uint32_t>());
    CKL();
    size_t nk = (size_t)n * k;
    TRY(ensure(c->ids, sizeof(int32_t) * nk));
    TRY(ensure(c->dists, sizeof(double) * nk));
    TRY(ensure(c->flags, nk));
    TRY(ensure(c->sizes, sizeof(int32_t) * n));
    k_init_lists<<<grid_for(c, (int64_t)nk, 256), 256, 0, c->st>>>(
        n, k, c->ids.as<int32_t>(), c->dists.as<double>(), c->flags.as<uint8_t>(),
        c->sizes.as<int32_t>());
    CKL();
    // per-round scratch sized for this union
    int W = 2 * k;
    TRY(ensure(c->indeg, sizeof(uint32_t) * (n + 1)));
    TRY(ensure(c->roff, sizeof(uint32_t) * (n + 1)));
    TRY(ensure(c->rev, sizeof(uint32_t) * nk));
    TRY(ensure(c->heavy, sizeof(int32_t) * n));
    TRY(ensure(c->giant, sizeof(int32_t) * n));
    TRY(ensure(c->nbh, sizeof(uint32_t) * (size_t)n * W));
    TRY(ensure(c->nlen, sizeof(int32_t) * n));
    TRY(ensure(c->hpairs, sizeof(uint32_t) * (n + 1)));
    TRY(ensure(c->poff, sizeof(uint64_t) * (n + 1)));
    TRY(ensure(c->worst0, sizeof(double) * n));
    TRY(ensure(c->active, sizeof(int32_t) * n));
    TRY(ensure(c->bound, sizeof(uint32_t) * (n + 1)));
    TRY(ensure(c->boff, sizeof(uint64_t) * (n + 1)));
    TRY(ensure(c->mcount, sizeof(uint32_t) * (n + 1)));
    TRY(ensure(c->moff, sizeof(uint32_t) * (n + 1)));
    TRY(ensure(c->mcur, sizeof(uint32_t) * (n + 1)));
    CK(cudaMemsetAsync(c->indeg.p, 0, sizeof(uint32_t) * (n + 1), c->st));
    c->tk = 0;
    c->have_tail = false;
    c->shard_lo = 0;
    c->shard_hi = -1;
    c->have_order = false;
    c->begun = true;
    return KNNM_OK;
}

static int load_impl(knnm_ctx *c, const int32_t *rows, int64_t m, const int32_t *g_ids,
                     const double *g_dists, const int32_t *g_sizes, int32_t gk, int32_t k1,
                     bool on_device) {
    if (c) c->state_gen++;  // the lists may change: cached phi is stale
    phi_wait(c);
    if (!c) return fail(KNNM_ERR_ARG, "null ctx");
    if (!c->begun) return fail(KNNM_ERR_STATE, "knnm_begin first");
    if (m == 0) return KNNM_OK;
    if (!rows || !g_sizes || (gk > 0 && (!g_ids || !g_dists))) return fail(KNNM_ERR_ARG, "null argument");
    if (k1 < 0 || k1 > c->k || gk < k1) return fail(KNNM_ERR_ARG, "bad k1=%d (gk=%d k=%d)", k1, gk, c->k);
    CK(cudaSetDevice(c->device));
    PhaseTimer pt(c, PH_OTHER);
    int tk = c->k - k1;
    if (tk > 0) {
        if (c->have_tail && c->tk != tk) return fail(KNNM_ERR_ARG, "inconsistent k1 across graphs");
        if (!c->have_tail) {
            size_t nt = (size_t)c->n * tk;
            TRY(ensure(c->tail_ids, sizeof(int32_t) * nt));
            TRY(ensure(c->tail_d, sizeof(double) * nt));
            TRY(ensure(c->tail_s, sizeof(int32_t) * c->n));
            k_init_lists<<<grid_for(c, (int64_t)nt, 256), 256, 0, c->st>>>(
                c->n, tk, c->tail_ids.as<int32_t>(), c->tail_d.as<double>(), nullptr,
                c->tail_s.as<int32_t>());
            CKL();
            c->tk = tk;
            c->have_tail = true;
        }
    }
    const int32_t *gi = g_ids, *gs = g_sizes;
    const double *gd = g_dists;
    TRY(ensure(c->stage[0], sizeof(int32_t) * m));
    TRY(h2d(c, c->stage[0].p, rows, sizeof(int32_t) * m));
    if (!on_device) {
        size_t mg = (size_t)m * (gk > 0 ? gk : 1);
        TRY(ensure(c->stage[1], sizeof(int32_t) * mg));
        TRY(ensure(c->stage[2], sizeof(double) * mg));
        TRY(ensure(c->stage[3], sizeof(int32_t) * m));
        if (gk > 0) {
            TRY(h2d(c, c->stage[1].p, g_ids, sizeof(int32_t) * m * gk));
            TRY(h2d(c, c->stage[2].p, g_dists, sizeof(double) * m * gk));
        }
        TRY(h2d(c, c->stage[3].p, g_sizes, sizeof(int32_t) * m));
        gi = c->stage[1].as<int32_t>();
        gd = c->stage[2].as<double>();
        gs = c->stage[3].as<int32_t>();
    }
    if (gk > 0) {
        k_load_graph<<<grid_for(c, m * gk, 256), 256, 0, c->st>>>(
            c->stage[0].as<int32_t>(), m, gi, gd, gs, gk, k1, c->k, ugid_of(c), c->n,
            c->ids.as<int32_t>(), c->dists.as<double>(), c->sizes.as<int32_t>(),
            tk > 0 ? c->tail_ids.as<int32_t>() : nullptr, tk > 0 ? c->tail_d.as<double>() : nullptr,
            tk > 0 ? c->tail_s.as<int32_t>() : nullptr, tk, c->f32chk.as<unsigned long long>());
        CKL();
    }
    CK(cudaStreamSynchronize(c->st));  // staging buffers are reused by the next call
    {
        unsigned long long bad = 0;
        CK(cudaMemcpy(&bad, c->f32chk.p, sizeof(bad), cudaMemcpyDeviceToHost));
        if (bad) c->lists_f32 = false;
    }
    return KNNM_OK;
}

int knnm_load_graph(knnm_ctx *c, const int32_t *rows, int64_t m, const int32_t *g_ids,
                    const double *g_dists, const int32_t *g_sizes, int32_t gk, int32_t k1) {
    return load_impl(c, rows, m, g_ids, g_dists, g_sizes, gk, k1, false);
}

int knnm_load_graph_dev(knnm_ctx *c, const int32_t *rows, int64_t m, const int32_t *g_ids,
                        const double *g_dists, const int32_t *g_sizes, int32_t gk, int32_t k1) {
    return load_impl(c, rows, m, g_ids, g_dists, g_sizes, gk, k1, true);
}

static int insert_impl(knnm_ctx *c, const int32_t *rows, int64_t mrows, int32_t count,
                       const int32_t *nids, int64_t m, int64_t *accepted, bool nids_on_device) {
    if (c) c->state_gen++;  // the lists may change: cached phi is stale
    phi_wait(c);
    if (!c) return fail(KNNM_ERR_ARG, "null ctx");
    if (!c->begun) return fail(KNNM_ERR_STATE, "knnm_begin first");
    if (accepted) *accepted = 0;
    if (m == 0) return KNNM_OK;
    if (!rows || (!nids && !nids_on_device)) return fail(KNNM_ERR_ARG, "null argument");
    CK(cudaSetDevice(c->device));
    TRY(ensure(c->stage[0], sizeof(int32_t) * m));
    TRY(ensure(c->stage[1], sizeof(int32_t) * m));
    if (count > 0) {
        TRY(ensure(c->stage[3], sizeof(int32_t) * mrows));
        TRY(h2d(c, c->stage[3].p, rows, sizeof(int32_t) * mrows));
        k_repeat_rows<<<grid_for(c, m, 256), 256, 0, c->st>>>(c->stage[3].as<int32_t>(), count, m,
                                                             c->stage[0].as<int32_t>());
        CKL();
    } else {
        TRY(h2d(c, c->stage[0].p, rows, sizeof(int32_t) * m));
    }
    if (!nids_on_device) TRY(h2d(c, c->stage[1].p, nids, sizeof(int32_t) * m));
    double *capd = nullptr;
    if (c->capture) {
        TRY(ensure(c->stage[2], sizeof(double) * m));
        capd = c->stage[2].as<double>();
    }
    unsigned long long *cnt = c->counters.as<unsigned long long>();
    int64_t acc_total = 0;
    bool direct = false;
    if (count > 0) {
        // row-grouped inserts with distinct rows take the direct per-row path
        TRY(ensure(c->segheavy, sizeof(uint32_t) * (size_t)((c->n + 31) / 32 + 1)));
        CK(cudaMemsetAsync(c->segheavy.p, 0, sizeof(uint32_t) * (size_t)((c->n + 31) / 32 + 1), c->st));
        CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * C_NUM, c->st));
        k_rows_distinct<<<grid_for(c, mrows, 256), 256, 0, c->st>>>(
            c->stage[3].as<int32_t>(), mrows, c->segheavy.as<uint32_t>(), cnt);
        CKL();
        unsigned long long dups = 0;
        CK(cudaMemcpyAsync(&c->hcnt[C_DUPROWS], cnt + C_DUPROWS, sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        dups = c->hcnt[C_DUPROWS];
        direct = dups == 0;
    }
    if (direct) {
        PhaseTimer pt(c, PH_UPDATE);
        CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * C_NUM, c->st));
        const int E = (c->k + 31) / 32;
        const int certi = (int)(c->cert && c->metric != KNNM_COSINE);
        // non-certified rows (exact fp64 values): batched folds from d = 64
        const bool batch = !c->cert_u8 && !certi && c->d >= 64;
        const int thr = batch ? 128 : 256;
        const int blocks = grid_for(c, mrows * 32, thr, 8);
#define KNNM_IRD_LAUNCH(EE, BB)                                                                      \
    k_insert_rows_direct<EE, BB><<<blocks, thr, 0, c->st>>>(                                        \
        c->stage[3].as<int32_t>(), mrows, count, c->stage[1].as<int32_t>(), c->subp, c->dp, c->d,    \
        c->metric, certi, c->cert_u8 ? c->sub16p : nullptr,                                          \
        c->rowb, c->cert_u8 ? c->subnormp : nullptr, c->ids.as<int32_t>(), c->dists.as<double>(),   \
        c->flags.as<uint8_t>(), c->sizes.as<int32_t>(), c->k, capd, cnt, lazy_of(c))
        if (E == 1) {
            if (batch) KNNM_IRD_LAUNCH(1, true);
            else KNNM_IRD_LAUNCH(1, false);
        } else {
            if (batch) KNNM_IRD_LAUNCH(2, true);
            else KNNM_IRD_LAUNCH(2, false);
        }
#undef KNNM_IRD_LAUNCH
        CKL();
        TRY(sync_counters(c));
        acc_total = (int64_t)c->hcnt[C_ACCEPTED];
    }
    const int64_t chunk = (int64_t)std::max<uint64_t>(bucket_budget(c), 1u << 20);
    for (int64_t c0 = 0; c0 < m && !direct; c0 += chunk) {
        const int64_t cm = std::min<int64_t>(chunk, m - c0);
        const int32_t *rows_d = c->stage[0].as<int32_t>() + c0;
        CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * C_NUM, c->st));
        {
            PhaseTimer pt(c, PH_OTHER);
            // ordinal memberships of weight 1: slot = rank of the entry
            // among the entries of its row (apply_updates_directed order)
            CK(cudaMemsetAsync(c->mcount.p, 0, sizeof(uint32_t) * (c->n + 1), c->st));
            CK(cudaMemsetAsync(c->mcur.p, 0, sizeof(uint32_t) * (c->n + 1), c->st));
            k_directed_memb<false><<<grid_for(c, cm, 256), 256, 0, c->st>>>(
                rows_d, cm, c->mcount.as<uint32_t>(), nullptr, nullptr, nullptr);
            CKL();
            TRY(scan<uint32_t, uint32_t>(c, c->mcount.as<uint32_t>(), c->moff.as<uint32_t>(), c->n));
            TRY(scan<uint32_t, uint64_t>(c, c->mcount.as<uint32_t>(), c->boff.as<uint64_t>(), c->n));
            TRY(ensure_memb(c, (uint64_t)cm, (uint64_t)cm));
            TRY(ensure_slots(c, (uint64_t)cm));
            k_directed_memb<true><<<grid_for(c, cm, 256), 256, 0, c->st>>>(
                rows_d, cm, nullptr, c->moff.as<uint32_t>(), c->mcur.as<uint32_t>(),
                c->memb.as<MembRec>());
            CKL();
            TRY(rank_memberships(c, 1u));
            k_directed_emit<<<grid_for(c, cm, 256, 32), 256, 0, c->st>>>(
                rows_d, c->stage[1].as<int32_t>() + c0, cm, c->subp, c->dp, c->d, c->metric,
                (int)(c->cert && c->metric != KNNM_COSINE), c->sizes.as<int32_t>(), c->dists.as<double>(), c->k, c->boff.as<uint64_t>(),
                c->start.as<uint32_t>(), c->Bd.as<double>(), c->Bs.as<int32_t>(),
                capd ? capd + c0 : nullptr, c->cert_u8 ? c->sub16p : nullptr, c->rowb,
                c->cert_u8 ? c->subnormp : nullptr);
            CKL();
        }
        {
            PhaseTimer pt(c, PH_UPDATE);
            c->slots_mode = SLOTS_PLAIN;  // k_directed_emit writes Bd/Bs
            TRY(run_updates(c));
        }
        acc_total += (int64_t)c->hcnt[C_ACCEPTED];
    }
    c->stats.init_evals += m;
    c->stats.accepted += acc_total;
    if (c->capture) {
        size_t o = c->cap_pa.size();
        c->cap_pa.resize(o + m);
        c->cap_pb.resize(o + m);
        c->cap_pd.resize(o + m);
        if (count > 0) {
            for (int64_t i = 0; i < m; i++) c->cap_pa[o + i] = rows[i / count];
        } else {
            memcpy(c->cap_pa.data() + o, rows, sizeof(int32_t) * m);
        }
        if (nids_on_device)
            TRY(d2h(c, c->cap_pb.data() + o, c->stage[1].p, sizeof(int32_t) * m));
        else
            memcpy(c->cap_pb.data() + o, nids, sizeof(int32_t) * m);
        TRY(d2h(c, c->cap_pd.data() + o, capd, sizeof(double) * m));
        CK(cudaStreamSynchronize(c->st));
    }
    TRY(resolve_timers(c));
    if (accepted) *accepted = acc_total;
    return KNNM_OK;
}

int knnm_insert_directed(knnm_ctx *c, const int32_t *rows, const int32_t *nids, int64_t m,
                         int64_t *accepted) {
    return insert_impl(c, rows, m, 0, nids, m, accepted, false);
}

int knnm_insert_rows(knnm_ctx *c, const int32_t *rows, int64_t mrows, int32_t count,
                     const int32_t *nids, int64_t *accepted) {
    if (count < 0) return fail(KNNM_ERR_ARG, "negative count");
    if (count == 0 || mrows == 0) {
        if (accepted) *accepted = 0;
        return KNNM_OK;
    }
    return insert_impl(c, rows, mrows, count, nids, mrows * (int64_t)count, accepted, false);
}

static int insert_impl(knnm_ctx *c, const int32_t *rows, int64_t mrows, int32_t count,
                       const int32_t *nids, int64_t m, int64_t *accepted, bool nids_on_device);

static int dup_check(knnm_ctx *c, const int64_t *rows_dev, int64_t nchk, int64_t *bad_out,
                     int64_t *nbad) {
    unsigned long long *cnt = c->counters.as<unsigned long long>();
    CK(cudaMemsetAsync(cnt + C_CAND, 0, sizeof(unsigned long long), c->st));
    int64_t work = rows_dev ? nchk : c->draw_n;
    k_dup_rows<<<grid_for(c, work, 256), 256, 0, c->st>>>(c->draws.as<int64_t>(), c->draw_n,
                                                           c->draw_t, rows_dev, nchk,
                                                           c->draw_bad.as<int64_t>(), cnt);
    CKL();
    TRY(sync_counters(c));
    int64_t nb = (int64_t)c->hcnt[C_CAND];
    if (nb > 0) {
        CK(cudaMemcpyAsync(bad_out, c->draw_bad.p, sizeof(int64_t) * nb, cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        std::sort(bad_out, bad_out + nb);  // np.nonzero order: ascending rows
    }
    *nbad = nb;
    return KNNM_OK;
}

// Generate N = (#rows) * t numpy-identical draws on the device (see
// k_pcg_raw).  rows == nullptr: fill the whole draw matrix; else overwrite
// the listed rows (device array).  *consumed = raw u32 values used.
static int pcg_fill(knnm_ctx *c, const uint64_t *st, int has0, uint32_t uint0, uint64_t m,
                    int64_t N, const int64_t *rows_dev, int64_t *consumed) {
    if (m == 0 || m > 0xFFFFFFFFull) return fail(KNNM_ERR_LIMIT, "draw range %llu", (unsigned long long)m);
    if (N == 0) {
        *consumed = 0;
        return KNNM_OK;
    }
    int64_t R = N + N / 512 + 256;
    for (int attempt = 0; attempt < 8; attempt++) {
        TRY(ensure(c->stage[2], sizeof(uint32_t) * 2 * (size_t)(R + 1)));
        TRY(ensure(c->scan_pos, sizeof(uint64_t) * (size_t)(R + 1)));
        uint32_t *val = c->stage[2].as<uint32_t>(), *acc = val + (R + 1);
        const int per = 16;
        const int64_t nout = (R + 1) / 2 + 1;
        k_pcg_raw<<<grid_for(c, (nout + per - 1) / per, 256, 8), 256, 0, c->st>>>(
            st[0], st[1], st[2], st[3], has0, uint0, m, R, per, val, acc);
        CKL();
        TRY(scan<uint32_t, uint64_t>(c, acc, c->scan_pos.as<uint64_t>(), R));
        uint64_t total = 0;
        CK(cudaMemcpyAsync(&total, c->scan_pos.as<uint64_t>() + R, sizeof(uint64_t), cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        if ((int64_t)total < N) {  // more Lemire rejections than the slack
            R = R * 2;
            continue;
        }
        unsigned long long *cnt = c->counters.as<unsigned long long>();
        k_pcg_compact<<<grid_for(c, R, 256), 256, 0, c->st>>>(val, acc, c->scan_pos.as<uint64_t>(), R, N,
                                                           c->draws.as<int64_t>(), rows_dev, c->draw_t,
                                                           cnt + C_MAXC);
        CKL();
        TRY(sync_counters(c));
        *consumed = (int64_t)c->hcnt[C_MAXC] + 1;
        return KNNM_OK;
    }
    return fail(KNNM_ERR_LIMIT, "could not generate %lld draws", (long long)N);
}

int knnm_draws_gen(knnm_ctx *c, const uint64_t *pcg, int32_t has_uint32, uint32_t uinteger,
                   uint64_t m, int64_t nrows, int32_t t, int64_t *consumed, int64_t *bad,
                   int64_t *nbad) {
    if (!c || !pcg || !consumed || !bad || !nbad || nrows < 0 || t < 1) return fail(KNNM_ERR_ARG, "bad argument");
    CK(cudaSetDevice(c->device));
    PhaseTimer pt(c, PH_OTHER);
    const size_t mm = (size_t)nrows * t;
    TRY(ensure(c->draws, sizeof(int64_t) * (mm + 1)));
    TRY(ensure(c->draw_bad, sizeof(int64_t) * (nrows + 1)));
    TRY(ensure(c->draw_rows, sizeof(int64_t) * (nrows + 1)));
    c->draw_n = nrows;
    c->draw_t = t;
    TRY(pcg_fill(c, pcg, has_uint32, uinteger, m, (int64_t)mm, nullptr, consumed));
    return dup_check(c, nullptr, 0, bad, nbad);
}

int knnm_draws_regen(knnm_ctx *c, const uint64_t *pcg, int32_t has_uint32, uint32_t uinteger,
                     uint64_t m, const int64_t *rows, int64_t nrows, int64_t *consumed, int64_t *bad,
                     int64_t *nbad) {
    if (!c || !pcg || !rows || !consumed || !bad || !nbad) return fail(KNNM_ERR_ARG, "bad argument");
    if (nrows > c->draw_n) return fail(KNNM_ERR_ARG, "too many rows");
    CK(cudaSetDevice(c->device));
    PhaseTimer pt(c, PH_OTHER);
    if (nrows == 0) {
        *consumed = 0;
        *nbad = 0;
        return KNNM_OK;
    }
    TRY(h2d(c, c->draw_rows.p, rows, sizeof(int64_t) * nrows));
    TRY(pcg_fill(c, pcg, has_uint32, uinteger, m, nrows * (int64_t)c->draw_t, c->draw_rows.as<int64_t>(),
                 consumed));
    return dup_check(c, c->draw_rows.as<int64_t>(), nrows, bad, nbad);
}

int knnm_draws_load(knnm_ctx *c, const int64_t *cand, int64_t nrows, int32_t t, int64_t *bad,
                    int64_t *nbad) {
    if (!c || !cand || !bad || !nbad || nrows < 0 || t < 1) return fail(KNNM_ERR_ARG, "bad argument");
    CK(cudaSetDevice(c->device));
    PhaseTimer pt(c, PH_OTHER);
    size_t m = (size_t)nrows * t;
    TRY(ensure(c->draws, sizeof(int64_t) * m));
    TRY(ensure(c->draw_bad, sizeof(int64_t) * (nrows + 1)));
    TRY(ensure(c->draw_rows, sizeof(int64_t) * (nrows + 1)));
    TRY(h2d(c, c->draws.p, cand, sizeof(int64_t) * m));
    c->draw_n = nrows;
    c->draw_t = t;
    return dup_check(c, nullptr, 0, bad, nbad);
}

int knnm_draws_replace(knnm_ctx *c, const int64_t *rows, int64_t nrows, const int64_t *vals,
                       int64_t *bad, int64_t *nbad) {
    if (!c || !rows || !vals || !bad || !nbad) return fail(KNNM_ERR_ARG, "bad argument");
    if (nrows > c->draw_n) return fail(KNNM_ERR_ARG, "too many rows");
    CK(cudaSetDevice(c->device));
    PhaseTimer pt(c, PH_OTHER);
    if (nrows == 0) {
        *nbad = 0;
        return KNNM_OK;
    }
    TRY(ensure(c->stage[2], sizeof(int64_t) * (size_t)nrows * c->draw_t));
    TRY(h2d(c, c->draw_rows.p, rows, sizeof(int64_t) * nrows));
    TRY(h2d(c, c->stage[2].p, vals, sizeof(int64_t) * (size_t)nrows * c->draw_t));
    k_put_rows<<<grid_for(c, nrows * c->draw_t, 256), 256, 0, c->st>>>(
        c->draws.as<int64_t>(), c->draw_t, c->draw_rows.as<int64_t>(), nrows, c->stage[2].as<int64_t>());
    CKL();
    return dup_check(c, c->draw_rows.as<int64_t>(), nrows, bad, nbad);
}

int knnm_draws_insert_range(knnm_ctx *c, const int32_t *rows, const int32_t *pool, int64_t npool,
                            int64_t r0, int64_t r1, int64_t *accepted) {
    if (c) c->state_gen++;  // the lists may change: cached phi is stale
    phi_wait(c);
    if (!c || !rows || !pool) return fail(KNNM_ERR_ARG, "bad argument");
    if (!c->begun) return fail(KNNM_ERR_STATE, "knnm_begin first");
    if (r0 < 0 || r1 < r0 || r1 > c->draw_n) return fail(KNNM_ERR_ARG, "bad draw rows [%lld, %lld)", (long long)r0, (long long)r1);
    CK(cudaSetDevice(c->device));
    const int64_t m = (r1 - r0) * c->draw_t;
    if (m == 0) {
        if (accepted) *accepted = 0;
        return KNNM_OK;
    }
    TRY(ensure(c->pool, sizeof(int32_t) * npool));
    TRY(h2d(c, c->pool.p, pool, sizeof(int32_t) * npool));
    TRY(ensure(c->stage[1], sizeof(int32_t) * m));
    k_pool_map<<<grid_for(c, m, 256), 256, 0, c->st>>>(c->draws.as<int64_t>() + r0 * c->draw_t, m,
                                                         c->pool.as<int32_t>(), c->stage[1].as<int32_t>());
    CKL();
    return insert_impl(c, rows + r0, r1 - r0, c->draw_t, nullptr, m, accepted, true);
}

int knnm_draws_insert(knnm_ctx *c, const int32_t *rows, const int32_t *pool, int64_t npool,
                      int64_t *accepted) {
    if (!c) return fail(KNNM_ERR_ARG, "null ctx");
    return knnm_draws_insert_range(c, rows, pool, npool, 0, c->draw_n, accepted);
}

// Fixed-point limb planes of the union rows for k_join_tc (once per merge).
static int ensure_limbs(knnm_ctx *c) {
    if (c->limbs_ready) return KNNM_OK;
    const int64_t n = c->n;
    TRY(ensure(c->limbs, (size_t)n * 3 * c->tcj_dpad));
    TRY(ensure(c->lnx, sizeof(double) * (size_t)n));
    TRY(ensure(c->lax, sizeof(double) * (size_t)n));
    k_make_limbs<<<grid_for(c, n * 32, 256, 16), 256, 0, c->st>>>(c->subp, c->dp, c->d, n, c->tcj_dpad,
                                                                  c->tcj_scale, c->limbs.as<uint8_t>(),
                                                                  c->lnx.as<double>(), c->lax.as<double>());
    CKL();
    c->limbs_ready = true;
    return KNNM_OK;
}

// fp64 copy of the union rows (+ the roots of the cosine norms) for
// k_join_dense (once per merge).
static int ensure_sub64(knnm_ctx *c) {
    if (c->sub64_ready) return KNNM_OK;
    const int64_t n = c->n;
    TRY(ensure(c->sub64, sizeof(double) * (size_t)n * c->dp));
    k_to_f64<<<grid_for(c, n * c->dp, 256), 256, 0, c->st>>>(c->subp, n * c->dp, c->sub64.as<double>());
    CKL();
    if (metric_is_cos(c)) {
        TRY(ensure(c->nsq, sizeof(double) * (size_t)n));
        k_sqrt64<<<grid_for(c, n, 256), 256, 0, c->st>>>(c->nrm64.as<double>(), n, c->nsq.as<double>());
        CKL();
    }
    c->sub64_ready = true;
    return KNNM_OK;
}

// Route of the local join for this round (dataset, k, rev_cap, mode).
struct JoinRoute {
    bool use_mma, tiled, lazy, tc, dense;
    int dense_rows;  // k_join_dense circular row buffer
    size_t smem, smem_tiled, smem_mma;
};

static int join_route(knnm_ctx *c, int W, int mode, JoinRoute *r) {
    const size_t smem = sizeof(float) * (size_t)W * c->dp;
    const size_t smem_tiled = sizeof(float) * (size_t)W * (c->dp + 4);
    const int Wp = mj_rows(W, mode);
    const size_t mj_per_warp = mj_meta_bytes(Wp) + (size_t)Wp * (c->rowb + 16);
    const size_t smem_mma = MJ_WARPS * mj_per_warp;
    const bool use_mma = c->cert_dot && smem_mma <= 200 * 1024 &&
                         (c->join_variant == 2 || c->join_variant < 0);
    // the d-chunked lazy route streams rows through fixed-size buffers, so it
    // takes every non-certified long-row dataset and anything whose whole
    // hood does not fit shared memory (e.g. d = 960 with k >= 27)
    const bool tiled_fits = smem_tiled <= 200 * 1024;
    const bool tiled = !use_mma && c->join_variant != 0 &&
                       (c->join_variant == 1 || tiled_fits || c->d > c->lazy_min_d);
    const bool lazy = tiled && ((!c->cert && c->d > c->lazy_min_d) || !tiled_fits);
    if (!use_mma && !tiled && smem > 200 * 1024)
        return fail(KNNM_ERR_LIMIT, "neighbourhood of %d x %d floats exceeds shared memory", W, c->dp);
    if (tiled && !lazy && !tiled_fits)
        return fail(KNNM_ERR_LIMIT, "neighbourhood of %d x %d floats exceeds shared memory", W, c->dp);
    c->slots_mode = use_mma ? SLOTS_PACKED
                    : tiled ? (lazy ? SLOTS_LAZY : c->cert ? SLOTS_PACKED : SLOTS_PLAIN)
                            : SLOTS_PLAIN;
    // lazy rows on the 5th-generation tensor cores (rigorous fixed-point
    // bounds, k_join_tc) when the data is non-negative and the hood's three
    // accumulators fit TMEM
    r->tc = lazy && c->tcj_data && W <= TJC_MAX_W && (c->join_variant == 3 || c->join_variant < 0);
    c->tcj_round = r->tc;
    // short non-certified rows: every admissible pair exact in register-
    // blocked fp64 tiles (k_join_dense) when the hood's fp64 rows fit
    r->dense_rows = dj_rows(W, c->dp, metric_is_cos(c));
    r->dense = tiled && !lazy && !c->cert && r->dense_rows > 0 &&
               (c->join_variant == 4 || (c->join_variant < 0 && c->d >= 64));
    r->use_mma = use_mma;
    r->tiled = tiled;
    r->lazy = lazy;
    r->smem = smem;
    r->smem_tiled = smem_tiled;
    r->smem_mma = smem_mma;
    return KNNM_OK;
}

// One hood chunk of a round: membership layout -> bucket offsets -> local
// join -> (unless local_only) apply.  ``counted``: k_assemble already
// counted (and, with fused_memb, wrote) the memberships of exactly these
// hoods.  Chunks must run in ascending hood order (the reference's per-row
// order is (u, p, q)).
static int join_chunk(knnm_ctx *c, int32_t mode, int W, const int32_t *act, int64_t nact,
                      uint64_t pairs2, bool counted, bool fused_memb, bool local_only,
                      int64_t *acc_out) {
    const int64_t n = c->n;
    unsigned long long *cnt = c->counters.as<unsigned long long>();
    JoinRoute rt;
    TRY(join_route(c, W, mode, &rt));
    const bool use_mma = rt.use_mma, tiled = rt.tiled, lazy = rt.lazy;
    const size_t smem = rt.smem, smem_tiled = rt.smem_tiled, smem_mma = rt.smem_mma;
    c->stats.join_row_bytes = use_mma ? c->rowb : 4 * c->dp;
    // long rows (large d): more warps share one staged hood
    const int tj_threads = smem_tiled > 16 * 1024 ? TJ_WARPS_BIG * 32 : TJ_THREADS;
    // lower bounds of the exact value from the fp32 one (LazyExact)
    const double lo_rel = 1.0 - (double)(c->d + 8) * ldexp(1.0, -23);
    const double lo_abs = (double)(4 * c->d + 64) * ldexp(1.0, -24);
    CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * C_NUM, c->st));
    {
        PhaseTimer pt(c, PH_JOIN);
        // reference-order slot layout (see MembRec in knnm_kernels.cuh);
        // k_assemble already counted every active hood's memberships
        // (and, when fused, wrote their records)
        const bool fused = counted && fused_memb;
        if (!fused) CK(cudaMemsetAsync(c->mcur.p, 0, sizeof(uint32_t) * (n + 1), c->st));
        const int hgrid = grid_for(c, nact * 32, 256, 16);
        if (!counted) {
            CK(cudaMemsetAsync(c->bound.p, 0, sizeof(uint32_t) * (n + 1), c->st));
            CK(cudaMemsetAsync(c->mcount.p, 0, sizeof(uint32_t) * (n + 1), c->st));
            k_hood_memb<false><<<hgrid, 256, 0, c->st>>>(
                act, (int)nact, c->nbh.as<uint32_t>(), c->nlen.as<int32_t>(), W,
                c->labels.as<int8_t>(), mode, c->bound.as<uint32_t>(),
                c->mcount.as<uint32_t>(), nullptr, nullptr, nullptr);
            CKL();
        }
        // fused: bucket sizes are written by rank_memberships below
        if (!fused) TRY(scan<uint32_t, uint64_t>(c, c->bound.as<uint32_t>(), c->boff.as<uint64_t>(), n));
        // tensor-core join, unsharded: generation-tagged slots, no prefill
        const bool tagged = use_mma && !local_only && c->gen_slots && n < (int64_t)(1 << 24);
        if (tagged) TRY(ensure_slots_tagged(c, pairs2));
        else TRY(ensure_slots(c, pairs2, !use_mma));
        if (!fused) {
            TRY(scan<uint32_t, uint32_t>(c, c->mcount.as<uint32_t>(), c->moff.as<uint32_t>(), n));
            TRY(ensure_memb(c, (uint64_t)n * W, (uint64_t)n * W));
            k_hood_memb<true><<<hgrid, 256, 0, c->st>>>(
                act, (int)nact, c->nbh.as<uint32_t>(), c->nlen.as<int32_t>(), W,
                c->labels.as<int8_t>(), mode, nullptr, nullptr, c->moff.as<uint32_t>(),
                c->mcur.as<uint32_t>(), c->memb.as<MembRec>());
            CKL();
        }
        TRY(rank_memberships(c, (uint32_t)W, fused));
        if (fused) TRY(scan<uint32_t, uint64_t>(c, c->bound.as<uint32_t>(), c->boff.as<uint64_t>(), n));
        const uint64_t *boff = c->boff.as<uint64_t>();
        const uint32_t *stt = c->start.as<uint32_t>();
        double *Bd = c->Bd.as<double>();
        int32_t *Bs = c->Bs.as<int32_t>();
        PhaseTimer ptk(c, PH_JOINK);  // the local-join kernel alone (roofline)
        if (use_mma) {
            int per_sm = 1;
            // 32-entry position blocks per hood
            const int nb = W <= 32 ? 1 : W <= 64 ? 2 : 4;
            const void *fn;
#define KNNM_MJ_FN(U, N) (mode == 0 ? (const void *)k_join_mma<U, N, 0>                     \
                  : mode == 1 ? (const void *)k_join_mma<U, N, 1> : (const void *)k_join_mma<U, N, 2>)
            if (c->cert_u8) fn = nb == 1 ? KNNM_MJ_FN(true, 1) : nb == 2 ? KNNM_MJ_FN(true, 2) : KNNM_MJ_FN(true, 4);
            else fn = nb == 1 ? KNNM_MJ_FN(false, 1) : nb == 2 ? KNNM_MJ_FN(false, 2) : KNNM_MJ_FN(false, 4);
#undef KNNM_MJ_FN
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, MJ_WARPS * 32, smem_mma));
            unsigned grid = (unsigned)std::min<int64_t>((nact + MJ_WARPS - 1) / MJ_WARPS,
                                                        (int64_t)c->sms * std::max(per_sm, 1));
            if (grid == 0) grid = 1;
            int nact32 = (int)nact, Wi = W, modei = mode, rowbi = c->rowb;
            const uint32_t *nbhp = c->nbh.as<uint32_t>();
            const int32_t *nlp = c->nlen.as<int32_t>();
            const int8_t *labp = c->labels.as<int8_t>();
            const uint8_t *s16 = c->sub16p;
            // per-row worst / norm / bucket base in one 16-byte record
            TRY(ensure(c->rowmeta, sizeof(RowMeta) * (size_t)n));
            k_rowmeta<<<grid_for(c, n, 256), 256, 0, c->st>>>(n, c->worst0.as<double>(), c->subnormp,
                                                             boff, c->rowmeta.as<RowMeta>());
            CKL();
            const RowMeta *rmp = c->rowmeta.as<RowMeta>();
            uint32_t gtag = c->slot_gen << 24;  // 0: NaN-prefilled slots
            void *args[] = {(void *)&act, (void *)&nact32, (void *)&nbhp, (void *)&nlp, (void *)&Wi,
                            (void *)&labp, (void *)&modei, (void *)&s16, (void *)&rowbi,
                            (void *)&rmp, (void *)&stt, (void *)&Bd, (void *)&Bs, (void *)&gtag};
            CK(cudaLaunchKernel(fn, dim3(grid), dim3(MJ_WARPS * 32), args, smem_mma, c->st));
        } else if (tiled) {
            // non-certified rows: exact values in the join from the
            // staged rows for short rows; for long rows the exact
            // evaluation is deferred to the apply (LazyExact), which
            // needs it for few slots only
            const void *fn;
            if (lazy) fn = nullptr;  // k_join_chunked below
            else if (c->cert) fn = c->metric == 1 ? (const void *)k_join_tiled<1, true, false>
                                             : (const void *)k_join_tiled<0, true, false>;
            else fn = c->metric == 1 ? (const void *)k_join_tiled<1, false, false>
                      : c->metric == 2 ? (const void *)k_join_tiled<2, false, false>
                                       : (const void *)k_join_tiled<0, false, false>;
            int per_sm = 1;
            if (fn) CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, tj_threads, smem_tiled));
            unsigned grid = (unsigned)std::min<int64_t>(nact, (int64_t)c->sms * std::max(per_sm, 1));
            if (grid == 0) grid = 1;
            int na = (int)nact;
            const double *nrm = c->metric == KNNM_COSINE ? c->nrm64.as<double>() : nullptr;
#define KNNM_TJ_ARGS                                                                          \
act, na, c->nbh.as<uint32_t>(), c->nlen.as<int32_t>(), W, c->labels.as<int8_t>(), mode,  \
c->subp, c->dp, c->d, c->worst0.as<double>(), boff, stt, Bd, Bs, lo_rel, lo_abs, nrm, cnt
#define KNNM_TJ_LAUNCH(T, C, L) k_join_tiled<T, C, L><<<grid, tj_threads, smem_tiled, c->st>>>(KNNM_TJ_ARGS)
            if (c->cert && !lazy) {
                if (c->metric == 1) KNNM_TJ_LAUNCH(1, true, false);
                else KNNM_TJ_LAUNCH(0, true, false);
            } else if (rt.dense) {
                TRY(ensure_sub64(c));
                const bool cos = metric_is_cos(c);
                const int RB = dj_rec_bytes(W, cos);
                TRY(ensure(c->djrec, (size_t)nact * RB));
                const int rgrid = grid_for(c, nact * 32, 256, 16);
                if (cos)
                    k_dense_rec<true><<<rgrid, 256, 0, c->st>>>(act, na, c->nbh.as<uint32_t>(), c->nlen.as<int32_t>(), W,
                                                               c->worst0.as<double>(), boff, stt, nrm, c->nsq.as<double>(),
                                                               c->djrec.as<uint8_t>(), RB);
                else
                    k_dense_rec<false><<<rgrid, 256, 0, c->st>>>(act, na, c->nbh.as<uint32_t>(), c->nlen.as<int32_t>(), W,
                                                                c->worst0.as<double>(), boff, stt, nullptr, nullptr,
                                                                c->djrec.as<uint8_t>(), RB);
                CKL();
                const int nrows = rt.dense_rows;
                const size_t smem_dj = dj_smem_bytes(W, c->dp, cos, nrows);
                const unsigned gdj = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nact, (int64_t)c->sms));
#define KNNM_DJ_LAUNCH(T)                                                                        \
k_join_dense<T><<<gdj, DJ_THREADS, smem_dj, c->st>>>(na, W, mode, c->sub64.as<double>(), c->dp, c->d, \
c->djrec.as<uint8_t>(), RB, nrows, Bd, Bs, cnt)
                if (c->metric == 1) KNNM_DJ_LAUNCH(1);
                else if (c->metric == 2) KNNM_DJ_LAUNCH(2);
                else KNNM_DJ_LAUNCH(0);
#undef KNNM_DJ_LAUNCH
                c->stats.dense_join_launches += 1;
            } else if (rt.tc) {
                TRY(ensure_limbs(c));
                // one CTA per SM: a deep ring of (hood, K block) stages
                const int stages = tjc_stages(W);
                const unsigned gtc = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nact, (int64_t)c->sms));
                k_join_tc<<<gtc, TJC_THREADS, tjc_smem_bytes(W, stages), c->st>>>(
                    act, na, c->nbh.as<uint32_t>(), c->nlen.as<int32_t>(), W, mode, c->limbs.as<uint8_t>(),
                    c->tcj_dpad, c->d, stages, c->lnx.as<double>(), c->lax.as<double>(), 1.0 / c->tcj_scale,
                    c->worst0.as<double>(), boff, stt, Bd, Bs);
                c->stats.tc_join_launches += 1;
            } else if (lazy) {
                // rows stream through two CJ_DC-dimension buffers
                const size_t smem_cj = CJ_NBUF * (size_t)W * (CJ_DC / 4 + 1) * sizeof(float4);
                const void *fc = c->metric == 1 ? (const void *)k_join_chunked<1>
                                 : c->metric == 2 ? (const void *)k_join_chunked<2>
                                                  : (const void *)k_join_chunked<0>;
                int per_cj = 1;
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_cj, fc, CJ_WARPS * 32, smem_cj));
                const unsigned gcj = (unsigned)std::max<int64_t>(
                    1, std::min<int64_t>(nact, (int64_t)c->sms * std::max(per_cj, 1)));
#define KNNM_CJ_LAUNCH(T)                                                                          \
k_join_chunked<T><<<gcj, CJ_WARPS * 32, smem_cj, c->st>>>(                                     \
act, na, c->nbh.as<uint32_t>(), c->nlen.as<int32_t>(), W, mode, c->subp, c->dp,           \
c->worst0.as<double>(), boff, stt, Bd, Bs, lo_rel, lo_abs)
                if (c->metric == 1) KNNM_CJ_LAUNCH(1);
                else if (c->metric == 2) KNNM_CJ_LAUNCH(2);
                else KNNM_CJ_LAUNCH(0);
#undef KNNM_CJ_LAUNCH
            } else {
                if (c->metric == 1) KNNM_TJ_LAUNCH(1, false, false);
                else if (c->metric == 2) KNNM_TJ_LAUNCH(2, false, false);
                else KNNM_TJ_LAUNCH(0, false, false);
            }
#undef KNNM_TJ_LAUNCH
#undef KNNM_TJ_ARGS
        } else {
#define KNNM_JE_ARGS                                                                          \
act, c->nbh.as<uint32_t>(), c->nlen.as<int32_t>(), W, c->labels.as<int8_t>(), mode,       \
c->subp, c->dp, c->d, c->worst0.as<double>(), boff, stt, Bd, Bs
            if (c->metric == 1)
                k_join_exact<1><<<(unsigned)nact, JOIN_THREADS, smem, c->st>>>(KNNM_JE_ARGS);
            else if (c->metric == 2)
                k_join_exact<2><<<(unsigned)nact, JOIN_THREADS, smem, c->st>>>(KNNM_JE_ARGS);
            else
                k_join_exact<0><<<(unsigned)nact, JOIN_THREADS, smem, c->st>>>(KNNM_JE_ARGS);
#undef KNNM_JE_ARGS
        }
        CKL();
        c->stats.join_launches += 1;
    }
    if (local_only) {  // slots stay for the exchange (knnm_local_views)
        TRY(sync_counters(c));
        c->stats.exact_evals += (int64_t)c->hcnt[C_EXACT];
        return KNNM_OK;
    }
    {
        PhaseTimer pt(c, PH_UPDATE);
        TRY(run_updates(c));
    }
    c->stats.exact_evals += (int64_t)c->hcnt[C_EXACT];
    *acc_out += (int64_t)c->hcnt[C_ACCEPTED];
    return KNNM_OK;
}

// Hood chunks for a round whose 2P slots exceed the candidate budget:
// consecutive hood ranges (ascending, which keeps the reference's per-row
// order: keys are (u, p, q)), each holding at most ``budget`` slots (a single
// hood larger than that gets a chunk of its own).
static int plan_chunks(knnm_ctx *c, uint64_t budget, std::vector<std::vector<int32_t>> &lists,
                       std::vector<uint64_t> &pairs2) {
    const int64_t n = c->n;
    std::vector<uint64_t> hpoff(n + 1);
    std::vector<uint32_t> hh(n);
    CK(cudaMemcpyAsync(hpoff.data(), c->poff.p, sizeof(uint64_t) * (n + 1), cudaMemcpyDeviceToHost,
                       c->st));
    CK(cudaMemcpyAsync(hh.data(), c->hpairs.p, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    c->stats.join_redos += 1;
    lists.clear();
    pairs2.clear();
    int64_t lo = 0;
    while (lo < n) {
        int64_t hi = lo;
        std::vector<int32_t> lst;
        while (hi < n && (2 * (hpoff[hi + 1] - hpoff[lo]) <= budget || hi == lo)) {
            if (hh[hi]) lst.push_back((int32_t)hi);
            hi++;
        }
        if (!lst.empty()) {
            lists.push_back(std::move(lst));
            pairs2.push_back(2 * (hpoff[hi] - hpoff[lo]));
        }
        lo = hi;
    }
    return KNNM_OK;
}

static int round_impl(knnm_ctx *c, int32_t mode, int32_t rev_cap, uint64_t round_seed,
                      int64_t *pairs, int64_t *accepted, bool local_only) {
    if (c) c->state_gen++;  // the lists may change: cached phi is stale
    // (no phi_wait here: a pending phi overlaps the reverse, assembly and
    // join; run_updates waits before the apply writes the lists)
    if (!c) return fail(KNNM_ERR_ARG, "null ctx");
    if (!c->begun) return fail(KNNM_ERR_STATE, "knnm_begin first");
    if (mode < 0 || mode > 2) return fail(KNNM_ERR_ARG, "mode %d", mode);
    if (rev_cap < 0 || rev_cap > c->k) return fail(KNNM_ERR_ARG, "rev_cap %d", rev_cap);
    CK(cudaSetDevice(c->device));
    c->slots_mode = SLOTS_PLAIN;  // set by the join route below
    int64_t n = c->n;
    int k = c->k;
    int W = k + rev_cap;
    // owned rows: all of them, or the shard set by knnm_set_shard
    const int64_t lo = local_only ? c->shard_lo : 0;
    bool fused_memb = false;  // k_assemble writes the membership records
    const int64_t hi = local_only ? (c->shard_hi < 0 ? n : c->shard_hi) : n;
    unsigned long long *cnt = c->counters.as<unsigned long long>();
    CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * C_NUM, c->st));
    {
        PhaseTimer pt(c, PH_REVERSE);
        CK(cudaMemsetAsync(c->indeg.p, 0, sizeof(uint32_t) * (n + 1), c->st));
        if (c->new_cap > 0 && c->new_cap < k) {  // rho < 1: sample the new entries
            k_sample_new<<<grid_for(c, n, 128), 128, 0, c->st>>>(c->sizes.as<int32_t>(), n, k,
                                                                 c->flags.as<uint8_t>(), c->new_cap,
                                                                 round_seed);
            CKL();
        }
        TRY(ensure(c->live, (size_t)n));
        CK(cudaMemsetAsync(c->live.p, 0, (size_t)n, c->st));
        k_rev_count<<<grid_for(c, n * k, 256), 256, 0, c->st>>>(
            c->ids.as<int32_t>(), c->flags.as<uint8_t>(), c->sizes.as<int32_t>(), n, k,
            c->indeg.as<uint32_t>(), lo, hi, c->live.as<uint8_t>());
        CKL();
        TRY(scan<uint32_t, uint32_t>(c, c->indeg.as<uint32_t>(), c->roff.as<uint32_t>(), n));
        k_rev_fill<<<grid_for(c, n * k, 256), 256, 0, c->st>>>(
            c->ids.as<int32_t>(), c->flags.as<uint8_t>(), c->sizes.as<int32_t>(), n, k,
            c->roff.as<uint32_t>(), c->indeg.as<uint32_t>(), c->rev.as<uint32_t>(), lo, hi,
            c->live.as<uint8_t>());
        CKL();
        k_find_heavy<<<grid_for(c, hi - lo, 256), 256, 0, c->st>>>(
            c->roff.as<uint32_t>(), lo, hi, std::max(rev_cap, WARP_REV_MAX), c->heavy.as<int32_t>(), cnt,
            c->live.as<uint8_t>(), c->giant.as<int32_t>(), BLOCK_SORT_MAX);
        CKL();
        // heavy segments: most fit a 2 x 16 KB sort (several blocks per SM),
        // the rest a 2 x 64 KB one
        k_rev_heavy<<<c->sms * 8, 256, 2 * sizeof(uint32_t) * HEAVY_SORT_SMALL, c->st>>>(
            c->heavy.as<int32_t>(), cnt, c->roff.as<uint32_t>(), c->rev.as<uint32_t>(), rev_cap,
            round_seed, nullptr, HEAVY_SORT_SMALL, 0);
        CKL();
        k_rev_heavy<<<c->sms * 2, 256, 2 * sizeof(uint32_t) * BLOCK_SORT_MAX, c->st>>>(
            c->heavy.as<int32_t>(), cnt, c->roff.as<uint32_t>(), c->rev.as<uint32_t>(), rev_cap,
            round_seed, nullptr, BLOCK_SORT_MAX, HEAVY_SORT_SMALL);
        CKL();
        // rows too long for a block's shared memory (in-degree above
        // BLOCK_SORT_MAX): one block in global scratch sized for any degree
        // (<= n); it finds them from the device-side list, so no host sync
        if (next_pow2((uint32_t)n) > (uint32_t)BLOCK_SORT_MAX) {
            TRY(ensure(c->gscratch32, 2 * sizeof(uint32_t) * next_pow2((uint32_t)n)));
            k_rev_heavy<<<1, 1024, 0, c->st>>>(c->giant.as<int32_t>(), cnt, c->roff.as<uint32_t>(),
                                               c->rev.as<uint32_t>(), rev_cap, round_seed,
                                               c->gscratch32.as<uint32_t>(), BLOCK_SORT_MAX, 0);
            CKL();
        }
    }
    if (!local_only && !c->have_order && c->locality_iters > 0) {
        PhaseTimer pt(c, PH_ASSEMBLE);
        TRY(build_locality_order(c));
    }
    {
        PhaseTimer pt(c, PH_ASSEMBLE);
        if (local_only) {
            // the join needs the round-start worst of every row (lists are
            // replicated); hoods outside the shard contribute no pairs
            k_worst0_all<<<grid_for(c, n, 256), 256, 0, c->st>>>(c->sizes.as<int32_t>(),
                                                                 c->dists.as<double>(), n, k,
                                                                 c->worst0.as<double>());
            CKL();
            CK(cudaMemsetAsync(c->hpairs.p, 0, sizeof(uint32_t) * (n + 1), c->st));
        }
        CK(cudaMemsetAsync(c->bound.p, 0, sizeof(uint32_t) * (n + 1), c->st));
        CK(cudaMemsetAsync(c->mcount.p, 0, sizeof(uint32_t) * (n + 1), c->st));
        // membership records written by k_assemble itself (unsharded rounds):
        // row x's segment holds indeg(x) + k + 1 records (see k_assemble)
        fused_memb = !local_only && lo == 0 && hi == n;
        if (fused_memb) {
            TRY(ensure_memb(c, (uint64_t)n * (uint64_t)(2 * k + 1), (uint64_t)n * W));
            TRY(ensure(c->mpack, sizeof(unsigned long long) * (size_t)n));
            k_mpack_init<<<grid_for(c, n, 256), 256, 0, c->st>>>(c->roff.as<uint32_t>(), n, k,
                                                                 c->mpack.as<unsigned long long>());
            CKL();
        }
#define KNNM_ASM_LAUNCH(M)                                                                          \
        k_assemble<M><<<grid_for(c, (hi - lo) * 32, ASM_WARPS * 32, 16), ASM_WARPS * 32, 0, c->st>>>(  \
            c->ids.as<int32_t>(), c->flags.as<uint8_t>(), c->sizes.as<int32_t>(),                   \
            c->dists.as<double>(), hi, k, rev_cap, c->roff.as<uint32_t>(), c->rev.as<uint32_t>(),   \
            round_seed, c->labbits.as<uint32_t>(), mode, W, c->nbh.as<uint32_t>(),                  \
            c->nlen.as<int32_t>(), c->hpairs.as<uint32_t>(), c->worst0.as<double>(),                \
            c->active.as<int32_t>(), cnt, lo, c->bound.as<uint32_t>(), c->mcount.as<uint32_t>(),    \
            (!local_only && c->have_order) ? c->order.as<int32_t>() : nullptr,                      \
            fused_memb ? c->memb.as<MembRec>() : nullptr,                                           \
            fused_memb ? c->mpack.as<unsigned long long>() : nullptr, c->live.as<uint8_t>())
        if (mode == 0) KNNM_ASM_LAUNCH(0);
        else if (mode == 1) KNNM_ASM_LAUNCH(1);
        else KNNM_ASM_LAUNCH(2);
#undef KNNM_ASM_LAUNCH
        CKL();
        TRY(scan<uint32_t, uint64_t>(c, c->hpairs.as<uint32_t>(), c->poff.as<uint64_t>(), n));
    }
    uint64_t P = 0;
    CK(cudaMemcpyAsync(&c->hcnt[C_NUM - 1], c->poff.as<uint64_t>() + n, sizeof(uint64_t), cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(c->hcnt, c->counters.p, sizeof(unsigned long long) * (C_NUM - 1), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    P = c->hcnt[C_NUM - 1];
    unsigned long long nactive = c->hcnt[C_ACTIVE];
    c->stats.members += (int64_t)c->hcnt[C_MEMBERS];
    c->stats.active_hoods += (int64_t)nactive;
    c->stats.heavy_rev_rows += (int64_t)c->hcnt[C_HEAVY_REV];
    c->stats.pairs += (int64_t)P;
    c->stats.rounds += 1;

    if (c->capture && P > 0) {
        DBuf pa, pb, pd;
        TRY(ensure(pa, sizeof(int32_t) * P));
        TRY(ensure(pb, sizeof(int32_t) * P));
        TRY(ensure(pd, sizeof(double) * P));
        k_capture_pairs<<<(unsigned)((n + 127) / 128), 128, 0, c->st>>>(
            c->nbh.as<uint32_t>(), c->nlen.as<int32_t>(), 0, n, W, c->labels.as<int8_t>(), mode,
            c->poff.as<uint64_t>(), c->subp, c->dp, c->d, c->metric, pa.as<int32_t>(),
            pb.as<int32_t>(), pd.as<double>());
        CKL();
        size_t o = c->cap_pa.size();
        c->cap_pa.resize(o + P);
        c->cap_pb.resize(o + P);
        c->cap_pd.resize(o + P);
        TRY(d2h(c, c->cap_pa.data() + o, pa.p, sizeof(int32_t) * P));
        TRY(d2h(c, c->cap_pb.data() + o, pb.p, sizeof(int32_t) * P));
        TRY(d2h(c, c->cap_pd.data() + o, pd.p, sizeof(double) * P));
        CK(cudaStreamSynchronize(c->st));
        release(pa);
        release(pb);
        release(pd);
    }

    int64_t acc_total = 0;
    JoinRoute rt0;  // the slot format is fixed even when this rank has no pairs
    TRY(join_route(c, W, mode, &rt0));
    const uint64_t budget = bucket_budget(c, rt0.use_mma);
    if (local_only) {
        // sharded round: the join runs chunk by chunk in knnm_local_join,
        // with the exchange of each chunk's slots in between
        c->lc_mode = mode;
        c->lc_W = W;
        c->lc_single = true;
        c->lc_nact = (int64_t)nactive;
        c->lc_lists.clear();
        c->lc_pairs2.clear();
        if (P > 0) {
            if (2 * P <= budget) {
                c->lc_pairs2.push_back(2 * P);
            } else {
                c->lc_single = false;
                TRY(plan_chunks(c, budget, c->lc_lists, c->lc_pairs2));
            }
        }
        TRY(resolve_timers(c));
        if (pairs) *pairs = (int64_t)P;
        if (accepted) *accepted = 0;
        return KNNM_OK;
    }
    if (P > 0) {
        if (2 * P <= budget) {
            // phi inside the round's final wait, unless the caller reduces it
            // asynchronously (knnm_phi_async) while the next round runs
            c->phi_in_updates = !c->st2;
            const int rc = join_chunk(c, mode, W, c->active.as<int32_t>(), (int64_t)nactive, 2 * P,
                                      true, fused_memb, false, &acc_total);
            c->phi_in_updates = false;
            TRY(rc);
        } else {
            std::vector<std::vector<int32_t>> lists;
            std::vector<uint64_t> p2;
            TRY(plan_chunks(c, budget, lists, p2));
            for (size_t i = 0; i < lists.size(); i++) {
                CK(cudaMemcpyAsync(c->active.p, lists[i].data(), sizeof(int32_t) * lists[i].size(),
                                   cudaMemcpyHostToDevice, c->st));
                TRY(join_chunk(c, mode, W, c->active.as<int32_t>(), (int64_t)lists[i].size(), p2[i],
                               false, fused_memb, false, &acc_total));
                CK(cudaStreamSynchronize(c->st));
            }
        }
    }
    c->stats.accepted += acc_total;
    TRY(resolve_timers(c));
    if (pairs) *pairs = (int64_t)P;
    if (accepted) *accepted = acc_total;
    return KNNM_OK;
}

int knnm_round(knnm_ctx *c, int32_t mode, int32_t rev_cap, uint64_t round_seed, int64_t *pairs,
               int64_t *accepted) {
    return round_impl(c, mode, rev_cap, round_seed, pairs, accepted, false);
}

int knnm_set_shard(knnm_ctx *c, int64_t lo, int64_t hi) {
    if (!c) return fail(KNNM_ERR_ARG, "null ctx");
    if (!c->begun) return fail(KNNM_ERR_STATE, "knnm_begin first");
    if (lo < 0 || hi < lo || hi > c->n) return fail(KNNM_ERR_ARG, "bad shard [%lld, %lld)", (long long)lo, (long long)hi);
    c->shard_lo = lo;
    c->shard_hi = hi;
    return KNNM_OK;
}

int knnm_round_local(knnm_ctx *c, int32_t mode, int32_t rev_cap, uint64_t round_seed,
                     int64_t *pairs_local) {
    if (!c) return fail(KNNM_ERR_ARG, "null ctx");
    if (!c->begun) return fail(KNNM_ERR_STATE, "knnm_begin first");
    if (c->capture) return fail(KNNM_ERR_STATE, "on_pair capture is not supported in sharded rounds");
    // an empty round leaves empty slot views
    CK(cudaSetDevice(c->device));
    CK(cudaMemsetAsync(c->bound.p, 0, sizeof(uint32_t) * (c->n + 1), c->st));
    CK(cudaMemsetAsync(c->boff.p, 0, sizeof(uint64_t) * (c->n + 1), c->st));
    TRY(ensure(c->dirty, (size_t)c->n + 1));
    CK(cudaMemsetAsync(c->dirty.p, 0, (size_t)c->n + 1, c->st));
    return round_impl(c, mode, rev_cap, round_seed, pairs_local, nullptr, true);
}

int knnm_local_chunks(knnm_ctx *c, int32_t *nchunks) {
    if (!c || !nchunks) return fail(KNNM_ERR_ARG, "null argument");
    if (!c->begun) return fail(KNNM_ERR_STATE, "knnm_begin first");
    *nchunks = (int32_t)c->lc_pairs2.size();
    return KNNM_OK;
}

int knnm_local_join(knnm_ctx *c, int32_t chunk) {
    if (!c) return fail(KNNM_ERR_ARG, "null ctx");
    if (!c->begun) return fail(KNNM_ERR_STATE, "knnm_begin first");
    if (chunk < 0) return fail(KNNM_ERR_ARG, "chunk %d", chunk);
    CK(cudaSetDevice(c->device));
    const int64_t n = c->n;
    if ((size_t)chunk >= c->lc_pairs2.size()) {
        // this rank has fewer chunks than the busiest one: empty slot views
        CK(cudaMemsetAsync(c->bound.p, 0, sizeof(uint32_t) * (n + 1), c->st));
        CK(cudaMemsetAsync(c->boff.p, 0, sizeof(uint64_t) * (n + 1), c->st));
        return KNNM_OK;
    }
    int64_t acc = 0;
    if (c->lc_single)
        return join_chunk(c, c->lc_mode, c->lc_W, c->active.as<int32_t>(), c->lc_nact,
                          c->lc_pairs2[0], true, false, true, &acc);
    const std::vector<int32_t> &lst = c->lc_lists[chunk];
    CK(cudaMemcpyAsync(c->active.p, lst.data(), sizeof(int32_t) * lst.size(), cudaMemcpyHostToDevice,
                       c->st));
    return join_chunk(c, c->lc_mode, c->lc_W, c->active.as<int32_t>(), (int64_t)lst.size(),
                      c->lc_pairs2[chunk], false, false, true, &acc);
}

int knnm_wait_stream(knnm_ctx *c, void *stream) {
    if (!c) return fail(KNNM_ERR_ARG, "null ctx");
    CK(cudaSetDevice(c->device));
    if (!c->ev_wait) CK(cudaEventCreateWithFlags(&c->ev_wait, cudaEventDisableTiming));
    CK(cudaEventRecord(c->ev_wait, (cudaStream_t)stream));
    CK(cudaStreamWaitEvent(c->st, c->ev_wait, 0));
    return KNNM_OK;
}

int knnm_signal_stream(knnm_ctx *c, void *stream) {
    if (!c) return fail(KNNM_ERR_ARG, "null ctx");
    CK(cudaSetDevice(c->device));
    if (!c->ev_sig) CK(cudaEventCreateWithFlags(&c->ev_sig, cudaEventDisableTiming));
    CK(cudaEventRecord(c->ev_sig, c->st));
    CK(cudaStreamWaitEvent((cudaStream_t)stream, c->ev_sig, 0));
    return KNNM_OK;
}

int knnm_set_cand_budget(knnm_ctx *c, int64_t bytes) {
    if (!c) return fail(KNNM_ERR_ARG, "null ctx");
    if (bytes < 0) return fail(KNNM_ERR_ARG, "budget %lld", (long long)bytes);
    // 0 restores the default; a tiny budget forces one hood per chunk
    c->cand_budget_bytes = bytes == 0 ? ((size_t)40 << 30) : (size_t)bytes;
    return KNNM_OK;
}

int knnm_local_views(knnm_ctx *c, void **cnt, void **boff, void **Bd, void **Bs) {
    if (!c) return fail(KNNM_ERR_ARG, "null ctx");
    if (!c->begun) return fail(KNNM_ERR_STATE, "knnm_begin first");
    TRY(ensure_slots_noinit(c, 1));
    if (cnt) *cnt = c->bound.p;
    if (boff) *boff = c->boff.p;
    if (Bd) *Bd = c->Bd.p;
    // packed slots carry the source row in Bd: nothing to exchange in Bs
    if (Bs) *Bs = c->slots_mode == SLOTS_PACKED ? nullptr : c->Bs.p;
    return KNNM_OK;
}

int knnm_local_compact(knnm_ctx *c, void **cnt, void **boff, void **Bd, void **Bs, int64_t *total) {
    if (!c) return fail(KNNM_ERR_ARG, "null ctx");
    if (!c->begun) return fail(KNNM_ERR_STATE, "knnm_begin first");
    CK(cudaSetDevice(c->device));
    TRY(ensure_slots_noinit(c, 1));
    const int64_t n = c->n;
    const bool packed = c->slots_mode == SLOTS_PACKED;
    TRY(ensure(c->wcnt, sizeof(uint32_t) * (size_t)(n + 1)));
    TRY(ensure(c->woff, sizeof(uint64_t) * (size_t)(n + 1)));
    const int blocks = grid_for(c, n * 32, 256, 16);
    k_slot_wcount<<<blocks, 256, 0, c->st>>>(n, c->boff.as<uint64_t>(), c->Bd.as<double>(),
                                             c->wcnt.as<uint32_t>());
    CKL();
    TRY(scan<uint32_t, uint64_t>(c, c->wcnt.as<uint32_t>(), c->woff.as<uint64_t>(), n));
    uint64_t tot = 0;
    CK(cudaMemcpyAsync(&c->hcnt[C_NUM - 1], c->woff.as<uint64_t>() + n, sizeof(uint64_t),
                       cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    tot = c->hcnt[C_NUM - 1];
    TRY(ensure(c->cBd, sizeof(double) * (size_t)(tot + 1)));
    if (!packed) TRY(ensure(c->cBs, sizeof(int32_t) * (size_t)(tot + 1)));
    k_slot_compact<<<blocks, 256, 0, c->st>>>(n, c->boff.as<uint64_t>(), c->woff.as<uint64_t>(),
                                              c->Bd.as<double>(), packed ? nullptr : c->Bs.as<int32_t>(),
                                              c->cBd.as<double>(), packed ? nullptr : c->cBs.as<int32_t>());
    CKL();
    CK(cudaStreamSynchronize(c->st));
    if (cnt) *cnt = c->wcnt.p;
    if (boff) *boff = c->woff.p;
    if (Bd) *Bd = c->cBd.p;
    if (Bs) *Bs = packed ? nullptr : c->cBs.p;
    if (total) *total = (int64_t)tot;
    return KNNM_OK;
}

int knnm_round_apply(knnm_ctx *c, int32_t nsrc, const uint32_t *recv_cnt, const uint64_t *recv_base,
                     const double *recv_Bd, const int32_t *recv_Bs, int64_t *accepted) {
    if (c) c->state_gen++;  // the lists may change: cached phi is stale
    phi_wait(c);
    if (!c || nsrc < 1 || !recv_cnt || !recv_base) return fail(KNNM_ERR_ARG, "bad argument");
    if (!c->begun) return fail(KNNM_ERR_STATE, "knnm_begin first");
    CK(cudaSetDevice(c->device));
    const int64_t lo = c->shard_lo, hi = c->shard_hi < 0 ? c->n : c->shard_hi, no = hi - lo;
    unsigned long long *cnt = c->counters.as<unsigned long long>();
    CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * C_NUM, c->st));
    if (accepted) *accepted = 0;
    if (no == 0) return KNNM_OK;
    PhaseTimer pt(c, PH_UPDATE);
    TRY(ensure(c->stage[2], sizeof(uint64_t) * (size_t)nsrc * (no + 1)));
    uint64_t *off = c->stage[2].as<uint64_t>();
    for (int s = 0; s < nsrc; s++) {
        TRY(scan<uint32_t, uint64_t>(c, recv_cnt + (size_t)s * no, off + (size_t)s * (no + 1), no));
        if (recv_base[s]) {
            k_add_base<<<grid_for(c, no + 1, 256), 256, 0, c->st>>>(off + (size_t)s * (no + 1), no + 1,
                                                                   recv_base[s]);
            CKL();
        }
    }
    const int E = (c->k + 31) / 32;
    const int blocks = grid_for(c, no * 32, APPLY_WARPS * 32, 16);
#define KNNM_APM_LAUNCH(EE, LZ)                                                                 \
    k_apply_stream_multi<EE, LZ><<<blocks, APPLY_WARPS * 32, 0, c->st>>>(                      \
        lo, no, c->k, nsrc, off, recv_cnt, recv_Bd, recv_Bs, c->ids.as<int32_t>(),             \
        c->dists.as<double>(), c->flags.as<uint8_t>(), c->sizes.as<int32_t>(), cnt, lazy_of(c), \
        c->dirty.as<uint8_t>())
    if (E == 1) {
        if (c->slots_mode == SLOTS_LAZY) KNNM_APM_LAUNCH(1, SLOTS_LAZY);
        else if (c->slots_mode == SLOTS_PACKED) KNNM_APM_LAUNCH(1, SLOTS_PACKED);
        else KNNM_APM_LAUNCH(1, SLOTS_PLAIN);
    } else {
        if (c->slots_mode == SLOTS_LAZY) KNNM_APM_LAUNCH(2, SLOTS_LAZY);
        else if (c->slots_mode == SLOTS_PACKED) KNNM_APM_LAUNCH(2, SLOTS_PACKED);
        else KNNM_APM_LAUNCH(2, SLOTS_PLAIN);
    }
#undef KNNM_APM_LAUNCH
    CKL();
    TRY(sync_counters(c));
    c->stats.accepted += (int64_t)c->hcnt[C_ACCEPTED];
    c->stats.exact_evals += (int64_t)c->hcnt[C_EXACT];
    if (accepted) *accepted = (int64_t)c->hcnt[C_ACCEPTED];
    return KNNM_OK;
}

int knnm_pack_rows(knnm_ctx *c, int32_t all, void **buf, int64_t *count, int32_t *rec_bytes) {
    if (!c || !buf || !count) return fail(KNNM_ERR_ARG, "null argument");
    if (!c->begun) return fail(KNNM_ERR_STATE, "knnm_begin first");
    CK(cudaSetDevice(c->device));
    const int64_t lo = c->shard_lo, hi = c->shard_hi < 0 ? c->n : c->shard_hi, no = hi - lo;
    const int rb = row_rec_bytes(c->k);
    if (rec_bytes) *rec_bytes = rb;
    TRY(ensure(c->dirty, (size_t)c->n + 1));
    TRY(ensure(c->live, (size_t)c->n + 1));
    TRY(ensure(c->rsel, sizeof(uint32_t) * (size_t)(no + 1)));
    TRY(ensure(c->rsoff, sizeof(uint64_t) * (size_t)(no + 1)));
    uint64_t cntr = 0;
    if (no > 0) {
        k_row_select<<<grid_for(c, no, 256), 256, 0, c->st>>>(lo, no, all, c->live.as<uint8_t>(),
                                                              c->dirty.as<uint8_t>(), c->rsel.as<uint32_t>());
        CKL();
        TRY(scan<uint32_t, uint64_t>(c, c->rsel.as<uint32_t>(), c->rsoff.as<uint64_t>(), no));
        CK(cudaMemcpyAsync(&c->hcnt[C_NUM - 1], c->rsoff.as<uint64_t>() + no, sizeof(uint64_t),
                           cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        cntr = c->hcnt[C_NUM - 1];
    }
    TRY(ensure(c->rpack, (size_t)rb * (size_t)(cntr + 1)));
    if (cntr > 0) {
        k_pack_rows<<<grid_for(c, no * 32, 256, 16), 256, 0, c->st>>>(
            lo, no, c->k, c->rsel.as<uint32_t>(), c->rsoff.as<uint64_t>(), c->ids.as<int32_t>(),
            c->dists.as<double>(), c->flags.as<uint8_t>(), c->sizes.as<int32_t>(),
            c->rpack.as<uint8_t>());
        CKL();
    }
    *buf = c->rpack.p;
    *count = (int64_t)cntr;
    return KNNM_OK;
}

int knnm_unpack_rows(knnm_ctx *c, const void *buf, int64_t count) {
    if (c) c->state_gen++;  // the lists change: cached phi is stale
    phi_wait(c);
    if (!c || (count > 0 && !buf) || count < 0) return fail(KNNM_ERR_ARG, "bad argument");
    if (!c->begun) return fail(KNNM_ERR_STATE, "knnm_begin first");
    if (count == 0) return KNNM_OK;
    CK(cudaSetDevice(c->device));
    k_unpack_rows<<<grid_for(c, count * 32, 256, 16), 256, 0, c->st>>>(
        count, c->k, (const uint8_t *)buf, c->ids.as<int32_t>(), c->dists.as<double>(),
        c->flags.as<uint8_t>(), c->sizes.as<int32_t>());
    CKL();
    return KNNM_OK;
}

int knnm_state_views(knnm_ctx *c, void **ids, void **dists, void **flags, void **sizes) {
    if (c) c->state_gen++;  // the lists may change: cached phi is stale
    phi_wait(c);
    if (!c) return fail(KNNM_ERR_ARG, "null ctx");
    if (!c->begun) return fail(KNNM_ERR_STATE, "knnm_begin first");
    if (ids) *ids = c->ids.p;
    if (dists) *dists = c->dists.p;
    if (flags) *flags = c->flags.p;
    if (sizes) *sizes = c->sizes.p;
    return KNNM_OK;
}

// TMA descriptor of a row-major u8 matrix (rows x rb bytes), boxes of
// TB_KB bytes x box_rows rows, 128-byte swizzle (the UMMA operand layout).
static int tb_tensor_map(CUtensorMap *map, const void *ptr, int64_t rows, int rb, int box_rows) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess) return fail(KNNM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t gdim[2] = {(cuuint64_t)rb, (cuuint64_t)rows};
    const cuuint64_t gstride[1] = {(cuuint64_t)rb};
    const cuuint32_t box[2] = {(cuuint32_t)TB_KB, (cuuint32_t)box_rows};
    const cuuint32_t estride[2] = {1, 1};
    const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(ptr), gdim, gstride, box,
                              estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(KNNM_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return KNNM_OK;
}

// Brute force on the tensor cores (knnm_bf.cuh): certified u8 data, L2.
// X = the candidate rows (union rows, or the whole dataset for vector
// queries), Q = the query rows as a dense u8 matrix with their norms.
static int bf_tc(knnm_ctx *c, const uint8_t *X, const int32_t *xnorm, int64_t nx, int rb, const uint8_t *Q,
                 const int32_t *qnorm, const int64_t *qself, int64_t nq, int k, int32_t *oi, double *od) {
    const int nkb = (rb + TB_KB - 1) / TB_KB;
    const size_t smem = tb_smem_bytes(nkb, k);
    CUtensorMap mq, mx;
    TRY(tb_tensor_map(&mq, Q, nq, rb, TB_M));
    TRY(tb_tensor_map(&mx, X, nx, rb, TB_N));
    static size_t smem_set = 0;
    if (smem > smem_set) {
        CK(cudaFuncSetAttribute(k_bf_tc_u8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        smem_set = smem;
    }
    const int64_t nqb = (nq + TB_M - 1) / TB_M, ntiles = (nx + TB_N - 1) / TB_N;
    // data slices so that small query sets still fill the SMs
    int S = (int)std::min<int64_t>({(int64_t)16, std::max<int64_t>(1, (c->sms + nqb - 1) / nqb), ntiles});
    const int64_t tps = (ntiles + S - 1) / S;
    S = (int)((ntiles + tps - 1) / tps);
    TRY(ensure(c->bfpart, sizeof(uint64_t) * (size_t)S * nq * k));
    k_bf_tc_u8<<<dim3((unsigned)nqb, (unsigned)S), TB_THREADS, smem, c->st>>>(
        mq, mx, nq, nx, nkb, qnorm, xnorm, qself, k, tps, c->bfpart.as<uint64_t>());
    CKL();
    k_bf_tc_finish<<<grid_for(c, nq, 128), 128, 0, c->st>>>(c->bfpart.as<uint64_t>(), nq, k, S, oi, od);
    CKL();
    c->stats.bf_tc_launches += 1;
    return KNNM_OK;
}

int knnm_bf_topk(knnm_ctx *c, const float *queries, const int64_t *rows, int64_t nq, int32_t k,
                 int32_t exclude_self, int32_t *out_ids, double *out_dists) {
    if (!c || (!queries && !rows) || !out_ids || !out_dists) return fail(KNNM_ERR_ARG, "null argument");
    if (!c->have_data) return fail(KNNM_ERR_STATE, "knnm_set_dataset first");
    if (k < 1 || k > BF_MAXK) return fail(KNNM_ERR_LIMIT, "brute-force k=%d outside [1, %d]", k, BF_MAXK);
    if (nq == 0) return KNNM_OK;
    CK(cudaSetDevice(c->device));
    PhaseTimer pt(c, PH_OTHER);
    // row queries: candidates are the rows of the current union (local ids);
    // vector queries: candidates are the whole dataset
    if (rows && !c->begun) return fail(KNNM_ERR_STATE, "row queries need knnm_begin");
    const float *data = rows ? c->subp : c->vec.as<float>();
    const int64_t n = rows ? c->n : c->n_all;
    const float *qd = nullptr;
    const int64_t *rd = nullptr;
    if (rows) {
        TRY(ensure(c->stage[0], sizeof(int64_t) * nq));
        TRY(h2d(c, c->stage[0].p, rows, sizeof(int64_t) * nq));
        rd = c->stage[0].as<int64_t>();
    } else {
        TRY(ensure(c->stage[0], sizeof(float) * (size_t)nq * c->dp));
        if (c->dp == c->d) {
            TRY(h2d(c, c->stage[0].p, queries, sizeof(float) * (size_t)nq * c->d));
        } else {
            TRY(ensure(c->stage[1], sizeof(float) * (size_t)nq * c->d));
            TRY(h2d(c, c->stage[1].p, queries, sizeof(float) * (size_t)nq * c->d));
            k_pad_rows<<<grid_for(c, nq * c->dp, 256), 256, 0, c->st>>>(c->stage[1].as<float>(), c->d, c->dp,
                                                                    nq, c->stage[0].as<float>());
            CKL();
        }
        qd = c->stage[0].as<float>();
    }
    TRY(ensure(c->stage[2], (sizeof(int32_t) + sizeof(double)) * (size_t)nq * k + 8));
    int32_t *oi = c->stage[2].as<int32_t>();
    double *od = reinterpret_cast<double *>(c->stage[2].as<char>() + ((sizeof(int32_t) * (size_t)nq * k + 7) & ~(size_t)7));
    // tensor-core route: exact integer Gram tiles (u8 rows, L2)
    const int rb = (c->d + 31) & ~31;
    bool tc = c->bf_u8 && c->metric == KNNM_L2 && k <= TB_MAX_K && c->bf_variant != 0 &&
              tb_smem_bytes((rb + TB_KB - 1) / TB_KB, k) <= 227 * 1024 && n >= 1;
    if (tc && !rows) {
        // vector queries must themselves be integers in [0, 255]
        unsigned long long *cnt = c->counters.as<unsigned long long>();
        unsigned long long init[3] = {0ull, 0ull, 0xffffffffull};
        CK(cudaMemcpyAsync(cnt + C_NUM - 3, init, sizeof(init), cudaMemcpyHostToDevice, c->st));
        k_data_stats<<<grid_for(c, nq * c->dp, 256), 256, 0, c->st>>>(qd, nq * c->dp, cnt + C_NUM - 3);
        CKL();
        TRY(sync_counters(c));
        const uint32_t mxk = (uint32_t)c->hcnt[C_NUM - 2], mnk = (uint32_t)c->hcnt[C_NUM - 1];
        // ordered keys of 0.0f and 255.0f (see k_data_stats)
        tc = c->hcnt[C_NUM - 3] == 0 && mnk >= 0x80000000u && mxk <= (0x437f0000u | 0x80000000u);
        CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * C_NUM, c->st));
    }
    if (c->bf_variant == 1 && !tc) return fail(KNNM_ERR_LIMIT, "tensor-core brute force needs u8 L2 data, k <= %d", TB_MAX_K);
    c->bf_last_route = tc ? 1 : 0;
    if (tc) {
        const uint8_t *X;
        const int32_t *xn;
        if (c->cert_u8) {  // the join's u8 copy (same row length)
            X = rows ? c->sub16p : c->vec16.as<uint8_t>();
            xn = reinterpret_cast<const int32_t *>(rows ? c->subnormp : c->norms.as<float>());
        } else {
            TRY(ensure(c->bfx, (size_t)n * rb));
            TRY(ensure(c->bfxn, sizeof(int32_t) * (size_t)n));
            k_to_u8<<<grid_for(c, n * 32, 256, 16), 256, 0, c->st>>>(data, c->dp, n, rb, c->bfx.as<uint8_t>(),
                                                                    reinterpret_cast<float *>(c->bfxn.p));
            CKL();
            X = c->bfx.as<uint8_t>();
            xn = c->bfxn.as<int32_t>();
        }
        TRY(ensure(c->bfq, (size_t)nq * rb));
        TRY(ensure(c->bfqn, sizeof(int32_t) * (size_t)nq));
        if (rows) {
            k_bf_gather_u8<<<grid_for(c, nq * (rb / 16), 256), 256, 0, c->st>>>(
                X, rb, xn, rd, nq, c->bfq.as<uint8_t>(), c->bfqn.as<int32_t>());
        } else {
            k_to_u8<<<grid_for(c, nq * 32, 256, 16), 256, 0, c->st>>>(qd, c->dp, nq, rb, c->bfq.as<uint8_t>(),
                                                                     reinterpret_cast<float *>(c->bfqn.p));
        }
        CKL();
        TRY(bf_tc(c, X, xn, n, rb, c->bfq.as<uint8_t>(), c->bfqn.as<int32_t>(), (rows && exclude_self) ? rd : nullptr,
                  nq, k, oi, od));
    } else {
        const size_t smem = (size_t)BF_THREADS * k * (sizeof(double) + sizeof(int32_t));
        const unsigned grid = (unsigned)std::min<int64_t>(nq, (int64_t)c->sms * 8);
#define KNNM_BF_ARGS data, n, c->dp, c->d, qd, c->dp, rd, nq, k, exclude_self, oi, od
        if (c->metric == 1) k_bf_topk<1><<<grid, BF_THREADS, smem, c->st>>>(KNNM_BF_ARGS);
        else if (c->metric == 2) k_bf_topk<2><<<grid, BF_THREADS, smem, c->st>>>(KNNM_BF_ARGS);
        else k_bf_topk<0><<<grid, BF_THREADS, smem, c->st>>>(KNNM_BF_ARGS);
#undef KNNM_BF_ARGS
        CKL();
    }
    TRY(d2h(c, out_ids, oi, sizeof(int32_t) * (size_t)nq * k));
    TRY(d2h(c, out_dists, od, sizeof(double) * (size_t)nq * k));
    CK(cudaStreamSynchronize(c->st));
    return KNNM_OK;
}

int knnm_pair_dists(knnm_ctx *c, const int32_t *pa, const int32_t *pb, int64_t m, double *out) {
    if (!c || ((!pa || !pb || !out) && m > 0)) return fail(KNNM_ERR_ARG, "null argument");
    if (!c->begun) return fail(KNNM_ERR_STATE, "knnm_begin first");
    if (m == 0) return KNNM_OK;
    CK(cudaSetDevice(c->device));
    PhaseTimer pt(c, PH_OTHER);
    TRY(ensure(c->stage[0], sizeof(int32_t) * (size_t)m));
    TRY(ensure(c->stage[1], sizeof(int32_t) * (size_t)m));
    TRY(ensure(c->stage[2], sizeof(double) * (size_t)m));
    TRY(h2d(c, c->stage[0].p, pa, sizeof(int32_t) * (size_t)m));
    TRY(h2d(c, c->stage[1].p, pb, sizeof(int32_t) * (size_t)m));
    k_pair_dists<<<grid_for(c, m, 256), 256, 0, c->st>>>(c->stage[0].as<int32_t>(), c->stage[1].as<int32_t>(), m,
                                                         c->subp, c->dp, c->d, c->metric, c->stage[2].as<double>());
    CKL();
    TRY(d2h(c, out, c->stage[2].p, sizeof(double) * (size_t)m));
    CK(cudaStreamSynchronize(c->st));
    return KNNM_OK;
}

int knnm_set_bf_variant(knnm_ctx *c, int32_t variant) {
    if (!c) return fail(KNNM_ERR_ARG, "null ctx");
    if (variant < -1 || variant > 1) return fail(KNNM_ERR_ARG, "bf variant %d", variant);
    c->bf_variant = variant;
    return KNNM_OK;
}

int knnm_bf_route(knnm_ctx *c, int32_t *route) {
    if (!c || !route) return fail(KNNM_ERR_ARG, "null argument");
    *route = c->bf_last_route;
    return KNNM_OK;
}

// Merge path: number of a-elements among the first p outputs of the merge
// of two strictly ascending, disjoint arrays.
static int64_t merge_split(const int64_t *a, int64_t na, const int64_t *b, int64_t nb, int64_t p) {
    int64_t lo = std::max<int64_t>(0, p - nb), hi = std::min<int64_t>(p, na);
    while (lo < hi) {
        const int64_t i = (lo + hi) >> 1, j = p - i;
        if (i < na && j > 0 && b[j - 1] > a[i]) lo = i + 1;  // b[j-1] must come after a[i]
        else hi = i;
    }
    return lo;
}

// Branch-free two-pointer merge of a[i..ia1) and b[j..jb1) into uni[o..):
// both rows are written every step and only the side(s) holding the smaller
// id advance, so each row's last write is its own (a shared id yields one
// union entry that both rows point at).  Returns whether an id was shared.
static int32_t merge_run(const int64_t *a, int64_t i, int64_t ia1, const int64_t *b, int64_t j,
                         int64_t jb1, int64_t o, int64_t *uni, int32_t *rows_a, int32_t *rows_b,
                         int8_t *labels, int64_t *o_end) {
    int32_t sh = 0;
    while (i < ia1 && j < jb1) {
        const int64_t x = a[i], y = b[j];
        const int ta = x <= y, tb = y <= x;
        uni[o] = ta ? x : y;
        if (labels) labels[o] = (int8_t)(ta ? 0 : 1);
        rows_a[i] = (int32_t)o;
        rows_b[j] = (int32_t)o;
        sh |= ta & tb;
        i += ta;
        j += tb;
        o++;
    }
    for (; i < ia1; i++) {
        uni[o] = a[i];
        if (labels) labels[o] = 0;
        rows_a[i] = (int32_t)o++;
    }
    for (; j < jb1; j++) {
        uni[o] = b[j];
        if (labels) labels[o] = 1;
        rows_b[j] = (int32_t)o++;
    }
    if (o_end) *o_end = o;
    return sh;
}

int knnm_merge_members(const int64_t *a, int64_t na, const int64_t *b, int64_t nb, int64_t *uni,
                       int32_t *rows_a, int32_t *rows_b, int64_t *nu, int32_t *shared, int8_t *labels) {
    if ((na > 0 && (!a || !rows_a)) || (nb > 0 && (!b || !rows_b)) || !uni || !nu)
        return fail(KNNM_ERR_ARG, "bad argument");
    if (na + nb >= (1ll << 31)) return fail(KNNM_ERR_LIMIT, "union too large");
    const int64_t total = na + nb;
    const int T = total < (1 << 16) ? 1
                : (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    // ascending checks and the merge, split over T host threads (merge path)
    std::vector<int32_t> bad(T, 0), sh(T, 0);
    auto work = [&](int t) {
        const int64_t p0 = total * t / T, p1 = total * (t + 1) / T;
        const int64_t ca0 = na * t / T, ca1 = na * (t + 1) / T, cb0 = nb * t / T, cb1 = nb * (t + 1) / T;
        for (int64_t i = std::max<int64_t>(ca0, 1); i < ca1; i++) bad[t] |= a[i] <= a[i - 1];
        for (int64_t i = std::max<int64_t>(cb0, 1); i < cb1; i++) bad[t] |= b[i] <= b[i - 1];
        if (T == 1) return;
        const int64_t i0 = merge_split(a, na, b, nb, p0), i1 = merge_split(a, na, b, nb, p1);
        sh[t] = merge_run(a, i0, i1, b, p0 - i0, p1 - i1, p0, uni, rows_a, rows_b, labels, nullptr);
    };
    if (T == 1) {
        work(0);
    } else {
        std::vector<std::thread> th;
        for (int t = 1; t < T; t++) th.emplace_back(work, t);
        work(0);
        for (auto &x : th) x.join();
    }
    for (int t = 0; t < T; t++)
        if (bad[t]) return fail(KNNM_ERR_ARG, "ids must be strictly ascending");
    int32_t s = 0;
    for (int t = 0; t < T; t++) s |= sh[t];
    int64_t o = total;
    if (T == 1 || s) {
        // serial merge (also the exact tie semantics when ids are shared:
        // the parallel split assumes disjoint inputs)
        s = merge_run(a, 0, na, b, 0, nb, 0, uni, rows_a, rows_b, labels, &o);
    }
    *nu = o;
    if (shared) *shared = s;
    return KNNM_OK;
}

// Content fingerprint of a host buffer (the dataset cache key): the 64-bit
// words w_i folded as sum(w_i * (2i + 1)) mod 2^64 per thread slice, the
// slices combined with a mix.  Any single-word change alters the sum (odd
// multipliers are invertible mod 2^64).  Host threads, memory-bound.
int knnm_fingerprint(const void *p, int64_t bytes, uint64_t *out) {
    if ((!p && bytes > 0) || bytes < 0 || !out) return fail(KNNM_ERR_ARG, "bad argument");
    const uint64_t *w = (const uint64_t *)p;
    const int64_t nw = bytes / 8;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int64_t nt = std::min<int64_t>(std::min(16u, hw), std::max<int64_t>(1, nw >> 18));
    std::vector<uint64_t> part((size_t)nt, 0);
    auto body = [&](int64_t t) {
        const int64_t a = nw * t / nt, b = nw * (t + 1) / nt;
        uint64_t h0 = 0, h1 = 0;
        int64_t i = a;
        for (; i + 1 < b; i += 2) {
            h0 += w[i] * (2 * (uint64_t)i + 1);
            h1 += w[i + 1] * (2 * (uint64_t)i + 3);
        }
        if (i < b) h0 += w[i] * (2 * (uint64_t)i + 1);
        part[(size_t)t] = h0 + h1;
    };
    std::vector<std::thread> th;
    for (int64_t t = 1; t < nt; t++) th.emplace_back(body, t);
    body(0);
    for (auto &x : th) x.join();
    uint64_t h = 0x9e3779b97f4a7c15ull ^ (uint64_t)bytes;
    for (uint64_t v : part) h += v;
    uint64_t tail = 0;
    memcpy(&tail, (const char *)p + nw * 8, (size_t)(bytes - nw * 8));
    h += tail * 0xff51afd7ed558ccdull;
    h ^= h >> 33;
    h *= 0xc4ceb9fe1a85ec53ull;
    h ^= h >> 33;
    *out = h;
    return KNNM_OK;
}

int knnm_sample_distinct_rows(uint64_t *pcg, int32_t *has_uint32, uint32_t *uinteger, int64_t n,
                              int32_t k, const int32_t *exclude, int64_t nrows, int64_t *out) {
    if (!pcg || !has_uint32 || !uinteger || !out || (nrows > 0 && !exclude) || k < 0)
        return fail(KNNM_ERR_ARG, "bad argument");
    HostPcg p;
    p.s = ((unsigned __int128)pcg[0] << 64) | pcg[1];
    p.inc = ((unsigned __int128)pcg[2] << 64) | pcg[3];
    p.has = *has_uint32;
    p.u = *uinteger;
    for (int64_t r = 0; r < nrows; r++) {
        const int64_t ex = exclude[r];
        const int64_t pool = (ex >= 0 && ex < n) ? n - 1 : n;  // core.py:222-230
        if (k > pool) return fail(KNNM_ERR_ARG, "not enough values to sample from");
        if (pool > 0xFFFFFFFFll) return fail(KNNM_ERR_LIMIT, "population too large");
    }
    HostPcg p0 = p;
    if (nrows >= 4096 && sample_rows_parallel(p, n, k, exclude, nrows, out)) {
        pcg[0] = (uint64_t)(p.s >> 64);
        pcg[1] = (uint64_t)p.s;
        *has_uint32 = p.has;
        *uinteger = p.u;
        return KNNM_OK;
    }
    p = p0;
    std::vector<uint64_t> hs;
    std::vector<int64_t> tmp;
    for (int64_t r = 0; r < nrows; r++) {
        const int64_t ex = exclude[r];
        const int64_t pool = (ex >= 0 && ex < n) ? n - 1 : n;  // core.py:222-230
        if (k > pool) return fail(KNNM_ERR_ARG, "not enough values to sample from");
        if (pool > 0xFFFFFFFFll) return fail(KNNM_ERR_LIMIT, "population too large");
        int64_t *o = out + r * k;
        host_choice(p, pool, k, o, hs, tmp);
        if (ex >= 0 && ex < n)
            for (int t = 0; t < k; t++) o[t] += o[t] >= ex ? 1 : 0;
    }
    pcg[0] = (uint64_t)(p.s >> 64);
    pcg[1] = (uint64_t)p.s;
    *has_uint32 = p.has;
    *uinteger = p.u;
    return KNNM_OK;
}

// Launch the phi reduction (numpy's pairwise tree over the present
// distances); *res = device address of the result.
static int phi_kernels(knnm_ctx *c, const double **res, cudaStream_t stream) {
    int64_t N = c->n * c->k;
    if (c->phi.N != N) {
        build_phi_tree(c->phi, N);
        size_t nl = c->phi.leaf_lo.size(), ni = c->phi.left.size();
        TRY(ensure(c->phi_leaf_lo, sizeof(int64_t) * nl));
        TRY(ensure(c->phi_leaf_len, sizeof(int32_t) * nl));
        TRY(ensure(c->phi_leaves, sizeof(double) * nl));
        TRY(ensure(c->phi_left, sizeof(int32_t) * (ni + 1)));
        TRY(ensure(c->phi_right, sizeof(int32_t) * (ni + 1)));
        TRY(ensure(c->phi_inner, sizeof(double) * (ni + 1)));
        TRY(ensure(c->phi_level, sizeof(int32_t) * c->phi.level_start.size()));
        CK(cudaMemcpy(c->phi_leaf_lo.p, c->phi.leaf_lo.data(), sizeof(int64_t) * nl, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c->phi_leaf_len.p, c->phi.leaf_len.data(), sizeof(int32_t) * nl, cudaMemcpyHostToDevice));
        if (ni) {
            CK(cudaMemcpy(c->phi_left.p, c->phi.left.data(), sizeof(int32_t) * ni, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(c->phi_right.p, c->phi.right.data(), sizeof(int32_t) * ni, cudaMemcpyHostToDevice));
        }
        CK(cudaMemcpy(c->phi_level.p, c->phi.level_start.data(),
                      sizeof(int32_t) * c->phi.level_start.size(), cudaMemcpyHostToDevice));
    }
    int64_t nl = (int64_t)c->phi.leaf_lo.size();
    int64_t ni = (int64_t)c->phi.left.size();
    k_phi_leaves<<<(unsigned)((nl + 127) / 128), 128, 0, stream>>>(
        c->dists.as<double>(), c->sizes.as<int32_t>(), c->k, c->phi_leaf_lo.as<int64_t>(),
        c->phi_leaf_len.as<int32_t>(), nl, c->phi_leaves.as<double>());
    CKL();
    if (ni > 0) {
        // wide levels: one grid each; the narrow top of the tree in one block
        const int nlev = (int)c->phi.level_start.size() - 1;
        int h = 0;
        for (; h < nlev; h++) {
            const int lo = c->phi.level_start[h], hi = c->phi.level_start[h + 1];
            if (hi - lo < 4096) break;
            k_phi_level<<<(unsigned)((hi - lo + 255) / 256), 256, 0, stream>>>(
                c->phi_left.as<int32_t>(), c->phi_right.as<int32_t>(), lo, hi,
                c->phi_leaves.as<double>(), c->phi_inner.as<double>());
            CKL();
        }
        if (h < nlev) {
            k_phi_tree<<<1, 1024, 0, stream>>>(c->phi_left.as<int32_t>(), c->phi_right.as<int32_t>(),
                                              c->phi_level.as<int32_t>() + h, nlev - h,
                                              c->phi_leaves.as<double>(), c->phi_inner.as<double>());
            CKL();
        }
        *res = c->phi_inner.as<double>() + (ni - 1);
    } else {
        *res = c->phi_leaves.as<double>();
    }
    return KNNM_OK;
}

int knnm_phi_async(knnm_ctx *c, int32_t slot) {
    if (!c || slot < 0 || slot >= KNNM_PHI_SLOTS) return fail(KNNM_ERR_ARG, "bad argument");
    if (!c->begun) return fail(KNNM_ERR_STATE, "knnm_begin first");
    CK(cudaSetDevice(c->device));
    if (!c->st2) {
        CK(cudaStreamCreateWithFlags(&c->st2, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&c->ev_lists, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_phi, cudaEventDisableTiming));
        CK(cudaHostAlloc((void **)&c->hphi, sizeof(double) * KNNM_PHI_SLOTS, cudaHostAllocDefault));
    }
    if (c->n * c->k == 0) {
        CK(cudaStreamSynchronize(c->st2));
        c->hphi[slot] = 0.0;
        return KNNM_OK;
    }
    // the lists as of now on st, reduced on st2
    CK(cudaEventRecord(c->ev_lists, c->st));
    CK(cudaStreamWaitEvent(c->st2, c->ev_lists, 0));
    const double *r = nullptr;
    TRY(phi_kernels(c, &r, c->st2));
    CK(cudaMemcpyAsync(c->hphi + slot, r, sizeof(double), cudaMemcpyDeviceToHost, c->st2));
    CK(cudaEventRecord(c->ev_phi, c->st2));
    c->phi_pending = true;
    return KNNM_OK;
}

int knnm_phi_fetch(knnm_ctx *c, int32_t slot, double *out) {
    if (!c || !out || slot < 0 || slot >= KNNM_PHI_SLOTS) return fail(KNNM_ERR_ARG, "bad argument");
    if (!c->st2) return fail(KNNM_ERR_STATE, "knnm_phi_async first");
    CK(cudaSetDevice(c->device));
    CK(cudaStreamSynchronize(c->st2));
    *out = c->hphi[slot];
    return KNNM_OK;
}

int knnm_phi(knnm_ctx *c, double *out) {
    if (!c || !out) return fail(KNNM_ERR_ARG, "null argument");
    if (!c->begun) return fail(KNNM_ERR_STATE, "knnm_begin first");
    CK(cudaSetDevice(c->device));
    if (c->n * c->k == 0) {
        *out = 0.0;
        return KNNM_OK;
    }
    if (c->phi_gen == c->state_gen) {  // computed by the last round, lists unchanged since
        *out = c->phi_val;
        return KNNM_OK;
    }
    PhaseTimer pt(c, PH_OTHER);
    const double *r = nullptr;
    TRY(phi_kernels(c, &r, c->st));
    CK(cudaMemcpyAsync(&c->phi_val, r, sizeof(double), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    c->phi_gen = c->state_gen;
    *out = c->phi_val;
    return KNNM_OK;
}

static int export_impl(knnm_ctx *c, int32_t merge_rear, int32_t *out_ids, double *out_dists,
                       int32_t *out_sizes, bool on_device) {
    if (c) c->state_gen++;  // the lists may change: cached phi is stale
    phi_wait(c);
    if (!c || !out_ids || !out_dists || !out_sizes) return fail(KNNM_ERR_ARG, "null argument");
    if (!c->begun) return fail(KNNM_ERR_STATE, "knnm_begin first");
    CK(cudaSetDevice(c->device));
    PhaseTimer pt(c, PH_OTHER);
    int64_t n = c->n, nk = c->n * c->k;
    const bool rear = merge_rear && c->have_tail && c->tk > 0;
    // device outputs are written in place by the last kernel (no copies)
    TRY(ensure(c->out_ids, sizeof(int32_t) * nk));
    int32_t *exp_ids = (on_device && !rear) ? out_ids : c->out_ids.as<int32_t>();
    k_export<<<grid_for(c, nk, 256), 256, 0, c->st>>>(c->ids.as<int32_t>(), ugid_of(c), nk, exp_ids);
    CKL();
    const void *src_i = exp_ids, *src_d = c->dists.p, *src_s = c->sizes.p;
    if (rear) {
        TRY(ensure(c->out_d, sizeof(double) * nk));
        TRY(ensure(c->out_s, sizeof(int32_t) * n));
        TRY(ensure(c->stage[0], sizeof(int32_t) * nk));
        int32_t *oi = on_device ? out_ids : c->stage[0].as<int32_t>();
        double *od = on_device ? out_dists : c->out_d.as<double>();
        int32_t *os = on_device ? out_sizes : c->out_s.as<int32_t>();
        const size_t mr_smem = mr_smem_bytes(c->k, c->tk);
        k_merge_rear<<<(unsigned)((n + MR_ROWS - 1) / MR_ROWS), MR_ROWS, mr_smem, c->st>>>(
            c->out_ids.as<int32_t>(), c->dists.as<double>(), c->sizes.as<int32_t>(),
            c->tail_ids.as<int32_t>(), c->tail_d.as<double>(), c->tail_s.as<int32_t>(), n, c->k,
            c->tk, oi, od, os);
        CKL();
        src_i = oi;
        src_d = od;
        src_s = os;
    }
    if (on_device) {
        if (!rear) {
            CK(cudaMemcpyAsync(out_dists, src_d, sizeof(double) * nk, cudaMemcpyDeviceToDevice, c->st));
            CK(cudaMemcpyAsync(out_sizes, src_s, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, c->st));
        }
    } else {
        TRY(d2h(c, out_ids, src_i, sizeof(int32_t) * nk));
        TRY(d2h(c, out_dists, src_d, sizeof(double) * nk));
        TRY(d2h(c, out_sizes, src_s, sizeof(int32_t) * n));
    }
    CK(cudaStreamSynchronize(c->st));
    return KNNM_OK;
}

int knnm_export(knnm_ctx *c, int32_t merge_rear, int32_t *out_ids, double *out_dists,
                int32_t *out_sizes) {
    return export_impl(c, merge_rear, out_ids, out_dists, out_sizes, false);
}

int knnm_export_dev(knnm_ctx *c, int32_t merge_rear, int32_t *out_ids, double *out_dists,
                    int32_t *out_sizes) {
    return export_impl(c, merge_rear, out_ids, out_dists, out_sizes, true);
}

int knnm_get_state(knnm_ctx *c, int32_t *ids, double *dists, uint8_t *flags, int32_t *sizes) {
    if (!c) return fail(KNNM_ERR_ARG, "null ctx");
    if (!c->begun) return fail(KNNM_ERR_STATE, "knnm_begin first");
    CK(cudaSetDevice(c->device));
    size_t nk = (size_t)c->n * c->k;
    if (ids) TRY(d2h(c, ids, c->ids.p, sizeof(int32_t) * nk));
    if (dists) TRY(d2h(c, dists, c->dists.p, sizeof(double) * nk));
    if (flags) TRY(d2h(c, flags, c->flags.p, nk));
    if (sizes) TRY(d2h(c, sizes, c->sizes.p, sizeof(int32_t) * c->n));
    CK(cudaStreamSynchronize(c->st));
    return KNNM_OK;
}

int knnm_set_capture(knnm_ctx *c, int32_t on) {
    if (!c) return fail(KNNM_ERR_ARG, "null ctx");
    c->capture = on != 0;
    c->cap_pa.clear();
    c->cap_pb.clear();
    c->cap_pd.clear();
    return KNNM_OK;
}

int knnm_capture_count(knnm_ctx *c, int64_t *count) {
    if (!c || !count) return fail(KNNM_ERR_ARG, "null argument");
    *count = (int64_t)c->cap_pa.size();
    return KNNM_OK;
}

int knnm_capture_fetch(knnm_ctx *c, int32_t *pa, int32_t *pb, double *pd, int64_t count) {
    if (!c) return fail(KNNM_ERR_ARG, "null ctx");
    if (count != (int64_t)c->cap_pa.size()) return fail(KNNM_ERR_ARG, "count mismatch");
    if (count) {
        memcpy(pa, c->cap_pa.data(), sizeof(int32_t) * count);
        memcpy(pb, c->cap_pb.data(), sizeof(int32_t) * count);
        memcpy(pd, c->cap_pd.data(), sizeof(double) * count);
    }
    c->cap_pa.clear();
    c->cap_pb.clear();
    c->cap_pd.clear();
    return KNNM_OK;
}

int knnm_set_locality(knnm_ctx *c, int32_t iters) {
    if (!c || iters < 0) return fail(KNNM_ERR_ARG, "bad argument");
    c->locality_iters = iters;
    c->have_order = false;
    return KNNM_OK;
}

int knnm_set_u8(knnm_ctx *c, int32_t on) {
    if (!c) return fail(KNNM_ERR_ARG, "null ctx");
    c->u8_enabled = on != 0;
    return KNNM_OK;
}

int knnm_set_sample(knnm_ctx *c, int32_t new_cap) {
    if (!c) return fail(KNNM_ERR_ARG, "null ctx");
    if (new_cap < 0) return fail(KNNM_ERR_ARG, "new_cap must be >= 0");
    c->new_cap = new_cap;
    return KNNM_OK;
}

int knnm_set_join_variant(knnm_ctx *c, int32_t variant) {
    if (!c || variant < -1 || variant > 4) return fail(KNNM_ERR_ARG, "variant %d", variant);
    c->join_variant = variant;
    return KNNM_OK;
}

int knnm_get_info(knnm_ctx *c, int32_t *cert, int32_t *dp) {
    if (!c) return fail(KNNM_ERR_ARG, "null ctx");
    if (cert) *cert = (c->cert ? 1 : 0) | (c->cert_dot ? 2 : 0) | (c->cert_u8 ? 4 : 0);
    if (dp) *dp = c->dp;
    return KNNM_OK;
}

int knnm_set_profiling(knnm_ctx *c, int32_t on) {
    if (!c) return fail(KNNM_ERR_ARG, "null ctx");
    c->profiling = on != 0;
    return KNNM_OK;
}

int knnm_get_stats(knnm_ctx *c, knnm_stats *out) {
    if (!c || !out) return fail(KNNM_ERR_ARG, "null argument");
    TRY(resolve_timers(c));
    *out = c->stats;
    out->join_ms = c->phase_ms[PH_JOIN];
    out->reverse_ms = c->phase_ms[PH_REVERSE];
    out->assemble_ms = c->phase_ms[PH_ASSEMBLE];
    out->update_ms = c->phase_ms[PH_UPDATE];
    out->other_ms = c->phase_ms[PH_OTHER];
    out->join_kernel_ms = c->phase_ms[PH_JOINK];
    out->apply_kernel_ms = c->phase_ms[PH_APPLYK];
    return KNNM_OK;
}

int knnm_reset_stats(knnm_ctx *c) {
    if (!c) return fail(KNNM_ERR_ARG, "null ctx");
    TRY(resolve_timers(c));
    c->stats = knnm_stats{};
    for (double &v : c->phase_ms) v = 0;
    return KNNM_OK;
}

int knnm_mark(knnm_ctx *c, int32_t slot) {
    if (!c || slot < 0 || slot >= 8) return fail(KNNM_ERR_ARG, "bad slot");
    CK(cudaSetDevice(c->device));
    if (!c->marks[slot]) CK(cudaEventCreate(&c->marks[slot]));
    CK(cudaEventRecord(c->marks[slot], c->st));
    return KNNM_OK;
}

int knnm_elapsed(knnm_ctx *c, int32_t a, int32_t b, double *ms) {
    if (!c || !ms || a < 0 || a >= 8 || b < 0 || b >= 8 || !c->marks[a] || !c->marks[b])
        return fail(KNNM_ERR_ARG, "bad slots");
    float f = 0;
    CK(cudaEventSynchronize(c->marks[b]));
    CK(cudaEventElapsedTime(&f, c->marks[a], c->marks[b]));
    *ms = f;
    return KNNM_OK;
}

int knnm_sync(knnm_ctx *c) {
    if (!c) return fail(KNNM_ERR_ARG, "null ctx");
    CK(cudaStreamSynchronize(c->st));
    return KNNM_OK;
}

}  // extern "C"

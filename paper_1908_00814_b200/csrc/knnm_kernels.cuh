// knnm_kernels.cuh -- sm_100a kernels of the S-Merge / J-Merge round engine.
//
// Each kernel cites the reference numba kernel (pkg/src/knnmerge/_kernels.py)
// whose result it reproduces bit-for-bit.  Design notes live in DESIGN.md.
#pragma once
#include <cuda_fp16.h>

#include <type_traits>

#include "knnm_device.cuh"

namespace knnm {

constexpr int WARP_REV_MAX = 256;      // reverse segments a warp sorts itself
constexpr int BLOCK_SORT_MAX = 16384;  // elements a block sorts in shared memory
constexpr int HEAVY_SORT_SMALL = 4096; // ... in the first (small shared memory) heavy pass
constexpr int MAX_W = 128;             // k + rev_cap upper bound
constexpr int SEG_SMEM = 256;          // membership segments ranked in shared memory

// Reference-order slots.  Row r's update bucket has one slot per admissible
// (hood, partner) pair it takes part in, laid out in the reference's
// sequential order: hoods ascending, then partner position ascending (pairs
// (x, p) with x < p, then (p, x) with x > p, _kernels.py:424-436).  Slot
// base of (hood u, member at position p) = boff[r] + start[u * W + p]; the
// partner's rank within the hood comes from per-class position prefix counts.
struct __align__(8) MembRec {  // one (hood, member) membership, bucketed by member row
    uint32_t key;     // hood id u (or directed-insert ordinal)
    uint16_t weight;  // slots the membership occupies (admissible partners)
    uint16_t pos;     // the member's hood position p (0 for directed inserts)
};
// where a record's exclusive rank goes: u * W + p (hoods), or the ordinal
// (directed inserts: wout = 1, pos = 0)
__device__ __forceinline__ uint32_t memb_out(const MembRec &r, uint32_t wout) { return r.key * wout + r.pos; }

// Streaming (read-once) load of a membership record.
__device__ __forceinline__ MembRec ldcs_memb(const MembRec *p) {
    const uint2 v = __ldcs(reinterpret_cast<const uint2 *>(p));
    return MembRec{v.x, (uint16_t)(v.y & 0xFFFFu), (uint16_t)(v.y >> 16)};
}

// Admissible partner classes of a member, by pair mode and member class
// (class = (label != 0) * 2 + !new; _kernels.py:391-399).  bit c set ->
// members of class c are partners; SELF: the member's own class is in the
// mask (it is not its own partner).
__host__ __device__ __forceinline__ int partner_mask(int mode, int cls) {
    if (mode == 0) return cls == 0 ? 0x3 : 0x1;
    if (mode == 1) return cls == 0 ? 0xC : cls == 1 ? 0x4 : cls == 2 ? 0x3 : 0x1;
    return cls == 0 ? 0xC : cls == 1 ? 0x4 : cls == 2 ? 0xF : 0x5;
}
__host__ __device__ __forceinline__ bool partner_self(int mode, int cls) {
    return (mode == 0 && cls == 0) || (mode == 2 && cls == 2);
}

// Q[ct * (MAX_W + 1) + x] = admissible partners of a class-ct member at nbh
// positions < x, i.e. sum over the classes c in partner_mask(mode, ct) of the
// class-c members before position x.
typedef uint8_t PosPrefix[4 * (MAX_W + 1)];

// Rank of partner position px among the admissible partners of the member
// (class ct, position pt) -- the slot offset inside the membership's range.
__device__ __forceinline__ uint32_t pair_rank(const uint8_t *__restrict__ Q, int mode, int ct, int pt,
                                              int px) {
    return (uint32_t)Q[ct * (MAX_W + 1) + px] - (uint32_t)(partner_self(mode, ct) && pt < px);
}

// Warp-cooperative: fill Q from the per-position classes clsv[b] of lanes
// (position b * 32 + lane; class 4 = no member).
__device__ __forceinline__ void build_pos_prefix(uint8_t *Q, const int (&clsv)[4], int mode,
                                                 unsigned lane) {
    int base[4] = {0, 0, 0, 0};
    int mk[4];
#pragma unroll
    for (int c = 0; c < 4; c++) mk[c] = partner_mask(mode, c);
#pragma unroll
    for (int b = 0; b < 4; b++) {
        int before[4];
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const unsigned m = __ballot_sync(FULL_MASK, clsv[b] == c);
            before[c] = base[c] + __popc(m & lanemask_lt());
            base[c] += __popc(m);
        }
#pragma unroll
        for (int ct = 0; ct < 4; ct++) {
            int q = 0;
#pragma unroll
            for (int c = 0; c < 4; c++) q += (mk[ct] >> c & 1) ? before[c] : 0;
            Q[ct * (MAX_W + 1) + b * 32 + lane] = (uint8_t)q;
        }
    }
}

// ---------------------------------------------------------------------------
// Scan: exclusive prefix sum, out has n+1 entries (out[n] = total).
// ---------------------------------------------------------------------------
constexpr int SCAN_THREADS = 512;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

template <typename TI, typename TO>
__global__ void k_scan_tiles(const TI *__restrict__ in, TO *__restrict__ out, int64_t n,
                             TO *__restrict__ tile_sums) {
    __shared__ TO warp_tot[SCAN_THREADS / 32];
    int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    TO v[SCAN_ITEMS];
    TO run = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; i++) {
        TO x = (base + i < n) ? (TO)in[base + i] : (TO)0;
        v[i] = run;
        run += x;
    }
    unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    TO incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        TO y = __shfl_up_sync(FULL_MASK, incl, o);
        if (lane >= (unsigned)o) incl += y;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        TO w = lane < SCAN_THREADS / 32 ? warp_tot[lane] : (TO)0;
        TO wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            TO y = __shfl_up_sync(FULL_MASK, wi, o);
            if (lane >= (unsigned)o) wi += y;
        }
        if (lane < SCAN_THREADS / 32) warp_tot[lane] = wi - w;
        if (lane == SCAN_THREADS / 32 - 1) tile_sums[blockIdx.x] = wi;
    }
    __syncthreads();
    TO off = warp_tot[warp] + (incl - run);
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; i++)
        if (base + i < n) out[base + i] = v[i] + off;
}

template <typename TO>
__global__ void k_scan_add(TO *__restrict__ out, int64_t n, const TO *__restrict__ tile_off) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] += tile_off[i / SCAN_TILE];
}

template <typename TO>
__global__ void k_scan_total(TO *__restrict__ out, int64_t n, const TO *__restrict__ tile_off,
                             int64_t ntiles) {
    out[n] = tile_off[ntiles];
}

// ---------------------------------------------------------------------------
// State setup
// ---------------------------------------------------------------------------
__global__ void k_gather_norms(const float *__restrict__ src, const int64_t *__restrict__ gids,
                               int64_t n, float *__restrict__ dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[gids[i]];
}

__global__ void k_gather_rows(const float *__restrict__ src, int dp, const int64_t *__restrict__ gids,
                              int64_t n, float *__restrict__ dst) {
    int64_t q = dp / 4;
    int64_t total = n * q;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = i / q, c = i % q;
        reinterpret_cast<float4 *>(dst)[r * q + c] =
            reinterpret_cast<const float4 *>(src)[gids[r] * q + c];
    }
}

// Fused membership segments: mpack[x] = (roff[x] + x * (k + 1)) << 32 (the
// base of row x's fixed-capacity record segment, count 0).
__global__ void k_mpack_init(const uint32_t *__restrict__ roff, int64_t n, int k,
                             unsigned long long *__restrict__ mpack) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n;
         x += (int64_t)gridDim.x * blockDim.x)
        mpack[x] = (unsigned long long)(roff[x] + (uint32_t)x * (uint32_t)(k + 1)) << 32;
}

// Exact fp64 squared norm of every row (sequential, as _kernels.py:65-70).
__global__ void k_row_sqnorm64(const float *__restrict__ sub, int dp, int d, int64_t n,
                               double *__restrict__ out) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x)
        out[r] = exact_sqnorm(sub + r * dp, d);
}

__global__ void k_pad_rows(const float *__restrict__ src, int d, int dp, int64_t n,
                           float *__restrict__ dst) {
    int64_t total = n * dp;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = i / dp, c = i % dp;
        dst[i] = c < d ? src[r * d + c] : 0.0f;
    }
}

__global__ void k_init_lists(int64_t n, int k, int32_t *ids, double *dists, uint8_t *flags,
                             int32_t *sizes) {
    int64_t total = n * k;
    double inf = __longlong_as_double(0x7ff0000000000000LL);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        ids[i] = -1;
        dists[i] = inf;
        if (flags) flags[i] = 0;
        if (i < n) sizes[i] = 0;
    }
}

__device__ __forceinline__ int32_t lookup_local(const int64_t *__restrict__ ug, int64_t n, int64_t g) {
    // np.searchsorted(union, g) (side='left'); ug == nullptr: the union is
    // 0 .. n-1 (identity)
    if (!ug) return (int32_t)(g < 0 ? 0 : g < n ? g : n);
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (ug[mid] < g) lo = mid + 1; else hi = mid;
    }
    return (int32_t)lo;
}

// split (graph.py:202-229) + _localize_rows (merge.py:129-143) + rear rows.
__global__ void k_load_graph(const int32_t *__restrict__ rows, int64_t m, const int32_t *__restrict__ gi,
                             const double *__restrict__ gd, const int32_t *__restrict__ gs, int gk,
                             int k1, int k, const int64_t *__restrict__ ug, int64_t n, int32_t *ids,
                             double *dists, int32_t *sizes, int32_t *tail_ids, double *tail_d,
                             int32_t *tail_s, int tk, unsigned long long *not_f32) {
    int64_t total = m * (int64_t)gk;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t j = i / gk;
        int t = (int)(i % gk);
        int64_t r = rows[j];
        int sz = gs[j];
        int hs = sz < k1 ? sz : k1;
        if (t < hs) {
            int32_t g = gi[i];
            ids[r * k + t] = g >= 0 ? lookup_local(ug, n, g) : -1;
            dists[r * k + t] = gd[i];
            // lists the fp32 apply may hold: every loaded distance exact in fp32
            if (g >= 0 && (double)(float)gd[i] != gd[i]) atomicAdd(not_f32, 1ull);
        } else if (t >= k1 && t < sz && tk > 0) {
            tail_ids[r * tk + (t - k1)] = gi[i];
            tail_d[r * tk + (t - k1)] = gd[i];
        }
        if (t == 0) {
            if (k1 > 0) sizes[r] = hs;  // k1 == 0: heads are empty (rows start empty)
            if (tk > 0) tail_s[r] = sz > k1 ? sz - k1 : 0;
        }
    }
}

__global__ void k_repeat_rows(const int32_t *__restrict__ rows, int count, int64_t m,
                              int32_t *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = rows[i / count];
}

// ---------------------------------------------------------------------------
// numpy PCG64 (XSL-RR 128/64) + Generator.integers(0, m) on the device.
// A bit-exact restatement of numpy/random/src/pcg64/pcg64.h (step, output,
// next_uint32 with the has_uint32 half-buffer) and of
// buffered_bounded_lemire_uint32 (distributions.c) -- the draws of
// merge.py:156-163 (rng.integers(0, m, size=(nrows, t))).  The raw 32-bit
// stream is produced in parallel by LCG jump-ahead; Lemire rejections are
// removed by a scan, so draw j is the j-th accepted raw value, exactly as
// numpy's sequential loop consumes them.  The host advances numpy's
// generator state by the consumed raw count afterwards.
// ---------------------------------------------------------------------------
typedef unsigned __int128 u128;

__host__ __device__ __forceinline__ u128 pcg_mult() {
    return ((u128)0x2360ED051FC65DA4ULL << 64) | (u128)0x4385DF649FCCF645ULL;
}

__device__ __forceinline__ uint64_t pcg_out(u128 st) {
    const uint64_t x = (uint64_t)(st >> 64) ^ (uint64_t)st;
    const unsigned r = (unsigned)(st >> 122);
    return (x >> r) | (x << ((64u - r) & 63u));
}

// state after `delta` LCG steps (pcg_advance_lcg_128)
__device__ __forceinline__ u128 pcg_advance(u128 st, u128 inc, uint64_t delta) {
    u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = inc;
    while (delta > 0) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    return acc_mult * st + acc_plus;
}

// Raw u32 stream r = 0..R-1 -> (value, accepted).  With a buffered half
// (has0), raw 0 is uint0 and raw r >= 1 comes from output (r-1)/2; else raw
// r comes from output r/2 (low half first).  Each thread covers `per`
// consecutive outputs.
__global__ void k_pcg_raw(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo, int has0,
                          uint32_t uint0, uint64_t m, int64_t R, int per, uint32_t *val,
                          uint32_t *acc) {
    const u128 st0 = ((u128)st_hi << 64) | st_lo, inc = ((u128)inc_hi << 64) | inc_lo;
    const uint32_t thr = (uint32_t)((0xFFFFFFFFull - (m - 1)) % m);
    const int64_t nout = (R - (has0 ? 1 : 0) + 1) / 2;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t * per < nout;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o0 = t * per;
        u128 st = pcg_advance(st0, inc, (uint64_t)o0);
        for (int q = 0; q < per && o0 + q < nout; q++) {
            st = st * pcg_mult() + inc;
            const uint64_t v = pcg_out(st);
            const int64_t rbase = (has0 ? 1 : 0) + 2 * (o0 + q);
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int64_t r = rbase + h;
                if (r < R) {
                    const uint32_t x = h ? (uint32_t)(v >> 32) : (uint32_t)v;
                    const uint64_t mm = (uint64_t)x * m;
                    val[r] = (uint32_t)(mm >> 32);
                    acc[r] = ((uint32_t)mm >= thr) ? 1u : 0u;
                }
            }
        }
    }
    if (has0 && blockIdx.x == 0 && threadIdx.x == 0) {
        const uint64_t mm = (uint64_t)uint0 * m;
        val[0] = (uint32_t)(mm >> 32);
        acc[0] = ((uint32_t)mm >= thr) ? 1u : 0u;
    }
}

// Compact accepted raw values into draws[0..N) (row-major into the listed
// rows of the draw matrix when rows != nullptr); record the raw index of
// the N-th accepted value.
__global__ void k_pcg_compact(const uint32_t *__restrict__ val, const uint32_t *__restrict__ acc,
                              const uint64_t *__restrict__ pos, int64_t R, int64_t N,
                              int64_t *draws, const int64_t *__restrict__ rows, int t,
                              unsigned long long *last) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < R;
         r += (int64_t)gridDim.x * blockDim.x) {
        if (!acc[r]) continue;
        const uint64_t j = pos[r];
        if (j >= (uint64_t)N) continue;
        const int64_t dst = rows ? rows[j / t] * t + (int64_t)(j % t) : (int64_t)j;
        draws[dst] = (int64_t)val[r];
        if (j == (uint64_t)N - 1) *last = (unsigned long long)r;
    }
}

// Random-append candidate matrix (merge.py:146-163): flag rows of an
// (nrows, t) int64 draw matrix that contain a repeated value.  Only rows in
// `rows` (or all rows when rows == nullptr) are checked.
__global__ void k_dup_rows(const int64_t *__restrict__ cand, int64_t nrows, int t,
                           const int64_t *__restrict__ rows, int64_t nchk, int64_t *bad,
                           unsigned long long *counters) {
    int64_t total = rows ? nchk : nrows;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = rows ? rows[i] : i;
        const int64_t *row = cand + r * t;
        bool dup = false;
        for (int a = 1; a < t && !dup; a++) {
            int64_t x = row[a];
            for (int b = 0; b < a; b++)
                if (row[b] == x) { dup = true; break; }
        }
        if (dup) bad[atomicAdd(&counters[C_CAND], 1ull)] = r;
    }
}

// Replace rows of the draw matrix with redrawn values.
__global__ void k_put_rows(int64_t *cand, int t, const int64_t *__restrict__ rows, int64_t nbad,
                           const int64_t *__restrict__ vals) {
    int64_t total = nbad * t;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x)
        cand[rows[i / t] * t + i % t] = vals[i];
}

// nids = pool[cand] as int32 local ids.
__global__ void k_pool_map(const int64_t *__restrict__ cand, int64_t m, const int32_t *__restrict__ pool,
                           int32_t *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = pool[cand[i]];
}

// ---------------------------------------------------------------------------
// Directed init inserts: distances + candidate emission
// (_eval_pairs -> pair_dists_dense, then apply_updates_directed order).
// ---------------------------------------------------------------------------
// Certified data (integer entries, d * range^2 < 2^24): every fp32 partial
// sum is an exact integer, so any summation order gives the reference's value.
__device__ __forceinline__ double cert_dist(const float *__restrict__ a, const float *__restrict__ b,
                                            int dp, int tag) {
    const float4 *a4 = reinterpret_cast<const float4 *>(a);
    const float4 *b4 = reinterpret_cast<const float4 *>(b);
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    for (int c = 0; c < (dp >> 2); c++) {
        const float4 x = __ldg(a4 + c), y = __ldg(b4 + c);
        const float t0 = x.x - y.x, t1 = x.y - y.y, t2 = x.z - y.z, t3 = x.w - y.w;
        if (tag == 1) {
            s0 = fmaf(t0, t0, s0); s1 = fmaf(t1, t1, s1); s2 = fmaf(t2, t2, s2); s3 = fmaf(t3, t3, s3);
        } else {
            s0 += fabsf(t0); s1 += fabsf(t1); s2 += fabsf(t2); s3 += fabsf(t3);
        }
    }
    return (double)((s0 + s1) + (s2 + s3));
}

// u8 rows (entries in [0, 255], the u8 certificate): exact integer
// |a|^2 + |b|^2 - 2 a.b from 128-bit loads and dp4a (rowb bytes per row).
__device__ __forceinline__ double u8_dist(const uint8_t *__restrict__ a, const uint8_t *__restrict__ b, int rowb,
                                          float na, float nb) {
    const uint4 *a4 = reinterpret_cast<const uint4 *>(a);
    const uint4 *b4 = reinterpret_cast<const uint4 *>(b);
    unsigned dot = 0;
    for (int c = 0; c < (rowb >> 4); c++) {
        const uint4 x = __ldg(a4 + c), y = __ldg(b4 + c);
        dot = __dp4a(x.x, y.x, dot);
        dot = __dp4a(x.y, y.y, dot);
        dot = __dp4a(x.z, y.z, dot);
        dot = __dp4a(x.w, y.w, dot);
    }
    return (double)((long long)__float_as_int(na) + (long long)__float_as_int(nb) - 2ll * (long long)dot);
}

__global__ void k_directed_emit(const int32_t *__restrict__ rows, const int32_t *__restrict__ nids,
                                int64_t m, const float *__restrict__ sub, int dp, int d, int tag, int cert,
                                const int32_t *__restrict__ sizes, const double *__restrict__ dists,
                                int k, const uint64_t *__restrict__ boff,
                                const uint32_t *__restrict__ start, double *__restrict__ Bd,
                                int32_t *__restrict__ Bs, double *cap_d, const uint8_t *__restrict__ sub8,
                                int rowb, const float *__restrict__ norms8) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = rows[i], s = nids[i];
        const double dd = sub8 ? u8_dist(sub8 + (int64_t)r * rowb, sub8 + (int64_t)s * rowb, rowb, norms8[r], norms8[s])
                        : cert ? cert_dist(sub + (int64_t)r * dp, sub + (int64_t)s * dp, dp, tag)
                               : exact_dist_tag(tag, sub + (int64_t)r * dp, sub + (int64_t)s * dp, d);
        if (cap_d) cap_d[i] = dd;
        const uint64_t slot = boff[r] + start[i];
        // slots are pre-filled with NaN; only updates that can pass are written
        if (!(sizes[r] == k && dd >= dists[(int64_t)r * k + k - 1])) {
            Bd[slot] = dd;
            Bs[slot] = s;
        }
    }
}

// Row-grouped directed inserts (insert_rows / draws_insert: every row given
// once, with `count` candidates in order): apply_updates_directed
// (_kernels.py:208-214) is _insert per candidate in input order, rows
// independent, so one warp per row applies them straight from registers --
// no bucket layout, ranking or slot round trip.  Distances as k_directed_emit.
// BATCH (non-certified rows): a chunk's up to 32 exact values are folded
// together by lazy_batch_t (cp.async-staged dimension blocks, one pair per
// lane) instead of one strided sequential scan per lane.
template <int E, bool BATCH>
__global__ void __launch_bounds__(BATCH ? 128 : 256)
k_insert_rows_direct(const int32_t *__restrict__ rows, int64_t mrows, int count,
                     const int32_t *__restrict__ nids, const float *__restrict__ sub, int dp, int d,
                     int tag, int cert, const uint8_t *__restrict__ sub8, int rowb,
                     const float *__restrict__ norms8, int32_t *ids, double *dists, uint8_t *flags,
                     int32_t *sizes, int k, double *cap_d, unsigned long long *counters, LazyExact z) {
    __shared__ LazyBatchSmem s_b[BATCH ? 4 : 1];
    const unsigned lane = lane_id();
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    unsigned long long acc = 0;
    for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < mrows; i += nw) {
        const int32_t r = rows[i];
        WarpRow<E, double> s;
        row_load<E, double>(s, ids, dists, flags, sizes, r, k, lane);
        int a = 0;
        for (int t0 = 0; t0 < count; t0 += 32) {
            const int t = t0 + (int)lane;
            int32_t src = 0;
            double dd = 0.0;
            const int cnt = count - t0 < 32 ? count - t0 : 32;
            if constexpr (BATCH) {
                LazyBatchSmem &b = s_b[threadIdx.x >> 5];
                if (t < count) {
                    src = nids[i * count + t];
                    b.sid[lane] = src;
                }
                __syncwarp();
                if (z.tag == 1) dd = lazy_batch_t<1>(z, r, cnt, b, lane);
                else if (z.tag == 0) dd = lazy_batch_t<0>(z, r, cnt, b, lane);
                else dd = lazy_batch_t<2>(z, r, cnt, b, lane);
                if (t < count && cap_d) cap_d[i * count + t] = dd;
                __syncwarp();
            } else if (t < count) {
                src = nids[i * count + t];
                dd = sub8 ? u8_dist(sub8 + (int64_t)r * rowb, sub8 + (int64_t)src * rowb, rowb, norms8[r], norms8[src])
                   : cert ? cert_dist(sub + (int64_t)r * dp, sub + (int64_t)src * dp, dp, tag)
                          : exact_dist_tag(tag, sub + (int64_t)r * dp, sub + (int64_t)src * dp, d);
                if (cap_d) cap_d[i * count + t] = dd;
            }
            for (int j = 0; j < cnt; j++) {
                const int sj = __shfl_sync(FULL_MASK, src, j);
                const double dj = __shfl_sync(FULL_MASK, dd, j);
                if constexpr (E == 1) a += warp_insert1<double>(s, k, sj, dj, lane);
                else a += warp_insert<E, true, double>(s, k, sj, dj, lane);
            }
        }
        if (a) row_store<E, double>(s, ids, dists, flags, sizes, r, k, lane);
        acc += (unsigned long long)a;
    }
    if (lane == 0 && acc) atomicAdd(&counters[C_ACCEPTED], acc);
}

// Duplicate-row test for the direct path: counters[C_DUPROWS] > 0 when a
// row occurs twice in rows[0, m).
__global__ void k_rows_distinct(const int32_t *__restrict__ rows, int64_t m, uint32_t *bits,
                                unsigned long long *counters) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t r = (uint32_t)rows[i];
        const uint32_t b = 1u << (r & 31);
        if (atomicOr(&bits[r >> 5], b) & b) atomicAdd(&counters[C_DUPROWS], 1ull);
    }
}

// ---------------------------------------------------------------------------
// Reverse CSR (_kernels.py:262-281): in-degree histogram, then scatter of
// (source << 1 | new-flag).  Segment order is restored where it matters
// (Fisher-Yates subsampling) by sorting on the source id in the assemble step.
// ---------------------------------------------------------------------------
// Sample rate rho < 1 (classic NN-Descent; the reference is rho = 1): of
// row u's new entries (list order), at most new_cap take part in this
// round, chosen by the reverse sampler's partial Fisher-Yates (splitmix64,
// state seed ^ SALT ^ (u+1)*gamma, one warm-up step; oracle orc_sample_new).
// The others get flag 2: skipped by the reverse lists and the hood, and
// still new after the round (k_assemble restores them).  Thread per row.
constexpr uint64_t FWD_SALT = 0x6a09e667f3bcc909ULL;
__global__ void k_sample_new(const int32_t *__restrict__ sizes, int64_t n, int k, uint8_t *flags,
                             int new_cap, uint64_t seed) {
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
         u += (int64_t)gridDim.x * blockDim.x) {
        const int sz = sizes[u];
        uint8_t pos[64];
        int c = 0;
        for (int t = 0; t < sz; t++)
            if (flags[u * k + t]) pos[c++] = (uint8_t)t;
        if (c <= new_cap) continue;
        uint8_t idx[64];
        uint64_t keep = 0;
        for (int t = 0; t < c; t++) idx[t] = (uint8_t)t;
        const uint64_t st0 = (seed ^ FWD_SALT) ^ ((uint64_t)(u + 1) * U64_GAMMA);
        for (int t = 0; t < new_cap; t++) {
            const uint64_t z = mix64(st0 + (uint64_t)(t + 2) * U64_GAMMA);
            const int r = t + (int)(z % (uint64_t)(c - t));
            const uint8_t tmp = idx[t];
            idx[t] = idx[r];
            idx[r] = tmp;
            keep |= 1ull << idx[t];
        }
        for (int t = 0; t < c; t++)
            if (!((keep >> t) & 1)) flags[u * k + pos[t]] = 2;
    }
}

// (flag 2 = a new entry sitting out this round under rho-sampling, see
// k_sample_new: it takes no part in the reverse lists)
// Also marks live[x] = 1 for every row whose hood can hold a new entry this
// round: rows with a flagged forward entry and targets of new forward
// entries (their reverse edge is new).  Other hoods have no admissible pair
// (_kernels.py:391-399 needs new_p or new_q): k_assemble skips them.
// Both reverse kernels walk the n*k list entries with 32-bit indices
// (n*k < 2^31, checked in knnm_begin) and take REV_U entries per thread per
// step, their loads issued together: the per-entry chain (entry -> target's
// offset / counter -> store) is latency-bound, so independent entries in
// flight are what hides it.
constexpr int REV_U = 4;

__global__ void k_rev_count(const int32_t *__restrict__ ids, const uint8_t *__restrict__ flags,
                            const int32_t *__restrict__ sizes, int64_t n, int k, uint32_t *indeg,
                            int64_t tlo, int64_t thi, uint8_t *live) {
    const uint32_t total = (uint32_t)(n * k), uk = (uint32_t)k;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < total; i0 += REV_U * stride) {
        int32_t j[REV_U];
        uint32_t f[REV_U], r[REV_U];
        bool in[REV_U];
#pragma unroll
        for (int q = 0; q < REV_U; q++) {
            const uint32_t i = i0 + q * stride;
            in[q] = i < total;
            r[q] = in[q] ? i / uk : 0u;
            j[q] = in[q] ? ids[i] : -1;
            f[q] = in[q] ? flags[i] : 0u;
            in[q] = in[q] && (int)(i - r[q] * uk) < sizes[r[q]];
        }
#pragma unroll
        for (int q = 0; q < REV_U; q++) {
            if (!in[q]) continue;
            if (f[q] != 0) live[r[q]] = 1;  // new or sitting out (its flag is restored)
            if (f[q] != 2 && j[q] >= tlo && j[q] < thi) {
                atomicAdd(&indeg[j[q]], 1u);
                if (f[q] == 1) live[j[q]] = 1;
            }
        }
    }
}

// Only targets whose hood will be assembled (live, see k_rev_count) get
// their reverse segment filled; the offsets still count every edge.
__global__ void k_rev_fill(const int32_t *__restrict__ ids, const uint8_t *__restrict__ flags,
                           const int32_t *__restrict__ sizes, int64_t n, int k,
                           const uint32_t *__restrict__ roff, uint32_t *indeg, uint32_t *rev,
                           int64_t tlo, int64_t thi, const uint8_t *__restrict__ live) {
    const uint32_t total = (uint32_t)(n * k), uk = (uint32_t)k;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < total; i0 += REV_U * stride) {
        int32_t j[REV_U];
        uint32_t f[REV_U], r[REV_U], p[REV_U];
        bool ok[REV_U];
#pragma unroll
        for (int q = 0; q < REV_U; q++) {
            const uint32_t i = i0 + q * stride;
            ok[q] = i < total;
            r[q] = ok[q] ? i / uk : 0u;
            j[q] = ok[q] ? ids[i] : -1;
            f[q] = ok[q] ? flags[i] : 2u;
            ok[q] = ok[q] && (int)(i - r[q] * uk) < sizes[r[q]] && j[q] >= tlo && j[q] < thi && f[q] != 2;
        }
#pragma unroll
        for (int q = 0; q < REV_U; q++) ok[q] = ok[q] && live[j[q]];
#pragma unroll
        for (int q = 0; q < REV_U; q++)
            if (ok[q]) p[q] = roff[j[q]] + atomicSub(&indeg[j[q]], 1u) - 1u;
#pragma unroll
        for (int q = 0; q < REV_U; q++)
            if (ok[q]) rev[p[q]] = (r[q] << 1) | f[q];
    }
}

__global__ void k_find_heavy(const uint32_t *__restrict__ roff, int64_t lo, int64_t n, int limit,
                             int32_t *heavy, unsigned long long *counters,
                             const uint8_t *__restrict__ live, int32_t *giant, int smem_max) {
    for (int64_t u = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
         u += (int64_t)gridDim.x * blockDim.x) {
        uint32_t deg = roff[u + 1] - roff[u];
        if (deg > (uint32_t)limit && live[u]) {
            unsigned long long p = atomicAdd(&counters[C_HEAVY_REV], 1ull);
            heavy[p] = (int32_t)u;
            // too long for a block's shared memory: the global-scratch pass
            if (next_pow2(deg) > (uint32_t)smem_max) giant[atomicAdd(&counters[C_GIANT], 1ull)] = (int32_t)u;
            atomicMax(&counters[C_MAXDEG], (unsigned long long)deg);
        }
    }
}

// Partial Fisher-Yates subsample (_kernels.py:345-361) for one vertex whose
// reverse segment is sorted in seg[0..deg).  Writes the rev_cap selected
// entries into out[0..rev_cap).  Block-cooperative; idx has >= deg slots.
__device__ void block_fy_select(uint32_t *seg, uint32_t *idx, uint32_t *R, uint32_t deg,
                                int rev_cap, uint64_t seed, int64_t u, uint32_t *out) {
    for (uint32_t j = threadIdx.x; j < deg; j += blockDim.x) idx[j] = j;
    uint64_t st0 = seed ^ ((uint64_t)(u + 1) * U64_GAMMA);
    for (int t = threadIdx.x; t < rev_cap; t += blockDim.x) {
        uint64_t z = mix64(st0 + (uint64_t)(t + 2) * U64_GAMMA);
        R[t] = (uint32_t)t + (uint32_t)(z % (uint64_t)(deg - (uint32_t)t));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int t = 0; t < rev_cap; t++) {
            uint32_t r = R[t];
            uint32_t tmp = idx[t];
            idx[t] = idx[r];
            idx[r] = tmp;
        }
    }
    __syncthreads();
    // read all selections before any write (out may alias seg's storage)
    uint32_t v = 0;
    if ((int)threadIdx.x < rev_cap) v = seg[idx[threadIdx.x]];
    __syncthreads();
    if ((int)threadIdx.x < rev_cap) out[threadIdx.x] = v;
}

// Heavy reverse segments: one block per vertex, shared-memory sort.  The
// selected entries overwrite the first rev_cap slots of the segment.
// gscratch == nullptr: the rows of `heavy` that fit shared memory; else the
// `giant` list (counters[C_GIANT]) in global scratch.
// Segments with smem_min < next_pow2(deg) <= smem_max are sorted in shared
// memory (launched once with a small smem_max, so that many blocks share an
// SM, and once for the rest); gscratch != nullptr: the giant pass.
__global__ void k_rev_heavy(const int32_t *__restrict__ heavy, const unsigned long long *counters,
                            const uint32_t *__restrict__ roff, uint32_t *rev, int rev_cap,
                            uint64_t seed, uint32_t *gscratch, int smem_max, int smem_min) {
    extern __shared__ uint32_t hs[];
    __shared__ uint32_t R[MAX_W];
    unsigned long long cnt = counters[gscratch ? C_GIANT : C_HEAVY_REV];
    for (unsigned long long h = blockIdx.x; h < cnt; h += gridDim.x) {
        int64_t u = heavy[h];
        uint32_t lo = roff[u];
        uint32_t deg = roff[u + 1] - lo;
        uint32_t P2 = next_pow2(deg);
        bool in_smem = P2 <= (uint32_t)smem_max;
        if (!in_smem && gscratch == nullptr) continue;  // a later pass
        if (in_smem && gscratch != nullptr) continue;
        if (gscratch == nullptr && P2 <= (uint32_t)smem_min) continue;  // an earlier pass
        uint32_t *seg = in_smem ? hs : gscratch;
        uint32_t *idx = seg + P2;
        for (uint32_t j = threadIdx.x; j < P2; j += blockDim.x) seg[j] = j < deg ? rev[lo + j] : 0xffffffffu;
        __syncthreads();
        bitonic_block<uint32_t>(seg, P2);
        block_fy_select(seg, idx, R, deg, rev_cap, seed, u, rev + lo);
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Locality order of hoods (performance only: results do not depend on the
// order hoods are processed in, since updates land in reference-order slots).
// Min-label propagation over the forward lists groups vertices by graph
// region; a counting sort by label gives the assembly (and join) order, so
// concurrently processed hoods share members and the gathers hit L2.
// ---------------------------------------------------------------------------
// Only "old" entries (the input subgraphs' lists) carry labels: the random
// cross appends are new-flagged and would turn the graph into an expander.
__global__ void k_label_prop(const int32_t *__restrict__ ids, const uint8_t *__restrict__ flags,
                             const int32_t *__restrict__ sizes, int64_t n, int k,
                             const int32_t *__restrict__ lin, int32_t *lout) {
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
         u += (int64_t)gridDim.x * blockDim.x) {
        int32_t m = lin[u];
        const int sz = sizes[u];
        for (int t = 0; t < sz; t++) {
            if (flags[u * k + t]) continue;
            const int32_t v = lin[ids[u * k + t]];
            m = v < m ? v : m;
        }
        lout[u] = m;
    }
}

// labels (int8, one per row) -> bitmap, one bit per row.
__global__ void k_label_bits(const int8_t *__restrict__ labels, int64_t n, uint32_t *__restrict__ bits) {
    const int64_t nw = (n + 31) >> 5;
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nw;
         w += (int64_t)gridDim.x * blockDim.x) {
        uint32_t b = 0;
        for (int i = 0; i < 32; i++) {
            const int64_t r = w * 32 + i;
            if (r < n && labels[r] != 0) b |= 1u << i;
        }
        bits[w] = b;
    }
}

__global__ void k_iota(int32_t *a, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        a[i] = (int32_t)i;
}

__global__ void k_label_hist(const int32_t *__restrict__ lab, int64_t n, uint32_t *hist) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&hist[lab[i]], 1u);
}

__global__ void k_label_scatter(const int32_t *__restrict__ lab, int64_t n,
                                const uint32_t *__restrict__ off, uint32_t *cur, int32_t *order) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t l = lab[i];
        order[off[l] + atomicAdd(&cur[l], 1u)] = (int32_t)i;
    }
}

// ---------------------------------------------------------------------------
// Neighbourhood assembly (_kernels.py:316-383) + flag clear
// (construct.py:142) + pair counting (_kernels.py:402-417, closed form) +
// round-start worst snapshot for the exact prefilter.  One warp per vertex.
// nbh entries are packed (local id << 1 | new).
// ---------------------------------------------------------------------------
constexpr int ASM_WARPS = 8;

// Sort a[0..m) (u32, m <= 32 * NE) with a register bitonic sort and write it
// back (padding slots become 0xffffffff).
template <int NE>
__device__ __forceinline__ void warp_sort_smem_u32(uint32_t *a, int m, unsigned lane) {
    uint32_t v[NE];
#pragma unroll
    for (int e = 0; e < NE; e++) {
        const int j = e * 32 + (int)lane;
        v[e] = j < m ? a[j] : 0xffffffffu;
    }
    warp_sort_reg<NE, uint32_t>(v, lane);
#pragma unroll
    for (int e = 0; e < NE; e++) a[e * 32 + lane] = v[e];
    __syncwarp();
}

__device__ __forceinline__ void warp_sort_any_u32(uint32_t *a, int m, unsigned lane) {
    __syncwarp();
    if (m <= 32) warp_sort_smem_u32<1>(a, m, lane);
    else if (m <= 64) warp_sort_smem_u32<2>(a, m, lane);
    else if (m <= 128) warp_sort_smem_u32<4>(a, m, lane);
    else warp_sort_smem_u32<8>(a, m, lane);
}

__device__ __forceinline__ uint64_t pairs_closed_form(int mode, int an, int ao, int bn, int bo) {
    uint64_t a = an + ao, b = bn + bo, w = a + b, wo = ao + bo;
    if (mode == 0) return w * (w - 1) / 2 - wo * (wo - (wo ? 1 : 0)) / 2;
    uint64_t cross = a * b - (uint64_t)ao * bo;
    if (mode == 1) return cross;
    return cross + b * (b - (b ? 1 : 0)) / 2 - (uint64_t)bo * (bo - (bo ? 1 : 0)) / 2;
}

__device__ __forceinline__ uint32_t members_closed_form(int mode, int an, int ao, int bn, int bo) {
    int a = an + ao, b = bn + bo, w = a + b, wn = an + bn, wo = ao + bo;
    if (mode == 0) return (w >= 2 ? wn : 0) + (wn >= 1 ? wo : 0);
    uint32_t m = (b >= 1 ? an : 0) + (bn >= 1 ? ao : 0);
    if (mode == 1) return m + (a >= 1 ? bn : 0) + (an >= 1 ? bo : 0);
    return m + ((a >= 1 || b >= 2) ? bn : 0) + ((an >= 1 || bn >= 1) ? bo : 0);
}

template <int MODE>
__global__ void __launch_bounds__(ASM_WARPS * 32, 6)
k_assemble(const int32_t *__restrict__ ids, uint8_t *flags, const int32_t *__restrict__ sizes,
           const double *__restrict__ dists, int64_t n, int k, int rev_cap,
           const uint32_t *__restrict__ roff, const uint32_t *__restrict__ rev, uint64_t seed,
           const uint32_t *__restrict__ labbits, int mode_rt, int W, uint32_t *nbh, int32_t *nlen,
           uint32_t *hpairs, double *worst0, int32_t *active, unsigned long long *counters,
           int64_t lo, uint32_t *bound, uint32_t *mcount, const int32_t *__restrict__ order,
           MembRec *memb, unsigned long long *mpack, const uint8_t *__restrict__ live) {
    constexpr int mode = MODE;  // (mode_rt == MODE)
    (void)mode_rt;
    __shared__ uint32_t s_seg[ASM_WARPS][WARP_REV_MAX];
    __shared__ uint32_t s_idx[ASM_WARPS][WARP_REV_MAX];
    __shared__ uint32_t s_R[ASM_WARPS][MAX_W];
    __shared__ uint32_t s_buf[ASM_WARPS][MAX_W];
    unsigned lane = lane_id(), wib = threadIdx.x >> 5;
    uint32_t *seg = s_seg[wib], *idx = s_idx[wib], *R = s_R[wib], *buf = s_buf[wib];
    int64_t nw = (int64_t)gridDim.x * ASM_WARPS;
    unsigned long long members = 0;
    for (int64_t uu = lo + (int64_t)blockIdx.x * ASM_WARPS + wib; uu < n; uu += nw) {
        const int64_t u = order ? (int64_t)order[uu] : uu;
        int sz = sizes[u];
        // issued early: they overlap the forward-list pass below
        const double dlast = dists[u * k + k - 1];
        const uint32_t ro0 = roff[u], ro1 = roff[u + 1];
        if (!live[u]) {
            // no new entry can reach this hood: no pairs, flags already clear
            if (lane == 0) {
                worst0[u] = sz == k ? dlast : __longlong_as_double(0x7ff0000000000000LL);
                nlen[u] = 0;
                hpairs[u] = 0;
            }
            continue;
        }
        // forward entries (rho-skipped ones, flag 2, sit out) and the flag
        // clear of construct.py:142 (skipped ones stay new)
        int m = 0;
        for (int t0 = 0; t0 < k; t0 += 32) {
            const int t = t0 + (int)lane;
            uint32_t f = 0, id = 0;
            if (t < sz) {
                id = (uint32_t)ids[u * k + t];
                f = flags[u * k + t];
            }
            const bool keep = t < sz && f != 2;
            const unsigned bal = __ballot_sync(FULL_MASK, keep);
            if (keep) buf[m + __popc(bal & lanemask_lt())] = (id << 1) | f;
            m += __popc(bal);
            if (t < k) flags[u * k + t] = f == 2 ? 1 : 0;
        }
        __syncwarp();
        if (lane == 0) worst0[u] = sz == k ? dlast : __longlong_as_double(0x7ff0000000000000LL);
        uint32_t lo = ro0, deg = ro1 - lo;
        if (deg <= (uint32_t)rev_cap) {
            for (uint32_t j = lane; j < deg; j += 32) buf[m + j] = rev[lo + j];
            m += deg;
        } else if (deg <= (uint32_t)WARP_REV_MAX) {
            for (uint32_t j = lane; j < deg; j += 32) {
                seg[j] = rev[lo + j];
                idx[j] = j;
            }
            uint64_t st0 = seed ^ ((uint64_t)(u + 1) * U64_GAMMA);
            for (int t = lane; t < rev_cap; t += 32) {
                uint64_t z = mix64(st0 + (uint64_t)(t + 2) * U64_GAMMA);
                R[t] = (uint32_t)t + (uint32_t)(z % (uint64_t)(deg - (uint32_t)t));
            }
            warp_sort_any_u32(seg, (int)deg, lane);
            if (lane == 0) {
                for (int t = 0; t < rev_cap; t++) {
                    uint32_t r = R[t];
                    uint32_t tmp = idx[t];
                    idx[t] = idx[r];
                    idx[r] = tmp;
                }
            }
            __syncwarp();
            for (int t = lane; t < rev_cap; t += 32) buf[m + t] = seg[idx[t]];
            m += rev_cap;
        } else {
            for (int t = lane; t < rev_cap; t += 32) buf[m + t] = rev[lo + t];  // pre-selected
            m += rev_cap;
        }
        warp_sort_any_u32(buf, m, lane);  // m <= k + rev_cap <= MAX_W
        // compact runs of equal ids; the last element of a run carries OR(flags)
        int w = 0;
        int an = 0, ao = 0, bn = 0, bo = 0;
        for (int base = 0; base < m; base += 32) {
            int j = base + lane;
            bool end = false;
            uint32_t v = 0;
            if (j < m) {
                v = buf[j];
                end = (j == m - 1) || ((buf[j + 1] >> 1) != (v >> 1));
            }
            unsigned em = __ballot_sync(FULL_MASK, end);
            int lab = 0;
            if (end) {
                // label bitmap (1 bit per row: 8x denser than the int8 labels,
                // so the random gathers mostly hit L1)
                lab = (labbits[(v >> 1) >> 5] >> ((v >> 1) & 31)) & 1u;
                // hood entry: id << 2 | label << 1 | new (the label rides along
                // so the join needs no dependent labels[] load)
                const uint32_t ent = ((v >> 1) << 2) | ((uint32_t)lab << 1) | (v & 1);
                const int at = w + __popc(em & lanemask_lt());
                nbh[u * W + at] = ent;
                R[at] = ent;  // staged for the membership pass below (R is free now)
            }
            bool nw_ = end && (v & 1);
            an += __popc(__ballot_sync(FULL_MASK, end && lab == 0 && nw_));
            ao += __popc(__ballot_sync(FULL_MASK, end && lab == 0 && !nw_));
            bn += __popc(__ballot_sync(FULL_MASK, end && lab != 0 && nw_));
            bo += __popc(__ballot_sync(FULL_MASK, end && lab != 0 && !nw_));
            w += __popc(em);
        }
        const uint64_t pc = pairs_closed_form(mode, an, ao, bn, bo);
        if (lane == 0) {
            nlen[u] = w;
            hpairs[u] = (uint32_t)pc;
            if (pc > 0) {
                unsigned long long p = atomicAdd(&counters[C_ACTIVE], 1ull);
                active[p] = (int32_t)u;
                members += members_closed_form(mode, an, ao, bn, bo);
            }
        }
        __syncwarp();
        if (bound != nullptr && pc > 0) {
            // membership counting for the reference-order slot layout (the
            // first pass of k_hood_memb, fused): admissible partners per member
            const int cnt4[4] = {an, ao, bn, bo};
            for (int j = lane; j < w; j += 32) {
                const uint32_t e = R[j];
                const int cls = (mode == 0 ? 0 : (int)((e >> 1) & 1)) * 2 + ((e & 1) ? 0 : 1);
                const int mk = partner_mask(mode, cls);
                int part = -(int)partner_self(mode, cls);
#pragma unroll
                for (int c = 0; c < 4; c++)
                    if (mk & (1 << c)) part += cnt4[c];
                if (part > 0) {
                    const uint32_t x = e >> 2;
                    // fused: the row totals come from k_seg_rank instead
                    if (!memb) atomicAdd(&bound[x], (uint32_t)part);
                    if (memb) {
                        // fused membership record (unsharded, unchunked
                        // rounds): row x lies in at most indeg(x) + k hoods
                        // (x in fwd(u) <=> u in rev(x); x in rev(u) <=> u in
                        // fwd(x)), so its records fit a segment of that
                        // capacity; mpack[x] = segment base << 32 | count, so
                        // one atomic yields the record's address
                        const unsigned long long at = atomicAdd(&mpack[x], 1ull);
                        memb[(uint32_t)(at >> 32) + (uint32_t)at] =
                            MembRec{(uint32_t)u, (uint16_t)part, (uint16_t)j};
                    } else {
                        atomicAdd(&mcount[x], 1u);
                    }
                }
            }
        }
    }
    if (lane == 0 && members) atomicAdd(&counters[C_MEMBERS], members);
}

// Update-slot formats.  PLAIN: Bd f64 distance + Bs int32 source.  LAZY:
// PLAIN, where the sign bit marks an fp32 approximation (LazyExact).
// PACKED (certified routes, whose distances are integers < 2^24 and hence
// exact in fp32): one u64 per slot in the Bd buffer, fp32 distance bits in
// the high word, source row in the low word -- one store per update.  The
// all-ones prefill reads as NaN in every format ("cannot pass").
constexpr int SLOTS_PLAIN = 0, SLOTS_LAZY = 1, SLOTS_PACKED = 2;

__device__ __forceinline__ unsigned long long pack_slot(double d, int src) {
    return ((unsigned long long)__float_as_uint((float)d) << 32) | (uint32_t)src;
}

// ---------------------------------------------------------------------------
// Local join, exact route (_kernels.py:402-437 pair enumeration +
// _kernels.py:113-119 distances + the candidate side of
// apply_updates_grouped).  One CTA per active hood.  Member vectors are
// staged in shared memory (128-bit loads); every admissible pair (p < q) is
// evaluated with the exact fp64 metric; each directed update that can still
// be accepted (d < round-start worst of its target) is emitted with its
// reference-order key.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool admissible(int na, int nb, int la, int lb, int mode) {
    // _kernels.py:391-399
    if (!(na || nb)) return false;
    if (mode == 1) return la != lb;
    if (mode == 2) return la != lb || (la == 1 && lb == 1);
    return true;
}

constexpr int JOIN_THREADS = 128;

template <int TAG>
__global__ void __launch_bounds__(JOIN_THREADS)
k_join_exact(const int32_t *__restrict__ active, const uint32_t *__restrict__ nbh,
             const int32_t *__restrict__ nlen, int W, const int8_t *__restrict__ labels, int mode,
             const float *__restrict__ sub, int dp, int d, const double *__restrict__ worst0,
             const uint64_t *__restrict__ boff, const uint32_t *__restrict__ start,
             double *__restrict__ Bd, int32_t *__restrict__ Bs) {
    extern __shared__ float4 sv4[];
    __shared__ int s_id[MAX_W];
    __shared__ int s_new[MAX_W];
    __shared__ int s_cls[MAX_W];
    __shared__ double s_w[MAX_W];
    __shared__ uint64_t s_st[MAX_W];
    __shared__ PosPrefix s_P;
    const float *sv = reinterpret_cast<const float *>(sv4);
    const int64_t u = active[blockIdx.x];
    const int w = nlen[u];
    if (threadIdx.x < 32) {
        const unsigned lane = lane_id();
        int clsv[4];
#pragma unroll
        for (int b = 0; b < 4; b++) {
            const int j = b * 32 + (int)lane;
            clsv[b] = 4;
            if (j < w) {
                const uint32_t e = nbh[u * W + j];
                const int id = (int)(e >> 2);
                const int lab = mode == 0 ? 0 : (int)((e >> 1) & 1);
                clsv[b] = lab * 2 + ((e & 1) ? 0 : 1);
                s_id[j] = id;
                s_new[j] = e & 1;
                s_cls[j] = clsv[b];
                s_w[j] = worst0[id];
                s_st[j] = boff[id] + start[u * W + j];
            }
        }
        build_pos_prefix(s_P, clsv, mode, lane);
    }
    __syncthreads();
    const int q4 = dp >> 2;
    for (int i = threadIdx.x; i < w * q4; i += blockDim.x) {
        const int r = i / q4, c = i - r * q4;
        sv4[i] = __ldg(reinterpret_cast<const float4 *>(sub + (int64_t)s_id[r] * dp) + c);
    }
    __syncthreads();
    const int total = w * w;
    for (int L = threadIdx.x; L < total; L += blockDim.x) {
        const int p = L / w, q = L - (L / w) * w;
        if (q <= p || !admissible(s_new[p], s_new[q], s_cls[p] >> 1, s_cls[q] >> 1, mode)) continue;
        const double dd = exact_dist<TAG>(sv + p * dp, sv + q * dp, d);
        const uint64_t spq = s_st[p] + pair_rank(s_P, mode, s_cls[p], p, q);
        const uint64_t sqp = s_st[q] + pair_rank(s_P, mode, s_cls[q], q, p);
        // slots are pre-filled with NaN ("cannot pass"); only updates that
        // can still be accepted (d < round-start worst) are written
        if (dd < s_w[p]) { Bd[spq] = dd; Bs[spq] = s_id[q]; }
        if (dd < s_w[q]) { Bd[sqp] = dd; Bs[sqp] = s_id[p]; }
    }
}

// ---------------------------------------------------------------------------
// Local join, tiled route (the product kernel).  One CTA per active hood
// (grid-stride).  Member vectors are staged into shared memory by TMA bulk
// copies (cp.async.bulk, one per member row, completion on an mbarrier).
// Members are re-ordered into classes (label, new-first) so the admissible
// region is a union of dense blocks:
//     CROSS        A x B                    (A = label 0, B = label 1)
//     CROSS_OR_S2  A x B  +  B x B (upper)
//     ALL          M x M (upper)
// Each thread owns 2x2 register tiles of the block (fp32 SIMT FMA, 128-bit
// shared loads, broadcast-friendly lane layout).  Tiles that hold only
// old x old pairs are skipped.
//   CERT  : the dataset carries an exactness certificate (integer values,
//           d * range^2 < 2^24): every fp32 partial sum is an exact integer,
//           so the fp32 value IS the reference's fp64 value.
//   !CERT : the fp32 value is stored as an approximation (sign bit set) when
//           its rigorous lower bound can beat the target's round-start worst;
//           the apply evaluates the exact fp64 metric only for slots that can
//           still pass the row's current state (LazyExact, knnm_device.cuh).
// Emission as in k_join_exact: reference-order key (u, p, q), exact-safe
// prefilter against the round-start worst of each target.
// ---------------------------------------------------------------------------
constexpr int TJ_WARPS = 2;       // warps per hood for small rows
constexpr int TJ_WARPS_BIG = 8;   // warps per hood when rows are long (large d)
constexpr int TJ_THREADS = TJ_WARPS * 32;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    }
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int TAG, bool CERT, bool LAZY>
__global__ void __launch_bounds__(TJ_WARPS_BIG * 32)
k_join_tiled(const int32_t *__restrict__ active, int nactive, const uint32_t *__restrict__ nbh,
             const int32_t *__restrict__ nlen, int W, const int8_t *__restrict__ labels, int mode,
             const float *__restrict__ sub, int dp, int d, const double *__restrict__ worst0,
             const uint64_t *__restrict__ boff, const uint32_t *__restrict__ start,
             double *__restrict__ Bd, int32_t *__restrict__ Bs, double lo_rel, double lo_abs,
             const double *__restrict__ nrm64, unsigned long long *counters) {
    extern __shared__ __align__(128) float4 sv4[];
    __shared__ int s_id[MAX_W];
    __shared__ int s_pos[MAX_W];
    __shared__ int s_new[MAX_W];
    __shared__ double s_w[MAX_W];
    __shared__ float s_nrm[MAX_W];
    __shared__ uint64_t s_st[MAX_W];
    __shared__ int s_sc[MAX_W];
    __shared__ PosPrefix s_P;
    __shared__ int s_cls[4];
    __shared__ __align__(8) uint64_t s_bar;
    // exact-in-join route (!CERT && !LAZY): screened-pair queue (< nthreads
    // left over + one wave of nwarps patches x 128 pairs) and exact norms
    constexpr bool QUEUE = !CERT && !LAZY;
    __shared__ uint32_t s_q[QUEUE ? TJ_WARPS_BIG * 32 + TJ_WARPS_BIG * 128 : 1];
    __shared__ double s_nrm64[QUEUE && TAG == 2 ? MAX_W : 1];
    __shared__ int s_qlen;
    __shared__ unsigned long long s_nexact;
    const int tid = threadIdx.x;
    const unsigned lane = lane_id();
    const int warp = tid >> 5;
    const int nwarps = blockDim.x >> 5;
    const int q4 = dp >> 2;
    const int qs = q4 + 1;  // padded row stride in float4
    if (tid == 0) {
        mbar_init(&s_bar, 1);
        s_qlen = 0;
        s_nexact = 0;
    }
    __syncthreads();
    uint32_t phase = 0;

    for (int hi = blockIdx.x; hi < nactive; hi += gridDim.x) {
        const int64_t u = active[hi];
        const int w = nlen[u];
        // ---- classify members: class = (label != 0) * 2 + (!new) ----------
        if (tid < 32) {
            uint32_t ev[4];
            int clsv[4];
            int cnts[4] = {0, 0, 0, 0};
#pragma unroll
            for (int b = 0; b < 4; b++) {
                const int j = b * 32 + (int)lane;
                ev[b] = j < w ? nbh[u * W + j] : 0u;
            }
#pragma unroll
            for (int b = 0; b < 4; b++) {
                const int j = b * 32 + (int)lane;
                int cls = 4;
                if (j < w) {
                    const int lab = mode == 0 ? 0 : (int)((ev[b] >> 1) & 1);
                    cls = lab * 2 + ((ev[b] & 1) ? 0 : 1);
                }
                clsv[b] = cls;
#pragma unroll
                for (int c = 0; c < 4; c++) cnts[c] += __popc(__ballot_sync(FULL_MASK, cls == c));
            }
            const int base_cls[4] = {0, cnts[0], cnts[0] + cnts[1], cnts[0] + cnts[1] + cnts[2]};
            int fill[4] = {0, 0, 0, 0};
#pragma unroll
            for (int b = 0; b < 4; b++) {
                const int j = b * 32 + (int)lane;
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    const unsigned m = __ballot_sync(FULL_MASK, clsv[b] == c);
                    if (clsv[b] == c) {
                        const int slot = base_cls[c] + fill[c] + __popc(m & lanemask_lt());
                        const int id = (int)(ev[b] >> 2);
                        s_id[slot] = id;
                        s_pos[slot] = j;
                        s_new[slot] = (int)(ev[b] & 1);
                        s_sc[slot] = c;
                        s_w[slot] = worst0[id];
                        if (QUEUE && TAG == 2) s_nrm64[slot] = nrm64[id];
                        s_st[slot] = boff[id] + start[u * W + j];
                    }
                    fill[c] += __popc(m);
                }
            }
            build_pos_prefix(s_P, clsv, mode, lane);
            if (lane < 4) s_cls[lane] = cnts[lane];
        }
        __syncthreads();
        // ---- stage the member rows with TMA bulk copies ---------------------
        // smem row stride = dp + 4 floats: consecutive rows start 16 B apart
        // modulo 128 B, so 8 distinct rows per wavefront are conflict-free.
        // slot s lives in smem row (s & 1) * H + (s >> 1): the two rows of a
        // 2x2 tile sit in different halves, so consecutive tiles of a warp
        // read consecutive rows (16 B apart modulo 128 B: conflict-free).
        const int H = (w + 1) >> 1;
        if (warp == 0) {  // the copies are issued by all lanes of warp 0
            fence_proxy_async();
            const uint32_t row_bytes = (uint32_t)dp * 4u;
            if (lane == 0) mbar_expect_tx(&s_bar, row_bytes * (uint32_t)w);
            __syncwarp();
            for (int sl = (int)lane; sl < w; sl += 32)
                bulk_g2s(sv4 + (size_t)((sl & 1) * H + (sl >> 1)) * qs, sub + (int64_t)s_id[sl] * dp,
                         row_bytes, &s_bar);
        }
        mbar_wait(&s_bar, phase);
        phase ^= 1u;
        if (TAG == 2) {
            // fp32 norms for the cosine screen
            for (int sl = warp; sl < w; sl += nwarps) {
                float acc = 0.f;
                for (int c = lane; c < q4; c += 32) {
                    float4 a = sv4[(size_t)((sl & 1) * H + (sl >> 1)) * qs + c];
                    acc = fmaf(a.x, a.x, acc);
                    acc = fmaf(a.y, a.y, acc);
                    acc = fmaf(a.z, a.z, acc);
                    acc = fmaf(a.w, a.w, acc);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL_MASK, acc, o);
                if (lane == 0) s_nrm[sl] = acc;
            }
            __syncthreads();
        }
        // ---- blocks ----------------------------------------------------------
        const int nAn = s_cls[0], nAo = s_cls[1], nBn = s_cls[2];
        const int nA = nAn + nAo;
        // block 0 and (CROSS_OR_S2 only) block 1; plain scalars, no local arrays
        const int b0r0 = 0, b0r1 = mode == 0 ? w : nA, b0c0 = mode == 0 ? 0 : nA, b0c1 = w;
        const int b0rn = nAn, b0cn = mode == 0 ? nAn : nBn, b0tri = mode == 0;
        const int b1r0 = nA, b1r1 = w, b1c0 = nA, b1c1 = w, b1rn = nBn, b1cn = nBn;
        const int nblk = mode == 2 ? 2 : 1;
        const int nrt0 = (b0r1 - b0r0 + 1) >> 1, nct0 = (b0c1 - b0c0 + 1) >> 1;
        const int nrt1 = (b1r1 - b1r0 + 1) >> 1, nct1 = (b1c1 - b1c0 + 1) >> 1;
        const int pc0 = (nct0 + 7) >> 3, np0 = ((nrt0 + 3) >> 2) * pc0;
        const int pc1 = (nct1 + 7) >> 3, np1 = nblk == 2 ? ((nrt1 + 3) >> 2) * pc1 : 0;
        // each warp takes 4 x 8 patches of 2 x 2 tiles (8 rows x 16 cols)
        auto rowp = [&](int sl) { return sv4 + (size_t)((sl & 1) * H + (sl >> 1)) * qs; };
        // fp32 2x2 tile of patch pid; returns whether the lane's tile is live
        auto patch = [&](int pid, int &i0, int &j0, int &r1, int &c1, bool &tri, float (&acc)[2][2]) {
            const bool second = pid >= np0;
            const int lp = second ? pid - np0 : pid;
            const int pcs = second ? pc1 : pc0;
            const int pr = lp / pcs, pcc = lp - pr * pcs;
            const int rt = pr * 4 + (int)(lane >> 3), ct = pcc * 8 + (int)(lane & 7);
            const int r0 = second ? b1r0 : b0r0;
            const int c0 = second ? b1c0 : b0c0;
            r1 = second ? b1r1 : b0r1;
            c1 = second ? b1c1 : b0c1;
            const int rn = second ? b1rn : b0rn, cn = second ? b1cn : b0cn;
            tri = second ? true : (bool)b0tri;
            i0 = r0 + 2 * rt;
            j0 = c0 + 2 * ct;
            bool live = i0 < r1 && j0 < c1;
            if (live && tri && rt > ct) live = false;             // below diagonal
            if (live && 2 * rt >= rn && 2 * ct >= cn) live = false;  // old x old
            const bool vi1 = i0 + 1 < r1, vj1 = j0 + 1 < c1;
            acc[0][0] = acc[0][1] = acc[1][0] = acc[1][1] = 0.f;
            if (live) {
                const float4 *a0p = rowp(i0);
                const float4 *a1p = rowp(vi1 ? i0 + 1 : i0);
                const float4 *b0p = rowp(j0);
                const float4 *b1p = rowp(vj1 ? j0 + 1 : j0);
#pragma unroll 4
                for (int c = 0; c < q4; c++) {
                    float4 a0 = a0p[c], a1 = a1p[c], b0 = b0p[c], b1 = b1p[c];
                    if (TAG == 1) {
#define KNNM_L2_ACC(ACC, X, Y)                         \
    {                                                  \
        float t_;                                      \
        t_ = X.x - Y.x; ACC = fmaf(t_, t_, ACC);       \
        t_ = X.y - Y.y; ACC = fmaf(t_, t_, ACC);       \
        t_ = X.z - Y.z; ACC = fmaf(t_, t_, ACC);       \
        t_ = X.w - Y.w; ACC = fmaf(t_, t_, ACC);       \
    }
                        KNNM_L2_ACC(acc[0][0], a0, b0);
                        KNNM_L2_ACC(acc[0][1], a0, b1);
                        KNNM_L2_ACC(acc[1][0], a1, b0);
                        KNNM_L2_ACC(acc[1][1], a1, b1);
#undef KNNM_L2_ACC
                    } else if (TAG == 0) {
#define KNNM_L1_ACC(ACC, X, Y)                                                          \
    {                                                                                   \
        ACC += fabsf(X.x - Y.x); ACC += fabsf(X.y - Y.y);                               \
        ACC += fabsf(X.z - Y.z); ACC += fabsf(X.w - Y.w);                               \
    }
                        KNNM_L1_ACC(acc[0][0], a0, b0);
                        KNNM_L1_ACC(acc[0][1], a0, b1);
                        KNNM_L1_ACC(acc[1][0], a1, b0);
                        KNNM_L1_ACC(acc[1][1], a1, b1);
#undef KNNM_L1_ACC
                    } else {
#define KNNM_DOT_ACC(ACC, X, Y)                                                          \
    {                                                                                    \
        ACC = fmaf(X.x, Y.x, ACC); ACC = fmaf(X.y, Y.y, ACC);                            \
        ACC = fmaf(X.z, Y.z, ACC); ACC = fmaf(X.w, Y.w, ACC);                            \
    }
                        KNNM_DOT_ACC(acc[0][0], a0, b0);
                        KNNM_DOT_ACC(acc[0][1], a0, b1);
                        KNNM_DOT_ACC(acc[1][0], a1, b0);
                        KNNM_DOT_ACC(acc[1][1], a1, b1);
#undef KNNM_DOT_ACC
                    }
                }
            }
            return live;
        };
        // admissible pair (ii, jj) of a tile
        auto pair_ok = [&](bool live, int ii, int jj, int r1, int c1, bool tri) {
            bool ok = live && ii < r1 && jj < c1;
            if (ok && tri) ok = ii < jj;
            if (ok) ok = s_new[ii] || s_new[jj];
            return ok;
        };
        // write both directions of a pair to their reference-order slots
        // (value dd; lb = a lower bound of the exact distance, or dd itself)
        auto emit = [&](int ii, int jj, double dd, double lb) {
            const bool e1 = lb < s_w[ii];  // id[ii] <- id[jj]
            const bool e2 = lb < s_w[jj];  // id[jj] <- id[ii]
            const int pi = s_pos[ii], pj = s_pos[jj];
            if (e1) {
                const uint64_t sij = s_st[ii] + pair_rank(s_P, mode, s_sc[ii], pi, pj);
                Bd[sij] = dd;
                Bs[sij] = s_id[jj];
            }
            if (e2) {
                const uint64_t sji = s_st[jj] + pair_rank(s_P, mode, s_sc[jj], pj, pi);
                Bd[sji] = dd;
                Bs[sji] = s_id[ii];
            }
        };
        // approximate value v (>= 0) and a rigorous lower bound of the exact
        // distance from the fp32 one; values outside the fp32-safe range give
        // bound 0 / -lo_abs (always evaluated exactly)
        auto approx = [&](int ii, int jj, float f, float &v) {
            double lb;
            if (TAG == 2) {
                const float na = s_nrm[ii], nb = s_nrm[jj];
                if (na >= 1e-30f && nb >= 1e-30f && na <= 1e30f && nb <= 1e30f) {
                    v = fmaxf(1.0f - f / (sqrtf(na) * sqrtf(nb)), 0.0f);
                    lb = (double)v - lo_abs;
                } else {
                    v = 0.0f;
                    lb = -lo_abs;
                }
            } else {
                v = (f >= 1e-30f && f <= 1e30f) ? f : 0.0f;
                lb = (double)v * lo_rel;
            }
            return lb;
        };
        const int npatch = np0 + np1;
        if (!QUEUE) {
        for (int pid = warp; pid < npatch; pid += nwarps) {
            int i0, j0, r1, c1;
            bool tri;
            float acc[2][2];
            const bool live = patch(pid, i0, j0, r1, c1, tri, acc);
#pragma unroll
            for (int s = 0; s < 4; s++) {
                const int ii = i0 + (s >> 1), jj = j0 + (s & 1);
                if (!pair_ok(live, ii, jj, r1, c1, tri)) continue;
                const float f = acc[s >> 1][s & 1];
                if (CERT) {
                    // every fp32 value is exact: packed slots
                    const double dd = (double)f;
                    unsigned long long *Bp = reinterpret_cast<unsigned long long *>(Bd);
                    if (dd < s_w[ii])
                        Bp[s_st[ii] + pair_rank(s_P, mode, s_sc[ii], s_pos[ii], s_pos[jj])] = pack_slot(dd, s_id[jj]);
                    if (dd < s_w[jj])
                        Bp[s_st[jj] + pair_rank(s_P, mode, s_sc[jj], s_pos[jj], s_pos[ii])] = pack_slot(dd, s_id[ii]);
                } else {
                    // LAZY: store the approximation (sign bit set); the apply
                    // evaluates it exactly only if it can still pass
                    float v;
                    const double lb = approx(ii, jj, f, v);
                    if (lb < s_w[ii] || lb < s_w[jj]) emit(ii, jj, -(double)v, lb);
                }
            }
        }
        } else {
            // exact in the join: fp32 screen in synchronized waves (one patch
            // per warp per wave); pairs that may pass go to a shared queue,
            // drained in whole multiples of the block (one exact fp64
            // evaluation per thread from the staged rows, no divergence, no
            // straggler warp at the hood barrier)
            const int nthreads = blockDim.x;
            const int nwaves = (npatch + nwarps - 1) / nwarps;
            for (int wave = 0; wave < nwaves; wave++) {
                const int pid = wave * nwarps + warp;
                if (pid < npatch) {
                    int i0, j0, r1, c1;
                    bool tri;
                    float acc[2][2];
                    const bool live = patch(pid, i0, j0, r1, c1, tri, acc);
#pragma unroll
                    for (int s = 0; s < 4; s++) {
                        const int ii = i0 + (s >> 1), jj = j0 + (s & 1);
                        bool maybe = pair_ok(live, ii, jj, r1, c1, tri);
                        if (maybe) {
                            float v;
                            const double lb = approx(ii, jj, acc[s >> 1][s & 1], v);
                            maybe = lb < s_w[ii] || lb < s_w[jj];
                        }
                        const unsigned m = __ballot_sync(FULL_MASK, maybe);
                        int base = 0;
                        if (lane == 0 && m) base = atomicAdd(&s_qlen, __popc(m));
                        base = __shfl_sync(FULL_MASK, base, 0);
                        if (maybe) s_q[base + __popc(m & lanemask_lt())] = (uint32_t)(ii | (jj << 8));
                    }
                }
                __syncthreads();
                const int qlen = s_qlen;
                const bool last = wave == nwaves - 1;
                if (qlen >= nthreads || (last && qlen > 0)) {
                    const int take = last ? qlen : (qlen / nthreads) * nthreads;
                    for (int e = qlen - take + tid; e < qlen; e += nthreads) {
                        const uint32_t code = s_q[e];
                        const int ii = (int)(code & 0xFF), jj = (int)(code >> 8);
                        const float *ra = reinterpret_cast<const float *>(rowp(ii));
                        const float *rb = reinterpret_cast<const float *>(rowp(jj));
                        const double dd = TAG == 2 ? exact_cos_norms(ra, rb, d, s_nrm64[ii], s_nrm64[jj])
                                                   : exact_dist<TAG>(ra, rb, d);
                        emit(ii, jj, dd, dd);
                    }
                    __syncthreads();
                    if (tid == 0) {
                        s_qlen = qlen - take;
                        s_nexact += (unsigned long long)take;
                    }
                    __syncthreads();
                }
            }
        }
        __syncthreads();  // smem reused by the next hood
    }
    if (QUEUE && tid == 0 && s_nexact) atomicAdd(&counters[C_EXACT], s_nexact);
}

// ---------------------------------------------------------------------------
// Local join, chunked lazy route (non-certified rows with d > LAZY_MIN_D):
// the tiled route's arithmetic and emission (approximate slots, LazyExact),
// but the hood's rows stream through two CJ_DC-dimension shared buffers by
// TMA (chunk c + 2 loads while c + 1 is computed), so a CTA stages ~1 KB per
// member instead of a whole 3.8 KB row: several CTAs fit an SM and the row
// fetches overlap the fp32 work.  Each warp keeps its tiles' running sums in
// registers across chunks (the same sequential fmaf chains as the tiled
// route); hoods with more than CJ_TPW patches per warp take extra passes.
// ---------------------------------------------------------------------------
constexpr int CJ_DC = 128;  // dimensions per chunk
constexpr int CJ_TPW = 2;   // patches per warp per pass
constexpr int CJ_WARPS = 8;
constexpr int CJ_NBUF = 2;  // chunk buffers (3 measured slower: 480 vs 467 ms at config 3, fewer CTAs per SM)

template <int TAG>
__global__ void __launch_bounds__(CJ_WARPS * 32, 4)
k_join_chunked(const int32_t *__restrict__ active, int nactive, const uint32_t *__restrict__ nbh,
               const int32_t *__restrict__ nlen, int W, int mode, const float *__restrict__ sub,
               int dp, const double *__restrict__ worst0, const uint64_t *__restrict__ boff,
               const uint32_t *__restrict__ start, double *__restrict__ Bd, int32_t *__restrict__ Bs,
               double lo_rel, double lo_abs) {
    extern __shared__ __align__(128) float4 cv4[];
    __shared__ int s_id[MAX_W];
    __shared__ int s_pos[MAX_W];
    __shared__ int s_new[MAX_W];
    __shared__ double s_w[MAX_W];
    __shared__ float s_nrm[MAX_W];
    __shared__ uint64_t s_st[MAX_W];
    __shared__ int s_sc[MAX_W];
    __shared__ PosPrefix s_P;
    __shared__ int s_cls[4];
    __shared__ __align__(8) uint64_t s_bar[CJ_NBUF];
    const int tid = threadIdx.x;
    const unsigned lane = lane_id();
    const int warp = tid >> 5;
    constexpr int nwarps = CJ_WARPS;
    constexpr int QC = CJ_DC / 4 + 1;  // padded chunk row stride in float4
    const int nch = (dp + CJ_DC - 1) / CJ_DC;
    if (tid == 0)
        for (int b = 0; b < CJ_NBUF; b++) mbar_init(&s_bar[b], 1);
    __syncthreads();
    uint32_t phases = 0;  // bit b: parity of buffer b's next completion

    for (int hi = blockIdx.x; hi < nactive; hi += gridDim.x) {
        const int64_t u = active[hi];
        const int w = nlen[u];
        // ---- classify members (as k_join_tiled) ------------------------------
        if (tid < 32) {
            uint32_t ev[4];
            int clsv[4];
            int cnts[4] = {0, 0, 0, 0};
#pragma unroll
            for (int b = 0; b < 4; b++) {
                const int j = b * 32 + (int)lane;
                ev[b] = j < w ? nbh[u * W + j] : 0u;
            }
#pragma unroll
            for (int b = 0; b < 4; b++) {
                const int j = b * 32 + (int)lane;
                int cls = 4;
                if (j < w) {
                    const int lab = mode == 0 ? 0 : (int)((ev[b] >> 1) & 1);
                    cls = lab * 2 + ((ev[b] & 1) ? 0 : 1);
                }
                clsv[b] = cls;
#pragma unroll
                for (int c = 0; c < 4; c++) cnts[c] += __popc(__ballot_sync(FULL_MASK, cls == c));
            }
            int f0 = 0, f1 = cnts[0], f2 = cnts[0] + cnts[1], f3 = cnts[0] + cnts[1] + cnts[2];
#pragma unroll
            for (int b = 0; b < 4; b++) {
                const int j = b * 32 + (int)lane;
                const unsigned k0 = __ballot_sync(FULL_MASK, clsv[b] == 0);
                const unsigned k1 = __ballot_sync(FULL_MASK, clsv[b] == 1);
                const unsigned k2 = __ballot_sync(FULL_MASK, clsv[b] == 2);
                const unsigned k3 = __ballot_sync(FULL_MASK, clsv[b] == 3);
                const unsigned lt = lanemask_lt();
                const int c = clsv[b];
                const int slot = c == 0 ? f0 + __popc(k0 & lt) : c == 1 ? f1 + __popc(k1 & lt)
                               : c == 2 ? f2 + __popc(k2 & lt) : c == 3 ? f3 + __popc(k3 & lt) : -1;
                f0 += __popc(k0);
                f1 += __popc(k1);
                f2 += __popc(k2);
                f3 += __popc(k3);
                if (slot >= 0) {
                    const int id = (int)(ev[b] >> 2);
                    s_id[slot] = id;
                    s_pos[slot] = j;
                    s_new[slot] = (int)(ev[b] & 1);
                    s_sc[slot] = c;
                    s_w[slot] = worst0[id];
                    s_st[slot] = boff[id] + start[u * W + j];
                    s_nrm[slot] = 0.f;
                }
            }
            build_pos_prefix(s_P, clsv, mode, lane);
            if (lane < 4) s_cls[lane] = cnts[lane];
        }
        __syncthreads();
        const int H = (w + 1) >> 1;  // even/odd slot split (see k_join_tiled)
        auto rowc = [&](int buf, int sl) { return cv4 + ((size_t)buf * W + (size_t)((sl & 1) * H + (sl >> 1))) * QC; };
        // TMA: chunk c of every member row into buffer c % CJ_NBUF
        auto issue = [&](int c) {
            if (warp == 0) {  // the copies are issued by all lanes of warp 0
                const int b = c % CJ_NBUF;
                const int cw = min(CJ_DC, dp - c * CJ_DC);
                const uint32_t bytes = (uint32_t)cw * 4u;
                fence_proxy_async();
                if (lane == 0) mbar_expect_tx(&s_bar[b], bytes * (uint32_t)w);
                __syncwarp();
                for (int sl = (int)lane; sl < w; sl += 32)
                    bulk_g2s(rowc(b, sl), sub + (int64_t)s_id[sl] * dp + (int64_t)c * CJ_DC, bytes, &s_bar[b]);
            }
        };
        // ---- blocks / patches (as k_join_tiled) ------------------------------
        const int nAn = s_cls[0], nAo = s_cls[1], nBn = s_cls[2];
        const int nA = nAn + nAo;
        const int b0r0 = 0, b0r1 = mode == 0 ? w : nA, b0c0 = mode == 0 ? 0 : nA, b0c1 = w;
        const int b0rn = nAn, b0cn = mode == 0 ? nAn : nBn, b0tri = mode == 0;
        const int b1r0 = nA, b1r1 = w, b1c0 = nA, b1c1 = w, b1rn = nBn, b1cn = nBn;
        const int nblk = mode == 2 ? 2 : 1;
        const int nrt0 = (b0r1 - b0r0 + 1) >> 1, nct0 = (b0c1 - b0c0 + 1) >> 1;
        const int nrt1 = (b1r1 - b1r0 + 1) >> 1, nct1 = (b1c1 - b1c0 + 1) >> 1;
        // 2x2 tiles enumerated row-major over the block(s); thread tid takes
        // tiles tid, tid + blockDim, ... (consecutive lanes share the a-row and
        // read consecutive b-rows: conflict-free, see the even/odd split)
        const int nt0 = nrt0 * nct0, nt1 = nblk == 2 ? nrt1 * nct1 : 0;
        const int npatch = nt0 + nt1;  // (tiles)
        auto geom = [&](int tix, int &i0, int &j0, int &r1, int &c1, bool &tri) {
            const bool second = tix >= nt0;
            const int lt = second ? tix - nt0 : tix;
            const int ncols = second ? nct1 : nct0;
            const int rt = lt / ncols, ct = lt - rt * ncols;
            const int r0 = second ? b1r0 : b0r0, c0 = second ? b1c0 : b0c0;
            r1 = second ? b1r1 : b0r1;
            c1 = second ? b1c1 : b0c1;
            const int rn = second ? b1rn : b0rn, cn = second ? b1cn : b0cn;
            tri = second ? true : (bool)b0tri;
            i0 = r0 + 2 * rt;
            j0 = c0 + 2 * ct;
            bool live = i0 < r1 && j0 < c1;
            if (live && tri && rt > ct) live = false;
            if (live && 2 * rt >= rn && 2 * ct >= cn) live = false;
            return live;
        };
        constexpr int PASS = CJ_TPW * nwarps * 32;
        for (int pg = 0; pg < (npatch > 0 ? npatch : 1); pg += PASS) {
            const bool norms = TAG == 2 && pg == 0;  // fp32 norms accumulate in the first pass
            float acc[CJ_TPW][2][2];
#pragma unroll
            for (int t = 0; t < CJ_TPW; t++) acc[t][0][0] = acc[t][0][1] = acc[t][1][0] = acc[t][1][1] = 0.f;
            for (int c = 0; c < CJ_NBUF - 1 && c < nch; c++) issue(c);
            for (int c = 0; c < nch; c++) {
                const int b = c % CJ_NBUF;
                // chunk c + NBUF - 1 goes into the buffer chunk c - 1 left
                // free (the barrier at the end of the previous step)
                if (c + CJ_NBUF - 1 < nch) issue(c + CJ_NBUF - 1);
                mbar_wait(&s_bar[b], (phases >> b) & 1u);
                phases ^= 1u << b;
                const int q4c = min(CJ_DC, dp - c * CJ_DC) >> 2;
#pragma unroll
                for (int t = 0; t < CJ_TPW; t++) {
                    const int pid = pg + t * nwarps * 32 + tid;
                    if (pid >= npatch) continue;
                    int i0, j0, r1, c1;
                    bool tri;
                    if (!geom(pid, i0, j0, r1, c1, tri)) continue;
                    const float4 *a0p = rowc(b, i0);
                    const float4 *a1p = rowc(b, i0 + 1 < r1 ? i0 + 1 : i0);
                    const float4 *b0p = rowc(b, j0);
                    const float4 *b1p = rowc(b, j0 + 1 < c1 ? j0 + 1 : j0);
                    float x00 = acc[t][0][0], x01 = acc[t][0][1], x10 = acc[t][1][0], x11 = acc[t][1][1];
#pragma unroll 4
                    for (int q = 0; q < q4c; q++) {
                        const float4 a0 = a0p[q], a1 = a1p[q], b0 = b0p[q], b1 = b1p[q];
                        if (TAG == 1) {
#define KNNM_CJ_L2(ACC, X, Y)                      \
    {                                              \
        float t_;                                  \
        t_ = X.x - Y.x; ACC = fmaf(t_, t_, ACC);   \
        t_ = X.y - Y.y; ACC = fmaf(t_, t_, ACC);   \
        t_ = X.z - Y.z; ACC = fmaf(t_, t_, ACC);   \
        t_ = X.w - Y.w; ACC = fmaf(t_, t_, ACC);   \
    }
                            KNNM_CJ_L2(x00, a0, b0);
                            KNNM_CJ_L2(x01, a0, b1);
                            KNNM_CJ_L2(x10, a1, b0);
                            KNNM_CJ_L2(x11, a1, b1);
#undef KNNM_CJ_L2
                        } else if (TAG == 0) {
#define KNNM_CJ_L1(ACC, X, Y)                                                      \
    {                                                                              \
        ACC += fabsf(X.x - Y.x); ACC += fabsf(X.y - Y.y);                          \
        ACC += fabsf(X.z - Y.z); ACC += fabsf(X.w - Y.w);                          \
    }
                            KNNM_CJ_L1(x00, a0, b0);
                            KNNM_CJ_L1(x01, a0, b1);
                            KNNM_CJ_L1(x10, a1, b0);
                            KNNM_CJ_L1(x11, a1, b1);
#undef KNNM_CJ_L1
                        } else {
#define KNNM_CJ_DOT(ACC, X, Y)                                                     \
    {                                                                              \
        ACC = fmaf(X.x, Y.x, ACC); ACC = fmaf(X.y, Y.y, ACC);                      \
        ACC = fmaf(X.z, Y.z, ACC); ACC = fmaf(X.w, Y.w, ACC);                      \
    }
                            KNNM_CJ_DOT(x00, a0, b0);
                            KNNM_CJ_DOT(x01, a0, b1);
                            KNNM_CJ_DOT(x10, a1, b0);
                            KNNM_CJ_DOT(x11, a1, b1);
#undef KNNM_CJ_DOT
                        }
                    }
                    acc[t][0][0] = x00;
                    acc[t][0][1] = x01;
                    acc[t][1][0] = x10;
                    acc[t][1][1] = x11;
                }
                if (norms) {
                    for (int sl = warp; sl < w; sl += nwarps) {
                        float a = 0.f;
                        const float4 *rp = rowc(b, sl);
                        for (int q = lane; q < q4c; q += 32) {
                            const float4 v = rp[q];
                            a = fmaf(v.x, v.x, a);
                            a = fmaf(v.y, v.y, a);
                            a = fmaf(v.z, v.z, a);
                            a = fmaf(v.w, v.w, a);
                        }
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(FULL_MASK, a, o);
                        if (lane == 0) s_nrm[sl] += a;
                    }
                }
                __syncthreads();  // buffer b is free again

            }
            // ---- emission: approximate slots (LazyExact), as k_join_tiled ----
#pragma unroll
            for (int t = 0; t < CJ_TPW; t++) {
                const int pid = pg + t * nwarps * 32 + tid;
                if (pid >= npatch) continue;
                int i0, j0, r1, c1;
                bool tri;
                const bool live = geom(pid, i0, j0, r1, c1, tri);
#pragma unroll
                for (int s4 = 0; s4 < 4; s4++) {
                    const int ii = i0 + (s4 >> 1), jj = j0 + (s4 & 1);
                    bool ok = live && ii < r1 && jj < c1;
                    if (ok && tri) ok = ii < jj;
                    if (ok) ok = s_new[ii] || s_new[jj];
                    if (!ok) continue;
                    const float f = acc[t][s4 >> 1][s4 & 1];
                    float v;
                    double lb;
                    if (TAG == 2) {
                        const float na = s_nrm[ii], nb = s_nrm[jj];
                        if (na >= 1e-30f && nb >= 1e-30f && na <= 1e30f && nb <= 1e30f) {
                            v = fmaxf(1.0f - f / (sqrtf(na) * sqrtf(nb)), 0.0f);
                            lb = (double)v - lo_abs;
                        } else {
                            v = 0.0f;
                            lb = -lo_abs;
                        }
                    } else {
                        v = (f >= 1e-30f && f <= 1e30f) ? f : 0.0f;
                        lb = (double)v * lo_rel;
                    }
                    const double dd = -(double)v;
                    const int pi = s_pos[ii], pj = s_pos[jj];
                    if (lb < s_w[ii]) {
                        const uint64_t sij = s_st[ii] + pair_rank(s_P, mode, s_sc[ii], pi, pj);
                        Bd[sij] = dd;
                        Bs[sij] = s_id[jj];
                    }
                    if (lb < s_w[jj]) {
                        const uint64_t sji = s_st[jj] + pair_rank(s_P, mode, s_sc[jj], pj, pi);
                        Bd[sji] = dd;
                        Bs[sji] = s_id[ii];
                    }
                }
            }
        }
        __syncthreads();  // metadata reused by the next hood
    }
}

// ---------------------------------------------------------------------------
// Local join, tensor-core route for datasets with a dot-form exactness
// certificate (integer entries, |v| <= 2048, 2*d*max|v|^2 < 2^24): rows are
// staged as fp16 (exact), the member Gram block is computed with
// mma.sync.m16n8k16 (fp16 x fp16 -> fp32; every partial sum is an integer
// below 2^24, hence exact), and dist = |a|^2 + |b|^2 - 2 a.b with exact
// per-point norms is bit-identical to the reference's fp64 sequential sum.
// One warp per hood, software-pipelined: while the warp computes hood i, the
// TMA engine fetches hood i+1's rows into the other buffer.
// ---------------------------------------------------------------------------
constexpr int MJ_WARPS = 4;  // independent warps per CTA (one hood each)

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2,
                                        uint32_t &r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t &r0, uint32_t &r1) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];"
                 : "=r"(r0), "=r"(r1)
                 : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Per-row join metadata, gathered with one 16-byte load per member: the
// round-start worst rounded up to fp32 (for an fp32 distance d:
// d < wru <=> d < worst), the row norm (int bits on the u8 route) and the
// row's first bucket slot.
struct __align__(16) RowMeta {
    float wru;
    float nrm;
    uint64_t boff;
};

__global__ void k_rowmeta(int64_t n, const double *__restrict__ worst0, const float *__restrict__ norms,
                          const uint64_t *__restrict__ boff, RowMeta *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = RowMeta{__double2float_ru(worst0[i]), norms[i], boff[i]};
}

// One member of a staged hood (32 bytes: two 128-bit shared loads).
struct __align__(16) MjRec {
    float w;      // round-start worst of the member's row, rounded up to fp32
                  // (for an fp32 distance d: d < w <=> d < worst)
    float pad_;
    uint64_t st;  // first bucket slot of the membership
    int id;       // member row
    float nrm;    // row norm (int bits on the u8 route)
    int pk;       // nbh position | new << 8 | class << 9 | partner_self << 11
    uint32_t q4;  // byte c: partners of a class-c member at positions < this one
};

// Staged rows per warp: a hood (<= W) plus the tile tails past it.  Row
// tiles start at 0 except mode 2's second block (start nA: tails up to 15
// rows); column tiles of 8 start anywhere (tails up to 7 rows).
__host__ __device__ constexpr int mj_rows(int W, int mode) {
    return mode == 2 ? W + 16 : (((W + 15) & ~15) > W + 8 ? ((W + 15) & ~15) : W + 8);
}

__host__ __device__ constexpr size_t mj_meta_bytes(int Wp) {
    return (16 + (size_t)Wp * sizeof(MjRec) + 127) & ~(size_t)127;
}

__device__ __forceinline__ void mma16832_u8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                            uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ MjRec lds_rec(const MjRec *p) {
    const float4 a = reinterpret_cast<const float4 *>(p)[0];
    const float4 b = reinterpret_cast<const float4 *>(p)[1];
    MjRec r;
    r.w = a.x;
    r.st = ((uint64_t)(uint32_t)__float_as_int(a.w) << 32) | (uint32_t)__float_as_int(a.z);
    r.id = __float_as_int(b.x);
    r.nrm = b.y;
    r.pk = __float_as_int(b.z);
    r.q4 = (uint32_t)__float_as_int(b.w);
    return r;
}

// Slot of the update "member a receives partner b" (reference order, see
// pair_rank): membership start + rank of b's position among a's partners,
// i.e. byte class(a) of b's q4 (the position prefix count), minus a itself
// when a is its own class's partner and precedes b.  The record's st holds
// the byte address of its first slot, so a slot is one 32-bit offset from
// it.  (Mode 1: no class is its own partner, so there is no self correction.)
template <int MODE>
__device__ __forceinline__ unsigned long long *mj_slot_ptr(const MjRec &a, const MjRec &b) {
    const int ca = (a.pk >> 9) & 3;
    uint32_t off = (b.q4 >> (8 * ca)) & 0xFFu;
    if (MODE != 1) off -= (uint32_t)(((a.pk >> 11) & 1) && (a.pk & 0xFF) < (b.pk & 0xFF));
    return reinterpret_cast<unsigned long long *>(a.st) + off;
}

// U8 = true: rows are u8 (integer data in [0, 255]); the Gram block uses
// mma.m16n8k32 u8 x u8 -> s32, exact integer arithmetic; norms are integers.
// U8 = false: fp16 rows, m16n8k16 fp16 -> fp32 (exact under the dot-form
// certificate).  `rowb` = staged bytes per row (multiple of 32).  NB = 32-entry
// blocks of a hood (W <= 32 * NB).  MODE = the pair mode (0 all, 1 cross,
// 2 cross-or-S2), a template parameter so partner masks and block shapes
// are constants.  Distances are compared and packed in fp32 against each
// member's round-start worst rounded up to fp32 (exact for fp32 values).
//
// One warp per hood, software-pipelined three deep: while hood i's rows are
// in flight (TMA) and its Gram block computes, hood i+1's per-member metadata
// gathers (worst, norm, bucket offset) and hood i+2's neighbour entries are
// already loading into registers.
template <bool U8, int NB, int MODE>
__global__ void __launch_bounds__(MJ_WARPS * 32, 4)
k_join_mma(const int32_t *__restrict__ active, int nactive, const uint32_t *__restrict__ nbh,
           const int32_t *__restrict__ nlen, int W, const int8_t *__restrict__ labels, int mode_rt,
           const uint8_t *__restrict__ sub16, int rowb, const RowMeta *__restrict__ rmeta,
           const uint32_t *__restrict__ start, double *__restrict__ Bd, int32_t *__restrict__ Bs,
           uint32_t gtag) {
    // gtag: the round's slot generation << 24 (0: NaN-prefilled slots)
    // the pair mode is a template parameter (mode_rt == MODE): partner masks,
    // block shapes and the slot correction fold into constants
    constexpr int mode = MODE;
    (void)mode_rt;
    extern __shared__ __align__(128) char mj_smem[];
    const unsigned lane = lane_id();
    const int warp = threadIdx.x >> 5;
    const int Wp = mj_rows(W, MODE);
    const int rs = rowb + 16;  // padded row stride: conflict-free ldmatrix
    const size_t per_warp = mj_meta_bytes(Wp) + (size_t)Wp * rs;
    char *base = mj_smem + (size_t)warp * per_warp;
    uint64_t *bar = reinterpret_cast<uint64_t *>(base);
    MjRec *rec = reinterpret_cast<MjRec *>(base + 16);
    char *rows = base + mj_meta_bytes(Wp);
    if (lane == 0) mbar_init(bar, 1);
    // zero the row buffer once: slots beyond w feed the MMA tile tails
    for (size_t i = lane * 16; i < (size_t)Wp * rs; i += 32 * 16)
        *reinterpret_cast<float4 *>(rows + i) = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncwarp();
    uint32_t phase = 0;
    const uint32_t row_bytes = (uint32_t)rowb;
    const uint32_t rbase = smem_u32(rows);
    const int stride = gridDim.x * MJ_WARPS;
    const unsigned lt = lanemask_lt();

    // neighbour entries of hood u (all W positions; masked by length later)
    auto load_ev = [&](bool ok, int64_t u, uint32_t (&ev)[NB]) {
#pragma unroll
        for (int b = 0; b < NB; b++) {
            const int j = b * 32 + (int)lane;
            ev[b] = (ok && j < W) ? __ldg(nbh + u * W + j) : 0u;
        }
    };
    // per-member metadata of hood u (independent gathers, issued together)
    // (results are consumed one hood later: no arithmetic on them here, or
    // the warp would wait for the loads right away)
    auto gather = [&](int64_t u, int w, const uint32_t (&ev)[NB], float (&mw)[NB], float (&mn)[NB],
                      uint64_t (&mb)[NB], uint32_t (&ms)[NB]) {
#pragma unroll
        for (int b = 0; b < NB; b++) {
            const int j = b * 32 + (int)lane;
            if (j < w) {
                const int id = (int)(ev[b] >> 2);
                const uint4 rm = __ldg(reinterpret_cast<const uint4 *>(rmeta + id));
                mw[b] = __uint_as_float(rm.x);
                mn[b] = __uint_as_float(rm.y);
                mb[b] = ((uint64_t)rm.w << 32) | rm.z;
                ms[b] = __ldg(start + u * W + j);
            } else {
                mw[b] = 0.f;
                mn[b] = 0.f;
                mb[b] = 0;
                ms[b] = 0;
            }
        }
    };

    int hi = blockIdx.x * MJ_WARPS + warp;
    int64_t u0 = hi < nactive ? __ldg(active + hi) : 0;
    int w0 = hi < nactive ? __ldg(nlen + u0) : 0;
    uint32_t ev0[NB];
    load_ev(hi < nactive, u0, ev0);
    int64_t u1 = hi + stride < nactive ? __ldg(active + hi + stride) : 0;
    int w1 = hi + stride < nactive ? __ldg(nlen + u1) : 0;
    uint32_t ev1[NB];
    load_ev(hi + stride < nactive, u1, ev1);
    int64_t u2 = hi + 2 * stride < nactive ? __ldg(active + hi + 2 * stride) : 0;
    float mw0[NB];
    float mn0[NB];
    uint64_t mb0[NB];
    uint32_t ms0[NB];
    gather(u0, w0, ev0, mw0, mn0, mb0, ms0);

    for (; hi < nactive; hi += stride) {
        const int w = w0;
        // ---- classify members into (label, new-first) slots ------------------
        int clsv[NB];
        int c0n = 0, c1n = 0, c2n = 0, c3n = 0;
#pragma unroll
        for (int b = 0; b < NB; b++) {
            const int j = b * 32 + (int)lane;
            const int lab = (j < w && mode != 0) ? (int)((ev0[b] >> 1) & 1) : 0;
            clsv[b] = j < w ? lab * 2 + ((ev0[b] & 1) ? 0 : 1) : 4;
            c0n += __popc(__ballot_sync(FULL_MASK, clsv[b] == 0));
            c1n += __popc(__ballot_sync(FULL_MASK, clsv[b] == 1));
            c2n += __popc(__ballot_sync(FULL_MASK, clsv[b] == 2));
            c3n += __popc(__ballot_sync(FULL_MASK, clsv[b] == 3));
        }
        fence_proxy_async();  // prior generic reads of the rows vs. async-proxy writes
        if (lane == 0) mbar_expect_tx(bar, row_bytes * (uint32_t)w);
        __syncwarp();
        {
            int f0 = 0, f1 = c0n, f2 = c0n + c1n, f3 = c0n + c1n + c2n;  // class bases
            int g0 = 0, g1 = 0, g2 = 0, g3 = 0;  // class members at earlier positions
            const int mk0 = partner_mask(mode, 0), mk1 = partner_mask(mode, 1);
            const int mk2 = partner_mask(mode, 2), mk3 = partner_mask(mode, 3);
#pragma unroll
            for (int b = 0; b < NB; b++) {
                const unsigned k0 = __ballot_sync(FULL_MASK, clsv[b] == 0);
                const unsigned k1 = __ballot_sync(FULL_MASK, clsv[b] == 1);
                const unsigned k2 = __ballot_sync(FULL_MASK, clsv[b] == 2);
                const unsigned k3 = __ballot_sync(FULL_MASK, clsv[b] == 3);
                const int c = clsv[b];
                const int be0 = g0 + __popc(k0 & lt), be1 = g1 + __popc(k1 & lt);
                const int be2 = g2 + __popc(k2 & lt), be3 = g3 + __popc(k3 & lt);
                const int sl = c == 0 ? f0 + be0 : c == 1 ? f1 + be1 : c == 2 ? f2 + be2
                             : c == 3 ? f3 + be3 : -1;
                g0 += __popc(k0);
                g1 += __popc(k1);
                g2 += __popc(k2);
                g3 += __popc(k3);
                // position prefix counts of this position for each member class
                // (the PosPrefix table row, kept in the member's record)
                auto q = [&](int mk) {
                    return (uint32_t)((mk & 1 ? be0 : 0) + (mk & 2 ? be1 : 0) + (mk & 4 ? be2 : 0) +
                                      (mk & 8 ? be3 : 0));
                };
                const uint32_t q4 = q(mk0) | (q(mk1) << 8) | (q(mk2) << 16) | (q(mk3) << 24);
                if (sl >= 0) {
                    // each lane stages its own members' rows (parallel TMA issue)
                    const int id = (int)(ev0[b] >> 2);
                    const int j = b * 32 + (int)lane;
                    bulk_g2s(rows + (size_t)sl * rs, sub16 + (int64_t)id * rowb, row_bytes, bar);
                    const int pk = j | (int)((ev0[b] & 1) << 8) | (c << 9) | ((int)partner_self(mode, c) << 11);
                    // st: byte address of the membership's first slot
                    const uint64_t st = reinterpret_cast<uint64_t>(Bd) + 8ull * (mb0[b] + ms0[b]);
                    float4 *dst = reinterpret_cast<float4 *>(rec + sl);
                    dst[0] = make_float4(mw0[b], 0.f,
                                         __int_as_float((int)(uint32_t)st), __int_as_float((int)(uint32_t)(st >> 32)));
                    dst[1] = make_float4(__int_as_float(id), mn0[b], __int_as_float(pk),
                                         __int_as_float((int)q4));
                }
            }
        }
        // ---- prefetch: hood i+1 metadata, hood i+2 entries, hood i+3 id --------
        float mw1[NB];
        float mn1[NB];
        uint64_t mb1[NB];
        uint32_t ms1[NB];
        gather(u1, w1, ev1, mw1, mn1, mb1, ms1);
        const bool ok2 = hi + 2 * stride < nactive;
        const int w2 = ok2 ? __ldg(nlen + u2) : 0;
        uint32_t ev2[NB];
        load_ev(ok2, u2, ev2);
        const int64_t u3 = hi + 3 * stride < nactive ? __ldg(active + hi + 3 * stride) : 0;
        __syncwarp();
        mbar_wait(bar, phase);
        phase ^= 1u;
        // ---- Gram blocks and emission -----------------------------------------
        const int nA = c0n + c1n;
        const int nblk = mode == 2 ? 2 : 1;
        const int g = lane >> 2, t4 = lane & 3;
        for (int bk = 0; bk < nblk; bk++) {
            const int r0 = bk ? nA : 0, r1 = bk ? w : (mode == 0 ? w : nA);
            const int cc0 = bk ? nA : (mode == 0 ? 0 : nA), cc1 = w;
            const int rn = bk ? c2n : c0n, cn = bk ? c2n : (mode == 0 ? c0n : c2n);
            const bool tri = bk ? true : (mode == 0);
            for (int m0 = r0; m0 < r1; m0 += 16) {
                // this lane's two row members of the tile row (hoisted)
                const int ia = m0 + g, ib = m0 + g + 8;
                const MjRec ra = lds_rec(rec + (ia < r1 ? ia : r0));
                const MjRec rb = lds_rec(rec + (ib < r1 ? ib : r0));
                for (int n0 = cc0; n0 < cc1; n0 += 8) {
                    if (m0 - r0 >= rn && n0 - cc0 >= cn) continue;  // old x old
                    if (tri && n0 + 7 <= m0) continue;              // below diagonal
                    float acc[4] = {0.f, 0.f, 0.f, 0.f};
                    int iacc[4] = {0, 0, 0, 0};
                    const uint32_t a_addr = rbase + (uint32_t)((m0 + (lane & 15)) * rs + (lane >> 4) * 16);
                    // tile column j holds member n0 + (j >> 1) + 4 (j & 1): a lane's two
                    // columns are members n0 + t4 and n0 + t4 + 4, so the four lanes of a
                    // row store to consecutive slots (one or two 32-byte sectors per
                    // store instruction and row instead of two or three)
                    const uint32_t b_addr = rbase + (uint32_t)((n0 + ((lane & 7) >> 1) + 4 * (lane & 1)) * rs +
                                                               ((lane >> 3) & 1) * 16);
                    // 32 bytes of K per step: 16 fp16 or 32 u8 elements; the
                    // ldmatrix byte layout is the same for both
#pragma unroll 4
                    for (int kb = 0; kb < rowb; kb += 32) {
                        uint32_t a0, a1, a2, a3, b0, b1;
                        ldsm_x4(a_addr + kb, a0, a1, a2, a3);
                        ldsm_x2(b_addr + kb, b0, b1);
                        if (U8)
                            mma16832_u8(iacc, a0, a1, a2, a3, b0, b1);
                        else
                            mma16816(acc, a0, a1, a2, a3, b0, b1);
                    }
                    const int ja = n0 + t4, jb = ja + 4;
                    const MjRec ca = lds_rec(rec + (ja < cc1 ? ja : cc0));
                    const MjRec cb = lds_rec(rec + (jb < cc1 ? jb : cc0));
#pragma unroll
                    for (int s = 0; s < 4; s++) {
                        const MjRec &R = (s >> 1) ? rb : ra;
                        const MjRec &C = (s & 1) ? cb : ca;
                        const int ii = (s >> 1) ? ib : ia, jj = (s & 1) ? jb : ja;
                        bool ok = ii < r1 && jj < cc1;
                        if (ok && tri) ok = ii < jj;
                        if (ok) ok = ((R.pk | C.pk) >> 8) & 1;  // at least one new
                        if (!ok) continue;
                        // fp32 distance: an exact integer (u8) / exact under the
                        // dot-form certificate (fp16)
                        const float dd =
                            U8 ? (float)((__float_as_int(R.nrm) + __float_as_int(C.nrm)) - 2 * iacc[s])
                               : (R.nrm + C.nrm) - 2.0f * acc[s];
                        const unsigned long long pv = (unsigned long long)__float_as_uint(dd) << 32;
                        if (dd < R.w) __stcs(mj_slot_ptr<MODE>(R, C), pv | gtag | (uint32_t)C.id);  // id[ii] <- id[jj]
                        if (dd < C.w) __stcs(mj_slot_ptr<MODE>(C, R), pv | gtag | (uint32_t)R.id);  // id[jj] <- id[ii]
                    }
                }
            }
        }
        __syncwarp();
        // ---- rotate the pipeline ------------------------------------------------
        w0 = w1;
        u1 = u2;
        w1 = w2;
        u2 = u3;
#pragma unroll
        for (int b = 0; b < NB; b++) {
            ev0[b] = ev1[b];
            ev1[b] = ev2[b];
            mw0[b] = mw1[b];
            mn0[b] = mn1[b];
            mb0[b] = mb1[b];
            ms0[b] = ms1[b];
        }
    }
}

// u8 copy of the dataset (integers in [0, 255], zero-padded to dpu) and exact
// integer row norms (stored as int bit patterns in the float norms array).
__global__ void k_to_u8(const float *__restrict__ v, int dp, int64_t n, int dpu,
                        uint8_t *__restrict__ out, float *__restrict__ norms) {
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n;
         r += (int64_t)gridDim.x * (blockDim.x >> 5)) {
        const unsigned lane = lane_id();
        int acc = 0;
        for (int c = lane; c < dpu; c += 32) {
            const int x = c < dp ? (int)v[r * dp + c] : 0;
            out[r * dpu + c] = (uint8_t)x;
            acc += x * x;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL_MASK, acc, o);
        if (lane == 0) norms[r] = __int_as_float(acc);
    }
}

// fp16 copy of the dataset (zero-padded to dph) and exact fp32 row norms.
__global__ void k_to_half(const float *__restrict__ v, int dp, int64_t n, int dph,
                          __half *__restrict__ out, float *__restrict__ norms) {
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n;
         r += (int64_t)gridDim.x * (blockDim.x >> 5)) {
        const unsigned lane = lane_id();
        float acc = 0.f;
        for (int c = lane; c < dph; c += 32) {
            float x = c < dp ? v[r * dp + c] : 0.f;
            out[r * dph + c] = __float2half_rn(x);
            acc = fmaf(x, x, acc);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL_MASK, acc, o);
        if (lane == 0) norms[r] = acc;
    }
}

// Dataset exactness certificate: integer-valued entries and their range.
__global__ void k_data_stats(const float *__restrict__ v, int64_t total, unsigned long long *out) {
    // out[0] = count of non-integer / non-finite entries, out[1] = max as
    // ordered bits, out[2] = min as ordered bits (float -> sortable u32)
    unsigned long long bad = 0;
    unsigned int mx = 0, mn = 0xffffffffu;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        float x = v[i];
        if (!(fabsf(x) < 16777216.0f) || rintf(x) != x) bad++;
        unsigned int b = __float_as_uint(x);
        unsigned int key = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
        mx = key > mx ? key : mx;
        mn = key < mn ? key : mn;
    }
    if (bad) atomicAdd(&out[0], bad);
    atomicMax(&out[1], (unsigned long long)mx);
    atomicMin(&out[2], (unsigned long long)mn);
}

// Hood memberships.  Pass 1 (k_hood_prep): every member of an active hood
// adds its number of admissible partners to its row's slot count and one to
// its membership count.  Pass 2 (k_hood_memb): the memberships are bucketed
// by member row (unordered; k_seg_rank orders them).
template <bool FILL>
__global__ void k_hood_memb(const int32_t *__restrict__ active, int nactive,
                            const uint32_t *__restrict__ nbh, const int32_t *__restrict__ nlen,
                            int W, const int8_t *__restrict__ labels, int mode, uint32_t *bound,
                            uint32_t *mcount, const uint32_t *__restrict__ moff, uint32_t *mcur,
                            MembRec *memb) {
    const unsigned lane = lane_id();
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t hi = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); hi < nactive;
         hi += nw) {
        const int64_t u = active[hi];
        const int w = nlen[u];
        uint32_t ev[4];
        int clsv[4];
        int cnt[4] = {0, 0, 0, 0};
#pragma unroll
        for (int b = 0; b < 4; b++) {
            const int j = b * 32 + (int)lane;
            ev[b] = j < w ? nbh[u * W + j] : 0u;
        }
#pragma unroll
        for (int b = 0; b < 4; b++) {
            const int j = b * 32 + (int)lane;
            int cls = 4;
            if (j < w) {
                const int lab = mode == 0 ? 0 : (int)((ev[b] >> 1) & 1);
                cls = lab * 2 + ((ev[b] & 1) ? 0 : 1);
            }
            clsv[b] = cls;
#pragma unroll
            for (int c = 0; c < 4; c++) cnt[c] += __popc(__ballot_sync(FULL_MASK, cls == c));
        }
#pragma unroll
        for (int b = 0; b < 4; b++) {
            const int j = b * 32 + (int)lane;
            if (j < w) {
                const int cls = clsv[b];
                const int mk = partner_mask(mode, cls);
                int part = -(int)partner_self(mode, cls);
#pragma unroll
                for (int c = 0; c < 4; c++)
                    if (mk & (1 << c)) part += cnt[c];
                if (part > 0) {
                    const int32_t id = (int32_t)(ev[b] >> 2);
                    if (!FILL) {
                        atomicAdd(&bound[id], (uint32_t)part);
                        atomicAdd(&mcount[id], 1u);
                    } else {
                        const uint32_t at = moff[id] + atomicAdd(&mcur[id], 1u);
                        memb[at] = MembRec{(uint32_t)u, (uint16_t)part, (uint16_t)j};
                    }
                }
            }
        }
    }
}

// Directed inserts: entry t of rows[] is a membership of weight 1, key t.
template <bool FILL>
__global__ void k_directed_memb(const int32_t *__restrict__ rows, int64_t m, uint32_t *mcount,
                                const uint32_t *__restrict__ moff, uint32_t *mcur, MembRec *memb) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = rows[i];
        if (!FILL) {
            atomicAdd(&mcount[r], 1u);
        } else {
            const uint32_t at = moff[r] + atomicAdd(&mcur[r], 1u);
            memb[at] = MembRec{(uint32_t)i, 1, 0};
        }
    }
}

// Per row: exclusive weighted rank of each membership by key (ascending
// hood / ordinal; keys are unique per row) -> start[out] = first slot of that
// membership in the row's bucket.  Warp per row: m <= 32 from registers (a
// shuffle loop), m <= SEG_SMEM by a shared-memory bitonic sort of
// (key << 32 | index) and a weighted exclusive scan; longer rows (hubs) go
// to a list ranked by k_seg_rank_heavy with a whole block per row.
// Rank a row's m <= 32 * NE memberships: keys sorted in registers, weights
// and output positions staged in shared memory, weighted exclusive scan.
template <int NE>
__device__ __forceinline__ uint32_t seg_rank_sorted(uint32_t lo, int m, const MembRec *__restrict__ memb,
                                                uint32_t *__restrict__ start, uint32_t *sw, uint32_t *so,
                                                unsigned lane, uint32_t wout) {
    uint64_t v[NE];
#pragma unroll
    for (int e = 0; e < NE; e++) {
        const int i = e * 32 + (int)lane;
        if (i < m) {
            const MembRec re = memb[lo + i];
            v[e] = ((uint64_t)re.key << 32) | (uint32_t)i;
            sw[i] = re.weight;
            so[i] = memb_out(re, wout);
        } else {
            v[e] = ~0ull;
        }
    }
    __syncwarp();
    warp_sort_reg<NE, uint64_t>(v, lane);
    uint32_t carry = 0;
#pragma unroll
    for (int e = 0; e < NE; e++) {
        const int i = e * 32 + (int)lane;
        const uint32_t idx = (uint32_t)v[e];
        const uint32_t w = i < m ? sw[idx] : 0u;
        uint32_t inc = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(FULL_MASK, inc, o);
            if ((int)lane >= o) inc += t;
        }
        if (i < m) start[so[idx]] = carry + inc - w;
        carry += __shfl_sync(FULL_MASK, inc, 31);
    }
    __syncwarp();
    return carry;  // the row's total weight
}

constexpr int SEG_WARPS = 8;
__global__ void __launch_bounds__(SEG_WARPS * 32)
k_seg_rank(int64_t n, const uint32_t *__restrict__ moff, const MembRec *__restrict__ memb,
           uint32_t *__restrict__ start, const unsigned long long *__restrict__ mpack,
           int32_t *heavy, unsigned long long *counters, uint32_t *__restrict__ total, uint32_t wout) {
    __shared__ uint32_t s_out[SEG_WARPS][SEG_SMEM];  // output positions of the sorted path
    __shared__ uint32_t s_wt[SEG_WARPS][SEG_SMEM];
    const unsigned lane = lane_id(), wib = threadIdx.x >> 5;
    const int64_t nw = (int64_t)gridDim.x * SEG_WARPS;
    // segment of row x: [moff[x], moff[x+1]) (compacted), or the fused
    // fixed-capacity segment of k_assemble (mpack[x] = base << 32 | count)
    auto seg = [&](int64_t x, uint32_t &a, uint32_t &b) {
        if (mpack) {
            const unsigned long long v = mpack[x];
            a = (uint32_t)(v >> 32);
            b = a + (uint32_t)v;
        } else {
            a = moff[x];
            b = moff[x + 1];
        }
    };
    // rows with m <= 32 memberships (almost all): one membership per lane in
    // registers; the next row's segment is loaded while the current one is
    // ranked (pipeline: offsets two rows ahead, records one row ahead)
    int64_t r = (int64_t)blockIdx.x * SEG_WARPS + wib;
    uint32_t lo1 = 0, hi1 = 0, lo2 = 0, hi2 = 0;
    MembRec rec1 = MembRec{0u, 0, 0};
    if (r < n) {
        seg(r, lo1, hi1);
        if (lane < hi1 - lo1) rec1 = ldcs_memb(memb + lo1 + lane);
    }
    if (r + nw < n) seg(r + nw, lo2, hi2);
    for (; r < n; r += nw) {
        const uint32_t lo = lo1;
        const int m = (int)(hi1 - lo1);
        const MembRec rec = rec1;
        lo1 = lo2;
        hi1 = hi2;
        rec1 = (r + nw < n && lane < hi1 - lo1) ? ldcs_memb(memb + lo1 + lane) : MembRec{0u, 0, 0};
        if (r + 2 * nw < n) seg(r + 2 * nw, lo2, hi2);
        if (m == 0) continue;
        if (m <= 32) {
            // keys (hood ids < 2^30, or chunk ordinals) fit 32 bits
            uint32_t acc = 0;
            const uint32_t key = (uint32_t)rec.key;
#pragma unroll 4
            for (int f = 0; f < m; f++) {
                const uint32_t kf = __shfl_sync(FULL_MASK, key, f);
                const uint32_t wf = __shfl_sync(FULL_MASK, rec.weight, f);
                acc += kf < key ? wf : 0u;
            }
            if ((int)lane < m) start[memb_out(rec, wout)] = acc;
            if (total) {
                const uint32_t t = __reduce_add_sync(FULL_MASK, (int)lane < m ? rec.weight : 0u);
                if (lane == 0) total[r] = t;
            }
            continue;
        }
        if (m <= 64) {
            // two memberships per lane, the same weighted count of smaller
            // keys (keys are unique within a row: hood ids / ordinals)
            const MembRec rb = (int)lane + 32 < m ? ldcs_memb(memb + lo + 32 + lane) : MembRec{~0u, 0, 0};
            uint32_t acc0 = 0, acc1 = 0;
            const uint32_t key0 = (uint32_t)rec.key, key1 = (uint32_t)rb.key;
#pragma unroll 4
            for (int f = 0; f < m; f++) {
                const uint32_t kk = f < 32 ? key0 : key1;
                const uint32_t ww = f < 32 ? rec.weight : rb.weight;
                const uint32_t kf = __shfl_sync(FULL_MASK, kk, f & 31);
                const uint32_t wf = __shfl_sync(FULL_MASK, ww, f & 31);
                acc0 += kf < key0 ? wf : 0u;
                acc1 += kf < key1 ? wf : 0u;
            }
            start[memb_out(rec, wout)] = acc0;
            if ((int)lane + 32 < m) start[memb_out(rb, wout)] = acc1;
            if (total) {
                const uint32_t t = __reduce_add_sync(FULL_MASK, rec.weight + rb.weight);
                if (lane == 0) total[r] = t;
            }
            continue;
        }
        if (m > SEG_SMEM) {  // hub row: ranked by a whole block later
            if (lane == 0) heavy[atomicAdd(&counters[C_SEGHEAVY], 1ull)] = (int32_t)r;
            continue;
        }
        // 64 < m <= SEG_SMEM: register bitonic sort of (key << 32 | index),
        // then the weights scanned in that order
        const uint32_t t = m <= 128
            ? seg_rank_sorted<4>(lo, m, memb, start, s_wt[wib], s_out[wib], lane, wout)
            : seg_rank_sorted<8>(lo, m, memb, start, s_wt[wib], s_out[wib], lane, wout);
        if (total && lane == 0) total[r] = t;
        __syncwarp();
    }
}

// Hub rows (> SEG_SMEM memberships): one block per row, keys staged in
// shared memory, rank = weighted count of smaller keys.  The row list and its
// length (counters[C_SEGHEAVY]) come from k_seg_rank: no host round trip.
constexpr int SEGH_THREADS = 256;
constexpr int SEGH_SMEM = 4096;  // keys staged in shared memory per block
__global__ void __launch_bounds__(SEGH_THREADS)
k_seg_rank_heavy(const uint32_t *__restrict__ moff, const MembRec *__restrict__ memb,
                 uint32_t *__restrict__ start, const unsigned long long *__restrict__ mpack,
                 const int32_t *__restrict__ heavy, const unsigned long long *__restrict__ counters,
                 uint32_t *__restrict__ total, uint32_t wout) {
    __shared__ uint64_t s_k[SEGH_SMEM];
    __shared__ uint32_t s_w[SEGH_SMEM];
    const int64_t nh = (int64_t)counters[C_SEGHEAVY];
    for (int64_t h = blockIdx.x; h < nh; h += gridDim.x) {
        const int64_t x = heavy[h];
        uint32_t lo, hi;
        if (mpack) {
            const unsigned long long v = mpack[x];
            lo = (uint32_t)(v >> 32);
            hi = lo + (uint32_t)v;
        } else {
            lo = moff[x];
            hi = moff[x + 1];
        }
        const int m = (int)(hi - lo);
        const int ms = m < SEGH_SMEM ? m : SEGH_SMEM;
        uint32_t part = 0;
        for (int e = threadIdx.x; e < m; e += blockDim.x) {
            const MembRec re = memb[lo + e];
            if (e < ms) {
                s_k[e] = re.key;
                s_w[e] = re.weight;
            }
            part += re.weight;
        }
        // row total (total[] is zero for rows ranked here: fused rounds
        // leave the bucket sizes to the ranking)
        if (total && part) atomicAdd(&total[x], part);
        __syncthreads();
        for (int e = threadIdx.x; e < m; e += blockDim.x) {
            const MembRec re = memb[lo + e];
            uint32_t acc = 0;
            for (int f = 0; f < ms; f++) acc += s_k[f] < re.key ? s_w[f] : 0u;
            for (int f = ms; f < m; f++) {
                const MembRec rf = memb[lo + f];
                acc += rf.key < re.key ? rf.weight : 0u;
            }
            start[memb_out(re, wout)] = acc;
        }
        __syncthreads();
    }
}


// pair_dists_dense (_kernels.py:113-119): exact reference distance of each
// (pa[i], pb[i]) pair of union rows, one thread per pair.
__global__ void k_pair_dists(const int32_t *__restrict__ pa, const int32_t *__restrict__ pb, int64_t m,
                             const float *__restrict__ sub, int dp, int d, int tag, double *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = exact_dist_tag(tag, sub + (int64_t)pa[i] * dp, sub + (int64_t)pb[i] * dp, d);
}

// on_pair capture: every admissible pair of every hood in (u, p, q) order.
__global__ void k_capture_pairs(const uint32_t *__restrict__ nbh, const int32_t *__restrict__ nlen,
                                int64_t lo, int64_t hi, int W, const int8_t *__restrict__ labels,
                                int mode, const uint64_t *__restrict__ poff, const float *sub,
                                int dp, int d, int tag, int32_t *pa, int32_t *pb, double *pd) {
    int64_t u = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= hi) return;
    uint64_t pos = poff[u];
    int w = nlen[u];
    for (int p = 0; p < w; p++) {
        uint32_t ep = nbh[u * W + p];
        for (int q = p + 1; q < w; q++) {
            uint32_t eq = nbh[u * W + q];
            int ip = ep >> 2, iq = eq >> 2;
            if (admissible(ep & 1, eq & 1, labels[ip], labels[iq], mode)) {
                pa[pos] = ip;
                pb[pos] = iq;
                pd[pos] = exact_dist_tag(tag, sub + (int64_t)ip * dp, sub + (int64_t)iq * dp, d);
                pos++;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Sequential per-row insertion in reference order (apply_updates_grouped's
// row loop, _kernels.py:248-254, each step _insert _kernels.py:159-192).
// One warp per row; the row's candidates are sorted by reference key first.
// ---------------------------------------------------------------------------
constexpr int APPLY_WARPS = 4;

// Stream row r's bucket slots [boff[r], boff[r+1]) in order: 32 distances per
// step (coalesced), candidates that cannot pass the current worst are
// skipped by ballot, the rest go through warp_insert in slot order -- which
// is the reference's sequential order, so no sorting is needed.
template <int E, int MODE, bool F32 = false>
__global__ void __launch_bounds__(APPLY_WARPS * 32, 6)
k_apply_stream(int64_t n, int k, const uint64_t *__restrict__ boff, const double *__restrict__ Bd,
               const int32_t *__restrict__ Bs, int32_t *ids, double *dists, uint8_t *flags,
               int32_t *sizes, unsigned long long *counters, LazyExact z, uint32_t gen) {
    // gen (packed slots only): the round's slot generation; a slot whose tag
    // differs was not written this round (0: NaN-prefilled format)
    constexpr bool LAZY = MODE == SLOTS_LAZY;
    __shared__ LazyBatchSmem s_lz[LAZY ? APPLY_WARPS : 1];
    const unsigned lane = lane_id(), wib = threadIdx.x >> 5;
    const int64_t nw = (int64_t)gridDim.x * APPLY_WARPS;
    unsigned long long acc = 0, slots = 0, written = 0, nexact = 0, rin = 0, rout = 0;
    for (int64_t r = (int64_t)blockIdx.x * APPLY_WARPS + wib; r < n; r += nw) {
        const uint64_t lo = boff[r];
        const int64_t ns = (int64_t)(boff[r + 1] - lo);
        if (ns == 0) continue;
        slots += (unsigned long long)ns;
        rin++;
        const double inf = __longlong_as_double(0x7ff0000000000000LL);
        // the next 32 slot distances are loaded while this chunk is applied
        // slots are read once: streaming loads keep L2 for the lists
        double dnext = (int64_t)lane < ns ? __ldcs(Bd + lo + lane) : inf;
        // F32: every list distance is an exact fp32 value (packed rounds on
        // certified data whose loaded lists passed the exactness check)
        using T = typename std::conditional<F32, float, double>::type;
        WarpRow<E, T> s;
        row_load<E, T>(s, ids, dists, flags, sizes, r, k, lane);
        int a = 0;
        uint32_t cpos = 0xffffffffu;  // lazy batch cache (slot index, exact value)
        double cval = 0.0;
        for (int64_t c0 = 0; c0 < ns; c0 += 32) {
            const int64_t j = c0 + lane;
            double dl = dnext;
            dnext = j + 32 < ns ? __ldcs(Bd + lo + j + 32) : inf;
            // an unwritten slot (NaN) belongs to a row that was full at round
            // start and a distance >= its worst: it can never pass
            int src;
            const int cnt = ns - c0 < 32 ? (int)(ns - c0) : 32;
            if constexpr (MODE == SLOTS_PACKED) {
                const unsigned long long v = __double_as_longlong(dl);
                const float f = __uint_as_float((uint32_t)(v >> 32));
                const bool wr = gen ? (((uint32_t)v >> 24) == gen) : (f == f);
                const T dt = wr ? (T)f : dist_inf<T>();
                if (j < ns && wr) written++;
                const bool pre = j < ns && (dt < s.worst || (s.sz < k && dt < dist_inf<T>()));
                if (!__any_sync(FULL_MASK, pre)) continue;
                src = gen ? (int)((uint32_t)v & 0xFFFFFFu) : (int)(uint32_t)v;
                a += warp_apply_chunk<E, T>(s, k, src, dt, cnt, lane);
            } else {
                if constexpr (LAZY) {
                    if (j < ns && dl == dl) written++;
                    bool need;
                    dl = lazy_resolve<E>(s, k, j < ns, dl, Bs, lo + j, z, src, need);
                    if (__any_sync(FULL_MASK, need))
                        lazy_chunk_eval<E>(s, k, z, r, Bd, Bs, lo, ns, c0, need, src, dl, cpos, cval, s_lz[wib],
                                           lane, nexact);
                    if (!__any_sync(FULL_MASK, dl < inf)) continue;
                } else {
                    if (dl != dl) dl = inf;
                    else if (j < ns) written++;
                    const bool pre = j < ns && (dl < s.worst || (s.sz < k && dl < inf));
                    if (!__any_sync(FULL_MASK, pre)) continue;
                    src = pre ? Bs[lo + j] : 0;
                }
                a += warp_apply_chunk<E, T>(s, k, src, dl, cnt, lane);
            }
        }
        if (a) {
            row_store<E, T>(s, ids, dists, flags, sizes, r, k, lane);
            rout++;
        }
        acc += a;
    }
    if (lane == 0 && acc) atomicAdd(&counters[C_ACCEPTED], acc);
    if (lane == 0 && slots) atomicAdd(&counters[C_CAND], slots);
    if (lane == 0 && rin) atomicAdd(&counters[C_ROWS_IN], rin);
    if (lane == 0 && rout) atomicAdd(&counters[C_ROWS_OUT], rout);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        written += __shfl_xor_sync(FULL_MASK, written, o);
        nexact += __shfl_xor_sync(FULL_MASK, nexact, o);
    }
    if (lane == 0 && written) atomicAdd(&counters[C_WRITTEN], written);
    if (lane == 0 && (nexact & ((1ull << 40) - 1))) atomicAdd(&counters[C_EXACT], nexact & ((1ull << 40) - 1));
    if (lane == 0 && (nexact >> 40)) atomicAdd(&counters[C_LZ_BATCHES], nexact >> 40);
}

// Written-slot compaction for the sharded exchange: an unwritten slot (NaN
// in its f64 view: the prefill, or all-ones when packed) can never be
// accepted.  One warp per row; written slots keep their order.
__global__ void k_slot_wcount(int64_t n, const uint64_t *__restrict__ boff, const double *__restrict__ Bd,
                              uint32_t *__restrict__ wcnt) {
    const unsigned lane = lane_id();
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += nw) {
        const uint64_t lo = boff[r], hi = boff[r + 1];
        uint32_t c = 0;
        for (uint64_t j = lo + lane; j - lane < hi; j += 32) {
            const double v = j < hi ? Bd[j] : __longlong_as_double(-1LL);
            c += __popc(__ballot_sync(FULL_MASK, v == v));
        }
        if (lane == 0) wcnt[r] = c;
    }
}

__global__ void k_slot_compact(int64_t n, const uint64_t *__restrict__ boff, const uint64_t *__restrict__ woff,
                               const double *__restrict__ Bd, const int32_t *__restrict__ Bs,
                               double *__restrict__ oBd, int32_t *__restrict__ oBs) {
    const unsigned lane = lane_id();
    const unsigned lt = lanemask_lt();
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += nw) {
        const uint64_t lo = boff[r], hi = boff[r + 1];
        uint64_t o = woff[r];
        for (uint64_t j = lo + lane; j - lane < hi; j += 32) {
            const double v = j < hi ? Bd[j] : __longlong_as_double(-1LL);
            const bool w = v == v;
            const unsigned m = __ballot_sync(FULL_MASK, w);
            if (w) {
                const uint64_t at = o + __popc(m & lt);
                oBd[at] = v;
                if (oBs) oBs[at] = Bs[j];
            }
            o += __popc(m);
        }
    }
}

// Round-start worst of every row (sharded rounds: the join needs the
// snapshot of rows owned by other ranks; lists are replicated).
__global__ void k_worst0_all(const int32_t *__restrict__ sizes, const double *__restrict__ dists,
                             int64_t n, int k, double *worst0) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x)
        worst0[r] = sizes[r] == k ? dists[r * k + k - 1] : __longlong_as_double(0x7ff0000000000000LL);
}

// Sharded rounds: row r (owned, r in [lo, lo+no)) receives one slot block per
// source rank; blocks are processed in source order, which is hood order,
// which is the reference's order.  off[s * (no+1) + i] = element offset of
// row lo+i's segment in the receive buffers.
template <int E, int MODE>
__global__ void __launch_bounds__(APPLY_WARPS * 32, 6)
k_apply_stream_multi(int64_t lo, int64_t no, int k, int nsrc, const uint64_t *__restrict__ off,
                     const uint32_t *__restrict__ cnt, const double *__restrict__ Bd,
                     const int32_t *__restrict__ Bs, int32_t *ids, double *dists, uint8_t *flags,
                     int32_t *sizes, unsigned long long *counters, LazyExact z,
                     uint8_t *dirty) {
    constexpr bool LAZY = MODE == SLOTS_LAZY;
    __shared__ LazyBatchSmem s_lz[LAZY ? APPLY_WARPS : 1];
    const unsigned lane = lane_id(), wib = threadIdx.x >> 5;
    const int64_t nw = (int64_t)gridDim.x * APPLY_WARPS;
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    unsigned long long acc = 0, nexact = 0;
    for (int64_t i = (int64_t)blockIdx.x * APPLY_WARPS + wib; i < no; i += nw) {
        const int64_t r = lo + i;
        bool any = false;
        for (int s = 0; s < nsrc && !any; s++) any = cnt[(int64_t)s * no + i] != 0;
        if (!any) continue;
        WarpRow<E> st;
        row_load<E>(st, ids, dists, flags, sizes, r, k, lane);
        int a = 0;
        for (int s = 0; s < nsrc; s++) {
            const uint64_t base = off[(int64_t)s * (no + 1) + i];
            const int64_t ns = cnt[(int64_t)s * no + i];
            uint32_t cpos = 0xffffffffu;  // lazy batch cache of this segment
            double cval = 0.0;
            for (int64_t c0 = 0; c0 < ns; c0 += 32) {
                const int64_t j = c0 + lane;
                double dl = j < ns ? Bd[base + j] : inf;
                int src;
                if (LAZY) {
                    bool need;
                    dl = lazy_resolve<E>(st, k, j < ns, dl, Bs, base + j, z, src, need);
                    if (__any_sync(FULL_MASK, need))
                        lazy_chunk_eval<E>(st, k, z, r, Bd, Bs, base, ns, c0, need, src, dl, cpos, cval,
                                           s_lz[wib], lane, nexact);
                    if (!__any_sync(FULL_MASK, dl < inf)) continue;
                } else if (MODE == SLOTS_PACKED) {
                    const unsigned long long v = __double_as_longlong(dl);
                    const float f = __uint_as_float((uint32_t)(v >> 32));
                    dl = f != f ? inf : (double)f;
                    const bool pre = j < ns && (dl < st.worst || (st.sz < k && dl < inf));
                    if (!__any_sync(FULL_MASK, pre)) continue;
                    src = (int)(uint32_t)v;
                } else {
                    if (dl != dl) dl = inf;
                    const bool pre = j < ns && (dl < st.worst || (st.sz < k && dl < inf));
                    if (!__any_sync(FULL_MASK, pre)) continue;
                    src = pre ? Bs[base + j] : 0;
                }
                const int c = ns - c0 < 32 ? (int)(ns - c0) : 32;
                a += warp_apply_chunk<E>(st, k, src, dl, c, lane);
            }
        }
        if (a) {
            row_store<E>(st, ids, dists, flags, sizes, r, k, lane);
            if (lane == 0) dirty[r] = 1;
        }
        acc += a;
    }
    if (lane == 0 && acc) atomicAdd(&counters[C_ACCEPTED], acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nexact += __shfl_xor_sync(FULL_MASK, nexact, o);
    if (lane == 0 && (nexact & ((1ull << 40) - 1))) atomicAdd(&counters[C_EXACT], nexact & ((1ull << 40) - 1));
    if (lane == 0 && (nexact >> 40)) atomicAdd(&counters[C_LZ_BATCHES], nexact >> 40);
}

// ---- replication of owned rows (sharded rounds) --------------------------
// A row record: f64 dists[k] | i32 ids[k] | i32 row | i32 size | u8 flags[k],
// padded to 8 bytes (row_rec_bytes).  Rows changed by a sharded round are
// the owned rows whose flags the assembly cleared (live: any flag set at
// round start) or that accepted an insert (dirty).
__host__ __device__ inline int row_rec_bytes(int k) { return (12 * k + 8 + k + 7) & ~7; }

__global__ void k_row_select(int64_t lo, int64_t no, int all, const uint8_t *__restrict__ live,
                             const uint8_t *__restrict__ dirty, uint32_t *sel) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < no;
         i += (int64_t)gridDim.x * blockDim.x)
        sel[i] = (all || live[lo + i] || dirty[lo + i]) ? 1u : 0u;
}

// one warp per selected row: coalesced row reads, record writes
__global__ void k_pack_rows(int64_t lo, int64_t no, int k, const uint32_t *__restrict__ sel,
                            const uint64_t *__restrict__ soff, const int32_t *__restrict__ ids,
                            const double *__restrict__ dists, const uint8_t *__restrict__ flags,
                            const int32_t *__restrict__ sizes, uint8_t *out) {
    const unsigned lane = lane_id();
    const int rb = row_rec_bytes(k);
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < no; i += nw) {
        if (!sel[i]) continue;
        const int64_t r = lo + i;
        uint8_t *rec = out + (size_t)soff[i] * rb;
        double *d = (double *)rec;
        int32_t *id = (int32_t *)(rec + 8 * (size_t)k);
        for (int t = lane; t < k; t += 32) {
            d[t] = dists[r * k + t];
            id[t] = ids[r * k + t];
            rec[12 * k + 8 + t] = flags[r * k + t];
        }
        if (lane == 0) {
            id[k] = (int32_t)r;
            id[k + 1] = sizes[r];
        }
    }
}

__global__ void k_unpack_rows(int64_t count, int k, const uint8_t *__restrict__ in, int32_t *ids,
                              double *dists, uint8_t *flags, int32_t *sizes) {
    const unsigned lane = lane_id();
    const int rb = row_rec_bytes(k);
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < count; i += nw) {
        const uint8_t *rec = in + (size_t)i * rb;
        const double *d = (const double *)rec;
        const int32_t *id = (const int32_t *)(rec + 8 * (size_t)k);
        const int64_t r = id[k];
        for (int t = lane; t < k; t += 32) {
            dists[r * k + t] = d[t];
            ids[r * k + t] = id[t];
            flags[r * k + t] = rec[12 * k + 8 + t];
        }
        if (lane == 0) sizes[r] = id[k + 1];
    }
}

__global__ void k_add_base(uint64_t *off, int64_t m, uint64_t base) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
        off[i] += base;
}

// ---------------------------------------------------------------------------
// Exact brute force (construct.py:273-348, _kernels.py:445-506).  The
// reference inserts candidates in ascending id order, so its lists are the
// top-k by (dist, id) with exact fp64 distances -- any evaluation order that
// keeps (dist, id) order gives the same lists.  One block per query; each
// thread keeps a sorted top-k of its strided share, then the block merges
// with k rounds of (dist, id) arg-min.
// ---------------------------------------------------------------------------
constexpr int BF_THREADS = 256;
constexpr int BF_MAXK = 64;

__device__ __forceinline__ bool dist_id_less(double d1, int32_t i1, double d2, int32_t i2) {
    return d1 < d2 || (d1 == d2 && i1 < i2);
}

template <int TAG>
__global__ void __launch_bounds__(BF_THREADS)
k_bf_topk(const float *__restrict__ data, int64_t n, int dp, int d, const float *__restrict__ queries,
          int qdp, const int64_t *__restrict__ qrows, int64_t nq, int k, int exclude_self,
          int32_t *out_ids, double *out_dists) {
    extern __shared__ double bf_sm[];  // q (dp doubles, unused) + BF_THREADS * k candidates
    double *cd = bf_sm;
    int32_t *ci = reinterpret_cast<int32_t *>(bf_sm + (size_t)BF_THREADS * k);
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    for (int64_t qi = blockIdx.x; qi < nq; qi += gridDim.x) {
        const float *q = qrows ? data + qrows[qi] * dp : queries + qi * qdp;
        const int64_t self = (qrows && exclude_self) ? qrows[qi] : -1;
        double td[BF_MAXK];
        int32_t ti[BF_MAXK];
        for (int t = 0; t < k; t++) { td[t] = inf; ti[t] = 0x7fffffff; }
        for (int64_t i = threadIdx.x; i < n; i += BF_THREADS) {
            if (i == self) continue;
            const double dd = exact_dist<TAG>(q, data + i * dp, d);
            if (!dist_id_less(dd, (int32_t)i, td[k - 1], ti[k - 1])) continue;
            int t = k - 1;
            while (t > 0 && dist_id_less(dd, (int32_t)i, td[t - 1], ti[t - 1])) {
                td[t] = td[t - 1];
                ti[t] = ti[t - 1];
                t--;
            }
            td[t] = dd;
            ti[t] = (int32_t)i;
        }
        for (int t = 0; t < k; t++) {
            cd[threadIdx.x * k + t] = td[t];
            ci[threadIdx.x * k + t] = ti[t];
        }
        __syncthreads();
        // k rounds of block arg-min over the per-thread heads
        __shared__ double s_bd[BF_THREADS / 32];
        __shared__ int32_t s_bi[BF_THREADS / 32];
        __shared__ int s_bt[BF_THREADS / 32];
        __shared__ int s_win;
        int head = 0;  // next unused entry of this thread's list
        for (int r = 0; r < k; r++) {
            double bd = head < k ? cd[threadIdx.x * k + head] : inf;
            int32_t bi = head < k ? ci[threadIdx.x * k + head] : 0x7fffffff;
            int bt = threadIdx.x;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double od = __shfl_xor_sync(FULL_MASK, bd, o);
                const int32_t oi = __shfl_xor_sync(FULL_MASK, bi, o);
                const int ot = __shfl_xor_sync(FULL_MASK, bt, o);
                if (dist_id_less(od, oi, bd, bi)) { bd = od; bi = oi; bt = ot; }
            }
            if ((threadIdx.x & 31) == 0) {
                s_bd[threadIdx.x >> 5] = bd;
                s_bi[threadIdx.x >> 5] = bi;
                s_bt[threadIdx.x >> 5] = bt;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                int w = 0;
                for (int x = 1; x < BF_THREADS / 32; x++)
                    if (dist_id_less(s_bd[x], s_bi[x], s_bd[w], s_bi[w])) w = x;
                s_win = s_bt[w];
                const bool real = s_bd[w] < inf;
                out_ids[qi * k + r] = real ? s_bi[w] : -1;
                out_dists[qi * k + r] = s_bd[w];
            }
            __syncthreads();
            if ((int)threadIdx.x == s_win) head++;
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------------------
// phi (construct.py:79-83) with numpy's pairwise summation tree.
// ---------------------------------------------------------------------------
__global__ void k_phi_leaves(const double *__restrict__ dists, const int32_t *__restrict__ sizes, int k,
                             const int64_t *__restrict__ leaf_lo, const int32_t *__restrict__ leaf_len,
                             int64_t nleaves, double *out) {
    int64_t li = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (li >= nleaves) return;
    int64_t lo = leaf_lo[li];
    int n = leaf_len[li];
    // elements are visited in index order: (row, slot) advance incrementally
    // (no division per element)
    int64_t u = lo / k;
    int t = (int)(lo - u * k);
    int sz = sizes[u];
    int64_t e = lo;
    auto next = [&]() -> double {
        const double v = t < sz ? dists[e] : 0.0;
        e++;
        if (++t == k) {
            t = 0;
            u++;
            sz = e < lo + n ? sizes[u] : 0;
        }
        return v;
    };
    double res;
    if (n < 8) {
        res = 0.0;
        for (int i = 0; i < n; i++) res = __dadd_rn(res, next());
    } else {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; j++) r[j] = next();
        int i;
        for (i = 8; i < n - (n % 8); i += 8) {
#pragma unroll
            for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], next());
        }
        res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                        __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n; i++) res = __dadd_rn(res, next());
    }
    out[li] = res;
}

// One tree level (nodes [lo, hi) of the height-sorted node array).
__global__ void k_phi_level(const int32_t *__restrict__ left, const int32_t *__restrict__ right,
                            int lo, int hi, const double *__restrict__ leaves, double *inner) {
    const int i = lo + blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hi) return;
    const int l = left[i], r = right[i];
    const double a = l >= 0 ? inner[l] : leaves[-l - 1];
    const double b = r >= 0 ? inner[r] : leaves[-r - 1];
    inner[i] = __dadd_rn(a, b);
}

// Internal nodes sorted by height; ref >= 0 -> internal node, ref < 0 -> leaf (-ref-1).
__global__ void k_phi_tree(const int32_t *__restrict__ left, const int32_t *__restrict__ right,
                           const int32_t *__restrict__ level_start, int nlevels,
                           const double *__restrict__ leaves, double *inner) {
    for (int h = 0; h < nlevels; h++) {
        for (int i = level_start[h] + threadIdx.x; i < level_start[h + 1]; i += blockDim.x) {
            int l = left[i], r = right[i];
            double a = l >= 0 ? inner[l] : leaves[-l - 1];
            double b = r >= 0 ? inner[r] : leaves[-r - 1];
            inner[i] = __dadd_rn(a, b);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Export (construct.py:212-223) and rear merge (_kernels.py:529-563).
// ---------------------------------------------------------------------------
__global__ void k_export(const int32_t *__restrict__ ids, const int64_t *__restrict__ ug, int64_t total,
                         int32_t *out_ids) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t v = ids[i];
        out_ids[i] = v >= 0 ? (ug ? (int32_t)ug[v] : v) : -1;
    }
}

// One thread per row, MR_ROWS rows per block: the block's U rows, rear rows
// and outputs are staged in shared memory with coalesced copies (a thread
// walking its own rows in global memory touched a new sector per element).
constexpr int MR_ROWS = 64;

__host__ __device__ constexpr size_t mr_smem_bytes(int k, int rk) {
    return (size_t)MR_ROWS * (size_t)(2 * k + rk) * (sizeof(double) + sizeof(int32_t));
}

__global__ void __launch_bounds__(MR_ROWS)
k_merge_rear(const int32_t *__restrict__ ui, const double *__restrict__ ud,
             const int32_t *__restrict__ us, const int32_t *__restrict__ ri,
             const double *__restrict__ rd, const int32_t *__restrict__ rs, int64_t n,
             int k, int rk, int32_t *oi, double *od, int32_t *os) {
    extern __shared__ __align__(16) char mr_smem[];
    const int64_t r0 = (int64_t)blockIdx.x * MR_ROWS;
    const int nr = (int)((n - r0) < MR_ROWS ? (n - r0) : MR_ROWS);
    double *sad = reinterpret_cast<double *>(mr_smem);      // [MR_ROWS][k]
    double *sbd = sad + MR_ROWS * k;                         // [MR_ROWS][rk]
    double *sod = sbd + MR_ROWS * rk;                        // [MR_ROWS][k]
    int32_t *sai = reinterpret_cast<int32_t *>(sod + MR_ROWS * k);
    int32_t *sbi = sai + MR_ROWS * k;
    int32_t *soi = sbi + MR_ROWS * rk;
    // coalesced staging of the block's rows (contiguous in global memory)
    for (int e = threadIdx.x; e < nr * k; e += MR_ROWS) {
        sad[e] = ud[r0 * k + e];
        sai[e] = ui[r0 * k + e];
    }
    for (int e = threadIdx.x; e < nr * rk; e += MR_ROWS) {
        sbd[e] = rd[r0 * rk + e];
        sbi[e] = ri[r0 * rk + e];
    }
    __syncthreads();
    const int lr = threadIdx.x;
    if (lr < nr) {
        const int64_t u = r0 + lr;
        const int32_t *a_i = sai + lr * k;
        const double *a_d = sad + lr * k;
        const int32_t *b_i = sbi + lr * rk;
        const double *b_d = sbd + lr * rk;
        int32_t *o_i = soi + lr * k;
        double *o_d = sod + lr * k;
        // graph.py:259-280 / _kernels.py:529-563: (dist, id) merge, U first
        // on ties, ids already output skipped, at most k kept
        int a = 0, b = 0, w = 0, na = us[u], nb = rs[u];
        while (w < k && (a < na || b < nb)) {
            int32_t cid;
            double cd;
            if (a < na && (b >= nb || a_d[a] < b_d[b] || (a_d[a] == b_d[b] && a_i[a] <= b_i[b]))) {
                cid = a_i[a];
                cd = a_d[a];
                a++;
            } else {
                cid = b_i[b];
                cd = b_d[b];
                b++;
            }
            bool dup = false;
            for (int t = 0; t < w; t++)
                if (o_i[t] == cid) { dup = true; break; }
            if (!dup) {
                o_i[w] = cid;
                o_d[w] = cd;
                w++;
            }
        }
        for (int t = w; t < k; t++) {
            o_i[t] = -1;
            o_d[t] = __longlong_as_double(0x7ff0000000000000LL);
        }
        os[u] = w;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nr * k; e += MR_ROWS) {
        od[r0 * k + e] = sod[e];
        oi[r0 * k + e] = soi[e];
    }
}

}  // namespace knnm

// knnm_device.cuh -- device helpers shared by the knnm kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define FULL_MASK 0xffffffffu

// Device-side bounds checks of the debug build (-DKNNM_DEBUG; compute-sanitizer
// is not available on the GPU pool): a failed check traps with its line.
#ifdef KNNM_DEBUG
#include <cassert>
#define KNNM_CHECK(cond) assert(cond)
#else
#define KNNM_CHECK(cond) ((void)0)
#endif

namespace knnm {

constexpr uint64_t U64_GAMMA = 0x9E3779B97F4A7C15ULL;  // _kernels.py:33
constexpr uint64_t U64_MIX1 = 0xBF58476D1CE4E5B9ULL;   // _kernels.py:34
constexpr uint64_t U64_MIX2 = 0x94D049BB133111EBULL;   // _kernels.py:35

// Indices into the per-context device counter block.
enum Counter {
    C_CAND = 0,       // candidate records emitted (directed updates)
    C_ACCEPTED = 1,   // accepted insertions
    C_ACTIVE = 2,     // active hoods (>= 1 admissible pair)
    C_HEAVY_REV = 3,  // vertices whose reverse segment needs block selection
    C_MAXDEG = 4,     // max reverse degree among heavy vertices
    C_MEMBERS = 5,    // sum |M_u| over hoods
    C_HEAVY_APPLY = 6,// rows with more candidates than the warp path holds
    C_GIANT_APPLY = 7,// rows with more candidates than the block smem path holds
    C_OVERFLOW = 8,   // candidate buffer overflow (must stay 0)
    C_EXACT = 9,      // pairs re-evaluated in fp64 after the fp32 screen
    C_MAXC = 10,      // max candidates on a giant row
    C_WRITTEN = 11,   // update slots written by the join (prefilter survivors)
    C_SEGHEAVY = 12,  // rows with > SEG_SMEM memberships (block-ranked)
    C_GIANT = 13,     // heavy rows whose reverse segment exceeds a block's smem
    C_DUPROWS = 14,   // rows given twice to a row-grouped insert (direct path check)
    C_ROWS_IN = 15,   // rows the apply loaded (>= 1 slot)
    C_ROWS_OUT = 16,  // rows the apply stored (>= 1 accepted insert)
    C_LZ_BATCHES = 17,// lazy exact-evaluation batches (folds of up to 32 pairs)
    C_NUM = 20
};

// splitmix64 output for a state that was already advanced (_kernels.py:306-313).
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * U64_MIX1;
    z = (z ^ (z >> 27)) * U64_MIX2;
    return z ^ (z >> 31);
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__host__ __device__ __forceinline__ uint32_t next_pow2(uint32_t x) {
    uint32_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

// ---------------------------------------------------------------------------
// Exact metric (_kernels.py:43-80): fp64 accumulation of fp32 inputs, strictly
// sequential, no contraction (explicit _rn intrinsics are never fused).
// ---------------------------------------------------------------------------
template <int TAG>
__device__ __forceinline__ double exact_dist(const float *__restrict__ a,
                                             const float *__restrict__ b, int d) {
    if (TAG == 1) {
        double acc = 0.0;
        for (int t = 0; t < d; t++) {
            double df = __dsub_rn((double)a[t], (double)b[t]);
            acc = __dadd_rn(acc, __dmul_rn(df, df));
        }
        return acc;
    } else if (TAG == 0) {
        double acc = 0.0;
        for (int t = 0; t < d; t++) acc = __dadd_rn(acc, fabs(__dsub_rn((double)a[t], (double)b[t])));
        return acc;
    } else {
        double dot = 0.0, na = 0.0, nb = 0.0;
        for (int t = 0; t < d; t++) {
            double x = (double)a[t], y = (double)b[t];
            dot = __dadd_rn(dot, __dmul_rn(x, y));
            na = __dadd_rn(na, __dmul_rn(x, x));
            nb = __dadd_rn(nb, __dmul_rn(y, y));
        }
        if (na == 0.0 || nb == 0.0) return (na == nb) ? 0.0 : 1.0;
        if (dot > 0.0 && __dmul_rn(dot, dot) >= __dmul_rn(na, nb)) return 0.0;
        double r = __dsub_rn(1.0, __ddiv_rn(dot, __dmul_rn(__dsqrt_rn(na), __dsqrt_rn(nb))));
        return r < 0.0 ? 0.0 : r;
    }
}

// Cosine with the two fp64 norms precomputed: the reference accumulates
// na = sum x*x and nb = sum y*y in the same sequential loop as the dot
// (_kernels.py:65-70); each depends only on its own vector, so computing them
// once per vector gives the same bits.  Post-processing as _kernels.py:71-80.
__device__ __forceinline__ double exact_cos_norms(const float *__restrict__ a, const float *__restrict__ b,
                                                  int d, double na, double nb) {
    double dot = 0.0;
    for (int t = 0; t < d; t++) dot = __dadd_rn(dot, __dmul_rn((double)a[t], (double)b[t]));
    if (na == 0.0 || nb == 0.0) return (na == nb) ? 0.0 : 1.0;
    if (dot > 0.0 && __dmul_rn(dot, dot) >= __dmul_rn(na, nb)) return 0.0;
    double r = __dsub_rn(1.0, __ddiv_rn(dot, __dmul_rn(__dsqrt_rn(na), __dsqrt_rn(nb))));
    return r < 0.0 ? 0.0 : r;
}

// One step of the exact reference sums (_kernels.py:43-80): acc + term(x, y)
// with the reference's fp64 roundings (cosine: the dot; norms precomputed).
// The same step with x already in fp64 (exactly (double) of an fp32 value).
template <int TAG>
__device__ __forceinline__ double exact_term_d(double acc, double x, float y) {
    if (TAG == 1) {
        const double df = __dsub_rn(x, (double)y);
        return __dadd_rn(acc, __dmul_rn(df, df));
    }
    if (TAG == 0) return __dadd_rn(acc, fabs(__dsub_rn(x, (double)y)));
    return __dadd_rn(acc, __dmul_rn(x, (double)y));
}

template <int TAG>
__device__ __forceinline__ double exact_term(double acc, float x, float y) {
    if (TAG == 1) {
        const double df = __dsub_rn((double)x, (double)y);
        return __dadd_rn(acc, __dmul_rn(df, df));
    }
    if (TAG == 0) return __dadd_rn(acc, fabs(__dsub_rn((double)x, (double)y)));
    return __dadd_rn(acc, __dmul_rn((double)x, (double)y));  // dot (norms precomputed)
}

__device__ __forceinline__ double exact_sqnorm(const float *__restrict__ a, int d) {
    double acc = 0.0;
    for (int t = 0; t < d; t++) {
        const double x = (double)a[t];
        acc = __dadd_rn(acc, __dmul_rn(x, x));
    }
    return acc;
}

__device__ __forceinline__ double cos_finish(double dot, double na, double nb) {
    if (na == 0.0 || nb == 0.0) return (na == nb) ? 0.0 : 1.0;
    if (dot > 0.0 && __dmul_rn(dot, dot) >= __dmul_rn(na, nb)) return 0.0;
    double r = __dsub_rn(1.0, __ddiv_rn(dot, __dmul_rn(__dsqrt_rn(na), __dsqrt_rn(nb))));
    return r < 0.0 ? 0.0 : r;
}

__device__ __forceinline__ double exact_dist_tag(int tag, const float *a, const float *b, int d) {
    if (tag == 1) return exact_dist<1>(a, b, d);
    if (tag == 2) return exact_dist<2>(a, b, d);
    return exact_dist<0>(a, b, d);
}

// ---------------------------------------------------------------------------
// Bitonic sorts over shared (or global) arrays of power-of-two length.
// Group = one warp (sync = __syncwarp) or one block (sync = __syncthreads).
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void bitonic_warp(T *a, uint32_t P2, unsigned lane) {
    for (uint32_t k2 = 2; k2 <= P2; k2 <<= 1) {
        for (uint32_t j = k2 >> 1; j > 0; j >>= 1) {
            for (uint32_t i = lane; i < P2; i += 32) {
                uint32_t ixj = i ^ j;
                if (ixj > i) {
                    T x = a[i], y = a[ixj];
                    bool asc = (i & k2) == 0;
                    if ((x > y) == asc) { a[i] = y; a[ixj] = x; }
                }
            }
            __syncwarp();
        }
    }
}

template <typename T>
__device__ __forceinline__ void bitonic_block(T *a, uint32_t P2) {
    for (uint32_t k2 = 2; k2 <= P2; k2 <<= 1) {
        for (uint32_t j = k2 >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < P2; i += blockDim.x) {
                uint32_t ixj = i ^ j;
                if (ixj > i) {
                    T x = a[i], y = a[ixj];
                    bool asc = (i & k2) == 0;
                    if ((x > y) == asc) { a[i] = y; a[ixj] = x; }
                }
            }
            __syncthreads();
        }
    }
}

// Register bitonic sort of one u64 per lane (ascending by lane).
__device__ __forceinline__ uint64_t bitonic_reg32(uint64_t v, unsigned lane) {
#pragma unroll
    for (int k2 = 2; k2 <= 32; k2 <<= 1) {
#pragma unroll
        for (int j = k2 >> 1; j > 0; j >>= 1) {
            uint64_t o = __shfl_xor_sync(FULL_MASK, v, j);
            bool up = (lane & k2) == 0;
            bool lower = (lane & j) == 0;
            uint64_t mn = v < o ? v : o, mx = v < o ? o : v;
            v = (lower == up) ? mn : mx;
        }
    }
    return v;
}

// Register bitonic sort of NE keys per lane; element index i = e * 32 + lane,
// ascending in i afterwards.  Cross-lane stages use shuffles, in-lane stages
// plain register swaps (no shared memory, no barriers).
template <int NE, typename T = uint64_t>
__device__ __forceinline__ void warp_sort_reg(T (&v)[NE], unsigned lane) {
#pragma unroll
    for (int k2 = 2; k2 <= 32 * NE; k2 <<= 1) {
#pragma unroll
        for (int j = k2 >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
                const int je = j >> 5;
#pragma unroll
                for (int e = 0; e < NE; e++) {
                    if ((e & je) == 0) {
                        const int f = e | je;
                        const bool asc = (((e * 32 + (int)lane) & k2) == 0);
                        T x = v[e], y = v[f];
                        if ((x > y) == asc) { v[e] = y; v[f] = x; }
                    }
                }
            } else {
#pragma unroll
                for (int e = 0; e < NE; e++) {
                    T o = __shfl_xor_sync(FULL_MASK, v[e], j);
                    const bool asc = (((e * 32 + (int)lane) & k2) == 0);
                    const bool lower = (lane & j) == 0;
                    T mn = v[e] < o ? v[e] : o, mx = v[e] < o ? o : v[e];
                    v[e] = (lower == asc) ? mn : mx;
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// One row of the k-NN state held by a warp: entry t = e*32 + lane.
// warp_insert() is _insert (_kernels.py:159-192) executed cooperatively.
// ---------------------------------------------------------------------------
// T = double, or float when every distance of the row is exactly an fp32
// value (certified data: integers below 2^24) -- half the shuffle traffic.
template <int E, typename T = double>
struct WarpRow {
    int idf[E];  // (id << 1) | new-flag: one register moves both (ids < 2^30)
    T d[E];
    int sz;
    T worst;  // dists[k-1] when sz == k
};

template <typename T>
__device__ __forceinline__ T dist_inf() {
    return (T)__longlong_as_double(0x7ff0000000000000LL);
}

template <int E, typename T>
__device__ __forceinline__ void row_load(WarpRow<E, T> &s, const int32_t *ids, const double *dists,
                                         const uint8_t *flags, const int32_t *sizes, int64_t r,
                                         int k, unsigned lane) {
#pragma unroll
    for (int e = 0; e < E; e++) {
        int t = e * 32 + lane;
        if (t < k) {
            s.idf[e] = (int)((uint32_t)ids[r * k + t] << 1) | (flags[r * k + t] & 1);
            s.d[e] = (T)dists[r * k + t];
        } else {
            s.idf[e] = -2;  // id -1, flag 0
            s.d[e] = dist_inf<T>();
        }
    }
    s.sz = sizes[r];
    s.worst = (T)0;
#pragma unroll
    for (int e = 0; e < E; e++)
        if (e == ((k - 1) >> 5)) s.worst = __shfl_sync(FULL_MASK, s.d[e], (k - 1) & 31);
}

template <int E, typename T>
__device__ __forceinline__ void row_store(const WarpRow<E, T> &s, int32_t *ids, double *dists,
                                          uint8_t *flags, int32_t *sizes, int64_t r, int k,
                                          unsigned lane) {
#pragma unroll
    for (int e = 0; e < E; e++) {
        int t = e * 32 + lane;
        if (t < k) {
            ids[r * k + t] = s.idf[e] >> 1;  // arithmetic: -2 -> -1
            dists[r * k + t] = (double)s.d[e];
            flags[r * k + t] = (uint8_t)(s.idf[e] & 1);
        }
    }
    if (lane == 0) sizes[r] = s.sz;
}

// Returns 1 (warp-uniform) when the candidate is accepted.  CHECK = false
// when the caller already knows the row is not full or nd < worst.
template <int E, bool CHECK = true, typename T = double>
__device__ __forceinline__ int warp_insert(WarpRow<E, T> &s, int k, int src, T nd, unsigned lane) {
    if (CHECK && s.sz == k && nd >= s.worst) return 0;
    // duplicate test and insertion point in one pass over the entries
    bool dup = false;
    int pos = s.sz;
#pragma unroll
    for (int e = E - 1; e >= 0; e--) {
        const int t = e * 32 + lane;
        const int id = s.idf[e] >> 1;
        const bool in = t < s.sz;
        dup |= in && id == src;
        const bool before = in && (nd < s.d[e] || (nd == s.d[e] && src < id));
        const unsigned b = __ballot_sync(FULL_MASK, before);
        if (b) pos = e * 32 + __ffs(b) - 1;
    }
    if (__any_sync(FULL_MASK, dup)) return 0;
    int last;
    if (s.sz == k) {
        last = k - 1;
    } else {
        last = s.sz;
        s.sz += 1;
    }
#pragma unroll
    for (int e = E - 1; e >= 0; e--) {
        int up_i = __shfl_up_sync(FULL_MASK, s.idf[e], 1);
        T up_d = __shfl_up_sync(FULL_MASK, s.d[e], 1);
        if (e > 0) {
            const int pi = __shfl_sync(FULL_MASK, s.idf[e > 0 ? e - 1 : 0], 31);
            const T pd = __shfl_sync(FULL_MASK, s.d[e > 0 ? e - 1 : 0], 31);
            if (lane == 0) { up_i = pi; up_d = pd; }
        }
        const int t = e * 32 + lane;
        if (t > pos && t <= last) { s.idf[e] = up_i; s.d[e] = up_d; }
        if (t == pos) { s.idf[e] = (int)((uint32_t)src << 1) | 1; s.d[e] = nd; }
    }
    if (s.sz == k) {
#pragma unroll
        for (int e = 0; e < E; e++)
            if (e == ((k - 1) >> 5)) s.worst = __shfl_sync(FULL_MASK, s.d[e], (k - 1) & 31);
    }
    return 1;
}

// ---------------------------------------------------------------------------
// Lazy exact evaluation (non-certified datasets).  The tiled join stores the
// fp32 screen value f of a pair with the sign bit set ("approximate"); the
// apply resolves it to the reference's fp64 value only when its rigorous
// lower bound can still beat the row's current worst.  Decisions are always
// taken on exact values, so the outcome is the reference's.
//   L2 / L1 : exact >= f * lo_rel    (|f / exact - 1| <= (d + 8) 2^-23)
//   cosine  : exact >= f - lo_abs    (|f - exact| <= (4 d + 64) 2^-24)
// ---------------------------------------------------------------------------
struct LazyExact {
    int64_t nrows;        // rows of sub (bounds checks of the debug build)
    int ahead;            // look-ahead chunks of a speculative batch (lazy_chunk_eval)
    const float *sub;     // subset rows, dp floats each (zero padded)
    const double *nrm64;  // exact fp64 squared norms per row (cosine only)
    int dp, d, tag;
    double lo_rel, lo_abs;
    // estimate of the exact value from above, f * hi_rel + hi_abs: only
    // steers the speculation of lazy_chunk_eval (a slot it leaves out is
    // evaluated on demand), so it need not be rigorous
    double hi_rel, hi_abs;
};

__device__ __forceinline__ bool slot_is_approx(double v) { return __double_as_longlong(v) < 0; }

__device__ __forceinline__ double slot_lower(double v, const LazyExact z) {
    const double f = -v;
    return z.tag == 2 ? f - z.lo_abs : f * z.lo_rel;
}
__device__ __forceinline__ double slot_upper(double v, const LazyExact z) { return -v * z.hi_rel + z.hi_abs; }

// Resolve the lane's slot for row r: returns the distance to apply (+inf when
// the slot cannot pass the row's current state).  need = approximate slot
// whose lower bound beats the current worst: its exact value must be
// computed (lazy_chunk_eval) before the chunk is applied.
template <int E>
__device__ __forceinline__ double lazy_resolve(const WarpRow<E> &s, int k, bool in, double dl,
                                               const int32_t *__restrict__ Bs, uint64_t pos,
                                               const LazyExact z, int &src, bool &need) {
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    if (dl != dl) dl = inf;  // unwritten slot
    const bool apx = z.sub && in && slot_is_approx(dl);
    const double lb = apx ? slot_lower(dl, z) : dl;
    const bool pre = in && (lb < s.worst || (s.sz < k && lb < inf));
    src = pre ? Bs[pos] : 0;
    need = pre && apx;
    if (__any_sync(FULL_MASK, need)) {
        // a candidate already in the list is rejected whatever its distance
        // (_kernels.py insertion: worst test, then duplicate test): no exact
        // evaluation for it
#pragma unroll
        for (int e = 0; e < E; e++)
            for (int t = 0; t < 32; t++) {
                const int id = __shfl_sync(FULL_MASK, s.idf[e], t) >> 1;
                if (e * 32 + t < s.sz && id == src) need = false;
            }
    }
    if (!pre || apx) return inf;  // approximate: replaced by the exact value if needed
    return dl;
}

// ---------------------------------------------------------------------------
// Batched speculative lazy evaluation.  The sequential fold of one exact
// value is a chain of d dependent fp64 adds, so a warp is only busy when many
// pairs fold at once: when a chunk of a row needs exact values, the warp also
// takes, from the next LZB_AHEAD chunks of the same slot segment, every
// approximate slot that could pass the row's current state (lower bound below
// the current worst, id not listed) -- up to 32 pairs -- and folds all of them
// together, one pair per lane.  The values are kept in a per-lane cache keyed
// by slot index and handed out when their chunks come up.  The decisions are
// unchanged (they are still taken on exact values at each slot's turn); a
// speculative value that is never asked for is wasted work only.
// ---------------------------------------------------------------------------
constexpr int LZB_AHEAD = 32;  // chunks of look-ahead per batch (default of LazyExact::ahead; with the
                               // simulated-worst filter 16 / 24 / 32 / 48 measure 276 / 272 / 273 / 270 ms at config 3)

struct __align__(16) LazyBatchSmem {
    // y[buf][j * 32 + 4 * (g ^ (j & 7)) + e]: dimension t0 + 4 g + e of pair
    // j's candidate row (16-byte groups XOR-swizzled by row: a warp's float4
    // reads of one group from 32 rows are conflict-free per quarter-warp)
    float y[2][32 * 32];
    float x[2][32];     // the row's own dimensions t0 .. t0 + 31
    double xd[32];      // the same in fp64 (one conversion per dimension, not per pair)
    int sid[32];        // candidate row of pair j
    uint32_t spos[32];  // slot index (within the row's segment) of pair j
};

__device__ __forceinline__ void cp_async16(float *dst, const float *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}

// Exact values of batch pairs 0 .. P-1 (row r against b.sid[j]); lane j
// folds pair j.  The 32-dimension blocks of the rows are staged by 16-byte
// cp.async copies (a warp instruction moves one block of four rows) into two
// buffers: block t + 1 is in flight while block t is folded.
template <int TAG>
__device__ __noinline__ double lazy_batch_t(const LazyExact z, int64_t r, int P, LazyBatchSmem &b, unsigned lane) {
    const float *ra = z.sub + r * z.dp;
    const int my = (int)lane < P ? b.sid[lane] : 0;
    KNNM_CHECK(P >= 1 && P <= 32 && r >= 0 && r < z.nrows && my >= 0 && my < z.nrows);
    const int nblk = (z.d + 31) >> 5;
    const int g = (int)(lane & 7);
    auto issue = [&](int blk) {
        const int t0 = blk * 32, buf = blk & 1;
        // chunk c = i * 32 + lane: row c >> 3, group c & 7 (= lane & 7)
        if (t0 + 4 * g < z.dp) {
            if (lane < 8) cp_async16(&b.x[buf][4 * g], ra + t0 + 4 * g);
            for (int j = (int)(lane >> 3); j < P; j += 4)
                cp_async16(&b.y[buf][j * 32 + 4 * (g ^ (j & 7))], z.sub + (int64_t)b.sid[j] * z.dp + t0 + 4 * g);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    double acc = 0.0;
    issue(0);
    for (int blk = 0; blk < nblk; blk++) {
        if (blk + 1 < nblk) issue(blk + 1);
        else asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncwarp();
        b.xd[lane] = (double)b.x[blk & 1][lane];  // the conversion unit is the scarce pipe
        __syncwarp();
        if ((int)lane < P) {
            const double2 *xs = reinterpret_cast<const double2 *>(b.xd);
            const float *yr = b.y[blk & 1] + lane * 32;
            const int sw = (int)(lane & 7);
            const int nb = z.d - blk * 32 < 32 ? z.d - blk * 32 : 32;
            if (nb == 32) {
#pragma unroll 2
                for (int q = 0; q < 8; q++) {
                    const double2 x01 = xs[2 * q], x23 = xs[2 * q + 1];
                    const float4 yv = *reinterpret_cast<const float4 *>(yr + 4 * (q ^ sw));
                    acc = exact_term_d<TAG>(acc, x01.x, yv.x);
                    acc = exact_term_d<TAG>(acc, x01.y, yv.y);
                    acc = exact_term_d<TAG>(acc, x23.x, yv.z);
                    acc = exact_term_d<TAG>(acc, x23.y, yv.w);
                }
            } else {
                for (int i = 0; i < nb; i++) acc = exact_term_d<TAG>(acc, b.xd[i], yr[4 * ((i >> 2) ^ sw) + (i & 3)]);
            }
        }
        __syncwarp();
    }
    if (TAG == 2 && (int)lane < P) acc = cos_finish(acc, z.nrm64[r], z.nrm64[my]);
    return acc;
}

template <int E>
__device__ __forceinline__ bool row_lists(const WarpRow<E> &s, int src) {
    bool hit = false;
#pragma unroll
    for (int e = 0; e < E; e++)
        for (int t = 0; t < 32; t++) {
            const int id = __shfl_sync(FULL_MASK, s.idf[e], t) >> 1;
            hit |= e * 32 + t < s.sz && id == src;
        }
    return hit;
}

// Resolve the need lanes of chunk c0 of a slot segment (slots seg[0, ns) of
// row r): from the cache, else by a new batch starting at this chunk.
// cpos/cval: the lane's cache entry (slot index, exact value).
template <int E>
__device__ __forceinline__ void lazy_chunk_eval(const WarpRow<E> &s, int k, const LazyExact z, int64_t r,
                                                const double *__restrict__ Bd, const int32_t *__restrict__ Bs,
                                                uint64_t seg, int64_t ns, int64_t c0, bool need, int src,
                                                double &dl, uint32_t &cpos, double &cval, LazyBatchSmem &b,
                                                unsigned lane, unsigned long long &nexact) {
    const uint32_t mypos = (uint32_t)(c0 + lane);
    // cache hits
    unsigned m = __ballot_sync(FULL_MASK, need);
    unsigned miss = 0;
    while (m) {
        const int i = __ffs(m) - 1;
        m &= m - 1;
        const uint32_t p = (uint32_t)(c0 + i);
        const unsigned h = __ballot_sync(FULL_MASK, cpos == p);
        if (h) {
            const double v = __shfl_sync(FULL_MASK, cval, __ffs(h) - 1);
            if ((int)lane == i) dl = v;
        } else {
            miss |= 1u << i;
        }
    }
    if (!miss) return;
    // a new batch: this chunk's misses, then look-ahead candidates in order
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    // Simulated worst: lane t (t < k, row full) counts the batch's candidates
    // whose upper estimate lies below its entry d[t]; once k - t of them do,
    // the row's worst will have dropped to d[t] or below by the time the
    // later slots get their turn, so look-ahead slots whose lower bound is
    // not below that are left out of the batch (most would have been
    // evaluated for nothing: 257 M evaluations for 179 M needed at config 3).
    const bool sim = E == 1 && s.sz == k;
    int simcnt = 0;
    double wsim = s.worst;
    auto sim_add = [&](unsigned cm, double ub) {  // cm: lanes holding a candidate, ub: its estimate
        if constexpr (E == 1) {  // (rows of one entry per lane)
            if (!sim) return;
            while (cm) {
                const int i = __ffs(cm) - 1;
                cm &= cm - 1;
                const double u = __shfl_sync(FULL_MASK, ub, i);
                simcnt += u < s.d[0] ? 1 : 0;
            }
            const unsigned ok = __ballot_sync(FULL_MASK, (int)lane < k && simcnt >= k - (int)lane);
            if (ok) wsim = __shfl_sync(FULL_MASK, s.d[0], __ffs(ok) - 1);
        }
    };
    int P = 0;
    {
        const bool mine = (miss >> lane) & 1u;
        const unsigned mm = __ballot_sync(FULL_MASK, mine);
        if (mine) {
            const int at = __popc(mm & lanemask_lt());
            KNNM_CHECK(src >= 0 && src < z.nrows);
            b.sid[at] = src;
            b.spos[at] = mypos;
        }
        P = __popc(mm);
        if (sim) sim_add(mm, mine ? slot_upper(Bd[seg + mypos], z) : inf);
    }
#pragma unroll 1
    for (int a = 1; a <= z.ahead; a++) {
        const int64_t cc = c0 + 32 * a;
        if (P >= 32 || cc >= ns) break;
        const int64_t j = cc + lane;
        const bool in = j < ns;
        const double v = in ? Bd[seg + j] : inf;
        const bool apx = in && slot_is_approx(v);
        const double lb = apx ? slot_lower(v, z) : inf;
        bool cand = apx && (lb < wsim || (s.sz < k && lb < inf));
        const int sv = cand ? Bs[seg + j] : 0;
        if (__any_sync(FULL_MASK, cand)) {
            const bool listed = row_lists<E>(s, sv);
            cand = cand && !listed;
        }
        const unsigned cm = __ballot_sync(FULL_MASK, cand);
        if (cm) sim_add(cm, cand ? slot_upper(v, z) : inf);
        const int at = P + __popc(cm & lanemask_lt());
        if (cand && at < 32) {
            KNNM_CHECK(sv >= 0 && sv < z.nrows);
            b.sid[at] = sv;
            b.spos[at] = (uint32_t)j;
        }
        __syncwarp();
        P += __popc(cm);
    }
    if (P > 32) P = 32;
    __syncwarp();
    double v;
    if (z.tag == 1) v = lazy_batch_t<1>(z, r, P, b, lane);
    else if (z.tag == 0) v = lazy_batch_t<0>(z, r, P, b, lane);
    else v = lazy_batch_t<2>(z, r, P, b, lane);
    if (lane == 0) nexact += (unsigned long long)P | (1ull << 40);  // pairs | batches << 40
    cpos = (int)lane < P ? b.spos[lane] : 0xffffffffu;
    cval = v;
    __syncwarp();
    // the misses of this chunk are batch entries 0 .. popc(miss) - 1
    const int rank = __popc(miss & lanemask_lt());
    const double mv = __shfl_sync(FULL_MASK, v, rank & 31);
    if ((miss >> lane) & 1u) dl = mv;
}

// _insert for rows held one entry per lane (k <= 32), cheapest tests first:
// a duplicate id costs one vote; "full and nd >= worst" is read off a
// ballot (worst = entry k-1, rows sorted by (d, id)) instead of a tracked
// worst.  Returns 1 (warp-uniform) when accepted.  s.worst is left stale:
// the caller refreshes it (warp_apply_chunk).
// FULL: the row is known to hold k entries (the usual state: no size vote,
// no growth).
template <typename T, bool FULL = false>
__device__ __forceinline__ int warp_insert1(WarpRow<1, T> &s, int k, int src, T nd, unsigned lane) {
    const int idf = s.idf[0];
    const T d = s.d[0];
    const bool in = (int)lane < (FULL ? k : s.sz);
    const int id = idf >> 1;
    if (__any_sync(FULL_MASK, in && id == src)) return 0;  // already listed
    // (sz is the same in every lane; a vote makes that visible to the compiler,
    // so the tests below are uniform branches)
    const bool full = FULL ? true : __all_sync(FULL_MASK, s.sz == k);
    const unsigned bs = __ballot_sync(FULL_MASK, in && nd < d);
    // nd >= worst (distance only).  FULL callers pass only candidates below the
    // current worst (warp_apply_chunk refreshes its live mask after every insert)
    if (!FULL && full && !((bs >> (k - 1)) & 1u)) return 0;
    const unsigned b = bs | __ballot_sync(FULL_MASK, in && nd == d && src < id);
    const int pos = b ? __ffs(b) - 1 : s.sz;
    const int last = full ? k - 1 : s.sz;
    const int up_i = __shfl_up_sync(FULL_MASK, idf, 1);
    const T up_d = __shfl_up_sync(FULL_MASK, d, 1);
    const bool here = (int)lane == pos, shift = (int)lane > pos && (int)lane <= last;
    s.idf[0] = here ? (int)(((uint32_t)src << 1) | 1u) : shift ? up_i : idf;
    s.d[0] = here ? nd : shift ? up_d : d;
    if (!full) s.sz += 1;
    return 1;
}

// Apply up to 32 in-order candidates held one per lane (lanes [0, cnt)).
// Candidates that cannot pass the "full and nd >= worst" test are skipped
// without changing the outcome (worst is non-increasing once a row is full).
template <int E, typename T = double>
__device__ __forceinline__ int warp_apply_chunk(WarpRow<E, T> &s, int k, int src_l, T d_l,
                                                int cnt, unsigned lane) {
    if constexpr (E == 1) {
        int acc = 0;
        unsigned m = __ballot_sync(FULL_MASK, (int)lane < cnt && d_l < dist_inf<T>() &&
                                                  (s.sz < k || d_l < s.worst));
        // rows still filling up (first inserts of a fresh row)
        while (m && s.sz < k) {
            const int i = __ffs(m) - 1;
            m &= m - 1;
            acc += warp_insert1<T>(s, k, __shfl_sync(FULL_MASK, src_l, i), __shfl_sync(FULL_MASK, d_l, i), lane);
            if (s.sz == k) {
                s.worst = __shfl_sync(FULL_MASK, s.d[0], (k - 1) & 31);
                m &= __ballot_sync(FULL_MASK, d_l < s.worst);
            }
        }
        while (m) {
            const int i = __ffs(m) - 1;
            m &= m - 1;
            if (warp_insert1<T, true>(s, k, __shfl_sync(FULL_MASK, src_l, i), __shfl_sync(FULL_MASK, d_l, i),
                                      lane)) {
                acc++;
                // the worst only decreases once the row is full: candidates it
                // now excludes leave the loop with one ballot instead of a
                // turn each (so every candidate that gets a turn is below
                // the worst of its turn)
                s.worst = __shfl_sync(FULL_MASK, s.d[0], (k - 1) & 31);
                m &= __ballot_sync(FULL_MASK, d_l < s.worst);
            }
        }
        return acc;
    }
    int acc = 0;
    // d_l = +inf marks an empty slot (real distances are finite); a candidate
    // live at chunk start is re-tested against the current worst when its
    // turn comes (the worst only decreases once the row is full)
    unsigned m = __ballot_sync(FULL_MASK, (int)lane < cnt && d_l < dist_inf<T>() &&
                                              (s.sz < k || d_l < s.worst));
    while (m) {
        const int i = __ffs(m) - 1;
        m &= m - 1;
        const int src = __shfl_sync(FULL_MASK, src_l, i);
        const T nd = __shfl_sync(FULL_MASK, d_l, i);
        if (!(s.sz < k || nd < s.worst)) continue;
        // a listed id (the common rejection in later rounds) costs one vote
        bool dup = false;
#pragma unroll
        for (int e = 0; e < E; e++) dup |= e * 32 + (int)lane < s.sz && (s.idf[e] >> 1) == src;
        if (__any_sync(FULL_MASK, dup)) continue;
        acc += warp_insert<E, false, T>(s, k, src, nd, lane);
    }
    return acc;
}

}  // namespace knnm

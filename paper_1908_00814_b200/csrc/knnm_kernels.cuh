// knnm_kernels.cuh -- sm_100a kernels of the S-Merge / J-Merge round engine.
//
// Each kernel cites the reference numba kernel (pkg/src/knnmerge/_kernels.py)
// whose result it reproduces bit-for-bit.  Design notes live in DESIGN.md.
#pragma once
#include "knnm_device.cuh"

namespace knnm {

constexpr int WARP_REV_MAX = 256;      // reverse segments a warp sorts itself
constexpr int BLOCK_SORT_MAX = 16384;  // elements a block sorts in shared memory
constexpr int APPLY_WARP_MAX = 1024;   // candidates per row handled by one warp
constexpr int MAX_W = 128;             // k + rev_cap upper bound

struct CandA {  // emitted directed update (unsorted)
    uint64_t key;  // reference order: (u*W + p)*W + q, or the init ordinal
    double d;
    int32_t src;
    int32_t tgt;
};
struct CandB {  // bucketed by target row
    uint64_t key;
    double d;
    int32_t src;
    int32_t pad;
};

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
    // np.searchsorted(union, g) (side='left')
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
                             int32_t *tail_s, int tk) {
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
__global__ void k_directed_emit(const int32_t *__restrict__ rows, const int32_t *__restrict__ nids,
                                int64_t m, int64_t key0, const float *__restrict__ sub, int dp,
                                int d, int tag, const int32_t *__restrict__ sizes,
                                const double *__restrict__ dists, int k, CandA *A, uint32_t *tcnt,
                                unsigned long long *counters, double *cap_d) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool valid = i < m;
    bool emit = false;
    int32_t r = 0, s = 0;
    double dd = 0.0;
    if (valid) {
        r = rows[i];
        s = nids[i];
        dd = exact_dist_tag(tag, sub + (int64_t)r * dp, sub + (int64_t)s * dp, d);
        if (cap_d) cap_d[i] = dd;
        // exact-safe prefilter: the row is untouched until the apply phase
        emit = !(sizes[r] == k && dd >= dists[(int64_t)r * k + k - 1]);
    }
    unsigned lane = lane_id();
    unsigned mk = __ballot_sync(FULL_MASK, emit);
    unsigned long long base = 0;
    if (lane == 0 && mk) base = atomicAdd(&counters[C_CAND], (unsigned long long)__popc(mk));
    base = __shfl_sync(FULL_MASK, base, 0);
    if (emit) {
        unsigned long long pos = base + __popc(mk & lanemask_lt());
        A[pos] = CandA{(uint64_t)(key0 + i), dd, s, r};
        atomicAdd(&tcnt[r], 1u);
    }
}

// ---------------------------------------------------------------------------
// Reverse CSR (_kernels.py:262-281): in-degree histogram, then scatter of
// (source << 1 | new-flag).  Segment order is restored where it matters
// (Fisher-Yates subsampling) by sorting on the source id in the assemble step.
// ---------------------------------------------------------------------------
__global__ void k_rev_count(const int32_t *__restrict__ ids, const int32_t *__restrict__ sizes,
                            int64_t n, int k, uint32_t *indeg) {
    int64_t total = n * k;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = i / k;
        int t = (int)(i % k);
        if (t < sizes[r]) atomicAdd(&indeg[ids[i]], 1u);
    }
}

__global__ void k_rev_fill(const int32_t *__restrict__ ids, const uint8_t *__restrict__ flags,
                           const int32_t *__restrict__ sizes, int64_t n, int k,
                           const uint32_t *__restrict__ roff, uint32_t *indeg, uint32_t *rev) {
    int64_t total = n * k;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = i / k;
        int t = (int)(i % k);
        if (t < sizes[r]) {
            int32_t j = ids[i];
            uint32_t p = roff[j] + atomicSub(&indeg[j], 1u) - 1u;
            rev[p] = ((uint32_t)r << 1) | (uint32_t)flags[i];
        }
    }
}

__global__ void k_find_heavy(const uint32_t *__restrict__ roff, int64_t n, int limit,
                             int32_t *heavy, unsigned long long *counters) {
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
         u += (int64_t)gridDim.x * blockDim.x) {
        uint32_t deg = roff[u + 1] - roff[u];
        if (deg > (uint32_t)limit) {
            unsigned long long p = atomicAdd(&counters[C_HEAVY_REV], 1ull);
            heavy[p] = (int32_t)u;
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
__global__ void k_rev_heavy(const int32_t *__restrict__ heavy, const unsigned long long *counters,
                            const uint32_t *__restrict__ roff, uint32_t *rev, int rev_cap,
                            uint64_t seed, uint32_t *gscratch, int smem_max) {
    extern __shared__ uint32_t hs[];
    __shared__ uint32_t R[MAX_W];
    unsigned long long cnt = counters[C_HEAVY_REV];
    for (unsigned long long h = blockIdx.x; h < cnt; h += gridDim.x) {
        int64_t u = heavy[h];
        uint32_t lo = roff[u];
        uint32_t deg = roff[u + 1] - lo;
        uint32_t P2 = next_pow2(deg);
        bool in_smem = P2 <= (uint32_t)smem_max;
        if (!in_smem && gscratch == nullptr) continue;  // giant: second pass
        if (in_smem && gscratch != nullptr) continue;
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
// Neighbourhood assembly (_kernels.py:316-383) + flag clear
// (construct.py:142) + pair counting (_kernels.py:402-417, closed form) +
// round-start worst snapshot for the exact prefilter.  One warp per vertex.
// nbh entries are packed (local id << 1 | new).
// ---------------------------------------------------------------------------
constexpr int ASM_WARPS = 8;

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

__global__ void __launch_bounds__(ASM_WARPS * 32)
k_assemble(const int32_t *__restrict__ ids, uint8_t *flags, const int32_t *__restrict__ sizes,
           const double *__restrict__ dists, int64_t n, int k, int rev_cap,
           const uint32_t *__restrict__ roff, const uint32_t *__restrict__ rev, uint64_t seed,
           const int8_t *__restrict__ labels, int mode, int W, uint32_t *nbh, int32_t *nlen,
           uint32_t *hpairs, double *worst0, int32_t *active, unsigned long long *counters) {
    __shared__ uint32_t s_seg[ASM_WARPS][WARP_REV_MAX];
    __shared__ uint32_t s_idx[ASM_WARPS][WARP_REV_MAX];
    __shared__ uint32_t s_R[ASM_WARPS][MAX_W];
    __shared__ uint32_t s_buf[ASM_WARPS][MAX_W];
    unsigned lane = lane_id(), wib = threadIdx.x >> 5;
    uint32_t *seg = s_seg[wib], *idx = s_idx[wib], *R = s_R[wib], *buf = s_buf[wib];
    int64_t nw = (int64_t)gridDim.x * ASM_WARPS;
    unsigned long long members = 0;
    for (int64_t u = (int64_t)blockIdx.x * ASM_WARPS + wib; u < n; u += nw) {
        int sz = sizes[u];
        for (int t = lane; t < sz; t += 32)
            buf[t] = ((uint32_t)ids[u * k + t] << 1) | (uint32_t)flags[u * k + t];
        __syncwarp();
        for (int t = lane; t < k; t += 32) flags[u * k + t] = 0;
        if (lane == 0) worst0[u] = sz == k ? dists[u * k + k - 1] : __longlong_as_double(0x7ff0000000000000LL);
        uint32_t lo = roff[u], deg = roff[u + 1] - lo;
        int m = sz;
        if (deg <= (uint32_t)rev_cap) {
            for (uint32_t j = lane; j < deg; j += 32) buf[m + j] = rev[lo + j];
            m += deg;
        } else if (deg <= (uint32_t)WARP_REV_MAX) {
            uint32_t P2 = next_pow2(deg);
            for (uint32_t j = lane; j < P2; j += 32) {
                seg[j] = j < deg ? rev[lo + j] : 0xffffffffu;
                idx[j] = j;
            }
            uint64_t st0 = seed ^ ((uint64_t)(u + 1) * U64_GAMMA);
            for (int t = lane; t < rev_cap; t += 32) {
                uint64_t z = mix64(st0 + (uint64_t)(t + 2) * U64_GAMMA);
                R[t] = (uint32_t)t + (uint32_t)(z % (uint64_t)(deg - (uint32_t)t));
            }
            __syncwarp();
            bitonic_warp<uint32_t>(seg, P2, lane);
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
        __syncwarp();
        uint32_t P2u = next_pow2((uint32_t)(m > 1 ? m : 1));
        for (uint32_t j = m + lane; j < P2u; j += 32) buf[j] = 0xffffffffu;
        __syncwarp();
        bitonic_warp<uint32_t>(buf, P2u, lane);
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
                nbh[u * W + w + __popc(em & lanemask_lt())] = v;
                lab = labels[v >> 1];
            }
            bool nw_ = end && (v & 1);
            an += __popc(__ballot_sync(FULL_MASK, end && lab == 0 && nw_));
            ao += __popc(__ballot_sync(FULL_MASK, end && lab == 0 && !nw_));
            bn += __popc(__ballot_sync(FULL_MASK, end && lab != 0 && nw_));
            bo += __popc(__ballot_sync(FULL_MASK, end && lab != 0 && !nw_));
            w += __popc(em);
        }
        if (lane == 0) {
            nlen[u] = w;
            uint64_t pc = pairs_closed_form(mode, an, ao, bn, bo);
            hpairs[u] = (uint32_t)pc;
            if (pc > 0) {
                unsigned long long p = atomicAdd(&counters[C_ACTIVE], 1ull);
                active[p] = (int32_t)u;
                members += members_closed_form(mode, an, ao, bn, bo);
            }
        }
        __syncwarp();
    }
    if (lane == 0 && members) atomicAdd(&counters[C_MEMBERS], members);
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
             CandA *A, unsigned long long cap, uint32_t *tcnt, unsigned long long *counters) {
    extern __shared__ float4 sv4[];
    __shared__ int s_id[MAX_W];
    __shared__ int s_new[MAX_W];
    __shared__ int s_lab[MAX_W];
    __shared__ double s_w[MAX_W];
    const float *sv = reinterpret_cast<const float *>(sv4);
    int64_t u = active[blockIdx.x];
    int w = nlen[u];
    for (int i = threadIdx.x; i < w; i += blockDim.x) {
        uint32_t e = nbh[u * W + i];
        int id = (int)(e >> 1);
        s_id[i] = id;
        s_new[i] = e & 1;
        s_lab[i] = labels[id];
        s_w[i] = worst0[id];
    }
    __syncthreads();
    int q4 = dp >> 2;
    for (int i = threadIdx.x; i < w * q4; i += blockDim.x) {
        int r = i / q4, c = i - r * q4;
        sv4[i] = __ldg(reinterpret_cast<const float4 *>(sub + (int64_t)s_id[r] * dp) + c);
    }
    __syncthreads();
    unsigned lane = lane_id();
    int total = w * w;
    for (int base = 0; base < total; base += blockDim.x) {
        int L = base + threadIdx.x;
        int p = L / w, q = L - (L / w) * w;
        bool ok = L < total && q > p && admissible(s_new[p], s_new[q], s_lab[p], s_lab[q], mode);
        double dd = 0.0;
        if (ok) dd = exact_dist<TAG>(sv + p * dp, sv + q * dp, d);
        bool e1 = ok && dd < s_w[p];  // id[p] <- id[q]
        bool e2 = ok && dd < s_w[q];  // id[q] <- id[p]
        unsigned m1 = __ballot_sync(FULL_MASK, e1), m2 = __ballot_sync(FULL_MASK, e2);
        int tot = __popc(m1) + __popc(m2);
        unsigned long long b0 = 0;
        if (lane == 0 && tot) b0 = atomicAdd(&counters[C_CAND], (unsigned long long)tot);
        b0 = __shfl_sync(FULL_MASK, b0, 0);
        uint64_t key = ((uint64_t)u * W + p) * W + q;
        if (e1) {
            unsigned long long pos = b0 + __popc(m1 & lanemask_lt());
            if (pos < cap) {
                A[pos] = CandA{key, dd, s_id[q], s_id[p]};
                atomicAdd(&tcnt[s_id[p]], 1u);
            } else {
                atomicAdd(&counters[C_OVERFLOW], 1ull);
            }
        }
        if (e2) {
            unsigned long long pos = b0 + __popc(m1) + __popc(m2 & lanemask_lt());
            if (pos < cap) {
                A[pos] = CandA{key, dd, s_id[p], s_id[q]};
                atomicAdd(&tcnt[s_id[q]], 1u);
            } else {
                atomicAdd(&counters[C_OVERFLOW], 1ull);
            }
        }
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
//   !CERT : the fp32 value screens with a rigorous error margin; pairs that
//           may pass are re-evaluated with the exact fp64 metric from the
//           staged vectors.
// Emission as in k_join_exact: reference-order key (u, p, q), exact-safe
// prefilter against the round-start worst of each target.
// ---------------------------------------------------------------------------
constexpr int TJ_WARPS = 2;
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

template <int TAG, bool CERT>
__global__ void __launch_bounds__(TJ_THREADS)
k_join_tiled(const int32_t *__restrict__ active, int nactive, const uint32_t *__restrict__ nbh,
             const int32_t *__restrict__ nlen, int W, const int8_t *__restrict__ labels, int mode,
             const float *__restrict__ sub, int dp, int d, const double *__restrict__ worst0,
             CandA *A, unsigned long long cap, uint32_t *tcnt, unsigned long long *counters,
             double mrel, double mabs) {
    extern __shared__ __align__(128) float4 sv4[];
    __shared__ int s_id[MAX_W];
    __shared__ int s_pos[MAX_W];
    __shared__ int s_new[MAX_W];
    __shared__ double s_w[MAX_W];
    __shared__ float s_nrm[MAX_W];
    __shared__ int s_cls[4];
    __shared__ __align__(8) uint64_t s_bar;
    const float *sv = reinterpret_cast<const float *>(sv4);
    const int tid = threadIdx.x;
    const unsigned lane = lane_id();
    const int warp = tid >> 5;
    const int q4 = dp >> 2;
    const int qs = q4 + 1;  // padded row stride in float4
    if (tid == 0) mbar_init(&s_bar, 1);
    __syncthreads();
    uint32_t phase = 0;
    unsigned long long n_exact = 0;

    for (int hi = blockIdx.x; hi < nactive; hi += gridDim.x) {
        const int64_t u = active[hi];
        const int w = nlen[u];
        // ---- classify members: class = (label != 0) * 2 + (!new) ----------
        if (tid < 32) {
            int cnts[4] = {0, 0, 0, 0};
            int base_cls[4];
            // first pass: class counts
            for (int b = 0; b < w; b += 32) {
                int j = b + lane;
                int cls = 4;
                if (j < w) {
                    uint32_t e = nbh[u * W + j];
                    int lab = mode == 0 ? 0 : (labels[e >> 1] != 0);
                    cls = lab * 2 + ((e & 1) ? 0 : 1);
                }
#pragma unroll
                for (int c = 0; c < 4; c++) cnts[c] += __popc(__ballot_sync(FULL_MASK, cls == c));
            }
            base_cls[0] = 0;
            base_cls[1] = cnts[0];
            base_cls[2] = cnts[0] + cnts[1];
            base_cls[3] = base_cls[2] + cnts[2];
            int fill[4] = {0, 0, 0, 0};
            for (int b = 0; b < w; b += 32) {
                int j = b + lane;
                int cls = 4;
                uint32_t e = 0;
                if (j < w) {
                    e = nbh[u * W + j];
                    int lab = mode == 0 ? 0 : (labels[e >> 1] != 0);
                    cls = lab * 2 + ((e & 1) ? 0 : 1);
                }
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    unsigned m = __ballot_sync(FULL_MASK, cls == c);
                    if (cls == c) {
                        int slot = base_cls[c] + fill[c] + __popc(m & lanemask_lt());
                        int id = (int)(e >> 1);
                        s_id[slot] = id;
                        s_pos[slot] = j;
                        s_new[slot] = (int)(e & 1);
                        s_w[slot] = worst0[id];
                    }
                    fill[c] += __popc(m);
                }
            }
            if (lane < 4) s_cls[lane] = cnts[lane];
        }
        __syncthreads();
        // ---- stage the member rows with TMA bulk copies ---------------------
        // smem row stride = dp + 4 floats: consecutive rows start 16 B apart
        // modulo 128 B, so 8 distinct rows per wavefront are conflict-free.
        if (tid == 0) {
            fence_proxy_async();
            const uint32_t row_bytes = (uint32_t)dp * 4u;
            mbar_expect_tx(&s_bar, row_bytes * (uint32_t)w);
            for (int sl = 0; sl < w; sl++)
                bulk_g2s(sv4 + (size_t)sl * qs, sub + (int64_t)s_id[sl] * dp, row_bytes, &s_bar);
        }
        mbar_wait(&s_bar, phase);
        phase ^= 1u;
        if (TAG == 2) {
            // fp32 norms for the cosine screen
            for (int sl = warp; sl < w; sl += TJ_WARPS) {
                float acc = 0.f;
                for (int c = lane; c < q4; c += 32) {
                    float4 a = sv4[(size_t)sl * qs + c];
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
        for (int pid = warp; pid < np0 + np1; pid += TJ_WARPS) {
            const bool second = pid >= np0;
            const int lp = second ? pid - np0 : pid;
            const int pcs = second ? pc1 : pc0;
            const int pr = lp / pcs, pcc = lp - pr * pcs;
            const int rt = pr * 4 + (int)(lane >> 3), ct = pcc * 8 + (int)(lane & 7);
            const int r0 = second ? b1r0 : b0r0, r1 = second ? b1r1 : b0r1;
            const int c0 = second ? b1c0 : b0c0, c1 = second ? b1c1 : b0c1;
            const int rn = second ? b1rn : b0rn, cn = second ? b1cn : b0cn;
            const bool tri = second ? true : (bool)b0tri;
            const int i0 = r0 + 2 * rt, j0 = c0 + 2 * ct;
            bool live = i0 < r1 && j0 < c1;
            if (live && tri && rt > ct) live = false;             // below diagonal
            if (live && 2 * rt >= rn && 2 * ct >= cn) live = false;  // old x old
            const bool vi1 = i0 + 1 < r1, vj1 = j0 + 1 < c1;
            float acc[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
            if (live) {
                const float4 *a0p = sv4 + (size_t)i0 * qs;
                const float4 *a1p = sv4 + (size_t)(vi1 ? i0 + 1 : i0) * qs;
                const float4 *b0p = sv4 + (size_t)j0 * qs;
                const float4 *b1p = sv4 + (size_t)(vj1 ? j0 + 1 : j0) * qs;
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
            // ---- finalize the 4 pairs of the tile --------------------------
#pragma unroll
            for (int s = 0; s < 4; s++) {
                const int ii = i0 + (s >> 1), jj = j0 + (s & 1);
                bool ok = live && ii < r1 && jj < c1;
                if (ok && tri) ok = ii < jj;
                if (ok) ok = s_new[ii] || s_new[jj];
                double dd = 0.0;
                bool e1 = false, e2 = false;
                if (ok) {
                    const double wi = s_w[ii], wj = s_w[jj];
                    const double wmax = wi > wj ? wi : wj;
                    float f = acc[s >> 1][s & 1];
                    if (CERT) {
                        dd = (double)f;
                    } else {
                        bool maybe;
                        if (TAG == 2) {
                            float na = s_nrm[ii], nb = s_nrm[jj];
                            if (na == 0.f || nb == 0.f) {
                                maybe = true;
                            } else {
                                float cs = 1.0f - f / (sqrtf(na) * sqrtf(nb));
                                maybe = (double)cs <= wmax + mabs;
                            }
                        } else {
                            maybe = (double)f <= wmax * mrel;
                        }
                        if (maybe) {
                            dd = exact_dist<TAG>(sv + (size_t)ii * qs * 4, sv + (size_t)jj * qs * 4, d);
                            n_exact++;
                        } else {
                            dd = __longlong_as_double(0x7ff0000000000000LL);
                        }
                    }
                    e1 = dd < wi;  // id[ii] <- id[jj]
                    e2 = dd < wj;  // id[jj] <- id[ii]
                }
                unsigned m1 = __ballot_sync(FULL_MASK, e1), m2 = __ballot_sync(FULL_MASK, e2);
                int tot = __popc(m1) + __popc(m2);
                if (tot) {
                    unsigned long long bb = 0;
                    if (lane == 0) bb = atomicAdd(&counters[C_CAND], (unsigned long long)tot);
                    bb = __shfl_sync(FULL_MASK, bb, 0);
                    if (e1 || e2) {
                        const int pi = s_pos[ii], pj = s_pos[jj];
                        const int p = pi < pj ? pi : pj, q = pi < pj ? pj : pi;
                        const uint64_t key = ((uint64_t)u * W + p) * W + q;
                        const int idi = s_id[ii], idj = s_id[jj];
                        if (e1) {
                            unsigned long long pos = bb + __popc(m1 & lanemask_lt());
                            if (pos < cap) {
                                A[pos] = CandA{key, dd, idj, idi};
                                atomicAdd(&tcnt[idi], 1u);
                            }
                        }
                        if (e2) {
                            unsigned long long pos = bb + __popc(m1) + __popc(m2 & lanemask_lt());
                            if (pos < cap) {
                                A[pos] = CandA{key, dd, idi, idj};
                                atomicAdd(&tcnt[idj], 1u);
                            }
                        }
                    }
                }
            }
        }
        __syncthreads();  // smem reused by the next hood
    }
    if (!CERT) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) n_exact += __shfl_xor_sync(FULL_MASK, n_exact, o);
        if (lane == 0 && n_exact) atomicAdd(&counters[C_EXACT], n_exact);
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
            int ip = ep >> 1, iq = eq >> 1;
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
// Candidate bucketing by target row (the counting sort of
// apply_updates_grouped, _kernels.py:227-247).
// ---------------------------------------------------------------------------
__global__ void k_scatter(const CandA *__restrict__ A, unsigned long long count,
                          const uint32_t *__restrict__ toff, uint32_t *tcnt, CandB *B) {
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        CandA c = A[i];
        uint32_t p = toff[c.tgt] + atomicSub(&tcnt[c.tgt], 1u) - 1u;
        B[p] = CandB{c.key, c.d, c.src, 0};
    }
}

// ---------------------------------------------------------------------------
// Sequential per-row insertion in reference order (apply_updates_grouped's
// row loop, _kernels.py:248-254, each step _insert _kernels.py:159-192).
// One warp per row; the row's candidates are sorted by reference key first.
// ---------------------------------------------------------------------------
constexpr int APPLY_WARPS = 4;

// Sort a row's c <= 32*NE candidates in registers by reference key, then
// apply them in order, 32 at a time.
template <int E, int NE>
__device__ __forceinline__ int apply_sorted_reg(WarpRow<E> &s, int k, const CandB *__restrict__ Bp,
                                                int c, int ib, uint64_t mask, unsigned lane) {
    uint64_t v[NE];
#pragma unroll
    for (int e = 0; e < NE; e++) {
        int j = e * 32 + (int)lane;
        v[e] = j < c ? ((Bp[j].key << ib) | (uint64_t)j) : ~0ull;
    }
    warp_sort_reg<NE>(v, lane);
    int a = 0;
#pragma unroll
    for (int e = 0; e < NE; e++) {
        const int base = e * 32;
        if (base >= c) break;
        int src = 0;
        double dd = 0.0;
        if (base + (int)lane < c) {
            const CandB &cb = Bp[(uint32_t)(v[e] & mask)];
            src = cb.src;
            dd = cb.d;
        }
        a += warp_apply_chunk<E>(s, k, src, dd, c - base < 32 ? c - base : 32, lane);
    }
    return a;
}

template <int E>
__global__ void __launch_bounds__(APPLY_WARPS * 32)
k_apply(int64_t n, int k, const uint32_t *__restrict__ toff, const CandB *__restrict__ B, int ib,
        int32_t *ids, double *dists, uint8_t *flags, int32_t *sizes, int32_t *heavy,
        unsigned long long *counters) {
    __shared__ uint64_t s_sort[APPLY_WARPS][APPLY_WARP_MAX];
    unsigned lane = lane_id(), wib = threadIdx.x >> 5;
    uint64_t *srt = s_sort[wib];
    int64_t nw = (int64_t)gridDim.x * APPLY_WARPS;
    unsigned long long acc = 0;
    for (int64_t r = (int64_t)blockIdx.x * APPLY_WARPS + wib; r < n; r += nw) {
        uint32_t lo = toff[r];
        int c = (int)(toff[r + 1] - lo);
        if (c == 0) continue;
        if (c > APPLY_WARP_MAX) {
            if (lane == 0) {
                heavy[atomicAdd(&counters[C_HEAVY_APPLY], 1ull)] = (int32_t)r;
                atomicMax(&counters[C_MAXC], (unsigned long long)c);
            }
            continue;
        }
        WarpRow<E> s;
        row_load<E>(s, ids, dists, flags, sizes, r, k, lane);
        const uint64_t mask = (1ull << ib) - 1ull;
        int a = 0;
        if (c <= 32) {
            a += apply_sorted_reg<E, 1>(s, k, B + lo, c, ib, mask, lane);
        } else if (c <= 64) {
            a += apply_sorted_reg<E, 2>(s, k, B + lo, c, ib, mask, lane);
        } else if (c <= 128) {
            a += apply_sorted_reg<E, 4>(s, k, B + lo, c, ib, mask, lane);
        } else if (c <= 256) {
            a += apply_sorted_reg<E, 8>(s, k, B + lo, c, ib, mask, lane);
        } else {
            uint32_t P2 = next_pow2((uint32_t)c);
            for (uint32_t j = lane; j < P2; j += 32)
                srt[j] = (int)j < c ? ((B[lo + j].key << ib) | j) : ~0ull;
            __syncwarp();
            bitonic_warp<uint64_t>(srt, P2, lane);
            for (int base = 0; base < c; base += 32) {
                int j = base + lane;
                int src = 0;
                double dd = 0.0;
                if (j < c) {
                    const CandB &cb = B[lo + (uint32_t)(srt[j] & mask)];
                    src = cb.src;
                    dd = cb.d;
                }
                a += warp_apply_chunk<E>(s, k, src, dd, c - base < 32 ? c - base : 32, lane);
            }
            __syncwarp();
        }
        row_store<E>(s, ids, dists, flags, sizes, r, k, lane);
        acc += a;
    }
    if (lane == 0 && acc) atomicAdd(&counters[C_ACCEPTED], acc);
}

// Rows with more than APPLY_WARP_MAX candidates: one block sorts (shared
// memory, or a global scratch for giant rows), warp 0 inserts.
template <int E>
__global__ void k_apply_heavy(const int32_t *__restrict__ heavy, int64_t k_, const uint32_t *__restrict__ toff,
                              const CandB *__restrict__ B, int ib, int32_t *ids, double *dists,
                              uint8_t *flags, int32_t *sizes, unsigned long long *counters,
                              uint64_t *gscratch, int smem_max, int32_t *giant) {
    extern __shared__ uint64_t hsrt[];
    int k = (int)k_;
    unsigned long long cnt = counters[C_HEAVY_APPLY];
    unsigned lane = lane_id();
    for (unsigned long long h = blockIdx.x; h < cnt; h += gridDim.x) {
        int64_t r = heavy[h];
        uint32_t lo = toff[r];
        uint32_t c = toff[r + 1] - lo;
        uint32_t P2 = next_pow2(c);
        bool in_smem = P2 <= (uint32_t)smem_max;
        if (gscratch == nullptr && !in_smem) continue;  // giant rows: second pass
        if (gscratch != nullptr && in_smem) continue;
        uint64_t *srt = in_smem ? hsrt : gscratch;
        uint64_t mask = (1ull << ib) - 1ull;
        for (uint32_t j = threadIdx.x; j < P2; j += blockDim.x)
            srt[j] = j < c ? ((B[lo + j].key << ib) | j) : ~0ull;
        __syncthreads();
        bitonic_block<uint64_t>(srt, P2);
        if (threadIdx.x < 32) {
            WarpRow<E> s;
            row_load<E>(s, ids, dists, flags, sizes, r, k, lane);
            int a = 0;
            for (uint32_t base = 0; base < c; base += 32) {
                uint32_t j = base + lane;
                int src = 0;
                double dd = 0.0;
                if (j < c) {
                    const CandB &cb = B[lo + (uint32_t)(srt[j] & mask)];
                    src = cb.src;
                    dd = cb.d;
                }
                a += warp_apply_chunk<E>(s, k, src, dd, c - base < 32 ? (int)(c - base) : 32, lane);
            }
            row_store<E>(s, ids, dists, flags, sizes, r, k, lane);
            if (lane == 0 && a) atomicAdd(&counters[C_ACCEPTED], (unsigned long long)a);
        }
        __syncthreads();
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
    auto val = [&](int64_t e) -> double {
        int64_t u = e / k;
        int t = (int)(e - u * k);
        return t < sizes[u] ? dists[e] : 0.0;
    };
    double res;
    if (n < 8) {
        res = 0.0;
        for (int i = 0; i < n; i++) res = __dadd_rn(res, val(lo + i));
    } else {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; j++) r[j] = val(lo + j);
        int i;
        for (i = 8; i < n - (n % 8); i += 8) {
#pragma unroll
            for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], val(lo + i + j));
        }
        res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                        __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n; i++) res = __dadd_rn(res, val(lo + i));
    }
    out[li] = res;
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
        out_ids[i] = v >= 0 ? (int32_t)ug[v] : -1;
    }
}

__global__ void k_merge_rear(const int32_t *__restrict__ ui, const double *__restrict__ ud,
                             const int32_t *__restrict__ us, const int32_t *__restrict__ ri,
                             const double *__restrict__ rd, const int32_t *__restrict__ rs, int64_t n,
                             int k, int rk, int32_t *oi, double *od, int32_t *os) {
    int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n) return;
    const int32_t *a_i = ui + u * k;
    const double *a_d = ud + u * k;
    const int32_t *b_i = ri + u * rk;
    const double *b_d = rd + u * rk;
    int32_t *o_i = oi + u * k;
    double *o_d = od + u * k;
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

}  // namespace knnm

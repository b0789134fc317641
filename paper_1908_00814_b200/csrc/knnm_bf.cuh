// knnm_bf.cuh -- exact brute-force k-NN on the 5th-generation tensor cores
// (tcgen05 + TMEM + TMA), for the ground truth of recall measurements
// (reference construct.py:273-348 brute_force_graph / brute_force_queries,
// _kernels.py:445-506 bf_graph_dense / bf_queries_dense).
//
// Certified u8 datasets (every entry an integer in [0, 255]; the config-2 /
// config-5 stand-ins): the Gram tile Q . X^T is computed EXACTLY by
// tcgen05.mma kind::i8 (u8 x u8 -> s32), so L2^2 = |q|^2 + |x|^2 - 2 q.x is
// the exact integer the reference's sequential fp64 sum produces (all
// partial sums are integers below 2^53).  The reference inserts candidates
// in ascending id order with the rule "reject when full and d >= worst",
// which makes its lists the top-k by (distance, id); every epilogue thread
// here also sees its candidates in ascending id order and keeps a sorted
// (dist << 32 | id) list, so the result is the reference's bit for bit.
//
// CTA layout (one CTA per 128-query block and data slice):
//   warp 0        TMA producer: the query tile once, then 256-row data tiles
//                 (K = 128 bytes per stage, SWIZZLE_128B) into a 4-deep ring
//   warp 1        TMEM allocator + MMA issuer (one elected thread):
//                 M=128 x N=256 x K=32 per instruction, two 256-column s32
//                 accumulators in TMEM so the epilogue of tile t overlaps
//                 the MMA of tile t+1
//   warps 2..9    epilogue: tcgen05.ld 32x32b.x32 (warp w reads TMEM lanes
//                 32*(w%4)..+31, i.e. 32 queries; warps w and w+4 split the
//                 256 columns), distance from the row norms, strict
//                 "d < worst" test and a sorted insert into a per-thread
//                 list in shared memory; the two half-lists of a query are
//                 merged at the end.
#pragma once

#include <cuda.h>
#include <cstdint>

#include "knnm_device.cuh"

namespace knnm {

constexpr int TB_M = 128;          // queries per CTA (TMEM lanes)
constexpr int TB_N = 256;          // data rows per tile (MMA N)
constexpr int TB_KB = 128;         // bytes of K per stage (one 128-byte swizzle row)
constexpr int TB_STAGES = 4;
constexpr int TB_EPI_WARPS = 8;
constexpr int TB_THREADS = (2 + TB_EPI_WARPS) * 32;
constexpr int TB_MAX_KB = 4;       // u8 rows up to 512 bytes
constexpr int TB_MAX_K = 32;       // list length held per epilogue thread
constexpr int TB_LIST_STRIDE = TB_EPI_WARPS * 32;  // entry t of thread i at [t * stride + i]
constexpr uint32_t TB_A_BYTES = TB_M * TB_KB;      // 16 KB per K block
constexpr uint32_t TB_B_BYTES = TB_N * TB_KB;      // 32 KB per stage

__host__ __device__ constexpr size_t tb_smem_bytes(int nkb, int k) {
    return 1024 /* alignment slack */ + (size_t)nkb * TB_A_BYTES + (size_t)TB_STAGES * TB_B_BYTES +
           (size_t)TB_LIST_STRIDE * k * 8 + 16 * 8 /* barriers */ + 16;
}

// K-major, 128-byte swizzled operand tile (8-row groups of 1024 bytes):
// start address >> 4, LBO = 1 (unused for swizzled K-major), SBO = 1024 B,
// descriptor version 1 (sm_100), layout SWIZZLE_128B.  Stepping K by 32
// bytes inside the swizzle row adds 2 to the start-address field.
__device__ __forceinline__ uint64_t tb_desc(uint32_t saddr) {
    return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// Instruction descriptor, kind::i8: D s32, A and B unsigned 8-bit, both
// K-major, N = 256, M = 128.
constexpr uint32_t TB_IDESC = (2u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(TB_N >> 3) << 17) |
                              ((uint32_t)(TB_M >> 4) << 24);

__device__ __forceinline__ void tb_tma_2d(void *dst, const CUtensorMap *map, int x, int y, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tb_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tc_mma_i8(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }" ::"r"(dtmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// 32 consecutive TMEM columns of this warp's 32 lanes -> v[0..31].
__device__ __forceinline__ void tc_ld32(uint32_t taddr, int32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
          "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
          "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
          "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Sorted insert of ``key`` into a thread's list (entries at lst[t * stride]);
// returns the new worst distance (0xffffffff while the list is not full).
__device__ __forceinline__ uint32_t tb_insert(uint64_t *lst, int k, uint64_t key) {
    int t = k - 1;
    while (t > 0) {
        const uint64_t prev = lst[(t - 1) * TB_LIST_STRIDE];
        if (!(key < prev)) break;
        lst[t * TB_LIST_STRIDE] = prev;
        t--;
    }
    lst[t * TB_LIST_STRIDE] = key;
    return (uint32_t)(lst[(k - 1) * TB_LIST_STRIDE] >> 32);
}

// Per CTA: queries [qb * 128, +128) x data tiles [slice range).  Output:
// out[(slice * nq + q) * k + t] = (dist << 32 | id) sorted ascending,
// all-ones for missing entries.
__global__ void __launch_bounds__(TB_THREADS, 1)
k_bf_tc_u8(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_x, int64_t nq,
           int64_t nx, int nkb, const int32_t *__restrict__ qnorm, const int32_t *__restrict__ xnorm,
           const int64_t *__restrict__ qself, int k, int64_t tiles_per_slice, uint64_t *__restrict__ out) {
    extern __shared__ uint8_t tb_raw[];
    const uint32_t raw = smem_u32(tb_raw);
    uint8_t *base = tb_raw + (((raw + 1023u) & ~1023u) - raw);
    uint8_t *sA = base;
    uint8_t *sB = sA + (size_t)nkb * TB_A_BYTES;
    uint64_t *lists = reinterpret_cast<uint64_t *>(sB + (size_t)TB_STAGES * TB_B_BYTES);
    uint64_t *bars = lists + (size_t)TB_LIST_STRIDE * k;
    uint64_t *full = bars, *empty = bars + TB_STAGES, *tfull = bars + 2 * TB_STAGES,
             *tempty = tfull + 2, *abar = tempty + 2;
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(abar + 1);

    const int warp = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    const int64_t q0 = (int64_t)blockIdx.x * TB_M;
    const int64_t ntiles_all = (nx + TB_N - 1) / TB_N;
    const int64_t t_lo = (int64_t)blockIdx.y * tiles_per_slice;
    const int64_t t_hi = t_lo + tiles_per_slice < ntiles_all ? t_lo + tiles_per_slice : ntiles_all;
    const int64_t ntiles = t_hi > t_lo ? t_hi - t_lo : 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < TB_STAGES; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; a++) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], TB_EPI_WARPS);
        }
        mbar_init(abar, 1);
    }
    if (warp == 1) {
        // 512 columns: two 256-column s32 accumulators
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (warp >= 2) {
        const int i = threadIdx.x - 64;
        for (int t = 0; t < k; t++) lists[t * TB_LIST_STRIDE + i] = ~0ull;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *s_tmem;

    if (warp == 0) {
        if (lane == 0) {
            mbar_expect_tx(abar, (uint32_t)nkb * TB_A_BYTES);
            for (int kb = 0; kb < nkb; kb++) tb_tma_2d(sA + (size_t)kb * TB_A_BYTES, &tm_q, kb * TB_KB, (int)q0, abar);
            int st = 0;
            uint32_t ph = 0;
            for (int64_t t = 0; t < ntiles; t++) {
                const int row0 = (int)((t_lo + t) * TB_N);
                for (int kb = 0; kb < nkb; kb++) {
                    mbar_wait(&empty[st], ph ^ 1);
                    mbar_expect_tx(&full[st], TB_B_BYTES);
                    tb_tma_2d(sB + (size_t)st * TB_B_BYTES, &tm_x, kb * TB_KB, row0, &full[st]);
                    if (++st == TB_STAGES) { st = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            mbar_wait(abar, 0);
            tc_fence_after();
            const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
            int st = 0;
            uint32_t ph = 0, aph = 0;
            for (int64_t t = 0; t < ntiles; t++) {
                const int acc = (int)(t & 1);
                mbar_wait(&tempty[acc], aph ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(acc * TB_N);
                for (int kb = 0; kb < nkb; kb++) {
                    mbar_wait(&full[st], ph);
                    tc_fence_after();
                    const uint64_t ad = tb_desc(a0 + (uint32_t)kb * TB_A_BYTES);
                    const uint64_t bd = tb_desc(b0 + (uint32_t)st * TB_B_BYTES);
#pragma unroll
                    for (int kk = 0; kk < TB_KB / 32; kk++)
                        tc_mma_i8(d, ad + 2 * kk, bd + 2 * kk, TB_IDESC, (kb | kk) != 0);
                    tc_commit(&empty[st]);  // the stage is free once these MMAs retire
                    if (++st == TB_STAGES) { st = 0; ph ^= 1; }
                }
                tc_commit(&tfull[acc]);  // accumulator ready for the epilogue
                if (acc == 1) aph ^= 1;
            }
        }
        __syncwarp();
    } else {
        const int ew = warp - 2;            // 0..7
        const int quad = warp & 3;          // TMEM lane quadrant this warp may read
        const int half = ew >> 2;           // column half [half * 128, +128)
        const int i = threadIdx.x - 64;     // list owner index
        uint64_t *lst = lists + i;
        const int64_t q = q0 + quad * 32 + (int)lane;
        const bool live = q < nq;
        const int32_t nqv = live ? __ldg(qnorm + q) : 0;
        const int64_t self = (live && qself) ? __ldg(qself + q) : -1;
        uint32_t worst = 0xffffffffu;
        uint32_t aph = 0;
        for (int64_t t = 0; t < ntiles; t++) {
            const int acc = (int)(t & 1);
            mbar_wait(&tfull[acc], aph);
            tc_fence_after();
            const int64_t col0 = (t_lo + t) * TB_N + half * 128;
#pragma unroll 1
            for (int c = 0; c < 4; c++) {
                int32_t v[32];
                tc_ld32(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * TB_N + half * 128 + c * 32), v);
                const int64_t cb = col0 + c * 32;
                // |x|^2 of these 32 columns (the same for every lane: broadcast loads)
                int32_t xn[32];
                if (cb + 32 <= nx) {
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        const int4 w4 = __ldg(reinterpret_cast<const int4 *>(xnorm + cb + j));
                        xn[j] = w4.x; xn[j + 1] = w4.y; xn[j + 2] = w4.z; xn[j + 3] = w4.w;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 32; j++) xn[j] = cb + j < nx ? __ldg(xnorm + cb + j) : 0x7fffffff;
                }
                if (live) {
#pragma unroll
                    for (int j = 0; j < 32; j++) {
                        const uint32_t dist = (uint32_t)(nqv + xn[j] - 2 * v[j]);
                        if (dist < worst && cb + j < nx && cb + j != self)
                            worst = tb_insert(lst, k, ((uint64_t)dist << 32) | (uint32_t)(cb + j));
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) tb_arrive(&tempty[acc]);
            if (acc == 1) aph ^= 1;
        }
        // merge the two column halves of each query (threads i and i + 128)
        asm volatile("bar.sync 1, %0;" ::"r"(TB_EPI_WARPS * 32) : "memory");
        if (half == 0 && live) {
            const uint64_t *a = lists + i, *b = lists + i + 128;
            uint64_t *o = out + ((int64_t)blockIdx.y * nq + q) * k;
            int ia = 0, ib = 0;
            for (int t = 0; t < k; t++) {
                const uint64_t va = a[ia * TB_LIST_STRIDE], vb = b[ib * TB_LIST_STRIDE];
                if (va <= vb) { o[t] = va; ia++; } else { o[t] = vb; ib++; }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

// S sorted partial lists per query -> the top k, as (local id or -1, exact
// fp64 distance or +inf).
__global__ void k_bf_tc_finish(const uint64_t *__restrict__ part, int64_t nq, int k, int S, int32_t *out_ids,
                               double *out_dists) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
        int head[16];
        for (int s = 0; s < S; s++) head[s] = 0;
        for (int t = 0; t < k; t++) {
            uint64_t best = ~0ull;
            int bs = -1;
            for (int s = 0; s < S; s++) {
                if (head[s] >= k) continue;
                const uint64_t v = part[((int64_t)s * nq + q) * k + head[s]];
                if (v < best) { best = v; bs = s; }
            }
            if (bs >= 0) head[bs]++;
            const bool real = best != ~0ull;
            out_ids[q * k + t] = real ? (int32_t)(uint32_t)best : -1;
            out_dists[q * k + t] = real ? (double)(uint32_t)(best >> 32) : __longlong_as_double(0x7ff0000000000000LL);
        }
    }
}

// Query rows gathered into a dense u8 matrix (row stride rb bytes) with
// their norms (certified data: the rows of the union copy).
__global__ void k_bf_gather_u8(const uint8_t *__restrict__ src, int rb, const int32_t *__restrict__ norms,
                               const int64_t *__restrict__ rows, int64_t nq, uint8_t *__restrict__ dst,
                               int32_t *__restrict__ qn) {
    const int vec = rb / 16;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nq * vec;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = i / vec;
        const int c = (int)(i % vec);
        const int64_t r = rows[q];
        reinterpret_cast<int4 *>(dst + q * rb)[c] = reinterpret_cast<const int4 *>(src + r * rb)[c];
        if (c == 0) qn[q] = norms[r];
    }
}

}  // namespace knnm

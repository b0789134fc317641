// knnm_tcjoin.cuh -- the local join's screen on the 5th-generation tensor
// cores, for the lazy route (non-certified L2 rows longer than lazy_min_d,
// config 3: d = 960): the hood's Gram block is computed EXACTLY in integers
// by tcgen05.mma kind::i8 on a 24-bit fixed-point image of the rows, which
// gives a rigorous lower bound of every pair's reference distance; the
// bound goes into the lazy slot and the apply evaluates the exact fp64
// value only when the bound can still beat the row's current worst
// (reference: _kernels.py:43-80 dense_dist, 402-437 fill_pairs; the slot
// layout and emission are k_join_chunked's).
//
// Fixed point (non-negative data, max value <= 2^e): Q = min(floor(x 2^(24-e)),
// 2^24 - 1), three u8 limbs Q = L0 2^16 + L1 2^8 + L2, stored as limb planes
// (row r: [L0 | L1 | L2], each dg = roundup(d, 16) bytes).  With
// s = 2^(e-24), 0 <= x - Q s <= s, and for a pair
//   S = sum Qx Qy = G0 2^32 + G1 2^24 + G2 2^16 + G3 2^8 + G4,
//   G0 = L0.L0, G1 = L0.L1 + L1.L0, G2 = L0.L2 + L1.L1 + L2.L0 (int32, exact)
// and G3, G4 >= 0 bounded by d (2 255^2 2^8 + 255^2).  So
//   x.y <= s^2 (S_low + Dmax) + s (sum x + sum y) + d s^2,
//   L2 = |x|^2 + |y|^2 - 2 x.y >= |x|^2 + |y|^2 - 2 (that),
// and the reference's sequential fp64 sum is >= L2 (1 - (d + 3) 2^-53).
//
// One CTA per SM (8 warps) walks its hoods as one stream of (hood, two
// 128-byte K blocks) items through a ring of shared-memory stages filled by 16-byte
// cp.async (manual 128-byte swizzle), LA items ahead of the tensor core:
// the row gathers of the next items are in flight while the current item's
// MMAs and the finished hood's epilogue run.  A stage holds the three limb
// tiles of the hood's members back to back (npw = roundup(W, 16) rows
// each); the M = 128 MMA reads 128 rows from a tile's start, the rows past
// the hood being whatever follows (don't-care rows of the output).  One
// thread issues the six limb products per 32-byte K step (A = B = the same
// tiles, N = the hood's width rounded to 16) into three s32 accumulators in
// TMEM (two sets, by hood parity, so a hood's epilogue -- warps (q, q + 4)
// read TMEM lane quarter q with tcgen05.ld and emit the pairs of their rows
// -- runs one item later, while the next hood's MMAs proceed).
#pragma once

#include <cstdint>

#include "knnm_bf.cuh"

namespace knnm {

constexpr int TJC_THREADS = 512;  // 16 warps (roles: see k_join_tc)
constexpr int TJC_KB = 128;          // K bytes per block (one swizzle atom row)
#ifndef KNNM_TJC_KI
#define KNNM_TJC_KI 2
#endif
constexpr int TJC_KI = KNNM_TJC_KI;   // K blocks per ring item
constexpr int TJC_MAX_W = 80;        // 3 accumulators x 80 columns <= 256
constexpr int TJC_MAX_STAGES = 16;
constexpr size_t TJC_SMEM_CAP = 200 * 1024;
constexpr double TJC_GMAX_TAIL = 33357825.0;  // 2 255^2 2^8 + 255^2 (dropped G3, G4 per dim)

// ring geometry for hood width W: stage stride 3 npw 128 B, plus the last
// tile's 128-row read-over
__host__ __device__ inline int tjc_npw(int W) { return (W + 15) & ~15; }
__host__ __device__ inline size_t tjc_stage_bytes(int W) { return (size_t)3 * TJC_KI * tjc_npw(W) * TJC_KB; }
__host__ __device__ inline size_t tjc_tail_bytes(int W) { return (size_t)(128 - tjc_npw(W)) * TJC_KB; }
__host__ inline int tjc_stages(int W) {
    const size_t avail = TJC_SMEM_CAP - 1024 - tjc_tail_bytes(W);
    const int s = (int)(avail / tjc_stage_bytes(W));
    return s < TJC_MAX_STAGES ? s : TJC_MAX_STAGES;
}
__host__ inline size_t tjc_smem_bytes(int W, int stages) {
    return 1024 + (size_t)stages * tjc_stage_bytes(W) + tjc_tail_bytes(W);
}

struct TjcMeta {
    int id[TJC_MAX_W];
    uint8_t pos[TJC_MAX_W];
    uint8_t nw[TJC_MAX_W];
    uint8_t sc[TJC_MAX_W];
    double w[TJC_MAX_W];   // round-start worst
    double nx[TJC_MAX_W];  // |x|^2 (fp64, sequential: within d 2^-53 of the real value)
    double ax[TJC_MAX_W];  // sum x (upper bound)
    uint64_t st[TJC_MAX_W];
    PosPrefix P;
    int width;
};

// instruction descriptor: kind::i8, D s32, A/B u8 K-major, M = 128, N = n
__device__ __forceinline__ uint32_t tjc_idesc(int n) {
    return (2u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ void tc_ld16(uint32_t taddr, int32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tc_ld4(uint32_t taddr, int32_t (&v)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(taddr));
}
template <int CB>
__device__ __forceinline__ void tc_ldn(uint32_t taddr, int32_t (&v)[CB]) {
    if constexpr (CB == 16) tc_ld16(taddr, v);
    else tc_ld4(taddr, v);
}
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// One lane of the (converged) warp; the compiler then knows the region is
// single-threaded and feeds tcgen05.mma from uniform registers directly
// (with `lane == 0` it wraps every MMA in a vote/branch loop).
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n .reg .b32 rx;\n .reg .pred px;\n elect.sync rx|px, 0xffffffff;\n selp.u32 %0, 1, 0, px;\n}\n"
        : "=r"(pred));
    return pred != 0;
}

__device__ __forceinline__ void cp16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}

// A hood's length and neighbour entries, loaded one hood ahead of their use
// (the classification warps are a chain of dependent global loads: hood id
// -> length / entries -> per-member gathers; without the look-ahead two
// warps delivered a hood every 2.6 us, the floor of the whole kernel).
struct TjcPre {
    int w;
    uint32_t ev[4];
};
__device__ __forceinline__ void tjc_prefetch(TjcPre &p, bool ok, int64_t u, const uint32_t *__restrict__ nbh,
                                             const int32_t *__restrict__ nlen, int W, unsigned lane) {
    p.w = ok ? __ldg(nlen + u) : 0;
#pragma unroll
    for (int b = 0; b < 4; b++) {
        const int j = b * 32 + (int)lane;
        p.ev[b] = (ok && j < W) ? __ldg(nbh + u * W + j) : 0u;  // masked by the length below
    }
}

// classification warp: members of hood u in class order (as k_join_chunked) into m
__device__ __forceinline__ void tjc_classify(TjcMeta &m, int64_t u, const TjcPre &pre, int W, int mode,
                                             const double *__restrict__ nx, const double *__restrict__ ax,
                                             const double *__restrict__ worst0, const uint64_t *__restrict__ boff,
                                             const uint32_t *__restrict__ start, unsigned lane) {
    const int w = pre.w;
    uint32_t ev[4];
    int clsv[4];
    int cnts[4] = {0, 0, 0, 0};
#pragma unroll
    for (int b = 0; b < 4; b++) {
        const int j = b * 32 + (int)lane;
        ev[b] = j < w ? pre.ev[b] : 0u;
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
            m.id[slot] = id;
            m.pos[slot] = (uint8_t)j;
            m.nw[slot] = (uint8_t)(ev[b] & 1);
            m.sc[slot] = (uint8_t)c;
            m.w[slot] = worst0[id];
            m.nx[slot] = nx[id];
            m.ax[slot] = ax[id];
            m.st[slot] = boff[id] + start[u * W + j];
        }
    }
    build_pos_prefix(m.P, clsv, mode, lane);
    if (lane == 0) m.width = w;
}

// epilogue of one hood by 8 warps.  A warp may read only the TMEM lane
// quarter warp % 4 (rows 32 q4 ..), so the warps of a quarter split the
// columns: blocks of CB columns dealt round-robin to the quarter's `nparts`
// warps (part = this warp's index among them); each thread emits the
// admissible pairs (i = its row, j > i).  Hoods of up to 64 members occupy
// quarters 0 and 1 only: four warps per quarter with 4-column blocks
// (k_join_tc's narrow layout) instead of two with 16-column blocks.
template <int CB>
__device__ __forceinline__ void tjc_epilogue(const TjcMeta &m, uint32_t tacc, int npw, int mode, int d, double s,
                                             double *__restrict__ Bd, int32_t *__restrict__ Bs, int q4, int part,
                                             int nparts, unsigned lane) {
    const double s2 = s * s;
    const double eps = ldexp(1.0, -50);
    const double tail = (double)d * TJC_GMAX_TAIL;
    const double nrel = 1.0 - (double)(d + 4) * ldexp(1.0, -53);
    const double lrel = 1.0 - (double)(d + 8) * ldexp(1.0, -53);
    const int w = m.width;
    const int npad = (w + 15) & ~15;
    const int i = q4 * 32 + (int)lane;
    const bool rowok = i < w;
    const int ri = rowok ? i : 0;
    const double nxi = m.nx[ri], axi = m.ax[ri], wi = m.w[ri];
    const int newi = m.nw[ri], sci = m.sc[ri], posi = m.pos[ri], idi = m.id[ri];
    const uint64_t sti = m.st[ri];
    const int labi = sci >> 1;
    for (int c0 = part * CB; c0 < npad; c0 += nparts * CB) {
        if (q4 * 32 >= w || c0 + CB - 1 <= q4 * 32) continue;  // no pair (i < j < w) here (warp-uniform)
        int32_t g0[CB], g1[CB], g2[CB];
        const uint32_t ta = tacc + ((uint32_t)(q4 * 32) << 16) + (uint32_t)c0;
        tc_ldn<CB>(ta, g0);
        tc_ldn<CB>(ta + (uint32_t)npw, g1);
        tc_ldn<CB>(ta + 2u * (uint32_t)npw, g2);
        tc_wait_ld();
        if (!rowok) continue;
#pragma unroll
        for (int tt = 0; tt < CB; tt++) {
            const int j = c0 + tt;
            if (j <= i || j >= w) continue;
            // admissible (_kernels.py:391-399) and at least one new
            const int labj = m.sc[j] >> 1;
            if (!(newi || m.nw[j])) continue;
            if (mode == 1 && labi == labj) continue;
            if (mode == 2 && !(labi != labj || labi == 1)) continue;
            const long long sl = ((long long)g0[tt] << 32) + ((long long)g1[tt] << 24) + ((long long)g2[tt] << 16);
            double up = ((double)sl + tail) * s2 * (1.0 + eps);
            up = (up + s * (axi + m.ax[j]) * (1.0 + eps) + (double)d * s2) * (1.0 + eps);
            double lbv = (nxi + m.nx[j]) * nrel - 2.0 * up;
            lbv = lbv > 0.0 ? lbv * lrel : 0.0;
            const double dd = -lbv;  // approximate slot (sign bit set, -0.0 included)
            const int pj = m.pos[j];
            if (lbv < wi) {
                const uint64_t sij = sti + pair_rank(m.P, mode, sci, posi, pj);
                Bd[sij] = dd;
                Bs[sij] = m.id[j];
            }
            if (lbv < m.w[j]) {
                const uint64_t sji = m.st[j] + pair_rank(m.P, mode, m.sc[j], pj, posi);
                Bd[sji] = dd;
                Bs[sji] = idi;
            }
        }
    }
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// arrives on bar when the calling thread's earlier cp.async copies have landed
__device__ __forceinline__ void cp_async_arrive(uint64_t *bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// 16-byte copy, or 16 zero bytes when !valid (src-size 0)
__device__ __forceinline__ void cp16z(uint32_t dst, const void *src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0)
                 : "memory");
}

// Warp roles (mbarrier handshakes, no CTA-wide barrier in the steady state):
//   MMA (one elected lane)  item t waits full[t % S], issues the limb MMAs,
//                     commits empty[t % S]; a hood's last item also commits
//                     accf[hood % NS]
//   classify (2 warps)  members of hood h (warp h % 2) into meta[h % R] once
//                     hood h - R's epilogue released it -> metaf
//   loaders (5 warps)  row gathers: item t into stage t % S once the MMAs of
//                     item t - S retired (cp.async, arrive-on-completion)
//   epilogue (8 warps)  hood h from TMEM set h % NS -> acce[h % NS], metae[h % R]
// A warp reads only the TMEM lane quarter warp % 4, and a hood's rows sit in
// lanes 0 .. w - 1.  Narrow hoods (W <= 64, the usual case) therefore put
// all eight epilogue warps on quarters 0 and 1 -- warps {0,4,8,12} and
// {1,5,9,13}, four column parts each -- and the other roles on the warps
// of quarters 2 and 3 (MMA 3; classify 7, 11; loaders 2, 6, 10, 14, 15).
// Wide hoods keep two epilogue warps per quarter (MMA 0; classify 1-2;
// loaders 3-7; epilogue 8-15).  With the epilogue on two warps per busy
// quarter it, not the tensor core, set the pace (19.3 -> 11.6 ms without it).
// NS = accumulator sets that fit TMEM's 512 columns (3 for W <= 48), so the
// tensor core runs up to NS - 1 hoods ahead of the epilogue.
#ifndef KNNM_TJC_R
#define KNNM_TJC_R 4
#endif
constexpr int TJC_R = KNNM_TJC_R;     // member-metadata ring (hoods)
constexpr int TJC_LOADERS = 5 * 32;   // five loader warps

__global__ void __launch_bounds__(TJC_THREADS, 1)
k_join_tc(const int32_t *__restrict__ active, int nactive, const uint32_t *__restrict__ nbh,
          const int32_t *__restrict__ nlen, int W, int mode, const uint8_t *__restrict__ limbs, int dg, int d,
          int stages, const double *__restrict__ nx, const double *__restrict__ ax, double s,
          const double *__restrict__ worst0, const uint64_t *__restrict__ boff,
          const uint32_t *__restrict__ start, double *__restrict__ Bd, int32_t *__restrict__ Bs) {
    extern __shared__ uint8_t tjc_raw[];
    __shared__ TjcMeta meta[TJC_R];
    __shared__ __align__(8) uint64_t s_full[TJC_MAX_STAGES], s_empty[TJC_MAX_STAGES];
    __shared__ __align__(8) uint64_t s_metaf[TJC_R], s_metae[TJC_R], s_accf[4], s_acce[4];
    __shared__ uint32_t s_tmem;
    const uint32_t sbase = (smem_u32(tjc_raw) + 1023u) & ~1023u;
    const int tid = threadIdx.x;
    const unsigned lane = lane_id();
    const int warp = tid >> 5;
    const int nkb = (dg + TJC_KB - 1) / TJC_KB;  // 128-byte K blocks per row
    const int nki = (nkb + TJC_KI - 1) / TJC_KI;  // items per hood
    const int rowb = 3 * dg;                      // limb-plane row stride (global)
    const int npw = tjc_npw(W);
    const uint32_t tile = (uint32_t)npw * TJC_KB;  // one (limb, K block) tile of a stage
    const uint32_t sstride = 3u * TJC_KI * tile;
    const int nh = (int)blockIdx.x < nactive ? (nactive - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const int T = nh * nki;
    const int ns0 = 512 / (3 * npw), NS = ns0 < 4 ? ns0 : 4;  // accumulator sets
    // roles (see above): 0 MMA, 1 classify, 2 loader, 3 epilogue; idx = index within the role
    const bool wide = W > 64;
    int role, idx;
    if (wide) {
        role = warp == 0 ? 0 : warp <= 2 ? 1 : warp < 8 ? 2 : 3;
        idx = warp == 0 ? 0 : warp <= 2 ? warp - 1 : warp < 8 ? warp - 3 : (warp - 8) >> 2;
    } else if ((warp & 3) <= 1) {
        role = 3;
        idx = warp >> 2;
    } else if (warp == 3) {
        role = 0;
        idx = 0;
    } else if (warp == 7 || warp == 11) {
        role = 1;
        idx = warp == 7 ? 0 : 1;
    } else {
        role = 2;
        idx = warp == 15 ? 4 : warp >> 2;  // 2, 6, 10, 14 -> 0..3; 15 -> 4
    }
    const int q4 = warp & 3, part = idx;  // epilogue: lane quarter, column part

    if (tid == 0) {
        for (int b = 0; b < stages; b++) {
            mbar_init(&s_full[b], TJC_LOADERS);
            mbar_init(&s_empty[b], 1);
        }
        for (int b = 0; b < TJC_R; b++) {
            mbar_init(&s_metaf[b], 32);
            mbar_init(&s_metae[b], 256);
        }
        for (int b = 0; b < 4; b++) {
            mbar_init(&s_accf[b], 1);
            mbar_init(&s_acce[b], 256);
        }
    }
    if (warp == 0) {  // NS accumulator sets of 3 x npw columns
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;

    if (role == 0) {
        if (elect_one()) {
            // The issuing thread is one instruction stream: everything it can
            // keep as a running counter (hood, K item, stage and accumulator
            // set with their barrier parities, the instruction descriptors) it
            // does -- a skeleton of this kernel without MMAs, copies and
            // epilogue took 5.4 of the kernel's 13.5 ms, all of it this
            // thread's index arithmetic (runtime divisions per item).
            const uint32_t i3 = tjc_idesc(3 * npw), i2 = tjc_idesc(2 * npw), i1 = tjc_idesc(npw);
            int h = 0, kq = 0, st = 0, hs = 0;      // hood, item of the hood, stage, accumulator set
            uint32_t fph = 0, aph = 0;              // parities of full[st] and of acce[hs]'s previous use
            for (int t = 0; t < T; t++) {
                if (kq == 0) {
                    mbar_wait(&s_metaf[h % TJC_R], (uint32_t)(h / TJC_R) & 1u);
                    if (h >= NS) mbar_wait(&s_acce[hs], aph ^ 1u);
                }
                mbar_wait(&s_full[st], fph);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                tc_fence_after();
                const uint32_t sb = sbase + (uint32_t)st * sstride;
                // The limb tiles of a K block lie back to back ([L0 | L1 | L2],
                // npw rows each), so one MMA with N = 3 npw takes L0 against
                // all three (G0, G1, G2 partial), N = 2 npw takes L1 against
                // [L0 | L1] (G1, G2) and N = npw takes L2 against L0 (G2):
                // three instructions per K step instead of six, same products.
                const uint32_t acc = tmem + (uint32_t)(hs * 3 * npw);
                const uint32_t d0 = acc, d1 = acc + (uint32_t)npw, d2 = acc + 2u * (uint32_t)npw;
                // Same-shape MMAs back to back: the three products write
                // overlapping accumulator columns with different N, and the
                // tensor core drains between such instructions (interleaved
                // per K step they ran at ~120 cycles each, three times the
                // pipelined rate).  Integer sums: the order is free.
#pragma unroll
                for (int p3 = 0; p3 < 3; p3++) {
#pragma unroll
                    for (int j = 0; j < TJC_KI; j++) {
                        const int kb = kq * TJC_KI + j;
                        if (kb >= nkb) break;
                        const uint64_t b0 = tb_desc(sb + (uint32_t)(3 * j) * tile);
                        const uint64_t bp = tb_desc(sb + (uint32_t)(3 * j + p3) * tile);
#pragma unroll
                        for (int kk = 0; kk < TJC_KB / 32; kk++) {
                            if (p3 == 0) tc_mma_i8(d0, b0 + 2 * kk, b0 + 2 * kk, i3, (kb | kk) == 0 ? 0u : 1u);  // L0 x [L0 | L1 | L2]
                            else if (p3 == 1) tc_mma_i8(d1, bp + 2 * kk, b0 + 2 * kk, i2, 1u);  // L1 x [L0 | L1]
                            else tc_mma_i8(d2, bp + 2 * kk, b0 + 2 * kk, i1, 1u);               // L2 x L0
                        }
                    }
                }
                tc_commit(&s_empty[st]);
                if (++st == stages) {
                    st = 0;
                    fph ^= 1u;
                }
                if (++kq == nki) {  // the hood's last item: its accumulators are complete
                    tc_commit(&s_accf[hs]);
                    kq = 0;
                    h++;
                    if (++hs == NS) {
                        hs = 0;
                        aph ^= 1u;
                    }
                }
            }
        }
        __syncwarp();
    } else if (role == 1) {
        // two register sets (A: this warp's even turns, B: odd) so a
        // prefetched hood is consumed without register moves
        auto hood_of = [&](int h) { return h < nh ? (int64_t)__ldg(active + blockIdx.x + (int64_t)h * gridDim.x) : 0; };
        auto step = [&](int h, int64_t u, const TjcPre &pre) {
            const int slot = h % TJC_R;
            if (h >= TJC_R) mbar_wait(&s_metae[slot], (uint32_t)((h - TJC_R) / TJC_R) & 1u);
            tjc_classify(meta[slot], u, pre, W, mode, nx, ax, worst0, boff, start, lane);
            __syncwarp();
            mbar_arrive(&s_metaf[slot]);
        };
        int h = idx;
        int64_t uA = hood_of(h), uB = hood_of(h + 2);
        TjcPre pA, pB;
        tjc_prefetch(pA, h < nh, uA, nbh, nlen, W, lane);
        for (; h < nh; h += 4) {
            tjc_prefetch(pB, h + 2 < nh, uB, nbh, nlen, W, lane);
            const int64_t uA2 = hood_of(h + 4);
            step(h, uA, pA);
            if (h + 2 >= nh) break;
            tjc_prefetch(pA, h + 4 < nh, uA2, nbh, nlen, W, lane);
            const int64_t uB2 = hood_of(h + 6);
            step(h + 2, uB, pB);
            uA = uA2;
            uB = uB2;
        }
    } else if (role == 2) {
        // thread -> (16-byte column c of the item's KI K blocks, rows r0,
        // r0 + rstep, ...): the column, its K block and the swizzle phase are
        // fixed per thread; each step copies the three limbs of one row chunk
        static_assert(TJC_LOADERS % (8 * TJC_KI) == 0, "loader threads per row chunk set");
        const int lt = idx * 32 + (int)lane;  // 0 .. TJC_LOADERS - 1
        const int c = lt & (8 * TJC_KI - 1), r0 = lt / (8 * TJC_KI);
        constexpr int rstep = TJC_LOADERS / (8 * TJC_KI);
        const int j = c >> 3, c16 = c & 7;
        int h = 0, kq = 0, st = 0;  // running counters instead of divisions per item
        uint32_t eph = 1;           // parity of empty[st]'s previous use (first pass: nothing to wait for)
        for (int t = 0; t < T; t++) {
            if (t >= stages) mbar_wait(&s_empty[st], eph);
            if (kq == 0) mbar_wait(&s_metaf[h % TJC_R], (uint32_t)(h / TJC_R) & 1u);
            const TjcMeta &m = meta[h % TJC_R];
            const int w = m.width;
            if (kq * TJC_KI + j < nkb) {  // else: block past the row, no MMA reads it
                const int col = kq * TJC_KI * TJC_KB + c * 16;
                const bool in = col < dg;  // columns past the padded row read as zero
                const uint8_t *src0 = limbs + (in ? col : 0);
                const uint32_t db = sbase + (uint32_t)st * sstride + (uint32_t)(3 * j) * tile;
                for (int r = r0; r < w; r += rstep) {
                    const uint8_t *src = src0 + (int64_t)m.id[r] * rowb;
                    const uint32_t dst = db + (uint32_t)r * 128u + (uint32_t)((c16 ^ (r & 7)) << 4);
                    cp16z(dst, src, in);
                    cp16z(dst + tile, src + dg, in);
                    cp16z(dst + 2u * tile, src + 2 * dg, in);
                }
            }
            cp_async_arrive(&s_full[st]);
            if (++st == stages) {
                st = 0;
                eph ^= 1u;
            }
            if (++kq == nki) {
                kq = 0;
                h++;
            }
        }
    } else {
        for (int h = 0; h < nh; h++) {
            const int slot = h % TJC_R;
            mbar_wait(&s_metaf[slot], (uint32_t)(h / TJC_R) & 1u);
            mbar_wait(&s_accf[h % NS], (uint32_t)(h / NS) & 1u);
            tc_fence_after();
            if (wide)
                tjc_epilogue<16>(meta[slot], tmem + (uint32_t)((h % NS) * 3 * npw), npw, mode, d, s, Bd, Bs, q4,
                                 part, 2, lane);
            else
                tjc_epilogue<4>(meta[slot], tmem + (uint32_t)((h % NS) * 3 * npw), npw, mode, d, s, Bd, Bs, q4,
                                part, 4, lane);
            tc_fence_before();
            mbar_arrive(&s_acce[h % NS]);
            mbar_arrive(&s_metae[slot]);
        }
    }
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

// Limb planes of the union rows (fixed point of non-negative rows, see the
// header) plus |x|^2 (fp64, sequential) and an upper bound of sum x.
__global__ void k_make_limbs(const float *__restrict__ sub, int dp, int d, int64_t n, int dg, double scale,
                             uint8_t *__restrict__ limbs, double *__restrict__ nx, double *__restrict__ ax) {
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n;
         r += (int64_t)gridDim.x * (blockDim.x >> 5)) {
        const unsigned lane = lane_id();
        uint8_t *o = limbs + r * (int64_t)(3 * dg);
        double sa = 0.0;
        for (int c = lane; c < dg; c += 32) {
            const float x = c < d ? sub[r * dp + c] : 0.f;
            double q = floor((double)x * scale);
            q = q < 0.0 ? 0.0 : q > 16777215.0 ? 16777215.0 : q;
            const uint32_t Q = (uint32_t)q;
            o[c] = (uint8_t)(Q >> 16);
            o[dg + c] = (uint8_t)(Q >> 8);
            o[2 * dg + c] = (uint8_t)Q;
            sa += (double)x;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) sa += __shfl_xor_sync(FULL_MASK, sa, off);
        if (lane == 0) {
            nx[r] = exact_sqnorm(sub + r * dp, d);
            ax[r] = sa * (1.0 + (double)(d + 4) * ldexp(1.0, -52));  // >= the real sum
        }
    }
}

}  // namespace knnm

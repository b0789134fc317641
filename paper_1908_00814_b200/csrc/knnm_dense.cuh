// knnm_dense.cuh -- the local join for non-certified short rows (config 4:
// d = 100 cosine; config 1: d = 32 L2 uniform): every admissible pair's
// exact fp64 distance from register-blocked fp64 tiles, no fp32 screen.
//
// Reference: _kernels.py:43-80 (dense_dist: per-dimension fp64 sums in index
// order, separate multiply and add), 391-399 (_pair_admissible), 402-437
// (fill_pairs order -> reference-order slots, as in k_join_tiled).
//
// Why no screen: with a round-start worst that passes most pairs (config 4:
// 63% of all pairs needed the exact value), screening in fp32 and
// re-evaluating survivors one pair per thread costs more than evaluating
// every pair exactly, if the exact evaluation is blocked so its operands
// come from registers: each lane holds a 4 x 2 tile of fp64 accumulators
// and reads two dimensions of its four rows and two columns per step (six
// 16-byte shared loads for 16 pair-dimensions).  The sums run in the
// reference's order per pair (t = 0 .. d-1, __dmul_rn then __dadd_rn), so
// every value is the reference's value bit for bit.
//
// Data flow (one CTA per SM, warp-specialised, no CTA-wide barrier in the
// hood loop):
//   k_dense_rec   one warp per active hood gathers what the join needs per
//                 member (nbh entry, round-start worst, first slot, cosine
//                 norm and root) into a fixed-size record in HBM;
//   k_join_dense  warp 0 (loader) bulk-copies the records into a ring of
//                 DJ_NRR shared slots and, as soon as a record is there, the
//                 member rows -- fp64 rows of the union (fp32 -> fp64 is
//                 exact; B200 converts at 16 lanes/clk/SM against 64 fp64
//                 ops, so rows are converted once per merge, not per hood)
//                 -- into a circular shared row buffer in nbh position order
//                 (mbarrier tx-count completion, up to DJ_NH hoods in
//                 flight; rows no rectangle touches are skipped);
//                 warp 1 (classifier) orders each hood's members by class
//                 and builds the pair-rank table and the rectangles;
//                 warps 2..15 (consumers) take 4 x 2-tile patches of the
//                 oldest ready hood from a per-hood counter and arrive on
//                 the hood's "empty" barrier when it has no patches left, so
//                 a warp moves on to the next hood while others finish the
//                 previous one; the loader reclaims rows and record slots in
//                 hood order.  (Loading and classifying in one warp delivered
//                 a hood every 4.7 us -- 38 of the 48 ms of config 4's first
//                 round with the arithmetic removed.)
// Shared rows have S = dp + 2 doubles (S / 2 odd: the rows a load touches
// start in distinct 16-byte bank groups).  Members are ordered by class
// (label, new first), so the admissible set of a hood is a union of at most
// four rectangles:
//   mode 1 (CROSS)       A_new x B          + A_old x B_new
//   mode 0 (ALL)         new x new (upper)  + new x old
//   mode 2 (CROSS_OR_S2) mode 1's two       + B_new x B_new (upper) + B_new x B_old
// (A = label 0, B = label 1); triangular rectangles skip patches below the
// diagonal.
#pragma once

#include "knnm_kernels.cuh"
#include "knnm_tcjoin.cuh"

namespace knnm {

constexpr int DJ_THREADS = 512;  // warp 0: loader; warp 1: classifier; warps 2..15: consumers
constexpr int DJ_CONS = DJ_THREADS / 32 - 2;
constexpr int DJ_NH = 8;         // hoods in flight (descriptor / barrier ring)
constexpr int DJ_NRR = 12;       // record slots (requested DJ_NRR - DJ_NH hoods ahead)
constexpr size_t DJ_SMEM_CAP = 225 * 1024;

__host__ __device__ inline int dj_stride(int dp) { return dp + 2; }  // doubles per shared row
// per-hood record (HBM, bulk-copied whole): header {int w}, then per member
// position: nbh entry (u32), round-start worst (f64), first slot (u64),
// [cosine: exact norm (f64), its root (f64)]
__host__ __device__ inline int dj_wr(int W) { return (W + 3) & ~3; }
__host__ __device__ inline int dj_rec_bytes(int W, bool cos) { return 16 + dj_wr(W) * (cos ? 36 : 20); }

// Lane tile: 4 rows x 2 columns of fp64 accumulators.  Two lane layouts,
// chosen per rectangle by padded area: lay 0 = 8 x 4 lanes (patch 32 x 8),
// lay 1 = 4 x 8 lanes (patch 16 x 16).  In both, the rows a quarter-warp
// reads are one address (2 shared wavefronts per 16-byte load; the columns'
// loads take 4).
__host__ __device__ inline int dj_prows(int lay) { return lay ? 16 : 32; }
__host__ __device__ inline int dj_pcols(int lay) { return lay ? 16 : 8; }

struct DjRect {
    int r0, r1, c0, c1, tri, lay, npc, pstart;
};

// One hood's class order (slot -> nbh position, class), pair-rank table and
// rectangles; the per-member values stay in the record, indexed by position.
struct __align__(16) DjMeta {
    uint8_t pos[MAX_W];
    uint8_t sc[MAX_W];
    PosPrefix P;
    DjRect rect[4];
    int nrect, npatch, width, next;
};

__host__ inline size_t dj_fixed_bytes(int W, bool cos) {
    return (size_t)DJ_NRR * dj_rec_bytes(W, cos) + DJ_NH * sizeof(DjMeta) +
           (3 * DJ_NH + DJ_NRR) * sizeof(uint64_t) + 2 * DJ_NH * sizeof(int);
}
// rows of the circular shared row buffer (0: a whole hood does not fit twice,
// the route does not apply)
__host__ inline int dj_rows(int W, int dp, bool cos) {
    const size_t row = (size_t)dj_stride(dp) * sizeof(double);
    const size_t fixed = dj_fixed_bytes(W, cos);
    if (fixed >= DJ_SMEM_CAP) return 0;
    const int C = (int)((DJ_SMEM_CAP - fixed) / row);
    return C >= 2 * W ? C : 0;
}
__host__ inline size_t dj_smem_bytes(int W, int dp, bool cos, int C) {
    return (size_t)C * dj_stride(dp) * sizeof(double) + dj_fixed_bytes(W, cos);
}

// 1 - dot / (|a| |b|) with the reference's special cases (_kernels.py:62-80);
// na, nb: the exact fp64 norms; sa, sb: their correctly rounded roots.
__device__ __forceinline__ double dj_cos_final(double dot, double na, double nb, double sa, double sb) {
    if (na == 0.0 || nb == 0.0) return (na == nb) ? 0.0 : 1.0;
    if (dot > 0.0 && __dmul_rn(dot, dot) >= __dmul_rn(na, nb)) return 0.0;
    const double r = __dsub_rn(1.0, __ddiv_rn(dot, __dmul_rn(sa, sb)));
    return r < 0.0 ? 0.0 : r;
}

template <int TAG>
__device__ __forceinline__ double dj_term(double acc, double x, double y) {
    if (TAG == 1) {
        const double df = __dsub_rn(x, y);
        return __dadd_rn(acc, __dmul_rn(df, df));
    }
    if (TAG == 0) return __dadd_rn(acc, fabs(__dsub_rn(x, y)));
    return __dadd_rn(acc, __dmul_rn(x, y));
}

// Per-hood records (see dj_rec_bytes): one warp per active hood.
template <bool COS>
__global__ void k_dense_rec(const int32_t *__restrict__ active, int nactive, const uint32_t *__restrict__ nbh,
                            const int32_t *__restrict__ nlen, int W, const double *__restrict__ worst0,
                            const uint64_t *__restrict__ boff, const uint32_t *__restrict__ start,
                            const double *__restrict__ nrm64, const double *__restrict__ nsq,
                            uint8_t *__restrict__ rec, int RB) {
    const unsigned lane = lane_id();
    const int Wr = dj_wr(W);
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t hi = gw; hi < nactive; hi += nw) {
        const int64_t u = active[hi];
        const int w = nlen[u];
        uint8_t *R = rec + hi * (int64_t)RB;
        uint32_t *E = reinterpret_cast<uint32_t *>(R + 16);
        double *W0 = reinterpret_cast<double *>(R + 16 + 4 * Wr);
        uint64_t *ST = reinterpret_cast<uint64_t *>(R + 16 + 12 * Wr);
        if (lane == 0) *reinterpret_cast<int *>(R) = w;
        for (int j = (int)lane; j < w; j += 32) {
            const uint32_t e = nbh[u * W + j];
            const int id = (int)(e >> 2);
            E[j] = e;
            W0[j] = worst0[id];
            ST[j] = boff[id] + start[u * W + j];
            if (COS) {
                reinterpret_cast<double *>(R + 16 + 20 * Wr)[j] = nrm64[id];
                reinterpret_cast<double *>(R + 16 + 28 * Wr)[j] = nsq[id];
            }
        }
    }
}

__global__ void k_to_f64(const float *__restrict__ src, int64_t total, double *__restrict__ dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = (double)src[i];
}

__global__ void k_sqrt64(const double *__restrict__ a, int64_t n, double *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = __dsqrt_rn(a[i]);
}

// Producer: order a hood's members by class (class = (label != 0) * 2 +
// !new, _kernels.py:391-399) from its record, build the pair-rank table and
// the rectangles.
__device__ __forceinline__ void dj_classify(DjMeta &M, const uint8_t *R, int mode, unsigned lane, int (&cnts)[4]) {
    const int w = *reinterpret_cast<const int *>(R);
    const uint32_t *E = reinterpret_cast<const uint32_t *>(R + 16);
    uint32_t ev[4];
    int clsv[4];
    cnts[0] = cnts[1] = cnts[2] = cnts[3] = 0;
#pragma unroll
    for (int b = 0; b < 4; b++) {
        const int j = b * 32 + (int)lane;
        ev[b] = j < w ? E[j] : 0u;
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
                M.pos[slot] = (uint8_t)j;
                M.sc[slot] = (uint8_t)c;
            }
            fill[c] += __popc(m);
        }
    }
    build_pos_prefix(M.P, clsv, mode, lane);
    if (lane == 0) {
        const int nAn = cnts[0], nA = cnts[0] + cnts[1], nBn = cnts[2];
        int nr = 0, np = 0;
        auto add = [&](int r0, int r1, int c0, int c1, int tri) {
            if (r1 > r0 && c1 > c0) {
                int h = r1 - r0, wd = c1 - c0;
                const int a0 = ((h + 31) & ~31) * ((wd + 7) & ~7), a1 = ((h + 15) & ~15) * ((wd + 15) & ~15);
                // a full rectangle may also run transposed (distances and
                // the emission are symmetric in the pair): 32 x 8 patches
                // along its long side, e.g. 5 new x 40 members -> 2 patches
                // instead of 3 (16 x 16) or 5 (32 x 8)
                const int a0t = tri ? 0x7fffffff : ((wd + 31) & ~31) * ((h + 7) & ~7);
                int lay = a1 < a0 ? 1 : 0;
                if (a0t < (lay ? a1 : a0)) {
                    lay = 0;
                    int t = r0; r0 = c0; c0 = t;
                    t = r1; r1 = c1; c1 = t;
                    t = h; h = wd; wd = t;
                }
                const int npc = (wd + dj_pcols(lay) - 1) / dj_pcols(lay);
                M.rect[nr++] = DjRect{r0, r1, c0, c1, tri, lay, npc, np};
                np += ((h + dj_prows(lay) - 1) / dj_prows(lay)) * npc;
            }
        };
        if (mode == 0) {
            add(0, nAn, 0, nAn, 1);
            add(0, nAn, nAn, w, 0);
        } else {
            add(0, nAn, nA, w, 0);
            add(nAn, nA, nA, nA + nBn, 0);
            if (mode == 2) {
                add(nA, nA + nBn, nA, nA + nBn, 1);
                add(nA, nA + nBn, nA + nBn, w, 0);
            }
        }
        M.nrect = nr;
        M.npatch = np;
        M.width = w;
        M.next = 0;
    }
}

template <int TAG>
__global__ void __launch_bounds__(DJ_THREADS, 1)
k_join_dense(int nactive, int W, int mode, const double *__restrict__ sub64, int dp, int d,
             const uint8_t *__restrict__ rec, int RB, int C, double *__restrict__ Bd, int32_t *__restrict__ Bs,
             unsigned long long *counters) {
    extern __shared__ __align__(128) uint8_t dsm[];
    const int S = dj_stride(dp), S2 = S >> 1;
    double *F0 = reinterpret_cast<double *>(dsm);  // C rows of S doubles (circular)
    uint8_t *R0 = dsm + (size_t)C * S * sizeof(double);
    DjMeta *M0 = reinterpret_cast<DjMeta *>(R0 + (size_t)DJ_NRR * RB);
    uint64_t *full = reinterpret_cast<uint64_t *>(M0 + DJ_NH);
    uint64_t *empty = full + DJ_NH;
    uint64_t *metaf = empty + DJ_NH;
    uint64_t *recb = metaf + DJ_NH;
    int *s_base = reinterpret_cast<int *>(recb + DJ_NRR);  // first ring row of the hood in slot h
    int *s_wid = s_base + DJ_NH;                           // its width (loader's release bookkeeping)
    __shared__ unsigned long long s_nev;
    const int tid = threadIdx.x;
    const unsigned lane = lane_id();
    const int warp = tid >> 5;
    const int Wr = dj_wr(W);
    const int J = ((int)blockIdx.x < nactive) ? (nactive - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
    const int n2 = (d + 1) >> 1;  // double2 steps (a padded odd dimension adds +0)
    if (tid == 0) {
        for (int h = 0; h < DJ_NH; h++) {
            mbar_init(&full[h], 1);
            mbar_init(&empty[h], DJ_CONS);
            mbar_init(&metaf[h], 1);
        }
        for (int r = 0; r < DJ_NRR; r++) mbar_init(&recb[r], 1);
        s_nev = 0;
    }
    __syncthreads();
    unsigned long long nev = 0;
    if (warp == 0) {
        // ------------------------------- loader -------------------------------
        // Hoods are released by the consumers in order; rel counts the
        // releases observed so far.  Hood j needs: ring slot j % NH (hood
        // j - NH released), its record (requested when hood j - NRR was
        // released), and w free rows in the circular buffer.  Rows go in
        // nbh position order, so the copies depend on the record alone (the
        // class order is the classifier warp's business: one warp doing
        // both delivered a hood every 4.7 us, 80% of the kernel's time).
        auto rec_req = [&](int j) {  // lane 0
            uint64_t *bar = &recb[j % DJ_NRR];
            mbar_expect_tx(bar, (uint32_t)RB);
            bulk_g2s(R0 + (size_t)(j % DJ_NRR) * RB, rec + ((int64_t)blockIdx.x + (int64_t)j * gridDim.x) * RB,
                     (uint32_t)RB, bar);
        };
        if (lane == 0)
            for (int j = 0; j < DJ_NRR && j < J; j++) rec_req(j);
        int rel = 0;
        int64_t head = 0, tail = 0;  // rows allocated / released (monotonic)
        auto release_one = [&]() {
            mbar_wait(&empty[rel % DJ_NH], (uint32_t)(rel / DJ_NH) & 1u);
            tail += s_wid[rel % DJ_NH];
            if (lane == 0 && rel + DJ_NRR < J) rec_req(rel + DJ_NRR);  // its record slot is free
            rel++;
        };
        const uint32_t row_bytes = (uint32_t)dp * 8u;
        for (int j = 0; j < J; j++) {
            while (rel < j - DJ_NH + 1) release_one();
            const int r = j % DJ_NRR, h = j % DJ_NH;
            mbar_wait(&recb[r], (uint32_t)(j / DJ_NRR) & 1u);
            const uint8_t *R = R0 + (size_t)r * RB;
            const int w = *reinterpret_cast<const int *>(R);
            while (head + w - tail > C) release_one();
            const uint32_t *E = reinterpret_cast<const uint32_t *>(R + 16);
            // Rows no rectangle touches are not fetched (their ring rows stay
            // stale): with A = label 0, B = label 1, old A members pair only
            // with new B members and old B members only with new A members
            // (modes 1, 2; mode 2's B x B block needs a new B member).
            uint32_t ev[4];
            int cls[4], cn[4] = {0, 0, 0, 0};
#pragma unroll
            for (int b = 0; b < 4; b++) {
                const int p = b * 32 + (int)lane;
                ev[b] = p < w ? E[p] : 0u;
                const int lab = mode == 0 ? 0 : (int)((ev[b] >> 1) & 1);
                cls[b] = p < w ? lab * 2 + ((ev[b] & 1) ? 0 : 1) : 4;
#pragma unroll
                for (int c = 0; c < 4; c++) cn[c] += __popc(__ballot_sync(FULL_MASK, cls[b] == c));
            }
            const bool needAo = mode == 0 || cn[2] > 0;
            const bool needBo = mode == 0 || cn[0] > 0 || (mode == 2 && cn[2] > 0);
            const int nfetch = cn[0] + (needAo ? cn[1] : 0) + cn[2] + (needBo ? cn[3] : 0);
            fence_proxy_async();  // the consumers' reads of the recycled rows vs. the bulk copies
            if (lane == 0) {
                s_base[h] = (int)(head % C);
                s_wid[h] = w;
                mbar_expect_tx(&full[h], row_bytes * (uint32_t)nfetch);
            }
            __syncwarp();
#pragma unroll
            for (int b = 0; b < 4; b++) {
                const int p = b * 32 + (int)lane;
                const bool need = cls[b] == 0 || cls[b] == 2 || (cls[b] == 1 && needAo) || (cls[b] == 3 && needBo);
                if (need)
                    bulk_g2s(F0 + (size_t)((head + p) % C) * S, sub64 + (int64_t)(ev[b] >> 2) * dp, row_bytes,
                             &full[h]);
            }
            head += w;
        }
    } else if (warp == 1) {
        // ----------------------------- classifier ----------------------------
        for (int j = 0; j < J; j++) {
            const int r = j % DJ_NRR, h = j % DJ_NH;
            if (j >= DJ_NH) mbar_wait(&empty[h], (uint32_t)((j - DJ_NH) / DJ_NH) & 1u);  // slot free
            mbar_wait(&recb[r], (uint32_t)(j / DJ_NRR) & 1u);
            int cn[4];
            dj_classify(M0[h], R0 + (size_t)r * RB, mode, lane, cn);
            __syncwarp();
            if (lane == 0) mbar_arrive(&metaf[h]);
        }
    } else {
        // ------------------------------ consumers -----------------------------
        const double2 *dv2 = reinterpret_cast<const double2 *>(F0);
        for (int j = 0; j < J; j++) {
            const int r = j % DJ_NRR, h = j % DJ_NH;
            mbar_wait(&metaf[h], (uint32_t)(j / DJ_NH) & 1u);
            mbar_wait(&full[h], (uint32_t)(j / DJ_NH) & 1u);
            DjMeta &M = M0[h];
            const uint8_t *R = R0 + (size_t)r * RB;
            const uint32_t *E = reinterpret_cast<const uint32_t *>(R + 16);
            const double *W0 = reinterpret_cast<const double *>(R + 16 + 4 * Wr);
            const uint64_t *ST = reinterpret_cast<const uint64_t *>(R + 16 + 12 * Wr);
            const double *N64 = reinterpret_cast<const double *>(R + 16 + 20 * Wr);
            const double *SQ = reinterpret_cast<const double *>(R + 16 + 28 * Wr);
            const int base = s_base[h];
            const int npatch = M.npatch, nrect = M.nrect;
            while (true) {
                int pid = 0;
                if (lane == 0) pid = atomicAdd(&M.next, 1);
                pid = __shfl_sync(FULL_MASK, pid, 0);
                if (pid >= npatch) break;
                int g = 0;
                while (g + 1 < nrect && pid >= M.rect[g + 1].pstart) g++;
                const DjRect Rc = M.rect[g];
                const int lp = pid - Rc.pstart;
                const int pr = lp / Rc.npc, pc = lp - pr * Rc.npc;
                const int R0r = Rc.r0 + pr * dj_prows(Rc.lay), C0 = Rc.c0 + pc * dj_pcols(Rc.lay);
                if (Rc.tri && R0r >= C0 + dj_pcols(Rc.lay) - 1) continue;  // all below the diagonal
                const int rs = Rc.lay ? 4 : 8, cs = Rc.lay ? 8 : 4;  // lane strides
                const int i0 = R0r + (Rc.lay ? (int)(lane >> 3) : (int)(lane >> 2));
                const int j0 = C0 + (Rc.lay ? (int)(lane & 7) : (int)(lane & 3));
                const double2 *pa[4], *pb[2];
#pragma unroll
                for (int m = 0; m < 4; m++) {  // ring rows are in nbh position order
                    int row = base + (int)M.pos[min(i0 + m * rs, Rc.r1 - 1)];
                    pa[m] = dv2 + (size_t)(row >= C ? row - C : row) * S2;
                }
#pragma unroll
                for (int n = 0; n < 2; n++) {
                    int row = base + (int)M.pos[min(j0 + n * cs, Rc.c1 - 1)];
                    pb[n] = dv2 + (size_t)(row >= C ? row - C : row) * S2;
                }
                double acc[4][2];
#pragma unroll
                for (int m = 0; m < 4; m++) acc[m][0] = acc[m][1] = 0.0;
#pragma unroll 2
                for (int t = 0; t < n2; t++) {
                    double2 a[4], b[2];
#pragma unroll
                    for (int m = 0; m < 4; m++) a[m] = pa[m][t];
#pragma unroll
                    for (int n = 0; n < 2; n++) b[n] = pb[n][t];
#pragma unroll
                    for (int m = 0; m < 4; m++)
#pragma unroll
                        for (int n = 0; n < 2; n++) acc[m][n] = dj_term<TAG>(acc[m][n], a[m].x, b[n].x);
#pragma unroll
                    for (int m = 0; m < 4; m++)
#pragma unroll
                        for (int n = 0; n < 2; n++) acc[m][n] = dj_term<TAG>(acc[m][n], a[m].y, b[n].y);
                }
#pragma unroll
                for (int s8 = 0; s8 < 8; s8++) {
                    const int ii = i0 + (s8 >> 1) * rs, jj = j0 + (s8 & 1) * cs;
                    if (!(ii < Rc.r1 && jj < Rc.c1 && (!Rc.tri || ii < jj))) continue;
                    nev++;
                    const double dot = acc[s8 >> 1][s8 & 1];
                    const int pi = M.pos[ii], pj = M.pos[jj];
                    const double wi = W0[pi], wj = W0[pj];
                    double dd;
                    if (TAG == 2) {
                        const double na = N64[pi], nb = N64[pj], sa = SQ[pi], sb = SQ[pj];
                        // cheap exclusion before the division: |q| <= ~1 for
                        // finite non-degenerate operands, fp32 error << 1e-5
                        const double p = __dmul_rn(sa, sb);
                        if (p > 1e-30 && p < 1e30 && fabs(dot) < 1e30) {
                            const float rf = 1.0f - __fdividef((float)dot, (float)p);
                            if ((double)rf > fmax(wi, wj) + 1e-5) continue;
                        }
                        dd = dj_cos_final(dot, na, nb, sa, sb);
                    } else {
                        dd = dot;
                    }
                    if (dd < wi) {  // id[ii] <- id[jj]
                        const uint64_t sij = ST[pi] + pair_rank(M.P, mode, M.sc[ii], pi, pj);
                        Bd[sij] = dd;
                        Bs[sij] = (int32_t)(E[pj] >> 2);
                    }
                    if (dd < wj) {  // id[jj] <- id[ii]
                        const uint64_t sji = ST[pj] + pair_rank(M.P, mode, M.sc[jj], pj, pi);
                        Bd[sji] = dd;
                        Bs[sji] = (int32_t)(E[pi] >> 2);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[h]);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nev += __shfl_xor_sync(FULL_MASK, nev, o);
    if (lane == 0 && nev) atomicAdd(&s_nev, nev);
    __syncthreads();
    if (tid == 0 && s_nev) atomicAdd(&counters[C_EXACT], s_nev);
}

}  // namespace knnm

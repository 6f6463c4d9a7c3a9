// stream_solve.cuh — the shared-LHS batched banded solve for the interleaved
// layout (pent_solve / tri_solve) as a persistent,
// warp-specialised, TMA-streamed two-phase partitioned solve for sm_100a.
//
// Why (measured on B200): a CTA that loads its whole share of
// a system group into registers, solves, and stores reaches only 3-4 TB/s
// even with no arithmetic; persistent CTAs that keep a ring of TMA tile loads
// in flight reach 5.6-6.3 TB/s.  So nothing is held on chip across CTAs: each
// system is cut into row tiles of R rows and every tile is visited twice.
//
//   P1(tile): TMA-load f (HBM); one lane per system sweeps the tile's rows
//             (the thesis's thread-per-system recurrence) with
//             zero tile inflows: g in place in shared memory, then the back
//             substitution streams the local solution y to global memory
//             (it stays in L2).  The tile's affine aggregates (forward carry
//             A_f, backward carry A_b) and, for cyclic systems, the forward
//             values on the Navon / Sherman–Morrison rows are published.
//   group scan: once every P1 tile of a group is counted, a designated CTA's
//             scan warp chains the aggregates along each system (lane per
//             system): tile inflows (Fin, Bin) and the periodic pair x_l
//             (eq:first_two).
//   P2(tile): TMA re-load y (L2) and apply x = y + RF Fin + RB Bin - Z x_l
//             (LHS-only response rows), store x.
//
// HBM traffic per unknown: f once, x once (16 B fp64); y and the O(1/R)
// aggregates live in the 126 MB L2 (P1 runs at most `lead` tiles ahead of
// P2).  FP64 work: 5 ops per unknown in P1 (+2 cyclic), 4-6 in P2 — no chunk
// scans inside a tile.  Tile-level algebra (LHS-only tables, tile_tables_kernel):
//   Fout = A_f + Mf_t Fin,   Bout = A_b + Hf_t Fin + Mb_t Bin,
//   y_true = y_local + RF Fin + RB Bin.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "band_core.cuh"

namespace pb {

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *b, int cnt)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity)
{
    asm volatile(
        "{\n .reg .pred p;\n"
        "LAB_WAIT:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra LAB_WAIT;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t *b, uint32_t parity)
{
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void red_add_relaxed(int *p, int v)
{
    asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *m, int c0, int c1, int c2, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(dst)),
        "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ unsigned long long gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void named_bar(int id, int n)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ int ld_acquire(const int *p)
{
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_relaxed(const int *p)
{
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ int atom_add_acq_rel(int *p, int v)
{
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void st_release(int *p, int v)
{
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---------------------------------------------------------------- plan tables
// LHS-only tables of the streaming solve (built once by pent_factor/tri_factor,
// dtype T unless noted):
//   coef  rows_alloc x 8     solve coefficients (band_core.cuh), identity rows
//                            beyond the system
//   tab   NRB*PC x TAB_STRIDE chunk scan tables, chunks grouped per tile
//   rsp   NRB x 4 x R        response of the local tile solution to the tile
//                            inflows: y_true = y_local + RF (Fin) + RB (Bin)
//   mft, mbt, hft  NRB x 4   tile transfer / response matrices (row-major 2x2)
//   gsp   4 x 2              response of g at spec row j to its tile's Fin
//   srb   4 (int)            tile index of spec row j (-1: unused)
//   scal  SCAL_LEN (fp64)    periodic finalisation scalars (band_core.cuh)
template <typename T>
struct StreamTabs {
    const T *coef, *tab, *mft, *mbt, *hft, *gsp, *rsp;
    const double *scal;
    int srb[4];
    int64_t srow[4];
};

// Per-call scratch (stream-ordered allocation by the launcher):
//   agg  [gt][NRB][W][4]  P1 tile aggregates (A_f0, A_f1, A_b0, A_b1)
//   inf  [gt][NRB][W][4]  group-scan result: tile inflows (Fin0, Fin1, Bin0, Bin1)
//   spec [gt][W][4]       forward values on the spec rows (zero tile inflow)
//   xl   [gt][W][2]       periodic pair
//   cnt, flag [gt]        P1 tiles completed (counted by each CTA's sync warp), scan-done flag
template <typename T>
struct StreamScratch {
    T *agg, *inf, *spec, *xl;
    int *cnt, *flag;
};

template <typename T>
struct StreamArgs {
    StreamTabs<T> tb;
    StreamScratch<T> sc;
    T *x;               // rhs / solution base
    int64_t n, M, bstride;
    int count;          // rhs batches (pent_solve_many)
    int nrb;            // tiles per system
    int K;              // CTAs per tile row block
    int64_t groups;     // system groups per batch = ceil(M / W)
    int lead;           // P1 tiles producer A may run ahead of producer B
    unsigned long long *trace;   // dev timeline: [cta][team][item][8] globaltimer stamps (nullptr = off)
};

// ---------------------------------------------------------------- geometry
// A tile is W = 32 systems (one per lane) x R rows: 32 KB, one TMA box.
// fp64: 256-byte rows, R = 128; fp32: 128-byte rows, R = 256.
template <typename T>
struct StreamGeom {
    static constexpr int W = 32;
    static constexpr int R = sizeof(T) == 8 ? 128 : 256;
};
constexpr int STREAM_SA = 3, STREAM_SB = 2;       // ring slots: P1 (A), P2 (B)
constexpr int STREAM_WA = 2, STREAM_WB = 2;       // consumer warps per ring
constexpr int STREAM_THREADS = 32 * (4 + STREAM_WA + STREAM_WB);   // producers A, B, sync, scan + consumers
constexpr int DONE_Q = 8;                         // P1-completion queue depth (sync warp)
constexpr int MAX_NRB = 64;                       // == STREAM_MAX_NRB (band_tile.cuh)

template <typename T>
struct StreamSmem {
    static constexpr int W = StreamGeom<T>::W, R = StreamGeom<T>::R;
    T slot[STREAM_SA + STREAM_SB][R * W];   // ring A (P1) then ring B (P2); 32 KB each
    T coef[R][COEF_STRIDE];                 // this CTA's rows (F0 F1 F2 - B1 B2 Z1 Z2)
    T rsp[R][4];                            // RF0 RF1 RB0 RB1 of this CTA's rows
    T tmat[MAX_NRB][12];                    // per tile: Mf_t, Mb_t, Hf_t (row-major 2x2)
    T side[STREAM_SB][W * 6];               // ring B: the tile's inflows [W][4] and x_l [W][2]
    T scanbuf[MAX_NRB][W / 2][4];           // group scan: one half of a group's aggregates
    uint64_t scanbar;                       // group scan: bulk-load barrier
    uint64_t full[STREAM_SA + STREAM_SB], empty[STREAM_SA + STREAM_SB];
    uint64_t done[DONE_Q];                  // P1 tile finished (one warp per tile)
    int p1_fenced;                          // P1 tiles whose stores are published (for producer B)
    int p2_issued;                          // P2 loads issued (P1 lead control)
};

// periodic pair (Navon eq:first_two, P:1596-1612 / Sherman–Morrison P:2384):
// y = (x_0, x_1) before correction, sp = forward values on the spec rows
template <typename T, int K>
__device__ __forceinline__ void local_xl(const double *sc, T y1, T y2, const T (&sp)[4], T &xl0, T &xl1)
{
    if (K == 2) {
        const T ym1 = sp[1], ym2 = sp[0] - T(sc[10]) * sp[1];
        const T q0 = sp[2] - (T(sc[4]) * y1 + T(sc[5]) * ym2 + T(sc[6]) * ym1);
        const T q1 = sp[3] - (T(sc[7]) * y1 + T(sc[8]) * y2 + T(sc[9]) * ym1);
        xl0 = T(sc[0]) * q0 + T(sc[1]) * q1;
        xl1 = T(sc[2]) * q0 + T(sc[3]) * q1;
    } else {
        xl0 = (y1 + T(sc[0]) * sp[0]) / T(sc[1]);
        xl1 = T(0);
    }
}

// ---------------------------------------------------------------- group scan
// Tile inflows of one group, lane = system: the forward chain over the tiles,
// then the backward chain, with loads batched (GB tiles per batch) so each
// batch costs one L2 round trip.
//   forward:  Fin_0 = 0,        Fin_{r+1} = A_f[r] + Mf_t[r] Fin_r
//   backward: Bin_{last} = 0,   Bin_{r-1} = A_b[r] + Hf_t[r] Fin_r + Mb_t[r] Bin_r
// then the periodic pair from Bout_0 = (y_1, y_2) and the spec rows.
template <typename T, int K, bool PER>
__device__ __forceinline__ void group_scan(const StreamArgs<T> &A, StreamSmem<T> &sm, int64_t g, int lane,
                                           uint32_t &sphase)
{
    constexpr int W = StreamGeom<T>::W, H = W / 2;
    const int nrb = A.nrb;
#pragma unroll 1
    for (int half = 0; half < 2; ++half) {
        // ---- one bulk copy per tile: the half-group's 16 systems x 4 values (512 B fp64)
        const uint32_t chunk = (uint32_t)(H * 4 * sizeof(T));
        if (lane == 0) mbar_expect_tx(&sm.scanbar, chunk * nrb);
        __syncwarp();
        for (int r = lane; r < nrb; r += 32)
            bulk_load(sm.scanbuf[r], A.sc.agg + ((g * nrb + r) * W + half * H) * 4, chunk, &sm.scanbar);
        mbar_wait(&sm.scanbar, sphase);
        sphase ^= 1;
        if (lane < H) {
            // forward: Fin in place of A_f; backward constants d_r = A_b[r] + Hf_t[r] Fin_r in place of A_b
            T F0 = T(0), F1 = T(0);
#pragma unroll 4
            for (int r = 0; r < nrb; ++r) {
                T *e = sm.scanbuf[r][lane];
                const T *m = sm.tmat[r];
                const T a0 = e[0], a1 = e[1];
                e[0] = F0;
                e[1] = F1;
                e[2] += m[8] * F0 + m[9] * F1;
                e[3] += m[10] * F0 + m[11] * F1;
                const T n0 = a0 + m[0] * F0 + m[1] * F1, n1 = a1 + m[2] * F0 + m[3] * F1;
                F0 = n0, F1 = n1;
            }
            // backward: Bin in place of d
            T B0 = T(0), B1 = T(0);
#pragma unroll 4
            for (int r = nrb - 1; r >= 0; --r) {
                T *e = sm.scanbuf[r][lane];
                const T *m = sm.tmat[r] + 4;
                const T d0 = e[2], d1 = e[3];
                e[2] = B0;
                e[3] = B1;
                const T n0 = d0 + m[0] * B0 + m[1] * B1, n1 = d1 + m[2] * B0 + m[3] * B1;
                B0 = n0, B1 = n1;
            }
            if (PER) {
                // periodic pair: true forward values on the spec rows, y = Bout_0
                const int sys = half * H + lane;
                T sp[4];
#pragma unroll
                for (int jx = 0; jx < 4; ++jx) {
                    const int r = A.tb.srb[jx];
                    sp[jx] = T(0);
                    if (r >= 0)
                        sp[jx] = __ldcg(A.sc.spec + (g * W + sys) * 4 + jx) + __ldg(A.tb.gsp + jx * 2) * sm.scanbuf[r][lane][0] +
                                 __ldg(A.tb.gsp + jx * 2 + 1) * sm.scanbuf[r][lane][1];
                }
                T xl0, xl1;
                local_xl<T, K>(A.tb.scal, B0, B1, sp, xl0, xl1);
                A.sc.xl[(g * W + sys) * 2 + 0] = xl0;
                A.sc.xl[(g * W + sys) * 2 + 1] = xl1;
            }
        }
        __syncwarp();
        // inflows out (coalesced: the warp writes one tile's 512 B at a time)
        for (int e = lane; e < nrb * H * 4; e += 32) {
            const int r = e / (H * 4), rest = e % (H * 4);
            A.sc.inf[((g * nrb + r) * W + half * H) * 4 + rest] = (&sm.scanbuf[r][0][0])[rest];
        }
        __syncwarp();
    }
}

#define PB_TR(slot)                                                                              \
    do {                                                                                         \
        if (A.trace && lane == 0 && j < 256)                                                     \
            A.trace[(((int64_t)blockIdx.x * 8 + cw) * 256 + j) * 8 + (slot)] = gtimer();         \
    } while (0)

// ---------------------------------------------------------------- the kernel
// Warps: 0 = ring-A producer, 1 = ring-B producer, 2 = sync warp, 3 = scan
// warp, then STREAM_WA consumer warps on ring A and STREAM_WB on ring B (one
// tile per warp at a time, lane = system).
//  two-phase (nrb > 1): ring A = P1 tiles, ring B = P2 tiles; the sync warp
//   publishes finished P1 tiles (gpu fence + per-group counter); the scan
//   warp runs the group scans of the groups this CTA is designated for
//   (i = rb, rb + nrb, ...); producer A runs at most `lead` tiles ahead of
//   producer B (L2 residency of y).
//  single tile (nrb == 1): every item is a complete solve (both rings).
template <typename T, int K, bool PER>
__global__ void __launch_bounds__(STREAM_THREADS, 1)
    stream_solve_kernel(const __grid_constant__ CUtensorMap tmap, const StreamArgs<T> A)
{
    using SM = StreamSmem<T>;
    constexpr int W = StreamGeom<T>::W, R = StreamGeom<T>::R, SA = STREAM_SA, SB = STREAM_SB;
    constexpr uint32_t TILE_BYTES = (uint32_t)(R * W * sizeof(T));
    extern __shared__ __align__(128) unsigned char smem_raw[];
    SM &sm = *reinterpret_cast<SM *>(smem_raw + ((128 - ((uintptr_t)smem_raw & 127)) & 127));

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nrb = A.nrb;
    const int rb = blockIdx.x % nrb, kk = blockIdx.x / nrb;
    const int64_t gt = A.groups * A.count;                 // groups over all batches
    const int ng = (int)((gt - kk + A.K - 1) / A.K);       // this CTA's groups: kk + A.K * i
    const bool two = nrb > 1;
    const int64_t row0 = (int64_t)rb * R;
    const int rows = (int)(A.n - row0 < R ? A.n - row0 : R);   // live rows of this tile row block

    // ---- setup: barriers, coefficient / response rows, tile matrices
    if (tid == 0) {
        for (int s = 0; s < SA + SB; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], 1);
        }
        for (int s = 0; s < DONE_Q; ++s) mbar_init(&sm.done[s], 1);
        mbar_init(&sm.scanbar, 1);
        sm.p1_fenced = 0;
        sm.p2_issued = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int e = tid; e < R * COEF_STRIDE; e += blockDim.x)
        sm.coef[e / COEF_STRIDE][e % COEF_STRIDE] = A.tb.coef[row0 * COEF_STRIDE + e];
    if (two) {
        for (int e = tid; e < R * 4; e += blockDim.x) {
            const int r = e / 4, c = e % 4;
            sm.rsp[r][c] = A.tb.rsp[((int64_t)rb * 4 + c) * R + r];
        }
        for (int e = tid; e < nrb * 12; e += blockDim.x) {
            const int r = e / 12, c = e % 12;
            sm.tmat[r][c] = c < 4 ? A.tb.mft[r * 4 + c] : c < 8 ? A.tb.mbt[r * 4 + c - 4] : A.tb.hft[r * 4 + c - 8];
        }
    }
    __syncthreads();
    auto gid = [&](int i) -> int64_t { return kk + (int64_t)A.K * i; };

    // ================= producers
    if (warp < 2) {
        if (lane != 0) return;
        const bool ringA = warp == 0;
        const int nslot = ringA ? SA : SB, base = ringA ? 0 : SA;
        int j = 0;
        for (int i = 0; i < ng; ++i) {
            // two-phase: every group on both rings; single tile: i % 4 == 3 on B, the rest on A
            if (!two && ((i % 4 != 3) != ringA)) continue;
            if (two) {
                volatile int *v2 = &sm.p2_issued, *vf = &sm.p1_fenced;
                if (ringA) {
                    // lead control; the sync warp's completion queue must not wrap
                    while (i >= *v2 + A.lead || i >= *vf + DONE_Q - 1) __nanosleep(64);
                } else {
                    while (i >= *vf) __nanosleep(64);   // P1 stores of this tile published
                    fence_proxy_async_global();
                }
            }
            const int s = base + j % nslot;
            if (j >= nslot) mbar_wait(&sm.empty[s], ((j / nslot) - 1) & 1);
            const int64_t g = gid(i);
            const int b = (int)(g / A.groups), gg = (int)(g % A.groups);
            if (two && !ringA) {
                // P2: the group scan's inflows travel with the tile (one barrier)
                const int *fl = A.sc.flag + g;
                if (A.trace && j < 256) A.trace[(((int64_t)blockIdx.x * 8 + 7) * 256 + j) * 8 + 0] = gtimer();
                while (ld_relaxed(fl) == 0) __nanosleep(32);
                if (A.trace && j < 256) A.trace[(((int64_t)blockIdx.x * 8 + 7) * 256 + j) * 8 + 1] = gtimer();
                fence_acq_rel_gpu();
                fence_proxy_async_global();
                const uint32_t side = (uint32_t)(W * 4 * sizeof(T)) + (PER ? (uint32_t)(W * 2 * sizeof(T)) : 0u);
                mbar_expect_tx(&sm.full[s], TILE_BYTES + side);
                T *sd = sm.side[s - SA];
                bulk_load(sd, A.sc.inf + (g * nrb + rb) * W * 4, W * 4 * sizeof(T), &sm.full[s]);
                if (PER) bulk_load(sd + W * 4, A.sc.xl + g * W * 2, W * 2 * sizeof(T), &sm.full[s]);
            } else {
                mbar_expect_tx(&sm.full[s], TILE_BYTES);
            }
            tma_load_3d(sm.slot[s], &tmap, gg * W, rb * R, b, &sm.full[s]);
            if (two && !ringA) {
                asm volatile("" ::: "memory");
                *(volatile int *)&sm.p2_issued = i + 1;
            }
            ++j;
        }
        return;
    }
    // ================= sync warp: publish finished P1 tiles (never blocks on scans)
    if (warp == 2) {
        if (!two || lane != 0) return;
        int jd = 0;   // next local P1 tile to publish
        while (jd < ng) {
            int nd = 0;
            while (jd + nd < ng && nd < DONE_Q && mbar_test(&sm.done[(jd + nd) % DONE_Q], ((jd + nd) / DONE_Q) & 1))
                ++nd;
            if (nd > 0) {
                fence_acq_rel_gpu();          // the P1 warps' stores (cumulative through the mbarrier)
                fence_proxy_async_global();
                for (int u = 0; u < nd; ++u) red_add_relaxed(A.sc.cnt + gid(jd + u), 1);
                if (A.trace)
                    for (int u = 0; u < nd; ++u)
                        if (jd + u < 256) A.trace[(((int64_t)blockIdx.x * 8 + 5) * 256 + jd + u) * 8 + 7] = gtimer();
                *(volatile int *)&sm.p1_fenced = jd + nd;
                jd += nd;
            } else {
                __nanosleep(64);
            }
        }
        return;
    }
    // ================= scan warp: group scans of the groups this CTA is designated for
    if (warp == 3) {
        if (!two) return;
        const int cw = 6;
        int j = 0;
        uint32_t sphase = 0;
        for (int is = rb; is < ng; is += nrb, ++j) {
            const int64_t g = gid(is);
            PB_TR(0);
            if (lane == 0) {
                while (ld_relaxed(A.sc.cnt + g) != nrb) __nanosleep(128);
                fence_acq_rel_gpu();
            }
            __syncwarp();
            PB_TR(1);
            group_scan<T, K, PER>(A, sm, g, lane, sphase);
            __syncwarp();
            if (lane == 0) {
                fence_acq_rel_gpu();
                st_release(A.sc.flag + g, 1);
            }
            PB_TR(7);
        }
        return;
    }

    // ================= consumer warps (lane = system of the tile's group)
    const int cw = warp - 4;
    const bool ringA = cw < STREAM_WA;
    const int widx = ringA ? cw : cw - STREAM_WA, nw = ringA ? STREAM_WA : STREAM_WB;
    const int nslot = ringA ? SA : SB, sbase = ringA ? 0 : SA;
    const bool corr = two && !ringA;   // P2: apply the tile inflows
    const int64_t M = A.M;
    const int sr2 = (int)(A.n - 2 - row0), sr1 = sr2 + 1;   // rows n-2, n-1 in tile coordinates

    int j = -1;
    for (int i = 0; i < ng; ++i) {
        if (!two && ((i % 4 != 3) != ringA)) continue;
        ++j;   // index of this item in its ring
        if (j % nw != widx) continue;
        const int sl = sbase + j % nslot;
        const int64_t g = gid(i);
        const int b = (int)(g / A.groups);
        const int64_t sys = (g % A.groups) * W + lane;
        const int lim = sys < M ? rows : 0;   // rows this lane stores
        T *col = sm.slot[sl] + lane;          // element r of this lane's system at col[r * W]
        T *dst = A.x + (int64_t)b * A.bstride + row0 * M + sys;

        if (corr) {
            // ======== P2: x = y + RF Fin + RB Bin (- Z x_l); the inflows arrive with the tile
            PB_TR(0);
            mbar_wait(&sm.full[sl], (j / nslot) & 1);
            PB_TR(1);
            const T *sd = sm.side[sl - SA];
            const T F0 = sd[lane * 4], F1 = sd[lane * 4 + 1], B0 = sd[lane * 4 + 2], B1 = sd[lane * 4 + 3];
            T X0 = T(0), X1 = T(0);
            if (PER) X0 = sd[W * 4 + lane * 2], X1 = sd[W * 4 + lane * 2 + 1];
#pragma unroll 1
            for (int r0 = 0; r0 < R; r0 += 8) {
                T o[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int r = r0 + k;
                    const T *rs = sm.rsp[r];
                    T v = col[r * W] + rs[0] * F0 + rs[1] * F1 + rs[2] * B0 + rs[3] * B1;
                    if (PER) {
                        v -= sm.coef[r][6] * X0;
                        if (K == 2) {
                            v -= sm.coef[r][7] * X1;
                            v = r == sr2 ? X0 : v;
                            v = r == sr1 ? X1 : v;
                        }
                    }
                    o[k] = v;
                }
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (r0 + k < lim) __stcs(dst + (int64_t)(r0 + k) * M, o[k]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.empty[sl]);
            PB_TR(7);
            continue;
        }

        // ======== P1 (two-phase: local solve, zero tile inflows) or a single-tile solve
        PB_TR(0);
        mbar_wait(&sm.full[sl], (j / nslot) & 1);
        PB_TR(1);
        // forward, g in place.  Blocks of 8 rows: loads and the
        // off-chain products first, then the recurrence (one DFMA per row on the
        // g_{i-1} chain).
        T y0 = T(0), y1 = T(0);
#pragma unroll 1
        for (int r0 = 0; r0 < R; r0 += 8) {
            T a[8], c1[8], c2[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const T *c = sm.coef[r0 + k];
                a[k] = c[0] * col[(r0 + k) * W];
                c1[k] = c[1];
                c2[k] = c[2];
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                T t = a[k];
                if (K == 2) t -= c2[k] * y0;
                const T gv = t - c1[k] * y1;
                col[(r0 + k) * W] = gv;
                y0 = y1;
                y1 = gv;
            }
        }
        // forward values on the spec rows (two-phase: zero tile inflow)
        T sp[4] = {T(0), T(0), T(0), T(0)};
        if (PER) {
#pragma unroll
            for (int jx = 0; jx < 4; ++jx) {
                const int64_t sr = A.tb.srow[jx] - row0;
                if (sr >= 0 && sr < R) {
                    sp[jx] = col[sr * W];
                    if (two && lim > 0) A.sc.spec[(g * W + lane) * 4 + jx] = sp[jx];
                }
            }
        }
        T *ag = A.sc.agg + ((g * nrb + rb) * W + lane) * 4;
        if (two) {
            ag[0] = y0;   // A_f
            ag[1] = y1;
        }
        // back substitution: two-phase streams y (kept in L2 for P2);
        // single tile: x in place (cyclic: corrected below) or streamed out
        T z0 = T(0), z1 = T(0);
#pragma unroll 1
        for (int r0 = R - 8; r0 >= 0; r0 -= 8) {
            T gk[8], b1[8], b2[8];
#pragma unroll
            for (int k = 7; k >= 0; --k) {
                const T *c = sm.coef[r0 + k];
                gk[k] = col[(r0 + k) * W];
                b1[k] = c[4];
                b2[k] = c[5];
            }
            T o[8];
#pragma unroll
            for (int k = 7; k >= 0; --k) {
                T t = gk[k];
                if (K == 2) t -= b2[k] * z1;
                const T xx = t - b1[k] * z0;
                z1 = z0;
                z0 = xx;
                o[k] = xx;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int r = r0 + k;
                if (two) {
                    if (r < lim) dst[(int64_t)r * M] = o[k];   // default policy: re-read from L2 by P2
                } else if (PER) {
                    col[r * W] = o[k];
                } else if (r < lim) {
                    __stcs(dst + (int64_t)r * M, o[k]);
                }
            }
        }
        if (two) {
            ag[2] = z0;   // A_b
            ag[3] = z1;
            fence_proxy_async_global();   // y is re-read by P2's TMA (async proxy)
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&sm.empty[sl]);
                mbar_arrive(&sm.done[i % DONE_Q]);
            }
        } else {
            if (PER) {
                // single tile: periodic pair from (x_0, x_1) and the spec rows, then x - Z x_l
                T xl0, xl1;
                local_xl<T, K>(A.tb.scal, z0, z1, sp, xl0, xl1);
#pragma unroll 1
                for (int r0 = 0; r0 < R; r0 += 8) {
                    T o[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const int r = r0 + k;
                        T v = col[r * W] - sm.coef[r][6] * xl0;
                        if (K == 2) {
                            v -= sm.coef[r][7] * xl1;
                            v = r == sr2 ? xl0 : v;
                            v = r == sr1 ? xl1 : v;
                        }
                        o[k] = v;
                    }
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        if (r0 + k < lim) __stcs(dst + (int64_t)(r0 + k) * M, o[k]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.empty[sl]);
        }
        PB_TR(7);
    }
}

}  // namespace pb

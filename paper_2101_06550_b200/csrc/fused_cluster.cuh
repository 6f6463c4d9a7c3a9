// fused_cluster.cuh — the shared-LHS batched solve as ONE persistent kernel of
// thread-block clusters: the production path of pent_solve / tri_solve /
// pent_solve_many / pent_solve_strided, the ADI sweeps and the 1D CH step.
//
// Same tiles as fused_solve.cuh (a 64-row chunk of 32 systems per consumer
// warp, lane = system, TMA ring, P1 = zero-inflow forward sweep + carries,
// P2 = sweeps from the true inflows), but a CLUSTER of CS CTAs
// owns whole groups of 32 systems: CTA c of the cluster handles chunks
// [c*cpc, (c+1)*cpc) of the cluster's current group, so
//   * P1 writes its chunk record (yF, zB) into its own shared memory -- the
//     records never touch L2 or HBM;
//   * the carry scan of a group (the affine chunk maps Mf, Mb, H) runs on one
//     warp per CTA over its cpc chunks with the CTA aggregates exchanged
//     through distributed shared memory (DSMEM stores + remote mbarrier
//     arrives) -- exact, no truncation, no global atomics or flags;
//   * cyclic systems get Navon's / Sherman–Morrison's x_l (P:1596-1612,
//     P:2384) from one more DSMEM exchange (x_0, x_1 from CTA 0; g on the
//     cyclic rows from the CTA that owns them);
//   * P2 of group t-1 follows P1 of group t, so its re-read of f hits the L2
//     that P1 filled one group ago: the L2 working set is ~2 groups per
//     cluster, HBM traffic = read f once + write x once.
// Clusters are independent (each loops over groups k, k + NCL, ...), so no
// co-residency beyond the cluster's own (guaranteed by the cluster launch) is
// needed.
#pragma once
#include <cooperative_groups.h>

#include "fused_solve.cuh"

namespace pb {
namespace fc {

using namespace fs;
namespace cg = cooperative_groups;

constexpr int CSMAX = 16;        // cluster size (16 = non-portable)
constexpr int NWC = 4;           // consumer warps (= items per block)
constexpr int NTHREADS = 32 * (NWC + 2);   // + producer warp + scan warp

template <typename T>
struct CCfg {
    static constexpr int TILE = Q * TW;
    static constexpr int COEF = Q * COEF_STRIDE;    // >= Q * REC
    static constexpr int HALO = TW * 2;             // MODE_CH1D: rows r0 - 1 and r0 + kmax (periodic)
    static constexpr int E1K = 1024 / (int)sizeof(T);
    static constexpr int SLOT = (TILE + COEF + HALO + E1K - 1) / E1K * E1K;   // 1 KB multiple (swizzle)
    static constexpr int NS = sizeof(T) == 8 ? 8 : 16;
    static constexpr int CPC = sizeof(T) == 8 ? 16 : 32;    // max chunks per CTA per group
    static_assert(NS % NWC == 0, "ring slots must be a multiple of the consumer warps");
};

template <typename T>
struct CArgs {
    const T *rec, *coef, *ct, *rsp;
    const double *scal;
    T *x, *xout;
    T alpha;                 // MODE_CH1D
    int64_t n, M, bstride, pitch;
    int64_t srow[4];
    int nq, count, Gb, G;
    int cs, cpc, ncl;        // cluster size, chunks per CTA, clusters
    int flat;
};

template <typename T>
struct CSmem {
    T slot[CCfg<T>::NS][CCfg<T>::SLOT];
    T rec[2][CCfg<T>::CPC][TW][4];   // per group parity: (yF0, yF1, zB0, zB1) -> (yin0, yin1, zin0, zin1)
    T spec[2][4][TW];                // zero-inflow g on the cyclic rows this CTA owns
    T xl[2][TW][2];
    T aggF[CSMAX][TW][2], aggB[CSMAX][TW][2];   // cluster exchange (written by every CTA)
    T PF[CSMAX][4], PB[CSMAX][4];
    T xlx[TW][2], xlg[4][TW];
    uint64_t full[CCfg<T>::NS], empty[CCfg<T>::NS];
    uint64_t p1done[2], recfree[2], scandone[2];
    uint64_t xfwd, xbwd, xxl;
    int64_t item[CCfg<T>::NS];       // (p2 << 62) | (t << 20) | local chunk ; -1 exit ; -2 empty
};

// ---------------------------------------------------------------- cluster PTX
__device__ __forceinline__ uint32_t mapa(const void *p, uint32_t rank)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(su32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void arrive_remote(const uint64_t *b, uint32_t rank)
{
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa(b, rank)) : "memory");
}
__device__ __forceinline__ void wait_cluster(uint64_t *b, uint32_t parity)
{
    asm volatile(
        "{\n .reg .pred p;\n"
        "FC_WAITC:\n"
        " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra FC_WAITC;\n}" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void fence_cluster() { asm volatile("fence.acq_rel.cluster;" ::: "memory"); }
template <typename T>
__device__ __forceinline__ T *peer(T *p, int rank)
{
    return cg::this_cluster().map_shared_rank(p, rank);
}

// ---------------------------------------------------------------- the scan of one group (one warp per CTA)
template <typename T, int K, bool PER>
__device__ void cluster_scan(const CArgs<T> &A, CSmem<T> &S, int t, int c, int q0, int ncl, int lane)
{
    const int par = t & 1;
    T(*R)[TW][4] = S.rec[par];
    // ---- forward fold of my chunks: a = Mf a + yF, P = Mf P
    T P[4] = {T(1), T(0), T(0), T(1)}, a0 = T(0), a1 = T(0);
    T mn[4];
    if (ncl > 0) ldm4(A.ct + (int64_t)q0 * 12, mn);
    for (int i = 0; i < ncl; ++i) {
        T m[4] = {mn[0], mn[1], mn[2], mn[3]}, t0, t1;
        if (i + 1 < ncl) ldm4(A.ct + (int64_t)(q0 + i + 1) * 12, mn);   // next chunk's map in flight
        mv(m, a0, a1, t0, t1);
        a0 = t0 + R[i][lane][0];
        a1 = t1 + R[i][lane][1];
        mmul(m, P, P);
    }
    for (int r = 0; r < A.cs; ++r) {
        T *pa = peer(&S.aggF[c][lane][0], r);
        pa[0] = a0;
        pa[1] = a1;
        if (lane < 4) peer(&S.PF[c][0], r)[lane] = P[lane];
    }
    fence_cluster();
    __syncwarp();
    if (lane == 0)
        for (int r = 0; r < A.cs; ++r) arrive_remote(&S.xfwd, r);
    wait_cluster(&S.xfwd, (uint32_t)(t & 1));
    T y0 = T(0), y1 = T(0);
    for (int v = 0; v < c; ++v) {
        T t0, t1;
        mv(S.PF[v], y0, y1, t0, t1);
        y0 = t0 + S.aggF[v][lane][0];
        y1 = t1 + S.aggF[v][lane][1];
    }
    // ---- forward walk: yin_q, c_q = zB_q + H_q yin_q, true g on the cyclic rows
    T hn[4];
    if (ncl > 0) {
        ldm4(A.ct + (int64_t)q0 * 12, mn);
        ldm4(A.ct + (int64_t)q0 * 12 + 8, hn);
    }
    for (int i = 0; i < ncl; ++i) {
        const int q = q0 + i;
        T m[4] = {mn[0], mn[1], mn[2], mn[3]}, h[4] = {hn[0], hn[1], hn[2], hn[3]}, t0, t1;
        if (i + 1 < ncl) {
            ldm4(A.ct + (int64_t)(q + 1) * 12, mn);
            ldm4(A.ct + (int64_t)(q + 1) * 12 + 8, hn);
        }
        const T yf0 = R[i][lane][0], yf1 = R[i][lane][1];
        mv(h, y0, y1, t0, t1);
        R[i][lane][0] = y0;
        R[i][lane][1] = y1;
        R[i][lane][2] += t0;
        R[i][lane][3] += t1;
        if (PER) {
#pragma unroll
            for (int jx = 0; jx < 4; ++jx)
                if (A.srow[jx] >= 0 && A.srow[jx] / Q == q)
                    S.spec[par][jx][lane] += A.rsp[jx * 2] * y0 + A.rsp[jx * 2 + 1] * y1;
        }
        mv(m, y0, y1, t0, t1);
        y0 = t0 + yf0;
        y1 = t1 + yf1;
    }
    // ---- backward fold (high to low): cb = Mb cb + c_q, Pb = Mb Pb
    T Pb[4] = {T(1), T(0), T(0), T(1)}, c0 = T(0), c1 = T(0);
    if (ncl > 0) ldm4(A.ct + (int64_t)(q0 + ncl - 1) * 12 + 4, mn);
    for (int i = ncl - 1; i >= 0; --i) {
        T m[4] = {mn[0], mn[1], mn[2], mn[3]}, t0, t1;
        if (i > 0) ldm4(A.ct + (int64_t)(q0 + i - 1) * 12 + 4, mn);
        mv(m, c0, c1, t0, t1);
        c0 = t0 + R[i][lane][2];
        c1 = t1 + R[i][lane][3];
        mmul(m, Pb, Pb);
    }
    for (int r = 0; r < A.cs; ++r) {
        T *pa = peer(&S.aggB[c][lane][0], r);
        pa[0] = c0;
        pa[1] = c1;
        if (lane < 4) peer(&S.PB[c][0], r)[lane] = Pb[lane];
    }
    fence_cluster();
    __syncwarp();
    if (lane == 0)
        for (int r = 0; r < A.cs; ++r) arrive_remote(&S.xbwd, r);
    wait_cluster(&S.xbwd, (uint32_t)(t & 1));
    T z0 = T(0), z1 = T(0);
    for (int v = A.cs - 1; v > c; --v) {
        T t0, t1;
        mv(S.PB[v], z0, z1, t0, t1);
        z0 = t0 + S.aggB[v][lane][0];
        z1 = t1 + S.aggB[v][lane][1];
    }
    if (ncl > 0) ldm4(A.ct + (int64_t)(q0 + ncl - 1) * 12 + 4, mn);
    for (int i = ncl - 1; i >= 0; --i) {
        T m[4] = {mn[0], mn[1], mn[2], mn[3]}, t0, t1;
        if (i > 0) ldm4(A.ct + (int64_t)(q0 + i - 1) * 12 + 4, mn);
        const T cq0 = R[i][lane][2], cq1 = R[i][lane][3];
        R[i][lane][2] = z0;
        R[i][lane][3] = z1;
        mv(m, z0, z1, t0, t1);
        z0 = t0 + cq0;
        z1 = t1 + cq1;
    }
    if (!PER) return;
    // ---- cyclic pair: (x_0, x_1) from CTA 0, true g on the cyclic rows from their owners
    if (c == 0)
        for (int r = 0; r < A.cs; ++r) {
            T *px = peer(&S.xlx[lane][0], r);
            px[0] = z0;
            px[1] = z1;
        }
#pragma unroll
    for (int jx = 0; jx < 4; ++jx) {
        const int64_t qj = A.srow[jx] / Q;
        if (A.srow[jx] >= 0 && qj >= q0 && qj < q0 + ncl)
            for (int r = 0; r < A.cs; ++r) peer(&S.xlg[jx][0], r)[lane] = S.spec[par][jx][lane];
    }
    fence_cluster();
    __syncwarp();
    if (lane == 0)
        for (int r = 0; r < A.cs; ++r) arrive_remote(&S.xxl, r);
    wait_cluster(&S.xxl, (uint32_t)(t & 1));
    const T y1c = S.xlx[lane][0], y2c = S.xlx[lane][1];
    T gv[4];
#pragma unroll
    for (int jx = 0; jx < 4; ++jx) gv[jx] = A.srow[jx] >= 0 ? S.xlg[jx][lane] : T(0);
    const double *sc = A.scal;
    T xl0, xl1;
    if (K == 2) {
        // Navon (eq:first_two)
        const T ym1 = gv[1], ym2 = gv[0] - T(sc[10]) * gv[1];
        const T qa = gv[2] - (T(sc[4]) * y1c + T(sc[5]) * ym2 + T(sc[6]) * ym1);
        const T qb = gv[3] - (T(sc[7]) * y1c + T(sc[8]) * y2c + T(sc[9]) * ym1);
        xl0 = T(sc[0]) * qa + T(sc[1]) * qb;
        xl1 = T(sc[2]) * qa + T(sc[3]) * qb;
    } else {
        // Sherman–Morrison
        xl0 = (y1c + T(sc[0]) * gv[0]) / T(sc[1]);
        xl1 = T(0);
    }
    S.xl[par][lane][0] = xl0;
    S.xl[par][lane][1] = xl1;
}

// ---------------------------------------------------------------- item order of one CTA
// Iteration t (the cluster's t-th group): the P1 tiles of group t, then the P2
// tiles of group t-1, in blocks of NWC chunks (one per consumer warp).  The
// scan of group t-1 (cluster-wide: every CTA's P1 tiles of t-1 + three DSMEM
// exchanges) then has the whole P1 phase of iteration t to complete.
struct Seq {
    int nb;   // blocks of NWC per type
    __device__ int len(int t, int T) const
    {
        const int p1 = t < T ? nb : 0, p2 = t >= 1 ? nb : 0;
        return (p1 + p2) * NWC;
    }
    __device__ void block(int t, int T, int pos, int &type, int &bi) const
    {
        if (t >= T) { type = 1; bi = pos; return; }
        type = pos >= nb;
        bi = type ? pos - nb : pos;
    }
};

// ---------------------------------------------------------------- the kernel
template <typename T, int K, bool PER, int MODE, int LAY>
__global__ void __launch_bounds__(NTHREADS, 1) fc_kernel(const __grid_constant__ CUtensorMap tmap, const CArgs<T> A)
{
    using C = CCfg<T>;
    constexpr int NS = C::NS, TILE = C::TILE;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    CSmem<T> &sm = *reinterpret_cast<CSmem<T> *>((((uintptr_t)smem_raw) + 1023) & ~(uintptr_t)1023);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = (int)cg::this_cluster().block_rank();
    const int cl = blockIdx.x / A.cs;                       // cluster index
    const int q0 = c * A.cpc, ncl = max(0, min(A.cpc, A.nq - q0));
    const int T_ = cl < A.G ? (A.G - 1 - cl) / A.ncl + 1 : 0;   // groups of this cluster
    const Seq seq{(ncl + NWC - 1) / NWC};
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) {
            bar_init(&sm.full[i], 1);
            bar_init(&sm.empty[i], 1);
        }
        for (int p = 0; p < 2; ++p) {
            bar_init(&sm.p1done[p], max(ncl, 1));
            bar_init(&sm.recfree[p], max(ncl, 1));
            bar_init(&sm.scandone[p], 1);
        }
        bar_init(&sm.xfwd, A.cs);
        bar_init(&sm.xbwd, A.cs);
        bar_init(&sm.xxl, A.cs);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cg::this_cluster().sync();   // barriers initialised cluster-wide before any remote arrive

    if (warp == NWC) {
        // ---------------- producer
        if (lane == 0) {
            const uint64_t pol1 = policy_evict_last(), pol2 = policy_evict_first();
            int64_t j = 0;   // local slot sequence
            for (int t = 0; t <= T_; ++t) {
                const int len = seq.len(t, T_);
                for (int k = 0; k < len; ++k, ++j) {
                    const int sl = (int)(j % NS);
                    if (j >= NS) bar_wait(&sm.empty[sl], (uint32_t)(((j / NS) - 1) & 1));
                    int type, bi;
                    seq.block(t, T_, k / NWC, type, bi);
                    const int i = bi * NWC + k % NWC;        // local chunk
                    const int tg = type ? t - 1 : t;         // iteration of the item's group
                    if (i >= ncl) {
                        sm.item[sl] = -2;
                        bar_arrive(&sm.full[sl]);
                        continue;
                    }
                    sm.item[sl] = ((int64_t)type << 62) | ((int64_t)tg << 20) | i;
                    const int g = cl + tg * A.ncl;
                    const int b = g / A.Gb, gl = g - b * A.Gb;
                    const int64_t r0 = (int64_t)(q0 + i) * Q;
                    const int kmax = (int)min((int64_t)Q, A.n - r0);
                    T *slot = sm.slot[sl];
                    const uint32_t cb = up16((uint32_t)(kmax * (type ? COEF_STRIDE : REC) * sizeof(T)));
                    uint32_t bytes = TILE * sizeof(T) + cb + (MODE == MODE_CH1D ? C::HALO * sizeof(T) : 0);
                    bar_expect_tx(&sm.full[sl], bytes);
                    const uint64_t pol = type ? pol2 : pol1;
                    if (LAY == LAY_CONTIG) {
#pragma unroll
                        for (int bx = 0; bx < Q / Sw<T>::EB; ++bx) {
                            T *dst = slot + bx * TW * Sw<T>::EB;
                            const int r = (int)r0 + bx * Sw<T>::EB;
                            if (A.flat) tma_load2(dst, &tmap, r, (int)((int64_t)b * A.M + gl * TW), &sm.full[sl], pol);
                            else tma_load3(dst, &tmap, r, gl * TW, b, &sm.full[sl], pol);
                        }
                    } else if (A.flat) {
                        tma_load2(slot, &tmap, gl * TW, (int)((int64_t)b * A.n + r0), &sm.full[sl], pol);
                    } else {
                        tma_load3(slot, &tmap, gl * TW, (int)r0, b, &sm.full[sl], pol);
                    }
                    bulk_load(slot + TILE, type ? A.coef + r0 * COEF_STRIDE : A.rec + r0 * REC, cb, &sm.full[sl]);
                    if (MODE == MODE_CH1D) {
                        const T *ub = A.x + (int64_t)b * A.bstride + (int64_t)gl * TW;
                        const int64_t rlo = r0 == 0 ? A.n - 1 : r0 - 1, rhi = r0 + kmax == A.n ? 0 : r0 + kmax;
                        T *hs = slot + TILE + C::COEF;
                        bulk_load(hs, ub + rlo * A.pitch, TW * sizeof(T), &sm.full[sl]);
                        bulk_load(hs + TW, ub + rhi * A.pitch, TW * sizeof(T), &sm.full[sl]);
                    }
                }
            }
            for (int w = 0; w < NWC; ++w, ++j) {   // exit markers
                const int sl = (int)(j % NS);
                if (j >= NS) bar_wait(&sm.empty[sl], (uint32_t)(((j / NS) - 1) & 1));
                sm.item[sl] = -1;
                bar_arrive(&sm.full[sl]);
            }
        }
    } else if (warp < NWC) {
        // ---------------- consumers: slots j = warp, warp + NWC, ... (each slot owned by one warp)
        for (int64_t j = warp;; j += NWC) {
            const int sl = (int)(j % NS);
            bar_wait(&sm.full[sl], (uint32_t)((j / NS) & 1));
            const int64_t it = *(volatile int64_t *)&sm.item[sl];
            if (it == -1) {
                if (LAY == LAY_CONTIG && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
                break;
            }
            if (it < 0) {
                __syncwarp();
                if (lane == 0) bar_arrive(&sm.empty[sl]);
                continue;
            }
            const int type = (int)(it >> 62), tg = (int)((it >> 20) & ((1ll << 42) - 1)), i = (int)(it & 0xfffff);
            const int par = tg & 1;
            const int g = cl + tg * A.ncl;
            const int b = g / A.Gb, gl = g - b * A.Gb;
            const int q = q0 + i;
            const int64_t r0 = (int64_t)q * Q;
            const int kmax = (int)min((int64_t)Q, A.n - r0);
            const T *d = sm.slot[sl];
            const T *cf = d + TILE;
            const int64_t s_in_batch = (int64_t)gl * TW + lane;
            const bool ok = s_in_batch < A.M;
            if (MODE == MODE_CH1D) ch1d_rhs<T>(const_cast<T *>(d), d + TILE + C::COEF, kmax, lane, A.alpha);
            if (!type) {
                // ---- P1: zero-inflow forward sweep, carry, back-substitution functional
                T y0 = T(0), y1 = T(0), a0 = T(0), a1 = T(0), gs[4] = {T(0), T(0), T(0), T(0)};
                if (kmax == Q && !(PER && q >= A.srow[0] / Q)) {
#pragma unroll
                    for (int k = 0; k < Q; ++k) {
                        T f0, f1, f2, wa;
                        lds2(cf + k * REC, f0, f1);
                        lds2(cf + k * REC + 2, f2, wa);
                        const T wb = cf[k * REC + 4];
                        T gg = f0 * tld<T, LAY>(d, k, lane) - f1 * y1;
                        if (K == 2) gg -= f2 * y0;
                        y0 = y1;
                        y1 = gg;
                        a0 += wa * gg;
                        a1 += wb * gg;
                    }
                } else {
#pragma unroll 4
                    for (int k = 0; k < kmax; ++k) {
                        T f0, f1, f2, wa;
                        lds2(cf + k * REC, f0, f1);
                        lds2(cf + k * REC + 2, f2, wa);
                        const T wb = cf[k * REC + 4];
                        T gg = f0 * tld<T, LAY>(d, k, lane) - f1 * y1;
                        if (K == 2) gg -= f2 * y0;
                        y0 = y1;
                        y1 = gg;
                        a0 += wa * gg;
                        a1 += wb * gg;
                        if (PER) {
#pragma unroll
                            for (int jx = 0; jx < 4; ++jx)
                                if (A.srow[jx] == r0 + k) gs[jx] = gg;
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) bar_arrive(&sm.empty[sl]);
                // the record buffer of this parity is free once P2 of group tg-2 has read it
                if (tg >= 2) bar_wait(&sm.recfree[par], (uint32_t)(((tg - 2) >> 1) & 1));
                sm.rec[par][i][lane][0] = y0;
                sm.rec[par][i][lane][1] = y1;
                sm.rec[par][i][lane][2] = a0;
                sm.rec[par][i][lane][3] = a1;
                if (PER) {
#pragma unroll
                    for (int jx = 0; jx < 4; ++jx)
                        if (A.srow[jx] >= 0 && A.srow[jx] / Q == q) sm.spec[par][jx][lane] = gs[jx];
                }
                __syncwarp();
                if (lane == 0) bar_arrive(&sm.p1done[par]);
                continue;
            }
            // ---- P2: inflows and x_l of the group (scan done), sweeps, x out
            T v[Q];
#pragma unroll
            for (int k = 0; k < Q; ++k) v[k] = tld<T, LAY>(d, k, lane);
            bar_wait(&sm.scandone[par], (uint32_t)((tg >> 1) & 1));
            const T yi0 = sm.rec[par][i][lane][0], yi1 = sm.rec[par][i][lane][1];
            const T zi0 = sm.rec[par][i][lane][2], zi1 = sm.rec[par][i][lane][3];
            T xl0 = T(0), xl1 = T(0);
            if (PER) xl0 = sm.xl[par][lane][0], xl1 = sm.xl[par][lane][1];
            __syncwarp();
            if (lane == 0) bar_arrive(&sm.recfree[par]);
            if (kmax == Q) tile_solve<T, K, PER, true>(v, cf, Q, yi0, yi1, zi0, zi1, xl0, xl1);
            else tile_solve<T, K, PER, false>(v, cf, kmax, yi0, yi1, zi0, zi1, xl0, xl1);
            if (PER && K == 2 && r0 + Q > A.n - 2) {
                const int k2 = (int)(A.n - 2 - r0);
#pragma unroll
                for (int k = 0; k < Q; ++k) {
                    if (k == k2) v[k] = xl0;
                    if (k == k2 + 1) v[k] = xl1;
                }
            }
            if (LAY == LAY_CONTIG) {
                T *dm = const_cast<T *>(d);
#pragma unroll
                for (int k = 0; k < Q; ++k) tst<T, LAY>(dm, k, lane, v[k]);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
#pragma unroll
                    for (int bx = 0; bx < Q / Sw<T>::EB; ++bx) {
                        const int r = (int)r0 + bx * Sw<T>::EB;
                        if (r < A.n) {
                            if (A.flat) tma_store2(&tmap, r, (int)((int64_t)b * A.M + gl * TW), dm + bx * TW * Sw<T>::EB);
                            else tma_store3(&tmap, r, gl * TW, b, dm + bx * TW * Sw<T>::EB);
                        }
                    }
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    bar_arrive(&sm.empty[sl]);
                }
                __syncwarp();
                continue;
            }
            __syncwarp();
            if (lane == 0) bar_arrive(&sm.empty[sl]);
            if (ok) {
                int64_t Mo = A.pitch;
                asm volatile("" : "+l"(Mo));
                T *x = A.xout + (int64_t)b * A.bstride + r0 * Mo + s_in_batch;
#pragma unroll
                for (int k = 0; k < Q; ++k) {
                    if (kmax == Q || k < kmax) __stcs(x, v[k]);
                    x += Mo;
                }
            }
        }
    } else {
        // ---------------- scan warp: the cluster's groups in order
        for (int t = 0; t < T_; ++t) {
            const int par = t & 1;
            if (ncl > 0) bar_wait(&sm.p1done[par], (uint32_t)((t >> 1) & 1));
            cluster_scan<T, K, PER>(A, sm, t, c, q0, ncl, lane);
            __syncwarp();
            if (lane == 0) bar_arrive(&sm.scandone[par]);
        }
    }
    // no CTA may leave while a peer can still write into its shared memory
    cg::this_cluster().sync();
}

}  // namespace fc
}  // namespace pb

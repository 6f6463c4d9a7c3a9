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

constexpr int CSMAX = 8;         // cluster size (portable)
constexpr int NWC = 4;           // consumer warps (= items per block)
constexpr int NTHREADS = 32 * (NWC + 2);   // + producer warp + scan warp

template <typename T, int MODE>
struct CCfg {
    static constexpr int TILE = Q * TW;
    static constexpr int COEF = Q * COEF_STRIDE;    // >= Q * REC
    static constexpr int HALO = MODE == MODE_CH1D ? TW * 2 : 0;   // rows r0 - 1 and r0 + kmax (periodic)
    static constexpr int E1K = 1024 / (int)sizeof(T);
    static constexpr int SLOT = (TILE + COEF + HALO + E1K - 1) / E1K * E1K;   // 1 KB multiple (swizzle)
    static constexpr int NS = sizeof(T) == 8 ? 8 : 16;
    // max chunks per CTA per group (records in shared memory; fp64: 15 keeps the
    // plan inside the 227 KB opt-in limit with its 1 KB alignment slack)
    static constexpr int CPC = MODE == MODE_CH1D ? 8 : (sizeof(T) == 8 ? 15 : 32);
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
    int dbg;   // DEV ONLY (timing experiments): 1 skip scan, 4 skip sweeps
    long long *prof;   // DEV ONLY (FH_PROF builds)
};

template <typename T, int MODE>
struct CSmem {
    using C = CCfg<T, MODE>;
    static constexpr int NPAR = 2;   // record parities
    T slot[C::NS][C::SLOT];
    T rec[2][C::CPC][TW][4];         // per group parity: (yF0, yF1, zB0, zB1) -> (yin0, yin1, zin0, zin1)
    T spec[2][4][TW];                // zero-inflow g on the cyclic rows this CTA owns
    T xl[2][TW][2];
    // one cluster exchange per group: CTA c's summary -- zero-inflow forward
    // outflow a and backward outflow b (per lane), forward / backward transfer
    // maps P, Pb and the coupling K of b to the forward inflow (uniform) -- and,
    // from the owners of the cyclic rows, their zero-inflow g and its coupling r
    // to the owner's forward inflow.  Rewritten for the next group only after
    // every CTA has consumed it (xcons).
    T xa[CSMAX][TW][2], xb[CSMAX][TW][2];
    T yv[CSMAX][TW][2];              // scan temporaries: every CTA's forward inflow
    T xP[CSMAX][12];
    T xg[4][TW], xr[4][2];
    T phi[C::CPC][8];                // scan temporaries: Phi_i (chunk inflow per unit CTA inflow), H_i Phi_i
    T cpriv[NWC][C::COEF];           // per consumer warp: its tile's coefficient rows (the slot is released early)
    uint64_t full[C::NS], empty[C::NS];
    uint64_t p1done[2], recfree[2], scandone[2];
    uint64_t xch, xcons;
    int64_t item[C::NS];             // (p2 << 62) | (t << 20) | local chunk ; -1 exit ; -2 empty
    int64_t seq[C::NS];              // sequence number of the item in the slot (written before its fill)
    int claim;                       // consumer ticket: the next item to take
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
// Chunk q's true inflows are affine in the CTA's forward inflow Y and backward
// inflow Z (P:1712-1724 in chunked form): the CTA folds its chunks with Y = Z =
// 0 while tracking the (lane-independent) 2x2 responses, publishes one summary
// to every CTA of the cluster, and after that single exchange every CTA
// resolves Y_c, Z_c of all CTAs, (x_0, x_1), the true g on the cyclic rows and
// x_l locally, then walks its own chunks.  A one-CTA cluster owns the whole
// system: Y = Z = 0 and no exchange.
//   ctl  this CTA's chunk maps (ct rows q0 .. q0+ncl-1, 12 values each)
//   rsp  the cyclic rows' g per unit forward inflow (8 values)
#ifdef FH_PROF
#define FHP(i) do { if (pt) { long long _n = clock64(); pt[i] += _n - _t; _t = _n; } } while (0)
#else
#define FHP(i) do {} while (0)
#endif
template <typename T>
__device__ __forceinline__ void ld4(const T *p, T *m)
{
    m[0] = p[0], m[1] = p[1], m[2] = p[2], m[3] = p[3];
}
__device__ __forceinline__ void st_peer2(uint32_t a, double x, double y)
{
    asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(x), "d"(y) : "memory");
}
__device__ __forceinline__ void st_peer2(uint32_t a, float x, float y)
{
    asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(x), "f"(y) : "memory");
}
__device__ __forceinline__ void st_peer(uint32_t a, double x)
{
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(x) : "memory");
}
__device__ __forceinline__ void st_peer(uint32_t a, float x)
{
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(a), "f"(x) : "memory");
}
template <typename T, int K, bool PER, int CSM, typename SM>
__device__ void cluster_scan(const CArgs<T> &A, SM &S, const T *ctl, const T *rsp, int t, int c, int q0, int ncl,
                             int lane, long long *pt = nullptr)
{
#ifdef FH_PROF
    long long _t = clock64();
#endif
    const int par = SM::NPAR == 2 ? (t & 1) : 0;
    T(*R)[TW][4] = S.rec[par];
    // ---- forward fold, zero inflow: yin0_i, Phi_i; c0_i = zB_i + H_i yin0_i; Hc_i = H_i Phi_i
    // (Phi, Hc, Pb, K: the responses to this CTA's inflows -- only a multi-CTA
    // cluster needs them)
    const bool multi = A.cs > 1;
    int li[4];   // local chunk of each cyclic row (-1: not mine)
#pragma unroll
    for (int jx = 0; jx < 4; ++jx) {
        const int64_t qq = A.srow[jx] >= 0 ? A.srow[jx] / Q - q0 : -1;
        li[jx] = PER && qq >= 0 && qq < ncl ? (int)qq : -1;
    }
    T Phi[4] = {T(1), T(0), T(0), T(1)}, y0 = T(0), y1 = T(0);
    T gj[4] = {T(0), T(0), T(0), T(0)}, rj[4][2] = {{T(0), T(0)}, {T(0), T(0)}, {T(0), T(0)}, {T(0), T(0)}};
    for (int i = 0; i < ncl; ++i) {
        T m[4], h[4], t0, t1;
        ld4(ctl + i * 12, m);
        ld4(ctl + i * 12 + 8, h);
        const T yf0 = R[i][lane][0], yf1 = R[i][lane][1];
        mv(h, y0, y1, t0, t1);
        R[i][lane][0] = y0;            // yin0_i
        R[i][lane][1] = y1;
        R[i][lane][2] += t0;           // c0_i
        R[i][lane][3] += t1;
        if (PER) {
#pragma unroll
            for (int jx = 0; jx < 4; ++jx)
                if (li[jx] == i) {
                    gj[jx] = S.spec[par][jx][lane] + rsp[jx * 2] * y0 + rsp[jx * 2 + 1] * y1;
                    rj[jx][0] = rsp[jx * 2] * Phi[0] + rsp[jx * 2 + 1] * Phi[2];
                    rj[jx][1] = rsp[jx * 2] * Phi[1] + rsp[jx * 2 + 1] * Phi[3];
                }
        }
        mv(m, y0, y1, t0, t1);
        y0 = t0 + yf0;
        y1 = t1 + yf1;
        if (multi) {
            T hc[4];
            mmul(h, Phi, hc);
            if (lane < 4) S.phi[i][lane] = Phi[lane], S.phi[i][4 + lane] = hc[lane];
            mmul(m, Phi, Phi);
        }
    }
    __syncwarp();
    FHP(0);
    // ---- backward fold, zero inflows: b = sum Mb.. c0_i, Pb = prod Mb, K = sum Mb.. Hc_i
    T Pb[4] = {T(1), T(0), T(0), T(1)}, Kc[4] = {T(0), T(0), T(0), T(0)}, b0 = T(0), b1 = T(0);
    for (int i = ncl - 1; i >= 0; --i) {
        T m[4], t0, t1;
        ld4(ctl + i * 12 + 4, m);
        mv(m, b0, b1, t0, t1);
        b0 = t0 + R[i][lane][2];
        b1 = t1 + R[i][lane][3];
        if (multi) {
            mmul(m, Pb, Pb);
            mmul(m, Kc, Kc);
#pragma unroll
            for (int e = 0; e < 4; ++e) Kc[e] += S.phi[i][4 + e];
        }
    }
    FHP(1);
    T Zc0 = T(0), Zc1 = T(0), y1c = b0, y2c = b1;   // one CTA: Y = Z = 0, (x_0, x_1) = my outflow
    T gv[4] = {gj[0], gj[1], gj[2], gj[3]};
    if (multi) {
        // ---- the one exchange: my summary to every CTA of the cluster (once every
        // CTA has consumed the previous group's)
        if (t >= 1) wait_cluster(&S.xcons, (uint32_t)((t - 1) & 1));
        FHP(2);
        for (int r = 0; r < A.cs; ++r) {
            st_peer2(mapa(&S.xa[c][lane][0], r), y0, y1);
            st_peer2(mapa(&S.xb[c][lane][0], r), b0, b1);
            if (lane < 4) {
                const uint32_t pp = mapa(&S.xP[c][0], r);
                st_peer(pp + lane * sizeof(T), Phi[lane]);
                st_peer(pp + (4 + lane) * sizeof(T), Pb[lane]);
                st_peer(pp + (8 + lane) * sizeof(T), Kc[lane]);
            }
            if (PER) {
#pragma unroll
                for (int jx = 0; jx < 4; ++jx)
                    if (A.srow[jx] >= 0 && A.srow[jx] / Q >= q0 && A.srow[jx] / Q < q0 + ncl) {
                        st_peer(mapa(&S.xg[jx][lane], r), gj[jx]);
                        if (lane < 2) st_peer(mapa(&S.xr[jx][lane], r), rj[jx][lane]);
                    }
            }
        }
        fence_cluster();
        __syncwarp();
        if (lane == 0)
            for (int r = 0; r < A.cs; ++r) arrive_remote(&S.xch, r);
        FHP(3);
        wait_cluster(&S.xch, (uint32_t)(t & 1));
        FHP(4);
        // ---- every CTA's forward inflow Y_v (kept per lane in S.yv), then backward inflows from the top
        {
            T ya = T(0), yb = T(0);
            for (int v = 0; v < A.cs; ++v) {
                S.yv[v][lane][0] = ya, S.yv[v][lane][1] = yb;
                T t0, t1;
                mv(S.xP[v], ya, yb, t0, t1);
                ya = t0 + S.xa[v][lane][0];
                yb = t1 + S.xa[v][lane][1];
            }
        }
        T Za = T(0), Zb = T(0);   // running backward inflow
        for (int v = A.cs - 1; v >= 0; --v) {
            if (v == c) Zc0 = Za, Zc1 = Zb;
            T t0, t1, u0, u1;
            mv(S.xP[v] + 4, Za, Zb, t0, t1);
            mv(S.xP[v] + 8, S.yv[v][lane][0], S.yv[v][lane][1], u0, u1);
            Za = t0 + u0 + S.xb[v][lane][0];
            Zb = t1 + u1 + S.xb[v][lane][1];
        }
        y1c = Za, y2c = Zb;
        // cyclic rows' g (read now: the exchange buffer is released right after)
        if (PER) {
#pragma unroll
            for (int jx = 0; jx < 4; ++jx)
                if (A.srow[jx] >= 0) {
                    const int ow = (int)(A.srow[jx] / Q) / A.cpc;   // owner CTA of the row's chunk
                    gv[jx] = S.xg[jx][lane] + S.xr[jx][0] * S.yv[ow][lane][0] + S.xr[jx][1] * S.yv[ow][lane][1];
                }
        }
        fence_cluster();
        __syncwarp();
        if (lane == 0)
            for (int r = 0; r < A.cs; ++r) arrive_remote(&S.xcons, r);   // this group's exchange consumed
        FHP(5);
        // ---- my chunks: yin_i = yin0_i + Phi_i Y, c_i = c0_i + Hc_i Y
        const T Y0 = S.yv[c][lane][0], Y1 = S.yv[c][lane][1];
        for (int i = 0; i < ncl; ++i) {
            T t0, t1, u0, u1;
            mv(S.phi[i], Y0, Y1, t0, t1);
            mv(S.phi[i] + 4, Y0, Y1, u0, u1);
            R[i][lane][0] += t0;
            R[i][lane][1] += t1;
            R[i][lane][2] += u0;
            R[i][lane][3] += u1;
        }
    }
    // ---- zin walk from Z_c
    T z0 = Zc0, z1 = Zc1;
    for (int i = ncl - 1; i >= 0; --i) {
        T m[4], t0, t1;
        ld4(ctl + i * 12 + 4, m);
        const T cq0 = R[i][lane][2], cq1 = R[i][lane][3];
        R[i][lane][2] = z0;
        R[i][lane][3] = z1;
        mv(m, z0, z1, t0, t1);
        z0 = t0 + cq0;
        z1 = t1 + cq1;
    }
    FHP(6);
    if (!PER) return;
    // ---- cyclic pair: (x_0, x_1) = CTA 0's backward outflow; g on the cyclic rows
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
    FHP(7);
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
    using C = CCfg<T, MODE>;
    constexpr int NS = C::NS, TILE = C::TILE;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1 KB aligned (the 128B swizzle of contiguous tiles); derived from smem_raw
    // by pointer arithmetic so the compiler keeps the shared address space
    CSmem<T, MODE> &sm = *reinterpret_cast<CSmem<T, MODE> *>(smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u));
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
        bar_init(&sm.xch, A.cs);
        bar_init(&sm.xcons, A.cs);
        for (int i = 0; i < NS; ++i) sm.seq[i] = -1;
        sm.claim = 0;
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
                        *(volatile int64_t *)&sm.seq[sl] = j;
                        bar_arrive(&sm.full[sl]);
                        continue;
                    }
                    sm.item[sl] = ((int64_t)type << 62) | ((int64_t)tg << 20) | i;
                    *(volatile int64_t *)&sm.seq[sl] = j;
                    const int g = cl + tg * A.ncl;
                    const int b = g / A.Gb, gl = g - b * A.Gb;
                    const int64_t r0 = (int64_t)(q0 + i) * Q;
                    const int kmax = (int)min((int64_t)Q, A.n - r0);
                    T *slot = sm.slot[sl];
                    const uint32_t cb = (A.dbg & 128) ? 0u : up16((uint32_t)(kmax * (type ? COEF_STRIDE : REC) * sizeof(T)));
                    uint32_t bytes = TILE * sizeof(T) + cb + C::HALO * sizeof(T);
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
                    if (cb) bulk_load(slot + TILE, type ? A.coef + r0 * COEF_STRIDE : A.rec + r0 * REC, cb, &sm.full[sl]);
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
                *(volatile int64_t *)&sm.seq[sl] = j;
                bar_arrive(&sm.full[sl]);
            }
        }
    } else if (warp < NWC) {
        // ---------------- consumers: each warp claims the next item (shared-memory
        // ticket), so a warp blocked on a dependency holds no slot and stalls no
        // other warp.  The slot's sequence tag is checked before its parity wait
        // (the fill of item j is the slot's phase j / NS once the tag reads j, so
        // the wait cannot alias another phase).  A tile's column goes to registers
        // and its coefficient rows to the warp's private buffer at once, so the
        // slot returns to the producer before the sweeps: the ring stays in flight.
        T *cp = sm.cpriv[warp];
        for (;;) {
            int64_t j = 0;
            if (lane == 0) j = atomicAdd(&sm.claim, 1);
            j = __shfl_sync(0xffffffffu, j, 0);
            const int sl = (int)(j % NS);
            while (*(volatile int64_t *)&sm.seq[sl] != j) {
            }
            bar_wait(&sm.full[sl], (uint32_t)((j / NS) & 1));
            const int64_t it = *(volatile int64_t *)&sm.item[sl];
            if (it == -1) break;
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
            const int64_t s_in_batch = (int64_t)gl * TW + lane;
            const bool ok = s_in_batch < A.M;
            if (MODE == MODE_CH1D) ch1d_rhs<T>(const_cast<T *>(d), d + TILE + C::COEF, kmax, lane, A.alpha);
            T v[Q];
#pragma unroll
            for (int k = 0; k < Q; ++k) v[k] = (A.dbg & 32) ? T(0) : tld<T, LAY>(d, k, lane);
            if (!(A.dbg & 16)) {
                // coefficient rows -> private buffer (16-byte shared loads / stores, lane-strided)
                constexpr int NV = C::COEF * (int)sizeof(T) / 16;
                const uint32_t src = su32(d + TILE), dst = su32(cp);
#pragma unroll
                for (int e = lane; e < NV; e += 32) {
                    uint32_t a, bq, cq, dq;
                    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(a), "=r"(bq), "=r"(cq), "=r"(dq) : "r"(src + e * 16));
                    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dst + e * 16), "r"(a), "r"(bq),
                                 "r"(cq), "r"(dq) : "memory");
                }
            }
            __syncwarp();
            if (lane == 0) bar_arrive(&sm.empty[sl]);
            if (!type) {
                // ---- P1: zero-inflow forward sweep, carry, back-substitution functional
                T y0 = T(0), y1 = T(0), a0 = T(0), a1 = T(0), gs[4] = {T(0), T(0), T(0), T(0)};
                const bool spec_tile = PER && q >= A.srow[0] / Q;
#pragma unroll
                for (int k = 0; k < Q; ++k) {
                    if (!(A.dbg & 4) && (kmax == Q || k < kmax)) {
                        T f0, f1, f2, wa, wb, wz;
                        lds2(cp + k * REC, f0, f1);
                        lds2(cp + k * REC + 2, f2, wa);
                        lds2(cp + k * REC + 4, wb, wz);
                        T tt = f0 * v[k];
                        if (K == 2) tt -= f2 * y0;
                        const T gg = tt - f1 * y1;   // newest carry last: one FMA on the chain
                        y0 = y1;
                        y1 = gg;
                        a0 += wa * gg;
                        a1 += wb * gg;
                        if (PER && spec_tile) {
#pragma unroll
                            for (int jx = 0; jx < 4; ++jx)
                                if (A.srow[jx] == r0 + k) gs[jx] = gg;
                        }
                    }
                }
                // the record buffer of this parity is free once P2 of group tg-2 has read it
                if (tg >= 2 && !(A.dbg & 64)) bar_wait(&sm.recfree[par], (uint32_t)(((tg - 2) >> 1) & 1));
                sm.rec[par][i][lane][0] = y0;
                sm.rec[par][i][lane][1] = y1;
                sm.rec[par][i][lane][2] = a0;
                sm.rec[par][i][lane][3] = a1;
                if (PER && spec_tile) {
#pragma unroll
                    for (int jx = 0; jx < 4; ++jx)
                        if (A.srow[jx] >= 0 && A.srow[jx] / Q == q) sm.spec[par][jx][lane] = gs[jx];
                }
                __syncwarp();
                if (lane == 0) bar_arrive(&sm.p1done[par]);
                continue;
            }
            // ---- P2: inflows and x_l of the group (scan done), sweeps, x out
            if (!(A.dbg & 64)) bar_wait(&sm.scandone[par], (uint32_t)((tg >> 1) & 1));
            const T yi0 = sm.rec[par][i][lane][0], yi1 = sm.rec[par][i][lane][1];
            const T zi0 = sm.rec[par][i][lane][2], zi1 = sm.rec[par][i][lane][3];
            T xl0 = T(0), xl1 = T(0);
            if (PER) xl0 = sm.xl[par][lane][0], xl1 = sm.xl[par][lane][1];
            __syncwarp();
            if (lane == 0) bar_arrive(&sm.recfree[par]);
            if (A.dbg & 4) {
            } else if (kmax == Q) tile_solve<T, K, PER, true>(v, cp, Q, yi0, yi1, zi0, zi1, xl0, xl1);
            else tile_solve<T, K, PER, false>(v, cp, kmax, yi0, yi1, zi0, zi1, xl0, xl1);
            if (PER && K == 2 && r0 + Q > A.n - 2) {
                const int k2 = (int)(A.n - 2 - r0);
#pragma unroll
                for (int k = 0; k < Q; ++k) {
                    if (k == k2) v[k] = xl0;
                    if (k == k2 + 1) v[k] = xl1;
                }
            }
            if (!ok || (A.dbg & 8)) continue;
            if (LAY == LAY_CONTIG) {
                // system = row of the output: 64 consecutive elements per lane
                T *x = A.xout + (int64_t)b * A.bstride + s_in_batch * A.pitch + r0;
                if (kmax == Q) {
#pragma unroll
                    for (int k = 0; k < Q; k += 16 / (int)sizeof(T)) {
                        if (sizeof(T) == 8)
                            __stcs(reinterpret_cast<double2 *>(x + k), make_double2((double)v[k], (double)v[k + 1]));
                        else
                            __stcs(reinterpret_cast<float4 *>(x + k),
                                   make_float4((float)v[k], (float)v[k + 1], (float)v[k + 2], (float)v[k + 3]));
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < Q; ++k)
                        if (k < kmax) __stcs(x + k, v[k]);
                }
                continue;
            }
            {
                // x in place: every row of the tile is one contiguous 32-system segment
                // (opaque stride: one running address instead of Q live ones)
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
            if (!(A.dbg & 1)) cluster_scan<T, K, PER, CSMAX>(A, sm, A.ct + (int64_t)q0 * 12, A.rsp, t, c, q0, ncl, lane);
            __syncwarp();
            if (lane == 0) bar_arrive(&sm.scandone[par]);
        }
    }
    // no CTA may leave while a peer can still write into its shared memory
    cg::this_cluster().sync();
}

}  // namespace fc
}  // namespace pb

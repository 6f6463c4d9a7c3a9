// twopass.cuh — the shared-LHS interleaved batched solve as two streaming
// kernels (pent_solve / tri_solve / pent_solve_many / pent_solve_strided on
// the interleaved layout whenever a system spans more than one held-tile CTA).
//
// The thesis solves one system per thread over all N rows (P:1712-1724,
// P:1729): at N = M = 8192 that is a 16 K-row dependent chain per thread and
// < 2 warps per SM.  Here a system is cut into chunks of Q = 64 rows and one
// warp owns one TILE = (chunk q, group g of 32 consecutive systems): lane =
// system, every tile row is one contiguous 256 B (fp64) / 128 B (fp32) segment
// of the interleaved array, and every coefficient read is a
// warp-uniform shared-memory broadcast.
//
//   tp_p1_kernel  P1 of every tile: forward sweep with zero inflow -> forward
//                 carry yF = (g_{r1-2}, g_{r1-1}); the chunk's zero-inflow
//                 back-substitution carry zB = sum_k W_k g_k (W_k = rows r0,
//                 r0+1 of L^{-1}, from the factor tables) accumulated on the
//                 fly.  Reads f once, writes 4 values per (system, chunk).
//   tp_scan_kernel one warp per group folds the chunk records:
//                 the affine chunk maps (Mf_q, Mb_q, H_q) folded over q -> the
//                 true inflows (yin_q, zin_q) and, cyclic, Navon's /
//                 Sherman–Morrison's pair x_l.
//   tp_p2_kernel  P2 of every tile, in REVERSE tile order (its first tiles are
//                 the ones P1 read last, still in L2): forward sweep from yin_q,
//                 back substitution from zin_q, cyclic correction x - Z x_l
//                 (eq:solve), x stored in place.
// The three launches are chained as programmatic dependents: each starts while
// its predecessor drains (P2 issues its first tile loads before it waits: f
// is not written by P1 or the scan).
//
// Every consumer warp streams its own tiles through its own ring of R slots
// (one TMA box + one bulk copy of the chunk's coefficient rows per slot) and
// issues the refills itself: a slot is only ever waited on by the warp that
// filled it, so an mbarrier parity wait cannot alias an older phase.
#pragma once
#include "fused_hold.cuh"

namespace pb {
namespace tp {

#ifdef TP_PROF
__device__ unsigned long long tp_prof[16];   // DEV ONLY: per-phase cycles summed over warps
#define TPQ(i) do { long long _n = clock64(); _acc[i] += _n - _t; _t = _n; } while (0)
#define TPQ_INIT long long _t = clock64(), _acc[16] = {0}
#define TPQ_DONE do { if (lane == 0) for (int _i = 0; _i < 16; ++_i) if (_acc[_i]) atomicAdd(&tp_prof[_i], (unsigned long long)_acc[_i]); } while (0)
#else
#define TPQ(i) do {} while (0)
#define TPQ_INIT do {} while (0)
#define TPQ_DONE do {} while (0)
#endif

using fs::Q;
using fs::REC;
using fs::TW;
using fs::bar_expect_tx;
using fs::bar_init;
using fs::bar_wait;
using fs::bulk_load;
using fs::lds2;
using fs::su32;
using fs::tma_load2;
using fs::tma_load3;

template <typename T>
struct Args {
    const T *rec, *coef, *ct, *rsp;
    const double *scal;
    T *x;               // right-hand sides, solved in place
    T *car;             // [G][nq][4][TW] chunk records: (yF0, yF1, zB0, zB1) -> (yin0, yin1, zin0, zin1)
    T *spec;            // [G][4][TW] zero-inflow g on the cyclic rows
    T *xl;              // [G][2][TW]
    int64_t n, M;       // rows, systems per batch
    int64_t bstride;    // elements between batches
    int64_t pitch;      // elements between rows
    int64_t ntiles;     // G * nq
    int64_t keep_from;  // P1 loads tiles >= keep_from with the default L2 policy (P2 re-reads them first)
    int64_t srow[4];
    int nq, Gb, G;
    int BG;             // groups per band (tile order: bands of BG groups, chunk-major inside a band)
    int flat;           // one 2-D map (M, n * count): row b * n + r
};

// tile t -> (group, chunk).  Bands of BG consecutive groups (BG * 32 systems:
// 4 KB of every row) in order; inside a band chunk-major, groups fastest, so
// the tiles in flight at any moment read a few contiguous row blocks of the
// interleaved array (DRAM-page friendly) while every band's groups complete
// early enough for their scans to overlap the streaming of later bands.
struct TC {
    int64_t g;
    int q;
};
template <typename T>
__device__ __forceinline__ TC tile_coords(const Args<T> &A, int64_t t)
{
    // 32-bit arithmetic (the launcher keeps ntiles < 2^31)
    const unsigned per = (unsigned)A.BG * (unsigned)A.nq, tt = (unsigned)t;
    const unsigned b = tt / per, rel = tt - b * per;
    const unsigned bg = min((unsigned)A.BG, (unsigned)A.G - b * (unsigned)A.BG);
    const unsigned q = rel / bg;
    TC c;
    c.q = (int)q;
    c.g = (int64_t)(b * (unsigned)A.BG + (rel - q * bg));
    return c;
}

// P2 sweeps of a full tile column in registers (coefficient rows cp in the
// band_core layout F0 F1 F2 - B1 B2 Z1 Z2), split so the slot refill can be
// issued between them: once the forward sweep has run, every value read from
// the slot has been consumed.  Each recurrence takes its newest carry last.
constexpr int PD2 = 4;
template <typename T, int K>
__device__ __forceinline__ void p2_fwd(T (&v)[Q], const T *cp, T y0, T y1)
{
    T c01[PD2][2], c2[PD2][2];
#pragma unroll
    for (int k = 0; k < PD2; ++k) {
        lds2(cp + k * COEF_STRIDE, c01[k][0], c01[k][1]);
        lds2(cp + k * COEF_STRIDE + 2, c2[k][0], c2[k][1]);
    }
#pragma unroll
    for (int k = 0; k < Q; ++k) {
        const int sl = k % PD2;
        const T f0 = c01[sl][0], f1 = c01[sl][1], f2 = c2[sl][0];
        if (k + PD2 < Q) {
            lds2(cp + (k + PD2) * COEF_STRIDE, c01[sl][0], c01[sl][1]);
            lds2(cp + (k + PD2) * COEF_STRIDE + 2, c2[sl][0], c2[sl][1]);
        }
        T t = f0 * v[k];
        if (K == 2) t -= f2 * y0;
        const T g = t - f1 * y1;
        y0 = y1;
        y1 = g;
        v[k] = g;
    }
}
template <typename T, int K, bool PER>
__device__ __forceinline__ void p2_bwd(T (&v)[Q], const T *cp, T z0, T z1, T xl0, T xl1)
{
    T cb[PD2][2], cz[PD2][2];
#pragma unroll
    for (int j = 0; j < PD2; ++j) {
        const int k = Q - 1 - j;
        lds2(cp + k * COEF_STRIDE + 4, cb[j][0], cb[j][1]);
        if (PER) lds2(cp + k * COEF_STRIDE + 6, cz[j][0], cz[j][1]);
    }
#pragma unroll
    for (int j = 0; j < Q; ++j) {
        const int k = Q - 1 - j, sl = j % PD2;
        const T b1 = cb[sl][0], b2 = cb[sl][1], z1v = PER ? cz[sl][0] : T(0), z2v = PER ? cz[sl][1] : T(0);
        if (j + PD2 < Q) {
            lds2(cp + (k - PD2) * COEF_STRIDE + 4, cb[sl][0], cb[sl][1]);
            if (PER) lds2(cp + (k - PD2) * COEF_STRIDE + 6, cz[sl][0], cz[sl][1]);
        }
        T t = v[k];
        if (K == 2) t -= b2 * z1;
        const T xx = t - b1 * z0;
        z1 = z0;
        z0 = xx;
        if (PER) {
            T o = xx - z1v * xl0;   // cyclic correction (Navon eq:solve / Sherman–Morrison)
            if (K == 2) o -= z2v * xl1;
            v[k] = o;
        } else {
            v[k] = xx;
        }
    }
}

// the 1-KB-aligned dynamic shared memory of either kernel
__device__ __forceinline__ unsigned char *smem_base()
{
    extern __shared__ __align__(1024) unsigned char tp_smem[];
    return tp_smem + ((1024u - (su32(tp_smem) & 1023u)) & 1023u);
}

// The tile (chunk q of group g) into dst.  Interleaved: one TMA box (32
// systems, 64 rows).  Contiguous (rows of a grid, the ADI x-sweep): Q/EB boxes
// of (EB unknowns = 128 B, 32 systems), 128B-swizzled (fs::csw) so the lanes
// read their own systems' unknown k conflict-free.
template <typename T, int LAY>
__device__ __forceinline__ void tile_box(const CUtensorMap *tm, const Args<T> &A, int64_t g, int q, T *dst,
                                         uint64_t *bar, uint64_t pol, bool store)
{
    const int b = (int)(g / A.Gb), gl = (int)(g - (int64_t)b * A.Gb);
    if (LAY == fs::LAY_CONTIG) {
#pragma unroll
        for (int bx = 0; bx < Q / fs::Sw<T>::EB; ++bx) {
            T *d = dst + bx * TW * fs::Sw<T>::EB;
            const int r = q * Q + bx * fs::Sw<T>::EB;
            if (store) {
                if (A.flat) fs::tma_store2(tm, r, (int)((int64_t)b * A.M + gl * TW), d);
                else fs::tma_store3(tm, r, gl * TW, b, d);
            } else {
                if (A.flat) tma_load2(d, tm, r, (int)((int64_t)b * A.M + gl * TW), bar, pol);
                else tma_load3(d, tm, r, gl * TW, b, bar, pol);
            }
        }
    } else if (store) {
        if (A.flat) fs::tma_store2(tm, gl * TW, (int)((int64_t)b * A.n + (int64_t)q * Q), dst);
        else fs::tma_store3(tm, gl * TW, q * Q, b, dst);
    } else {
        if (A.flat) tma_load2(dst, tm, gl * TW, (int)((int64_t)b * A.n + (int64_t)q * Q), bar, pol);
        else tma_load3(dst, tm, gl * TW, q * Q, b, bar, pol);
    }
}
template <typename T, int LAY>
__device__ __forceinline__ void issue_tile(const CUtensorMap *tm, const Args<T> &A, int64_t g, int q, T *dst,
                                           uint64_t *bar, const T *rows, uint32_t row_bytes, uint64_t pol,
                                           uint32_t extra_tx = 0)
{
    bar_expect_tx(bar, (uint32_t)(Q * TW * sizeof(T)) + row_bytes + extra_tx);
    tile_box<T, LAY>(tm, A, g, q, dst, bar, pol, false);
    bulk_load(dst + Q * TW, rows, row_bytes, bar);
}


// ---------------------------------------------------------------- P1 of one tile (one warp)
constexpr int PD = 4;   // coefficient rows software-pipelined this many rows ahead

// zero-inflow forward sweep of the tile (smem [Q][TW]) with the chunk's rows
// (F0, F1, F2, Wa, Wb, 0) -> forward carry (y0, y1), functional (a0, a1); hist
// = g of the last four rows swept (the cyclic rows are the last four of the
// system, hence of their tile).  FULL: kmax == Q.
template <typename T, int K, bool PER, bool FULL, int LAY>
__device__ __forceinline__ void p1_tile(const T *d, const T *c, int lane, int kmax, T &y0, T &y1, T &a0, T &a1,
                                        T (&hist)[4])
{
    y0 = y1 = a0 = a1 = T(0);
    T cf[PD][6], vv[PD];
#pragma unroll
    for (int u = 0; u < PD; ++u) {
        lds2(c + u * REC, cf[u][0], cf[u][1]);
        lds2(c + u * REC + 2, cf[u][2], cf[u][3]);
        lds2(c + u * REC + 4, cf[u][4], cf[u][5]);
        vv[u] = fs::tld<T, LAY>(d, u, lane);
    }
#pragma unroll
    for (int kk = 0; kk < Q; ++kk) {
        const int sl = kk % PD;
        const T f0 = cf[sl][0], f1 = cf[sl][1], f2 = cf[sl][2], wa = cf[sl][3], wb = cf[sl][4], v = vv[sl];
        if (kk + PD < Q) {
            lds2(c + (kk + PD) * REC, cf[sl][0], cf[sl][1]);
            lds2(c + (kk + PD) * REC + 2, cf[sl][2], cf[sl][3]);
            lds2(c + (kk + PD) * REC + 4, cf[sl][4], cf[sl][5]);
            vv[sl] = fs::tld<T, LAY>(d, kk + PD, lane);
        }
        if (FULL || kk < kmax) {
            T tt = f0 * v;
            if (K == 2) tt -= f2 * y0;
            const T gg = tt - f1 * y1;   // newest carry last: one FMA on the chain
            y0 = y1;
            y1 = gg;
            a0 += wa * gg;
            a1 += wb * gg;
            if (PER) hist[kk & 3] = gg;
        }
    }
}

// ---------------------------------------------------------------- P1 (+ the group scans)
template <typename T, int NC, int R>
struct P1Smem {
    // (1 KB multiples: the contiguous layout's 128B-swizzled boxes)
    static constexpr int SLOT = ((Q * TW + Q * REC) * (int)sizeof(T) + 1023) / 1024 * 1024 / (int)sizeof(T);
    T slot[NC][R][SLOT];
    uint64_t full[NC][R];
};

// NC consumer warps stream the tiles; nothing waits on anything but its own
// slot (no fences, no counters): the kernel boundary publishes the records.
template <typename T, int K, bool PER, int NC, int R, int LAY>
__global__ void __launch_bounds__(32 * NC, 1) tp_p1_kernel(const __grid_constant__ CUtensorMap tmap, const Args<T> A)
{
    using S = P1Smem<T, NC, R>;
    S &sm = *reinterpret_cast<S *>(smem_base());
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // the scan may launch now: it only touches the records after griddepcontrol.wait
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (lane == 0)
        for (int r = 0; r < R; ++r) bar_init(&sm.full[w][r], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const int64_t W = (int64_t)blockIdx.x * NC + w, NWT = (int64_t)gridDim.x * NC;
    const uint64_t pol_first = fs::policy_evict_first();
    const uint32_t rb = (uint32_t)(Q * REC * sizeof(T));
    auto issue = [&](int64_t t, int r) {
        const TC tc = tile_coords(A, t);
        uint64_t pol = pol_first;
        if (t >= A.keep_from) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
        issue_tile<T, LAY>(&tmap, A, tc.g, tc.q, sm.slot[w][r], &sm.full[w][r], A.rec + (int64_t)tc.q * Q * REC, rb,
                           pol);
    };
    if (lane == 0)
        for (int r = 0; r < R; ++r)
            if (W + r * NWT < A.ntiles) issue(W + r * NWT, r);
    int k = 0;
    TPQ_INIT;
    for (int64_t t = W; t < A.ntiles; t += NWT, ++k) {
        const int r = k % R;
        bar_wait(&sm.full[w][r], (uint32_t)((k / R) & 1));
        TPQ(0);
        const T *d = sm.slot[w][r];
        const T *c = d + Q * TW;
        const TC tc = tile_coords(A, t);
        const int64_t g = tc.g;
        const int q = tc.q;
        const int64_t r0 = (int64_t)q * Q;
        // zero-inflow forward sweep, carry and back-substitution functional
        T y0, y1, a0, a1;
        T hist[4] = {T(0), T(0), T(0), T(0)};
        if (A.n - r0 >= Q) p1_tile<T, K, PER, true, LAY>(d, c, lane, Q, y0, y1, a0, a1, hist);
        else p1_tile<T, K, PER, false, LAY>(d, c, lane, (int)(A.n - r0), y0, y1, a0, a1, hist);
        TPQ(1);
        // every value read from the slot has been consumed by the sweep: the
        // slot can take its refill
        __syncwarp();
        if (lane == 0 && t + R * NWT < A.ntiles) issue(t + R * NWT, r);
        // arrival of the PREVIOUS tile: its records were stored one tile ago,
        // so the fence that publishes them has (almost) nothing left to wait for
        TPQ(2);
        T *o = A.car + (g * A.nq + q) * 4 * TW + lane;
        __stcg(o, y0);
        __stcg(o + TW, y1);
        __stcg(o + 2 * TW, a0);
        __stcg(o + 3 * TW, a1);
        if (PER) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t rr = A.srow[j] - r0;
                if (A.srow[j] >= 0 && rr >= 0 && rr < Q) {
                    const int jj = (int)(rr & 3);
                    __stcg(A.spec + (g * 4 + j) * TW + lane, jj == 0 ? hist[0] : jj == 1 ? hist[1] : jj == 2 ? hist[2] : hist[3]);
                }
            }
        }
    }
    TPQ_DONE;
}

// ---------------------------------------------------------------- the scan kernel
// One CTA per group, one warp per segment of SL consecutive chunks (lane =
// system), all of a segment's records loaded up front (one memory latency).
//   pass A (segment inflows zero): y <- Mf_i y + yF_i gives the segment's
//     forward outflow a; cz0_i = zB_i + H_i y; its backward outflow for zero
//     outflow from above, b = sum_i Qb_i cz0_i (Qb_i = Mb_c0 ... Mb_{i-1}),
//     accumulated forward; the lane-uniform maps P = prod Mf, Pb = prod Mb and
//     Kc = sum_i Qb_i H_i Phi_i (Phi_i = Mf_{i-1} ... Mf_c0: b's response to
//     the segment's forward inflow Y).
//   combine (every warp, from shared memory): Y_{s+1} = P_s Y_s + a_s;
//     Z above the last segment = 0, Z_{s-1} = Pb_s Z_s + Kc_s Y_s + b_s.
//   pass B: the walks again from the true (Y_s, Z_s) -> yin_i, zin_i stored.
// The same affine algebra as hold_scan (fused_hold.cuh); cyclic: the true g
// on the four last rows and (x_0, x_1) = Z_{-1} give Navon's / Sherman–
// Morrison's x_l.  A programmatic dependent of P1 (launches while P1 runs).
constexpr int SL = 16;      // chunks per segment
constexpr int SEGMAX = 8;   // warps per CTA (the full register budget each)
constexpr int NSEG = 32;    // segments per group: nq <= 512 (a warp folds segments w, w + 8, ...)
// shared memory of one scan CTA, sized by its segment count nsg:
// a, b, ys [nsg][TW][2] | m [nsg][12] (P, Pb, Kc) | gv [4][TW] | chunk maps ct[nq][12]
template <typename T>
struct ScanView {
    T (*a)[TW][2];
    T (*b)[TW][2];
    T (*ys)[TW][2];
    T (*m)[12];
    T (*gv)[TW];
    T *ctm;
};
template <typename T>
__host__ __device__ inline size_t scan_smem_elems(int nsg, int nq)
{
    return ((size_t)nsg * (TW * 2 * 3 + 12) + 4 * TW + 1) / 2 * 2 + (size_t)nq * 12;
}

// SLT: chunks per segment (SL; 8 for systems of <= 8 chunks, whose records
// then need half the registers: more resident warps)
template <typename T, int K, bool PER, int SLT = SL>
__global__ void __launch_bounds__(32 * SEGMAX, SLT <= 8 ? 2 : 1) tp_scan_kernel(const Args<T> A)
{
    extern __shared__ __align__(16) unsigned char tp_scan_smem[];
    const int nsg0 = (A.nq + SLT - 1) / SLT;
    ScanView<T> sm;
    {
        T *p = reinterpret_cast<T *>(tp_scan_smem);
        sm.a = reinterpret_cast<T(*)[TW][2]>(p);
        sm.b = sm.a + nsg0;
        sm.ys = sm.b + nsg0;
        sm.m = reinterpret_cast<T(*)[12]>(sm.ys + nsg0);
        sm.gv = reinterpret_cast<T(*)[TW]>(sm.m + nsg0);
        sm.ctm = p + (((size_t)nsg0 * (TW * 2 * 3 + 12) + 4 * TW + 1) / 2 * 2);   // 16-byte aligned
    }
    T *ctm = sm.ctm;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    for (int e = threadIdx.x; e < A.nq * 12; e += blockDim.x) ctm[e] = A.ct[e];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
    const int nsg = (A.nq + SLT - 1) / SLT;
    const int64_t g = blockIdx.x;
    T *cg0 = A.car + g * A.nq * 4 * TW + lane;
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // ---- pass A: every segment of this warp with zero inflows
    for (int sg = w; sg < nsg; sg += nwarp) {
        const int c0 = sg * SLT, nc = min(SLT, A.nq - c0);
        const T *cr = cg0 + (int64_t)c0 * 4 * TW;
        T r[SLT][4];
#pragma unroll
        for (int i = 0; i < SLT; ++i)
            if (i < nc) {
#pragma unroll
                for (int e = 0; e < 4; ++e) r[i][e] = __ldcg(cr + (i * 4 + e) * TW);
            }
        T y0 = T(0), y1 = T(0), b0 = T(0), b1 = T(0);
        T Ph[4] = {T(1), T(0), T(0), T(1)}, Qb[4] = {T(1), T(0), T(0), T(1)}, Kc[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
        for (int i = 0; i < SLT; ++i)
            if (i < nc) {
                const T *m = ctm + (c0 + i) * 12;
                T mf[4], mb[4], h[4];
                lds2(m, mf[0], mf[1]);
                lds2(m + 2, mf[2], mf[3]);
                lds2(m + 4, mb[0], mb[1]);
                lds2(m + 6, mb[2], mb[3]);
                lds2(m + 8, h[0], h[1]);
                lds2(m + 10, h[2], h[3]);
                const T c0v = r[i][2] + (h[0] * y0 + h[1] * y1), c1v = r[i][3] + (h[2] * y0 + h[3] * y1);
                b0 += Qb[0] * c0v + Qb[1] * c1v;
                b1 += Qb[2] * c0v + Qb[3] * c1v;
                const T n0 = (mf[0] * y0 + mf[1] * y1) + r[i][0], n1 = (mf[2] * y0 + mf[3] * y1) + r[i][1];
                y0 = n0, y1 = n1;
                T hp[4], qh[4];
                fs::mmul(h, Ph, hp);
                fs::mmul(Qb, hp, qh);
#pragma unroll
                for (int e = 0; e < 4; ++e) Kc[e] += qh[e];
                fs::mmul(Qb, mb, Qb);
                fs::mmul(mf, Ph, Ph);
            }
        sm.a[sg][lane][0] = y0, sm.a[sg][lane][1] = y1;
        sm.b[sg][lane][0] = b0, sm.b[sg][lane][1] = b1;
        if (lane < 4) sm.m[sg][lane] = Ph[lane], sm.m[sg][4 + lane] = Qb[lane], sm.m[sg][8 + lane] = Kc[lane];
    }
    __syncthreads();
    // ---- combine (warp 0): every segment's true inflows Y (forward) and Z
    // (from above) into shared memory, (x_0, x_1) = the outflow of segment 0
    if (w == 0) {
        T ya = T(0), yb = T(0);
        for (int v = 0; v < nsg; ++v) {
            sm.ys[v][lane][0] = ya, sm.ys[v][lane][1] = yb;
            T t0, t1;
            fs::mv(sm.m[v], ya, yb, t0, t1);
            ya = t0 + sm.a[v][lane][0];
            yb = t1 + sm.a[v][lane][1];
        }
        T za = T(0), zb = T(0);
        for (int v = nsg - 1; v >= 0; --v) {
            T t0, t1, u0, u1;
            fs::mv(sm.m[v] + 4, za, zb, t0, t1);
            fs::mv(sm.m[v] + 8, sm.ys[v][lane][0], sm.ys[v][lane][1], u0, u1);
            sm.a[v][lane][0] = za, sm.a[v][lane][1] = zb;   // a[v] := Z above segment v
            za = t0 + u0 + sm.b[v][lane][0];
            zb = t1 + u1 + sm.b[v][lane][1];
        }
        sm.b[0][lane][0] = za, sm.b[0][lane][1] = zb;   // b[0] := (x_0, x_1)
    }
    __syncthreads();
    const T x0 = sm.b[0][lane][0], x1 = sm.b[0][lane][1];
    // ---- pass B: the walks again from the true (Y, Z) of each of this warp's segments
    for (int sg = w; sg < nsg; sg += nwarp) {
        const int c0 = sg * SLT, nc = min(SLT, A.nq - c0);
        T *cr = cg0 + (int64_t)c0 * 4 * TW;
        int qs[4] = {-1, -1, -1, -1};
        if (PER) {
#pragma unroll
            for (int j = 0; j < 4; ++j) qs[j] = A.srow[j] >= 0 ? (int)(A.srow[j] / Q) - c0 : -1;
        }
        T r[SLT][4], cz[SLT][2];
#pragma unroll
        for (int i = 0; i < SLT; ++i)
            if (i < nc) {
#pragma unroll
                for (int e = 0; e < 4; ++e) r[i][e] = __ldcg(cr + (i * 4 + e) * TW);
            }
        T y0 = sm.ys[sg][lane][0], y1 = sm.ys[sg][lane][1];
#pragma unroll
        for (int i = 0; i < SLT; ++i)
            if (i < nc) {
                const T *m = ctm + (c0 + i) * 12;
                T mf[4], h[4];
                lds2(m, mf[0], mf[1]);
                lds2(m + 2, mf[2], mf[3]);
                lds2(m + 8, h[0], h[1]);
                lds2(m + 10, h[2], h[3]);
                cz[i][0] = r[i][2] + (h[0] * y0 + h[1] * y1);
                cz[i][1] = r[i][3] + (h[2] * y0 + h[3] * y1);
                if (PER) {
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (qs[j] == i)
                            sm.gv[j][lane] = __ldcg(A.spec + (g * 4 + j) * TW + lane) + (A.rsp[2 * j] * y0 +
                                                                                          A.rsp[2 * j + 1] * y1);
                }
                const T n0 = (mf[0] * y0 + mf[1] * y1) + r[i][0], n1 = (mf[2] * y0 + mf[3] * y1) + r[i][1];
                r[i][0] = y0, r[i][1] = y1;
                y0 = n0, y1 = n1;
            }
        T z0 = sm.a[sg][lane][0], z1 = sm.a[sg][lane][1];
#pragma unroll
        for (int i = SLT - 1; i >= 0; --i)
            if (i < nc) {
                T mb[4];
                lds2(ctm + (c0 + i) * 12 + 4, mb[0], mb[1]);
                lds2(ctm + (c0 + i) * 12 + 6, mb[2], mb[3]);
                r[i][2] = z0, r[i][3] = z1;
                const T n0 = (mb[0] * z0 + mb[1] * z1) + cz[i][0], n1 = (mb[2] * z0 + mb[3] * z1) + cz[i][1];
                z0 = n0, z1 = n1;
            }
#pragma unroll
        for (int i = 0; i < SLT; ++i)
            if (i < nc) {
#pragma unroll
                for (int e = 0; e < 4; ++e) __stcg(cr + (i * 4 + e) * TW, r[i][e]);
            }
    }
    if (!PER) return;
    __syncthreads();
    if (w != 0) return;
    // cyclic pair from (x_0, x_1) and the true g on the last rows
    const double *sc = A.scal;
    T gv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) gv[j] = A.srow[j] >= 0 ? sm.gv[j][lane] : T(0);
    T xl0, xl1;
    if (K == 2) {
        // Navon (eq:first_two)
        const T ym1 = gv[1], ym2 = gv[0] - T(sc[10]) * gv[1];
        const T qa = gv[2] - (T(sc[4]) * x0 + T(sc[5]) * ym2 + T(sc[6]) * ym1);
        const T qb = gv[3] - (T(sc[7]) * x0 + T(sc[8]) * x1 + T(sc[9]) * ym1);
        xl0 = T(sc[0]) * qa + T(sc[1]) * qb;
        xl1 = T(sc[2]) * qa + T(sc[3]) * qb;
    } else {
        // Sherman–Morrison
        xl0 = (x0 + T(sc[0]) * gv[0]) / T(sc[1]);
        xl1 = T(0);
    }
    __stcg(A.xl + (g * 2 + 0) * TW + lane, xl0);
    __stcg(A.xl + (g * 2 + 1) * TW + lane, xl1);
}

// ---------------------------------------------------------------- P2
template <typename T, int NC, int R>
struct P2Smem {
    // tile | coefficient rows | the tile's inflows [4][TW] | x_l [2][TW]
    static constexpr int INF = Q * TW + Q * COEF_STRIDE, XL = INF + 4 * TW;
    static constexpr int SLOT = ((XL + 2 * TW) * (int)sizeof(T) + 1023) / 1024 * 1024 / (int)sizeof(T);
    T slot[NC][R][SLOT];
    T cpriv[NC][Q * COEF_STRIDE];   // the current tile's coefficient rows (its slot is refilled early)
    uint64_t full[NC][R];
};

template <typename T, int K, bool PER, int NC, int R, int LAY>
__global__ void __launch_bounds__(32 * NC, 1) tp_p2_kernel(const __grid_constant__ CUtensorMap tmap, const Args<T> A)
{
    using S = P2Smem<T, NC, R>;
    S &sm = *reinterpret_cast<S *>(smem_base());
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0)
        for (int r = 0; r < R; ++r) bar_init(&sm.full[w][r], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const int64_t W = (int64_t)blockIdx.x * NC + w, NWT = (int64_t)gridDim.x * NC;
    const uint64_t pol = fs::policy_evict_first();
    const uint32_t rb = (uint32_t)(Q * COEF_STRIDE * sizeof(T));
    auto tile_of = [&](int64_t i) { return A.ntiles - 1 - i; };   // reverse order: L2-warm tiles first
    // the tile's inflows and x_l ride in the slot (bulk copies on the same
    // mbarrier: the tile's expect_tx covers them)
    const uint32_t ib = (uint32_t)(4 * TW * sizeof(T)), xb = PER ? (uint32_t)(2 * TW * sizeof(T)) : 0u;
    auto issue_in = [&](int64_t i, int r) {
        const TC tc = tile_coords(A, tile_of(i));
        T *dst = sm.slot[w][r];
        bulk_load(dst + S::INF, A.car + (tc.g * A.nq + tc.q) * 4 * TW, ib, &sm.full[w][r]);
        if (PER) bulk_load(dst + S::XL, A.xl + tc.g * 2 * TW, xb, &sm.full[w][r]);
    };
    auto issue = [&](int64_t i, int r, bool with_in) {
        const TC tc = tile_coords(A, tile_of(i));
        issue_tile<T, LAY>(&tmap, A, tc.g, tc.q, sm.slot[w][r], &sm.full[w][r],
                           A.coef + (int64_t)tc.q * Q * COEF_STRIDE, rb, pol, ib + xb);
        if (with_in) issue_in(i, r);
    };
    // f and the coefficients are not written by P1 or the scan: the first
    // tiles go out before the dependency wait, their inflows after it
    if (lane == 0)
        for (int r = 0; r < R; ++r)
            if (W + r * NWT < A.ntiles) issue(W + r * NWT, r, false);
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (lane == 0)
        for (int r = 0; r < R; ++r)
            if (W + r * NWT < A.ntiles) issue_in(W + r * NWT, r);
    T *cp = sm.cpriv[w];
    int k = 0;
    TPQ_INIT;
    for (int64_t i = W; i < A.ntiles; i += NWT, ++k) {
        const int r = k % R;
        const TC tc = tile_coords(A, tile_of(i));
        const int64_t g = tc.g;
        const int q = tc.q;
        const int64_t r0 = (int64_t)q * Q;
        const int kmax = (int)min((int64_t)Q, A.n - r0);
        const int b = (int)(g / A.Gb), gl = (int)(g - (int64_t)b * A.Gb);
        bar_wait(&sm.full[w][r], (uint32_t)((k / R) & 1));
        TPQ(8);
        const T *d = sm.slot[w][r];
        const T yi0 = d[S::INF + lane], yi1 = d[S::INF + TW + lane], zi0 = d[S::INF + 2 * TW + lane],
                zi1 = d[S::INF + 3 * TW + lane];
        T xl0 = T(0), xl1 = T(0);
        if (PER) xl0 = d[S::XL + lane], xl1 = d[S::XL + TW + lane];
        T v[Q];
#pragma unroll
        for (int kk = 0; kk < Q; ++kk) v[kk] = fs::tld<T, LAY>(d, kk, lane);
        {
            // the coefficient rows into the warp's private buffer (16-byte units)
            const float4 *src = reinterpret_cast<const float4 *>(d + Q * TW);
            float4 *dst = reinterpret_cast<float4 *>(cp);
            constexpr int NV = Q * COEF_STRIDE * (int)sizeof(T) / 16;
#pragma unroll
            for (int e = lane; e < NV; e += 32) dst[e] = src[e];
        }
        __syncwarp();   // cp complete
        // x goes back through the slot: the tile column into the slot, one TMA
        // store of the box, and the slot's refill once the store has read it
        if (kmax == Q) {
            TPQ(9);
            p2_fwd<T, K>(v, cp, yi0, yi1);
            TPQ(10);
            p2_bwd<T, K, PER>(v, cp, zi0, zi1, xl0, xl1);
            TPQ(11);
        } else {
            fs::tile_solve<T, K, PER, false>(v, cp, kmax, yi0, yi1, zi0, zi1, xl0, xl1);
        }
        if (PER && K == 2 && r0 + Q > A.n - 2) {
            const int k2 = (int)(A.n - 2 - r0);
#pragma unroll
            for (int kk = 0; kk < Q; ++kk) {
                if (kk == k2) v[kk] = xl0;
                if (kk == k2 + 1) v[kk] = xl1;
            }
        }
        T *dw = sm.slot[w][r];
#pragma unroll
        for (int kk = 0; kk < Q; ++kk) fs::tst<T, LAY>(dw, kk, lane, v[kk]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();   // (also: cp is rewritten by the next tile)
        if (lane == 0) {
            tile_box<T, LAY>(&tmap, A, g, q, dw, nullptr, 0, true);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            if (i + R * NWT < A.ntiles) {
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                issue(i + R * NWT, r, true);
            }
        }
        __syncwarp();
        TPQ(12);
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    TPQ_DONE;
}

}  // namespace tp
}  // namespace pb

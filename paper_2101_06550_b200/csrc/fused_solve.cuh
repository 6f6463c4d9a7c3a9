// fused_solve.cuh — the shared-LHS interleaved solve as ONE persistent kernel
// (pent_solve / tri_solve / pent_solve_many / the ADI y-sweep).
//
// The thesis solves one system per thread over all N rows (P:1712-1724,
// P:1729): at N = M = 8192 that is a dependent chain of 16 K rows per thread
// and < 2 warps per SM.  Here every system is cut into chunks of Q = 64 rows
// and one consumer warp owns one TILE = (chunk q, group g of 32 consecutive
// systems): lane = system, so every tile row is one contiguous 256 B (fp64) /
// 128 B (fp32) segment of the interleaved array and every
// coefficient read is a warp-uniform shared-memory broadcast.
//
// Three kinds of work share one launch:
//   P1(g, q)  forward sweep of the tile with zero inflow -> forward carry
//             yF = (g_{r1-2}, g_{r1-1}); the chunk's back-substitution carry
//             with zero inflow is a linear functional of g (zB = sum W_k g_k,
//             W_k = rows r0, r0+1 of L^{-1}), accumulated on the fly.  Reads f
//             from HBM once, writes 4 values per (system, chunk).
//   scan(g)   when all P1 tiles of group g are done, a team of NSW scan warps
//             composes the affine chunk maps (Mf_q, Mb_q, H_q) over q -> the
//             true inflows (yin_q, zin_q) and, cyclic, Navon's / Sherman–
//             Morrison's pair x_l.
//   P2(g, q)  forward sweep from yin_q, back substitution from zin_q with the
//             tile in registers, cyclic correction x - Z x_l (eq:solve), x
//             stored in place.  Its f re-read hits the L2 that P1(g) filled:
//             P2(g) is scheduled D groups after P1(g), D sized so the lag
//             window of f fits in L2 -> HBM traffic = read f once + write x once.
//
// Work order.  Items are numbered in one global order: for s = 0, 1, ...:
// the nq P1 tiles of group s, then the nq P2 tiles of group s - D.  Claims of
// NC consecutive items (one per consumer warp) are dealt round-robin to the
// CTAs (claim c -> CTA c mod grid), and every CTA, warp and scan team works
// through its share in that order.  The launch is cooperative, so all CTAs are
// co-resident, and the earliest incomplete item never waits on anything later
// (P1 waits on nothing; P2(g) waits only on the scan of g, whose P1 tiles all
// precede it and whose scan team -- groups dealt round-robin, in order --
// waits only on earlier groups' P1 tiles) -> no deadlock.  (A dynamic ticket
// gives the same guarantee without co-residency, but 16 K same-address
// atomics per solve serialise at ~45 ns each on B200: measured 759 us.)
//
// Per CTA: 1 producer warp (claims, flags, TMA), NC consumer warps, NSW scan
// warps.  Ring of NS slots (NS a multiple of NC): local item j goes to warp
// j % NC and slot j % NS, so every slot is owned by ONE consumer warp and a
// parity wait can never alias an older phase.  A slot holds the tile (TMA
// 3-D/2-D box), the chunk's coefficient rows (1-D bulk copy; L2-resident),
// and for P2 the tile's inflows and x_l (1-D bulk copies, issued after the
// producer has acquired the group's scan flag).
//
// Tables (built once per LHS by fs_tables_kernel, fp64 maths rounded to T):
//   rec[r]  = (F0, F1, F2, Wa, Wb, 0)        per row (P1)
//   coef[r] = band_core layout (F0 F1 F2 - B1 B2 Z1 Z2) (P2)
//   ct[q]   = (Mf_q, Mb_q, H_q) row-major 2x2 each
//   rsp[j]  = response of g on cyclic row srow[j] to its chunk's forward inflow
#pragma once
#include <cuda.h>

#include "band_core.cuh"
#include "common.cuh"

namespace pb {
namespace fs {

constexpr int Q = 64;    // rows per chunk (tile height)
constexpr int TW = 32;   // systems per tile (lanes)
constexpr int REC = 6;   // P1 row record length
constexpr int NC = 4;    // consumer warps (= items per claim)
constexpr int NSW = 3;   // scan warps (1 + NC + NSW = 8 warps: the full 255-register budget)
constexpr int NTHREADS = 32 * (NC + 1 + NSW);

// what the tile holds on arrival:
//   MODE_SOLVE  the right-hand side f (pent_solve / tri_solve / the ADI y-sweep)
//   MODE_CH1D   the 1D Cahn–Hilliard level C^n; f is formed on chip from the
//               tile and its two halo rows (eq6:1Dnumerical):
//               f_i = C_i + alpha (N_{i-1} - 2 N_i + N_{i+1}), N = C^3 - C
//               (the +C_i^n term of reading r12), and x = C^{n+1} goes to xout
constexpr int MODE_SOLVE = 0, MODE_CH1D = 1;
template <typename T>
constexpr int sbatch() { return 8; }   // scan records per register batch

template <typename T>
struct Cfg {
    static constexpr int TILE = Q * TW;             // elements
    static constexpr int COEF = Q * COEF_STRIDE;    // >= Q * REC
    static constexpr int INF = TW * 4;              // (yin, zin) blocks of the tile's 32 systems
    static constexpr int XL = TW * 2;
    static constexpr int HALO = TW * 2;             // MODE_CH1D: rows r0 - 1 and r0 + kmax (periodic)
    // (a multiple of 1 KB: every slot's tile must keep the 128B swizzle alignment)
    static constexpr int SLOT = (TILE + COEF + INF + XL + HALO + 1024 / (int)sizeof(T) - 1) / (1024 / (int)sizeof(T)) *
                                (1024 / (int)sizeof(T));
    static constexpr int NS = sizeof(T) == 8 ? 8 : 16;
    static_assert(NS % NC == 0, "ring slots must be a multiple of the consumer warps");
};

template <typename T>
struct Args {
    const T *rec, *coef, *ct, *rsp;
    const double *scal;
    T *car;             // chunk records [q][half][sys][2]: half 0 = yF (-> yin), half 1 = zB (-> zin)
    T *spec;            // [sys][4] zero-inflow g on the cyclic rows
    T *xl;              // [sys][2]
    T *x;               // the right-hand sides (MODE_SOLVE: solved in place; MODE_CH1D: C^n)
    T *xout;            // where P2 writes x (== x for MODE_SOLVE; C^{n+1} for MODE_CH1D)
    T alpha;            // MODE_CH1D: dt / dx^2
    int64_t bstride;    // elements between batches
    int64_t pitch;      // interleaved: elements between rows (>= M); contiguous: between systems (>= n)
    unsigned *cnt;      // [G] P1 tiles done, cumulative over launches (== epoch * nq when complete)
    unsigned *flag;     // [G] == this launch's epoch once the group is scanned
    unsigned *tick;     // [2] CTAs done (reset by the last CTA), [3] launches completed: this
                        // launch's epoch is tick[3] + 1 (kept on the device, so a solve captured
                        // in a CUDA graph is correct on every replay)
    int64_t n, M, nsys; // rows, systems per batch, padded systems over all batches (= 32 G)
    int64_t items, nclaims;
    int64_t srow[4];
    int nq, count, Gb, G, D;
    int qspec;          // first chunk holding a cyclic row (cyclic only)
    int flat;           // one 2-D map over all batches: interleaved (M, n*count), row b*n + r (n % Q == 0);
                        // contiguous (n, M*count), system b*M + s (M % 32 == 0)
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void lds2(const double *p, double &a, double &b)
{
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b) : "r"(su32(p)));
}
__device__ __forceinline__ void lds2(const float *p, float &a, float &b)
{
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(a), "=f"(b) : "r"(su32(p)));
}
__device__ __forceinline__ void bar_init(uint64_t *b, int cnt)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void bar_expect_tx(uint64_t *b, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t *b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t *b, uint32_t parity)
{
    asm volatile(
        "{\n .reg .pred p;\n"
        "FS_WAIT:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra FS_WAIT;\n}" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void tma_load3(void *dst, const CUtensorMap *m, int c0, int c1, int c2, uint64_t *bar,
                                          uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(su32(dst)),
        "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(su32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void tma_load2(void *dst, const CUtensorMap *m, int c0, int c1, uint64_t *bar, uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(su32(dst)),
        "l"(m), "r"(c0), "r"(c1), "r"(su32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void tma_store2(const CUtensorMap *m, int c0, int c1, const void *src)
{
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(m), "r"(c0), "r"(c1),
                 "r"(su32(src))
                 : "memory");
}
__device__ __forceinline__ void tma_store3(const CUtensorMap *m, int c0, int c1, int c2, const void *src)
{
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(m), "r"(c0),
                 "r"(c1), "r"(c2), "r"(su32(src))
                 : "memory");
}
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned *p, unsigned v)
{
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acquire() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void scan_bar() { asm volatile("bar.sync 1, %0;" ::"n"(32 * NSW) : "memory"); }
__device__ __forceinline__ uint32_t up16(uint32_t b) { return (b + 15u) & ~15u; }

// global item i -> (P2?, group, chunk); see the work order above
struct Item {
    int p2, g, q;
};
__device__ __forceinline__ Item decode(int64_t i, int nq, int G, int D)
{
    Item it;
    const int64_t a = (int64_t)D * nq;                  // phase A: P1 of groups 0 .. D-1
    const int64_t b = a + (int64_t)(G - D) * 2 * nq;    // phase B: (P1 of s, P2 of s - D), s = D .. G-1
    if (i < a) {
        it.p2 = 0;
        it.g = (int)(i / nq);
        it.q = (int)(i - (int64_t)it.g * nq);
    } else if (i < b) {
        const int64_t k = i - a, s = k / (2 * nq);
        const int r = (int)(k - s * 2 * nq);
        it.p2 = r >= nq;
        it.g = (int)(it.p2 ? s : s + D);
        it.q = it.p2 ? r - nq : r;
    } else {                                            // phase C: P2 of groups G-D .. G-1
        const int64_t k = i - b, s = k / nq;
        it.p2 = 1;
        it.g = (int)(G - D + s);
        it.q = (int)(k - s * nq);
    }
    return it;
}

// chunk record (q, sys): half 0 = (yF0, yF1) / (yin0, yin1), half 1 = (zB0, zB1)
// / (zin0, zin1); the 32 systems of a group are contiguous per (q, half)
__device__ __forceinline__ int64_t rec_off(int64_t q, int half, int64_t sys, int64_t nsys)
{
    return ((2 * q + half) * nsys + sys) * 2;
}

// ---------------------------------------------------------------- tile layouts in the slot
// LAY_INTER  (interleaved rhs, x[i*M + s]): the TMA box (32 systems, 64 rows)
//            lands as [row][lane] -> element (k, lane) at k*TW + lane.
// LAY_CONTIG (contiguous rhs, x[s*n + i]; the ADI x-sweep): the tile is EB =
//            128/sizeof(T) rows x 32 systems per TMA box (Q/EB boxes), box
//            rows = systems, 128B-swizzled: the 16-byte unit u of system s is
//            stored at unit u ^ (s & 7), so the 32 lanes reading the same row k
//            of their own system hit 8 distinct unit groups per 8 lanes
//            (conflict-free 16-byte reads, 4 wavefronts per warp).
constexpr int LAY_INTER = 0, LAY_CONTIG = 1;

template <typename T>
struct Sw {
    static constexpr int EB = 128 / (int)sizeof(T);   // rows per box (one 128-byte box row per system)
    static constexpr int EU = 16 / (int)sizeof(T);    // elements per 16-byte unit
};
// element offset of (row k, system lane) in a LAY_CONTIG tile
template <typename T>
__device__ __forceinline__ int csw(int k, int lane)
{
    constexpr int EB = Sw<T>::EB, EU = Sw<T>::EU;
    const int b = k / EB, kk = k % EB;
    return b * (TW * EB) + lane * EB + (((kk / EU) ^ (lane & 7)) * EU) + kk % EU;
}
template <typename T, int LAY>
__device__ __forceinline__ T tld(const T *d, int k, int lane)
{
    return LAY == LAY_INTER ? d[k * TW + lane] : d[csw<T>(k, lane)];
}
template <typename T, int LAY>
__device__ __forceinline__ void tst(T *d, int k, int lane, T v)
{
    if (LAY == LAY_INTER) d[k * TW + lane] = v;
    else d[csw<T>(k, lane)] = v;
}

// ---------------------------------------------------------------- tile kernels (one warp)
// P1: zero-inflow forward sweep, carry and back-substitution functional.
// FULL: kmax == Q (no row guards); SPEC: the tile holds cyclic rows (ks[j] =
// row srow[j] - r0 inside the tile, else -1)
template <typename T, int K, bool SPEC, bool FULL, int LAY>
__device__ __forceinline__ void tile_carry(const T *d, const T *c, int kmax, int lane, const int (&ks)[4],
                                           const Args<T> &A, int64_t sys, bool ok, int q)
{
    T y0 = T(0), y1 = T(0), a0 = T(0), a1 = T(0);
#pragma unroll(FULL ? Q : 4)
    for (int k = 0; k < (FULL ? Q : kmax); ++k) {
        T f0, f1, f2, wa, wb, wz;
        lds2(c + k * REC, f0, f1);
        lds2(c + k * REC + 2, f2, wa);
        lds2(c + k * REC + 4, wb, wz);
        T t = f0 * tld<T, LAY>(d, k, lane);
        if (K == 2) t -= f2 * y0;
        const T g = t - f1 * y1;
        y0 = y1;
        y1 = g;
        a0 += wa * g;
        a1 += wb * g;
        if (SPEC) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (ok && ks[j] == k) A.spec[sys * 4 + j] = g;
        }
    }
    if (ok) {
        T *o = A.car + rec_off(q, 0, sys, A.nsys);
        T *o2 = A.car + rec_off(q, 1, sys, A.nsys);
        o[0] = y0;
        o[1] = y1;
        o2[0] = a0;
        o2[1] = a1;
    }
}

// P2: forward sweep from (y0, y1), back substitution from (z0, z1), cyclic
// correction x - Z x_l, on the tile column in registers.  FULL: kmax == Q.
template <typename T, int K, bool PER, bool FULL>
__device__ __forceinline__ void tile_solve(T (&v)[Q], const T *c, int kmax, T y0, T y1, T z0, T z1, T xl0, T xl1)
{
    // each recurrence takes its newest carry last: one dependent FMA per row
    // on the critical path (g = (F0 f - F2 g_{k-2}) - F1 g_{k-1}; likewise x)
#pragma unroll
    for (int k = 0; k < Q; ++k) {
        if (FULL || k < kmax) {
            T f0, f1, f2, fz;
            lds2(c + k * COEF_STRIDE, f0, f1);
            lds2(c + k * COEF_STRIDE + 2, f2, fz);
            T t = f0 * v[k];
            if (K == 2) t -= f2 * y0;
            const T g = t - f1 * y1;
            y0 = y1;
            y1 = g;
            v[k] = g;
        }
    }
#pragma unroll
    for (int k = Q - 1; k >= 0; --k) {
        if (FULL || k < kmax) {
            T b1, b2;
            lds2(c + k * COEF_STRIDE + 4, b1, b2);
            T t = v[k];
            if (K == 2) t -= b2 * z1;
            const T xx = t - b1 * z0;
            z1 = z0;
            z0 = xx;
            v[k] = xx;
        }
    }
    if (PER) {
        // cyclic correction x - Z x_l (Navon eq:solve / Sherman–Morrison)
#pragma unroll
        for (int k = 0; k < Q; ++k) {
            T z1v, z2v;
            lds2(c + k * COEF_STRIDE + 6, z1v, z2v);
            T o = v[k] - z1v * xl0;
            if (K == 2) o -= z2v * xl1;
            v[k] = o;
        }
    }
}

// ---------------------------------------------------------------- scan of one group (NSW warps)
template <typename T>
__device__ __forceinline__ void mv(const T *m, T x0, T x1, T &r0, T &r1)
{
    r0 = m[0] * x0 + m[1] * x1;
    r1 = m[2] * x0 + m[3] * x1;
}
template <typename T>
__device__ __forceinline__ void mmul(const T *a, const T *b, T *r)   // r = a b (may alias)
{
    const T r0 = a[0] * b[0] + a[1] * b[2], r1 = a[0] * b[1] + a[1] * b[3];
    const T r2 = a[2] * b[0] + a[3] * b[2], r3 = a[2] * b[1] + a[3] * b[3];
    r[0] = r0, r[1] = r1, r[2] = r2, r[3] = r3;
}
template <typename T>
__device__ __forceinline__ void ldm4(const T *p, T *m)
{
    m[0] = __ldg(p), m[1] = __ldg(p + 1), m[2] = __ldg(p + 2), m[3] = __ldg(p + 3);
}
template <typename T>
__device__ __forceinline__ void ld_pair(const T *p, T &a, T &b)
{
    if (sizeof(T) == 8) {
        const double2 u = __ldcg(reinterpret_cast<const double2 *>(p));
        a = (T)u.x, b = (T)u.y;
    } else {
        const float2 u = __ldcg(reinterpret_cast<const float2 *>(p));
        a = (T)u.x, b = (T)u.y;
    }
}
template <typename T>
__device__ __forceinline__ void st_pair(T *p, T a, T b)
{
    if (sizeof(T) == 8) __stcg(reinterpret_cast<double2 *>(p), make_double2((double)a, (double)b));
    else __stcg(reinterpret_cast<float2 *>(p), make_float2((float)a, (float)b));
}
// record (q, sys) -> r[0..3] = (half 0, half 1)
template <typename T>
__device__ __forceinline__ void ld_rec(const Args<T> &A, int64_t q, int64_t sys, T *r)
{
    ld_pair(A.car + rec_off(q, 0, sys, A.nsys), r[0], r[1]);
    ld_pair(A.car + rec_off(q, 1, sys, A.nsys), r[2], r[3]);
}
template <typename T>
__device__ __forceinline__ void st_rec(const Args<T> &A, int64_t q, int64_t sys, const T *r)
{
    st_pair(A.car + rec_off(q, 0, sys, A.nsys), r[0], r[1]);
    st_pair(A.car + rec_off(q, 1, sys, A.nsys), r[2], r[3]);
}

template <typename T>
struct ScanSmem {
    T agg[NSW][TW][2];
    T pm[NSW][4];
    T gsp[4][TW];
    int grp;
};

// The team's NSW warps split the group's chunks into NSW segments: fold each
// segment (forward affine maps), combine the segment maps through shared
// memory, walk the segment writing yin_q and c_q = zB_q + H_q yin_q; then the
// same backward with Mb over c_q -> zin_q.  Records stay in place:
// (yF, zB) -> (yin, zin).  Cyclic: warp 0 evaluates x_l.
template <typename T, int K, bool PER>
__device__ void scan_group(const Args<T> &A, ScanSmem<T> &S, int g, int sw, int lane)
{
    const int64_t sys = (int64_t)g * TW + lane;
    const int nq = A.nq, cps = (nq + NSW - 1) / NSW;
    const int qa = min(nq, sw * cps), qe = min(nq, qa + cps);
    constexpr int SB = sbatch<T>();

    // ---- forward fold of my segment: a = (Mf a + yF) over q, P = prod Mf
    T P[4] = {T(1), T(0), T(0), T(1)}, a0 = T(0), a1 = T(0);
    for (int q0 = qa; q0 < qe; q0 += SB) {
        T R[SB][4];
#pragma unroll
        for (int i = 0; i < SB; ++i)
            if (q0 + i < qe) ld_rec(A, q0 + i, sys, R[i]);
#pragma unroll
        for (int i = 0; i < SB; ++i)
            if (q0 + i < qe) {
                T m[4], t0, t1;
                ldm4(A.ct + (int64_t)(q0 + i) * 12, m);
                mv(m, a0, a1, t0, t1);
                a0 = t0 + R[i][0];
                a1 = t1 + R[i][1];
                mmul(m, P, P);
            }
    }
    S.agg[sw][lane][0] = a0;
    S.agg[sw][lane][1] = a1;
    if (lane == 0)
        for (int e = 0; e < 4; ++e) S.pm[sw][e] = P[e];
    scan_bar();
    T y0 = T(0), y1 = T(0);
    for (int v = 0; v < sw; ++v) {
        T t0, t1;
        mv(S.pm[v], y0, y1, t0, t1);
        y0 = t0 + S.agg[v][lane][0];
        y1 = t1 + S.agg[v][lane][1];
    }
    // ---- forward walk: yin_q replaces yF_q, c_q = zB_q + H_q yin_q replaces zB_q
    for (int q0 = qa; q0 < qe; q0 += SB) {
        T R[SB][4];
#pragma unroll
        for (int i = 0; i < SB; ++i)
            if (q0 + i < qe) ld_rec(A, q0 + i, sys, R[i]);
#pragma unroll
        for (int i = 0; i < SB; ++i)
            if (q0 + i < qe) {
                const int q = q0 + i;
                T m[4], h[4], t0, t1;
                ldm4(A.ct + (int64_t)q * 12, m);
                ldm4(A.ct + (int64_t)q * 12 + 8, h);
                const T yf0 = R[i][0], yf1 = R[i][1];
                mv(h, y0, y1, t0, t1);
                R[i][0] = y0;
                R[i][1] = y1;
                R[i][2] += t0;
                R[i][3] += t1;
                if (PER && q >= A.qspec) {
#pragma unroll
                    for (int jx = 0; jx < 4; ++jx)
                        if (A.srow[jx] >= 0 && A.srow[jx] / Q == q)
                            S.gsp[jx][lane] = __ldcg(A.spec + sys * 4 + jx) + A.rsp[jx * 2] * y0 + A.rsp[jx * 2 + 1] * y1;
                }
                mv(m, y0, y1, t0, t1);
                y0 = t0 + yf0;
                y1 = t1 + yf1;
                st_rec(A, q, sys, R[i]);
            }
    }
    // ---- backward fold of my segment (high to low): c = Mb c + c_q, Pb = prod Mb
    T Pb[4] = {T(1), T(0), T(0), T(1)}, c0 = T(0), c1 = T(0);
    for (int q1 = qe; q1 > qa; q1 -= SB) {
        T R[SB][4];
#pragma unroll
        for (int i = 0; i < SB; ++i)
            if (q1 - 1 - i >= qa) ld_rec(A, q1 - 1 - i, sys, R[i]);
#pragma unroll
        for (int i = 0; i < SB; ++i)
            if (q1 - 1 - i >= qa) {
                T m[4], t0, t1;
                ldm4(A.ct + (int64_t)(q1 - 1 - i) * 12 + 4, m);
                mv(m, c0, c1, t0, t1);
                c0 = t0 + R[i][2];
                c1 = t1 + R[i][3];
                mmul(m, Pb, Pb);
            }
    }
    scan_bar();   // forward aggregates consumed
    S.agg[sw][lane][0] = c0;
    S.agg[sw][lane][1] = c1;
    if (lane == 0)
        for (int e = 0; e < 4; ++e) S.pm[sw][e] = Pb[e];
    scan_bar();
    T z0 = T(0), z1 = T(0);
    for (int v = NSW - 1; v > sw; --v) {
        T t0, t1;
        mv(S.pm[v], z0, z1, t0, t1);
        z0 = t0 + S.agg[v][lane][0];
        z1 = t1 + S.agg[v][lane][1];
    }
    for (int q1 = qe; q1 > qa; q1 -= SB) {
        T R[SB][4];
#pragma unroll
        for (int i = 0; i < SB; ++i)
            if (q1 - 1 - i >= qa) ld_rec(A, q1 - 1 - i, sys, R[i]);
#pragma unroll
        for (int i = 0; i < SB; ++i)
            if (q1 - 1 - i >= qa) {
                const int q = q1 - 1 - i;
                T m[4], t0, t1;
                ldm4(A.ct + (int64_t)q * 12 + 4, m);
                const T cq0 = R[i][2], cq1 = R[i][3];
                R[i][2] = z0;
                R[i][3] = z1;
                mv(m, z0, z1, t0, t1);
                z0 = t0 + cq0;
                z1 = t1 + cq1;
                st_rec(A, q, sys, R[i]);
            }
    }
    if (PER && sw == 0) {
        // (x_0, x_1) of the non-cyclic solution = warp 0's z after its walk
        const T y1c = z0, y2c = z1;
        T gv[4];
#pragma unroll
        for (int jx = 0; jx < 4; ++jx) gv[jx] = A.srow[jx] >= 0 ? S.gsp[jx][lane] : T(0);
        const double *sc = A.scal;
        T xl0, xl1;
        if (K == 2) {
            // Navon (eq:first_two)
            const T ym1 = gv[1], ym2 = gv[0] - T(sc[10]) * gv[1];
            const T q0 = gv[2] - (T(sc[4]) * y1c + T(sc[5]) * ym2 + T(sc[6]) * ym1);
            const T q1 = gv[3] - (T(sc[7]) * y1c + T(sc[8]) * y2c + T(sc[9]) * ym1);
            xl0 = T(sc[0]) * q0 + T(sc[1]) * q1;
            xl1 = T(sc[2]) * q0 + T(sc[3]) * q1;
        } else {
            // Sherman–Morrison
            xl0 = (y1c + T(sc[0]) * gv[0]) / T(sc[1]);
            xl1 = T(0);
        }
        __stcg(A.xl + sys * 2 + 0, xl0);
        __stcg(A.xl + sys * 2 + 1, xl1);
    }
}

// ---------------------------------------------------------------- the kernel
template <typename T>
struct Smem {
    T slot[Cfg<T>::NS][Cfg<T>::SLOT];
    uint64_t full[Cfg<T>::NS], empty[Cfg<T>::NS];
    int64_t item[Cfg<T>::NS];   // global item of the slot; -1 exit, -2 empty (past the end)
    ScanSmem<T> scan;
};

// f of the 1D CH step, in place over the warp's own tile column (lane-private)
template <typename T>
__device__ __forceinline__ void ch1d_rhs(T *du, const T *halo, int kmax, int lane, T alpha)
{
    T um = halo[lane];
    T nm = um * um * um - um;
    T u0 = du[lane];
    T n0 = u0 * u0 * u0 - u0;
#pragma unroll 4
    for (int k = 0; k < kmax; ++k) {
        const T u1 = (k + 1 < kmax) ? du[(k + 1) * TW + lane] : halo[TW + lane];
        const T n1 = u1 * u1 * u1 - u1;
        du[k * TW + lane] = u0 + alpha * (nm - T(2) * n0 + n1);
        nm = n0;
        n0 = n1;
        u0 = u1;
    }
}

template <typename T, int K, bool PER, int MODE, int LAY>
__global__ void __launch_bounds__(NTHREADS, 1) fs_kernel(const __grid_constant__ CUtensorMap tmap, const Args<T> A)
{
    constexpr int NS = Cfg<T>::NS, TILE = Cfg<T>::TILE;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // 1024-byte aligned: the 128B swizzle pattern of LAY_CONTIG tiles repeats per 1 KB
    Smem<T> &sm = *reinterpret_cast<Smem<T> *>((((uintptr_t)smem_raw) + 1023) & ~(uintptr_t)1023);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) {
            bar_init(&sm.full[i], 1);
            bar_init(&sm.empty[i], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == NC) {
        // ---------------- producer: claim NC items at a time, one per consumer warp
        if (lane == 0) {
            const unsigned epoch = ld_relaxed(A.tick + 3) + 1u;
            const uint64_t pol1 = policy_evict_last(), pol2 = policy_evict_first();
            for (int64_t k = 0;; ++k) {
                const int64_t c = blockIdx.x + k * gridDim.x;   // this CTA's k-th claim (static)
                const bool done = c >= A.nclaims;
                Item it[NC];
                unsigned fl[NC];
#pragma unroll
                for (int w = 0; w < NC; ++w) {
                    const int64_t i = c * NC + w;
                    const bool live = !done && i < A.items;
                    it[w] = live ? decode(i, A.nq, A.G, A.D) : Item{0, 0, 0};
                    fl[w] = (live && it[w].p2) ? ld_relaxed(A.flag + it[w].g) : epoch;
                }
#pragma unroll
                for (int w = 0; w < NC; ++w) {
                    const int64_t j = k * NC + w, i = c * NC + w;
                    const int sl = (int)(j % NS);
                    if (j >= NS) bar_wait(&sm.empty[sl], (uint32_t)(((j / NS) - 1) & 1));
                    if (done || i >= A.items) {
                        sm.item[sl] = done ? -1 : -2;
                        bar_arrive(&sm.full[sl]);
                        continue;
                    }
                    const Item id = it[w];
                    if (id.p2) {
                        // the group's scan must be complete before its inflows are copied
                        if (fl[w] != epoch)
                            while (ld_acquire(A.flag + id.g) != epoch) __nanosleep(64);
                        fence_acquire();
                        fence_proxy_global();
                    }
                    sm.item[sl] = i;
                    const int b = id.g / A.Gb, gl = id.g - b * A.Gb;
                    const int64_t r0 = (int64_t)id.q * Q;
                    const int kmax = (int)min((int64_t)Q, A.n - r0);
                    T *slot = sm.slot[sl];
                    const uint32_t cb = up16((uint32_t)(kmax * (id.p2 ? COEF_STRIDE : REC) * sizeof(T)));
                    uint32_t bytes = TILE * sizeof(T) + cb;
                    if (id.p2) bytes += (Cfg<T>::INF + (PER ? Cfg<T>::XL : 0)) * sizeof(T);
                    if (MODE == MODE_CH1D) bytes += Cfg<T>::HALO * sizeof(T);
                    bar_expect_tx(&sm.full[sl], bytes);
                    const uint64_t pol = id.p2 ? pol2 : pol1;
                    if (LAY == LAY_CONTIG) {
                        // Q / EB boxes of (EB rows x 32 systems), 128B-swizzled
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
                    bulk_load(slot + TILE, id.p2 ? A.coef + r0 * COEF_STRIDE : A.rec + r0 * REC, cb, &sm.full[sl]);
                    if (MODE == MODE_CH1D) {
                        // the tile's periodic halo rows (32 contiguous systems each)
                        const T *ub = A.x + (int64_t)b * A.bstride + (int64_t)gl * TW;
                        const int64_t rlo = r0 == 0 ? A.n - 1 : r0 - 1, rhi = r0 + kmax == A.n ? 0 : r0 + kmax;
                        T *hs = slot + TILE + Cfg<T>::COEF + Cfg<T>::INF + Cfg<T>::XL;
                        bulk_load(hs, ub + rlo * A.pitch, TW * sizeof(T), &sm.full[sl]);
                        bulk_load(hs + TW, ub + rhi * A.pitch, TW * sizeof(T), &sm.full[sl]);
                    }
                    if (id.p2) {
                        T *ia = slot + TILE + Cfg<T>::COEF;
                        const int64_t s0 = (int64_t)id.g * TW;
                        constexpr uint32_t BB = 2 * TW * sizeof(T);   // one (q, half) block of the group
                        bulk_load(ia, A.car + rec_off(id.q, 0, s0, A.nsys), BB, &sm.full[sl]);
                        bulk_load(ia + 2 * TW, A.car + rec_off(id.q, 1, s0, A.nsys), BB, &sm.full[sl]);
                        if (PER)
                            bulk_load(slot + TILE + Cfg<T>::COEF + Cfg<T>::INF, A.xl + s0 * 2, Cfg<T>::XL * sizeof(T),
                                      &sm.full[sl]);
                    }
                }
                if (done) break;
            }
        }
    } else if (warp < NC) {
        // ---------------- consumers: local items j = warp, warp + NC, ... (slot j % NS, owned by this warp)
        for (int64_t j = warp;; j += NC) {
            const int sl = (int)(j % NS);
            bar_wait(&sm.full[sl], (uint32_t)((j / NS) & 1));
            const int64_t i = *(volatile int64_t *)&sm.item[sl];
            if (i == -1) {
                if (LAY == LAY_CONTIG && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
                break;
            }
            if (i < 0) {
                __syncwarp();
                if (lane == 0) bar_arrive(&sm.empty[sl]);
                continue;
            }
            const Item id = decode(i, A.nq, A.G, A.D);
            const int b = id.g / A.Gb, gl = id.g - b * A.Gb;
            const int64_t r0 = (int64_t)id.q * Q;
            const int kmax = (int)min((int64_t)Q, A.n - r0);
            const T *d = sm.slot[sl];
            const T *c = d + TILE;
            const int64_t s_in_batch = (int64_t)gl * TW + lane;
            const bool ok = s_in_batch < A.M;
            const int64_t sys = (int64_t)id.g * TW + lane;
            if (MODE == MODE_CH1D)
                ch1d_rhs<T>(const_cast<T *>(d), d + TILE + Cfg<T>::COEF + Cfg<T>::INF + Cfg<T>::XL, kmax, lane, A.alpha);
            if (!id.p2) {
                if (PER && id.q >= A.qspec) {
                    int ks[4];
#pragma unroll
                    for (int jx = 0; jx < 4; ++jx) {
                        const int64_t rr = A.srow[jx] - r0;
                        ks[jx] = (A.srow[jx] >= 0 && rr >= 0 && rr < Q) ? (int)rr : -1;
                    }
                    tile_carry<T, K, true, false, LAY>(d, c, kmax, lane, ks, A, sys, ok, id.q);
                } else {
                    const int ks[4] = {-1, -1, -1, -1};
                    if (kmax == Q) tile_carry<T, K, false, true, LAY>(d, c, Q, lane, ks, A, sys, ok, id.q);
                    else tile_carry<T, K, false, false, LAY>(d, c, kmax, lane, ks, A, sys, ok, id.q);
                }
                __syncwarp();
                if (lane == 0) bar_arrive(&sm.empty[sl]);
                // publish: this tile's records (and cyclic g values) -> the group's counter
                __threadfence();
                __syncwarp();
                if (lane == 0) atomicAdd(A.cnt + id.g, 1u);
                continue;
            }
            // P2: the column, inflows and x_l into registers
            T v[Q];
#pragma unroll
            for (int k = 0; k < Q; ++k) v[k] = tld<T, LAY>(d, k, lane);
            const T *inf = c + Cfg<T>::COEF;
            T y0, y1, z0, z1, xl0 = T(0), xl1 = T(0);
            lds2(inf + lane * 2, y0, y1);
            lds2(inf + 2 * TW + lane * 2, z0, z1);
            if (PER) lds2(inf + Cfg<T>::INF + lane * 2, xl0, xl1);
            if (kmax == Q) tile_solve<T, K, PER, true>(v, c, Q, y0, y1, z0, z1, xl0, xl1);
            else tile_solve<T, K, PER, false>(v, c, kmax, y0, y1, z0, z1, xl0, xl1);
            if (PER && K == 2 && r0 + Q > A.n - 2) {
                // Navon: the last two unknowns are x_l itself
                const int k2 = (int)(A.n - 2 - r0);
#pragma unroll
                for (int k = 0; k < Q; ++k) {
                    if (k == k2) v[k] = xl0;
                    if (k == k2 + 1) v[k] = xl1;
                }
            }
            if (LAY == LAY_CONTIG) {
                // x back into the slot (same swizzle) and out by TMA: systems are
                // rows of the output, so a register store would scatter 32 lines
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
                    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // slot read out: reusable
                    bar_arrive(&sm.empty[sl]);
                }
                __syncwarp();
                continue;
            }
            __syncwarp();
            if (lane == 0) bar_arrive(&sm.empty[sl]);
            if (ok) {
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
        // ---------------- scan team: groups claimed in order, each after its P1 tiles
        const int sw = warp - NC - 1;
        const unsigned epoch = ld_relaxed(A.tick + 3) + 1u;
        const unsigned need = epoch * (unsigned)A.nq;
        for (int g = blockIdx.x; g < A.G; g += gridDim.x) {   // groups in order (static)
            while (ld_acquire(A.cnt + g) != need) __nanosleep(128);
            scan_group<T, K, PER>(A, sm.scan, g, sw, lane);
            __threadfence();
            fence_proxy_global();
            scan_bar();   // all records / x_l of the group written
            if (sw == 0 && lane == 0) st_release(A.flag + g, epoch);
        }
    }
    // the last CTA out resets the tickets for the next launch (stream-ordered)
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(A.tick + 2, 1u) == gridDim.x - 1) {
            A.tick[2] = 0u;
            A.tick[3] = A.tick[3] + 1u;   // every CTA has read this launch's epoch
            __threadfence();
        }
    }
}

}  // namespace fs
}  // namespace pb

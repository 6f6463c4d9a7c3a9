// twopass.cuh — the streaming two-pass shared-LHS solve (interleaved layout).
//
// The thesis solves one system per thread over all N rows (P:1712-1724,
// P:1729); at N = M = 8192 that is a dependent chain of 16 K rows per thread
// and < 2 warps per SM.  Here every system is split into chunks of Q = 64 rows
// and one warp owns one TILE = (chunk q, 32 consecutive systems): lane = system,
// so every row of the tile is one contiguous 256 B (fp64) / 128 B (fp32)
// segment of the interleaved array and every coefficient load is a
// warp-uniform shared-memory broadcast.
//
//   pass 1 (tp_pass_kernel<P2 = false>): forward sweep of the tile with zero
//       inflow -> forward carry yF = (g_{r1-2}, g_{r1-1}); the back-substitution
//       carry of the chunk with zero inflow is a linear functional of g
//       (zB = sum_k W_k g_k, W_k from the factor), accumulated on the fly, so
//       pass 1 holds nothing and reads f once.
//   scan  (tp_scan_kernel): one warp per system composes the affine chunk maps
//       (Mf_q, Mb_q, H_q) with a Kogge–Stone scan over lanes -> the true forward
//       inflow yin_q and backward inflow zin_q of every chunk, and (cyclic) the
//       Navon / Sherman–Morrison pair x_l.
//   pass 2 (tp_pass_kernel<P2 = true>): forward sweep from yin_q, back
//       substitution from zin_q with the tile column in registers, cyclic
//       correction x - Z x_l, TMA store.  The launcher slabs the systems so its
//       f re-read hits the L2 that pass 1 filled.
//
// Both passes are persistent, warp-specialised TMA rings (one producer warp,
// NWC consumer warps, NS slots of one tile each): register-burst LDG loading
// of the same strips tops out at 3-4 TB/s on B200, a TMA ring at 5.6-6.3 TB/s
// (DESIGN.md §6.1).  Each slot also receives, by 1-D bulk copy, the chunk's
// coefficient rows and (pass 2) the tile's inflows and x_l.
//
// Tables (built once per LHS by tp_tables_kernel, fp64 maths rounded to T):
//   rec[r]  = (F0, F1, F2, Wa, Wb, 0)        per row (pass 1)
//   coef[r] = band_core layout (F0 F1 F2 - B1 B2 Z1 Z2) (pass 2)
//   ct[q]   = (Mf_q, Mb_q, H_q) row-major 2x2 each
//   rsp[j]  = response of g on cyclic row srow[j] to its chunk's forward inflow
#pragma once
#include <cuda.h>

#include "band_core.cuh"
#include "common.cuh"

namespace pb {
namespace tp {

constexpr int Q = 64;       // rows per chunk (tile height)
constexpr int TW = 32;      // systems per tile (lanes)
constexpr int REC = 6;      // pass-1 row record length
constexpr int NWC = 4;      // consumer warps per CTA, pass 2
#ifndef TP_NWC1
#define TP_NWC1 4
#endif
constexpr int NWC1 = TP_NWC1;   // consumer warps per CTA, pass 1
template <bool P2>
__host__ __device__ constexpr int nwc() { return P2 ? NWC : NWC1; }

template <typename T>
struct Cfg {
    static constexpr int TILE = Q * TW;                                   // elements
    static constexpr int SLOT1 = TILE + Q * REC;                          // pass-1 slot (elements)
    static constexpr int SLOT2 = TILE + Q * COEF_STRIDE;                  // pass-2 slot
    static constexpr int NS1 = (int)((220 * 1024) / (SLOT1 * sizeof(T)));
    static constexpr int NS2 = (int)((220 * 1024 - NWC * TILE * sizeof(T)) / (SLOT2 * sizeof(T)));
};

template <typename T>
struct Args {
    const T *rec, *coef, *ct, *rsp;
    const double *scal;
    // per-launch scratch; sys = batch * msp + (s - s0), msp = ms rounded up to TW
    // (so every tile's records start 16-byte aligned for the bulk copies)
    T *car;                  // [q][sys][4]: pass 1 (yF, zB) -> scan (yin, zin)
    T *spec;                 // [sys][4] zero-inflow g on the cyclic rows
    T *xl;                   // [sys][2]
    int64_t n, M;            // rows, systems per batch
    int64_t s0, ms, msp;     // systems [s0, s0 + ms) of each batch in this launch
    int64_t srow[4];
    int nq, count, G;        // chunks, batches, tiles across ms
    int qspec;               // first chunk holding a cyclic row (cyclic only)
    int keep;                // pass 1 loads with L2 evict_last (the slab fits in L2)
    int flat;                // batches contiguous and n % Q == 0: 2-D maps, row = b * n + r
    int p2g;                 // coefficient rows per stage: 0 = 1-D bulk copy, 2 = 2-D tensor load
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
        "TP_WAIT:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra TP_WAIT;\n}" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void tma_load(void *dst, const CUtensorMap *m, int c0, int c1, int c2, uint64_t *bar,
                                         uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(su32(dst)),
        "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(su32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void tma_load(void *dst, const CUtensorMap *m, int c0, int c1, int c2, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(su32(dst)),
        "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(su32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load2(void *dst, const CUtensorMap *m, int c0, int c1, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(su32(dst)),
        "l"(m), "r"(c0), "r"(c1), "r"(su32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store2(const CUtensorMap *m, int c0, int c1, const void *src)
{
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(m), "r"(c0), "r"(c1),
                 "r"(su32(src))
                 : "memory");
}
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ void tma_store(const CUtensorMap *m, int c0, int c1, int c2, const void *src)
{
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(m), "r"(c0),
                 "r"(c1), "r"(c2), "r"(su32(src))
                 : "memory");
}
__device__ __forceinline__ uint32_t up16(uint32_t b) { return (b + 15u) & ~15u; }
// programmatic dependent launch: the three kernels of a solve are launched with
// programmatic stream serialization; each waits for its predecessor's memory
// before touching shared data and lets its successor launch right away (the
// successor's CTAs cannot be resident until this grid's CTAs leave anyway)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

struct TileId {
    int q, b, g;
};
__device__ __forceinline__ TileId tile_of(int64_t t, int G, int count)
{
    TileId r;
    const int64_t per_q = (int64_t)G * count;
    r.q = (int)(t / per_q);
    const int64_t rem = t - (int64_t)r.q * per_q;
    r.b = (int)(rem / G);
    r.g = (int)(rem - (int64_t)r.b * G);
    return r;
}

// ---------------------------------------------------------------- passes
template <typename T, bool P2>
struct PassSmem {
    static constexpr int SLOT = P2 ? Cfg<T>::SLOT2 : Cfg<T>::SLOT1;
    static constexpr int NS = P2 ? Cfg<T>::NS2 : Cfg<T>::NS1;
    T slot[NS][SLOT];
    T out[P2 ? NWC : 1][P2 ? Cfg<T>::TILE : 2];           // pass 2: per-warp TMA store staging
    uint64_t full[NS], empty[NS];
};

// pass-1 tile: zero-inflow forward sweep, carry and back-substitution functional.
// FULL: kmax == Q (no row guards); SPEC: the tile holds cyclic rows (ks[j] =
// row srow[j] - r0 inside the tile, else -1)
template <typename T, int K, bool SPEC, bool FULL>
__device__ __forceinline__ void tile_carry(const T *d, const T *c, int kmax, int lane, const int (&ks)[4],
                                           const Args<T> &A, int64_t sys, bool ok, int q)
{
    T y0 = T(0), y1 = T(0), a0 = T(0), a1 = T(0);
#pragma unroll(FULL ? Q : 4)
    for (int k = 0; k < (FULL ? Q : kmax); ++k) {
        T f0, f1, f2, wa;
        lds2(c + k * REC, f0, f1);
        lds2(c + k * REC + 2, f2, wa);
        const T wb = c[k * REC + 4];
        T g = f0 * d[k * TW + lane] - f1 * y1;
        if (K == 2) g -= f2 * y0;
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
        T *o = A.car + ((int64_t)q * A.msp * A.count + sys) * 4;
        o[0] = y0;
        o[1] = y1;
        o[2] = a0;
        o[3] = a1;
    }
}

// pass-2 tile column (registers): forward sweep from (y0, y1), back
// substitution from (z0, z1), cyclic correction x - Z x_l.  FULL: kmax == Q,
// no row guards (the ragged last chunk takes the guarded copy)
template <bool GL, typename T>
__device__ __forceinline__ void cld2(const T *p, T &a, T &b)
{
    if (GL) {
        a = __ldg(p);
        b = __ldg(p + 1);
    } else {
        lds2(p, a, b);
    }
}

template <typename T, int K, bool PER, bool FULL, bool GL = false>
__device__ __forceinline__ void tile_solve(T (&v)[Q], const T *c, int kmax, T y0, T y1, T z0, T z1, T xl0, T xl1)
{
#pragma unroll
    for (int k = 0; k < Q; ++k) {
        if (FULL || k < kmax) {
            T f0, f1;
            cld2<GL>(c + k * COEF_STRIDE, f0, f1);
            T g = f0 * v[k] - f1 * y1;
            if (K == 2) g -= (GL ? __ldg(c + k * COEF_STRIDE + 2) : c[k * COEF_STRIDE + 2]) * y0;
            y0 = y1;
            y1 = g;
            v[k] = g;
        }
    }
#pragma unroll
    for (int k = Q - 1; k >= 0; --k) {
        if (FULL || k < kmax) {
            T b1, b2;
            cld2<GL>(c + k * COEF_STRIDE + 4, b1, b2);
            T xx = v[k] - b1 * z0;
            if (K == 2) xx -= b2 * z1;
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
            cld2<GL>(c + k * COEF_STRIDE + 6, z1v, z2v);
            T o = v[k] - z1v * xl0;
            if (K == 2) o -= z2v * xl1;
            v[k] = o;
        }
    }
}

// pass 2: (yin, zin) of tile t and x_l for this lane's system (plain loads)
template <typename T, bool PER>
__device__ __forceinline__ void load_inflow(const Args<T> &A, int64_t t, int lane, T (&r)[6])
{
    const TileId id = tile_of(t, A.G, A.count);
    const int64_t sys = (int64_t)id.b * A.msp + (int64_t)id.g * TW + lane;
    const T *p = A.car + ((int64_t)id.q * A.msp * A.count + sys) * 4;
    r[0] = __ldcg(p), r[1] = __ldcg(p + 1), r[2] = __ldcg(p + 2), r[3] = __ldcg(p + 3);
    r[4] = PER ? __ldcg(A.xl + sys * 2) : T(0);
    r[5] = PER ? __ldcg(A.xl + sys * 2 + 1) : T(0);
}

template <typename T, int K, bool PER, bool P2>
__global__ void __launch_bounds__(32 * (nwc<P2>() + 1), 1) tp_pass_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                     const __grid_constant__ CUtensorMap smap,
                                                                     const __grid_constant__ CUtensorMap cmap,
                                                                     const Args<T> A)
{
    using S = PassSmem<T, P2>;
    constexpr int NS = S::NS, TILE = Cfg<T>::TILE;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    S &sm = *reinterpret_cast<S *>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t ntile = (int64_t)A.nq * A.G * A.count;
    const int64_t nsys = A.msp * A.count;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) {
            bar_init(&sm.full[i], 1);
            bar_init(&sm.empty[i], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_wait();
    pdl_trigger();

    constexpr int NC = nwc<P2>();
    if (warp == NC) {
        // ---------------- producer
        if (lane != 0) return;
        // L2 hint only for pass 1 of a slabbed solve (keep the slab for pass 2).
        // Pass 2 loads carry no hint: evict_first-hinted TMA loads of the
        // tensor this kernel also TMA-stores to faulted intermittently
        // (tools/tp_stress.sh: 2 of 4 runs of 50 solves; none without the hint)
        const bool hint = !P2 && A.keep;
        const uint64_t pol = policy_evict_last();
        int j = 0;
        for (int64_t t = blockIdx.x; t < ntile; t += gridDim.x, ++j) {
            const int sl = j % NS;
            if (j >= NS) bar_wait(&sm.empty[sl], ((j / NS) - 1) & 1);
            const TileId id = tile_of(t, A.G, A.count);
            const int64_t r0 = (int64_t)id.q * Q;
            const int kmax = (int)min((int64_t)Q, A.n - r0);
            T *slot = sm.slot[sl];
            uint32_t bytes = TILE * sizeof(T);
            const uint32_t cb = up16((uint32_t)(kmax * (P2 ? COEF_STRIDE : REC) * sizeof(T)));
            bytes += A.p2g == 2 ? (uint32_t)(Q * (P2 ? COEF_STRIDE : REC) * sizeof(T)) : cb;
            const int64_t sys0 = (int64_t)id.b * A.msp + (int64_t)id.g * TW;
            const int nt = (int)min((int64_t)TW, A.ms - (int64_t)id.g * TW);
            bar_expect_tx(&sm.full[sl], bytes);
            if (A.flat)
                tma_load2(slot, &tmap, (int)(A.s0 + (int64_t)id.g * TW), (int)((int64_t)id.b * A.n + r0), &sm.full[sl]);
            else if (hint)
                tma_load(slot, &tmap, (int)(A.s0 + (int64_t)id.g * TW), (int)r0, id.b, &sm.full[sl], pol);
            else
                tma_load(slot, &tmap, (int)(A.s0 + (int64_t)id.g * TW), (int)r0, id.b, &sm.full[sl]);
            // (the tile's inflows are NOT bulk-copied in as well: a third and
            // fourth bulk copy per stage made pass 2 hang or fault
            // intermittently on B200 (tools/tp_stress2.sh); the consumers
            // prefetch them with plain loads one tile ahead instead)
            if (A.p2g == 2)   // the chunk's coefficient rows by a 2-D tensor load (row records x Q rows)
                tma_load2(slot + TILE, &cmap, 0, (int)r0, &sm.full[sl]);
            else
                bulk_load(slot + TILE, P2 ? A.coef + r0 * COEF_STRIDE : A.rec + r0 * REC, cb, &sm.full[sl]);
        }
        return;
    }

    // ---------------- consumers: warp w takes local tiles w, w + NWC, ...
    int j = warp;
    bool pend = false;
    T pf[6];   // pass 2: the next tile's (yin, zin, x_l) of this lane, loaded one tile ahead
    const int64_t tstep = (int64_t)NC * gridDim.x;
    if (P2 && blockIdx.x + (int64_t)warp * gridDim.x < ntile) load_inflow<T, PER>(A, blockIdx.x + (int64_t)warp * gridDim.x, lane, pf);
    for (int64_t t = blockIdx.x + (int64_t)warp * gridDim.x; t < ntile; t += tstep, j += NC) {
        const int sl = j % NS;
        bar_wait(&sm.full[sl], (j / NS) & 1);
        const TileId id = tile_of(t, A.G, A.count);
        const int64_t r0 = (int64_t)id.q * Q;
        const int kmax = (int)min((int64_t)Q, A.n - r0);
        const T *d = sm.slot[sl];
        const T *c = d + TILE;
        const int64_t sl_sys = (int64_t)id.g * TW + lane;        // system within the slab
        const bool ok = sl_sys < A.ms;
        const int64_t sys = (int64_t)id.b * A.msp + sl_sys;
        if (!P2) {
            if (PER && id.q >= A.qspec) {
                int ks[4];
#pragma unroll
                for (int jx = 0; jx < 4; ++jx) {
                    const int64_t rr = A.srow[jx] - r0;
                    ks[jx] = (A.srow[jx] >= 0 && rr >= 0 && rr < Q) ? (int)rr : -1;
                }
                tile_carry<T, K, true, false>(d, c, kmax, lane, ks, A, sys, ok, id.q);
            } else {
                const int ks[4] = {-1, -1, -1, -1};
                if (kmax == Q) tile_carry<T, K, false, true>(d, c, Q, lane, ks, A, sys, ok, id.q);
                else tile_carry<T, K, false, false>(d, c, kmax, lane, ks, A, sys, ok, id.q);
            }
            __syncwarp();
            if (lane == 0) bar_arrive(&sm.empty[sl]);
            continue;
        }
        // pass 2: the column, inflows and x_l into registers
        T v[Q];
#pragma unroll
        for (int k = 0; k < Q; ++k) v[k] = d[k * TW + lane];
        const T y0 = pf[0], y1 = pf[1], z0 = pf[2], z1 = pf[3], xl0 = pf[4], xl1 = pf[5];
        if (t + tstep < ntile) load_inflow<T, PER>(A, t + tstep, lane, pf);
        if (kmax == Q) tile_solve<T, K, PER, true>(v, c, Q, y0, y1, z0, z1, xl0, xl1);
        else tile_solve<T, K, PER, false>(v, c, kmax, y0, y1, z0, z1, xl0, xl1);
        // the slot is released after the solve (reads the coefficients in place)
        __syncwarp();
        if (lane == 0) bar_arrive(&sm.empty[sl]);
        if (PER && K == 2 && r0 + Q > A.n - 2) {
            // Navon: the last two unknowns are x_l itself
            const int k2 = (int)(A.n - 2 - r0);
#pragma unroll
            for (int k = 0; k < Q; ++k) {
                if (k == k2) v[k] = xl0;
                if (k == k2 + 1) v[k] = xl1;
            }
        }
        // stage the tile as NSW boxes of SW systems (128-byte rows) and TMA-store them.
        // (A single 256-byte-wide fp64 store box intermittently hung or faulted
        // on B200 under sustained back-to-back solves, tools/tp_stress2.sh;
        // 128-byte boxes, direct STG and bulk row copies never did.)
        constexpr int SW = 128 / (int)sizeof(T), NSW = TW / SW;
        if (lane == 0 && pend) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
        T *o = sm.out[warp];
#pragma unroll
        for (int k = 0; k < Q; ++k) o[(lane / SW) * Q * SW + k * SW + (lane % SW)] = v[k];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
#pragma unroll
            for (int h = 0; h < NSW; ++h)
                if (A.flat)
                    tma_store2(&smap, (int)(A.s0 + (int64_t)id.g * TW + h * SW), (int)((int64_t)id.b * A.n + r0),
                               o + h * Q * SW);
                else
                    tma_store(&smap, (int)(A.s0 + (int64_t)id.g * TW + h * SW), (int)r0, id.b, o + h * Q * SW);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        pend = true;
    }
    if (P2 && lane == 0 && pend) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---------------------------------------------------------------- scan
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

// CTA = 32 systems (lane = system) x NSEG chunk segments (warp = segment of
// consecutive chunks).  Every warp folds its segment lane-per-system (coalesced
// 1 KB record rows, warp-uniform chunk matrices), the NSEG segment maps are
// combined through shared memory, then every warp walks its segment again
// writing the inflows.  Records move in register batches of SB chunks.
constexpr int NSEG = 8, SB = 8;

template <typename T, int NW = NSEG>
struct ScanSmem {
    T agg[NW][TW][2];
    T pm[NW][4];
    T gsp[4][TW];
};

template <typename T>
__device__ __forceinline__ void ld_rec(const T *p, T *r)
{
    if (sizeof(T) == 8) {
        const double2 u = *reinterpret_cast<const double2 *>(p), w = *reinterpret_cast<const double2 *>(p + 2);
        r[0] = (T)u.x, r[1] = (T)u.y, r[2] = (T)w.x, r[3] = (T)w.y;
    } else {
        const float4 u = *reinterpret_cast<const float4 *>(p);
        r[0] = (T)u.x, r[1] = (T)u.y, r[2] = (T)u.z, r[3] = (T)u.w;
    }
}
template <typename T>
__device__ __forceinline__ void st_rec(T *p, const T *r)
{
    if (sizeof(T) == 8) {
        *reinterpret_cast<double2 *>(p) = make_double2((double)r[0], (double)r[1]);
        *reinterpret_cast<double2 *>(p + 2) = make_double2((double)r[2], (double)r[3]);
    } else {
        *reinterpret_cast<float4 *>(p) = make_float4((float)r[0], (float)r[1], (float)r[2], (float)r[3]);
    }
}

template <typename T, int K, bool PER>
__global__ void __launch_bounds__(32 * NSEG) tp_scan_kernel(const Args<T> A)
{
    pdl_wait();
    pdl_trigger();
    __shared__ ScanSmem<T> S;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t nsys = A.msp * A.count;
    const int64_t sys = (int64_t)blockIdx.x * TW + lane;   // msp is a multiple of TW: never past nsys
    const int nq = A.nq, cps = (nq + NSEG - 1) / NSEG;
    const int qa = min(nq, w * cps), qe = min(nq, qa + cps);
    T *car = A.car + sys * 4;
    const int64_t qstride = nsys * 4;

    // ---- forward fold of my segment: a = (Mf a + yF) over q, P = prod Mf
    T P[4] = {T(1), T(0), T(0), T(1)}, a0 = T(0), a1 = T(0);
    for (int q0 = qa; q0 < qe; q0 += SB) {
        T R[SB][4];
#pragma unroll
        for (int i = 0; i < SB; ++i)
            if (q0 + i < qe) ld_rec(car + (q0 + i) * qstride, R[i]);
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
    S.agg[w][lane][0] = a0;
    S.agg[w][lane][1] = a1;
    if (lane == 0)
        for (int e = 0; e < 4; ++e) S.pm[w][e] = P[e];
    __syncthreads();
    T y0 = T(0), y1 = T(0);
    for (int v = 0; v < w; ++v) {
        T t0, t1;
        mv(S.pm[v], y0, y1, t0, t1);
        y0 = t0 + S.agg[v][lane][0];
        y1 = t1 + S.agg[v][lane][1];
    }
    // ---- walk: yin_q replaces yF_q, c_q = zB_q + H_q yin_q replaces zB_q
    T gs[4] = {T(0), T(0), T(0), T(0)};
    bool own[4] = {false, false, false, false};
    for (int q0 = qa; q0 < qe; q0 += SB) {
        T R[SB][4];
#pragma unroll
        for (int i = 0; i < SB; ++i)
            if (q0 + i < qe) ld_rec(car + (q0 + i) * qstride, R[i]);
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
                        if (A.srow[jx] >= 0 && A.srow[jx] / Q == q) {
                            gs[jx] = A.spec[sys * 4 + jx] + A.rsp[jx * 2] * y0 + A.rsp[jx * 2 + 1] * y1;
                            own[jx] = true;
                        }
                }
                mv(m, y0, y1, t0, t1);
                y0 = t0 + yf0;
                y1 = t1 + yf1;
                st_rec(car + q * qstride, R[i]);
            }
    }
    if (PER) {
#pragma unroll
        for (int jx = 0; jx < 4; ++jx)
            if (own[jx]) S.gsp[jx][lane] = gs[jx];
    }
    // ---- backward fold of my segment (high to low): c = Mb c + c_q, Pb = prod Mb
    T Pb[4] = {T(1), T(0), T(0), T(1)}, c0 = T(0), c1 = T(0);
    for (int q1 = qe; q1 > qa; q1 -= SB) {
        T R[SB][4];
#pragma unroll
        for (int i = 0; i < SB; ++i)
            if (q1 - 1 - i >= qa) ld_rec(car + (q1 - 1 - i) * qstride, R[i]);
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
    __syncthreads();   // forward aggregates consumed
    S.agg[w][lane][0] = c0;
    S.agg[w][lane][1] = c1;
    if (lane == 0)
        for (int e = 0; e < 4; ++e) S.pm[w][e] = Pb[e];
    __syncthreads();
    T z0 = T(0), z1 = T(0);
    for (int v = NSEG - 1; v > w; --v) {
        T t0, t1;
        mv(S.pm[v], z0, z1, t0, t1);
        z0 = t0 + S.agg[v][lane][0];
        z1 = t1 + S.agg[v][lane][1];
    }
    for (int q1 = qe; q1 > qa; q1 -= SB) {
        T R[SB][4];
#pragma unroll
        for (int i = 0; i < SB; ++i)
            if (q1 - 1 - i >= qa) ld_rec(car + (q1 - 1 - i) * qstride, R[i]);
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
                st_rec(car + q * qstride, R[i]);
            }
    }
    if (PER && w == 0 && sys % A.msp < A.ms) {
        // (x_0, x_1) of the non-cyclic solution = warp 0's z after its walk
        const T y1c = z0, y2c = z1;
        T g[4];
#pragma unroll
        for (int jx = 0; jx < 4; ++jx) g[jx] = A.srow[jx] >= 0 ? S.gsp[jx][lane] : T(0);
        const double *sc = A.scal;
        T xl0, xl1;
        if (K == 2) {
            // Navon (eq:first_two)
            const T ym1 = g[1], ym2 = g[0] - T(sc[10]) * g[1];
            const T q0 = g[2] - (T(sc[4]) * y1c + T(sc[5]) * ym2 + T(sc[6]) * ym1);
            const T q1 = g[3] - (T(sc[7]) * y1c + T(sc[8]) * y2c + T(sc[9]) * ym1);
            xl0 = T(sc[0]) * q0 + T(sc[1]) * q1;
            xl1 = T(sc[2]) * q0 + T(sc[3]) * q1;
        } else {
            // Sherman–Morrison
            xl0 = (y1c + T(sc[0]) * g[0]) / T(sc[1]);
            xl1 = T(0);
        }
        A.xl[sys * 2 + 0] = xl0;
        A.xl[sys * 2 + 1] = xl1;
    }
}

// Register-resident scan (nq <= NW * CPS): the same segment scheme with NW = 16
// warps and each warp's <= CPS chunk records held in registers between the
// folds and walks, so the records are loaded once and stored once.
constexpr int NSEG_R = 16, CPS_R = 8;

template <typename T>
__device__ __forceinline__ void ldm4s(const T *p, T *m)
{
    lds2(p, m[0], m[1]);
    lds2(p + 2, m[2], m[3]);
}

template <typename T, int K, bool PER>
__global__ void __launch_bounds__(32 * NSEG_R) tp_scan_reg_kernel(const Args<T> A)
{
    pdl_wait();
    pdl_trigger();
    constexpr int NW = NSEG_R, CPS = CPS_R;
    __shared__ ScanSmem<T, NW> S;
    __shared__ __align__(16) T cts[NW * CPS][12];   // the chunk maps, staged once per CTA
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t nsys = A.msp * A.count;
    const int64_t sys = (int64_t)blockIdx.x * TW + lane;
    const int nq = A.nq, cps = (nq + NW - 1) / NW;
    const int qa = min(nq, w * cps), cnt = min(nq, qa + cps) - qa;
    T *car = A.car + sys * 4;
    const int64_t qstride = nsys * 4;
    for (int e = threadIdx.x; e < nq * 12; e += blockDim.x) (&cts[0][0])[e] = A.ct[e];
    T R[CPS][4];
#pragma unroll
    for (int i = 0; i < CPS; ++i)
        if (i < cnt) ld_rec(car + (qa + i) * qstride, R[i]);
    __syncthreads();   // chunk maps staged
    // ---- forward fold of my segment
    T P[4] = {T(1), T(0), T(0), T(1)}, a0 = T(0), a1 = T(0);
#pragma unroll
    for (int i = 0; i < CPS; ++i)
        if (i < cnt) {
            T m[4], t0, t1;
            ldm4s(cts[qa + i], m);
            mv(m, a0, a1, t0, t1);
            a0 = t0 + R[i][0];
            a1 = t1 + R[i][1];
            mmul(m, P, P);
        }
    S.agg[w][lane][0] = a0;
    S.agg[w][lane][1] = a1;
    if (lane == 0)
        for (int e = 0; e < 4; ++e) S.pm[w][e] = P[e];
    __syncthreads();
    T y0 = T(0), y1 = T(0);
    for (int v = 0; v < w; ++v) {
        T t0, t1;
        mv(S.pm[v], y0, y1, t0, t1);
        y0 = t0 + S.agg[v][lane][0];
        y1 = t1 + S.agg[v][lane][1];
    }
    // ---- forward walk: yin_q, c_q = zB_q + H_q yin_q; cyclic rows' true g
#pragma unroll
    for (int i = 0; i < CPS; ++i)
        if (i < cnt) {
            const int q = qa + i;
            T m[4], h[4], t0, t1;
            ldm4s(cts[q], m);
            ldm4s(cts[q] + 8, h);
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
                        S.gsp[jx][lane] = A.spec[sys * 4 + jx] + A.rsp[jx * 2] * y0 + A.rsp[jx * 2 + 1] * y1;
            }
            mv(m, y0, y1, t0, t1);
            y0 = t0 + yf0;
            y1 = t1 + yf1;
        }
    // ---- backward fold of my segment (high to low)
    T Pb[4] = {T(1), T(0), T(0), T(1)}, c0 = T(0), c1 = T(0);
#pragma unroll
    for (int i = CPS - 1; i >= 0; --i)
        if (i < cnt) {
            T m[4], t0, t1;
            ldm4s(cts[qa + i] + 4, m);
            mv(m, c0, c1, t0, t1);
            c0 = t0 + R[i][2];
            c1 = t1 + R[i][3];
            mmul(m, Pb, Pb);
        }
    __syncthreads();   // forward aggregates consumed
    S.agg[w][lane][0] = c0;
    S.agg[w][lane][1] = c1;
    if (lane == 0)
        for (int e = 0; e < 4; ++e) S.pm[w][e] = Pb[e];
    __syncthreads();
    T z0 = T(0), z1 = T(0);
    for (int v = NW - 1; v > w; --v) {
        T t0, t1;
        mv(S.pm[v], z0, z1, t0, t1);
        z0 = t0 + S.agg[v][lane][0];
        z1 = t1 + S.agg[v][lane][1];
    }
#pragma unroll
    for (int i = CPS - 1; i >= 0; --i)
        if (i < cnt) {
            T m[4], t0, t1;
            ldm4s(cts[qa + i] + 4, m);
            const T cq0 = R[i][2], cq1 = R[i][3];
            R[i][2] = z0;
            R[i][3] = z1;
            mv(m, z0, z1, t0, t1);
            z0 = t0 + cq0;
            z1 = t1 + cq1;
        }
#pragma unroll
    for (int i = 0; i < CPS; ++i)
        if (i < cnt) st_rec(car + (qa + i) * qstride, R[i]);
    if (PER && w == 0 && sys % A.msp < A.ms) {
        const T y1c = z0, y2c = z1;   // (x_0, x_1) of the non-cyclic solution
        T g[4];
#pragma unroll
        for (int jx = 0; jx < 4; ++jx) g[jx] = A.srow[jx] >= 0 ? S.gsp[jx][lane] : T(0);
        const double *sc = A.scal;
        T xl0, xl1;
        if (K == 2) {
            // Navon (eq:first_two)
            const T ym1 = g[1], ym2 = g[0] - T(sc[10]) * g[1];
            const T q0 = g[2] - (T(sc[4]) * y1c + T(sc[5]) * ym2 + T(sc[6]) * ym1);
            const T q1 = g[3] - (T(sc[7]) * y1c + T(sc[8]) * y2c + T(sc[9]) * ym1);
            xl0 = T(sc[0]) * q0 + T(sc[1]) * q1;
            xl1 = T(sc[2]) * q0 + T(sc[3]) * q1;
        } else {
            // Sherman–Morrison
            xl0 = (y1c + T(sc[0]) * g[0]) / T(sc[1]);
            xl1 = T(0);
        }
        A.xl[sys * 2 + 0] = xl0;
        A.xl[sys * 2 + 1] = xl1;
    }
}

// Short systems (nq <= SEQ_MAX chunks): one thread per system walks its chunks
// sequentially with the records in registers (no cross-warp combine); the
// chunk maps are staged in shared memory per CTA.
constexpr int SEQ_MAX = 16;

template <typename T, int K, bool PER>
__global__ void __launch_bounds__(256) tp_scan_seq_kernel(const Args<T> A)
{
    pdl_wait();
    pdl_trigger();
    __shared__ __align__(16) T cts[SEQ_MAX][12];
    const int nq = A.nq;
    for (int e = threadIdx.x; e < nq * 12; e += blockDim.x) (&cts[0][0])[e] = A.ct[e];
    __syncthreads();
    const int64_t nsys = A.msp * A.count;
    const int64_t sys = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (sys >= nsys) return;
    T *car = A.car + sys * 4;
    const int64_t qstride = nsys * 4;
    T R[SEQ_MAX][4];
#pragma unroll
    for (int q = 0; q < SEQ_MAX; ++q)
        if (q < nq) ld_rec(car + q * qstride, R[q]);
    T y0 = T(0), y1 = T(0), g[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
    for (int q = 0; q < SEQ_MAX; ++q)
        if (q < nq) {
            T m[4], h[4], t0, t1;
            ldm4s(cts[q], m);
            ldm4s(cts[q] + 8, h);
            const T yf0 = R[q][0], yf1 = R[q][1];
            mv(h, y0, y1, t0, t1);
            R[q][0] = y0;
            R[q][1] = y1;
            R[q][2] += t0;
            R[q][3] += t1;
            if (PER && q >= A.qspec) {
#pragma unroll
                for (int jx = 0; jx < 4; ++jx)
                    if (A.srow[jx] >= 0 && A.srow[jx] / Q == q)
                        g[jx] = A.spec[sys * 4 + jx] + A.rsp[jx * 2] * y0 + A.rsp[jx * 2 + 1] * y1;
            }
            mv(m, y0, y1, t0, t1);
            y0 = t0 + yf0;
            y1 = t1 + yf1;
        }
    T z0 = T(0), z1 = T(0);
#pragma unroll
    for (int q = SEQ_MAX - 1; q >= 0; --q)
        if (q < nq) {
            T m[4], t0, t1;
            ldm4s(cts[q] + 4, m);
            const T cq0 = R[q][2], cq1 = R[q][3];
            R[q][2] = z0;
            R[q][3] = z1;
            mv(m, z0, z1, t0, t1);
            z0 = t0 + cq0;
            z1 = t1 + cq1;
        }
#pragma unroll
    for (int q = 0; q < SEQ_MAX; ++q)
        if (q < nq) st_rec(car + q * qstride, R[q]);
    if (PER && sys % A.msp < A.ms) {
        const T y1c = z0, y2c = z1;   // (x_0, x_1) of the non-cyclic solution
        const double *sc = A.scal;
        T xl0, xl1;
        if (K == 2) {
            // Navon (eq:first_two)
            const T ym1 = g[1], ym2 = g[0] - T(sc[10]) * g[1];
            const T q0 = g[2] - (T(sc[4]) * y1c + T(sc[5]) * ym2 + T(sc[6]) * ym1);
            const T q1 = g[3] - (T(sc[7]) * y1c + T(sc[8]) * y2c + T(sc[9]) * ym1);
            xl0 = T(sc[0]) * q0 + T(sc[1]) * q1;
            xl1 = T(sc[2]) * q0 + T(sc[3]) * q1;
        } else {
            // Sherman–Morrison
            xl0 = (y1c + T(sc[0]) * g[0]) / T(sc[1]);
            xl1 = T(0);
        }
        A.xl[sys * 2 + 0] = xl0;
        A.xl[sys * 2 + 1] = xl1;
    }
}

}  // namespace tp
}  // namespace pb

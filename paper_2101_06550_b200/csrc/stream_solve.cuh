// stream_solve.cuh — the shared-LHS batched banded solve for the interleaved
// layout (pent_solve / tri_solve) as a persistent,
// warp-specialised, TMA-streamed two-phase partitioned solve for sm_100a.
//
// Why (measured on B200): a CTA that loads its whole share of
// a system group into registers, solves, and stores reaches only 3-4 TB/s
// even with no arithmetic (the load burst drains before anything else is in
// flight); persistent CTAs that keep a ring of TMA tile loads in flight reach
// 5.6-6.3 TB/s.  So nothing is held on chip across CTAs: each system is cut
// into row tiles of R rows and every tile is visited twice.
//
//   P1(tile): read f (HBM), partitioned zero-inflow sweeps -> the tile's
//             affine aggregates (forward carry A_f, backward carry A_b) and,
//             for cyclic systems, the forward values on the rows the Navon /
//             Sherman–Morrison 2x2 needs.  The CTA finishing the last P1 tile
//             of a group runs the group scan: the true inflows (Fin, Bin) of
//             every tile and the periodic pair x_l (eq:first_two).
//   P2(tile): read f again (L2-resident: P2 trails P1 by L groups), run the
//             4-sweep partitioned solve with the tile inflows, apply the
//             periodic correction, store x (STG, streaming).
//
// HBM traffic per unknown: f once, x once (16 B fp64); the second f read and
// the O(1/R) aggregates stay in the 126 MB L2.  The algebra inside a tile is
// band_core's (chunk sweeps + Kogge-Stone carry scan with LHS-only transfer
// matrices); the tile level uses the tile transfer matrices Mf_t, Mb_t and the
// response Hf_t of the backward carry to the forward inflow:
//   Fout = A_f + Mf_t Fin,   Bout = A_b + Hf_t Fin + Mb_t Bin.
//
// Roles: warp 0 = TMA producer (one elected lane), NG consumer groups of
// NC = W*PC threads; items alternate between groups; slots are released as
// soon as the tile is in registers, so up to S tiles are in flight per SM.
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
// A tile is W systems x R = PC*MR rows (one TMA box, 128-byte swizzled rows).
// Warp q of a team owns the SYS systems [q*SYS, (q+1)*SYS) of the tile; lane
// p owns the chunk of MR rows starting at p*MR, for all SYS systems (SYS
// independent recurrences per thread).  MR is odd so the 32 rows a warp reads
// at once fall on 8 distinct swizzle phases: the tile reads are
// conflict-free.  Chunk carries are scanned across the 32 lanes with warp
// shuffles, so a warp needs no barrier with any other warp.
template <typename T>
struct StreamGeom;
template <>
struct StreamGeom<double> {
    static constexpr int W = 16, SYS = 4, PC = 32, MR = 7, SA = 3, SB = 3;
};
template <>
struct StreamGeom<float> {
    static constexpr int W = 32, SYS = 8, PC = 32, MR = 7, SA = 3, SB = 3;
};
constexpr int STREAM_NQ = 4;      // warps per tile (W / SYS)
constexpr int STREAM_TEAMS = 3;   // consumer teams of STREAM_NQ warps: 0,1 on ring A, 2 on ring B
constexpr int STREAM_THREADS = 96 + STREAM_TEAMS * STREAM_NQ * 32;   // + producer A, producer B, sync warp
constexpr int NCOEF = 7;          // F0 F1 F2 B1 B2 Z1 Z2 (coefficient slots 0,1,2,4,5,6,7)
constexpr int DONE_Q = 8;         // P1-completion mbarriers (sync warp queue depth)

template <typename T>
struct StreamSmem {
    using G = StreamGeom<T>;
    static constexpr int W = G::W, PC = G::PC, MR = G::MR, R = PC * MR, SA = G::SA, SB = G::SB;
    static constexpr int SLOT = R * W;   // elements; R*W*sizeof(T) = 28 KB, a multiple of 1024 B
    T slot[SA + SB][SLOT];               // ring A (P1) then ring B (P2), 1024-B aligned
    T coef[NCOEF][MR][PC];               // this CTA's coefficient rows, chunk-fastest
    T rsp[4][MR][PC];                    // RF0 RF1 RB0 RB1 of this CTA's rows
    T tab[TAB_STRIDE][PC];               // chunk scan tables, chunk-fastest
    T wsc[STREAM_TEAMS * STREAM_NQ][10][G::SYS];   // per consumer warp: inflows, xl, spec rows
    uint64_t full[SA + SB], empty[SA + SB];
    uint64_t done[DONE_Q];               // P1 tile finished by its 4 warps (count 4)
    int p1_fenced;                       // P1 tiles whose stores are published (for producer B)
    int p2_issued;                       // P2 loads issued (P1 lead control)
};
// per-warp scratch slots (wsc[warp][slot][system])
constexpr int WS_FIN0 = 0, WS_FIN1 = 1, WS_BIN0 = 2, WS_BIN1 = 3, WS_XL0 = 4, WS_XL1 = 5, WS_SP = 6;

// element (r, c16) of a 128-byte-swizzled tile (TMA CU_TENSOR_MAP_SWIZZLE_128B):
// 16-byte chunk index XOR (row mod 8)
template <typename T>
__device__ __forceinline__ const T *swz(const T *tile, int r, int c16)
{
    return reinterpret_cast<const T *>(reinterpret_cast<const char *>(tile) + r * 128 + ((c16 ^ (r & 7)) << 4));
}

// one row of this warp's SYS systems: two 16-byte chunks
__device__ __forceinline__ void ld_row(const double *tile, int r, int q, double (&o)[4])
{
    const double2 a = *reinterpret_cast<const double2 *>(swz(tile, r, 2 * q));
    const double2 b = *reinterpret_cast<const double2 *>(swz(tile, r, 2 * q + 1));
    o[0] = a.x, o[1] = a.y, o[2] = b.x, o[3] = b.y;
}
__device__ __forceinline__ void ld_row(const float *tile, int r, int q, float (&o)[8])
{
    const float4 a = *reinterpret_cast<const float4 *>(swz(tile, r, 2 * q));
    const float4 b = *reinterpret_cast<const float4 *>(swz(tile, r, 2 * q + 1));
    o[0] = a.x, o[1] = a.y, o[2] = a.z, o[3] = a.w, o[4] = b.x, o[5] = b.y, o[6] = b.z, o[7] = b.w;
}
// STREAM: evict-first (final x); KEEP: default policy (P1's local solution,
// re-read by P2 from L2)
template <bool STREAM>
__device__ __forceinline__ void st_row(double *d, const double (&v)[4])
{
    if (STREAM) {
        __stcs(reinterpret_cast<double2 *>(d), make_double2(v[0], v[1]));
        __stcs(reinterpret_cast<double2 *>(d) + 1, make_double2(v[2], v[3]));
    } else {
        reinterpret_cast<double2 *>(d)[0] = make_double2(v[0], v[1]);
        reinterpret_cast<double2 *>(d)[1] = make_double2(v[2], v[3]);
    }
}
template <bool STREAM>
__device__ __forceinline__ void st_row(float *d, const float (&v)[8])
{
    if (STREAM) {
        __stcs(reinterpret_cast<float4 *>(d), make_float4(v[0], v[1], v[2], v[3]));
        __stcs(reinterpret_cast<float4 *>(d) + 1, make_float4(v[4], v[5], v[6], v[7]));
    } else {
        reinterpret_cast<float4 *>(d)[0] = make_float4(v[0], v[1], v[2], v[3]);
        reinterpret_cast<float4 *>(d)[1] = make_float4(v[4], v[5], v[6], v[7]);
    }
}

// ---------------------------------------------------------------- warp scans
// Kogge–Stone over the 32 lanes (chunks) of SYS independent affine carries:
// b_p += P_{p,l} b_{p-2^l} (forward, P = chunk tables Pf) or, with `rev`,
// b_p += P_{p,l} b_{p+2^l} (backward, Pb).  Inclusive result in b.
template <typename T, int SYS, bool REV>
__device__ __forceinline__ void warp_scan(T (&b0)[SYS], T (&b1)[SYS], int p, const T (*tab)[32], int tab_off)
{
#pragma unroll
    for (int l = 0; l < 5; ++l) {
        const int d = 1 << l;
        const T m0 = tab[tab_off + 4 * l + 0][p], m1 = tab[tab_off + 4 * l + 1][p];
        const T m2 = tab[tab_off + 4 * l + 2][p], m3 = tab[tab_off + 4 * l + 3][p];
        const bool ok = REV ? (p + d < 32) : (p >= d);
#pragma unroll
        for (int j = 0; j < SYS; ++j) {
            const T u0 = REV ? __shfl_down_sync(0xffffffffu, b0[j], d) : __shfl_up_sync(0xffffffffu, b0[j], d);
            const T u1 = REV ? __shfl_down_sync(0xffffffffu, b1[j], d) : __shfl_up_sync(0xffffffffu, b1[j], d);
            if (ok) {
                b0[j] += m0 * u0 + m1 * u1;
                b1[j] += m2 * u0 + m3 * u1;
            }
        }
    }
}

// ---------------------------------------------------------------- group scan
// Tile inflows of one (group, quad) from the published tile aggregates, run by
// the sync warp of the group's designated CTA once every P1 tile is counted.  Lane l owns tiles
// [l*span, (l+1)*span); affine operators (M, c): y -> c + M y are composed
// across lanes with a Kogge–Stone scan, so the latency is one L2 round trip
// plus 5 shuffle levels.
//   forward:  Fout_r = A_f[r] + Mf_t[r] Fin_r,                  Fin_0 = 0
//   backward: Bout_r = (A_b[r] + Hf_t[r] Fin_r) + Mb_t[r] Bin_r, Bin_last = 0
// then the periodic pair from Bout_0 = (y_1, y_2) and the spec rows.
constexpr int MAX_NRB = 64;  // == STREAM_MAX_NRB (band_tile.cuh), checked in stream_launch.cuh
constexpr int GS_SPAN = MAX_NRB / 32;

template <typename T>
struct Aff {
    T m0, m1, m2, m3, c0, c1;
};
// op o pre  (pre applied first)
template <typename T>
__device__ __forceinline__ Aff<T> compose(const Aff<T> &op, const Aff<T> &pre)
{
    Aff<T> r;
    r.m0 = op.m0 * pre.m0 + op.m1 * pre.m2;
    r.m1 = op.m0 * pre.m1 + op.m1 * pre.m3;
    r.m2 = op.m2 * pre.m0 + op.m3 * pre.m2;
    r.m3 = op.m2 * pre.m1 + op.m3 * pre.m3;
    r.c0 = op.c0 + op.m0 * pre.c0 + op.m1 * pre.c1;
    r.c1 = op.c1 + op.m2 * pre.c0 + op.m3 * pre.c1;
    return r;
}
template <typename T, bool UP>
__device__ __forceinline__ Aff<T> shfl_aff(const Aff<T> &a, int d)
{
    Aff<T> r;
#define PB_SH(f) r.f = UP ? __shfl_up_sync(0xffffffffu, a.f, d) : __shfl_down_sync(0xffffffffu, a.f, d)
    PB_SH(m0);
    PB_SH(m1);
    PB_SH(m2);
    PB_SH(m3);
    PB_SH(c0);
    PB_SH(c1);
#undef PB_SH
    return r;
}

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

template <typename T, int K, bool PER>
__device__ __noinline__ void group_scan(const StreamArgs<T> &A, int64_t g, int q, int lane)
{
    using G = StreamGeom<T>;
    constexpr int W = G::W, SYS = G::SYS;
    const int nrb = A.nrb;
    const int span = (nrb + 31) / 32;
    const int r_lo = lane * span;
    const int64_t sys0 = q * SYS;
    const T *agg = A.sc.agg + (g * nrb * W + sys0) * 4;   // tile r, system j at agg + (r*W + j)*4
    T *inf = A.sc.inf + (g * nrb * W + sys0) * 4;
    // all loads first (one L2 round trip), then SYS interleaved scans
    T af0[GS_SPAN][SYS], af1[GS_SPAN][SYS], ab0[GS_SPAN][SYS], ab1[GS_SPAN][SYS];
    T mf[GS_SPAN][4], mb[GS_SPAN][4], hf[GS_SPAN][4];
#pragma unroll
    for (int k = 0; k < GS_SPAN; ++k) {
        const int r = r_lo + k;
        const bool ok = k < span && r < nrb;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            mf[k][c] = ok ? __ldg(A.tb.mft + r * 4 + c) : T(c == 0 || c == 3);
            mb[k][c] = ok ? __ldg(A.tb.mbt + r * 4 + c) : T(c == 0 || c == 3);
            hf[k][c] = ok ? __ldg(A.tb.hft + r * 4 + c) : T(0);
        }
#pragma unroll
        for (int j = 0; j < SYS; ++j) {
            const T *a = agg + ((int64_t)r * W + j) * 4;
            af0[k][j] = ok ? __ldcg(a) : T(0);
            af1[k][j] = ok ? __ldcg(a + 1) : T(0);
            ab0[k][j] = ok ? __ldcg(a + 2) : T(0);
            ab1[k][j] = ok ? __ldcg(a + 3) : T(0);
        }
    }
    // ---- forward: lane composite (the matrix part is shared by all systems)
    T M0 = T(1), M1 = T(0), M2 = T(0), M3 = T(1);
    T C0[SYS], C1[SYS];
#pragma unroll
    for (int j = 0; j < SYS; ++j) C0[j] = C1[j] = T(0);
#pragma unroll
    for (int k = 0; k < GS_SPAN; ++k) {
#pragma unroll
        for (int j = 0; j < SYS; ++j) {
            const T n0 = af0[k][j] + mf[k][0] * C0[j] + mf[k][1] * C1[j];
            const T n1 = af1[k][j] + mf[k][2] * C0[j] + mf[k][3] * C1[j];
            C0[j] = n0;
            C1[j] = n1;
        }
        const T n0 = mf[k][0] * M0 + mf[k][1] * M2, n1 = mf[k][0] * M1 + mf[k][1] * M3;
        const T n2 = mf[k][2] * M0 + mf[k][3] * M2, n3 = mf[k][2] * M1 + mf[k][3] * M3;
        M0 = n0, M1 = n1, M2 = n2, M3 = n3;
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        // (M, C) <- (M, C) o (M', C') of lane - d
        const T u0 = __shfl_up_sync(0xffffffffu, M0, d), u1 = __shfl_up_sync(0xffffffffu, M1, d);
        const T u2 = __shfl_up_sync(0xffffffffu, M2, d), u3 = __shfl_up_sync(0xffffffffu, M3, d);
        const bool ok = lane >= d;
#pragma unroll
        for (int j = 0; j < SYS; ++j) {
            const T c0 = __shfl_up_sync(0xffffffffu, C0[j], d), c1 = __shfl_up_sync(0xffffffffu, C1[j], d);
            if (ok) {
                C0[j] += M0 * c0 + M1 * c1;
                C1[j] += M2 * c0 + M3 * c1;
            }
        }
        if (ok) {
            const T n0 = M0 * u0 + M1 * u2, n1 = M0 * u1 + M1 * u3;
            const T n2 = M2 * u0 + M3 * u2, n3 = M2 * u1 + M3 * u3;
            M0 = n0, M1 = n1, M2 = n2, M3 = n3;
        }
    }
    T fin0[GS_SPAN][SYS], fin1[GS_SPAN][SYS];
#pragma unroll
    for (int j = 0; j < SYS; ++j) {
        T F0 = __shfl_up_sync(0xffffffffu, C0[j], 1), F1 = __shfl_up_sync(0xffffffffu, C1[j], 1);
        if (lane == 0) F0 = F1 = T(0);
#pragma unroll
        for (int k = 0; k < GS_SPAN; ++k) {
            fin0[k][j] = F0;
            fin1[k][j] = F1;
            const T n0 = af0[k][j] + mf[k][0] * F0 + mf[k][1] * F1;
            const T n1 = af1[k][j] + mf[k][2] * F0 + mf[k][3] * F1;
            F0 = n0;
            F1 = n1;
            // backward constants d_r = A_b[r] + Hf_t[r] Fin_r
            ab0[k][j] += hf[k][0] * fin0[k][j] + hf[k][1] * fin1[k][j];
            ab1[k][j] += hf[k][2] * fin0[k][j] + hf[k][3] * fin1[k][j];
        }
    }
    // ---- backward: lane composite over its tiles (right to left), reverse lane scan
    M0 = T(1), M1 = T(0), M2 = T(0), M3 = T(1);
#pragma unroll
    for (int j = 0; j < SYS; ++j) C0[j] = C1[j] = T(0);
#pragma unroll
    for (int k = GS_SPAN - 1; k >= 0; --k) {
#pragma unroll
        for (int j = 0; j < SYS; ++j) {
            const T n0 = ab0[k][j] + mb[k][0] * C0[j] + mb[k][1] * C1[j];
            const T n1 = ab1[k][j] + mb[k][2] * C0[j] + mb[k][3] * C1[j];
            C0[j] = n0;
            C1[j] = n1;
        }
        const T n0 = mb[k][0] * M0 + mb[k][1] * M2, n1 = mb[k][0] * M1 + mb[k][1] * M3;
        const T n2 = mb[k][2] * M0 + mb[k][3] * M2, n3 = mb[k][2] * M1 + mb[k][3] * M3;
        M0 = n0, M1 = n1, M2 = n2, M3 = n3;
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const T u0 = __shfl_down_sync(0xffffffffu, M0, d), u1 = __shfl_down_sync(0xffffffffu, M1, d);
        const T u2 = __shfl_down_sync(0xffffffffu, M2, d), u3 = __shfl_down_sync(0xffffffffu, M3, d);
        const bool ok = lane + d < 32;
#pragma unroll
        for (int j = 0; j < SYS; ++j) {
            const T c0 = __shfl_down_sync(0xffffffffu, C0[j], d), c1 = __shfl_down_sync(0xffffffffu, C1[j], d);
            if (ok) {
                C0[j] += M0 * c0 + M1 * c1;
                C1[j] += M2 * c0 + M3 * c1;
            }
        }
        if (ok) {
            const T n0 = M0 * u0 + M1 * u2, n1 = M0 * u1 + M1 * u3;
            const T n2 = M2 * u0 + M3 * u2, n3 = M2 * u1 + M3 * u3;
            M0 = n0, M1 = n1, M2 = n2, M3 = n3;
        }
    }
    T y1[SYS], y2[SYS];
#pragma unroll
    for (int j = 0; j < SYS; ++j) {
        T B0 = __shfl_down_sync(0xffffffffu, C0[j], 1), B1 = __shfl_down_sync(0xffffffffu, C1[j], 1);
        if (lane == 31) B0 = B1 = T(0);
#pragma unroll
        for (int k = GS_SPAN - 1; k >= 0; --k) {
            const int r = r_lo + k;
            if (k < span && r < nrb) {
                T *o = inf + ((int64_t)r * W + j) * 4;
                o[0] = fin0[k][j];
                o[1] = fin1[k][j];
                o[2] = B0;
                o[3] = B1;
            }
            const T n0 = ab0[k][j] + mb[k][0] * B0 + mb[k][1] * B1;
            const T n1 = ab1[k][j] + mb[k][2] * B0 + mb[k][3] * B1;
            B0 = n0;
            B1 = n1;
        }
        y1[j] = B0;   // lane 0 ends at tile 0: Bout_0 = (x_0, x_1)
        y2[j] = B1;
    }
    if (!PER) return;
    // ---- periodic pair: spec rows (true forward values) and y = Bout_0 (lane 0)
    T sp[4][SYS];
#pragma unroll
    for (int jx = 0; jx < 4; ++jx) {
        const int r = A.tb.srb[jx];
        const bool mine = r >= 0 && r >= r_lo && r < r_lo + span;
        const int owner = r >= 0 ? r / span : 0;
        const T g0 = r >= 0 ? __ldg(A.tb.gsp + jx * 2) : T(0), g1 = r >= 0 ? __ldg(A.tb.gsp + jx * 2 + 1) : T(0);
#pragma unroll
        for (int j = 0; j < SYS; ++j) {
            T val = T(0);
            if (mine) {
                T f0 = T(0), f1 = T(0);
#pragma unroll
                for (int k2 = 0; k2 < GS_SPAN; ++k2)
                    if (k2 == r - r_lo) {
                        f0 = fin0[k2][j];
                        f1 = fin1[k2][j];
                    }
                val = __ldcg(A.sc.spec + (g * W + sys0 + j) * 4 + jx) + g0 * f0 + g1 * f1;
            }
            sp[jx][j] = __shfl_sync(0xffffffffu, val, owner);
        }
    }
    if (lane == 0) {
#pragma unroll
        for (int j = 0; j < SYS; ++j) {
            T spp[4] = {sp[0][j], sp[1][j], sp[2][j], sp[3][j]};
            T xl0, xl1;
            local_xl<T, K>(A.tb.scal, y1[j], y2[j], spp, xl0, xl1);
            A.sc.xl[(g * W + sys0 + j) * 2 + 0] = xl0;
            A.sc.xl[(g * W + sys0 + j) * 2 + 1] = xl1;
        }
    }
}

#define PB_TR(slot)                                                                                   \
    do {                                                                                              \
        if (A.trace && q == 0 && lane == 0 && j < 256)                                                \
            A.trace[(((int64_t)blockIdx.x * STREAM_TEAMS + team) * 256 + j) * 8 + (slot)] = gtimer(); \
    } while (0)

// ---------------------------------------------------------------- the kernel
// Warps: 0 = ring-A producer, 1 = ring-B producer, 2 = sync warp, then three
// teams of four consumer warps (teams 0,1 alternate on ring A, team 2 drains
// ring B).
//  two-phase (nrb > 1):
//   ring A / P1: the tile's local solve (zero tile inflows) written in place,
//     tile aggregates A_f, A_b (and spec-row values) published;
//   sync warp: publishes finished P1 tiles (gpu fence, per-group counter) and
//     runs the group scans of the groups this CTA is designated for;
//   ring B / P2: re-reads the local solution (L2) once the group scan is
//     done and applies x = y + RF Fin + RB Bin (- Z x_l for cyclic systems).
//   Producer A runs at most `lead` tiles ahead of producer B (L2 residency).
//  single tile (nrb == 1): every item is a complete solve (local periodic pair).
template <typename T, int K, bool PER>
__global__ void __launch_bounds__(STREAM_THREADS, 1)
    stream_solve_kernel(const __grid_constant__ CUtensorMap tmap, const StreamArgs<T> A)
{
    using SM = StreamSmem<T>;
    using G = StreamGeom<T>;
    constexpr int W = G::W, SYS = G::SYS, PC = G::PC, MR = G::MR, R = SM::R, SA = G::SA, SB = G::SB;
    constexpr uint32_t TILE_BYTES = (uint32_t)(R * W * sizeof(T));
    static_assert(PC == 32 && W == STREAM_NQ * SYS && SYS * sizeof(T) == 32, "geometry");
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    SM &sm = *reinterpret_cast<SM *>(smem_raw + ((1024 - ((uintptr_t)smem_raw & 1023)) & 1023));

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nrb = A.nrb;
    const int rb = blockIdx.x % nrb, kk = blockIdx.x / nrb;
    const int64_t gt = A.groups * A.count;                 // groups over all batches
    const int ng = (int)((gt - kk + A.K - 1) / A.K);       // this CTA's groups: kk + A.K * i
    const bool two = nrb > 1;
    const int64_t row0 = (int64_t)rb * R;

    // ---- setup: barriers, coefficient / response rows and chunk tables (chunk-fastest)
    if (tid == 0) {
        for (int s = 0; s < SA + SB; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], STREAM_NQ);
        }
        for (int s = 0; s < DONE_Q; ++s) mbar_init(&sm.done[s], STREAM_NQ);
        sm.p1_fenced = 0;
        sm.p2_issued = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    {
        constexpr int cslot[NCOEF] = {0, 1, 2, 4, 5, 6, 7};
        for (int e = tid; e < NCOEF * MR * PC; e += blockDim.x) {
            const int c = e / (MR * PC), k = (e / PC) % MR, p = e % PC;
            sm.coef[c][k][p] = A.tb.coef[(row0 + p * MR + k) * COEF_STRIDE + cslot[c]];
        }
        if (two)
            for (int e = tid; e < 4 * MR * PC; e += blockDim.x) {
                const int c = e / (MR * PC), k = (e / PC) % MR, p = e % PC;
                sm.rsp[c][k][p] = A.tb.rsp[((int64_t)rb * 4 + c) * R + p * MR + k];
            }
        for (int e = tid; e < TAB_STRIDE * PC; e += blockDim.x) {
            const int c = e / PC, p = e % PC;
            sm.tab[c][p] = A.tb.tab[((int64_t)rb * PC + p) * TAB_STRIDE + c];
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
            // two-phase: every group on both rings; single tile: i % 3 != 2 on A, the rest on B
            if (!two && ((i % 3 != 2) != ringA)) continue;
            if (two) {
                volatile int *v2 = &sm.p2_issued, *vf = &sm.p1_fenced;
                if (ringA) {
                    // lead control, and the sync warp's completion queue must not wrap
                    while (i >= *v2 + A.lead || i >= *vf + DONE_Q - 1) __nanosleep(64);
                } else {
                    while (i >= *vf) __nanosleep(64);   // P1 stores of this tile published
                }
            }
            const int s = base + j % nslot;
            if (j >= nslot) mbar_wait(&sm.empty[s], ((j / nslot) - 1) & 1);
            const int64_t g = gid(i);
            const int b = (int)(g / A.groups), gg = (int)(g % A.groups);
            mbar_expect_tx(&sm.full[s], TILE_BYTES);
            tma_load_3d(sm.slot[s], &tmap, gg * W, rb * R, b, &sm.full[s]);
            if (two && !ringA) {
                asm volatile("" ::: "memory");
                *(volatile int *)&sm.p2_issued = i + 1;
            }
            ++j;
        }
        return;
    }

    // ================= sync warp: publish P1 tiles, run designated group scans
    if (warp == 2) {
        if (!two) return;
        int jd = 0;              // next local P1 tile to publish
        int is = rb;             // next designated group (i = rb, rb + nrb, ...)
        while (jd < ng || is < ng) {
            bool progress = false;
            int nd = 0;
            if (lane == 0)
                while (jd + nd < ng && nd < DONE_Q && mbar_test(&sm.done[(jd + nd) % DONE_Q], ((jd + nd) / DONE_Q) & 1))
                    ++nd;
            nd = __shfl_sync(0xffffffffu, nd, 0);
            if (nd > 0) {
                if (lane == 0) {
                    fence_acq_rel_gpu();          // the P1 warps' stores (cumulative through the mbarrier)
                    fence_proxy_async_global();   // ... visible to P2's TMA re-read as well
                    for (int u = 0; u < nd; ++u) red_add_relaxed(A.sc.cnt + gid(jd + u), 1);
                    *(volatile int *)&sm.p1_fenced = jd + nd;
                }
                jd += nd;
                progress = true;
            }
            if (is < ng) {
                const int64_t g = gid(is);
                int c = 0;
                if (lane == 0) c = ld_relaxed(A.sc.cnt + g);
                c = __shfl_sync(0xffffffffu, c, 0);
                if (c == nrb) {
                    fence_acq_rel_gpu();
#pragma unroll 1
                    for (int qd = 0; qd < STREAM_NQ; ++qd) group_scan<T, K, PER>(A, g, qd, lane);
                    __syncwarp();
                    if (lane == 0) {
                        fence_acq_rel_gpu();
                        st_release(A.sc.flag + g, 1);
                    }
                    is += nrb;
                    progress = true;
                }
            }
            if (!progress) __nanosleep(128);
        }
        return;
    }

    // ================= consumer warps
    const int cw = warp - 3;                 // consumer warp 0..11
    const int team = cw / STREAM_NQ, q = cw % STREAM_NQ;
    const bool ringA = team < 2;
    const int nslot = ringA ? SA : SB, sbase = ringA ? 0 : SA;
    const bool corr = two && !ringA;         // P2: elementwise correction
    const int p = lane;
    const int64_t r0 = row0 + (int64_t)p * MR;
    const T(*tab)[32] = sm.tab;
    T(*ws)[SYS] = sm.wsc[cw];

    int j = -1;
    for (int i = 0; i < ng; ++i) {
        if (!two && ((i % 3 != 2) != ringA)) continue;
        ++j;   // index of this item in its ring
        if (ringA && (j & 1) != team) continue;
        const int sl = sbase + j % nslot;
        const int64_t g = gid(i);                  // global group (batch-major)
        const int b = (int)(g / A.groups);
        const int64_t gg = g % A.groups;
        const int64_t sys0 = gg * W + q * SYS;     // first system of this warp

        if (corr) {
            // ======== P2: x = y + RF Fin + RB Bin (- Z x_l); the inflows are fetched
            // before the tile wait so their L2 latency overlaps it
            if (lane == 0) {
                const int *fl = A.sc.flag + g;
                while (ld_relaxed(fl) == 0) __nanosleep(32);
                fence_acq_rel_gpu();
            }
            __syncwarp();
            PB_TR(3);
            T in[6];   // lane l: value (l % 6) of system l / 6 (SYS * 6 <= 48 values)
            if (lane < 4 * SYS) {
                const int s_ = lane / 4, c_ = lane % 4;
                ws[WS_FIN0 + c_][s_] = __ldcg(A.sc.inf + ((g * nrb + rb) * W + q * SYS + s_) * 4 + c_);
            }
            if (PER) {
                for (int e = lane; e < 2 * SYS; e += 32) {
                    const int s_ = e / 2, c_ = e % 2;
                    ws[WS_XL0 + c_][s_] = __ldcg(A.sc.xl + (g * W + q * SYS + s_) * 2 + c_);
                }
            }
            (void)in;
            PB_TR(0);
            mbar_wait(&sm.full[sl], (j / nslot) & 1);
            PB_TR(1);
            T v[MR][SYS];
#pragma unroll
            for (int k = 0; k < MR; ++k) ld_row(sm.slot[sl], p * MR + k, q, v[k]);
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.empty[sl]);
            T F0[SYS], F1[SYS], B0[SYS], B1[SYS], X0[SYS], X1[SYS];
#pragma unroll
            for (int s = 0; s < SYS; ++s) {
                F0[s] = ws[WS_FIN0][s], F1[s] = ws[WS_FIN1][s];
                B0[s] = ws[WS_BIN0][s], B1[s] = ws[WS_BIN1][s];
                if (PER) X0[s] = ws[WS_XL0][s], X1[s] = ws[WS_XL1][s];
            }
#pragma unroll
            for (int k = 0; k < MR; ++k) {
                const T rf0 = sm.rsp[0][k][p], rf1 = sm.rsp[1][k][p], rb0 = sm.rsp[2][k][p], rb1 = sm.rsp[3][k][p];
                T z1 = T(0), z2 = T(0);
                if (PER) z1 = sm.coef[5][k][p], z2 = sm.coef[6][k][p];
                const int64_t r = r0 + k;
#pragma unroll
                for (int s = 0; s < SYS; ++s) {
                    T o = v[k][s] + rf0 * F0[s] + rf1 * F1[s] + rb0 * B0[s] + rb1 * B1[s];
                    if (PER) {
                        o -= z1 * X0[s];
                        if (K == 2) {
                            o -= z2 * X1[s];
                            if (r == A.n - 2) o = X0[s];
                            if (r == A.n - 1) o = X1[s];
                        }
                    }
                    v[k][s] = o;
                }
            }
            PB_TR(4);
            int64_t Mo = A.M;
            asm volatile("" : "+l"(Mo));
            T *dst = A.x + (int64_t)b * A.bstride + r0 * Mo + sys0;
            const bool full_w = sys0 + SYS <= Mo;
#pragma unroll
            for (int k = 0; k < MR; ++k) {
                if (r0 + k >= A.n) break;
                T *d = dst + k * Mo;
                if (full_w) {
                    st_row<true>(d, v[k]);
                } else {
#pragma unroll
                    for (int s = 0; s < SYS; ++s)
                        if (sys0 + s < Mo) __stcs(d + s, v[k][s]);
                }
            }
            PB_TR(7);
            __syncwarp();   // ws reused by the next item
            continue;
        }

        // ======== P1 (two-phase) or a complete single-tile solve
        PB_TR(0);
        mbar_wait(&sm.full[sl], (j / nslot) & 1);
        PB_TR(1);
        T v[MR][SYS];
#pragma unroll
        for (int k = 0; k < MR; ++k) ld_row(sm.slot[sl], p * MR + k, q, v[k]);
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[sl]);   // this warp's part is in registers

        // ---- 1. forward sweep, zero inflow -> chunk carry; 2. lane scan
        T c0[SYS], c1[SYS];
#pragma unroll
        for (int s = 0; s < SYS; ++s) c0[s] = c1[s] = T(0);
#pragma unroll
        for (int k = 0; k < MR; ++k) {
            const T f0 = sm.coef[0][k][p], f1 = sm.coef[1][k][p], f2 = sm.coef[2][k][p];
#pragma unroll
            for (int s = 0; s < SYS; ++s) {
                T gv = f0 * v[k][s];
                if (K == 2) gv -= f2 * c0[s];
                gv -= f1 * c1[s];
                c0[s] = c1[s];
                c1[s] = gv;
            }
        }
        warp_scan<T, SYS, false>(c0, c1, p, tab, TAB_PF);
        PB_TR(2);
        T *ag = A.sc.agg + ((g * nrb + rb) * W + q * SYS) * 4;
        if (two && p == 31) {
            // A_f: the tile's forward carry with zero tile inflow
#pragma unroll
            for (int s = 0; s < SYS; ++s) {
                ag[s * 4 + 0] = c0[s];
                ag[s * 4 + 1] = c1[s];
            }
        }
        // ---- 3. forward sweep with the chunk inflow (zero tile inflow): v <- g
        {
            T y0[SYS], y1[SYS];
#pragma unroll
            for (int s = 0; s < SYS; ++s) {
                y0[s] = __shfl_up_sync(0xffffffffu, c0[s], 1);
                y1[s] = __shfl_up_sync(0xffffffffu, c1[s], 1);
                if (p == 0) y0[s] = y1[s] = T(0);
            }
#pragma unroll
            for (int k = 0; k < MR; ++k) {
                const T f0 = sm.coef[0][k][p], f1 = sm.coef[1][k][p], f2 = sm.coef[2][k][p];
#pragma unroll
                for (int s = 0; s < SYS; ++s) {
                    T gv = f0 * v[k][s];
                    if (K == 2) gv -= f2 * y0[s];
                    gv -= f1 * y1[s];
                    y0[s] = y1[s];
                    y1[s] = gv;
                    v[k][s] = gv;
                }
            }
        }
        // forward values on the spec rows (two-phase: zero tile inflow, to the
        // group scan; single tile: final, for the local periodic pair)
        if (PER) {
#pragma unroll
            for (int jx = 0; jx < 4; ++jx) {
                const int64_t sr = A.tb.srow[jx];
                const bool here = sr >= row0 && sr < row0 + R;   // warp-uniform
                if (here) {
                    const int owner = (int)((sr - row0) / MR), kx = (int)((sr - row0) % MR);
                    if (lane == owner) {
#pragma unroll
                        for (int s = 0; s < SYS; ++s) {
                            T val = T(0);
#pragma unroll
                            for (int k2 = 0; k2 < MR; ++k2)
                                if (k2 == kx) val = v[k2][s];
                            if (two)
                                A.sc.spec[(g * W + q * SYS + s) * 4 + jx] = val;
                            else
                                ws[WS_SP + jx][s] = val;
                        }
                    }
                }
            }
        }
        // ---- 4. back substitution, zero inflow -> chunk carry; 5. reverse lane scan
#pragma unroll
        for (int s = 0; s < SYS; ++s) c0[s] = c1[s] = T(0);
#pragma unroll
        for (int k = MR - 1; k >= 0; --k) {
            const T b1 = sm.coef[3][k][p], b2 = sm.coef[4][k][p];
#pragma unroll
            for (int s = 0; s < SYS; ++s) {
                T xx = v[k][s];
                if (K == 2) xx -= b2 * c1[s];
                xx -= b1 * c0[s];
                c1[s] = c0[s];
                c0[s] = xx;
            }
        }
        warp_scan<T, SYS, true>(c0, c1, p, tab, TAB_PB);
        if (two && p == 0) {
            // A_b: the tile's backward carry (chunk 0) with zero tile inflows
#pragma unroll
            for (int s = 0; s < SYS; ++s) {
                ag[s * 4 + 2] = c0[s];
                ag[s * 4 + 3] = c1[s];
            }
        }
        // single tile, cyclic: y = (x_0, x_1) is lane 0's inclusive carry
        if (PER && !two) {
            __syncwarp();
            if (lane == 0) {
#pragma unroll
                for (int s = 0; s < SYS; ++s) {
                    T spp[4] = {ws[WS_SP][s], ws[WS_SP + 1][s], ws[WS_SP + 2][s], ws[WS_SP + 3][s]};
                    T a0, a1;
                    local_xl<T, K>(A.tb.scal, c0[s], c1[s], spp, a0, a1);
                    ws[WS_XL0][s] = a0;
                    ws[WS_XL1][s] = a1;
                }
            }
            __syncwarp();
        }
        // ---- 6. back substitution with the chunk inflow (zero tile inflow)
        {
            T z0[SYS], z1[SYS], xl0[SYS], xl1[SYS];
#pragma unroll
            for (int s = 0; s < SYS; ++s) {
                z0[s] = __shfl_down_sync(0xffffffffu, c0[s], 1);
                z1[s] = __shfl_down_sync(0xffffffffu, c1[s], 1);
                if (p == 31) z0[s] = z1[s] = T(0);
                if (PER && !two) xl0[s] = ws[WS_XL0][s], xl1[s] = ws[WS_XL1][s];
            }
#pragma unroll
            for (int k = MR - 1; k >= 0; --k) {
                const T b1 = sm.coef[3][k][p], b2 = sm.coef[4][k][p];
                T zz1 = T(0), zz2 = T(0);
                if (PER && !two) zz1 = sm.coef[5][k][p], zz2 = sm.coef[6][k][p];
                const int64_t r = r0 + k;
#pragma unroll
                for (int s = 0; s < SYS; ++s) {
                    T xx = v[k][s];
                    if (K == 2) xx -= b2 * z1[s];
                    xx -= b1 * z0[s];
                    z1[s] = z0[s];
                    z0[s] = xx;
                    if (PER && !two) {
                        T o = xx - zz1 * xl0[s];
                        if (K == 2) {
                            o -= zz2 * xl1[s];
                            if (r == A.n - 2) o = xl0[s];
                            if (r == A.n - 1) o = xl1[s];
                        }
                        v[k][s] = o;
                    } else {
                        v[k][s] = xx;
                    }
                }
            }
        }
        PB_TR(4);
        // ---- store: the local solution (two-phase, kept in L2 for P2) or x
        {
            int64_t Mo = A.M;
            asm volatile("" : "+l"(Mo));
            T *dst = A.x + (int64_t)b * A.bstride + r0 * Mo + sys0;
            const bool full_w = sys0 + SYS <= Mo;
#pragma unroll
            for (int k = 0; k < MR; ++k) {
                if (r0 + k >= A.n) break;
                T *d = dst + k * Mo;
                if (full_w) {
                    if (two)
                        st_row<false>(d, v[k]);
                    else
                        st_row<true>(d, v[k]);
                } else {
#pragma unroll
                    for (int s = 0; s < SYS; ++s)
                        if (sys0 + s < Mo) d[s] = v[k][s];
                }
            }
        }
        if (two) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.done[i % DONE_Q]);   // P1 tile i: this warp's stores are issued
        }
        PB_TR(7);
        __syncwarp();   // ws reused by the next item
    }
}

}  // namespace pb

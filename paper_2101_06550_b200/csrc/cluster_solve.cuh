// cluster_solve.cuh — the shared-LHS batched banded solve for the interleaved
// layout (pent_solve / tri_solve; cyclic: Navon
// P:1585-1620 / Sherman–Morrison P:2332-2385) as a persistent thread-block-
// cluster kernel for sm_100a.
//
// A cluster of C CTAs owns one group of W systems at a time (W*8 B = 128 B
// per row in fp64, W = 32 systems in fp32); CTA c holds rows [512c, 512c+512)
// of the group in shared memory (64 KB).  Per group:
//   sweep 1  forward, zero inflow          -> chunk carries (16 chunks of 32 rows)
//   exchange 1 (DSMEM): CTA aggregates     -> every chunk's true forward inflow
//   sweep 2  forward with inflow, g in place
//   sweep 3  back substitution, zero inflow -> chunk carries
//   exchange 2 (DSMEM): CTA aggregates, spec rows -> true backward inflows, x_l
//   sweep 4  back substitution with inflow (+ cyclic correction), x in place
// then one TMA store writes x.  Each thread owns one (system, chunk) pair and
// runs the thesis's per-system recurrence over its 32 rows:
// 12 FP64 ops per unknown, no warp scans.  Three 64 KB buffers per CTA: while
// one group is solved, the next two are in flight (TMA), which is what the
// HBM needs (~100 KB in flight per SM).  The group never
// leaves the chip between its load and its store: 16 B of HBM traffic per
// unknown (fp64), the algorithmic minimum.
#pragma once
#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "band_core.cuh"

namespace pb {
namespace clu {

constexpr int RC = 512;      // rows per CTA
constexpr int MR = 32;       // rows per chunk
constexpr int PC = RC / MR;  // chunks per CTA (16)
constexpr int NB = 2;        // group buffers per CTA
constexpr int MAXC = 16;     // cluster size limit (non-portable above 8)

template <typename T>
struct Geom {
    static constexpr int W = sizeof(T) == 8 ? 16 : 32;   // systems per group: 128-byte rows
    static constexpr int NT = PC * W;                     // consumer threads (one per system x chunk)
};

template <typename T>
__host__ __device__ constexpr int W_OF() { return Geom<T>::W; }

template <typename T>
struct Smem {
    static constexpr int W = Geom<T>::W;
    static constexpr int PAIRS = PC / 2;
    T buf[NB][RC * W];          // group buffers (TMA destination / source)
    // coefficient rows of this CTA, chunk pairs interleaved: the two chunks a
    // fp64 warp spans read adjacent 16-byte words (one wavefront per load)
    T cF[MR][PAIRS][2][2];      // (F0, F1) of row k of chunk 2w+h
    T cB[MR][PAIRS][2][2];      // (B1, B2)
    T cF2[MR][PAIRS][2];        // F2
    T cf[PC][W][2];             // chunk carries
    T agg[W][2];                // this CTA's aggregate (to the peers); later the cyclic pair x_l
    T aggF[MAXC][W][2];         // exchange 1: CTA forward aggregates (written by peers)
    T aggB[MAXC][W][2];         // exchange 2: CTA backward aggregates
    T spec[4][W];               // exchange 2: forward values on the cyclic rows (from their owner)
    T mf[PC][4], mb[PC][4];     // chunk transfer matrices
    T mfc[MAXC][4], mbc[MAXC][4];   // CTA block transfer matrices
    alignas(16) T z[RC][2];               // cyclic correction vectors Z1, Z2 of this CTA's rows
    // transfer-matrix products (prologue) turning every fold into independent
    // 2x2 mat-vecs: TF[p][j] = Mf_{p-1} .. Mf_j (j <= p), TB[p][j] = Mb_p .. Mb_{j-1} (j >= p)
    T TF[PC + 1][PC + 1][4];
    T TB[PC + 1][PC + 1][4];
    // CTA level, for this CTA c
    T pcf[MAXC][4];             // Mfc_{c-1} .. Mfc_{c'+1}  (aggF of c' < c -> inflow of c)
    T pcb[MAXC][4];             // Mbc_{c+1} .. Mbc_{c'-1}  (aggB of c' > c -> inflow of c)
    T pcy[MAXC][4];             // Mbc_0 .. Mbc_{c'-1}      (aggB of c' -> x_0, x_1)
    uint64_t full[NB], empty[NB];
    uint64_t xf, xb;            // exchange barriers (C remote arrivals each)
};

template <typename T>
struct Args {
    const T *coef;              // rows_alloc x 8 (band_core.cuh layout)
    const T *cc;                // rows_alloc x 5 compact sweep coefficients (F0 F1 F2 B1 B2), read via L1
    const T *mf, *mb;           // per chunk (C*PC) x 4
    const T *mfc, *mbc;         // per CTA C x 4
    const double *scal;         // SCAL_LEN
    int64_t srow[4];
    int64_t n, M, bstride, groups;
    int count, C, ncl;
    T *x;
    unsigned long long *trace;   // dev timeline [cta][group<256][8] (nullptr = off)
};
__device__ __forceinline__ unsigned long long clu_gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define CLU_TR2(k)                                                                       \
    do {                                                                                 \
        if (A.trace && t < 256) A.trace[((int64_t)blockIdx.x * 256 + t) * 16 + (k)] = clu_gtimer(); \
    } while (0)
#define CLU_TR(k)                                                                        \
    do {                                                                                 \
        if (A.trace && tid == 0 && t < 256) A.trace[((int64_t)blockIdx.x * 256 + t) * 16 + (k)] = clu_gtimer(); \
    } while (0)

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

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
        "LAB_WAIT:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra LAB_WAIT;\n}" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
// wait with cluster-scope acquire (peers' DSMEM writes before their release-arrive)
__device__ __forceinline__ void bar_wait_cluster(uint64_t *b, uint32_t parity)
{
    asm volatile(
        "{\n .reg .pred p;\n"
        "LAB_WAITC:\n"
        " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra LAB_WAITC;\n}" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
// release-arrive on the same barrier in CTA `rank` of the cluster
__device__ __forceinline__ void bar_arrive_remote(uint64_t *b, uint32_t rank)
{
    asm volatile(
        "{\n .reg .b32 ra;\n"
        " mapa.shared::cluster.u32 ra, %0, %1;\n"
        " mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n}" ::"r"(su32(b)),
        "r"(rank)
        : "memory");
}
__device__ __forceinline__ void bar_arrive_remote_relaxed(uint64_t *b, uint32_t rank)
{
    asm volatile(
        "{\n .reg .b32 ra;\n"
        " mapa.shared::cluster.u32 ra, %0, %1;\n"
        " mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [ra];\n}" ::"r"(su32(b)),
        "r"(rank)
        : "memory");
}
__device__ __forceinline__ void fence_acq_rel_cluster() { asm volatile("fence.acq_rel.cluster;" ::: "memory"); }
template <typename T>
__device__ __forceinline__ void st_remote(T *p, uint32_t rank, T v);
template <>
__device__ __forceinline__ void st_remote<double>(double *p, uint32_t rank, double v)
{
    asm volatile(
        "{\n .reg .b32 ra;\n"
        " mapa.shared::cluster.u32 ra, %0, %1;\n"
        " st.shared::cluster.f64 [ra], %2;\n}" ::"r"(su32(p)),
        "r"(rank), "d"(v)
        : "memory");
}
template <>
__device__ __forceinline__ void st_remote<float>(float *p, uint32_t rank, float v)
{
    asm volatile(
        "{\n .reg .b32 ra;\n"
        " mapa.shared::cluster.u32 ra, %0, %1;\n"
        " st.shared::cluster.f32 [ra], %2;\n}" ::"r"(su32(p)),
        "r"(rank), "f"(v)
        : "memory");
}
__device__ __forceinline__ void tma_load(void *dst, const CUtensorMap *m, int c0, int c1, int c2, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            su32(dst)),
        "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(su32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store(const CUtensorMap *m, int c0, int c1, int c2, const void *src)
{
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(m), "r"(c0),
                 "r"(c1), "r"(c2), "r"(su32(src))
                 : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// y <- c + M y
template <typename T>
__device__ __forceinline__ void aff(T &y0, T &y1, T c0, T c1, const T *m)
{
    const T n0 = c0 + m[0] * y0 + m[1] * y1;
    const T n1 = c1 + m[2] * y0 + m[3] * y1;
    y0 = n0;
    y1 = n1;
}

// a += m x (2x2 mat-vec accumulate)
template <typename T>
__device__ __forceinline__ void mva(T &a0, T &a1, const T *m, T x0, T x1)
{
    a0 += m[0] * x0 + m[1] * x1;
    a1 += m[2] * x0 + m[3] * x1;
}

// read-only global load the compiler keeps in program order (bounds the
// register footprint of coefficient prefetching in the unrolled sweeps)
__device__ __forceinline__ double ldc(const double *p)
{
    double v;
    asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ float ldc(const float *p)
{
    float v;
    asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}

// Chunk sweeps over the 32 rows in shared memory (row k at col[k*W]), in
// blocks of 8 rows: the block's loads are issued together, then the
// recurrence runs (one dependent DFMA per row on the carry).
// vector loads of a coefficient row (AoS, 8 per row: F0 F1 F2 - B1 B2 Z1 Z2), L1 resident
__device__ __forceinline__ void ld_f(const double *c, double &f0, double &f1, double &f2)
{
    const double2 a = __ldg(reinterpret_cast<const double2 *>(c));
    f0 = a.x, f1 = a.y, f2 = __ldg(c + 2);
}
__device__ __forceinline__ void ld_f(const float *c, float &f0, float &f1, float &f2)
{
    const float4 a = __ldg(reinterpret_cast<const float4 *>(c));
    f0 = a.x, f1 = a.y, f2 = a.z;
}
__device__ __forceinline__ void ld_b(const double *c, double &b1, double &b2)
{
    const double2 a = __ldg(reinterpret_cast<const double2 *>(c + 4));
    b1 = a.x, b2 = a.y;
}
__device__ __forceinline__ void ld_b(const float *c, float &b1, float &b2)
{
    const float2 a = __ldg(reinterpret_cast<const float2 *>(c + 4));
    b1 = a.x, b2 = a.y;
}

// Chunk sweeps over the 32 rows in shared memory (row k at col[k*W]), in
// blocks of 8 rows: the block's loads are issued together, then the
// recurrence runs (one dependent DFMA per row on the carry).
template <typename T, int K, bool STORE>
__device__ __forceinline__ void fwd_blocks(T *col, const T *cr, T &y0, T &y1)
{
#pragma unroll 1
    for (int k0 = 0; k0 < MR; k0 += 8) {
        T a[8], c1[8], c2[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            T f0;
            ld_f(cr + (k0 + k) * COEF_STRIDE, f0, c1[k], c2[k]);
            a[k] = f0 * col[(k0 + k) * W_OF<T>()];
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            T gv = a[k];
            if (K == 2) gv -= c2[k] * y0;
            gv -= c1[k] * y1;
            y0 = y1;
            y1 = gv;
            if (STORE) col[(k0 + k) * W_OF<T>()] = gv;
        }
    }
}
template <typename T, int K, bool STORE>
__device__ __forceinline__ void bwd_blocks(T *col, const T *cr, T &z0, T &z1)
{
#pragma unroll 1
    for (int k0 = MR - 8; k0 >= 0; k0 -= 8) {
        T gk[8], b1[8], b2[8];
#pragma unroll
        for (int k = 7; k >= 0; --k) {
            gk[k] = col[(k0 + k) * W_OF<T>()];
            ld_b(cr + (k0 + k) * COEF_STRIDE, b1[k], b2[k]);
        }
#pragma unroll
        for (int k = 7; k >= 0; --k) {
            T xx = gk[k];
            if (K == 2) xx -= b2[k] * z1;
            xx -= b1[k] * z0;
            z1 = z0;
            z0 = xx;
            if (STORE) col[(k0 + k) * W_OF<T>()] = xx;
        }
    }
}

// R = A B (row-major 2x2)
template <typename T>
__device__ __forceinline__ void mm(const T *a, const T *b, T *r)
{
    const T r0 = a[0] * b[0] + a[1] * b[2], r1 = a[0] * b[1] + a[1] * b[3];
    const T r2 = a[2] * b[0] + a[3] * b[2], r3 = a[2] * b[1] + a[3] * b[3];
    r[0] = r0, r[1] = r1, r[2] = r2, r[3] = r3;
}
template <typename T>
__device__ __forceinline__ void set_id(T *r) { r[0] = T(1), r[1] = T(0), r[2] = T(0), r[3] = T(1); }

// shared loads the compiler keeps in program order (bounds the register
// footprint of the coefficient prefetch in the fully unrolled sweeps)
__device__ __forceinline__ void lds2(const double *p, double &a, double &b)
{
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b) : "r"(su32(p)));
}
__device__ __forceinline__ void lds2(const float *p, float &a, float &b)
{
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(a), "=f"(b) : "r"(su32(p)));
}
__device__ __forceinline__ double lds1(const double *p)
{
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(su32(p)));
    return v;
}
__device__ __forceinline__ float lds1(const float *p)
{
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(su32(p)));
    return v;
}

template <typename T, int K, bool PER>
__global__ void __launch_bounds__(Geom<T>::NT + 32, 1) cluster_solve_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                           const Args<T> A)
{
    namespace cg = cooperative_groups;
    constexpr int W = Geom<T>::W, NT = Geom<T>::NT;
    constexpr uint32_t BYTES = (uint32_t)(RC * W * sizeof(T));
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem<T> &sm = *reinterpret_cast<Smem<T> *>(smem_raw);
    const int tid = threadIdx.x;
    const int C = A.C;
    const uint32_t c = C > 1 ? cg::this_cluster().block_rank() : 0;
    const int cl = blockIdx.x / C;                  // cluster index
    const int64_t gt = A.groups * A.count;
    const int ng = (int)((gt - cl + A.ncl - 1) / A.ncl);   // groups of this cluster: cl + ncl*t
    const int64_t row0 = (int64_t)c * RC;

    if (tid == 0) {
        for (int b = 0; b < NB; ++b) {
            bar_init(&sm.full[b], 1);
            bar_init(&sm.empty[b], 1);
        }
        bar_init(&sm.xf, C);
        bar_init(&sm.xb, C);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int e = tid; e < RC; e += blockDim.x) {
        const int pp = e / MR, k = e % MR, w = pp / 2, h = pp % 2;
        const T *cr = A.coef + (row0 + e) * COEF_STRIDE;
        sm.cF[k][w][h][0] = cr[0];
        sm.cF[k][w][h][1] = cr[1];
        sm.cF2[k][w][h] = cr[2];
        sm.cB[k][w][h][0] = cr[4];
        sm.cB[k][w][h][1] = cr[5];
    }
    for (int e = tid; e < PC * 4; e += blockDim.x) {
        sm.mf[e / 4][e % 4] = A.mf[((int64_t)c * PC) * 4 + e];
        sm.mb[e / 4][e % 4] = A.mb[((int64_t)c * PC) * 4 + e];
    }
    for (int e = tid; e < C * 4; e += blockDim.x) {
        sm.mfc[e / 4][e % 4] = A.mfc[e];
        sm.mbc[e / 4][e % 4] = A.mbc[e];
    }
    for (int e = tid; e < RC * 2; e += blockDim.x) sm.z[e / 2][e % 2] = A.coef[(row0 + e / 2) * COEF_STRIDE + 6 + e % 2];
    __syncthreads();
    if (tid <= PC) {
        const int pp = tid;
        T m[4];
        set_id(m);
        for (int j = 0; j < 4; ++j) sm.TF[pp][pp][j] = m[j];
        for (int j = pp - 1; j >= 0; --j) {
            mm(m, sm.mf[j], m);
            for (int e = 0; e < 4; ++e) sm.TF[pp][j][e] = m[e];
        }
    } else if (tid >= 32 && tid <= 32 + PC) {
        const int pp = tid - 32;
        T m[4];
        set_id(m);
        for (int j = 0; j < 4; ++j) sm.TB[pp][pp][j] = m[j];
        for (int j = pp + 1; j <= PC; ++j) {
            mm(m, sm.mb[j - 1], m);
            for (int e = 0; e < 4; ++e) sm.TB[pp][j][e] = m[e];
        }
    } else if (tid == 64) {
        T m[4];
        set_id(m);
        for (int cc = (int)c - 1; cc >= 0; --cc) {
            for (int j = 0; j < 4; ++j) sm.pcf[cc][j] = m[j];
            mm(m, sm.mfc[cc], m);
        }
        set_id(m);
        for (int cc = (int)c + 1; cc < C; ++cc) {
            for (int j = 0; j < 4; ++j) sm.pcb[cc][j] = m[j];
            mm(m, sm.mbc[cc], m);
        }
    } else if (tid == 96) {
        T m[4];
        set_id(m);
        for (int cc = 0; cc < C; ++cc) {
            for (int j = 0; j < 4; ++j) sm.pcy[cc][j] = m[j];
            mm(m, sm.mbc[cc], m);
        }
    }
    __syncthreads();
    if (C > 1) cg::this_cluster().sync();   // peers' barriers initialised before any remote arrive

    auto coords = [&](int t, int &c0, int &c2) {
        const int64_t g = cl + (int64_t)A.ncl * t;
        c2 = (int)(g / A.groups);
        c0 = (int)(g % A.groups) * W;
    };

    // ================= producer warp: TMA loads, NB groups deep
    if (tid >= NT) {
        if (tid != NT) return;
        for (int t = 0; t < ng; ++t) {
            const int b = t % NB;
            if (t >= NB) bar_wait(&sm.empty[b], ((t / NB) - 1) & 1);
            int c0, c2;
            coords(t, c0, c2);
            bar_expect_tx(&sm.full[b], BYTES);
            tma_load(sm.buf[b], &tmap, c0, (int)row0, c2, &sm.full[b]);
            tma_load(sm.buf[b] + 256 * W, &tmap, c0, (int)row0 + 256, c2, &sm.full[b]);
        }
        return;
    }

    // ================= consumers: thread = (chunk p, system s); its 32 values live in registers
    const int s = tid % W, p = tid / W;
    const int pw = p / 2, ph2 = p % 2;                 // coefficient pair slot
    const int k0 = p * MR;                             // first row of the chunk in the CTA
    int pend = -1;                                     // buffer whose TMA store is pending
    for (int t = 0; t < ng; ++t) {
        const int b = t % NB;
        const uint32_t ph = t & 1;
        CLU_TR(0);
        if (tid == 0 && pend >= 0) {
            // the previous group's TMA store has finished reading its buffer
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            bar_arrive(&sm.empty[pend]);
        }
        bar_wait(&sm.full[b], (t / NB) & 1);
        CLU_TR(1);
        T *col = sm.buf[b] + s + k0 * W;   // row k of the chunk at col[k * W]
        T v[MR];
#pragma unroll
        for (int k = 0; k < MR; ++k) v[k] = col[k * W];
        CLU_TR(8);

        // ---- sweep 1: forward, zero inflow -> chunk carry
        {
            T y0 = T(0), y1 = T(0);
#pragma unroll
            for (int k = 0; k < MR; ++k) {
                T f0, f1;
                lds2(sm.cF[k][pw][ph2], f0, f1);
                T gv = f0 * v[k];
                if (K == 2) gv -= lds1(&sm.cF2[k][pw][ph2]) * y0;
                gv -= f1 * y1;
                y0 = y1;
                y1 = gv;
            }
            sm.cf[p][s][0] = y0;
            sm.cf[p][s][1] = y1;
        }
        CLU_TR(9);
        named_sync(1, NT);
        // ---- exchange 1: this CTA's forward aggregate to every peer
        if (p == 0) {
            T a0 = T(0), a1 = T(0);
            T e0 = T(0), e1 = T(0);
#pragma unroll
            for (int q = 0; q < PC; q += 2) {
                mva(a0, a1, sm.TF[PC][q + 1], sm.cf[q][s][0], sm.cf[q][s][1]);
                mva(e0, e1, sm.TF[PC][q + 2], sm.cf[q + 1][s][0], sm.cf[q + 1][s][1]);
            }
            a0 += e0;
            a1 += e1;
            sm.agg[s][0] = a0;
            sm.agg[s][1] = a1;
        }
        named_sync(1, NT);
        CLU_TR(10);
        if (p < C) {
            st_remote(&sm.aggF[c][s][0], (uint32_t)p, sm.agg[s][0]);
            st_remote(&sm.aggF[c][s][1], (uint32_t)p, sm.agg[s][1]);
        }
        named_sync(1, NT);
        // one cluster-scope fence (covers this CTA's DSMEM stores through the
        // CTA barrier above), then relaxed arrives on every peer's barrier
        if (tid == 0) {
            fence_acq_rel_cluster();
            for (int r = 0; r < C; ++r) bar_arrive_remote_relaxed(&sm.xf, (uint32_t)r);
            CLU_TR(2);
            bar_wait_cluster(&sm.xf, ph);   // one cluster-scope acquire, then a CTA barrier
            CLU_TR(3);
        }
        named_sync(1, NT);
        // ---- sweep 2: forward with the true inflow: v <- g
        {
            T y0 = T(0), y1 = T(0);
            {
                T u0 = T(0), u1 = T(0);
                for (int cc = 0; cc < (int)c; ++cc) mva(u0, u1, sm.pcf[cc], sm.aggF[cc][s][0], sm.aggF[cc][s][1]);
                mva(y0, y1, sm.TF[p][0], u0, u1);
                T e0 = T(0), e1 = T(0);
#pragma unroll
                for (int q = 0; q < PC - 1; ++q)
                    if (q < p) {
                        if (q & 1) mva(e0, e1, sm.TF[p][q + 1], sm.cf[q][s][0], sm.cf[q][s][1]);
                        else mva(y0, y1, sm.TF[p][q + 1], sm.cf[q][s][0], sm.cf[q][s][1]);
                    }
                y0 += e0;
                y1 += e1;
            }
            if (p == PC - 1 && s == 0) CLU_TR2(11);
#pragma unroll
            for (int k = 0; k < MR; ++k) {
                T f0, f1;
                lds2(sm.cF[k][pw][ph2], f0, f1);
                T gv = f0 * v[k];
                if (K == 2) gv -= lds1(&sm.cF2[k][pw][ph2]) * y0;
                gv -= f1 * y1;
                y0 = y1;
                y1 = gv;
                v[k] = gv;
            }
        }
        if (p == PC - 1 && s == 0) CLU_TR2(12);
        named_sync(1, NT);   // cf is rewritten below
        // ---- sweep 3: back substitution, zero inflow -> chunk carry
        {
            T z0 = T(0), z1 = T(0);
#pragma unroll
            for (int k = MR - 1; k >= 0; --k) {
                T b1, b2;
                lds2(sm.cB[k][pw][ph2], b1, b2);
                T xx = v[k];
                if (K == 2) xx -= b2 * z1;
                xx -= b1 * z0;
                z1 = z0;
                z0 = xx;
            }
            sm.cf[p][s][0] = z0;
            sm.cf[p][s][1] = z1;
        }
        // (cyclic) forward values on the spec rows (g in v): owner thread -> every peer
        if (PER) {
#pragma unroll
            for (int jx = 0; jx < 4; ++jx) {
                const int64_t sr = A.srow[jx] - row0 - k0;
                if (A.srow[jx] >= 0 && sr >= 0 && sr < MR) {
                    T val = T(0);
#pragma unroll
                    for (int k = 0; k < MR; ++k)
                        if (k == sr) val = v[k];
                    for (int r = 0; r < C; ++r) st_remote(&sm.spec[jx][s], (uint32_t)r, val);
                }
            }
        }
        named_sync(1, NT);
        if (p == 0) {
            T a0 = T(0), a1 = T(0);
            T e0 = T(0), e1 = T(0);
#pragma unroll
            for (int q = 0; q < PC; q += 2) {
                mva(a0, a1, sm.TB[0][q], sm.cf[q][s][0], sm.cf[q][s][1]);
                mva(e0, e1, sm.TB[0][q + 1], sm.cf[q + 1][s][0], sm.cf[q + 1][s][1]);
            }
            a0 += e0;
            a1 += e1;
            sm.agg[s][0] = a0;
            sm.agg[s][1] = a1;
        }
        named_sync(1, NT);
        // ---- exchange 2
        if (p < C) {
            st_remote(&sm.aggB[c][s][0], (uint32_t)p, sm.agg[s][0]);
            st_remote(&sm.aggB[c][s][1], (uint32_t)p, sm.agg[s][1]);
        }
        named_sync(1, NT);
        // one cluster-scope fence (covers this CTA's DSMEM stores through the
        // CTA barrier above), then relaxed arrives on every peer's barrier
        if (tid == 0) {
            fence_acq_rel_cluster();
            for (int r = 0; r < C; ++r) bar_arrive_remote_relaxed(&sm.xb, (uint32_t)r);
            CLU_TR(4);
            bar_wait_cluster(&sm.xb, ph);
            CLU_TR(5);
        }
        named_sync(1, NT);
        if (PER) {
            // y = (x_0, x_1): the backward composition of every CTA; then the 2x2
            if (p == 0) {
                T y1 = T(0), y2 = T(0);
                for (int cc = 0; cc < C; ++cc) mva(y1, y2, sm.pcy[cc], sm.aggB[cc][s][0], sm.aggB[cc][s][1]);
                const double *sc = A.scal;
                T xl0, xl1;
                if (K == 2) {
                    // Navon (eq:first_two)
                    const T ym1 = sm.spec[1][s], ym2 = sm.spec[0][s] - T(sc[10]) * sm.spec[1][s];
                    const T q0 = sm.spec[2][s] - (T(sc[4]) * y1 + T(sc[5]) * ym2 + T(sc[6]) * ym1);
                    const T q1 = sm.spec[3][s] - (T(sc[7]) * y1 + T(sc[8]) * y2 + T(sc[9]) * ym1);
                    xl0 = T(sc[0]) * q0 + T(sc[1]) * q1;
                    xl1 = T(sc[2]) * q0 + T(sc[3]) * q1;
                } else {
                    // Sherman–Morrison
                    xl0 = (y1 + T(sc[0]) * sm.spec[0][s]) / T(sc[1]);
                    xl1 = T(0);
                }
                sm.agg[s][0] = xl0;   // agg is free after exchange 2
                sm.agg[s][1] = xl1;
            }
            named_sync(1, NT);
        }
        // ---- sweep 4: back substitution with the true inflow (+ cyclic correction), x -> buffer
        {
            T z0 = T(0), z1 = T(0);
            {
                T u0 = T(0), u1 = T(0);
                for (int cc = (int)c + 1; cc < C; ++cc) mva(u0, u1, sm.pcb[cc], sm.aggB[cc][s][0], sm.aggB[cc][s][1]);
                mva(z0, z1, sm.TB[p + 1][PC], u0, u1);
                T e0 = T(0), e1 = T(0);
#pragma unroll
                for (int q = 1; q < PC; ++q)
                    if (q > p) {
                        if (q & 1) mva(e0, e1, sm.TB[p + 1][q], sm.cf[q][s][0], sm.cf[q][s][1]);
                        else mva(z0, z1, sm.TB[p + 1][q], sm.cf[q][s][0], sm.cf[q][s][1]);
                    }
                z0 += e0;
                z1 += e1;
            }
            if (p == 0 && s == 0) CLU_TR(13);
#pragma unroll
            for (int k = MR - 1; k >= 0; --k) {
                T b1, b2;
                lds2(sm.cB[k][pw][ph2], b1, b2);
                T xx = v[k];
                if (K == 2) xx -= b2 * z1;
                xx -= b1 * z0;
                z1 = z0;
                z0 = xx;
                v[k] = xx;
            }
            if (p == 0 && s == 0) CLU_TR(14);
            if (PER) {
                // cyclic correction x - Z x_l (Navon eq:solve / Sherman–Morrison)
                const T xl0 = sm.agg[s][0], xl1 = sm.agg[s][1];
                const int64_t rbase = row0 + k0;
#pragma unroll
                for (int k = 0; k < MR; ++k) {
                    T z1v, z2v;
                    lds2(sm.z[k0 + k], z1v, z2v);
                    T o = v[k] - z1v * xl0;
                    if (K == 2) {
                        o -= z2v * xl1;
                        if (rbase + k == A.n - 2) o = xl0;
                        if (rbase + k == A.n - 1) o = xl1;
                    }
                    v[k] = o;
                }
            }
            if (p == 0 && s == 0) CLU_TR(15);
#pragma unroll
            for (int k = 0; k < MR; ++k) col[k * W] = v[k];
        }
        // ---- x out: one TMA store per 256-row box; the buffer is released one group later
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        named_sync(1, NT);
        if (tid == 0) {
            int c0, c2;
            coords(t, c0, c2);
            tma_store(&tmap, c0, (int)row0, c2, sm.buf[b]);
            tma_store(&tmap, c0, (int)row0 + 256, c2, sm.buf[b] + 256 * W);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            CLU_TR(6);
            CLU_TR(7);
        }
        pend = b;
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

}  // namespace clu
}  // namespace pb

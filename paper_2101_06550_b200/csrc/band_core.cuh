// band_core.cuh — the partitioned (SPIKE-like) batched banded solve core for
// sm_100a, shared by pent_solve / tri_solve and the fused ADI sweeps.
//
// Method.  The thesis solves each system with one thread
// sweeping all N rows.  On B200 that leaves <2 warps per
// SM at N = M = 8192 and an N-long dependent FMA chain per thread, so here a
// system is split into chunks of MR rows, one chunk per thread:
//   1. forward sweep of the chunk with zero inflow -> 2-value carry;
//   2. carry scan across chunks (smem) and across the CTAs of a thread-block
//      cluster (DSMEM), using the chunk transfer matrices Mf (precomputed
//      once per LHS: they depend only on the shared factors);
//   3. forward sweep again with the true inflow (g of P:1712-1716);
//   4-5. the same for the back substitution with Mb;
//   6. periodic correction x = y - Z (x_{N-1}, x_N) (Navon, eq:solve /
//      eq:first_two) or x = y - coef z (Sherman–Morrison,
//      P:2380-2385).
// The whole system stays on chip (registers), so each unknown costs exactly
// one HBM read of f and one HBM write of x — the 16 B/unknown (fp64)
// algorithmic minimum; the thesis's g round trip (32 B) disappears.
//
// Recurrences (per row i, coefficient AoS row of 8 values):
//   g_i = F0_i f_i - F1_i g_{i-1} - F2_i g_{i-2}    F0 = 1/alpha, F1 = beta/alpha, F2 = eps/alpha
//   x_i = g_i - B1_i x_{i+1} - B2_i x_{i+2}         B1 = gamma, B2 = delta
//   periodic: Z1_i, Z2_i = (E^{-1} k)_i (penta) or z_i = (A'^{-1} u)_i (tri)
// Tridiagonal (Thomas): F0 = 1/(b_i - a_i chat_{i-1}),
// F1 = a_i F0, B1 = chat_i, F2 = B2 = 0 (K = 1 drops those terms).
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace pb {
namespace cg = cooperative_groups;

constexpr int COEF_STRIDE = 8;  // F0 F1 F2 - B1 B2 Z1 Z2
constexpr int MAX_CLUSTER = 16;
constexpr int MAX_LOG_PC = 5;    // chunks per CTA (PC) <= 32: one warp segment per system
// per-chunk scan table: Pf[l] (l < 5), Pb[l], PhiF, PhiB — 2x2 row-major each
constexpr int TAB_PF = 0, TAB_PB = 4 * MAX_LOG_PC, TAB_PHIF = 8 * MAX_LOG_PC, TAB_PHIB = 8 * MAX_LOG_PC + 4;
constexpr int TAB_STRIDE = 8 * MAX_LOG_PC + 8;

// scalar parameters of the periodic finalisation (fp64 on device)
//   penta: [0..3] Sinv (row-major 2x2), [4..9] H = (e_{N-1}, a_{N-1}, b_{N-1}, d_N, e_N, a_N),
//          [10] gamma_{m-2} (m = N-2, core size)
//   tri:   [0] v_N = -a_1/b_1, [1] 1 + v.z
constexpr int SCAL_LEN = 12;

template <typename T>
struct CoreArgs {
    const T *coef;          // (rows) x 8, AoS, identity rows beyond the system
    const T *tab;           // per-chunk scan tables (TAB_STRIDE per chunk)
    const T *mfc, *mbc;     // CTA-block transfer matrices, 4 per CTA of the cluster
    const double *scal;     // SCAL_LEN periodic scalars
    int64_t n;              // unknowns per system
    int C;                  // cluster size (CTAs sharing one system group)
    int64_t srow[4];        // rows whose forward value feeds the periodic 2x2 (-1: unused)
};

// Carry buffers are [system][chunk] with one pad column, so both the
// sweep-layout writes (system fastest across lanes) and the scan-layout reads
// (chunk fastest) are bank-conflict free.
template <typename T, int W, int PC>
struct CoreSmem {
    T cf0[W][PC + 1], cf1[W][PC + 1];
    T in0[W][PC + 1], in1[W][PC + 1];
    T aggF[MAX_CLUSTER][W][2];
    T aggB[MAX_CLUSTER][W][2];
    T spec[4][W];
    T xl[W][2];
};

__device__ __forceinline__ void cluster_sync_all() { cg::this_cluster().sync(); }

template <typename T>
__device__ __forceinline__ T *peer(T *p, int rank)
{
    return cg::this_cluster().map_shared_rank(p, rank);
}

// Coefficient rows are read from the CTA's shared-memory copy (stage_coef):
// every lane of a system group reads the same row, so the loads broadcast.
template <typename T>
__device__ __forceinline__ void ldcoef_f(const T *cr, T &f0, T &f1, T &f2)
{
    f0 = cr[0];
    f1 = cr[1];
    f2 = cr[2];
}
template <>
__device__ __forceinline__ void ldcoef_f<double>(const double *cr, double &f0, double &f1, double &f2)
{
    double2 a = *reinterpret_cast<const double2 *>(cr);
    f0 = a.x;
    f1 = a.y;
    f2 = cr[2];
}
template <>
__device__ __forceinline__ void ldcoef_f<float>(const float *cr, float &f0, float &f1, float &f2)
{
    float4 a = *reinterpret_cast<const float4 *>(cr);
    f0 = a.x;
    f1 = a.y;
    f2 = a.z;
}
template <typename T>
__device__ __forceinline__ void ldcoef_b(const T *cr, T &b1, T &b2)
{
    b1 = cr[4];
    b2 = cr[5];
}
template <>
__device__ __forceinline__ void ldcoef_b<double>(const double *cr, double &b1, double &b2)
{
    double2 a = *reinterpret_cast<const double2 *>(cr + 4);
    b1 = a.x;
    b2 = a.y;
}
template <>
__device__ __forceinline__ void ldcoef_b<float>(const float *cr, float &b1, float &b2)
{
    float2 a = *reinterpret_cast<const float2 *>(cr + 4);
    b1 = a.x;
    b2 = a.y;
}
template <typename T>
__device__ __forceinline__ void ldcoef_z(const T *cr, T &z1, T &z2)
{
    z1 = cr[6];
    z2 = cr[7];
}
template <>
__device__ __forceinline__ void ldcoef_z<double>(const double *cr, double &z1, double &z2)
{
    double2 a = *reinterpret_cast<const double2 *>(cr + 6);
    z1 = a.x;
    z2 = a.y;
}
template <>
__device__ __forceinline__ void ldcoef_z<float>(const float *cr, float &z1, float &z2)
{
    float2 a = *reinterpret_cast<const float2 *>(cr + 6);
    z1 = a.x;
    z2 = a.y;
}

// Copy the CTA's rc coefficient rows (global, contiguous) into shared memory.
// Callers synchronise before band_core reads them.
template <typename T, int NT>
__device__ __forceinline__ void stage_coef(T *dst, const T *src, int rc)
{
    const int nvec = rc * COEF_STRIDE * (int)sizeof(T) / 16;
    const int4 *s4 = reinterpret_cast<const int4 *>(src);
    int4 *d4 = reinterpret_cast<int4 *>(dst);
    for (int e = threadIdx.x; e < nvec; e += NT) d4[e] = __ldg(s4 + e);
}


// y <- c + M y  (M row-major 2x2 in global memory)
template <typename T>
__device__ __forceinline__ void affine(T &y0, T &y1, T c0, T c1, const T *M)
{
    T m0 = __ldg(M + 0), m1 = __ldg(M + 1), m2 = __ldg(M + 2), m3 = __ldg(M + 3);
    T n0 = c0 + m0 * y0 + m1 * y1;
    T n1 = c1 + m2 * y0 + m3 * y1;
    y0 = n0;
    y1 = n1;
}

// Segmented inclusive Kogge–Stone scan of affine carries over PC lanes:
// lane q holds the zero-inflow carry of chunk q; at level l,
// b_q += P_{q,l} b_{q-2^l} with P_{q,l} the product of the 2^l chunk
// transfer matrices ending at q (precomputed, LHS-only).
template <typename T, int PC>
__device__ __forceinline__ void seg_scan(T &b0, T &b1, int q, const T *P)
{
#pragma unroll
    for (int l = 0; (1 << l) < PC; ++l) {
        const int d = 1 << l;
        T u0 = __shfl_up_sync(0xffffffffu, b0, d, PC);
        T u1 = __shfl_up_sync(0xffffffffu, b1, d, PC);
        if (q >= d) {
            const T *m = P + 4 * l;
            T m0 = __ldg(m + 0), m1 = __ldg(m + 1), m2 = __ldg(m + 2), m3 = __ldg(m + 3);
            b0 += m0 * u0 + m1 * u1;
            b1 += m2 * u0 + m3 * u1;
        }
    }
}

// The solve core.  v[k] holds f for rows r0 .. r0+MR-1 of system lane s on
// entry and x on exit.  All threads of the CTA (and all CTAs of the cluster)
// must call it.  c = CTA rank in the cluster; r0 = c*PC*MR + p*MR.
// cs = the CTA's coefficient rows in shared memory (stage_coef), row 0 =
// global row c*PC*MR.
template <typename T, int K, int W, int NT, int MR, bool PER>
__device__ __forceinline__ void band_core(T (&v)[MR], const CoreArgs<T> &A, CoreSmem<T, W, NT / W> &S,
                                          const T *cs, int c, int s, int p, int64_t r0)
{
    constexpr int PC = NT / W;
    static_assert(PC <= 32 && (PC & (PC - 1)) == 0, "chunks per CTA must be a power of two <= 32");
    const int tid = threadIdx.x;
    const int C = A.C;
    const T *coef = cs + p * MR * COEF_STRIDE;
    // scan-layout coordinates: system ss, chunk-lane qq (one carry per thread)
    const int ss = tid / PC, qq = tid % PC;
    const T *tab_c = A.tab + (int64_t)c * PC * TAB_STRIDE;

    // ---- 1. forward sweep, zero inflow: carry (g_{r1-2}, g_{r1-1})
    {
        T y0 = T(0), y1 = T(0);
#pragma unroll
        for (int k = 0; k < MR; ++k) {
            T f0, f1, f2;
            ldcoef_f(coef + k * COEF_STRIDE, f0, f1, f2);
            T g = f0 * v[k];
            if (K == 2) g -= f2 * y0;
            g -= f1 * y1;   // newest carry last: one FMA on the chain
            y0 = y1;
            y1 = g;
        }
        S.cf0[s][p] = y0;
        S.cf1[s][p] = y1;
    }
    __syncthreads();
    // ---- 2. forward carry scan: warp segments (chunks), then cluster (DSMEM)
    {
        T b0 = S.cf0[ss][qq], b1 = S.cf1[ss][qq];
        seg_scan<T, PC>(b0, b1, qq, tab_c + qq * TAB_STRIDE + TAB_PF);
        T e0 = __shfl_up_sync(0xffffffffu, b0, 1, PC), e1 = __shfl_up_sync(0xffffffffu, b1, 1, PC);
        if (qq == 0) e0 = e1 = T(0);
        S.in0[ss][qq] = e0;
        S.in1[ss][qq] = e1;
        if (C > 1 && qq == PC - 1)
            for (int rr = 0; rr < C; ++rr) {
                T *pa = peer(&S.aggF[c][ss][0], rr);
                pa[0] = b0;
                pa[1] = b1;
            }
    }
    if (C > 1)
        cluster_sync_all();
    else
        __syncthreads();
    // ---- 3. forward sweep with the true inflow: v <- g
    {
        T y0 = S.in0[s][p], y1 = S.in1[s][p];
        if (C > 1) {
            T Y0 = T(0), Y1 = T(0);
            for (int cc = 0; cc < c; ++cc) affine(Y0, Y1, S.aggF[cc][s][0], S.aggF[cc][s][1], A.mfc + cc * 4);
            const T *phi = tab_c + p * TAB_STRIDE + TAB_PHIF;
            y0 += __ldg(phi + 0) * Y0 + __ldg(phi + 1) * Y1;
            y1 += __ldg(phi + 2) * Y0 + __ldg(phi + 3) * Y1;
        }
#pragma unroll
        for (int k = 0; k < MR; ++k) {
            T f0, f1, f2;
            ldcoef_f(coef + k * COEF_STRIDE, f0, f1, f2);
            T g = f0 * v[k];
            if (K == 2) g -= f2 * y0;
            g -= f1 * y1;   // newest carry last: one FMA on the chain
            y0 = y1;
            y1 = g;
            v[k] = g;
        }
    }
    if (PER) {
        // publish the forward values the periodic 2x2 needs (one owner each)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t k = A.srow[j] - r0;
            if (k >= 0 && k < MR) {
                T val = T(0);
#pragma unroll
                for (int kk = 0; kk < MR; ++kk)
                    if (kk == k) val = v[kk];
                if (C == 1)
                    S.spec[j][s] = val;
                else
                    for (int rr = 0; rr < C; ++rr) *peer(&S.spec[j][s], rr) = val;
            }
        }
    }
    // ---- 4. back substitution, zero inflow: carry (x_{r0}, x_{r0+1})
    {
        T z0 = T(0), z1 = T(0);
#pragma unroll
        for (int k = MR - 1; k >= 0; --k) {
            T b1, b2;
            ldcoef_b(coef + k * COEF_STRIDE, b1, b2);
            T xx = v[k];
            if (K == 2) xx -= b2 * z1;
            xx -= b1 * z0;
            z1 = z0;
            z0 = xx;
        }
        S.cf0[s][p] = z0;
        S.cf1[s][p] = z1;
    }
    __syncthreads();
    // ---- 5. backward carry scan (lanes in reverse chunk order)
    {
        const int q = PC - 1 - qq;
        T b0 = S.cf0[ss][q], b1 = S.cf1[ss][q];
        seg_scan<T, PC>(b0, b1, qq, tab_c + q * TAB_STRIDE + TAB_PB);
        T e0 = __shfl_up_sync(0xffffffffu, b0, 1, PC), e1 = __shfl_up_sync(0xffffffffu, b1, 1, PC);
        if (qq == 0) e0 = e1 = T(0);
        S.in0[ss][q] = e0;
        S.in1[ss][q] = e1;
        if (qq == PC - 1) {  // chunk 0: the CTA's aggregate
            if (C > 1) {
                for (int rr = 0; rr < C; ++rr) {
                    T *pa = peer(&S.aggB[c][ss][0], rr);
                    pa[0] = b0;
                    pa[1] = b1;
                }
            } else if (PER) {
                S.xl[ss][0] = b0;  // (y_1, y_2): first two values of the system
                S.xl[ss][1] = b1;
            }
        }
    }
    if (C > 1)
        cluster_sync_all();
    else
        __syncthreads();
    if (PER) {
        // spec is visible (barrier after step 4 / cluster barrier above)
        if (tid < W) {
            T y1, y2;
            if (C > 1) {
                y1 = T(0);
                y2 = T(0);
                for (int cc = C - 1; cc >= 0; --cc) affine(y1, y2, S.aggB[cc][tid][0], S.aggB[cc][tid][1], A.mbc + cc * 4);
            } else {
                y1 = S.xl[tid][0];
                y2 = S.xl[tid][1];
            }
            const double *sc = A.scal;
            if (K == 2) {
                // Navon (eq:first_two): (x_{N-1}, x_N) = Sinv [(f_{N-1}, f_N) - h^T y]
                T gm2 = S.spec[0][tid], gm1 = S.spec[1][tid], fn2 = S.spec[2][tid], fn1 = S.spec[3][tid];
                T ym1 = gm1;                    // last core row: x = g (gamma = delta = 0)
                T ym2 = gm2 - T(sc[10]) * gm1;  // second-to-last core row
                T q0 = fn2 - (T(sc[4]) * y1 + T(sc[5]) * ym2 + T(sc[6]) * ym1);
                T q1 = fn1 - (T(sc[7]) * y1 + T(sc[8]) * y2 + T(sc[9]) * ym1);
                S.xl[tid][0] = T(sc[0]) * q0 + T(sc[1]) * q1;
                S.xl[tid][1] = T(sc[2]) * q0 + T(sc[3]) * q1;
            } else {
                // Sherman–Morrison: coef = (v.y)/(1 + v.z), v = (1, 0.., v_N)
                T yn = S.spec[0][tid];
                S.xl[tid][0] = (y1 + T(sc[0]) * yn) / T(sc[1]);
                S.xl[tid][1] = T(0);
            }
        }
        __syncthreads();
    }
    // ---- 6. back substitution with the true inflow (+ periodic correction): v <- x
    {
        T z0 = S.in0[s][p], z1 = S.in1[s][p];
        if (C > 1) {
            T Z0 = T(0), Z1 = T(0);
            for (int cc = C - 1; cc > c; --cc) affine(Z0, Z1, S.aggB[cc][s][0], S.aggB[cc][s][1], A.mbc + cc * 4);
            const T *phi = tab_c + p * TAB_STRIDE + TAB_PHIB;
            z0 += __ldg(phi + 0) * Z0 + __ldg(phi + 1) * Z1;
            z1 += __ldg(phi + 2) * Z0 + __ldg(phi + 3) * Z1;
        }
        T xl0 = T(0), xl1 = T(0);
        if (PER) {
            xl0 = S.xl[s][0];
            xl1 = S.xl[s][1];
        }
#pragma unroll
        for (int k = MR - 1; k >= 0; --k) {
            T b1, b2;
            ldcoef_b(coef + k * COEF_STRIDE, b1, b2);
            T xx = v[k];
            if (K == 2) xx -= b2 * z1;
            xx -= b1 * z0;
            z1 = z0;
            z0 = xx;
            if (PER) {
                T zz1, zz2;
                ldcoef_z(coef + k * COEF_STRIDE, zz1, zz2);
                T o = xx - zz1 * xl0;
                if (K == 2) {
                    o -= zz2 * xl1;
                    const int64_t r = r0 + k;
                    if (r == A.n - 2) o = xl0;
                    if (r == A.n - 1) o = xl1;
                }
                v[k] = o;
            } else {
                v[k] = xx;
            }
        }
    }
}

}  // namespace pb

// banded.cu — pent_factor / pent_solve / tri_factor / tri_solve for sm_100a.
//
// Shared-LHS systems (cuPentConstantBatch / cuThomasConstantBatch)
// run the partitioned cluster kernel of band_core.cuh.  Per-system LHS
// (cuPentBatch) runs one thread per system, as in the thesis.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include <cudaTypedefs.h>

#include "band_tile.cuh"

namespace pb {

constexpr double PIVOT_TOL = 1e-14;  // reading r16

}  // namespace pb

struct pb_penta_s : pb::Band {};
struct pb_tri_s : pb::Band {};

namespace pb {

// ---------------------------------------------------------------- factorisation (device, fp64)
// Writes the AoS coefficient rows of one system: coef(i, j) at
// out[(i*8 + j) * ostr + s].  Inputs a..e at [i*istr + s].  Returns 0 or the
// failing row (+1) via *bad (negative code in *code).
struct Acc {
    const double *p;
    int64_t str, s;
    __device__ double operator()(int64_t i) const { return p[i * str + s]; }
};

template <typename T>
__device__ void put(T *out, int64_t ostr, int64_t s, int64_t i, int j, double v)
{
    out[(i * COEF_STRIDE + j) * ostr + s] = (T)v;
}

// 14-step LR of rows 0..nn-1, emitted directly as solve
// coefficients; rows nn..rows-1 become identity rows.
template <typename T>
__device__ int penta_factor_rows(int64_t nn, int64_t rows, Acc a, Acc b, Acc c, Acc d, Acc e, T *out,
                                 int64_t ostr, int64_t s, int64_t *bad)
{
    double gm2 = 0, dm2 = 0, gm1 = 0, dm1 = 0;  // gamma/delta of rows i-2, i-1
    for (int64_t i = 0; i < nn; ++i) {
        double be = 0, al;
        if (i == 0) {
            al = c(0);                                      // 1. alpha_1 = c_1
        } else if (i == 1) {
            be = b(1);                                      // 4. beta_2 = b_2
            al = c(1) - be * gm1;                           // 5.
        } else {
            be = b(i) - a(i) * gm2;                         // 8a / 9 / 12
            al = c(i) - a(i) * dm2 - be * gm1;              // 8b / 10 / 13
        }
        if (!(fabs(al) >= PIVOT_TOL)) {
            *bad = i;
            return PB_EZEROPIVOT;
        }
        double ga = (i <= nn - 2) ? (d(i) - be * dm1) / al : 0.0;  // 2 / 6 / 8c / 11
        double de = (i <= nn - 3) ? e(i) / al : 0.0;               // 3 / 7 / 8d
        double ep = (i >= 2) ? a(i) : 0.0;                          // 14. eps_i = a_i
        put(out, ostr, s, i, 0, 1.0 / al);
        put(out, ostr, s, i, 1, be / al);
        put(out, ostr, s, i, 2, ep / al);
        put(out, ostr, s, i, 3, 0.0);
        put(out, ostr, s, i, 4, ga);
        put(out, ostr, s, i, 5, de);
        put(out, ostr, s, i, 6, 0.0);
        put(out, ostr, s, i, 7, 0.0);
        gm2 = gm1;
        dm2 = dm1;
        gm1 = ga;
        dm1 = de;
    }
    for (int64_t i = nn; i < rows; ++i) {
        put(out, ostr, s, i, 0, 1.0);
        for (int j = 1; j < COEF_STRIDE; ++j) put(out, ostr, s, i, j, 0.0);
    }
    return PB_OK;
}

// Thomas prefactorisation emitted as coefficients; for
// periodic systems on A' (corners 2b_1 and b_N + a_1 c_N / b_1).
template <typename T>
__device__ int tri_factor_rows(int64_t n, int64_t rows, int periodic, Acc a, Acc b, Acc c, T *out, int64_t ostr,
                               int64_t s, int64_t *bad)
{
    double chp = 0;
    for (int64_t i = 0; i < n; ++i) {
        double bi = b(i);
        if (periodic && i == 0) bi = 2.0 * b(0);
        if (periodic && i == n - 1) bi = b(n - 1) + a(0) * c(n - 1) / b(0);
        double ai = (i > 0) ? a(i) : 0.0;
        double den = bi - ai * chp;
        if (!(fabs(den) >= PIVOT_TOL)) {
            *bad = i;
            return PB_EZEROPIVOT;
        }
        double ch = (i < n - 1) ? c(i) / den : 0.0;
        put(out, ostr, s, i, 0, 1.0 / den);
        put(out, ostr, s, i, 1, ai / den);
        put(out, ostr, s, i, 2, 0.0);
        put(out, ostr, s, i, 3, 0.0);
        put(out, ostr, s, i, 4, ch);
        put(out, ostr, s, i, 5, 0.0);
        put(out, ostr, s, i, 6, 0.0);
        put(out, ostr, s, i, 7, 0.0);
        chp = ch;
    }
    for (int64_t i = n; i < rows; ++i) {
        put(out, ostr, s, i, 0, 1.0);
        for (int j = 1; j < COEF_STRIDE; ++j) put(out, ostr, s, i, j, 0.0);
    }
    return PB_OK;
}

// Solve with the emitted coefficients (used by the factor kernels for the
// periodic precomputes): rhs in slot j (6 or 7) of rows 0..nn-1, in place.
__device__ void coef_solve_slot(double *out, int64_t ostr, int64_t s, int64_t nn, int j)
{
    auto C_ = [&](int64_t i, int q) -> double & { return out[(i * COEF_STRIDE + q) * ostr + s]; };
    double y0 = 0, y1 = 0;
    for (int64_t i = 0; i < nn; ++i) {
        double g = C_(i, 0) * C_(i, j) - C_(i, 1) * y1 - C_(i, 2) * y0;
        C_(i, j) = g;
        y0 = y1;
        y1 = g;
    }
    double z0 = 0, z1 = 0;
    for (int64_t i = nn - 1; i >= 0; --i) {
        double x = C_(i, j) - C_(i, 4) * z0 - C_(i, 5) * z1;
        C_(i, j) = x;
        z1 = z0;
        z0 = x;
    }
}

// One system's full factorisation + periodic precomputes, fp64 coefficients.
// scal(j) at sc[j*sstr + s].
__device__ int factor_system(int K, int64_t n, int periodic, int64_t rows, Acc a, Acc b, Acc c, Acc d, Acc e,
                             double *out, int64_t ostr, int64_t s, double *sc, int64_t sstr, int64_t *bad)
{
    auto C_ = [&](int64_t i, int q) -> double & { return out[(i * COEF_STRIDE + q) * ostr + s]; };
    for (int j = 0; j < SCAL_LEN; ++j) sc[j * sstr + s] = 0.0;
    if (K == 2) {
        int64_t nn = periodic ? n - 2 : n;
        int rc = penta_factor_rows<double>(nn, rows, a, b, c, d, e, out, ostr, s, bad);
        if (rc) return rc;
        if (!periodic) return PB_OK;
        // Navon: Z = E^{-1} k, k = columns N-1, N of the core rows
        int64_t m = nn;
        C_(0, 6) = a(0);        // row 1, col N-1
        C_(m - 2, 6) = e(m - 2); // row N-3, col N-1
        C_(m - 1, 6) = d(m - 1); // row N-2, col N-1
        C_(0, 7) = b(0);        // row 1, col N
        C_(1, 7) = a(1);        // row 2, col N
        C_(m - 1, 7) = e(m - 1); // row N-2, col N
        coef_solve_slot(out, ostr, s, m, 6);
        coef_solve_slot(out, ostr, s, m, 7);
        // h^T (rows N-1, N on core columns): row N-1: e_{N-1}@1, a_{N-1}@N-3, b_{N-1}@N-2;
        //                                     row N:   d_N@1, e_N@2, a_N@N-2
        double H[6] = {e(n - 2), a(n - 2), b(n - 2), d(n - 1), e(n - 1), a(n - 1)};
        double hz00 = H[0] * C_(0, 6) + H[1] * C_(m - 2, 6) + H[2] * C_(m - 1, 6);
        double hz01 = H[0] * C_(0, 7) + H[1] * C_(m - 2, 7) + H[2] * C_(m - 1, 7);
        double hz10 = H[3] * C_(0, 6) + H[4] * C_(1, 6) + H[5] * C_(m - 1, 6);
        double hz11 = H[3] * C_(0, 7) + H[4] * C_(1, 7) + H[5] * C_(m - 1, 7);
        // S = B - h^T E^{-1} k, B = [[c_{N-1}, d_{N-1}], [b_N, c_N]]
        double S0 = c(n - 2) - hz00, S1 = d(n - 2) - hz01, S2 = b(n - 1) - hz10, S3 = c(n - 1) - hz11;
        double det = S0 * S3 - S1 * S2;
        if (!(fabs(det) >= PIVOT_TOL)) return PB_ESINGULAR;
        sc[0 * sstr + s] = S3 / det;
        sc[1 * sstr + s] = -S1 / det;
        sc[2 * sstr + s] = -S2 / det;
        sc[3 * sstr + s] = S0 / det;
        for (int j = 0; j < 6; ++j) sc[(4 + j) * sstr + s] = H[j];
        sc[10 * sstr + s] = C_(m - 2, 4);  // gamma_{m-2}
        return PB_OK;
    } else {
        if (periodic && !(fabs(b(0)) >= PIVOT_TOL)) {
            *bad = 0;
            return PB_EZEROPIVOT;
        }
        int rc = tri_factor_rows<double>(n, rows, periodic, a, b, c, out, ostr, s, bad);
        if (rc || !periodic) return rc;
        // Sherman–Morrison: A' z = u, u = (-b_1, 0, .., c_N)  (r14)
        C_(0, 6) = -b(0);
        C_(n - 1, 6) = c(n - 1);
        coef_solve_slot(out, ostr, s, n, 6);
        double vN = -a(0) / b(0);
        double den = 1.0 + C_(0, 6) + vN * C_(n - 1, 6);
        if (!(fabs(den) >= PIVOT_TOL)) return PB_ESINGULAR;
        sc[0 * sstr + s] = vN;
        sc[1 * sstr + s] = den;
        return PB_OK;
    }
}

__global__ void factor_shared_kernel(int K, int64_t n, int periodic, int64_t rows, const double *a,
                                     const double *b, const double *c, const double *d, const double *e,
                                     double *coefD, double *scal, int64_t *status)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int64_t bad = -1;
    Acc A{a, 1, 0}, B{b, 1, 0}, Cc{c, 1, 0}, D{d ? d : a, 1, 0}, E{e ? e : a, 1, 0};
    int rc = factor_system(K, n, periodic, rows, A, B, Cc, D, E, coefD, 1, 0, scal, 1, &bad);
    status[0] = rc;
    status[1] = 0;
    status[2] = bad;
}

__global__ void factor_persys_kernel(int K, int64_t n, int64_t M, int periodic, const double *a,
                                     const double *b, const double *c, const double *d, const double *e,
                                     double *coefD, double *scal, int64_t *status)
{
    int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= M) return;
    int64_t bad = -1;
    Acc A{a, M, s}, B{b, M, s}, Cc{c, M, s}, D{d ? d : a, M, s}, E{e ? e : a, M, s};
    int rc = factor_system(K, n, periodic, n, A, B, Cc, D, E, coefD, M, s, scal, M, &bad);
    if (rc) {
        // report the first failing system (lowest index wins)
        // report the lowest failing system and its code
        unsigned long long key = ((unsigned long long)s << 20) | (unsigned long long)(-rc);
        atomicMin((unsigned long long *)&status[3], key);
    }
}

__global__ void cast_kernel(const double *src, float *dst, int64_t count)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = (float)src[i];
}

// Chunk transfer matrices of the homogeneous recurrences (fp64):
// Mf maps the inflow (g_{r0-2}, g_{r0-1}) of a chunk to its outflow
// (g_{r1-2}, g_{r1-1}); Mb maps (x_{r1}, x_{r1+1}) to (x_{r0}, x_{r0+1}).
__global__ void transfer_kernel(const double *coef, int64_t nchunks, int mr, double *mf, double *mb)
{
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= nchunks) return;
    const double *cr = coef + q * mr * COEF_STRIDE;
    for (int col = 0; col < 2; ++col) {
        double y0 = col == 0, y1 = col == 1;
        for (int k = 0; k < mr; ++k) {
            double g = -cr[k * 8 + 1] * y1 - cr[k * 8 + 2] * y0;
            y0 = y1;
            y1 = g;
        }
        mf[q * 4 + 0 + col] = y0;
        mf[q * 4 + 2 + col] = y1;
        double z0 = col == 0, z1 = col == 1;
        for (int k = mr - 1; k >= 0; --k) {
            double x = -cr[k * 8 + 4] * z0 - cr[k * 8 + 5] * z1;
            z1 = z0;
            z0 = x;
        }
        mb[q * 4 + 0 + col] = z0;
        mb[q * 4 + 2 + col] = z1;
    }
}

__device__ inline void mat_mul(const double *A, const double *B, double *R)  // R = A B
{
    double r0 = A[0] * B[0] + A[1] * B[2], r1 = A[0] * B[1] + A[1] * B[3];
    double r2 = A[2] * B[0] + A[3] * B[2], r3 = A[2] * B[1] + A[3] * B[3];
    R[0] = r0; R[1] = r1; R[2] = r2; R[3] = r3;
}

// Per-chunk scan tables (band_core.cuh): Pf[l] = Mf_q ... Mf_{q-2^l+1},
// Pb[l] = Mb_q ... Mb_{q+2^l-1}, PhiF = Mf_{q-1} ... Mf_0, PhiB = Mb_{q+1} ... Mb_{PC-1}
// (products within the chunk's CTA block), rounded to T.
template <typename T>
__global__ void scan_table_kernel(const double *mf, const double *mb, int64_t nchunks, int pc, T *tab)
{
    int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= nchunks) return;
    const int q = (int)(g % pc);
    const int64_t base = g - q;
    T *o = tab + g * TAB_STRIDE;
    for (int j = 0; j < TAB_STRIDE; ++j) o[j] = T(0);
    for (int l = 0; (1 << l) < pc; ++l) {
        double P[4] = {1, 0, 0, 1}, Q[4] = {1, 0, 0, 1};
        for (int t = 0; t < (1 << l); ++t) {
            int qf = q - t, qb = q + t;
            if (qf >= 0) mat_mul(P, mf + (base + qf) * 4, P);  // P = P * Mf_{q-t}
            if (qb < pc) mat_mul(Q, mb + (base + qb) * 4, Q);  // Q = Q * Mb_{q+t}
        }
        for (int j = 0; j < 4; ++j) {
            o[TAB_PF + 4 * l + j] = (T)P[j];
            o[TAB_PB + 4 * l + j] = (T)Q[j];
        }
    }
    double F[4] = {1, 0, 0, 1}, B[4] = {1, 0, 0, 1};
    for (int t = q - 1; t >= 0; --t) mat_mul(F, mf + (base + t) * 4, F);
    for (int t = q + 1; t < pc; ++t) mat_mul(B, mb + (base + t) * 4, B);
    for (int j = 0; j < 4; ++j) {
        o[TAB_PHIF + j] = (T)F[j];
        o[TAB_PHIB + j] = (T)B[j];
    }
}

template <typename T>
__global__ void block_transfer_kernel(const double *mf, const double *mb, int C, int pc, T *mfc, T *mbc)
{
    int c = threadIdx.x;
    if (c >= C) return;
    // forward: P = Mf_last ... Mf_first ; backward: Q = Mb_first ... Mb_last
    double P[4] = {1, 0, 0, 1}, Q[4] = {1, 0, 0, 1};
    for (int q = pc - 1; q >= 0; --q) mat_mul(P, mf + ((int64_t)c * pc + q) * 4, P);
    for (int q = 0; q < pc; ++q) mat_mul(Q, mb + ((int64_t)c * pc + q) * 4, Q);
    for (int j = 0; j < 4; ++j) {
        mfc[c * 4 + j] = (T)P[j];
        mbc[c * 4 + j] = (T)Q[j];
    }
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder()
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
        cudaGetLastError();
    });
    return fn;
}

// ---------------------------------------------------------------- one thread per system
// The thesis's cuPentBatch kernel shape: g stored in place.
// Used for per-system LHS and for any strides the fused solve cannot take:
// element i of system s of batch b at x[b*bstride + s*xs + i*xr].
template <typename T, int K, bool PER>
__global__ void band_persys_kernel(T *x, const T *coef, int64_t cstr, const double *scal, int64_t sstr,
                                   int64_t N, int64_t M, int64_t xs, int64_t xr, int64_t bstride)
{
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= M) return;
    T *X = x + (int64_t)blockIdx.y * bstride;
    auto IX = [&](int64_t i) -> int64_t { return s * xs + i * xr; };
    const int64_t cmul = cstr ? cstr : 1;
    auto CG = [&](int64_t i, int j) -> T { return coef[(i * COEF_STRIDE + j) * cmul + (cstr ? s : 0)]; };
    T y0 = 0, y1 = 0, sp[4] = {0, 0, 0, 0};
    for (int64_t i = 0; i < N; ++i) {
        T g = CG(i, 0) * X[IX(i)] - CG(i, 1) * y1;
        if (K == 2) g -= CG(i, 2) * y0;
        X[IX(i)] = g;
        y0 = y1;
        y1 = g;
        if (PER) {
            if (K == 2) {
                if (i == N - 4) sp[0] = g;
                if (i == N - 3) sp[1] = g;
                if (i == N - 2) sp[2] = g;
                if (i == N - 1) sp[3] = g;
            } else if (i == N - 1) {
                sp[0] = g;
            }
        }
    }
    T z0 = 0, z1 = 0;
    for (int64_t i = N - 1; i >= 0; --i) {
        T xx = X[IX(i)] - CG(i, 4) * z0;
        if (K == 2) xx -= CG(i, 5) * z1;
        X[IX(i)] = xx;
        z1 = z0;
        z0 = xx;
    }
    if (!PER) return;
    const int64_t ss = sstr ? s : 0;
    auto SC = [&](int j) -> T { return (T)scal[j * (sstr ? sstr : 1) + ss]; };
    T xl0, xl1 = 0;
    if (K == 2) {
        T y_0 = z0, y_1 = z1;
        T ym1 = sp[1], ym2 = sp[0] - SC(10) * sp[1];
        T q0 = sp[2] - (SC(4) * y_0 + SC(5) * ym2 + SC(6) * ym1);
        T q1 = sp[3] - (SC(7) * y_0 + SC(8) * y_1 + SC(9) * ym1);
        xl0 = SC(0) * q0 + SC(1) * q1;
        xl1 = SC(2) * q0 + SC(3) * q1;
    } else {
        xl0 = (z0 + SC(0) * sp[0]) / SC(1);
    }
    for (int64_t i = 0; i < N; ++i) {
        T o = X[IX(i)] - CG(i, 6) * xl0;
        if (K == 2) {
            o -= CG(i, 7) * xl1;
            if (i == N - 2) o = xl0;
            if (i == N - 1) o = xl1;
        }
        X[IX(i)] = o;
    }
}

// ---------------------------------------------------------------- tile configurations

static int choose_cfg(int64_t n, int64_t batch, int dtype, int *C_out)
{
    const TileCfg *T = dtype == PB_F64 ? CFG64 : CFG32;
    const int W = dtype == PB_F64 ? 16 : 32;
    const int64_t groups = (batch + W - 1) / W;
    int best = -1;
    int64_t best_ctas = -1;
    for (int k = NCFG - 1; k >= 0; --k) {  // largest chunks first
        int64_t rc = (int64_t)(T[k].nt / W) * T[k].mr;
        int64_t C = (n + rc - 1) / rc;
        if (C > 8) continue;
        int64_t ctas = groups * C;
        if (ctas >= 2 * 148) {
            *C_out = (int)C;
            return k;
        }
        if (ctas > best_ctas) {
            best_ctas = ctas;
            best = k;
        }
    }
    if (best >= 0) {
        int64_t rc = (int64_t)(T[best].nt / W) * T[best].mr;
        *C_out = (int)((n + rc - 1) / rc);
        return best;
    }
    // very long systems: up to a 16-CTA (non-portable) cluster with the largest chunks
    int k = NCFG - 1;
    int64_t rc = (int64_t)(T[k].nt / W) * T[k].mr;
    int64_t C = (n + rc - 1) / rc;
    if (C <= MAX_CLUSTER) {
        *C_out = (int)C;
        return k;
    }
    return -1;  // beyond cluster capacity: one thread per system
}

template <typename T, int K>
static int launch_persys_t(const Band *h, T *x, const pb_layout &L, cudaStream_t st)
{
    const bool shared = h->shared();
    const T *coef = (const T *)(shared ? h->coef : h->pcoef);
    const int64_t cstr = shared ? 0 : h->batch;
    const double *scal = shared ? h->scal : h->pscal;
    const int64_t sstr = shared ? 0 : h->batch;
    const int nt = 128;
    dim3 grid((unsigned)((L.n_inner + nt - 1) / nt), (unsigned)L.n_outer);
    if (h->periodic)
        band_persys_kernel<T, K, true><<<grid, nt, 0, st>>>(x, coef, cstr, scal, sstr, h->n, L.n_inner, L.inner_stride,
                                                            L.row_stride, L.outer_stride);
    else
        band_persys_kernel<T, K, false><<<grid, nt, 0, st>>>(x, coef, cstr, scal, sstr, h->n, L.n_inner, L.inner_stride,
                                                             L.row_stride, L.outer_stride);
    PB_LAUNCH_CHECK();
    return PB_OK;
}

// ---------------------------------------------------------------- factor / solve drivers
// max over the 64-row chunks of the max-abs entry of the forward and backward
// homogeneous chunk maps (fp64, from the master coefficients on the host)
static double chunk_map_growth(const Band *h)
{
    const int64_t n = h->n, rows = h->rows_alloc, nq = (n + 63) / 64;
    std::vector<double> cf((size_t)rows * COEF_STRIDE);
    if (cudaMemcpy(cf.data(), h->coefD, sizeof(double) * cf.size(), cudaMemcpyDeviceToHost) != cudaSuccess) {
        cudaGetLastError();
        return 0.0;
    }
    auto C = [&](int64_t r, int j) { return (h->K == 1 && (j == 2 || j == 5)) ? 0.0 : cf[(size_t)r * COEF_STRIDE + j]; };
    double g = 0.0;
    for (int64_t q = 0; q < nq; ++q) {
        const int64_t r0 = q * 64, kmax = std::min<int64_t>(64, n - r0);
        for (int col = 0; col < 2; ++col) {
            double y0 = col == 0, y1 = col == 1;
            for (int64_t i = 0; i < kmax; ++i) {
                const double gg = -C(r0 + i, 1) * y1 - C(r0 + i, 2) * y0;
                y0 = y1, y1 = gg;
            }
            double z0 = col == 0, z1 = col == 1;
            for (int64_t i = kmax - 1; i >= 0; --i) {
                const double x = -C(r0 + i, 4) * z0 - C(r0 + i, 5) * z1;
                z1 = z0, z0 = x;
            }
            g = std::max(g, std::max(std::max(fabs(y0), fabs(y1)), std::max(fabs(z0), fabs(z1))));
        }
    }
    return g;
}

static int factor_impl(Band *h, const double *a, const double *b, const double *c, const double *d, const double *e,
                       cudaStream_t st, int forced_k = -1, int forced_C = 0)
{
    const int64_t n = h->n, L = h->lhs_count;
    const size_t lb = sizeof(double) * (size_t)(n * L);
    Staged sa, sb, sc, sd, se;
    int rc;
    if ((rc = sa.in(a, lb, st, true)) || (rc = sb.in(b, lb, st, true)) || (rc = sc.in(c, lb, st, true))) return rc;
    if (h->K == 2 && ((rc = sd.in(d, lb, st, true)) || (rc = se.in(e, lb, st, true)))) return rc;
    int64_t *status = nullptr;
    PB_CUDA_TRY(cudaMallocAsync(&status, sizeof(int64_t) * 8, st));
    int64_t init[8] = {0, 0, -1, (int64_t)0x7fffffffffffffffLL, 0, 0, 0, 0};
    PB_CUDA_TRY(cudaMemcpyAsync(status, init, sizeof(init), cudaMemcpyHostToDevice, st));
    const double *D = h->K == 2 ? (const double *)sd.dev : nullptr, *E = h->K == 2 ? (const double *)se.dev : nullptr;
    if (h->shared()) {
        int C = 1;
        int k = forced_k >= 0 ? forced_k : choose_cfg(n, h->batch, h->dtype, &C);
        if (forced_k >= 0) C = forced_C;
        const int W = h->dtype == PB_F64 ? 16 : 32;
        int64_t rc_rows = 0;
        if (k >= 0) {
            const TileCfg &tc = (h->dtype == PB_F64 ? CFG64 : CFG32)[k];
            rc_rows = (int64_t)(tc.nt / W) * tc.mr;
            h->plan.nt = tc.nt;
            h->plan.mr = k;  // cfg index
            h->plan.w = W;
            h->plan.C = C;
            h->plan.nchunks = (int64_t)C * (tc.nt / W);
        } else {
            h->plan.C = 0;
        }
        h->rows_alloc = k >= 0 ? (int64_t)C * rc_rows : n;
        if (h->rows_alloc < n) h->rows_alloc = n;
        const int64_t chunk_rows = (n + 63) / 64 * 64;   // whole 64-row chunks for the fused solve tables
        if (h->rows_alloc < chunk_rows) h->rows_alloc = chunk_rows;
        if (h->periodic) {
            if (h->K == 2) {
                h->srow[0] = n - 4;
                h->srow[1] = n - 3;
                h->srow[2] = n - 2;
                h->srow[3] = n - 1;
            } else {
                h->srow[0] = n - 1;
            }
        }
        PB_CUDA_TRY(cudaMalloc(&h->coefD, sizeof(double) * COEF_STRIDE * h->rows_alloc));
        PB_CUDA_TRY(cudaMalloc(&h->scal, sizeof(double) * SCAL_LEN));
        factor_shared_kernel<<<1, 1, 0, st>>>(h->K, n, h->periodic, h->rows_alloc, (const double *)sa.dev,
                                               (const double *)sb.dev, (const double *)sc.dev, D, E, h->coefD,
                                               h->scal, status);
        PB_LAUNCH_CHECK();
        if (h->dtype == PB_F64) {
            h->coef = h->coefD;
        } else {
            PB_CUDA_TRY(cudaMalloc(&h->coef, sizeof(float) * COEF_STRIDE * h->rows_alloc));
            cast_kernel<<<64, 256, 0, st>>>(h->coefD, (float *)h->coef, COEF_STRIDE * h->rows_alloc);
            PB_LAUNCH_CHECK();
        }
        if (k >= 0) {
            const size_t es = dtype_size(h->dtype);
            const int tm = (h->dtype == PB_F64 ? CFG64 : CFG32)[k].mr;
            const int pc = h->plan.nt / W;
            const int64_t nch = h->plan.nchunks;
            double *mfD = nullptr, *mbD = nullptr;
            PB_CUDA_TRY(cudaMallocAsync(&mfD, sizeof(double) * 4 * nch, st));
            PB_CUDA_TRY(cudaMallocAsync(&mbD, sizeof(double) * 4 * nch, st));
            PB_CUDA_TRY(cudaMalloc(&h->plan.tab, es * TAB_STRIDE * nch));
            PB_CUDA_TRY(cudaMalloc(&h->plan.mfc, es * 4 * MAX_CLUSTER));
            PB_CUDA_TRY(cudaMalloc(&h->plan.mbc, es * 4 * MAX_CLUSTER));
            const unsigned g = (unsigned)((nch + 127) / 128);
            transfer_kernel<<<g, 128, 0, st>>>(h->coefD, nch, tm, mfD, mbD);
            PB_LAUNCH_CHECK();
            if (h->dtype == PB_F64) {
                scan_table_kernel<double><<<g, 128, 0, st>>>(mfD, mbD, nch, pc, (double *)h->plan.tab);
                PB_LAUNCH_CHECK();
                block_transfer_kernel<double><<<1, 32, 0, st>>>(mfD, mbD, C, pc, (double *)h->plan.mfc,
                                                               (double *)h->plan.mbc);
            } else {
                scan_table_kernel<float><<<g, 128, 0, st>>>(mfD, mbD, nch, pc, (float *)h->plan.tab);
                PB_LAUNCH_CHECK();
                block_transfer_kernel<float><<<1, 32, 0, st>>>(mfD, mbD, C, pc, (float *)h->plan.mfc,
                                                              (float *)h->plan.mbc);
            }
            PB_LAUNCH_CHECK();
            PB_CUDA_TRY(cudaFreeAsync(mfD, st));
            PB_CUDA_TRY(cudaFreeAsync(mbD, st));
        }
        if ((rc = fused_build_tables(h, st))) return rc;
    } else {
        const int64_t M = h->batch;
        double *pcD = nullptr;
        PB_CUDA_TRY(cudaMalloc(&pcD, sizeof(double) * COEF_STRIDE * n * M));
        PB_CUDA_TRY(cudaMalloc(&h->pscal, sizeof(double) * SCAL_LEN * M));
        factor_persys_kernel<<<(unsigned)((M + 127) / 128), 128, 0, st>>>(
            h->K, n, M, h->periodic, (const double *)sa.dev, (const double *)sb.dev, (const double *)sc.dev, D, E,
            pcD, h->pscal, status);
        PB_LAUNCH_CHECK();
        if (h->dtype == PB_F64) {
            h->pcoef = pcD;
        } else {
            PB_CUDA_TRY(cudaMalloc(&h->pcoef, sizeof(float) * COEF_STRIDE * n * M));
            cast_kernel<<<256, 256, 0, st>>>(pcD, (float *)h->pcoef, COEF_STRIDE * n * M);
            PB_LAUNCH_CHECK();
            PB_CUDA_TRY(cudaFreeAsync(pcD, st));
        }
    }
    int64_t hs[8];
    PB_CUDA_TRY(cudaMemcpyAsync(hs, status, sizeof(hs), cudaMemcpyDeviceToHost, st));
    PB_CUDA_TRY(cudaFreeAsync(status, st));
    PB_CUDA_TRY(cudaStreamSynchronize(st));  // the one sync of pent_factor
    if (h->shared()) {
        if (hs[0] != PB_OK) {
            int code = (int)hs[0];
            set_error(code, code == PB_EZEROPIVOT ? "zero pivot at row %lld" : "singular periodic correction",
                      (long long)hs[2]);
            set_pivot(0, hs[2]);
            return code;
        }
    } else if (hs[3] != (int64_t)0x7fffffffffffffffLL) {
        unsigned long long key = (unsigned long long)hs[3];
        int code = -(int)(key & 0xfffff);
        int64_t sys = (int64_t)(key >> 20);
        set_error(code, code == PB_EZEROPIVOT ? "zero pivot in system %lld" : "singular periodic correction in system %lld",
                  (long long)sys);
        set_pivot(sys, -1);
        return code;
    }
    if (h->shared() && h->n > 64) {
        h->chunk_growth = chunk_map_growth(h);
        h->seq_only = h->chunk_growth >= 1.0;
    }
    return PB_OK;
}

// Host right-hand sides (interleaved, one batch, shared LHS): the systems are
// cut into NCHUNK column blocks and pipelined over two internal streams --
// pitched H2D copy of block c+1 | fused solve of block c | pitched D2H of
// block c-1 -- so both PCIe directions and the solve overlap.  The caller's
// stream is joined at the start and the end; the call returns with the host
// buffer updated (the host-buffer contract of pentab.h).
static int pipelined_host_solve(const Band *h, void *host, const pb_layout &L, cudaStream_t st)
{
    constexpr int NCHUNK = 16, NS = 3;   // column blocks, streams (H2D of c+2 | solve of c+1 | D2H of c)
    const size_t es = dtype_size(h->dtype);
    const int64_t n = h->n, M = L.n_inner, P = L.row_stride;
    int64_t mc = (M + NCHUNK - 1) / NCHUNK;
    mc = (mc + 31) / 32 * 32;   // whole 32-system tiles, 16-byte pitch
    const int nch = (int)((M + mc - 1) / mc);
    struct Res {
        cudaStream_t s[NS] = {};
        cudaEvent_t e[NS + 1] = {};
        void *buf[NS] = {};
        cudaStream_t owner = nullptr;
        ~Res()
        {
            for (int k = 0; k < NS; ++k)
                if (buf[k]) cudaFreeAsync(buf[k], owner);
            for (auto ev : e)
                if (ev) cudaEventDestroy(ev);
        }
    } R;
    R.owner = st;
    {
        // the handle's pipeline streams (created once; their scratch is reused)
        std::lock_guard<std::mutex> lk(h->fplan.mu);
        for (int k = 0; k < NS; ++k) {
            if (!h->fplan.pipe[k]) PB_CUDA_TRY(cudaStreamCreateWithFlags(&h->fplan.pipe[k], cudaStreamNonBlocking));
            R.s[k] = h->fplan.pipe[k];
        }
    }
    for (int k = 0; k <= NS; ++k) PB_CUDA_TRY(cudaEventCreateWithFlags(&R.e[k], cudaEventDisableTiming));
    const size_t cbytes = es * (size_t)mc * (size_t)n;
    for (int k = 0; k < NS; ++k) PB_CUDA_TRY(cudaMallocAsync(&R.buf[k], cbytes, st));
    PB_CUDA_TRY(cudaEventRecord(R.e[NS], st));   // the caller's prior work (and the allocations)
    for (int k = 0; k < NS; ++k) PB_CUDA_TRY(cudaStreamWaitEvent(R.s[k], R.e[NS], 0));
    char *hb = (char *)host;
    for (int c = 0; c < nch; ++c) {
        const int k = c % NS;
        const int64_t s0 = (int64_t)c * mc, m = std::min<int64_t>(mc, M - s0);
        // block c reuses buffer k after block c-NS's D2H (same stream: ordered)
        PB_CUDA_TRY(cudaMemcpy2DAsync(R.buf[k], es * m, hb + es * s0, es * P, es * m, n, cudaMemcpyHostToDevice, R.s[k]));
        int rc = launch_fused(h, R.buf[k], PB_INTERLEAVED, 1, 0, R.s[k], m, m);
        if (rc) return rc;
        PB_CUDA_TRY(cudaMemcpy2DAsync(hb + es * s0, es * P, R.buf[k], es * m, es * m, n, cudaMemcpyDeviceToHost, R.s[k]));
    }
    for (int k = 0; k < NS; ++k) {
        PB_CUDA_TRY(cudaEventRecord(R.e[k], R.s[k]));
        PB_CUDA_TRY(cudaStreamWaitEvent(st, R.e[k], 0));
    }
    PB_CUDA_TRY(cudaStreamSynchronize(st));
    return PB_OK;
}

// The general solve: systems (s, b) at rhs + b*outer_stride + s*inner_stride,
// unknown i at + i*row_stride.  Shared LHS with either packed or
// pitched interleaved (inner_stride 1) or contiguous (row_stride 1) systems ->
// the fused streaming solve; packed layouts with unaligned buffers -> the
// register-tile kernel; anything else (and per-system LHS) -> one thread per
// system.  Host buffers are staged through device scratch (Staged).
int band_solve_layout(const Band *h, void *rhs, const pb_layout &L, cudaStream_t st)
{
    if (!h) return set_error(PB_EINVAL, "null handle");
    if (L.n_inner < 0 || L.n_outer < 0 || L.n_outer > 65535) return set_error(PB_EINVAL, "bad system / batch count");
    if (L.n_inner == 0 || L.n_outer == 0 || h->batch == 0) return PB_OK;
    if (!h->shared() && L.n_inner != h->batch) return set_error(PB_EINVAL, "per-system LHS: n_inner must equal batch");
    if (L.inner_stride < 1 || L.row_stride < 1 || (L.n_outer > 1 && L.outer_stride < 1))
        return set_error(PB_EINVAL, "strides must be positive");
    const int64_t n = h->n;
    const bool inter = L.inner_stride == 1 && L.row_stride >= L.n_inner;
    const bool contig = L.row_stride == 1 && L.inner_stride >= n;
    const size_t es = dtype_size(h->dtype);
    if (inter && L.n_outer == 1 && h->shared() && h->fplan.ok && !h->seq_only && L.n_inner >= 4096 && !is_device_ptr(rhs))
        return pipelined_host_solve(h, rhs, L, st);
    const int64_t span = (L.n_outer - 1) * L.outer_stride + (L.n_inner - 1) * L.inner_stride + (n - 1) * L.row_stride + 1;
    Staged sx;
    int rc = sx.in(rhs, es * (size_t)span, st, true);
    if (rc) return rc;
    sx.out_to(rhs);
    const bool a16 = (uintptr_t)sx.dev % 16 == 0 && (L.n_outer == 1 || (L.outer_stride * es) % 16 == 0);
    const bool fused = h->shared() && h->fplan.ok && !h->seq_only && a16 &&
                       ((inter && (L.row_stride * es) % 16 == 0) || (contig && (L.inner_stride * es) % 16 == 0));
    const bool packed = L.n_inner == h->batch && ((inter && L.row_stride == L.n_inner) || (contig && L.inner_stride == n)) &&
                        (L.n_outer == 1 || L.outer_stride >= L.n_inner * n);
    if (fused) {
        rc = launch_fused(h, sx.dev, inter ? PB_INTERLEAVED : PB_CONTIGUOUS, L.n_outer, L.outer_stride, st, L.n_inner,
                          inter ? L.row_stride : L.inner_stride);
    } else if (h->shared() && h->plan.C > 0 && packed && !h->seq_only) {
        const int layout = inter ? PB_INTERLEAVED : PB_CONTIGUOUS;
        rc = h->dtype == PB_F64
                 ? (h->K == 2 ? launch_tile_f64_k2(h, sx.dev, layout, L.n_outer, L.outer_stride, st)
                              : launch_tile_f64_k1(h, sx.dev, layout, L.n_outer, L.outer_stride, st))
                 : (h->K == 2 ? launch_tile_f32_k2(h, sx.dev, layout, L.n_outer, L.outer_stride, st)
                              : launch_tile_f32_k1(h, sx.dev, layout, L.n_outer, L.outer_stride, st));
    } else if (h->dtype == PB_F64) {
        rc = h->K == 2 ? launch_persys_t<double, 2>(h, (double *)sx.dev, L, st)
                       : launch_persys_t<double, 1>(h, (double *)sx.dev, L, st);
    } else {
        rc = h->K == 2 ? launch_persys_t<float, 2>(h, (float *)sx.dev, L, st)
                       : launch_persys_t<float, 1>(h, (float *)sx.dev, L, st);
    }
    if (rc) return rc;
    return sx.finish();
}

// the packed layouts of pent_solve / pent_solve_many / tri_solve
int band_solve(const Band *h, void *rhs, int layout, int64_t count, int64_t bstride, cudaStream_t st)
{
    if (!h) return set_error(PB_EINVAL, "null handle");
    if (layout != PB_INTERLEAVED && layout != PB_CONTIGUOUS) return set_error(PB_EINVAL, "bad layout");
    if (count < 0 || count > 65535) return set_error(PB_EINVAL, "bad count");
    const int64_t per = h->batch * h->n;
    if (count > 1 && bstride < per) return set_error(PB_EINVAL, "batch_stride < batch*n");
    pb_layout L;
    L.n_inner = h->batch;
    L.n_outer = count;
    L.outer_stride = count > 1 ? bstride : per;
    L.inner_stride = layout == PB_INTERLEAVED ? 1 : h->n;
    L.row_stride = layout == PB_INTERLEAVED ? h->batch : 1;
    return band_solve_layout(h, rhs, L, st);
}

template <typename H>
static int make_band(int K, int64_t batch, int64_t n, const double *a, const double *b, const double *c,
                     const double *d, const double *e, int64_t lhs_count, int periodic, int dtype, void *stream,
                     H **out)
{
    if (!out) return set_error(PB_EINVAL, "null out");
    *out = nullptr;
    const int64_t nmin = K == 2 ? (periodic ? 7 : 5) : 3;
    if (n < nmin) return set_error(PB_EINVAL, "n = %lld too small (need >= %lld)", (long long)n, (long long)nmin);
    if (batch < 0 || (lhs_count != 1 && lhs_count != batch) || lhs_count < 1)
        return set_error(PB_EINVAL, "bad batch/lhs_count");
    if (dtype != PB_F64 && dtype != PB_F32) return set_error(PB_EINVAL, "bad dtype");
    if (!a || !b || !c || (K == 2 && (!d || !e))) return set_error(PB_EINVAL, "null diagonal");
    if (pb_device_ok() != PB_OK) return PB_ECUDA;
    H *h = new H();
    h->K = K;
    h->batch = batch;
    h->n = n;
    h->lhs_count = lhs_count;
    h->periodic = periodic ? 1 : 0;
    h->dtype = dtype;
    int rc = factor_impl(h, a, b, c, d, e, (cudaStream_t)stream);
    if (rc) {
        delete h;
        return rc;
    }
    *out = h;
    return PB_OK;
}

// Uniform-scalar LHS (cuPentUniformBatch / cuThomasConstantBatch with equal
// entries on each diagonal): the scalars become the diagonals of
// one shared LHS; the factorisation is the same 14-step LR (it is not uniform
// near the ends).
__global__ void fill_diags_kernel(double *dg, int64_t n, double a, double b, double c, double d, double e)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        dg[i] = a;
        dg[n + i] = b;
        dg[2 * n + i] = c;
        dg[3 * n + i] = d;
        dg[4 * n + i] = e;
    }
}

template <typename H>
static int make_uniform(int K, int64_t batch, int64_t n, double a, double b, double c, double d, double e, int periodic,
                        int dtype, cudaStream_t st, H **out)
{
    if (!out) return set_error(PB_EINVAL, "null out");
    *out = nullptr;
    if (n < 1) return set_error(PB_EINVAL, "n = %lld too small", (long long)n);
    if (pb_device_ok() != PB_OK) return PB_ECUDA;
    double *dg = nullptr;
    PB_CUDA_TRY(cudaMallocAsync(&dg, sizeof(double) * 5 * n, st));
    fill_diags_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, st>>>(dg, n, a, b, c, d, e);
    PB_LAUNCH_CHECK();
    int rc = make_band<H>(K, batch, n, dg, dg + n, dg + 2 * n, dg + 3 * n, dg + 4 * n, 1, periodic, dtype, st, out);
    cudaFreeAsync(dg, st);
    return rc;
}

// Re-factor a per-system handle in place (cuPentBatchRewrite: the
// LHS changes every step): the same device kernels as pent_factor into the
// handle's own buffers -- no allocation after the first call, no host sync, no
// pivot report (a zero pivot yields non-finite solutions, r16).
static int refactor_band(Band *h, const double *a, const double *b, const double *c, const double *d, const double *e,
                         cudaStream_t st)
{
    if (!h) return set_error(PB_EINVAL, "null handle");
    if (h->shared()) return set_error(PB_EUNSUPPORTED, "refactor is for per-system LHS handles (factor a new shared one)");
    if (!a || !b || !c || (h->K == 2 && (!d || !e))) return set_error(PB_EINVAL, "null diagonal");
    const int64_t n = h->n, M = h->batch;
    if (M == 0) return PB_OK;
    if (!h->rstatus) PB_CUDA_TRY(cudaMalloc(&h->rstatus, sizeof(int64_t) * 8));
    double *dst = h->dtype == PB_F64 ? (double *)h->pcoef : h->pcoefD;
    if (!dst) {
        PB_CUDA_TRY(cudaMalloc(&h->pcoefD, sizeof(double) * COEF_STRIDE * n * M));
        dst = h->pcoefD;
    }
    factor_persys_kernel<<<(unsigned)((M + 127) / 128), 128, 0, st>>>(h->K, n, M, h->periodic, a, b, c,
                                                                      h->K == 2 ? d : nullptr, h->K == 2 ? e : nullptr,
                                                                      dst, h->pscal, h->rstatus);
    PB_LAUNCH_CHECK();
    if (h->dtype != PB_F64) {
        cast_kernel<<<256, 256, 0, st>>>(dst, (float *)h->pcoef, COEF_STRIDE * n * M);
        PB_LAUNCH_CHECK();
    }
    return PB_OK;
}

// Constant cyclic pentadiagonal (s, -4s, 1+6s, -4s, s): the ADI operators
// L_x = L_y = I + 2/3 D gamma dt d_xxxx, factored with a forced tile
// configuration for the fused sweeps of ch_adi.cu.
int const_penta_band(int64_t n, double sigma, int dtype, int cfg, int C, cudaStream_t st, Band **out)
{
    *out = nullptr;
    double *dg = nullptr;
    PB_CUDA_TRY(cudaMalloc(&dg, sizeof(double) * 5 * n));
    double *hv = (double *)malloc(sizeof(double) * 5 * n);
    const double v[5] = {sigma, -4 * sigma, 1 + 6 * sigma, -4 * sigma, sigma};
    for (int j = 0; j < 5; ++j)
        for (int64_t i = 0; i < n; ++i) hv[j * n + i] = v[j];
    cudaError_t e1 = cudaMemcpyAsync(dg, hv, sizeof(double) * 5 * n, cudaMemcpyHostToDevice, st);
    cudaError_t e2 = cudaStreamSynchronize(st);
    free(hv);
    if (e1 != cudaSuccess || e2 != cudaSuccess) {
        cudaFree(dg);
        return set_error(PB_ECUDA, "const_penta_band copy failed");
    }
    Band *h = new Band();
    h->K = 2;
    h->batch = n;
    h->n = n;
    h->lhs_count = 1;
    h->periodic = 1;
    h->dtype = dtype;
    int rc = factor_impl(h, dg, dg + n, dg + 2 * n, dg + 3 * n, dg + 4 * n, st, cfg, C);
    cudaFree(dg);
    if (rc) {
        delete h;
        return rc;
    }
    *out = h;
    return PB_OK;
}

}  // namespace pb

extern "C" {

int pent_factor(int64_t batch, int64_t n, const double *a, const double *b, const double *c, const double *d,
                const double *e, int64_t lhs_count, int periodic, int dtype, void *stream, pb_penta_t *out)
{
    return pb::make_band<pb_penta_s>(2, batch, n, a, b, c, d, e, lhs_count, periodic, dtype, stream, out);
}

int pent_solve(pb_penta_t h, void *rhs, int layout, void *stream)
{
    return pb::band_solve(h, rhs, layout, 1, 0, (cudaStream_t)stream);
}

int pent_solve_many(pb_penta_t h, void *rhs, int layout, int64_t count, int64_t batch_stride, void *stream)
{
    return pb::band_solve(h, rhs, layout, count, batch_stride, (cudaStream_t)stream);
}

int pent_refactor(pb_penta_t h, const double *a, const double *b, const double *c, const double *d, const double *e,
                  void *stream)
{
    return pb::refactor_band(h, a, b, c, d, e, (cudaStream_t)stream);
}

int pent_factor_uniform(int64_t batch, int64_t n, double a, double b, double c, double d, double e, int periodic,
                        int dtype, void *stream, pb_penta_t *out)
{
    return pb::make_uniform<pb_penta_s>(2, batch, n, a, b, c, d, e, periodic, dtype, (cudaStream_t)stream, out);
}

int pent_solve_strided(pb_penta_t h, void *rhs, const pb_layout *L, void *stream)
{
    if (!L) return pb::set_error(PB_EINVAL, "null layout");
    return pb::band_solve_layout(h, rhs, *L, (cudaStream_t)stream);
}

int pent_solve_info(pb_penta_t h, int layout, int *info)
{
    if (!h || !info || (layout != PB_INTERLEAVED && layout != PB_CONTIGUOUS))
        return pb::set_error(PB_EINVAL, "bad argument");
    info[0] = info[1] = info[2] = info[3] = -1;
    if (!h->shared() || !h->fplan.ok || h->seq_only) return PB_OK;
    return pb::fused_info(h, layout, h->batch, 1, info);
}

int pent_destroy(pb_penta_t h)
{
    delete h;
    return PB_OK;
}

int tri_factor(int64_t batch, int64_t n, const double *a, const double *b, const double *c, int64_t lhs_count,
               int periodic, int dtype, void *stream, pb_tri_t *out)
{
    return pb::make_band<pb_tri_s>(1, batch, n, a, b, c, nullptr, nullptr, lhs_count, periodic, dtype, stream, out);
}

int tri_solve(pb_tri_t h, void *rhs, int layout, void *stream)
{
    return pb::band_solve(h, rhs, layout, 1, 0, (cudaStream_t)stream);
}

int tri_refactor(pb_tri_t h, const double *a, const double *b, const double *c, void *stream)
{
    return pb::refactor_band(h, a, b, c, nullptr, nullptr, (cudaStream_t)stream);
}

int tri_factor_uniform(int64_t batch, int64_t n, double a, double b, double c, int periodic, int dtype, void *stream,
                       pb_tri_t *out)
{
    return pb::make_uniform<pb_tri_s>(1, batch, n, a, b, c, 0.0, 0.0, periodic, dtype, (cudaStream_t)stream, out);
}

int tri_solve_strided(pb_tri_t h, void *rhs, const pb_layout *L, void *stream)
{
    if (!L) return pb::set_error(PB_EINVAL, "null layout");
    return pb::band_solve_layout(h, rhs, *L, (cudaStream_t)stream);
}

int tri_destroy(pb_tri_t h)
{
    delete h;
    return PB_OK;
}

}  // extern "C"

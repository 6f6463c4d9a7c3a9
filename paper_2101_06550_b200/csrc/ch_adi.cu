// ch_adi.cu — the ADI Cahn–Hilliard time step of Eq 3.1 on sm_100a.
//
//   RHS     R = -2/3 (C^n - C^{n-1}) - 2/3 dt D gamma grad^4 Cbar
//               + 2/3 D dt grad^2 (C^3 - C)^n                    (adi_rhs_kernel)
//   x-sweep w = L_x^{-1} R along i      (fused streaming solve, contiguous layout)
//   y-sweep v = L_y^{-1} w along j      (fused streaming solve, interleaved layout)
//   combine C^{n+1} = Cbar + v = 2C^n - C^{n-1} + v, over C^{n-1} (adi_combine_kernel)
// then the level pointers rotate (cuSten Swap).
//
// Both sweeps are the shared-LHS batched solve of pent_solve (fused_solve.cuh):
// the x-sweep's systems are the grid rows (sim, j), contiguous along i, which
// the fused kernel reads and writes through 128B-swizzled TMA boxes (no HBM
// transpose; the thesis transposes the whole grid between sweeps);
// the y-sweep's systems are the grid columns i, interleaved along j (batch =
// one simulation, count = sims).  R, w and v live in one fp64 workspace for
// both state dtypes: R carries the explicit biharmonic term, 64 sigma |C| in
// magnitude, that the sweeps cancel back to O(|C|), so an fp32 R would cost
// ~eps32 * 64 sigma relative per step (reading r22).
//
// Readings: dx = L/n (r1); Cbar = 2C^n - C^{n-1} (r6); the
// explicit grad^4 carries D*gamma (r5); grad^2 is the 5-point stencil (r8);
// grad^4 = dx^4 + 2 dx^2 dy^2 + dy^4 with the Fig 3.1 cross stencil (r9).
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>

#include "band_tile.cuh"

namespace pb {

// ---------------------------------------------------------------- RHS
// CTA = RT_J rows x RT_I columns of one simulation; Cbar = 2C^n - C^{n-1} and
// C^n with their 2-point halo are staged once in shared memory (fp64), then
// thread = column slides down the rows with the 13-point / 5-point windows in
// registers (one new Cbar row and one new C^3 - C row per output).  R is fp64.
#ifndef RHS_RT_J
#define RHS_RT_J 8
#endif
#ifndef RHS_RT_I
#define RHS_RT_I 128
#endif
constexpr int RT_I = RHS_RT_I, RT_J = RHS_RT_J;
constexpr int RS_I = RT_I + 4, RS_J = RT_J + 4;

__device__ __forceinline__ int64_t wrapi(int64_t x, int64_t n)
{
    x %= n;
    return x < 0 ? x + n : x;
}

// ext = 0: whole periodic grids [sim][n][n]; ext = 1: one row block of `rows`
// rows in an extended (rows + 4) x n buffer (2 halo rows above and below,
// configs[4]), periodic in i only
// Cahn–Hilliard–Cook noise (ch_adi_step_cook, readings r25/r26): the
// counter-based N(0,1) pair (rho_x, rho_y) of one cell -- splitmix64 over
// (seed, step, sim, cell), two uniforms in (0,1), Box–Muller.
struct CookArgs {
    double k_noise;   // 2/3 dt sqrt(sigma / (dx^2 dt)) / (2 dx); 0 = no noise
    uint64_t key;     // mix(mix(seed) ^ step) (the sim is mixed in per CTA)
};
__host__ __device__ __forceinline__ uint64_t cook_mix(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__device__ __forceinline__ void cook_rho(uint64_t k, uint64_t cell, double &rx, double &ry)
{
    const uint64_t h1 = cook_mix(k ^ (2 * cell)), h2 = cook_mix(k ^ (2 * cell + 1));
    const double u1 = ((double)(h1 >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    const double u2 = ((double)(h2 >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    // cos / sin of 2 pi u2 (as the oracle) through sincospi: no argument reduction
    const double r = sqrt(-2.0 * log(u1));
    double sn, cs;
    sincospi(2.0 * u2, &sn, &cs);
    rx = r * cs;
    ry = r * sn;
}

template <typename TS>
__global__ void __launch_bounds__(RT_I) adi_rhs_kernel(const TS *__restrict__ cn, const TS *__restrict__ cm,
                                                       double *__restrict__ R, int64_t n, int64_t rows, int ext,
                                                       double k_dif, double k_bih, double k_lap)
{
    extern __shared__ __align__(16) double rhs_smem[];
    double(*sb)[RS_I] = reinterpret_cast<double(*)[RS_I]>(rhs_smem);                 // Cbar
    double(*sc)[RS_I] = reinterpret_cast<double(*)[RS_I]>(rhs_smem + RS_J * RS_I);   // C^n
    const int64_t i0 = (int64_t)blockIdx.x * RT_I, j0 = (int64_t)blockIdx.y * RT_J;
    const int64_t plane_in = (ext ? rows + 4 : n) * n;
    const TS *Cn = cn + (int64_t)blockIdx.z * plane_in;
    const TS *Cm = cm + (int64_t)blockIdx.z * plane_in;
    double *Ro = R + (int64_t)blockIdx.z * rows * n;
    // ---- stage (all loads of a batch first, then the stores)
#ifndef RHS_BATCH
#define RHS_BATCH 8
#endif
    constexpr int NE = RS_J * RS_I, PER = (NE + RT_I - 1) / RT_I, BATCH = RHS_BATCH;
#pragma unroll
    for (int u0 = 0; u0 < PER; u0 += BATCH) {
        TS a[BATCH], b[BATCH];
#pragma unroll
        for (int u = 0; u < BATCH; ++u) {
            const int e = threadIdx.x + (u0 + u) * RT_I;
            if (u0 + u < PER && e < NE) {
                const int r = e / RS_I, q = e % RS_I;
                const int64_t jj = ext ? min(j0 + r, rows + 3) : wrapi(j0 - 2 + r, n);
                const int64_t idx = jj * n + wrapi(i0 - 2 + q, n);
                a[u] = __ldg(Cn + idx);
                b[u] = __ldg(Cm + idx);
            }
        }
#pragma unroll
        for (int u = 0; u < BATCH; ++u) {
            const int e = threadIdx.x + (u0 + u) * RT_I;
            if (u0 + u < PER && e < NE) {
                const double x = (double)a[u], y = (double)b[u];
                (&sb[0][0])[e] = 2.0 * x - y;
                (&sc[0][0])[e] = x;
            }
        }
    }
    __syncthreads();
    const int t = threadIdx.x;
    const int64_t i = i0 + t;
    if (i >= n) return;
    const int c = t + 2;   // staged column of i
    // window registers: Cbar rows r-2..r+2 (5 columns), C^3 - C rows r-1..r+1 (3 columns)
    double b2[5], b1[5], b0[5], bp1[5], bp2[5], n1[3], n0[3], np1[3];
    auto ldb = [&](int r, double *o) {
#pragma unroll
        for (int d = 0; d < 5; ++d) o[d] = sb[r][c - 2 + d];
    };
    auto ldn = [&](int r, double *o) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const double x = sc[r][c - 1 + d];
            o[d] = x * x * x - x;
        }
    };
    ldb(0, b2);
    ldb(1, b1);
    ldb(2, b0);
    ldb(3, bp1);
    ldn(1, n1);
    ldn(2, n0);
    const int jmax = (int)min((int64_t)RT_J, rows - j0);
#pragma unroll 4
    for (int jj = 0; jj < jmax; ++jj) {
        ldb(jj + 4, bp2);
        ldn(jj + 3, np1);
        // 13-point biharmonic: dx^4 + dy^4 (1,-4,6,-4,1) + 2 x Fig 3.1 cross stencil
        const double bih = 20.0 * b0[2] - 8.0 * ((b0[1] + b0[3]) + (b1[2] + bp1[2])) +
                           2.0 * ((b1[1] + b1[3]) + (bp1[1] + bp1[3])) + ((b0[0] + b0[4]) + (b2[2] + bp2[2]));
        const double lap = (n0[0] + n0[2]) + (n1[1] + np1[1]) - 4.0 * n0[1];
        const double d = b0[2] - sc[jj + 2][c];   // C^n - C^{n-1} = Cbar - C^n
        __stcg(Ro + (j0 + jj) * n + i, k_dif * d + k_bih * bih + k_lap * lap);
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            b2[q] = b1[q];
            b1[q] = b0[q];
            b0[q] = bp1[q];
            bp1[q] = bp2[q];
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            n1[q] = n0[q];
            n0[q] = np1[q];
        }
    }
}

// R += 2/3 dt eta, eta_ij = sqrt(sigma/(dx^2 dt)) (div rho)_ij (readings r25,
// r26): a CTA stages one Box–Muller pair per cell of its 32 x 32 tile and the
// 1-cell halo (periodic) in shared memory -- 18 KB, so many CTAs per SM hide
// the fp64 log / sincos latency -- then adds the central-difference
// divergence to its outputs (R read and written once more: 16 B per point).
constexpr int CK_T = 32, CK_H = CK_T + 2;
__global__ void __launch_bounds__(256) cook_add_kernel(double *__restrict__ R, int64_t n, double k_noise, uint64_t key)
{
    __shared__ double nx[CK_H * CK_H], ny[CK_H * CK_H];
    const int64_t i0 = (int64_t)blockIdx.x * CK_T, j0 = (int64_t)blockIdx.y * CK_T, sim = blockIdx.z;
    const uint64_t k = cook_mix(key ^ (uint64_t)sim);
    for (int e = threadIdx.x; e < CK_H * CK_H; e += blockDim.x) {
        const int r = e / CK_H, q = e % CK_H;
        const int64_t jj = wrapi(j0 - 1 + r, n), ii = wrapi(i0 - 1 + q, n);
        cook_rho(k, (uint64_t)(jj * n + ii), nx[e], ny[e]);
    }
    __syncthreads();
    double *Rs = R + sim * n * n;
    for (int e = threadIdx.x; e < CK_T * CK_T; e += blockDim.x) {
        const int r = e / CK_T, q = e % CK_T;
        const int64_t j = j0 + r, i = i0 + q;
        if (j < n && i < n) {
            const int c = (r + 1) * CK_H + (q + 1);
            double *p = Rs + j * n + i;
            __stcg(p, __ldcg(p) + k_noise * ((nx[c + 1] - nx[c - 1]) + (ny[c + CK_H] - ny[c - CK_H])));
        }
    }
}

// C^{n+1} = Cbar^{n+1} + v = 2 C^n - C^{n-1} + v, written over C^{n-1}
template <typename TS>
__global__ void adi_combine_kernel(int64_t count, const TS *__restrict__ cn, TS *__restrict__ cm,
                                   const double *__restrict__ v)
{
    using V = typename std::conditional<sizeof(TS) == 8, double2, float2>::type;
    const int64_t nv = count / 2;
    const V *a = reinterpret_cast<const V *>(cn);
    V *b = reinterpret_cast<V *>(cm);
    const double2 *c = reinterpret_cast<const double2 *>(v);
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nv; k += (int64_t)gridDim.x * blockDim.x) {
        const V x = __ldcs(a + k), y = __ldcs(b + k);
        const double2 z = __ldcs(c + k);
        V o;
        o.x = (TS)((2.0 * (double)x.x - (double)y.x) + z.x);
        o.y = (TS)((2.0 * (double)x.y - (double)y.y) + z.y);
        __stcs(b + k, o);
    }
    for (int64_t k = nv * 2 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count;
         k += (int64_t)gridDim.x * blockDim.x)
        cm[k] = (TS)((2.0 * (double)cn[k] - (double)cm[k]) + v[k]);
}

// ---------------------------------------------------------------- host side
static std::mutex g_adi_mu;
static std::map<std::tuple<int, int64_t, uint64_t>, Band *> g_adi_cache;

// the cyclic (s, -4s, 1+6s, -4s, s) of L_x = L_y, fp64, factored once
static int adi_band(int64_t n, double sigma, cudaStream_t st, Band **out)
{
    int dev = 0;
    PB_CUDA_TRY(cudaGetDevice(&dev));
    uint64_t bits;
    memcpy(&bits, &sigma, sizeof(bits));
    auto key = std::make_tuple(dev, n, bits);
    std::lock_guard<std::mutex> lk(g_adi_mu);
    auto it = g_adi_cache.find(key);
    if (it != g_adi_cache.end()) {
        *out = it->second;
        return PB_OK;
    }
    Band *h = nullptr;
    int rc = const_penta_band(n, sigma, PB_F64, -1, 0, st, &h);
    if (rc) return rc;
    g_adi_cache[key] = h;
    *out = h;
    return PB_OK;
}

struct AdiCoef {
    double sigma, k_dif, k_bih, k_lap;
};
static AdiCoef adi_coef(int64_t n, double dt, const pb_ch_params *p)
{
    const double dx = p->L / (double)n;  // r1
    const double dx4 = dx * dx * dx * dx;
    AdiCoef c;
    c.sigma = (2.0 / 3.0) * p->D * p->gamma * dt / dx4;   // L_x = I + 2/3 D gamma dt d_xxxx
    c.k_dif = -2.0 / 3.0;
    c.k_bih = -(2.0 / 3.0) * dt * p->D * p->gamma / dx4;   // r5
    c.k_lap = (2.0 / 3.0) * p->D * dt / (dx * dx);
    return c;
}

template <typename TS>
static int launch_rhs(const TS *cn, const TS *cm, double *R, int64_t n, int64_t rows, int64_t sims, int ext,
                      const AdiCoef &c, cudaStream_t st, const CookArgs *ck = nullptr)
{
    constexpr size_t smem = sizeof(double) * 2 * RS_J * RS_I;
    static std::once_flag once;
    static cudaError_t attr = cudaSuccess;
    std::call_once(once, [] {
        attr = cudaFuncSetAttribute(adi_rhs_kernel<TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    if (attr != cudaSuccess) return set_error(PB_ECUDA, "adi_rhs_kernel smem attribute: %s", cudaGetErrorString(attr));
    dim3 grid((unsigned)((n + RT_I - 1) / RT_I), (unsigned)((rows + RT_J - 1) / RT_J), (unsigned)sims);
    adi_rhs_kernel<TS><<<grid, RT_I, smem, st>>>(cn, cm, R, n, rows, ext, c.k_dif, c.k_bih, c.k_lap);
    PB_LAUNCH_CHECK();
    if (ck && ck->k_noise != 0.0) {
        dim3 g2((unsigned)((n + CK_T - 1) / CK_T), (unsigned)((n + CK_T - 1) / CK_T), (unsigned)sims);
        cook_add_kernel<<<g2, 256, 0, st>>>(R, n, ck->k_noise, ck->key);
        PB_LAUNCH_CHECK();
    }
    return PB_OK;
}

template <typename TS>
static int launch_combine(int64_t count, const TS *cn, TS *cm, const double *v, cudaStream_t st)
{
    const unsigned g = (unsigned)std::min<int64_t>((count / 2 + 255) / 256, 148 * 16);
    adi_combine_kernel<TS><<<g > 0 ? g : 1, 256, 0, st>>>(count, cn, cm, v);
    PB_LAUNCH_CHECK();
    return PB_OK;
}

template <typename TS>
static int adi_run(pb_ch_state *s, double dt, const pb_ch_params *p, int64_t nsteps, cudaStream_t st,
                   const pb_ch_noise *noise = nullptr)
{
    const int64_t n = s->n, sims = s->sims, plane = n * n;
    const AdiCoef c = adi_coef(n, dt, p);
    Band *h = nullptr;
    int rc = adi_band(n, c.sigma, st, &h);
    if (rc) return rc;
    double *w = (double *)s->work;
    for (int64_t step = 0; step < nsteps; ++step) {
        const TS *cn = (const TS *)s->c_cur;
        TS *cm = (TS *)s->c_prev;
        CookArgs ck{0.0, 0};
        if (noise && noise->sigma > 0) {
            const double dx = p->L / (double)n;
            ck.k_noise = (2.0 / 3.0) * dt * sqrt(noise->sigma / (dx * dx * dt)) / (2.0 * dx);
            ck.key = cook_mix(cook_mix(noise->seed) ^ (uint64_t)(noise->step0 + step));
        }
        if ((rc = launch_rhs<TS>(cn, cm, w, n, n, sims, 0, c, st, &ck))) return rc;
        // x-sweep: systems = rows (sim, j), contiguous along i; y-sweep: systems =
        // columns i of each simulation, interleaved along j
        if ((rc = band_solve(h, w, PB_CONTIGUOUS, sims, plane, st))) return rc;
        if ((rc = band_solve(h, w, PB_INTERLEAVED, sims, plane, st))) return rc;
        if ((rc = launch_combine<TS>(sims * plane, cn, cm, w, st))) return rc;
        void *t = s->c_prev;  // C^{n+1} now lives in the old C^{n-1} buffer
        s->c_prev = s->c_cur;
        s->c_cur = t;
    }
    return PB_OK;
}

// w [rows][n] -> packed [parts][rows][nb]: column block q becomes a contiguous
// [rows][nb] slab, the send layout of the all-to-all transpose.
__global__ void dist_pack_kernel(int64_t rows, int64_t n, int64_t parts, const double *w, double *out)
{
    const int64_t nb = n / parts, total = rows * n;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = e / n, i = e % n, q = i / nb, ii = i % nb;
        out[(q * rows + j) * nb + ii] = w[e];
    }
}

// C^{n+1} = 2 C^n - C^{n-1} + v on the interior rows of a row block (written
// over C^{n-1}); v arrives as [parts][rows][nb] (block q = columns of rank q).
template <typename TS>
__global__ void dist_combine_kernel(int64_t rows, int64_t n, int64_t parts, const TS *cn, TS *cm, const double *v)
{
    const int64_t nb = n / parts, total = rows * n;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = e / n, i = e % n, q = i / nb, ii = i % nb;
        const int64_t x = (j + 2) * n + i;
        cm[x] = (TS)((2.0 * (double)cn[x] - (double)cm[x]) + v[(q * rows + j) * nb + ii]);
    }
}

template <typename TS>
static int dist_pass_a(int64_t rows, int64_t n, const void *cn, const void *cm, double *w, double dt,
                       const pb_ch_params *p, cudaStream_t st)
{
    const AdiCoef c = adi_coef(n, dt, p);
    Band *h = nullptr;
    int rc = adi_band(n, c.sigma, st, &h);
    if (rc) return rc;
    if ((rc = launch_rhs<TS>((const TS *)cn, (const TS *)cm, w, n, rows, 1, 1, c, st))) return rc;
    // x-sweep of the rank's rows: `rows` contiguous systems of length n
    if (!h->fplan.ok) return set_error(PB_EUNSUPPORTED, "no streaming plan for n = %lld", (long long)n);
    return launch_fused(h, w, PB_CONTIGUOUS, 1, 0, st, rows);
}

}  // namespace pb

extern "C" int ch_dist_pass_a(int64_t rows, int64_t n, int dtype, const void *cn_ext, const void *cm_ext, void *w,
                              double dt, const pb_ch_params *p, void *stream)
{
    using namespace pb;
    if (!p || !cn_ext || !cm_ext || !w || rows < 1 || n < 8 || rows > n) return set_error(PB_EINVAL, "bad args");
    if (dtype != PB_F64 && dtype != PB_F32) return set_error(PB_EINVAL, "bad dtype");
    if (n % 2 || (uintptr_t)w % 16) return set_error(PB_EINVAL, "ch_dist_pass_a needs even n and a 16-byte aligned w");
    if (!(dt > 0) || !(p->L > 0)) return set_error(PB_EINVAL, "dt and L must be positive");
    if (pb_device_ok() != PB_OK) return PB_ECUDA;
    if (!is_device_ptr(cn_ext) || !is_device_ptr(cm_ext) || !is_device_ptr(w))
        return set_error(PB_EINVAL, "ch_dist_pass_a buffers must be device memory");
    cudaStream_t st = (cudaStream_t)stream;
    return dtype == PB_F64 ? dist_pass_a<double>(rows, n, cn_ext, cm_ext, (double *)w, dt, p, st)
                           : dist_pass_a<float>(rows, n, cn_ext, cm_ext, (double *)w, dt, p, st);
}

// y-sweep of a rank's column block (configs[4]): L_y v = w along j for ncols
// interleaved fp64 columns of length n, in place, with the cached cyclic L_y.
extern "C" int ch_dist_ysweep(int64_t ncols, int64_t n, void *cols, double dt, const pb_ch_params *p, void *stream)
{
    using namespace pb;
    if (!p || !cols || ncols < 1 || n < 8) return set_error(PB_EINVAL, "bad args");
    if (!(dt > 0) || !(p->L > 0)) return set_error(PB_EINVAL, "dt and L must be positive");
    if ((ncols * 8) % 16 || (uintptr_t)cols % 16)
        return set_error(PB_EINVAL, "ch_dist_ysweep needs 16-byte aligned rows (even ncols)");
    if (pb_device_ok() != PB_OK) return PB_ECUDA;
    if (!is_device_ptr(cols)) return set_error(PB_EINVAL, "ch_dist_ysweep buffers must be device memory");
    cudaStream_t st = (cudaStream_t)stream;
    const AdiCoef c = adi_coef(n, dt, p);
    Band *h = nullptr;
    int rc = adi_band(n, c.sigma, st, &h);
    if (rc) return rc;
    if (!h->fplan.ok) return set_error(PB_EUNSUPPORTED, "no streaming plan for n = %lld", (long long)n);
    return launch_fused(h, cols, PB_INTERLEAVED, 1, 0, st, ncols);
}

extern "C" int ch_dist_pack(int64_t rows, int64_t n, int64_t parts, const void *w, void *packed, void *stream)
{
    using namespace pb;
    if (!w || !packed || rows < 1 || parts < 1 || n % parts) return set_error(PB_EINVAL, "bad args");
    if (pb_device_ok() != PB_OK) return PB_ECUDA;
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned g = (unsigned)std::min<int64_t>((rows * n + 255) / 256, 148 * 16);
    dist_pack_kernel<<<g, 256, 0, st>>>(rows, n, parts, (const double *)w, (double *)packed);
    PB_LAUNCH_CHECK();
    return PB_OK;
}

extern "C" int ch_dist_combine(int64_t rows, int64_t n, int64_t parts, int dtype, const void *cn_ext, void *cm_ext,
                               const void *v_packed, void *stream)
{
    using namespace pb;
    if (!cn_ext || !cm_ext || !v_packed || rows < 1 || parts < 1 || n % parts) return set_error(PB_EINVAL, "bad args");
    if (dtype != PB_F64 && dtype != PB_F32) return set_error(PB_EINVAL, "bad dtype");
    if (pb_device_ok() != PB_OK) return PB_ECUDA;
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned g = (unsigned)std::min<int64_t>((rows * n + 255) / 256, 148 * 16);
    if (dtype == PB_F64)
        dist_combine_kernel<double><<<g, 256, 0, st>>>(rows, n, parts, (const double *)cn_ext, (double *)cm_ext,
                                                       (const double *)v_packed);
    else
        dist_combine_kernel<float><<<g, 256, 0, st>>>(rows, n, parts, (const float *)cn_ext, (float *)cm_ext,
                                                      (const double *)v_packed);
    PB_LAUNCH_CHECK();
    return PB_OK;
}

extern "C" int ch_workspace_bytes(int64_t sims, int64_t n, int dtype, size_t *bytes)
{
    using namespace pb;
    if (!bytes || sims < 0 || n < 8 || (dtype != PB_F64 && dtype != PB_F32)) return set_error(PB_EINVAL, "bad args");
    *bytes = sizeof(double) * (size_t)sims * (size_t)n * (size_t)n;   // R -> w -> v, fp64 for both state dtypes
    return PB_OK;
}

static int ch_adi_entry(pb_ch_state *s, double dt, const pb_ch_params *p, int64_t nsteps, void *stream,
                        const pb_ch_noise *noise);

extern "C" int ch_adi_step(pb_ch_state *s, double dt, const pb_ch_params *p, int64_t nsteps, void *stream)
{
    return ch_adi_entry(s, dt, p, nsteps, stream, nullptr);
}

extern "C" int ch_adi_step_cook(pb_ch_state *s, double dt, const pb_ch_params *p, const pb_ch_noise *noise,
                                int64_t nsteps, void *stream)
{
    if (!noise || !(noise->sigma >= 0)) return pb::set_error(PB_EINVAL, "noise: sigma must be >= 0");
    return ch_adi_entry(s, dt, p, nsteps, stream, noise);
}

static int ch_adi_entry(pb_ch_state *s, double dt, const pb_ch_params *p, int64_t nsteps, void *stream,
                        const pb_ch_noise *noise)
{
    using namespace pb;
    if (!s || !p) return set_error(PB_EINVAL, "null state/params");
    if (s->n < 8 || s->sims < 0 || nsteps < 0) return set_error(PB_EINVAL, "need n >= 8, sims >= 0, nsteps >= 0");
    if (s->dtype != PB_F64 && s->dtype != PB_F32) return set_error(PB_EINVAL, "bad dtype");
    if (!(dt > 0) || !(p->L > 0)) return set_error(PB_EINVAL, "dt and L must be positive");
    if (s->sims > 65535) return set_error(PB_EINVAL, "sims > 65535 per call");
    if (pb_device_ok() != PB_OK) return PB_ECUDA;
    if (s->sims == 0 || nsteps == 0) return PB_OK;
    if (!s->c_cur || !s->c_prev || !s->work || s->c_cur == s->c_prev)
        return set_error(PB_EINVAL, "c_cur, c_prev, work must be distinct device buffers");
    if ((uintptr_t)s->work % 16 || (uintptr_t)s->c_cur % 16 || (uintptr_t)s->c_prev % 16)
        return set_error(PB_EINVAL, "ch_adi_step buffers must be 16-byte aligned");
    if (!is_device_ptr(s->c_cur) || !is_device_ptr(s->c_prev) || !is_device_ptr(s->work))
        return set_error(PB_EINVAL, "ch_adi_step buffers must be device memory");
    cudaStream_t st = (cudaStream_t)stream;
    return s->dtype == PB_F64 ? adi_run<double>(s, dt, p, nsteps, st, noise)
                              : adi_run<float>(s, dt, p, nsteps, st, noise);
}

// ch_adi.cu — the ADI Cahn–Hilliard time step of Eq 3.1 as two
// fused HBM passes per step on sm_100a.
//
//   pass A (rows j):    R = -2/3 (C^n - C^{n-1}) - 2/3 dt D gamma grad^4 Cbar
//                           + 2/3 D dt grad^2 (C^3 - C)^n          (stencil, smem-staged)
//                       w = L_x^{-1} R along i                      (band_core, cyclic)
//   pass B (columns i): v = L_y^{-1} w along j                      (band_core, cyclic)
//                       C^{n+1} = Cbar + v = 2C^n - C^{n-1} + v      (epilogue, into C^{n-1})
// then the host rotates the level pointers (cuSten Swap).
//
// HBM traffic per point and step: pass A reads C^n, C^{n-1} and writes w;
// pass B reads w, C^n, C^{n-1} and writes C^{n+1}: 7 field passes = 56 B (fp64),
// the algorithmic minimum of this two-pass design.  The thesis's separate
// cuSten RHS kernels, combine kernel and the full-grid transpose between the
// sweeps are gone: pass A transposes through shared memory, and
// pass B's systems (grid columns) are already in the interleaved layout.
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

template <typename T>
struct AdiArgs {
    CoreArgs<T> core;
    const T *cn;
    T *cm;
    T *w;
    int64_t n;
    T k_dif, k_bih, k_lap;  // R = k_dif (C^n - C^{n-1}) + k_bih BIH(Cbar) + k_lap LAP(C^3 - C)
    // row-partitioned grids (ch_dist_pass_a): `rows` local rows; cn / cm hold
    // rows + 4 rows (2 halo rows above and below, no wrap in j); w holds `rows`
    int64_t rows = 0;
    int ext = 0;
    // w layout: 0 = [sim][j][i]; else w[(j * wperm + sim) * n + i] with wperm = sims
    // (all simulations' columns of one grid row contiguous: the y-sweep is then ONE
    // batch of sims * n interleaved systems)
    int64_t wperm = 0;
};

constexpr int ADI_IB = 32;  // stencil column block

__device__ __forceinline__ int64_t wrapi(int64_t x, int64_t n)
{
    // one conditional step covers the stencil halos (|offset| <= 2 + a column block)
    // when n >= the column block; the loops only run for tiny grids
    x = x < 0 ? x + n : x;
    x = x >= n ? x - n : x;
    if ((uint64_t)x >= (uint64_t)n) {
        while (x < 0) x += n;
        while (x >= n) x -= n;
    }
    return x;
}

template <typename T, int W, int NT, int MR, bool EXT = false>
__global__ void __launch_bounds__(NT, (NT <= 256 ? 2 : 1)) adi_pass_a(const AdiArgs<T> A)
{
    constexpr int PC = NT / W, RC = PC * MR, WP = W + 1, IB = ADI_IB;
    constexpr int SB = IB + 4, SN = IB + 2;  // staged row strides (Cbar halo 2, NL halo 1)
    __shared__ CoreSmem<T, W, PC> S;
    extern __shared__ __align__(16) unsigned char dyn_smem[];
    // coefficient rows are read through L1 here (not staged): pass A's shared
    // memory (solve tile + stencil staging) then allows two CTAs per SM
    T *tile = reinterpret_cast<T *>(dyn_smem);   // [RC][W+1]: R, then w
    T *cb = tile + RC * WP;                      // [W+4][IB+4] Cbar
    T *nl = cb + (W + 4) * SB;                   // [W+2][IB+2] C^3 - C
    T *dl = nl + (W + 2) * SN;                   // [W][IB]     C^n - C^{n-1}
    const int tid = threadIdx.x, s = tid % W, p = tid / W;
    const int C = A.core.C;
    const int c = (C > 1) ? (int)cg::this_cluster().block_rank() : 0;
    const int64_t n = A.n, j0 = (int64_t)(blockIdx.x / C) * W;
    const int64_t rows = EXT ? A.rows : n;
    const int64_t plane_in = (EXT ? rows + 4 : n) * n, plane_w = rows * n;
    const T *Cn = A.cn + (int64_t)blockIdx.y * plane_in;
    const T *Cm = A.cm + (int64_t)blockIdx.y * plane_in;
    T *Wo = A.w + (int64_t)blockIdx.y * (A.wperm ? n : plane_w);
    const int64_t wrs = A.wperm ? A.wperm * n : n;   // w row stride
    const int64_t ib0 = (int64_t)c * RC;  // first solve row (grid column i) of this CTA
    const T *cs = A.core.coef + ib0 * COEF_STRIDE;

    // ---- stencil RHS into the solve tile, column block by column block
    for (int ib = 0; ib < RC; ib += IB) {
        const int64_t i0 = ib0 + ib;
        const bool live = i0 < n;  // CTA-uniform
        if (live) {
            // all of this thread's staging loads first (latency overlap), then the stores
            constexpr int NST = ((W + 4) * SB + NT - 1) / NT;
            T cnr[NST], cmr[NST];
#pragma unroll
            for (int u = 0; u < NST; ++u) {
                const int e = tid + u * NT;
                if (e < (W + 4) * SB) {
                    const int r = e / SB, q = e % SB;
                    // periodic in j (whole grid), or halo rows of a row block (ext)
                    const int64_t jr = EXT ? (j0 + r < rows + 3 ? j0 + r : rows + 3) : wrapi(j0 - 2 + r, n);
                    const int64_t idx = jr * n + wrapi(i0 - 2 + q, n);
                    cnr[u] = __ldg(Cn + idx);
                    cmr[u] = __ldg(Cm + idx);
                }
            }
#pragma unroll
            for (int u = 0; u < NST; ++u) {
                const int e = tid + u * NT;
                if (e < (W + 4) * SB) {
                    const int r = e / SB, q = e % SB;
                    const T cnv = cnr[u], cmv = cmr[u];
                    cb[e] = T(2) * cnv - cmv;
                    if (r >= 1 && r < W + 3 && q >= 1 && q < IB + 3) nl[(r - 1) * SN + (q - 1)] = cnv * cnv * cnv - cnv;
                    if (r >= 2 && r < W + 2 && q >= 2 && q < IB + 2) dl[(r - 2) * IB + (q - 2)] = cnv - cmv;
                }
            }
        }
        __syncthreads();
        for (int e = tid; e < W * IB; e += NT) {
            const int jj = e / IB, ii = e % IB;
            T R = T(0);
            if (live && i0 + ii < n) {
                const T *u = cb + (jj + 2) * SB + (ii + 2);
                // 13-point biharmonic: dx^4 + dy^4 (1,-4,6,-4,1) + 2 x Fig 3.1 cross stencil
                const T bih = T(20) * u[0] - T(8) * ((u[-1] + u[1]) + (u[-SB] + u[SB])) +
                              T(2) * ((u[-SB - 1] + u[-SB + 1]) + (u[SB - 1] + u[SB + 1])) +
                              ((u[-2] + u[2]) + (u[-2 * SB] + u[2 * SB]));
                const T *q_ = nl + (jj + 1) * SN + (ii + 1);
                const T lap = (q_[-1] + q_[1]) + (q_[-SN] + q_[SN]) - T(4) * q_[0];
                R = A.k_dif * dl[jj * IB + ii] + A.k_bih * bih + A.k_lap * lap;
            }
            tile[(ib + ii) * WP + jj] = R;
        }
        __syncthreads();
    }
    // ---- x-sweep: systems = grid rows j0 + s, unknowns along i
    T v[MR];
#pragma unroll
    for (int k = 0; k < MR; ++k) v[k] = tile[(p * MR + k) * WP + s];
    band_core<T, 2, W, NT, MR, true>(v, A.core, S, cs, c, s, p, ib0 + (int64_t)p * MR);
#pragma unroll
    for (int k = 0; k < MR; ++k) tile[(p * MR + k) * WP + s] = v[k];
    __syncthreads();
    // ---- w back to the natural [j][i] layout, coalesced along i
    for (int e = tid; e < W * RC; e += NT) {
        const int jj = e / RC, ii = e % RC;
        const int64_t j = j0 + jj, i = ib0 + ii;
        if (j < rows && i < n) __stcg(Wo + j * wrs + i, tile[ii * WP + jj]);
    }
}

template <typename T, int W, int NT, int MR>
__global__ void __launch_bounds__(NT, (NT <= 256 ? 2 : 1)) adi_pass_b(const AdiArgs<T> A)
{
    constexpr int PC = NT / W, RC = PC * MR;
    __shared__ CoreSmem<T, W, PC> S;
    extern __shared__ __align__(16) unsigned char dyn_smem[];
    T *cs = reinterpret_cast<T *>(dyn_smem);  // [RC][8] coefficient rows of this CTA
    const int tid = threadIdx.x, s = tid % W, p = tid / W;
    const int C = A.core.C;
    const int c = (C > 1) ? (int)cg::this_cluster().block_rank() : 0;
    stage_coef<T, NT>(cs, A.core.coef + (int64_t)c * RC * COEF_STRIDE, RC);
    const int64_t n = A.n, i = (int64_t)(blockIdx.x / C) * W + s;
    const int64_t plane = n * n;
    const T *Wi = A.w + (int64_t)blockIdx.y * plane;
    const T *Cn = A.cn + (int64_t)blockIdx.y * plane;
    T *Cm = A.cm + (int64_t)blockIdx.y * plane;
    const int64_t r0 = (int64_t)c * RC + (int64_t)p * MR;
    const bool ok = i < n;
    // ---- y-sweep: systems = grid columns i (interleaved: lanes = consecutive i)
    T v[MR];
    {
        const T *src = Wi + r0 * n + i;
#pragma unroll
        for (int k = 0; k < MR; ++k) v[k] = (ok && r0 + k < n) ? __ldcs(src + k * n) : T(0);
    }
    __syncthreads();  // coefficient table staged
    band_core<T, 2, W, NT, MR, true>(v, A.core, S, cs, c, s, p, r0);
    // ---- C^{n+1} = Cbar^{n+1} + v, written over C^{n-1} (same thread reads then writes)
    int64_t no = n;
    asm volatile("" : "+l"(no));
    if (ok) {
#pragma unroll
        for (int k = 0; k < MR; ++k) {
            if (r0 + k < n) {
                const int64_t idx = (r0 + k) * no + i;
                const T cnv = __ldcs(Cn + idx), cmv = __ldcs(Cm + idx);
                __stcs(Cm + idx, (T(2) * cnv - cmv) + v[k]);
            }
        }
    }
}

// ---------------------------------------------------------------- host side
template <typename T, int W, int NT, int MR>
static int launch_adi(const Band *h, const AdiArgs<T> &A, int64_t sims, cudaStream_t st, bool pass_a)
{
    constexpr int PC = NT / W, RC = PC * MR;
    const int C = h->plan.C;
    const int64_t groups = ((A.ext ? A.rows : A.n) + W - 1) / W;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(groups * C), (unsigned)sims, 1);
    cfg.blockDim = dim3(NT, 1, 1);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = C > 1 ? 1 : 0;
    if (pass_a) {
        auto kern = A.ext ? adi_pass_a<T, W, NT, MR, true> : adi_pass_a<T, W, NT, MR, false>;
        const size_t dyn = sizeof(T) * ((size_t)RC * (W + 1) + (W + 4) * (ADI_IB + 4) +
                                        (W + 2) * (ADI_IB + 2) + W * ADI_IB);
        int rc = prep_kernel(kern, dyn, C);
        if (rc) return rc;
        cfg.dynamicSmemBytes = dyn;
        PB_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, A));
    } else {
        auto kern = adi_pass_b<T, W, NT, MR>;
        const size_t dyn = sizeof(T) * (size_t)RC * COEF_STRIDE;
        int rc = prep_kernel(kern, dyn, C);
        if (rc) return rc;
        cfg.dynamicSmemBytes = dyn;
        PB_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, A));
    }
    PB_LAUNCH_CHECK();
    return PB_OK;
}

template <typename T>
static int launch_adi_cfg(const Band *h, const AdiArgs<T> &A, int64_t sims, cudaStream_t st, bool pass_a)
{
    const int k = h->plan.mr;
    if (sizeof(T) == 8) {
        switch (k) {
            case 0: return launch_adi<T, 16, 256, 4>(h, A, sims, st, pass_a);
            case 1: return launch_adi<T, 16, 256, 8>(h, A, sims, st, pass_a);
            case 2: return launch_adi<T, 16, 256, 16>(h, A, sims, st, pass_a);
            case 3: return launch_adi<T, 16, 256, 32>(h, A, sims, st, pass_a);
            case 4: return launch_adi<T, 16, 512, 32>(h, A, sims, st, pass_a);
        }
    } else {
        switch (k) {
            case 0: return launch_adi<T, 32, 256, 8>(h, A, sims, st, pass_a);
            case 1: return launch_adi<T, 32, 256, 16>(h, A, sims, st, pass_a);
            case 2: return launch_adi<T, 32, 256, 32>(h, A, sims, st, pass_a);
            case 3: return launch_adi<T, 32, 256, 64>(h, A, sims, st, pass_a);
            case 4: return launch_adi<T, 32, 512, 64>(h, A, sims, st, pass_a);
        }
    }
    return set_error(PB_EINVAL, "bad ADI cfg");
}

// Tile configuration for a sweep of length n: the smallest per-CTA row span
// that covers n (one CTA per system group), else the largest span with a
// cluster of ceil(n / span) CTAs (<= 16).
// shared memory of pass A (the larger pass) for tile configuration k
static size_t adi_smem(int k, int dtype)
{
    const TileCfg *T = dtype == PB_F64 ? CFG64 : CFG32;
    const int W = dtype == PB_F64 ? 16 : 32;
    const size_t es = dtype == PB_F64 ? 8 : 4;
    const size_t RC = (size_t)(T[k].nt / W) * T[k].mr, PC = T[k].nt / W;
    const size_t dyn = es * (RC * (W + 1) + (W + 4) * (ADI_IB + 4) + (W + 2) * (ADI_IB + 2) + W * ADI_IB);
    const size_t stat = es * (4 * W * (PC + 1) + 2 * MAX_CLUSTER * W * 2 + 4 * W + 2 * W);
    return dyn + stat;
}

static int adi_choose(int64_t n, int dtype, int *C)
{
    const TileCfg *T = dtype == PB_F64 ? CFG64 : CFG32;
    const int W = dtype == PB_F64 ? 16 : 32;
    const size_t limit = 227 * 1024;
    for (int k = 0; k < NCFG; ++k) {
        int64_t rc = (int64_t)(T[k].nt / W) * T[k].mr;
        if (rc >= n && adi_smem(k, dtype) <= limit) {
            *C = 1;
            return k;
        }
    }
    // multi-CTA cluster: the largest row span whose pass A fits in shared memory
    for (int k = NCFG - 1; k >= 0; --k) {
        if (adi_smem(k, dtype) > limit) continue;
        int64_t rc = (int64_t)(T[k].nt / W) * T[k].mr;
        int64_t c = (n + rc - 1) / rc;
        if (c > MAX_CLUSTER) return -1;
        *C = (int)c;
        return k;
    }
    return -1;
}

static std::mutex g_adi_mu;
static std::map<std::tuple<int, int64_t, int, uint64_t>, Band *> g_adi_cache;

static int adi_band(int64_t n, double sigma, int dtype, cudaStream_t st, Band **out)
{
    int dev = 0;
    PB_CUDA_TRY(cudaGetDevice(&dev));
    uint64_t bits;
    memcpy(&bits, &sigma, sizeof(bits));
    auto key = std::make_tuple(dev, n, dtype, bits);
    std::lock_guard<std::mutex> lk(g_adi_mu);
    auto it = g_adi_cache.find(key);
    if (it != g_adi_cache.end()) {
        *out = it->second;
        return PB_OK;
    }
    int C = 1;
    int k = adi_choose(n, dtype, &C);
    if (k < 0) return set_error(PB_EUNSUPPORTED, "ADI grid n = %lld exceeds the 16-CTA cluster span", (long long)n);
    Band *h = nullptr;
    int rc = const_penta_band(n, sigma, dtype, k, C, st, &h);
    if (rc) return rc;
    g_adi_cache[key] = h;
    *out = h;
    return PB_OK;
}

// C^{n+1} = Cbar^{n+1} + v = 2 C^n - C^{n-1} + v, written over C^{n-1} (16-byte vectors)
template <typename T>
__global__ void adi_combine_kernel(int64_t count, const T *__restrict__ cn, T *__restrict__ cm, const T *__restrict__ v)
{
    using V = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
    constexpr int E = 16 / sizeof(T);
    const int64_t nv = count / E;
    const V *a = reinterpret_cast<const V *>(cn);
    const V *c = reinterpret_cast<const V *>(v);
    V *b = reinterpret_cast<V *>(cm);
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nv; k += (int64_t)gridDim.x * blockDim.x) {
        const V x = __ldcs(a + k), y = __ldcs(b + k), z = __ldcs(c + k);
        V o;
        const T *xs = reinterpret_cast<const T *>(&x), *ys = reinterpret_cast<const T *>(&y),
                *zs = reinterpret_cast<const T *>(&z);
        T *os = reinterpret_cast<T *>(&o);
#pragma unroll
        for (int e = 0; e < E; ++e) os[e] = (T(2) * xs[e] - ys[e]) + zs[e];
        __stcs(b + k, o);
    }
    for (int64_t k = nv * E + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count;
         k += (int64_t)gridDim.x * blockDim.x)
        cm[k] = (T(2) * cn[k] - cm[k]) + v[k];
}

// the same combine with v in the permuted layout v[(j * sims + sim) * n + i]
template <typename T>
__global__ void adi_combine_perm_kernel(int64_t sims, int64_t n, const T *__restrict__ cn, T *__restrict__ cm,
                                        const T *__restrict__ v)
{
    using V = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
    constexpr int E = 16 / sizeof(T);
    const int64_t nr = n / E, rows = sims * n;   // vectors per grid row; grid rows (sim, j)
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < rows * nr; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = k / nr, iv = k - row * nr, sim = row / n, j = row - sim * n;
        const V *a = reinterpret_cast<const V *>(cn + row * n) + iv;
        V *b = reinterpret_cast<V *>(cm + row * n) + iv;
        const V *c = reinterpret_cast<const V *>(v + (j * sims + sim) * n) + iv;
        const V x = __ldcs(a), y = __ldcs(b), z = __ldcs(c);
        V o;
        const T *xs = reinterpret_cast<const T *>(&x), *ys = reinterpret_cast<const T *>(&y),
                *zs = reinterpret_cast<const T *>(&z);
        T *os = reinterpret_cast<T *>(&o);
#pragma unroll
        for (int e = 0; e < E; ++e) os[e] = (T(2) * xs[e] - ys[e]) + zs[e];
        __stcs(b, o);
    }
}

template <typename T>
static int adi_run(pb_ch_state *s, double dt, const pb_ch_params *p, int64_t nsteps, cudaStream_t st)
{
    const int64_t n = s->n;
    const double dx = p->L / (double)n;  // r1
    const double sigma = (2.0 / 3.0) * p->D * p->gamma * dt / (dx * dx * dx * dx);
    Band *h = nullptr;
    int rc = adi_band(n, sigma, s->dtype, st, &h);
    if (rc) return rc;
    AdiArgs<T> A;
    A.core.coef = (const T *)h->coef;
    A.core.tab = (const T *)h->plan.tab;
    A.core.mfc = (const T *)h->plan.mfc;
    A.core.mbc = (const T *)h->plan.mbc;
    A.core.scal = h->scal;
    A.core.n = n;
    A.core.C = h->plan.C;
    for (int j = 0; j < 4; ++j) A.core.srow[j] = h->srow[j];
    A.n = n;
    A.k_dif = T(-2.0 / 3.0);
    A.k_bih = T(-(2.0 / 3.0) * dt * p->D * p->gamma / (dx * dx * dx * dx));
    A.k_lap = T((2.0 / 3.0) * p->D * dt / (dx * dx));
    A.w = (T *)s->work;
    // y-sweep: the fused streaming solve over ONE batch of sims * n interleaved systems
    // (w in the permuted layout) + the C^{n+1} combine; the fused band_core pass B
    // serves the rest (unaligned buffers)
    const bool ysweep_tp = h->fplan.ok && (n * (int64_t)sizeof(T)) % 16 == 0 && (uintptr_t)s->work % 16 == 0 &&
                           (uintptr_t)s->c_cur % 16 == 0 && (uintptr_t)s->c_prev % 16 == 0;
    A.wperm = ysweep_tp ? s->sims : 0;
    for (int64_t step = 0; step < nsteps; ++step) {
        A.cn = (const T *)s->c_cur;
        A.cm = (T *)s->c_prev;
        if ((rc = launch_adi_cfg<T>(h, A, s->sims, st, true))) return rc;
        if (ysweep_tp) {
            // y-sweep = the batched interleaved solve (systems = columns i, one batch
            // per simulation) by the two-pass TMA solve, then the C^{n+1} combine
            // (w is in the permuted layout: one batch of sims * n systems)
            if ((rc = launch_fused(h, A.w, 1, 0, st, s->sims * n))) return rc;
            int dev = 0, nsm = 0;
            PB_CUDA_TRY(cudaGetDevice(&dev));
            PB_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
            adi_combine_perm_kernel<T><<<(unsigned)(nsm * 8), 256, 0, st>>>(s->sims, n, A.cn, A.cm, A.w);
            PB_LAUNCH_CHECK();
        } else if ((rc = launch_adi_cfg<T>(h, A, s->sims, st, false))) {
            return rc;
        }
        void *t = s->c_prev;  // C^{n+1} now lives in the old C^{n-1} buffer
        s->c_prev = s->c_cur;
        s->c_cur = t;
    }
    return PB_OK;
}

}  // namespace pb

namespace pb {

// w [rows][n] -> packed [parts][rows][nb]: column block q becomes a contiguous
// [rows][nb] slab, the send layout of the all-to-all transpose.
template <typename T>
__global__ void dist_pack_kernel(int64_t rows, int64_t n, int64_t parts, const T *w, T *out)
{
    const int64_t nb = n / parts, total = rows * n;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = e / n, i = e % n, q = i / nb, ii = i % nb;
        out[(q * rows + j) * nb + ii] = w[e];
    }
}

// C^{n+1} = 2 C^n - C^{n-1} + v on the interior rows of a row block (written
// over C^{n-1}); v arrives as [parts][rows][nb] (block q = columns of rank q).
template <typename T>
__global__ void dist_combine_kernel(int64_t rows, int64_t n, int64_t parts, const T *cn, T *cm, const T *v)
{
    const int64_t nb = n / parts, total = rows * n;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = e / n, i = e % n, q = i / nb, ii = i % nb;
        const int64_t x = (j + 2) * n + i;
        cm[x] = (T(2) * cn[x] - cm[x]) + v[(q * rows + j) * nb + ii];
    }
}

template <typename T>
static int dist_pass_a(int64_t rows, int64_t n, const void *cn, const void *cm, void *w, double dt,
                       const pb_ch_params *p, cudaStream_t st)
{
    const double dx = p->L / (double)n;  // r1
    const double sigma = (2.0 / 3.0) * p->D * p->gamma * dt / (dx * dx * dx * dx);
    Band *h = nullptr;
    int rc = adi_band(n, sigma, sizeof(T) == 8 ? PB_F64 : PB_F32, st, &h);
    if (rc) return rc;
    AdiArgs<T> A;
    A.core.coef = (const T *)h->coef;
    A.core.tab = (const T *)h->plan.tab;
    A.core.mfc = (const T *)h->plan.mfc;
    A.core.mbc = (const T *)h->plan.mbc;
    A.core.scal = h->scal;
    A.core.n = n;
    A.core.C = h->plan.C;
    for (int j = 0; j < 4; ++j) A.core.srow[j] = h->srow[j];
    A.n = n;
    A.k_dif = T(-2.0 / 3.0);
    A.k_bih = T(-(2.0 / 3.0) * dt * p->D * p->gamma / (dx * dx * dx * dx));
    A.k_lap = T((2.0 / 3.0) * p->D * dt / (dx * dx));
    A.cn = (const T *)cn;
    A.cm = (T *)cm;
    A.w = (T *)w;
    A.rows = rows;
    A.ext = 1;
    return launch_adi_cfg<T>(h, A, 1, st, true);
}

}  // namespace pb

extern "C" int ch_dist_pass_a(int64_t rows, int64_t n, int dtype, const void *cn_ext, const void *cm_ext, void *w,
                              double dt, const pb_ch_params *p, void *stream)
{
    using namespace pb;
    if (!p || !cn_ext || !cm_ext || !w || rows < 1 || n < 8 || rows > n) return set_error(PB_EINVAL, "bad args");
    if (dtype != PB_F64 && dtype != PB_F32) return set_error(PB_EINVAL, "bad dtype");
    if (!(dt > 0) || !(p->L > 0)) return set_error(PB_EINVAL, "dt and L must be positive");
    if (pb_device_ok() != PB_OK) return PB_ECUDA;
    if (!is_device_ptr(cn_ext) || !is_device_ptr(cm_ext) || !is_device_ptr(w))
        return set_error(PB_EINVAL, "ch_dist_pass_a buffers must be device memory");
    cudaStream_t st = (cudaStream_t)stream;
    return dtype == PB_F64 ? dist_pass_a<double>(rows, n, cn_ext, cm_ext, w, dt, p, st)
                           : dist_pass_a<float>(rows, n, cn_ext, cm_ext, w, dt, p, st);
}

// y-sweep of a rank's column block (configs[4]): L_y v = w along j for ncols
// interleaved columns of length n, in place, with the cached cyclic L_y.
extern "C" int ch_dist_ysweep(int64_t ncols, int64_t n, int dtype, void *cols, double dt, const pb_ch_params *p,
                              void *stream)
{
    using namespace pb;
    if (!p || !cols || ncols < 1 || n < 8) return set_error(PB_EINVAL, "bad args");
    if (dtype != PB_F64 && dtype != PB_F32) return set_error(PB_EINVAL, "bad dtype");
    if (!(dt > 0) || !(p->L > 0)) return set_error(PB_EINVAL, "dt and L must be positive");
    if ((ncols * (int64_t)dtype_size(dtype)) % 16 || (uintptr_t)cols % 16)
        return set_error(PB_EINVAL, "ch_dist_ysweep needs 16-byte aligned rows (ncols * sizeof(T) % 16 == 0)");
    if (pb_device_ok() != PB_OK) return PB_ECUDA;
    if (!is_device_ptr(cols)) return set_error(PB_EINVAL, "ch_dist_ysweep buffers must be device memory");
    cudaStream_t st = (cudaStream_t)stream;
    const double dx = p->L / (double)n;  // r1
    const double sigma = (2.0 / 3.0) * p->D * p->gamma * dt / (dx * dx * dx * dx);
    Band *h = nullptr;
    int rc = adi_band(n, sigma, dtype, st, &h);
    if (rc) return rc;
    if (!h->fplan.ok) return set_error(PB_EUNSUPPORTED, "no streaming plan for n = %lld", (long long)n);
    return launch_fused(h, cols, 1, 0, st, ncols);
}

extern "C" int ch_dist_pack(int64_t rows, int64_t n, int64_t parts, int dtype, const void *w, void *packed,
                            void *stream)
{
    using namespace pb;
    if (!w || !packed || rows < 1 || parts < 1 || n % parts) return set_error(PB_EINVAL, "bad args");
    if (dtype != PB_F64 && dtype != PB_F32) return set_error(PB_EINVAL, "bad dtype");
    if (pb_device_ok() != PB_OK) return PB_ECUDA;
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned g = (unsigned)std::min<int64_t>((rows * n + 255) / 256, 148 * 16);
    if (dtype == PB_F64)
        dist_pack_kernel<double><<<g, 256, 0, st>>>(rows, n, parts, (const double *)w, (double *)packed);
    else
        dist_pack_kernel<float><<<g, 256, 0, st>>>(rows, n, parts, (const float *)w, (float *)packed);
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
                                                      (const float *)v_packed);
    PB_LAUNCH_CHECK();
    return PB_OK;
}

extern "C" int ch_workspace_bytes(int64_t sims, int64_t n, int dtype, size_t *bytes)
{
    using namespace pb;
    if (!bytes || sims < 0 || n < 8 || (dtype != PB_F64 && dtype != PB_F32)) return set_error(PB_EINVAL, "bad args");
    *bytes = dtype_size(dtype) * (size_t)sims * (size_t)n * (size_t)n;
    return PB_OK;
}

extern "C" int ch_adi_step(pb_ch_state *s, double dt, const pb_ch_params *p, int64_t nsteps, void *stream)
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
    if (!is_device_ptr(s->c_cur) || !is_device_ptr(s->c_prev) || !is_device_ptr(s->work))
        return set_error(PB_EINVAL, "ch_adi_step buffers must be device memory");
    cudaStream_t st = (cudaStream_t)stream;
    return s->dtype == PB_F64 ? adi_run<double>(s, dt, p, nsteps, st) : adi_run<float>(s, dt, p, nsteps, st);
}

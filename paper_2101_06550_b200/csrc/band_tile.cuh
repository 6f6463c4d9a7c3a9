// band_tile.cuh — the shared-LHS tile kernel (band_core + global load/store)
// and its launcher; instantiated per (dtype, K) in banded_inst_*.cu so the
// nvcc builds run in parallel.
#pragma once
#include <map>
#include <mutex>

#include "band_core.cuh"
#include "common.cuh"

namespace pb {

// ---------------------------------------------------------------- handle
struct Plan {
    int nt = 0, mr = 0, w = 0, C = 0;
    int64_t nchunks = 0;
    void *tab = nullptr, *mfc = nullptr, *mbc = nullptr;  // dtype scan tables (band_core.cuh)
};

// fused streaming solve plan (fused_solve.cuh): row records, chunk maps,
// cyclic-row responses (dtype), and per-stream scratch.  Solves on different
// streams get different scratch (concurrent solves with one handle are safe);
// solves on one stream reuse theirs in stream order.
struct FusedScratch {
    void *buf = nullptr;
    size_t bytes = 0;
    int64_t nq = 0, nsys = 0;
    // two-pass solve (twopass.cuh): chunk records, cyclic rows, x_l; grow-only
    void *tbuf = nullptr;
    size_t tbytes = 0;
    // the last tensor map encoded for this stream, per layout (rhs pointer + shape key)
    uint64_t key[2][6] = {{0, 0, 0, 0, 0, 0}, {0, 0, 0, 0, 0, 0}};
    alignas(64) unsigned char tmap[2][128];
};
struct FusedPlan {
    int ok = 0, nq = 0;
    void *rec = nullptr, *ct = nullptr, *rsp = nullptr;
    mutable std::mutex mu;
    mutable std::map<cudaStream_t, FusedScratch> scratch;
    mutable cudaStream_t pipe[3] = {nullptr, nullptr, nullptr};   // internal streams of the host-buffer pipeline
};

struct Band {
    int K = 2;  // 2 = penta, 1 = tri
    int64_t batch = 0, n = 0, lhs_count = 1;
    int periodic = 0, dtype = PB_F64;
    // shared LHS
    int64_t rows_alloc = 0;
    double *coefD = nullptr;  // fp64 master (rows_alloc x 8)
    void *coef = nullptr;     // dtype copy (== coefD for fp64)
    double *scal = nullptr;   // SCAL_LEN
    Plan plan;
    FusedPlan fplan;
    int64_t srow[4] = {-1, -1, -1, -1};
    // the 64-row chunk maps of the factored LHS grow (max |Mf_q|, |Mb_q| >= 1):
    // chunked solves would amplify rounding through the carry scan, so this
    // handle is solved sequentially, one thread per system (the thesis's kernel)
    bool seq_only = false;
    double chunk_growth = 0.0;
    // per-system LHS
    void *pcoef = nullptr;    // dtype, [(i*8 + j) * batch + s]
    double *pscal = nullptr;  // [j * batch + s]
    double *pcoefD = nullptr; // fp64 factor scratch of fp32 per-system handles (pent_refactor)
    int64_t *rstatus = nullptr;   // device status of pent_refactor (never read back on the hot path)
    bool shared() const { return lhs_count == 1; }
    ~Band()
    {
        if (coef && coef != coefD) cudaFree(coef);
        cudaFree(coefD);
        cudaFree(scal);
        cudaFree(plan.tab);
        cudaFree(plan.mfc);
        cudaFree(plan.mbc);
        cudaFree(pcoef);
        cudaFree(pscal);
        cudaFree(pcoefD);
        cudaFree(rstatus);
        cudaFree(fplan.rec);
        cudaFree(fplan.ct);
        cudaFree(fplan.rsp);
        if (!fplan.scratch.empty() || fplan.pipe[0]) cudaDeviceSynchronize();   // queued solves may use the scratch
        for (auto &kv : fplan.scratch) {
            cudaFree(kv.second.buf);
            cudaFree(kv.second.tbuf);
        }
        for (auto s : fplan.pipe)
            if (s) cudaStreamDestroy(s);
    }
};

// ---------------------------------------------------------------- shared-LHS tile kernel
template <typename T>
struct TileArgs {
    CoreArgs<T> core;
    T *x;
    int64_t M, bstride;
};

template <typename T>
__device__ __forceinline__ T ld_stream(const T *p) { return __ldcs(p); }
template <typename T>
__device__ __forceinline__ void st_stream(T *p, T v) { __stcs(p, v); }

template <typename T, int K, int W, int NT, int MR, bool PER, int LAYOUT>
__global__ void __launch_bounds__(NT, (NT <= 256 ? 2 : 1)) band_tile_kernel(const TileArgs<T> A)
{
    constexpr int PC = NT / W;
    constexpr int RC = PC * MR;
    __shared__ CoreSmem<T, W, PC> S;
    extern __shared__ __align__(16) unsigned char dyn_smem[];
    const int tid = threadIdx.x, s = tid % W, p = tid / W;
    const int C = A.core.C;
    const int c = (C > 1) ? (int)cg::this_cluster().block_rank() : 0;
    const int64_t group = blockIdx.x / C;
    const int64_t sys = group * W + s;
    const int64_t N = A.core.n, M = A.M;
    const int64_t row0 = (int64_t)c * RC, r0 = row0 + (int64_t)p * MR;
    T *X = A.x + (int64_t)blockIdx.y * A.bstride;
    T *cs = reinterpret_cast<T *>(dyn_smem);       // [RC][8] coefficient rows of this CTA
    stage_coef<T, NT>(cs, A.core.coef + row0 * COEF_STRIDE, RC);
    T v[MR];
    if (LAYOUT == PB_INTERLEAVED) {
        // lanes = W consecutive systems of one row: W*sizeof(T) contiguous bytes
        const bool ok = sys < M;
        const T *src = X + r0 * M + sys;
#pragma unroll
        for (int k = 0; k < MR; ++k) v[k] = (ok && r0 + k < N) ? ld_stream(src + k * M) : T(0);
    } else {
        // systems contiguous: coalesced loads along the row, transposed into a
        // padded smem tile [RC][W+1] (conflict-free both ways)
        T *tile = cs + RC * COEF_STRIDE;
        for (int e = tid; e < W * RC; e += NT) {
            const int ss = e / RC, rr = e % RC;
            const int64_t sy = group * W + ss, r = row0 + rr;
            tile[rr * (W + 1) + ss] = (sy < M && r < N) ? ld_stream(X + sy * N + r) : T(0);
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < MR; ++k) v[k] = tile[(p * MR + k) * (W + 1) + s];
    }
    __syncthreads();  // coefficient table (and contiguous tile) staged
    band_core<T, K, W, NT, MR, PER>(v, A.core, S, cs, c, s, p, r0);
    if (LAYOUT == PB_INTERLEAVED) {
        // opaque stride: recompute the store addresses instead of keeping the
        // MR load addresses live across the solve (register pressure)
        int64_t Mo = M;
        asm volatile("" : "+l"(Mo));
        if (sys < M) {
            T *dst = X + r0 * Mo + sys;
#pragma unroll
            for (int k = 0; k < MR; ++k)
                if (r0 + k < N) st_stream(dst + k * Mo, v[k]);
        }
    } else {
        T *tile = cs + RC * COEF_STRIDE;
#pragma unroll
        for (int k = 0; k < MR; ++k) tile[(p * MR + k) * (W + 1) + s] = v[k];
        __syncthreads();
        for (int e = tid; e < W * RC; e += NT) {
            const int ss = e / RC, rr = e % RC;
            const int64_t sy = group * W + ss, r = row0 + rr;
            if (sy < M && r < N) st_stream(X + sy * N + r, tile[rr * (W + 1) + ss]);
        }
    }
}


struct TileCfg {
    int nt, mr;
};
// fp64: W = 16 systems per CTA (128 B per row); fp32: W = 32 (128 B per row)
static const TileCfg CFG64[] = {{256, 4}, {256, 8}, {256, 16}, {256, 32}, {512, 32}};
static const TileCfg CFG32[] = {{256, 8}, {256, 16}, {256, 32}, {256, 64}, {512, 64}};
constexpr int NCFG = 5;

template <typename KernT>
static int prep_kernel(KernT kern, size_t dyn, int C)
{
    // idempotent attribute setup (cheap; cached by the runtime)
    // static + dynamic > 48 KB needs the opt-in even when dyn itself is small
    if (dyn > 0) PB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    if (C > 8) PB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    return PB_OK;
}

template <typename T, int K, int W, int NT, int MR, bool PER, int LAYOUT>
static int launch_tile_t(const Band *h, T *x, int64_t count, int64_t bstride, cudaStream_t st)
{
    auto kern = band_tile_kernel<T, K, W, NT, MR, PER, LAYOUT>;
    constexpr int RC = (NT / W) * MR;
    const int C = h->plan.C;
    const size_t dyn = sizeof(T) * ((size_t)RC * COEF_STRIDE + (LAYOUT == PB_CONTIGUOUS ? (size_t)RC * (W + 1) : 0));
    int rc = prep_kernel(kern, dyn, C);
    if (rc) return rc;
    TileArgs<T> A;
    A.core.coef = (const T *)h->coef;
    A.core.tab = (const T *)h->plan.tab;
    A.core.mfc = (const T *)h->plan.mfc;
    A.core.mbc = (const T *)h->plan.mbc;
    A.core.scal = h->scal;
    A.core.n = h->n;
    A.core.C = C;
    for (int j = 0; j < 4; ++j) A.core.srow[j] = h->srow[j];
    A.x = x;
    A.M = h->batch;
    A.bstride = bstride;
    const int64_t groups = (h->batch + W - 1) / W;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(groups * C), (unsigned)count, 1);
    cfg.blockDim = dim3(NT, 1, 1);
    cfg.dynamicSmemBytes = dyn;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = C > 1 ? 1 : 0;
    PB_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, A));
    PB_LAUNCH_CHECK();
    return PB_OK;
}

template <typename T, int K, int W, int NT, int MR>
static int launch_tile_l(const Band *h, T *x, int layout, int64_t count, int64_t bstride, cudaStream_t st)
{
    const bool per = h->periodic != 0;
    if (layout == PB_INTERLEAVED)
        return per ? launch_tile_t<T, K, W, NT, MR, true, PB_INTERLEAVED>(h, x, count, bstride, st)
                   : launch_tile_t<T, K, W, NT, MR, false, PB_INTERLEAVED>(h, x, count, bstride, st);
    return per ? launch_tile_t<T, K, W, NT, MR, true, PB_CONTIGUOUS>(h, x, count, bstride, st)
               : launch_tile_t<T, K, W, NT, MR, false, PB_CONTIGUOUS>(h, x, count, bstride, st);
}



int const_penta_band(int64_t n, double sigma, int dtype, int cfg, int C, cudaStream_t st, Band **out);

int fused_build_tables(Band *h, cudaStream_t st);
// the cluster configuration {CS, cpc, clusters} of a fused solve of M x count systems
// (CS = 0: the global-scan kernel serves)
int fused_info(const Band *h, int layout, int64_t M, int64_t count, int *info);
// the dispatching solves behind pent_solve / pent_solve_many / pent_solve_strided / tri_*
int band_solve(const Band *h, void *rhs, int layout, int64_t count, int64_t bstride, cudaStream_t st);
int band_solve_layout(const Band *h, void *rhs, const pb_layout &L, cudaStream_t st);
// shared-LHS solve of `count` batches (batch k at x + k * bstride elements) in
// `layout` (PB_INTERLEAVED / PB_CONTIGUOUS); M = systems per batch (0: the
// handle's); pitch = elements between rows (interleaved) / systems (contiguous),
// 0 = packed
int launch_fused(const Band *h, void *x, int layout, int64_t count, int64_t bstride, cudaStream_t st, int64_t M = 0,
                 int64_t pitch = 0);
// one step of the batched 1D Cahn–Hilliard scheme (fused_solve.cuh MODE_CH1D):
// c -> cnew, M interleaved systems, alpha = dt/dx^2, h = the cyclic (s,-4s,1+6s,-4s,s)
int launch_fused_ch1d(const Band *h, const void *c, void *cnew, double alpha, int64_t M, cudaStream_t st);

// per-(dtype, K) entry points, defined in banded_inst_*.cu
int launch_tile_f64_k2(const Band *h, void *x, int layout, int64_t count, int64_t bstride, cudaStream_t st);
int launch_tile_f64_k1(const Band *h, void *x, int layout, int64_t count, int64_t bstride, cudaStream_t st);
int launch_tile_f32_k2(const Band *h, void *x, int layout, int64_t count, int64_t bstride, cudaStream_t st);
int launch_tile_f32_k1(const Band *h, void *x, int layout, int64_t count, int64_t bstride, cudaStream_t st);

}  // namespace pb

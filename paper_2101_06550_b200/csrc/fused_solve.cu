// fused_solve.cu — tables and host launcher of the fused streaming solve
// (fused_solve.cuh), both dtypes, penta (K = 2) and tri (K = 1).
#include <cudaTypedefs.h>
#include <math.h>
#include <string.h>

#include <array>
#include <vector>

#include "band_tile.cuh"
#include "fused_solve.cuh"

namespace pb {

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();

// One thread per chunk q (rows r0 .. r0+kmax-1), fp64 from the master coefficients.
//   rec[r]  = (F0, F1, F2, alpha_r, beta_r, 0): alpha/beta are the weights of g_r
//             in (x_{r0}, x_{r0+1}) of the chunk's back substitution with zero
//             inflow, i.e. rows r0, r0+1 of L^{-1} (L unit upper, L[j][j+1] = B1_j,
//             L[j][j+2] = B2_j): L^T alpha = e_{r0}, solved forward in r.
//   ct[q]   = Mf (inflow (g_{r0-2}, g_{r0-1}) -> outflow, f = 0),
//             Mb ((x_{r1}, x_{r1+1}) -> (x_{r0}, x_{r0+1}), g = 0),
//             H  (forward inflow -> zero-inflow back-substitution carry).
//   rsp[j]  = g on row srow[j] per unit forward inflow of its chunk.
template <typename T>
__global__ void fs_tables_kernel(const double *coef, int K, int64_t n, int nq, int64_t s0, int64_t s1, int64_t s2,
                                 int64_t s3, T *rec, T *ct, T *rsp)
{
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    const int64_t srow[4] = {s0, s1, s2, s3};
    const int64_t r0 = (int64_t)q * fs::Q;
    const int kmax = (int)min((int64_t)fs::Q, n - r0);
    const double *cr = coef + r0 * COEF_STRIDE;
    auto F1 = [&](int i) { return cr[i * COEF_STRIDE + 1]; };
    auto F2 = [&](int i) { return K == 2 ? cr[i * COEF_STRIDE + 2] : 0.0; };
    auto B1 = [&](int i) { return cr[i * COEF_STRIDE + 4]; };
    auto B2 = [&](int i) { return K == 2 ? cr[i * COEF_STRIDE + 5] : 0.0; };
    double am1 = 0, am2 = 0, bm1 = 0, bm2 = 0;
    double al[fs::Q], be[fs::Q];
    for (int i = 0; i < kmax; ++i) {
        const double b1 = i >= 1 ? B1(i - 1) : 0.0, b2 = i >= 2 ? B2(i - 2) : 0.0;
        const double a = (i == 0 ? 1.0 : 0.0) - b1 * am1 - b2 * am2;
        const double b = (i == 1 ? 1.0 : 0.0) - b1 * bm1 - b2 * bm2;
        am2 = am1, am1 = a, bm2 = bm1, bm1 = b;
        al[i] = a, be[i] = b;
        T *o = rec + (r0 + i) * fs::REC;
        o[0] = (T)cr[i * COEF_STRIDE + 0];
        o[1] = (T)F1(i);
        o[2] = (T)F2(i);
        o[3] = (T)a;
        o[4] = (T)b;
        o[5] = T(0);
    }
    for (int i = kmax; i < fs::Q; ++i)
        for (int j = 0; j < fs::REC; ++j) rec[(r0 + i) * fs::REC + j] = T(0);
    T *m = ct + (int64_t)q * 12;
    for (int col = 0; col < 2; ++col) {
        double y0 = col == 0, y1 = col == 1, h0 = 0, h1 = 0;
        for (int i = 0; i < kmax; ++i) {
            const double g = -F1(i) * y1 - F2(i) * y0;
            y0 = y1, y1 = g;
            h0 += al[i] * g;
            h1 += be[i] * g;
            for (int j = 0; j < 4; ++j)
                if (srow[j] == r0 + i) rsp[j * 2 + col] = (T)g;
        }
        m[0 + col] = (T)y0;
        m[2 + col] = (T)y1;
        m[8 + col] = (T)h0;
        m[10 + col] = (T)h1;
        double z0 = col == 0, z1 = col == 1;
        for (int i = kmax - 1; i >= 0; --i) {
            const double x = -B1(i) * z0 - B2(i) * z1;
            z1 = z0, z0 = x;
        }
        m[4 + col] = (T)z0;
        m[6 + col] = (T)z1;
    }
}

int fused_build_tables(Band *h, cudaStream_t st)
{
    const size_t es = dtype_size(h->dtype);
    const int64_t nq = (h->n + fs::Q - 1) / fs::Q;
    h->fplan.ok = 0;
    if (nq > (1 << 24) || h->rows_alloc < nq * fs::Q || !tensor_map_encoder()) return PB_OK;
    PB_CUDA_TRY(cudaMalloc(&h->fplan.rec, es * fs::REC * nq * fs::Q));
    PB_CUDA_TRY(cudaMalloc(&h->fplan.ct, es * 12 * nq));
    PB_CUDA_TRY(cudaMalloc(&h->fplan.rsp, es * 8));
    PB_CUDA_TRY(cudaMemsetAsync(h->fplan.rsp, 0, es * 8, st));
    const unsigned g = (unsigned)((nq + 63) / 64);
    if (h->dtype == PB_F64)
        fs_tables_kernel<double><<<g, 64, 0, st>>>(h->coefD, h->K, h->n, (int)nq, h->srow[0], h->srow[1], h->srow[2],
                                                   h->srow[3], (double *)h->fplan.rec, (double *)h->fplan.ct,
                                                   (double *)h->fplan.rsp);
    else
        fs_tables_kernel<float><<<g, 64, 0, st>>>(h->coefD, h->K, h->n, (int)nq, h->srow[0], h->srow[1], h->srow[2],
                                                  h->srow[3], (float *)h->fplan.rec, (float *)h->fplan.ct,
                                                  (float *)h->fplan.rsp);
    PB_LAUNCH_CHECK();
    h->fplan.nq = (int)nq;
    h->fplan.ok = 1;
    return PB_OK;
}

// Windowed inflows (fused_solve.cuh): the smallest L <= LMAX such that every
// product of L, L+1 and L+2 consecutive chunk maps (forward Mf, backward Mb) is
// below WIN_TOL in max-norm, so truncating the scan sums at L chunks changes
// nothing at fp64 rounding; a chunk needs x_l if its rows' cyclic correction
// columns Z1, Z2 exceed WIN_TOL (or it holds the last two unknowns, = x_l).
constexpr double WIN_TOL = 1e-18;

int fused_window_plan(Band *h)
{
    FusedPlan &P = h->fplan;
    P.win = 0;
    if (!P.ok) return PB_OK;
    const int64_t n = h->n, nq = P.nq, rows = h->rows_alloc;
    std::vector<double> cf((size_t)rows * COEF_STRIDE);
    PB_CUDA_TRY(cudaMemcpy(cf.data(), h->coefD, sizeof(double) * cf.size(), cudaMemcpyDeviceToHost));
    auto C = [&](int64_t r, int j) { return (h->K == 1 && (j == 2 || j == 5)) ? 0.0 : cf[(size_t)r * COEF_STRIDE + j]; };
    std::vector<std::array<double, 4>> mf(nq), mb(nq);
    for (int64_t q = 0; q < nq; ++q) {
        const int64_t r0 = q * fs::Q, kmax = std::min<int64_t>(fs::Q, n - r0);
        for (int col = 0; col < 2; ++col) {
            double y0 = col == 0, y1 = col == 1;
            for (int64_t i = 0; i < kmax; ++i) {
                const double g = -C(r0 + i, 1) * y1 - C(r0 + i, 2) * y0;
                y0 = y1, y1 = g;
            }
            mf[q][0 + col] = y0, mf[q][2 + col] = y1;
            double z0 = col == 0, z1 = col == 1;
            for (int64_t i = kmax - 1; i >= 0; --i) {
                const double x = -C(r0 + i, 4) * z0 - C(r0 + i, 5) * z1;
                z1 = z0, z0 = x;
            }
            mb[q][0 + col] = z0, mb[q][2 + col] = z1;
        }
    }
    auto mul = [](const std::array<double, 4> &a, const std::array<double, 4> &b) {
        return std::array<double, 4>{a[0] * b[0] + a[1] * b[2], a[0] * b[1] + a[1] * b[3], a[2] * b[0] + a[3] * b[2],
                                     a[2] * b[1] + a[3] * b[3]};
    };
    auto nrm = [](const std::array<double, 4> &a) {
        return std::max(std::max(fabs(a[0]), fabs(a[1])), std::max(fabs(a[2]), fabs(a[3])));
    };
    for (int L = 1; L <= fs::LMAX && !P.win; ++L) {
        bool ok = true;
        for (int64_t q = 0; q < nq && ok; ++q) {
            std::array<double, 4> F = {1, 0, 0, 1}, B = {1, 0, 0, 1};
            for (int l = 1; l <= L + 2 && q + l - 1 < nq; ++l) {
                F = mul(mf[q + l - 1], F);   // Mf_{q+l-1} .. Mf_q
                B = mul(B, mb[q + l - 1]);   // Mb_q .. Mb_{q+l-1}
                if (l >= L && (nrm(F) >= WIN_TOL || nrm(B) >= WIN_TOL)) ok = false;
            }
        }
        if (ok) P.win = L;
    }
    if (P.win && h->periodic) {
        std::vector<unsigned char> nx((size_t)nq, 0);
        for (int64_t r = 0; r < n; ++r)
            if (fabs(C(r, 6)) >= WIN_TOL || fabs(C(r, 7)) >= WIN_TOL || (h->K == 2 && r >= n - 2)) nx[r / fs::Q] = 1;
        PB_CUDA_TRY(cudaMalloc(&P.needxl, (size_t)nq));
        PB_CUDA_TRY(cudaMemcpy(P.needxl, nx.data(), (size_t)nq, cudaMemcpyHostToDevice));
    }
    return PB_OK;
}

// L2 budget for the lag window of f between P1(g) and P2(g) (the L2 is 126 MB;
// the window, the x write-back in flight and the scratch records share it)
constexpr double FS_L2_BUDGET = 40.0 * 1048576.0;       // group-scan mode (scan latency to cover)
constexpr double FS_L2_BUDGET_WIN = 24.0 * 1048576.0;   // windowed mode

static int sm_count()
{
    static int cached[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (dev < 64 && cached[dev]) return cached[dev];
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (dev < 64) cached[dev] = nsm;
    return nsm;
}

template <typename T, int K, bool PER, int MODE, int LAY>
static int fs_launch_t(const Band *h, T *x, T *xout, double alpha, int64_t count, int64_t bstride, cudaStream_t st,
                       int64_t Mo, int64_t pitch)
{
    auto kern = fs::fs_kernel<T, K, PER, MODE, LAY>;
    const size_t smem = sizeof(fs::Smem<T>) + 1024;   // + alignment to 1 KB
    static std::once_flag attr_once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(attr_once, [&] {
        attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    if (attr_err != cudaSuccess) return set_error(PB_ECUDA, "fs_kernel smem attribute: %s", cudaGetErrorString(attr_err));

    const int64_t M = Mo > 0 ? Mo : h->batch, n = h->n;
    const int64_t dpitch = LAY == fs::LAY_CONTIG ? n : M;   // the packed pitch
    const int64_t P = pitch > 0 ? pitch : dpitch;
    const int nq = h->fplan.nq;
    const int64_t Gb = (M + fs::TW - 1) / fs::TW, G = Gb * count;
    if (G > INT32_MAX / 2) return set_error(PB_EINVAL, "too many systems for one launch");
    const int64_t nsys = G * fs::TW;
    const int64_t items = 2 * G * nq, nclaims = (items + fs::NC - 1) / fs::NC;
    const size_t es = sizeof(T);
    // scratch: car [nq][nsys][4], spec [nsys][4], xl [nsys][2], cnt [G], flag [G], tick [4]
    // (tick[2] CTAs done, tick[3] launches done)
    const size_t off_spec = es * (size_t)nq * nsys * 4, off_xl = off_spec + es * nsys * 4;
    const size_t off_cnt = (off_xl + es * nsys * 2 + 255) / 256 * 256;
    const size_t off_flag = off_cnt + 4 * (size_t)G, off_tick = off_flag + 4 * (size_t)G;
    const size_t need = off_tick + 16;   // tick[4]

    fs::Args<T> A;
    {
        std::lock_guard<std::mutex> lk(h->fplan.mu);
        FusedScratch &S = h->fplan.scratch[st];
        if (need > S.bytes) {
            if (S.buf) {
                PB_CUDA_TRY(cudaStreamSynchronize(st));   // queued solves may still use the old scratch
                cudaFree(S.buf);
                S.buf = nullptr;
                S.bytes = 0;
            }
            PB_CUDA_TRY(cudaMalloc(&S.buf, need));
            S.bytes = need;
            S.nq = S.nsys = -1;
            memset(S.key, 0, sizeof(S.key));
        }
        char *base = (char *)S.buf;
        if (S.nq != nq || S.nsys != nsys) {
            // fresh scratch or new shape (the counters live at shape-dependent
            // offsets): clear counters, flags and tickets; epochs restart at 1
            PB_CUDA_TRY(cudaMemsetAsync(base + off_cnt, 0, need - off_cnt, st));
            S.nq = nq;
            S.nsys = nsys;
        }
        A.car = (T *)base;
        A.spec = (T *)(base + off_spec);
        A.xl = (T *)(base + off_xl);
        A.cnt = (unsigned *)(base + off_cnt);
        A.flag = (unsigned *)(base + off_flag);
        A.tick = (unsigned *)(base + off_tick);

        // tensor map over x, cached per stream.  Interleaved: dims (M, n, count),
        // box (32 systems, 64 rows, 1); contiguous: dims (n, M, count), box
        // (128 B of rows, 32 systems, 1), 128B swizzle.  OOB loads zero-fill and
        // OOB stores are clipped (ragged M and n).  Contiguous batches that tiles
        // cannot straddle use one 2-D view.
        const bool flat = P == dpitch && (LAY == fs::LAY_CONTIG
                              ? (count == 1 || (bstride == M * n && M % fs::TW == 0))
                              : (count == 1 || (bstride == M * n && n % fs::Q == 0 && n * count < ((int64_t)1 << 31))));
        const uint64_t key[6] = {(uint64_t)(uintptr_t)x, (uint64_t)M, (uint64_t)n, (uint64_t)count,
                                 (uint64_t)bstride, (uint64_t)P * 16 + sizeof(T) * 2 + LAY};
        uint64_t *skey = S.key[LAY];
        void *smap = S.tmap[LAY];
        if (memcmp(key, skey, sizeof(key)) != 0) {
            auto enc = tensor_map_encoder();
            if (!enc) return set_error(PB_ECUDA, "cuTensorMapEncodeTiled unavailable");
            const auto dt = sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
            const int rank = flat ? 2 : 3;
            const int64_t bs = count > 1 ? bstride : P * (LAY == fs::LAY_CONTIG ? M : n);
            CUresult r;
            cuuint32_t estr[3] = {1, 1, 1};
            if (LAY == fs::LAY_CONTIG) {
                cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)(flat ? M * count : M), (cuuint64_t)(flat ? 1 : count)};
                cuuint64_t strides[2] = {(cuuint64_t)(P * sizeof(T)), (cuuint64_t)(bs * sizeof(T))};
                cuuint32_t box[3] = {(cuuint32_t)fs::Sw<T>::EB, (cuuint32_t)fs::TW, 1};
                r = enc((CUtensorMap *)smap, dt, rank, (void *)x, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            } else {
                cuuint64_t dims[3] = {(cuuint64_t)M, (cuuint64_t)(flat ? n * count : n), (cuuint64_t)(flat ? 1 : count)};
                cuuint64_t strides[2] = {(cuuint64_t)(P * sizeof(T)), (cuuint64_t)(bs * sizeof(T))};
                cuuint32_t box[3] = {(cuuint32_t)fs::TW, (cuuint32_t)fs::Q, 1};
                r = enc((CUtensorMap *)smap, dt, rank, (void *)x, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            }
            if (r != CUDA_SUCCESS) return set_error(PB_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
            memcpy(skey, key, sizeof(key));
        }
        A.flat = flat ? 1 : 0;
        CUtensorMap tmap;
        memcpy(&tmap, smap, sizeof(tmap));

        A.rec = (const T *)h->fplan.rec;
        A.coef = (const T *)h->coef;
        A.ct = (const T *)h->fplan.ct;
        A.rsp = (const T *)h->fplan.rsp;
        A.scal = h->scal;
        A.x = x;
        A.xout = xout;
        A.alpha = (T)alpha;
        A.bstride = count > 1 ? bstride : P * (LAY == fs::LAY_CONTIG ? M : n);
        A.pitch = P;
        A.n = n;
        A.M = M;
        A.nsys = nsys;
        A.items = items;
        A.nclaims = nclaims;
        for (int j = 0; j < 4; ++j) A.srow[j] = h->srow[j];
        A.nq = nq;
        A.count = (int)count;
        A.Gb = (int)Gb;
        A.G = (int)G;
        const double gbytes = (double)fs::TW * (double)n * (double)es;
        A.win = h->fplan.win;
        A.needxl = h->fplan.needxl;
        int64_t D = (int64_t)((A.win ? FS_L2_BUDGET_WIN : FS_L2_BUDGET) / gbytes);
        A.D = (int)(D < 1 ? 1 : (D > G ? G : D));
        A.qspec = PER ? (int)(h->srow[0] / fs::Q) : nq;
        const int grid = (int)std::min<int64_t>(sm_count(), nclaims);
        // cooperative: all CTAs co-resident (the static work deal relies on it).
        // Launched under the lock: the scratch (and its cached map) is not
        // re-laid-out between this launch's setup and its enqueue
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)grid);
        cfg.blockDim = dim3(fs::NTHREADS);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        PB_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, tmap, A));
        PB_LAUNCH_CHECK();
    }
    return PB_OK;
}

template <typename T, int LAY>
static int fs_launch_dl(const Band *h, void *x, int64_t count, int64_t bstride, cudaStream_t st, int64_t M,
                        int64_t pitch)
{
    T *X = (T *)x;
    using namespace fs;
    if (h->K == 2)
        return h->periodic ? fs_launch_t<T, 2, true, MODE_SOLVE, LAY>(h, X, X, 0.0, count, bstride, st, M, pitch)
                           : fs_launch_t<T, 2, false, MODE_SOLVE, LAY>(h, X, X, 0.0, count, bstride, st, M, pitch);
    return h->periodic ? fs_launch_t<T, 1, true, MODE_SOLVE, LAY>(h, X, X, 0.0, count, bstride, st, M, pitch)
                       : fs_launch_t<T, 1, false, MODE_SOLVE, LAY>(h, X, X, 0.0, count, bstride, st, M, pitch);
}

int launch_fused(const Band *h, void *x, int layout, int64_t count, int64_t bstride, cudaStream_t st, int64_t M,
                 int64_t pitch)
{
    if (layout == PB_CONTIGUOUS)
        return h->dtype == PB_F64 ? fs_launch_dl<double, fs::LAY_CONTIG>(h, x, count, bstride, st, M, pitch)
                                  : fs_launch_dl<float, fs::LAY_CONTIG>(h, x, count, bstride, st, M, pitch);
    return h->dtype == PB_F64 ? fs_launch_dl<double, fs::LAY_INTER>(h, x, count, bstride, st, M, pitch)
                              : fs_launch_dl<float, fs::LAY_INTER>(h, x, count, bstride, st, M, pitch);
}

int launch_fused_ch1d(const Band *h, const void *c, void *cnew, double alpha, int64_t M, cudaStream_t st)
{
    if (!(h->K == 2 && h->periodic)) return set_error(PB_EINVAL, "ch1d needs the cyclic penta handle");
    if (h->dtype == PB_F64)
        return fs_launch_t<double, 2, true, fs::MODE_CH1D, fs::LAY_INTER>(h, (double *)c, (double *)cnew, alpha, 1, 0, st, M, 0);
    return fs_launch_t<float, 2, true, fs::MODE_CH1D, fs::LAY_INTER>(h, (float *)c, (float *)cnew, alpha, 1, 0, st, M, 0);
}

}  // namespace pb

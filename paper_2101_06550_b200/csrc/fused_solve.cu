// fused_solve.cu — tables and host launcher of the fused streaming solve
// (fused_solve.cuh), both dtypes, penta (K = 2) and tri (K = 1).
#include <cudaTypedefs.h>
#include <string.h>

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

// L2 budget for the lag window of f between P1(g) and P2(g) (the L2 is 126 MB;
// the window, the x write-back in flight and the scratch records share it)
constexpr double FS_L2_BUDGET = 40.0 * 1048576.0;

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

template <typename T, int K, bool PER>
static int fs_launch_t(const Band *h, T *x, int64_t count, int64_t bstride, cudaStream_t st, int64_t Mo)
{
    using C = fs::Cfg<T>;
    auto kern = fs::fs_kernel<T, K, PER>;
    const size_t smem = sizeof(fs::Smem<T>) + 128;
    static std::once_flag attr_once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(attr_once, [&] {
        attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    if (attr_err != cudaSuccess) return set_error(PB_ECUDA, "fs_kernel smem attribute: %s", cudaGetErrorString(attr_err));

    const int64_t M = Mo > 0 ? Mo : h->batch, n = h->n;
    const int nq = h->fplan.nq;
    const int64_t Gb = (M + fs::TW - 1) / fs::TW, G = Gb * count;
    if (G > INT32_MAX / 2) return set_error(PB_EINVAL, "too many systems for one launch");
    const int64_t nsys = G * fs::TW;
    const int64_t items = 2 * G * nq, nclaims = (items + fs::NC - 1) / fs::NC;
    const size_t es = sizeof(T);
    // scratch: car [nq][nsys][4], spec [nsys][4], xl [nsys][2], cnt [G], flag [G], tick [4]
    const size_t off_spec = es * (size_t)nq * nsys * 4, off_xl = off_spec + es * nsys * 4;
    const size_t off_cnt = (off_xl + es * nsys * 2 + 255) / 256 * 256;
    const size_t off_flag = off_cnt + 4 * (size_t)G, off_tick = off_flag + 4 * (size_t)G;
    const size_t need = off_tick + 16;

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
            S.epoch = 0;
            memset(S.key, 0, sizeof(S.key));
        }
        char *base = (char *)S.buf;
        const bool relayout = S.nq != nq || S.nsys != nsys;   // counters live at shape-dependent offsets
        S.nq = nq;
        S.nsys = nsys;
        if (++S.epoch == 0 || S.epoch == 1 || relayout) {   // fresh, wrapped or re-laid-out: clear counters, flags, tickets
            S.epoch = 1;
            PB_CUDA_TRY(cudaMemsetAsync(base + off_cnt, 0, need - off_cnt, st));
        }
        A.car = (T *)base;
        A.spec = (T *)(base + off_spec);
        A.xl = (T *)(base + off_xl);
        A.cnt = (unsigned *)(base + off_cnt);
        A.flag = (unsigned *)(base + off_flag);
        A.tick = (unsigned *)(base + off_tick);
        A.epoch = S.epoch;

        // tensor map over x: dims (M, n, count), box (32 systems, 64 rows, 1);
        // OOB loads zero-fill (ragged M and n).  Contiguous batches of whole
        // chunks use one 2-D (M, n*count) view.  Cached per stream.
        const bool flat = count == 1 || (bstride == M * n && n % fs::Q == 0 && n * count < ((int64_t)1 << 31));
        const uint64_t key[6] = {(uint64_t)(uintptr_t)x, (uint64_t)M, (uint64_t)n, (uint64_t)count,
                                 (uint64_t)bstride, (uint64_t)sizeof(T)};
        if (memcmp(key, S.key, sizeof(key)) != 0) {
            auto enc = tensor_map_encoder();
            if (!enc) return set_error(PB_ECUDA, "cuTensorMapEncodeTiled unavailable");
            const auto dt = sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
            const int rank = flat ? 2 : 3;
            const int64_t bs = count > 1 ? bstride : M * n;
            cuuint64_t dims[3] = {(cuuint64_t)M, (cuuint64_t)(flat ? n * count : n), (cuuint64_t)(flat ? 1 : count)};
            cuuint64_t strides[2] = {(cuuint64_t)(M * sizeof(T)), (cuuint64_t)(bs * sizeof(T))};
            cuuint32_t box[3] = {(cuuint32_t)fs::TW, (cuuint32_t)fs::Q, 1};
            cuuint32_t estr[3] = {1, 1, 1};
            CUresult r = enc((CUtensorMap *)S.tmap, dt, rank, (void *)x, dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) return set_error(PB_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
            memcpy(S.key, key, sizeof(key));
        }
        A.flat = flat ? 1 : 0;
        CUtensorMap tmap;
        memcpy(&tmap, S.tmap, sizeof(tmap));

        A.rec = (const T *)h->fplan.rec;
        A.coef = (const T *)h->coef;
        A.ct = (const T *)h->fplan.ct;
        A.rsp = (const T *)h->fplan.rsp;
        A.scal = h->scal;
        A.x = x;
        A.bstride = count > 1 ? bstride : M * n;
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
        int64_t D = (int64_t)(FS_L2_BUDGET / gbytes);
        A.D = (int)(D < 1 ? 1 : (D > G ? G : D));
        A.qspec = PER ? (int)(h->srow[0] / fs::Q) : nq;
        const int grid = (int)std::min<int64_t>(sm_count(), nclaims);
        // launched (and the scratch's epoch bumped) under the lock: launches of one
        // stream keep their epoch order
        kern<<<grid, fs::NTHREADS, smem, st>>>(tmap, A);
        PB_LAUNCH_CHECK();
    }
    return PB_OK;
}

template <typename T>
static int fs_launch_dt(const Band *h, void *x, int64_t count, int64_t bstride, cudaStream_t st, int64_t M)
{
    T *X = (T *)x;
    if (h->K == 2)
        return h->periodic ? fs_launch_t<T, 2, true>(h, X, count, bstride, st, M)
                           : fs_launch_t<T, 2, false>(h, X, count, bstride, st, M);
    return h->periodic ? fs_launch_t<T, 1, true>(h, X, count, bstride, st, M)
                       : fs_launch_t<T, 1, false>(h, X, count, bstride, st, M);
}

int launch_fused(const Band *h, void *x, int64_t count, int64_t bstride, cudaStream_t st, int64_t M)
{
    return h->dtype == PB_F64 ? fs_launch_dt<double>(h, x, count, bstride, st, M)
                              : fs_launch_dt<float>(h, x, count, bstride, st, M);
}

}  // namespace pb

// twopass.cu — tables and host launchers of the two-pass streaming solve
// (twopass.cuh), both dtypes.
#include <cudaTypedefs.h>
#include <stdlib.h>

#include "band_tile.cuh"
#include "twopass.cuh"

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
__global__ void tp_tables_kernel(const double *coef, int K, int64_t n, int nq, int64_t s0, int64_t s1, int64_t s2,
                                 int64_t s3, T *rec, T *ct, T *rsp)
{
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    const int64_t srow[4] = {s0, s1, s2, s3};
    const int64_t r0 = (int64_t)q * tp::Q;
    const int kmax = (int)min((int64_t)tp::Q, n - r0);
    const double *cr = coef + r0 * COEF_STRIDE;
    auto F1 = [&](int i) { return cr[i * COEF_STRIDE + 1]; };
    auto F2 = [&](int i) { return K == 2 ? cr[i * COEF_STRIDE + 2] : 0.0; };
    auto B1 = [&](int i) { return cr[i * COEF_STRIDE + 4]; };
    auto B2 = [&](int i) { return K == 2 ? cr[i * COEF_STRIDE + 5] : 0.0; };
    double am1 = 0, am2 = 0, bm1 = 0, bm2 = 0;
    double al[tp::Q], be[tp::Q];
    for (int i = 0; i < kmax; ++i) {
        const double b1 = i >= 1 ? B1(i - 1) : 0.0, b2 = i >= 2 ? B2(i - 2) : 0.0;
        const double a = (i == 0 ? 1.0 : 0.0) - b1 * am1 - b2 * am2;
        const double b = (i == 1 ? 1.0 : 0.0) - b1 * bm1 - b2 * bm2;
        am2 = am1, am1 = a, bm2 = bm1, bm1 = b;
        al[i] = a, be[i] = b;
        T *o = rec + (r0 + i) * tp::REC;
        o[0] = (T)cr[i * COEF_STRIDE + 0];
        o[1] = (T)F1(i);
        o[2] = (T)F2(i);
        o[3] = (T)a;
        o[4] = (T)b;
        o[5] = T(0);
    }
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

int twopass_build_tables(Band *h, cudaStream_t st)
{
    const size_t es = dtype_size(h->dtype);
    const int64_t nq = (h->n + tp::Q - 1) / tp::Q;
    h->tplan.ok = 0;
    if (nq > 65535 || !tensor_map_encoder()) return PB_OK;
    PB_CUDA_TRY(cudaMalloc(&h->tplan.rec, es * tp::REC * nq * tp::Q));
    PB_CUDA_TRY(cudaMalloc(&h->tplan.ct, es * 12 * nq));
    PB_CUDA_TRY(cudaMalloc(&h->tplan.rsp, es * 8));
    PB_CUDA_TRY(cudaMemsetAsync(h->tplan.rsp, 0, es * 8, st));
    const unsigned g = (unsigned)((nq + 63) / 64);
    if (h->dtype == PB_F64)
        tp_tables_kernel<double><<<g, 64, 0, st>>>(h->coefD, h->K, h->n, (int)nq, h->srow[0], h->srow[1], h->srow[2],
                                                   h->srow[3], (double *)h->tplan.rec, (double *)h->tplan.ct,
                                                   (double *)h->tplan.rsp);
    else
        tp_tables_kernel<float><<<g, 64, 0, st>>>(h->coefD, h->K, h->n, (int)nq, h->srow[0], h->srow[1], h->srow[2],
                                                  h->srow[3], (float *)h->tplan.rec, (float *)h->tplan.ct,
                                                  (float *)h->tplan.rsp);
    PB_LAUNCH_CHECK();
    h->tplan.nq = (int)nq;
    h->tplan.ok = 1;
    return PB_OK;
}

// systems per slab: pass 2 re-reads the slab's RHS, which pass 1 left in L2
// when the slab fits (PB_TP_SLAB_MB MB; default 0 = one slab: the per-slab
// scan has too little parallelism below ~4 K systems, measured slower)
static int64_t tp_slab_systems(int64_t M, int64_t n, int64_t count, size_t es)
{
    const char *e = getenv("PB_TP_SLAB_MB");
    const double mb = e ? atof(e) : 0.0;
    if (mb <= 0) return M;
    int64_t ms = (int64_t)(mb * 1048576.0 / ((double)n * (double)es * (double)count));
    ms = ms / 128 * 128;
    if (ms < 128) ms = 128;
    return ms >= M ? M : ms;
}

// launch with programmatic stream serialization (see pdl_wait in twopass.cuh)
template <typename Kern, typename... Args>
static cudaError_t launch_pdl(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <typename T, int K, bool PER, bool P2>
static int tp_pass_prep(size_t *smem)
{
    auto kern = tp::tp_pass_kernel<T, K, PER, P2>;
    *smem = sizeof(tp::PassSmem<T, P2>) + 128;
    PB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*smem));
    return PB_OK;
}

template <typename T, int K, bool PER>
static int launch_tp_t(const Band *h, T *x, int64_t count, int64_t bstride, cudaStream_t st, int64_t Mo = 0)
{
    const int64_t M = Mo > 0 ? Mo : h->batch, n = h->n;
    const int nq = h->tplan.nq;
    const int64_t ms = tp_slab_systems(M, n, count, sizeof(T));
    const int64_t msp = (ms + tp::TW - 1) / tp::TW * tp::TW;
    size_t sm1, sm2;
    int rc = tp_pass_prep<T, K, PER, false>(&sm1);
    if (!rc) rc = tp_pass_prep<T, K, PER, true>(&sm2);
    if (rc) return rc;
    int dev = 0, nsm = 0;
    PB_CUDA_TRY(cudaGetDevice(&dev));
    PB_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));

    // tensor map: dims (M, n, count), box (32 systems, 64 rows, 1); OOB loads
    // zero-fill, OOB stores are clipped (ragged M and n)
    // tensor maps over x: dims (M, n, count).  Loads: box (32 systems, 64 rows);
    // stores: box (128 bytes of systems, 64 rows).  OOB loads zero-fill, OOB
    // stores are clipped (ragged M and n)
    CUtensorMap tmap, smap, cmap1, cmap2;
    bool flat = false, cmaps_ok = false;
    {
        // coefficient rows as 2-D tensors: pass 1 rec (REC per row), pass 2 coef (COEF_STRIDE per row)
        auto enc = tensor_map_encoder();
        if (!enc) return set_error(PB_ECUDA, "cuTensorMapEncodeTiled unavailable");
        const auto dt = sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
        const int64_t rrows = (int64_t)nq * tp::Q;
        cuuint64_t d1[2] = {(cuuint64_t)tp::REC, (cuuint64_t)rrows}, s1[1] = {(cuuint64_t)(tp::REC * sizeof(T))};
        cuuint32_t b1[2] = {(cuuint32_t)tp::REC, (cuuint32_t)tp::Q}, e1[2] = {1, 1};
        CUresult r = enc(&cmap1, dt, 2, (void *)h->tplan.rec, d1, s1, b1, e1, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        cuuint64_t d2[2] = {(cuuint64_t)COEF_STRIDE, (cuuint64_t)h->rows_alloc},
                   s2[1] = {(cuuint64_t)(COEF_STRIDE * sizeof(T))};
        cuuint32_t b2[2] = {(cuuint32_t)COEF_STRIDE, (cuuint32_t)tp::Q};
        if (r == CUDA_SUCCESS)
            r = enc(&cmap2, dt, 2, (void *)h->coef, d2, s2, b2, e1, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        cmaps_ok = r == CUDA_SUCCESS;   // (fp32 rec rows are 24 B: not a legal TMA row; bulk copies then)
    }
    {
        const int64_t bs = count > 1 ? bstride : M * n;
        // contiguous batches whose systems are whole chunks: one 2-D (M, n*count) view
        // (3-D maps with count > 1 faulted intermittently under sustained
        // back-to-back solves, tools/iso_stress.sh)
        flat = count > 1 && bs == M * n && n % tp::Q == 0 && n * count < (int64_t)1 << 31;
        const int rank = flat ? 2 : 3;
        cuuint64_t dims[3] = {(cuuint64_t)M, (cuuint64_t)(flat ? n * count : n), (cuuint64_t)(flat ? 1 : count)};
        cuuint64_t strides[2] = {(cuuint64_t)(M * sizeof(T)), (cuuint64_t)(bs * sizeof(T))};
        cuuint32_t box[3] = {(cuuint32_t)tp::TW, (cuuint32_t)tp::Q, 1};
        cuuint32_t sbox[3] = {(cuuint32_t)(128 / sizeof(T)), (cuuint32_t)tp::Q, 1};
        cuuint32_t es[3] = {1, 1, 1};
        auto enc = tensor_map_encoder();
        if (!enc) return set_error(PB_ECUDA, "cuTensorMapEncodeTiled unavailable");
        const auto dt = sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
        CUresult r = enc(&tmap, dt, rank, (void *)x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r == CUDA_SUCCESS)
            r = enc(&smap, dt, rank, (void *)x, dims, strides, sbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return set_error(PB_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    }
    tp::Args<T> A;
    A.rec = (const T *)h->tplan.rec;
    A.coef = (const T *)h->coef;
    A.ct = (const T *)h->tplan.ct;
    A.rsp = (const T *)h->tplan.rsp;
    A.scal = h->scal;
    A.n = n;
    A.M = M;
    for (int j = 0; j < 4; ++j) A.srow[j] = h->srow[j];
    A.nq = nq;
    A.count = (int)count;
    A.qspec = PER ? (int)(h->srow[0] / tp::Q) : nq;
    A.msp = msp;
    A.keep = ms < M;   // slabbed: the slab is sized to stay in L2 until pass 2
    A.flat = flat ? 1 : 0;
    const char *p2g_env = getenv("PB_TP_P2G");   // 0 bulk, 2 tensor; unset = auto


    // per-handle scratch for one slab (reused by the slabs in stream order);
    // a solve on another stream first waits for the previous solve's event
    const size_t nsys = (size_t)msp * count;
    const size_t need = sizeof(T) * nsys * ((size_t)nq * 4 + 6) + 256;
    const TwoPassPlan &P = h->tplan;
    if (!P.done) PB_CUDA_TRY(cudaEventCreateWithFlags(&P.done, cudaEventDisableTiming));
    else PB_CUDA_TRY(cudaStreamWaitEvent(st, P.done, 0));
    if (need > P.scratch_bytes) {
        PB_CUDA_TRY(cudaEventSynchronize(P.done));
        PB_CUDA_TRY(cudaStreamSynchronize(st));
        cudaFree(P.scratch);
        P.scratch = nullptr;
        P.scratch_bytes = 0;
        PB_CUDA_TRY(cudaMalloc(&P.scratch, need));
        P.scratch_bytes = need;
    }
    void *scratch = P.scratch;
    A.car = (T *)scratch;
    A.spec = A.car + nsys * nq * 4;
    A.xl = A.spec + nsys * 4;
    for (int64_t s0 = 0; s0 < M; s0 += ms) {
        A.s0 = s0;
        A.ms = (M - s0) < ms ? (M - s0) : ms;
        A.G = (int)((A.ms + tp::TW - 1) / tp::TW);
        const int64_t ntile = (int64_t)nq * A.G * count;
        // coefficient rows per stage: 1-D bulk copy (fastest) unless more than 1024 tile
        // groups share a chunk -- then every in-flight stage copies the same rows, the
        // regime in which the bulk copies faulted -- where a 2-D tensor
        // load of the rows is used instead (measured fault-free there)
        A.p2g = p2g_env ? atoi(p2g_env) : (cmaps_ok && (int64_t)A.G * count > 1024 ? 2 : 0);
        if (A.p2g == 2 && !cmaps_ok) A.p2g = 0;
        const unsigned grid = (unsigned)(ntile < nsm ? ntile : nsm);
        PB_CUDA_TRY(launch_pdl(tp::tp_pass_kernel<T, K, PER, false>, dim3(grid), dim3(32 * (tp::NWC1 + 1)), sm1, st, tmap,
                               smap, cmap1, A));
        PB_LAUNCH_CHECK();
            if (nq <= tp::SEQ_MAX)
            PB_CUDA_TRY(launch_pdl(tp::tp_scan_seq_kernel<T, K, PER>, dim3((unsigned)((nsys + 255) / 256)), dim3(256), 0,
                                   st, A));
        else if (nq <= tp::NSEG_R * tp::CPS_R)
            PB_CUDA_TRY(launch_pdl(tp::tp_scan_reg_kernel<T, K, PER>, dim3((unsigned)(nsys / tp::TW)),
                                   dim3(32 * tp::NSEG_R), 0, st, A));
        else
            PB_CUDA_TRY(launch_pdl(tp::tp_scan_kernel<T, K, PER>, dim3((unsigned)(nsys / tp::TW)), dim3(32 * tp::NSEG),
                                   0, st, A));
        PB_LAUNCH_CHECK();
        PB_CUDA_TRY(launch_pdl(tp::tp_pass_kernel<T, K, PER, true>, dim3(grid), dim3(32 * (tp::NWC + 1)), sm2, st, tmap,
                               smap, cmap2, A));
        PB_LAUNCH_CHECK();
    }
    PB_CUDA_TRY(cudaEventRecord(P.done, st));
    return PB_OK;
}

template <typename T>
static int launch_tp_dt(const Band *h, void *x, int64_t count, int64_t bstride, cudaStream_t st, int64_t Mo = 0)
{
    T *X = (T *)x;
    if (h->K == 2)
        return h->periodic ? launch_tp_t<T, 2, true>(h, X, count, bstride, st, Mo)
                           : launch_tp_t<T, 2, false>(h, X, count, bstride, st, Mo);
    return h->periodic ? launch_tp_t<T, 1, true>(h, X, count, bstride, st, Mo)
                       : launch_tp_t<T, 1, false>(h, X, count, bstride, st, Mo);
}

// one batch of M systems sharing the handle's LHS (M need not equal h->batch)
int launch_tp_m(const Band *h, void *x, int64_t M, cudaStream_t st)
{
    return h->dtype == PB_F64 ? launch_tp_dt<double>(h, x, 1, M * h->n, st, M)
                              : launch_tp_dt<float>(h, x, 1, M * h->n, st, M);
}

int launch_tp_f64(const Band *h, void *x, int64_t count, int64_t bstride, cudaStream_t st)
{
    return launch_tp_dt<double>(h, x, count, bstride, st);
}
int launch_tp_f32(const Band *h, void *x, int64_t count, int64_t bstride, cudaStream_t st)
{
    return launch_tp_dt<float>(h, x, count, bstride, st);
}

}  // namespace pb

// stream_launch.cuh — host launcher of the streaming solve (stream_solve.cuh):
// tensor map, per-call scratch, grid sizing.  Included by
// stream_solve_f64.cu / stream_solve_f32.cu (one dtype each, parallel builds).
#pragma once
#include <cudaTypedefs.h>
#include <stdlib.h>

#include "band_tile.cuh"
#include "stream_solve.cuh"

namespace pb {

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();
static_assert(MAX_NRB == STREAM_MAX_NRB, "group-scan capacity mismatch");


template <typename T, int K, bool PER>
static int stream_prep(size_t *smem_out, int *blocks_per_sm)
{
    auto kern = stream_solve_kernel<T, K, PER>;
    const size_t smem = sizeof(StreamSmem<T>) + 128;   // + alignment
    PB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    PB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, STREAM_THREADS, smem));
    *smem_out = smem;
    *blocks_per_sm = occ;
    return PB_OK;
}

// co-resident CTAs of the persistent grid (0 if the kernel cannot run)
template <typename T>
static int stream_max_ctas_t(int K, int periodic)
{
    size_t smem;
    int occ = 0, dev = 0, nsm = 0;
    int rc = K == 2 ? (periodic ? stream_prep<T, 2, true>(&smem, &occ) : stream_prep<T, 2, false>(&smem, &occ))
                    : (periodic ? stream_prep<T, 1, true>(&smem, &occ) : stream_prep<T, 1, false>(&smem, &occ));
    if (rc) return 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return occ * nsm;
}

template <typename T, int K, bool PER>
static int launch_stream_t(const Band *h, T *x, int64_t count, int64_t bstride, cudaStream_t st)
{
    constexpr int W = StreamGeom<T>::W;
    auto kern = stream_solve_kernel<T, K, PER>;
    size_t smem;
    int occ;
    int rc = stream_prep<T, K, PER>(&smem, &occ);
    if (rc) return rc;
    int dev = 0, nsm = 0;
    PB_CUDA_TRY(cudaGetDevice(&dev));
    PB_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const int nrb = h->splan.nrb;
    const int64_t M = h->batch, n = h->n;
    const int64_t groups = (M + W - 1) / W, gt = groups * count;
    int K_ = (occ * nsm) / nrb;
    if (K_ < 1) return set_error(PB_EUNSUPPORTED, "stream solve: %d tiles per system exceed the resident grid", nrb);
    if (K_ > gt) K_ = (int)gt;

    // tensor map: dims (M, n, count), box (W, R, 1); strides must be 16 B multiples
    CUtensorMap tmap;
    {
        const int64_t bs = count > 1 ? bstride : M * n;
        cuuint64_t dims[3] = {(cuuint64_t)M, (cuuint64_t)n, (cuuint64_t)count};
        cuuint64_t strides[2] = {(cuuint64_t)(M * sizeof(T)), (cuuint64_t)(bs * sizeof(T))};
        cuuint32_t box[3] = {(cuuint32_t)W, (cuuint32_t)StreamGeom<T>::R, 1};
        cuuint32_t es[3] = {1, 1, 1};
        auto enc = tensor_map_encoder();
        if (!enc) return set_error(PB_ECUDA, "cuTensorMapEncodeTiled unavailable");
        CUresult r = enc(&tmap, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                         (void *)x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return set_error(PB_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    }

    StreamArgs<T> A;
    A.tb.coef = (const T *)h->coef;
    A.tb.tab = (const T *)h->splan.tab;
    A.tb.mft = (const T *)h->splan.mft;
    A.tb.mbt = (const T *)h->splan.mbt;
    A.tb.hft = (const T *)h->splan.hft;
    A.tb.gsp = (const T *)h->splan.gsp;
    A.tb.rsp = (const T *)h->splan.rsp;
    A.tb.scal = h->scal;
    for (int j = 0; j < 4; ++j) {
        A.tb.srb[j] = h->splan.srb[j];
        A.tb.srow[j] = h->srow[j];
    }
    A.x = x;
    A.n = n;
    A.M = M;
    A.bstride = bstride;
    A.count = (int)count;
    A.nrb = nrb;
    A.K = K_;
    A.groups = groups;
    {
        static const int lead = [] {
            const char *e = getenv("PB_STREAM_LEAD");
            return e ? atoi(e) : 6;
        }();
        A.lead = lead > 0 ? lead : 1;
    }
    {
        // dev timeline: PB_STREAM_TRACE=<device pointer> ([cta][team][256][8] u64)
        const char *e = getenv("PB_STREAM_TRACE");
        A.trace = e ? (unsigned long long *)strtoull(e, nullptr, 0) : nullptr;
    }
    A.sc = StreamScratch<T>{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    void *scratch = nullptr;
    if (nrb > 1) {
        // per-call scratch, stream ordered (concurrent solves with one handle stay independent)
        const size_t n_agg = (size_t)gt * nrb * W * 4, n_spec = (size_t)gt * W * 4, n_xl = (size_t)gt * W * 2;
        const size_t n_flag = (size_t)gt;
        const size_t bytes = sizeof(T) * (2 * n_agg + n_spec + n_xl) + sizeof(int) * 2 * n_flag + 256;
        PB_CUDA_TRY(cudaMallocAsync(&scratch, bytes, st));
        char *c = (char *)scratch;
        A.sc.cnt = (int *)c;
        A.sc.flag = A.sc.cnt + n_flag;
        c += ((sizeof(int) * 2 * n_flag + 255) / 256) * 256;
        A.sc.agg = (T *)c;
        A.sc.inf = A.sc.agg + n_agg;
        A.sc.spec = A.sc.inf + n_agg;
        A.sc.xl = A.sc.spec + n_spec;
        PB_CUDA_TRY(cudaMemsetAsync(scratch, 0, sizeof(int) * 2 * n_flag, st));
    }
    kern<<<(unsigned)(nrb * K_), STREAM_THREADS, smem, st>>>(tmap, A);
    PB_LAUNCH_CHECK();
    if (scratch) PB_CUDA_TRY(cudaFreeAsync(scratch, st));
    return PB_OK;
}

template <typename T>
static int launch_stream_dt(const Band *h, void *x, int64_t count, int64_t bstride, cudaStream_t st)
{
    T *X = (T *)x;
    if (h->K == 2)
        return h->periodic ? launch_stream_t<T, 2, true>(h, X, count, bstride, st)
                           : launch_stream_t<T, 2, false>(h, X, count, bstride, st);
    return h->periodic ? launch_stream_t<T, 1, true>(h, X, count, bstride, st)
                       : launch_stream_t<T, 1, false>(h, X, count, bstride, st);
}

}  // namespace pb

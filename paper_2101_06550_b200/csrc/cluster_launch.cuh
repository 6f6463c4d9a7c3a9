// cluster_launch.cuh — host side of the cluster solve (cluster_solve.cuh):
// plan tables, tensor map, persistent cluster grid.  Included by
// stream_solve_f64.cu / stream_solve_f32.cu.
#pragma once
#include <cudaTypedefs.h>
#include <stdlib.h>

#include "band_tile.cuh"
#include "cluster_solve.cuh"

namespace pb {

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();

template <typename T, int K, bool PER>
static int clu_prep(int C, size_t *smem_out, int *ncl_out)
{
    auto kern = clu::cluster_solve_kernel<T, K, PER>;
    const size_t smem = sizeof(clu::Smem<T>);
    PB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (C > 8) PB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(clu::Geom<T>::NT + 32);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    PB_CUDA_TRY(cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg));
    *smem_out = smem;
    *ncl_out = ncl;
    return PB_OK;
}

template <typename T>
int clu_max_clusters(int C, int K, int periodic)
{
    size_t smem;
    int ncl = 0;
    int rc = K == 2 ? (periodic ? clu_prep<T, 2, true>(C, &smem, &ncl) : clu_prep<T, 2, false>(C, &smem, &ncl))
                    : (periodic ? clu_prep<T, 1, true>(C, &smem, &ncl) : clu_prep<T, 1, false>(C, &smem, &ncl));
    return rc ? 0 : ncl;
}

template <typename T, int K, bool PER>
static int launch_clu_t(const Band *h, T *x, int64_t count, int64_t bstride, cudaStream_t st)
{
    constexpr int W = clu::Geom<T>::W;
    const int C = h->cplan.C;
    size_t smem;
    int ncl;
    int rc = clu_prep<T, K, PER>(C, &smem, &ncl);
    if (rc) return rc;
    if (ncl < 1) return set_error(PB_EUNSUPPORTED, "cluster solve: no resident %d-CTA cluster", C);
    const int64_t M = h->batch, n = h->n;
    const int64_t groups = (M + W - 1) / W, gt = groups * count;
    if (ncl > gt) ncl = (int)gt;
    CUtensorMap tmap;
    {
        const int64_t bs = count > 1 ? bstride : M * n;
        cuuint64_t dims[3] = {(cuuint64_t)M, (cuuint64_t)n, (cuuint64_t)count};
        cuuint64_t strides[2] = {(cuuint64_t)(M * sizeof(T)), (cuuint64_t)(bs * sizeof(T))};
        cuuint32_t box[3] = {(cuuint32_t)W, 256, 1};
        cuuint32_t es[3] = {1, 1, 1};
        auto enc = tensor_map_encoder();
        if (!enc) return set_error(PB_ECUDA, "cuTensorMapEncodeTiled unavailable");
        CUresult r = enc(&tmap, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                         (void *)x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return set_error(PB_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    }
    clu::Args<T> A;
    A.coef = (const T *)h->coef;
    A.cc = (const T *)h->cplan.cc;
    A.mf = (const T *)h->cplan.mf;
    A.mb = (const T *)h->cplan.mb;
    A.mfc = (const T *)h->cplan.mfc;
    A.mbc = (const T *)h->cplan.mbc;
    A.scal = h->scal;
    for (int j = 0; j < 4; ++j) A.srow[j] = h->srow[j];
    A.n = n;
    A.M = M;
    A.bstride = bstride;
    A.groups = groups;
    A.count = (int)count;
    A.C = C;
    A.ncl = ncl;
    A.x = x;
    {
        const char *e = getenv("PB_CLU_TRACE");   // dev timeline (device pointer)
        A.trace = e ? (unsigned long long *)strtoull(e, nullptr, 0) : nullptr;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(ncl * C));
    cfg.blockDim = dim3(clu::Geom<T>::NT + 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    PB_CUDA_TRY(cudaLaunchKernelEx(&cfg, clu::cluster_solve_kernel<T, K, PER>, tmap, A));
    PB_LAUNCH_CHECK();
    return PB_OK;
}

template <typename T>
static int launch_clu_dt(const Band *h, void *x, int64_t count, int64_t bstride, cudaStream_t st)
{
    T *X = (T *)x;
    if (h->K == 2)
        return h->periodic ? launch_clu_t<T, 2, true>(h, X, count, bstride, st)
                           : launch_clu_t<T, 2, false>(h, X, count, bstride, st);
    return h->periodic ? launch_clu_t<T, 1, true>(h, X, count, bstride, st)
                       : launch_clu_t<T, 1, false>(h, X, count, bstride, st);
}

}  // namespace pb

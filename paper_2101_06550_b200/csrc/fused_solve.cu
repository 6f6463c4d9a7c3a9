// fused_solve.cu — tables and host launcher of the fused streaming solve
// (fused_solve.cuh), both dtypes, penta (K = 2) and tri (K = 1).
#include <cudaTypedefs.h>
#include <math.h>
#include <string.h>


#include "band_tile.cuh"
#include "fused_cluster.cuh"

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

int fs_sm_count()
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

// per-(dtype, layout) translation units (fused_part.cuh): the instantiations
// are split so nvcc compiles them in parallel
int launch_fused_f64_inter(const Band *, void *, int64_t, int64_t, cudaStream_t, int64_t, int64_t);
int launch_fused_f64_contig(const Band *, void *, int64_t, int64_t, cudaStream_t, int64_t, int64_t);
int launch_fused_f32_inter(const Band *, void *, int64_t, int64_t, cudaStream_t, int64_t, int64_t);
int launch_fused_f32_contig(const Band *, void *, int64_t, int64_t, cudaStream_t, int64_t, int64_t);
int launch_ch1d_f64(const Band *, const void *, void *, double, int64_t, cudaStream_t);
int fused_info_f64_inter(const Band *, int64_t, int64_t, int *);
int fused_info_f64_contig(const Band *, int64_t, int64_t, int *);
int fused_info_f32_inter(const Band *, int64_t, int64_t, int *);
int fused_info_f32_contig(const Band *, int64_t, int64_t, int *);

int fused_info(const Band *h, int layout, int64_t M, int64_t count, int *info)
{
    if (layout == PB_CONTIGUOUS)
        return h->dtype == PB_F64 ? fused_info_f64_contig(h, M, count, info) : fused_info_f32_contig(h, M, count, info);
    return h->dtype == PB_F64 ? fused_info_f64_inter(h, M, count, info) : fused_info_f32_inter(h, M, count, info);
}
int launch_ch1d_f32(const Band *, const void *, void *, double, int64_t, cudaStream_t);

int launch_fused(const Band *h, void *x, int layout, int64_t count, int64_t bstride, cudaStream_t st, int64_t M,
                 int64_t pitch)
{
    if (layout == PB_CONTIGUOUS)
        return h->dtype == PB_F64 ? launch_fused_f64_contig(h, x, count, bstride, st, M, pitch)
                                  : launch_fused_f32_contig(h, x, count, bstride, st, M, pitch);
    return h->dtype == PB_F64 ? launch_fused_f64_inter(h, x, count, bstride, st, M, pitch)
                              : launch_fused_f32_inter(h, x, count, bstride, st, M, pitch);
}

int launch_fused_ch1d(const Band *h, const void *c, void *cnew, double alpha, int64_t M, cudaStream_t st)
{
    if (!(h->K == 2 && h->periodic)) return set_error(PB_EINVAL, "ch1d needs the cyclic penta handle");
    return h->dtype == PB_F64 ? launch_ch1d_f64(h, c, cnew, alpha, M, st) : launch_ch1d_f32(h, c, cnew, alpha, M, st);
}

}  // namespace pb

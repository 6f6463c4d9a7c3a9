// coarsen.cu — on-device coarsening statistics: the free
// energy F of every simulation of a batch (reading r24) and the
// growth rate beta = -(t/F) dF/dt of sampled F (reading r27).  The
// Cahn–Hilliard–Cook noise itself lives in the ADI RHS kernel (ch_adi.cu).
#include <algorithm>

#include "common.cuh"

namespace pb {

constexpr int FE_ROWS = 16;    // grid rows per CTA
constexpr int FE_THREADS = 256;

// partial[sim][blk] = sum over rows [blk*FE_ROWS, ...) of
//   1/4 (C^2 - 1)^2 + 1/2 gamma ((C_{i+1,j} - C_ij)^2 + (C_{i,j+1} - C_ij)^2) / dx^2
// (periodic forward differences), fp64, fixed reduction order.
template <typename TS>
__global__ void __launch_bounds__(FE_THREADS) free_energy_kernel(const TS *__restrict__ c, int64_t n, double half_g_idx2,
                                                                  double *__restrict__ partial)
{
    const int64_t sim = blockIdx.y, j0 = (int64_t)blockIdx.x * FE_ROWS;
    const TS *C = c + sim * n * n;
    double acc = 0.0;
    const int64_t jmax = min((int64_t)FE_ROWS, n - j0);
    for (int64_t jj = 0; jj < jmax; ++jj) {
        const int64_t j = j0 + jj, jp = j + 1 == n ? 0 : j + 1;
        for (int64_t i = threadIdx.x; i < n; i += FE_THREADS) {
            const int64_t ip = i + 1 == n ? 0 : i + 1;
            const double v = (double)C[j * n + i];
            const double gx = (double)C[j * n + ip] - v, gy = (double)C[jp * n + i] - v;
            const double b = v * v - 1.0;
            acc += 0.25 * b * b + half_g_idx2 * (gx * gx + gy * gy);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    __shared__ double ws[FE_THREADS / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < FE_THREADS / 32; ++w) s += ws[w];
        partial[sim * gridDim.x + blockIdx.x] = s;
    }
}

__global__ void free_energy_final_kernel(const double *__restrict__ partial, int64_t sims, int nblk, double dx2,
                                         double *__restrict__ F)
{
    const int64_t sim = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (sim >= sims) return;
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += partial[sim * nblk + b];
    F[sim] = s * dx2;
}

// beta[k][sim] = -(t_k / F_k) (F_b - F_a) / (t_b - t_a), (a, b) = (k-1, k+1)
// inside, one-sided at the ends
__global__ void beta_kernel(int64_t nt, int64_t sims, const double *__restrict__ t, const double *__restrict__ F,
                            double *__restrict__ beta)
{
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= nt * sims) return;
    const int64_t k = e / sims, s = e - k * sims;
    const int64_t a = k > 0 ? k - 1 : 0, b = k < nt - 1 ? k + 1 : nt - 1;
    const double dFdt = (F[b * sims + s] - F[a * sims + s]) / (t[b] - t[a]);
    beta[e] = -(t[k] / F[e]) * dFdt;
}

}  // namespace pb

extern "C" int ch_free_energy(const pb_ch_state *s, const pb_ch_params *p, double *F, void *stream)
{
    using namespace pb;
    if (!s || !p || !F) return set_error(PB_EINVAL, "null state/params/F");
    if (s->n < 2 || s->sims < 0 || (s->dtype != PB_F64 && s->dtype != PB_F32) || !(p->L > 0))
        return set_error(PB_EINVAL, "bad state or params");
    if (pb_device_ok() != PB_OK) return PB_ECUDA;
    if (s->sims == 0) return PB_OK;
    if (!is_device_ptr(s->c_cur) || !is_device_ptr(F)) return set_error(PB_EINVAL, "c_cur and F must be device memory");
    if (s->sims > 65535) return set_error(PB_EINVAL, "sims > 65535 per call");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = s->n;
    const double dx = p->L / (double)n;
    const int nblk = (int)((n + FE_ROWS - 1) / FE_ROWS);
    double *partial = nullptr;
    PB_CUDA_TRY(cudaMallocAsync(&partial, sizeof(double) * (size_t)nblk * s->sims, st));
    dim3 grid((unsigned)nblk, (unsigned)s->sims);
    const double hg = 0.5 * p->gamma / (dx * dx);
    if (s->dtype == PB_F64)
        free_energy_kernel<double><<<grid, FE_THREADS, 0, st>>>((const double *)s->c_cur, n, hg, partial);
    else
        free_energy_kernel<float><<<grid, FE_THREADS, 0, st>>>((const float *)s->c_cur, n, hg, partial);
    PB_LAUNCH_CHECK();
    free_energy_final_kernel<<<(unsigned)((s->sims + 127) / 128), 128, 0, st>>>(partial, s->sims, nblk, dx * dx, F);
    PB_LAUNCH_CHECK();
    PB_CUDA_TRY(cudaFreeAsync(partial, st));
    return PB_OK;
}

extern "C" int ch_coarsening_beta(int64_t nt, int64_t sims, const double *t, const double *F, double *beta,
                                  void *stream)
{
    using namespace pb;
    if (nt < 2 || sims < 0 || !t || !F || !beta) return set_error(PB_EINVAL, "need nt >= 2 and buffers");
    if (pb_device_ok() != PB_OK) return PB_ECUDA;
    if (sims == 0) return PB_OK;
    if (!is_device_ptr(t) || !is_device_ptr(F) || !is_device_ptr(beta))
        return set_error(PB_EINVAL, "t, F, beta must be device memory");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t tot = nt * sims;
    beta_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(nt, sims, t, F, beta);
    PB_LAUNCH_CHECK();
    return PB_OK;
}

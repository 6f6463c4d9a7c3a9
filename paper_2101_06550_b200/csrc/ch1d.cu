// ch1d.cu — batched 1D Cahn–Hilliard (thesis §6.2, eq6:1Dnumerical,
// P:2668-2731): per step and system,
//   (I + dt gamma d_xxxx) C^{n+1} = C^n + dt d_xx (C^3 - C)^n
// i.e. the cyclic pentadiagonal (s, -4s, 1+6s, -4s, s), s = gamma dt / dx^4,
// with f_i = C_i + alpha (N_{i-1} - 2 N_i + N_{i+1}), alpha = dt / dx^2,
// N = C^3 - C (the +C_i^n term is reading r12).  One launch per step: the
// fused streaming solve forms f on chip from the C^n tile (MODE_CH1D), so a
// step moves read C^n + write C^{n+1} through HBM (16 B per point fp64).
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>

#include "band_tile.cuh"

namespace pb {

static std::mutex g_ch1d_mu;
static std::map<std::tuple<int, int64_t, int, uint64_t>, Band *> g_ch1d_cache;

static int ch1d_band(int64_t n, double sigma, int dtype, cudaStream_t st, Band **out)
{
    int dev = 0;
    PB_CUDA_TRY(cudaGetDevice(&dev));
    uint64_t bits;
    memcpy(&bits, &sigma, sizeof(bits));
    auto key = std::make_tuple(dev, n, dtype, bits);
    std::lock_guard<std::mutex> lk(g_ch1d_mu);
    auto it = g_ch1d_cache.find(key);
    if (it != g_ch1d_cache.end()) {
        *out = it->second;
        return PB_OK;
    }
    Band *h = nullptr;
    int rc = const_penta_band(n, sigma, dtype, -1, 0, st, &h);
    if (rc) return rc;
    g_ch1d_cache[key] = h;
    *out = h;
    return PB_OK;
}

// f_i = C_i + alpha (N_{i-1} - 2 N_i + N_{i+1}), N = C^3 - C, periodic in i
// (interleaved [i][s]); used when the handle is solved sequentially (seq_only)
template <typename T>
__global__ void ch1d_rhs_kernel(const T *__restrict__ c, T *__restrict__ f, int64_t n, int64_t M, T alpha)
{
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * M; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / M, s = e - i * M;
        const T um = c[(i == 0 ? n - 1 : i - 1) * M + s], u = c[e], up = c[(i == n - 1 ? 0 : i + 1) * M + s];
        const T nm = um * um * um - um, n0 = u * u * u - u, np = up * up * up - up;
        f[e] = u + alpha * (nm - T(2) * n0 + np);
    }
}

}  // namespace pb

extern "C" int ch1d_step(pb_ch1d_state *s, double dt, const pb_ch1d_params *p, int64_t nsteps, void *stream)
{
    using namespace pb;
    if (!s || !p) return set_error(PB_EINVAL, "null state/params");
    if (s->n < 7 || s->batch < 0 || nsteps < 0) return set_error(PB_EINVAL, "need n >= 7, batch >= 0, nsteps >= 0");
    if (s->batch % 32) return set_error(PB_EINVAL, "batch must be a multiple of 32 (whole 32-system tiles)");
    if (s->dtype != PB_F64 && s->dtype != PB_F32) return set_error(PB_EINVAL, "bad dtype");
    if (!(dt > 0) || !(p->L > 0) || !(p->gamma >= 0)) return set_error(PB_EINVAL, "dt, L must be positive, gamma >= 0");
    if (pb_device_ok() != PB_OK) return PB_ECUDA;
    if (s->batch == 0 || nsteps == 0) return PB_OK;
    if (!s->c || !s->work || s->c == s->work) return set_error(PB_EINVAL, "c and work must be distinct device buffers");
    if ((uintptr_t)s->c % 16 || (uintptr_t)s->work % 16) return set_error(PB_EINVAL, "c and work must be 16-byte aligned");
    if (!is_device_ptr(s->c) || !is_device_ptr(s->work)) return set_error(PB_EINVAL, "ch1d buffers must be device memory");
    cudaStream_t st = (cudaStream_t)stream;
    const double dx = p->L / (double)s->n;   // r1
    const double sigma = p->gamma * dt / (dx * dx * dx * dx), alpha = dt / (dx * dx);
    Band *h = nullptr;
    int rc = ch1d_band(s->n, sigma, s->dtype, st, &h);
    if (rc) return rc;
    const bool fused = h->fplan.ok && !h->seq_only;
    for (int64_t k = 0; k < nsteps; ++k) {
        if (fused) {
            if ((rc = launch_fused_ch1d(h, s->c, s->work, alpha, s->batch, st))) return rc;
        } else {
            // growing chunk maps (kappa ~ 1e6+, e.g. Table 6.1's N = 4096): RHS kernel +
            // the sequential thread-per-system solve
            const unsigned g = (unsigned)std::min<int64_t>((s->n * s->batch + 255) / 256, 148 * 16);
            if (s->dtype == PB_F64)
                ch1d_rhs_kernel<double><<<g, 256, 0, st>>>((const double *)s->c, (double *)s->work, s->n, s->batch,
                                                           alpha);
            else
                ch1d_rhs_kernel<float><<<g, 256, 0, st>>>((const float *)s->c, (float *)s->work, s->n, s->batch,
                                                          (float)alpha);
            PB_LAUNCH_CHECK();
            pb_layout L;
            L.n_inner = s->batch;
            L.inner_stride = 1;
            L.n_outer = 1;
            L.outer_stride = 0;
            L.row_stride = s->batch;
            if ((rc = band_solve_layout(h, s->work, L, st))) return rc;
        }
        void *t = s->c;
        s->c = s->work;
        s->work = t;
    }
    return PB_OK;
}

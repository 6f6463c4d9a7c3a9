// stencil.cu — cuSten Compute2D{X,Y,XY}{p,np} with linear weights.
//
// B200 design: one CTA computes a TY x TX output tile.  The input tile plus
// its halo (top/bottom rows, left/right columns; periodic wrap or clipped) is
// staged once in shared memory with coalesced loads along i, then every thread
// evaluates its outputs from smem with the window weights held in a kernel
// parameter (broadcast, no constant-cache serialisation).  HBM traffic is one
// read and one write per point plus the halo re-reads (L2 hits).  The thesis's
// Unified-Memory tiling along y with stream prefetch is dropped:
// a 180 GB B200 holds every grid of this workload resident.
#include <string.h>

#include <algorithm>

#include "common.cuh"

namespace pb {

constexpr int ST_MAXW = 15;  // window <= 15 x 15 (extents <= 7 each side)
constexpr int ST_TX = 64, ST_TY = 16, ST_NT = 256;

struct StencilArgs {
    double w[ST_MAXW * ST_MAXW];
    int left, right, top, bottom;
    int64_t ny, nx;
    int periodic;
};

template <typename T>
__global__ void __launch_bounds__(ST_NT) stencil_kernel(const T *__restrict__ in, T *__restrict__ out,
                                                        const StencilArgs A)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *tile = reinterpret_cast<T *>(smem_raw);
    const int wx = A.left + A.right + 1, wy = A.top + A.bottom + 1;
    const int sx = ST_TX + wx - 1, sy = ST_TY + wy - 1;  // staged tile extent
    const int64_t i0 = (int64_t)blockIdx.x * ST_TX, j0 = (int64_t)blockIdx.y * ST_TY;
    const int64_t nx = A.nx, ny = A.ny;
    const int64_t plane = nx * ny;
    const T *g = in + (int64_t)blockIdx.z * plane;
    T *o = out + (int64_t)blockIdx.z * plane;
    // stage input rows j0-top .. j0+TY-1+bottom, columns i0-left .. i0+TX-1+right
    for (int e = threadIdx.x; e < sx * sy; e += ST_NT) {
        const int r = e / sx, q = e % sx;
        int64_t jj = j0 - A.top + r, ii = i0 - A.left + q;
        T v = T(0);
        if (A.periodic) {
            jj %= ny;
            if (jj < 0) jj += ny;
            ii %= nx;
            if (ii < 0) ii += nx;
            v = __ldg(g + jj * nx + ii);
        } else if (jj >= 0 && jj < ny && ii >= 0 && ii < nx) {
            v = __ldg(g + jj * nx + ii);
        }
        tile[r * sx + q] = v;
    }
    __syncthreads();
    // each thread: one column i, ST_TY / (ST_NT / ST_TX) rows
    const int tx = threadIdx.x % ST_TX, ty0 = threadIdx.x / ST_TX;
    constexpr int RSTEP = ST_NT / ST_TX;
    const int64_t i = i0 + tx;
    if (i >= nx) return;
    for (int ty = ty0; ty < ST_TY; ty += RSTEP) {
        const int64_t j = j0 + ty;
        if (j >= ny) break;
        if (!A.periodic && (j - A.top < 0 || j + A.bottom >= ny || i - A.left < 0 || i + A.right >= nx))
            continue;  // boundary cells untouched
        T acc = T(0);
        for (int r = 0; r < wy; ++r) {
            const T *row = tile + (ty + r) * sx + tx;
            const double *wr = A.w + r * wx;
            for (int q = 0; q < wx; ++q) acc += T(wr[q]) * row[q];
        }
        o[j * nx + i] = acc;
    }
}

}  // namespace pb

extern "C" int stencil_apply(const pb_grid *g, const void *in, void *out, const pb_window *w,
                             const double *weights, int boundary, void *stream)
{
    using namespace pb;
    if (!g || !w || !weights || !in || !out) return set_error(PB_EINVAL, "null argument");
    if (g->dtype != PB_F64 && g->dtype != PB_F32) return set_error(PB_EINVAL, "bad dtype");
    {
        // the output must not overlap the input anywhere (separate buffers)
        const size_t nb = dtype_size(g->dtype) * (size_t)(g->batch > 0 ? g->batch : 0) * (size_t)g->ny * (size_t)g->nx;
        const uintptr_t a0 = (uintptr_t)in, b0 = (uintptr_t)out;
        if (in == out || (nb > 0 && a0 < b0 + nb && b0 < a0 + nb))
            return set_error(PB_EINVAL, "in and out must not overlap (P:909)");
    }
    if (w->left < 0 || w->right < 0 || w->top < 0 || w->bottom < 0) return set_error(PB_EINVAL, "negative extent");
    const int wx = w->left + w->right + 1, wy = w->top + w->bottom + 1;
    if (wx > ST_MAXW || wy > ST_MAXW) return set_error(PB_EINVAL, "window larger than 15 x 15");
    if (g->batch < 0 || g->ny < 1 || g->nx < 1 || wx - 1 >= g->nx || wy - 1 >= g->ny)
        return set_error(PB_EINVAL, "window extents must be smaller than the grid");
    if (boundary != PB_PERIODIC && boundary != PB_NONPERIODIC) return set_error(PB_EINVAL, "bad boundary");
    if (pb_device_ok() != PB_OK) return PB_ECUDA;
    if (g->batch == 0) return PB_OK;
    cudaStream_t st = (cudaStream_t)stream;
    StencilArgs A;
    memset(&A, 0, sizeof(A));
    for (int k = 0; k < wx * wy; ++k) A.w[k] = weights[k];
    A.left = w->left;
    A.right = w->right;
    A.top = w->top;
    A.bottom = w->bottom;
    A.ny = g->ny;
    A.nx = g->nx;
    A.periodic = boundary == PB_PERIODIC;
    const size_t es = dtype_size(g->dtype);
    const size_t bytes = es * (size_t)(g->batch * g->ny * g->nx);
    Staged si, so;
    int rc;
    if ((rc = si.in(in, bytes, st, true))) return rc;
    // non-periodic leaves boundary cells untouched: the output must be copied in too
    if ((rc = so.in(out, bytes, st, true))) return rc;
    so.out_to(out);
    const size_t smem = es * (size_t)(ST_TX + wx - 1) * (ST_TY + wy - 1);
    // grid z is capped at 65535: launch the batch in slices
    const size_t plane = es * (size_t)g->ny * (size_t)g->nx;
    for (int64_t b0 = 0; b0 < g->batch; b0 += 65535) {
        const int64_t nbz = std::min<int64_t>(65535, g->batch - b0);
        dim3 grid((unsigned)((g->nx + ST_TX - 1) / ST_TX), (unsigned)((g->ny + ST_TY - 1) / ST_TY), (unsigned)nbz);
        const char *src = (const char *)si.dev + plane * (size_t)b0;
        char *dst = (char *)so.dev + plane * (size_t)b0;
        if (g->dtype == PB_F64)
            stencil_kernel<double><<<grid, ST_NT, smem, st>>>((const double *)src, (double *)dst, A);
        else
            stencil_kernel<float><<<grid, ST_NT, smem, st>>>((const float *)src, (float *)dst, A);
        PB_LAUNCH_CHECK();
    }
    if ((rc = si.finish())) return rc;
    return so.finish();
}

// mb_tile.cu — dev micro-benchmark (not product code): the HBM access pattern
// of band_tile_kernel's interleaved layout without the solve, to separate the
// memory-pattern ceiling from compute / barrier latency.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC tools/mb_tile.cu -o tools/libmb.so
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace cg = cooperative_groups;

// Each CTA: W consecutive systems x RC = (NT/W)*MR rows; thread (s, p) loads
// MR rows of system s (rows p*MR ..), optional barrier(s), stores them.
template <int W, int NT, int MR, int SYNC>
__global__ void __launch_bounds__(NT) tile_copy(const double *__restrict__ x, double *__restrict__ y, int64_t N,
                                                int64_t M, int C)
{
    constexpr int PC = NT / W, RC = PC * MR;
    const int tid = threadIdx.x, s = tid % W, p = tid / W;
    const int c = blockIdx.x % C;
    const int64_t group = blockIdx.x / C;
    const int64_t sys = group * W + s;
    const int64_t r0 = (int64_t)c * RC + (int64_t)p * MR;
    double v[MR];
#pragma unroll
    for (int k = 0; k < MR; ++k) v[k] = (r0 + k < N) ? __ldcs(x + (r0 + k) * M + sys) : 0.0;
    if (SYNC == 1) __syncthreads();
    if (SYNC == 2) cg::this_cluster().sync();
#pragma unroll
    for (int k = 0; k < MR; ++k) v[k] = v[k] * 1.0000001;
#pragma unroll
    for (int k = 0; k < MR; ++k)
        if (r0 + k < N) __stcs(y + (r0 + k) * M + sys, v[k]);
}

// Row-major streaming copy (reference ceiling): float4-wide grid-stride.
__global__ void stream_copy(const double2 *__restrict__ x, double2 *__restrict__ y, int64_t n2)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x)
        __stcs(y + i, __ldcs(x + i));
}

template <int W, int NT, int MR, int SYNC>
static void launch(const double *x, double *y, int64_t N, int64_t M, int C, cudaStream_t st)
{
    constexpr int RC = (NT / W) * MR;
    const int64_t crows = (N + RC - 1) / RC;  // CTAs per system group
    (void)C;
    const int Cc = (int)crows;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((M / W) * Cc));
    cfg.blockDim = dim3(NT);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = Cc;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = (SYNC == 2) ? 1 : 0;
    if (SYNC == 2 && Cc > 8) cudaFuncSetAttribute(tile_copy<W, NT, MR, SYNC>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchKernelEx(&cfg, tile_copy<W, NT, MR, SYNC>, x, y, N, M, Cc);
}

#define V(W, NT, MR)                                                   \
    case __COUNTER__: launch<W, NT, MR, 0>(x, y, N, M, 0, st); break; \
    case __COUNTER__: launch<W, NT, MR, 2>(x, y, N, M, 0, st); break;

extern "C" int mb_run(int variant, const double *x, double *y, int64_t N, int64_t M, int reps, float *ms)
{
    cudaStream_t st = 0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int r = -1; r < reps; ++r) {
        if (r == 0) cudaEventRecord(e0, st);
        switch (variant) {
            case 0: stream_copy<<<148 * 8, 512, 0, st>>>((const double2 *)x, (double2 *)y, N * M / 2); break;
            case 1: launch<16, 512, 32, 0>(x, y, N, M, 0, st); break;
            case 2: launch<16, 512, 32, 2>(x, y, N, M, 0, st); break;
            case 3: launch<16, 512, 16, 0>(x, y, N, M, 0, st); break;
            case 4: launch<16, 512, 16, 2>(x, y, N, M, 0, st); break;
            case 5: launch<32, 512, 32, 0>(x, y, N, M, 0, st); break;
            case 6: launch<32, 512, 16, 0>(x, y, N, M, 0, st); break;
            case 7: launch<64, 512, 32, 0>(x, y, N, M, 0, st); break;
            case 8: launch<16, 256, 32, 0>(x, y, N, M, 0, st); break;
            case 9: launch<16, 256, 32, 2>(x, y, N, M, 0, st); break;
            case 10: launch<32, 1024, 16, 0>(x, y, N, M, 0, st); break;
            case 11: launch<8, 256, 32, 0>(x, y, N, M, 0, st); break;
            case 12: launch<8, 256, 32, 2>(x, y, N, M, 0, st); break;
            case 13: launch<4, 128, 32, 0>(x, y, N, M, 0, st); break;
            case 14: launch<4, 128, 32, 2>(x, y, N, M, 0, st); break;
            case 15: launch<8, 128, 32, 0>(x, y, N, M, 0, st); break;
            case 16: launch<8, 128, 64, 2>(x, y, N, M, 0, st); break;
            case 17: launch<4, 64, 64, 2>(x, y, N, M, 0, st); break;
            case 18: launch<16, 256, 32, 0>(x, y, N, M, 0, st); break;
            case 19: launch<32, 256, 32, 0>(x, y, N, M, 0, st); break;
            default: return -1;
        }
    }
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(ms, e0, e1);
    *ms /= reps;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : (int)e;
}

// dependent-chain latency probes: fp64 FMA, fp32 FMA (cycles per op)
__global__ void lat_probe(double *out, float *outf, long long *cyc, int iters)
{
    double a = out[0], b = out[1], c = out[2];
    float af = outf[0], bf = outf[1], cf = outf[2];
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) c = fma(a, c, b);
    }
    long long t1 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) cf = fmaf(af, cf, bf);
    }
    long long t2 = clock64();
    out[3] = c;
    outf[3] = cf;
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
}
extern "C" int mb_lat(double *out, float *outf, long long *cyc, int iters)
{
    lat_probe<<<1, 1>>>(out, outf, cyc, iters);
    return (int)cudaDeviceSynchronize();
}

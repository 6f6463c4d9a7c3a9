// mb_compute.cu — dev micro-benchmark: the streaming solve's per-warp local
// tile solve (4 sweeps + 2 lane scans, SYS systems x MR rows per lane) on
// shared-memory-resident data, no global traffic; cycles per warp-item for
// 1..16 warps per SM.
#include "../paper_2101_06550_b200/csrc/stream_solve.cuh"

using namespace pb;

template <int STORE>
__global__ void __launch_bounds__(512, 1) compute_only(int items, long long *cyc, double *sink)
{
    using G = StreamGeom<double>;
    constexpr int SYS = G::SYS, MR = G::MR, PC = 32, R = PC * MR, W = G::W;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    double *tile = reinterpret_cast<double *>(smem_raw + ((1024 - ((uintptr_t)smem_raw & 1023)) & 1023));
    double(*coef)[MR][PC] = reinterpret_cast<double(*)[MR][PC]>(tile + R * W);
    double(*tab)[PC] = reinterpret_cast<double(*)[PC]>(tile + R * W + NCOEF * MR * PC);
    for (int e = threadIdx.x; e < R * W; e += blockDim.x) tile[e] = 1.0 + 1e-3 * (e % 97);
    for (int e = threadIdx.x; e < NCOEF * MR * PC; e += blockDim.x) (&coef[0][0][0])[e] = 0.5 + 1e-4 * (e % 13);
    for (int e = threadIdx.x; e < TAB_STRIDE * PC; e += blockDim.x) (&tab[0][0])[e] = 1e-3 * (e % 7);
    __syncthreads();
    const int lane = threadIdx.x & 31, q = (threadIdx.x >> 5) & 3, p = lane;
    double acc = 0;
    long long t0 = clock64();
    for (int it = 0; it < items; ++it) {
        double v[MR][SYS];
#pragma unroll
        for (int k = 0; k < MR; ++k) ld_row(tile, p * MR + k, q, v[k]);
        double c0[SYS], c1[SYS];
#pragma unroll
        for (int s = 0; s < SYS; ++s) c0[s] = c1[s] = 0;
#pragma unroll
        for (int k = 0; k < MR; ++k) {
            const double f0 = ldsh(&coef[0][k][p]), f1 = ldsh(&coef[1][k][p]), f2 = ldsh(&coef[2][k][p]);
#pragma unroll
            for (int s = 0; s < SYS; ++s) {
                double gv = f0 * v[k][s];
                gv -= f2 * c0[s];
                gv -= f1 * c1[s];
                c0[s] = c1[s];
                c1[s] = gv;
            }
        }
        warp_scan<double, SYS, false>(c0, c1, p, tab, TAB_PF);
        {
            double y0[SYS], y1[SYS];
#pragma unroll
            for (int s = 0; s < SYS; ++s) {
                y0[s] = __shfl_up_sync(0xffffffffu, c0[s], 1);
                y1[s] = __shfl_up_sync(0xffffffffu, c1[s], 1);
                if (p == 0) y0[s] = y1[s] = 0;
            }
#pragma unroll
            for (int k = 0; k < MR; ++k) {
                const double f0 = ldsh(&coef[0][k][p]), f1 = ldsh(&coef[1][k][p]), f2 = ldsh(&coef[2][k][p]);
#pragma unroll
                for (int s = 0; s < SYS; ++s) {
                    double gv = f0 * v[k][s];
                    gv -= f2 * y0[s];
                    gv -= f1 * y1[s];
                    y0[s] = y1[s];
                    y1[s] = gv;
                    v[k][s] = gv;
                }
            }
        }
#pragma unroll
        for (int s = 0; s < SYS; ++s) c0[s] = c1[s] = 0;
#pragma unroll
        for (int k = MR - 1; k >= 0; --k) {
            const double b1 = ldsh(&coef[3][k][p]), b2 = ldsh(&coef[4][k][p]);
#pragma unroll
            for (int s = 0; s < SYS; ++s) {
                double xx = v[k][s];
                xx -= b2 * c1[s];
                xx -= b1 * c0[s];
                c1[s] = c0[s];
                c0[s] = xx;
            }
        }
        warp_scan<double, SYS, true>(c0, c1, p, tab, TAB_PB);
        {
            double z0[SYS], z1[SYS];
#pragma unroll
            for (int s = 0; s < SYS; ++s) {
                z0[s] = __shfl_down_sync(0xffffffffu, c0[s], 1);
                z1[s] = __shfl_down_sync(0xffffffffu, c1[s], 1);
                if (p == 31) z0[s] = z1[s] = 0;
            }
#pragma unroll
            for (int k = MR - 1; k >= 0; --k) {
                const double b1 = ldsh(&coef[3][k][p]), b2 = ldsh(&coef[4][k][p]);
#pragma unroll
                for (int s = 0; s < SYS; ++s) {
                    double xx = v[k][s];
                    xx -= b2 * z1[s];
                    xx -= b1 * z0[s];
                    z1[s] = z0[s];
                    z0[s] = xx;
                    v[k][s] = xx;
                }
            }
        }
        if (STORE) {
            double *dst = sink + ((size_t)blockIdx.x * 16 + (threadIdx.x >> 5)) * 32 * MR * SYS + lane * SYS;
#pragma unroll
            for (int k = 0; k < MR; ++k) st_row<true>(dst + k * 32 * SYS, v[k]);
        } else {
#pragma unroll
            for (int k = 0; k < MR; ++k)
#pragma unroll
                for (int s = 0; s < SYS; ++s) acc += v[k][s];
        }
    }
    long long t1 = clock64();
    if (lane == 0) cyc[blockIdx.x * 16 + (threadIdx.x >> 5)] = t1 - t0;
    if (acc == 123.0) sink[0] = acc;
}

extern "C" int mbc_run(int warps, int items, int store, long long *cyc, double *sink, float *ms)
{
    const size_t smem = 1024 + sizeof(double) * (224 * 16 + NCOEF * 7 * 32 + TAB_STRIDE * 32);
    auto k = store ? compute_only<1> : compute_only<0>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<148, warps * 32, smem>>>(items, cyc, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(ms, e0, e1);
    return (int)cudaGetLastError();
}

// mb_sweep.cu — dev micro-benchmark: cycles per row of the cluster solve's
// chunk sweep (fwd_blocks / bwd_blocks) on shared memory, coefficients via L1.
#include "../paper_2101_06550_b200/csrc/cluster_solve.cuh"
using namespace pb;
using namespace pb::clu;

template <int MODE>
__global__ void __launch_bounds__(288, 1) sweep_bench(const double *cc, int reps, long long *cyc, double *sink)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *buf = reinterpret_cast<double *>(smem_raw);
    constexpr int W = 16;
    for (int e = threadIdx.x; e < 512 * W; e += blockDim.x) buf[e] = 1.0 + 1e-3 * (e % 17);
    __syncthreads();
    if (threadIdx.x >= 256) return;
    const int s = threadIdx.x % W, p = threadIdx.x / W;
    double *col = buf + s + p * 32 * W;
    const double *ccr = cc + p * 32 * 8;
    double y0 = 0, y1 = 0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        if (MODE == 0) fwd_blocks<double, 2, false>(col, ccr, y0, y1);
        if (MODE == 1) fwd_blocks<double, 2, true>(col, ccr, y0, y1);
        if (MODE == 2) bwd_blocks<double, 2, true>(col, ccr, y0, y1);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (y0 == 12345.0) sink[0] = y1;
}
extern "C" int mbs_run(int mode, const double *cc, int reps, long long *cyc, double *sink, float *ms)
{
    const size_t smem = 512 * 16 * 8;
    auto k = mode == 0 ? sweep_bench<0> : mode == 1 ? sweep_bench<1> : sweep_bench<2>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<148, 288, smem>>>(cc, reps, cyc, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(ms, e0, e1);
    return (int)cudaGetLastError();
}

// Dependent-latency micro-benchmarks (dev tool): DFMA / FFMA chains, LDS
// pointer chase, DSMEM store + fence.acq_rel.cluster round trip.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void dfma_chain(double *out, double a, double b, int n, long long *cyc)
{
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) x = fma(x, a, b);
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void ffma_chain(float *out, float a, float b, int n, long long *cyc)
{
    float x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) x = fmaf(x, a, b);
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lds_chase(int *out, int n, long long *cyc)
{
    __shared__ int s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i + 33) & 1023;
    __syncthreads();
    int p = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) p = s[p];
    long long t1 = clock64();
    out[threadIdx.x] = p;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void dsmem_rt(double *out, int n, long long *cyc)
{
    __shared__ double buf[64];
    auto cl = cg::this_cluster();
    const unsigned r = cl.block_rank(), peer = (r + 1) % cl.num_blocks();
    double *pb = cl.map_shared_rank(buf, peer);
    cl.sync();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        pb[threadIdx.x & 63] = i;
        asm volatile("fence.acq_rel.cluster;" ::: "memory");
    }
    long long t1 = clock64();
    cl.sync();
    out[r] = buf[0];
    if (threadIdx.x == 0 && r == 0) cyc[0] = t1 - t0;
}
__global__ void dsmem_ld(double *out, int n, long long *cyc)
{
    __shared__ double buf[64];
    auto cl = cg::this_cluster();
    const unsigned r = cl.block_rank(), peer = (r + 1) % cl.num_blocks();
    for (int i = threadIdx.x; i < 64; i += blockDim.x) buf[i] = (i + 1) & 63;
    cl.sync();
    double *pb = cl.map_shared_rank(buf, peer);
    int p = threadIdx.x & 63;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) p = (int)pb[p];
    long long t1 = clock64();
    cl.sync();
    out[r] = p;
    if (threadIdx.x == 0 && r == 0) cyc[0] = t1 - t0;
}
int main()
{
    double *od;
    float *of;
    int *oi;
    long long *cyc, h;
    cudaMalloc(&od, 4096 * 8);
    cudaMalloc(&of, 4096 * 4);
    cudaMalloc(&oi, 4096 * 4);
    cudaMalloc(&cyc, 8);
    const int n = 1000;
    for (int threads : {32, 256}) {
        dfma_chain<<<1, threads>>>(od, 1.0000001, 1e-9, n, cyc);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("DFMA dependent latency (%d threads/CTA): %.2f cycles\n", threads, (double)h / (16.0 * n));
        ffma_chain<<<1, threads>>>(of, 1.0000001f, 1e-9f, n, cyc);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("FFMA dependent latency (%d threads/CTA): %.2f cycles\n", threads, (double)h / (16.0 * n));
    }
    lds_chase<<<1, 32>>>(oi, n, cyc);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("LDS chase latency: %.2f cycles\n", (double)h / n);
    for (int cs : {2, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs);
        cfg.blockDim = dim3(32);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaFuncSetAttribute(dsmem_rt, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaFuncSetAttribute(dsmem_ld, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaError_t e = cudaLaunchKernelEx(&cfg, dsmem_rt, od, n, cyc);
        cudaDeviceSynchronize();
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("cluster %d: DSMEM store + fence.acq_rel.cluster: %.1f cycles (%s)\n", cs, (double)h / n, cudaGetErrorString(e));
        e = cudaLaunchKernelEx(&cfg, dsmem_ld, od, n, cyc);
        cudaDeviceSynchronize();
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("cluster %d: DSMEM load chase: %.1f cycles (%s)\n", cs, (double)h / n, cudaGetErrorString(e));
    }
    return 0;
}

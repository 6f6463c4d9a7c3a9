// mb2.cu — dev micro-benchmarks (not product code): HBM access patterns for
// W-wide column strips of a row-major N x M fp64 array (the interleaved
// layout of the batched solve), via TMA bulk tensor copies and via LDG, plus
// the L2-hit read bandwidth.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC tools/mb2.cu -o tools/libmb2.so
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *b, int cnt)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity)
{
    asm volatile(
        "{\n .reg .pred p;\n"
        "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *m, int c0, int c1, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(m), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap *m, int c0, int c1, const void *src)
{
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(m), "r"(c0),
                 "r"(c1), "r"(smem_u32(src))
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read()
{
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Persistent TMA copy: tiles of W x R (box), S-stage ring, one thread issues.
// order 0: row-block-major (consecutive tiles = neighbouring column groups),
// order 1: group-major.
template <int S>
__global__ void tma_copy(const __grid_constant__ CUtensorMap src, const __grid_constant__ CUtensorMap dst, int ngroups,
                         int nrb, int W, int R, int order)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) uint64_t full[S];
    const int tile_bytes = W * R * 8;
    const int ntiles = ngroups * nrb;
    if (threadIdx.x != 0) return;
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    auto coords = [&](int t, int &c0, int &c1) {
        int g, rb;
        if (order == 0) {
            rb = t / ngroups;
            g = t % ngroups;
        } else {
            g = t / nrb;
            rb = t % nrb;
        }
        c0 = g * W;
        c1 = rb * R;
    };
    // my tiles: blockIdx.x + k*gridDim.x
    int cnt = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) ++cnt;
    for (int k = 0; k < S && k < cnt; ++k) {
        int c0, c1;
        coords(blockIdx.x + k * gridDim.x, c0, c1);
        mbar_expect_tx(&full[k], tile_bytes);
        tma_load_2d(sm + k * tile_bytes, &src, c0, c1, &full[k]);
    }
    for (int k = 0; k < cnt; ++k) {
        const int s = k % S;
        mbar_wait(&full[s], (k / S) & 1);
        int c0, c1;
        coords(blockIdx.x + k * gridDim.x, c0, c1);
        tma_store_2d(&dst, c0, c1, sm + s * tile_bytes);
        bulk_commit();
        // refill the previous stage once its store has read smem
        if (k >= 1) {
            bulk_wait_read<1>();
            const int kk = k - 1 + S;
            if (kk < cnt) {
                const int ps = (k - 1) % S;
                coords(blockIdx.x + kk * gridDim.x, c0, c1);
                mbar_expect_tx(&full[ps], tile_bytes);
                tma_load_2d(sm + ps * tile_bytes, &src, c0, c1, &full[ps]);
            }
        }
    }
    bulk_wait_all();
}

// LDG "tile-order streaming": CTA = (group, row block); each warp streams rows,
// 32 lanes = (32/W) rows x W systems; load and store immediately.
__global__ void ldg_tile_stream(const double *__restrict__ x, double *__restrict__ y, int64_t N, int64_t M, int W, int RB)
{
    const int64_t ngroups = M / W;
    const int64_t g = blockIdx.x % ngroups, rb = blockIdx.x / ngroups;
    const int lanes_per_row = W, rows_per_pass = blockDim.x / W;
    const int s = threadIdx.x % lanes_per_row, r = threadIdx.x / lanes_per_row;
    for (int64_t i = rb * RB + r; i < (rb + 1) * RB && i < N; i += rows_per_pass) {
        const int64_t idx = i * M + g * W + s;
        __stcs(y + idx, __ldcs(x + idx));
    }
}

// L2-hit read bandwidth: every CTA reads [off, off+len) of a small buffer repeatedly.
__global__ void l2_read(const double2 *__restrict__ x, int64_t n2, int reps, double *out)
{
    double acc = 0;
    for (int r = 0; r < reps; ++r)
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
            double2 v = __ldcg(x + i);
            acc += v.x + v.y;
        }
    if (acc == 123.456) out[0] = acc;
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode()
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&fn, cudaEnableDefault, &q);
    }
    return fn;
}

static int make_map(CUtensorMap *m, const void *base, int64_t N, int64_t M, int W, int R)
{
    cuuint64_t dims[2] = {(cuuint64_t)M, (cuuint64_t)N};
    cuuint64_t strides[1] = {(cuuint64_t)M * 8};
    cuuint32_t box[2] = {(cuuint32_t)W, (cuuint32_t)R};
    cuuint32_t es[2] = {1, 1};
    CUresult r = get_encode()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void *)base, dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return (int)r;
}

extern "C" int mb2_tma(const double *x, double *y, int64_t N, int64_t M, int W, int R, int stages, int ctas_per_sm,
                       int order, int reps, float *ms)
{
    CUtensorMap ms_, md_;
    int rc = make_map(&ms_, x, N, M, W, R);
    if (rc) return 1000 + rc;
    rc = make_map(&md_, y, N, M, W, R);
    if (rc) return 2000 + rc;
    const int ngroups = (int)(M / W), nrb = (int)(N / R);
    const size_t smem = (size_t)stages * W * R * 8;
    void (*k)(CUtensorMap, CUtensorMap, int, int, int, int, int) = nullptr;
    switch (stages) {
        case 2: k = tma_copy<2>; break;
        case 3: k = tma_copy<3>; break;
        case 4: k = tma_copy<4>; break;
        case 6: k = tma_copy<6>; break;
        case 8: k = tma_copy<8>; break;
        case 12: k = tma_copy<12>; break;
        case 16: k = tma_copy<16>; break;
        default: return -1;
    }
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = 148 * ctas_per_sm;
    for (int r = -1; r < reps; ++r) {
        if (r == 0) cudaEventRecord(e0);
        k<<<grid, 32, smem>>>(ms_, md_, ngroups, nrb, W, R, order);
    }
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(ms, e0, e1);
    *ms /= reps;
    return (int)cudaGetLastError();
}

extern "C" int mb2_ldg_stream(const double *x, double *y, int64_t N, int64_t M, int W, int RB, int nt, int reps,
                              float *ms)
{
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int64_t grid = (M / W) * (N / RB);
    for (int r = -1; r < reps; ++r) {
        if (r == 0) cudaEventRecord(e0);
        ldg_tile_stream<<<(unsigned)grid, nt>>>(x, y, N, M, W, RB);
    }
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(ms, e0, e1);
    *ms /= reps;
    return (int)cudaGetLastError();
}

extern "C" int mb2_l2(const double *x, int64_t n, int reps, double *out, float *ms)
{
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    l2_read<<<148 * 4, 512>>>((const double2 *)x, n / 2, 1, out);
    cudaEventRecord(e0);
    l2_read<<<148 * 4, 512>>>((const double2 *)x, n / 2, reps, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(ms, e0, e1);
    return (int)cudaGetLastError();
}

// Persistent cluster "tile hold" emulation of the solve: each CTA (512 threads
// = 16 systems x 32 chunks of MR rows) owns rows [c*RC, (c+1)*RC) of a
// 16-system group; TMA prefetches the next group's rows into smem while the
// current one sits in registers through a fake dependent-FMA "solve" and two
// cluster barriers; results leave by STG (STORE_TMA=0) or STS + TMA store (1).
#include <cooperative_groups.h>
template <int MR, int STORE_TMA>
__global__ void __launch_bounds__(512, 1) tile_hold(const __grid_constant__ CUtensorMap src,
                                                    const __grid_constant__ CUtensorMap dst, double *y, int64_t M,
                                                    int ngroups, int C, int chain, int csync)
{
    namespace cg = cooperative_groups;
    constexpr int W = 16, RC = 32 * MR, BOX = 256, NBOX = RC / BOX > 0 ? RC / BOX : 1, BR = RC < BOX ? RC : BOX;
    extern __shared__ __align__(1024) unsigned char sm[];
    double *buf = reinterpret_cast<double *>(sm);
    double *obuf = buf + RC * W;
    __shared__ __align__(8) uint64_t full;
    const int tid = threadIdx.x, s = tid % W, p = tid / W;
    const int c = blockIdx.x % C, k = blockIdx.x / C, ncl = gridDim.x / C;
    if (tid == 0) {
        mbar_init(&full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int g = k;
    if (tid == 0 && g < ngroups) {
        mbar_expect_tx(&full, RC * W * 8);
        for (int b = 0; b < NBOX; ++b) tma_load_2d(buf + b * BR * W, &src, g * W, c * RC + b * BR, &full);
    }
    uint32_t phase = 0;
    for (; g < ngroups; g += ncl) {
        mbar_wait(&full, phase);
        phase ^= 1;
        double v[MR];
#pragma unroll
        for (int q = 0; q < MR; ++q) v[q] = buf[(p * MR + q) * W + s];
        __syncthreads();
        const int gn = g + ncl;
        if (tid == 0 && gn < ngroups) {
            mbar_expect_tx(&full, RC * W * 8);
            for (int b = 0; b < NBOX; ++b) tma_load_2d(buf + b * BR * W, &src, gn * W, c * RC + b * BR, &full);
        }
        // fake solve: `chain` dependent sweeps over the MR values
        double acc = 0.0;
        for (int it = 0; it < chain; ++it) {
#pragma unroll
            for (int q = 0; q < MR; ++q) {
                acc = fma(acc, 0.5, v[q]);
                v[q] = acc;
            }
            if (csync && (it & 1)) {
                if (C > 1)
                    cg::this_cluster().sync();
                else
                    __syncthreads();
            }
        }
        if (STORE_TMA == 0) {
            double *dstp = y + (int64_t)(c * RC + p * MR) * M + g * W + s;
#pragma unroll
            for (int q = 0; q < MR; ++q) __stcs(dstp + q * M, v[q]);
        } else {
            if (tid == 0) bulk_wait_read<0>();
            __syncthreads();
#pragma unroll
            for (int q = 0; q < MR; ++q) obuf[(p * MR + q) * W + s] = v[q];
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (tid == 0) {
                for (int b = 0; b < NBOX; ++b) tma_store_2d(&dst, g * W, c * RC + b * BR, obuf + b * BR * W);
                bulk_commit();
            }
        }
    }
    if (STORE_TMA && tid == 0) bulk_wait_all();
}

extern "C" int mb2_hold(const double *x, double *y, int64_t N, int64_t M, int mr, int store_tma, int chain, int csync,
                        int reps, float *ms, int *nclusters)
{
    const int RC = 32 * mr, BR = RC < 256 ? RC : 256;
    CUtensorMap ms_, md_;
    int rc = make_map(&ms_, x, N, M, 16, BR);
    if (rc) return 1000 + rc;
    rc = make_map(&md_, y, N, M, 16, BR);
    if (rc) return 2000 + rc;
    const int C = (int)(N / RC);
    void (*k)(CUtensorMap, CUtensorMap, double *, int64_t, int, int, int, int) = nullptr;
    if (mr == 32 && store_tma == 0) k = tile_hold<32, 0>;
    if (mr == 16 && store_tma == 0) k = tile_hold<16, 0>;
    if (mr == 16 && store_tma == 1) k = tile_hold<16, 1>;
    if (mr == 8 && store_tma == 1) k = tile_hold<8, 1>;
    if (mr == 8 && store_tma == 0) k = tile_hold<8, 0>;
    if (!k) return -1;
    const size_t smem = (size_t)RC * 16 * 8 * (store_tma ? 2 : 1);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (C > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(C);
    int ncl = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, k, &cfg);
    if (e != cudaSuccess) return 3000 + (int)e;
    *nclusters = ncl;
    cfg.gridDim = dim3(ncl * C);
    const int ngroups = (int)(M / 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int r = -1; r < reps; ++r) {
        if (r == 0) cudaEventRecord(e0);
        cudaLaunchKernelEx(&cfg, k, ms_, md_, y, M, ngroups, C, chain, csync);
    }
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(ms, e0, e1);
    *ms /= reps;
    return (int)cudaGetLastError();
}

// TMA copy restricted to `ctas` CTAs (e.g. 128 = what 8-CTA clusters can occupy)
extern "C" int mb2_tma_n(const double *x, double *y, int64_t N, int64_t M, int W, int R, int ctas, int reps, float *ms)
{
    CUtensorMap ms_, md_;
    make_map(&ms_, x, N, M, W, R);
    make_map(&md_, y, N, M, W, R);
    const size_t smem = (size_t)4 * W * R * 8;
    cudaFuncSetAttribute(tma_copy<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int r = -1; r < reps; ++r) {
        if (r == 0) cudaEventRecord(e0);
        tma_copy<4><<<ctas, 32, smem>>>(ms_, md_, (int)(M / W), (int)(N / R), W, R, 0);
    }
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(ms, e0, e1);
    *ms /= reps;
    return (int)cudaGetLastError();
}

// Two-phase (SPIKE with L2 re-read) traffic emulation: the work sequence
// interleaves P1(tile k) [load only] with P2(tile k-D) [load + store].
// Tiles are enumerated super-group by super-group (G groups of W systems),
// row-block-major inside a super-group.  Static round-robin over CTAs.
template <int S>
__global__ void tma_twophase(const __grid_constant__ CUtensorMap src, const __grid_constant__ CUtensorMap dst,
                             int ngroups, int nrb, int W, int R, int G, int D)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) uint64_t full[S];
    const int tile_bytes = W * R * 8;
    const int ntiles = ngroups * nrb;
    if (threadIdx.x != 0) return;
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int nitems = 2 * (ntiles + D);
    auto item = [&](int it, int &c0, int &c1, int &st) -> bool {  // false: no-op
        int k = it >> 1;
        st = it & 1;
        if (st) k -= D;
        if (k < 0 || k >= ntiles) return false;
        const int per_sg = G * nrb;
        const int sg = k / per_sg, r = k % per_sg;
        const int rb = r / G, gg = r % G;
        const int g = sg * G + gg;
        if (g >= ngroups) return false;
        c0 = g * W;
        c1 = rb * R;
        return true;
    };
    // my items: it = blockIdx.x + j*gridDim.x
    int cnt = 0;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) ++cnt;
    int c0, c1, st;
    int issued = 0;
    auto issue = [&](int j) {
        const int s = j % S;
        if (item(blockIdx.x + j * gridDim.x, c0, c1, st)) {
            mbar_expect_tx(&full[s], tile_bytes);
            tma_load_2d(sm + s * tile_bytes, &src, c0, c1, &full[s]);
        } else {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])) : "memory");
        }
    };
    for (; issued < S && issued < cnt; ++issued) issue(issued);
    for (int j = 0; j < cnt; ++j) {
        const int s = j % S;
        mbar_wait(&full[s], (j / S) & 1);
        if (item(blockIdx.x + j * gridDim.x, c0, c1, st) && st) {
            tma_store_2d(&dst, c0, c1, sm + s * tile_bytes);
        }
        bulk_commit();
        bulk_wait_read<0>();
        if (issued < cnt) issue(issued++);
    }
    bulk_wait_all();
}

extern "C" int mb2_twophase(const double *x, double *y, int64_t N, int64_t M, int W, int R, int G, int D, int ctas,
                            int reps, float *ms)
{
    CUtensorMap ms_, md_;
    if (make_map(&ms_, x, N, M, W, R)) return 1;
    if (make_map(&md_, y, N, M, W, R)) return 2;
    const size_t smem = (size_t)4 * W * R * 8;
    cudaFuncSetAttribute(tma_twophase<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int r = -1; r < reps; ++r) {
        if (r == 0) cudaEventRecord(e0);
        tma_twophase<4><<<ctas, 32, smem>>>(ms_, md_, (int)(M / W), (int)(N / R), W, R, G, D);
    }
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(ms, e0, e1);
    *ms /= reps;
    return (int)cudaGetLastError();
}

// fused_part.cuh — launchers of the fused solve kernels (fused_cluster.cuh,
// fused_solve.cuh) for one (dtype, layout); included by fused_part_*.cu with
// FS_T / FS_LAY / FS_NAME defined, so the instantiations compile in parallel.
#include <cudaTypedefs.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "band_tile.cuh"
#include "fused_cluster.cuh"
#include "fused_hold.cuh"
#include "twopass.cuh"

namespace pb {

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();
int fs_sm_count();

// L2 budget for the lag window of f between P1(g) and P2(g) (the L2 is 126 MB;
// the window, the x write-back in flight and the scratch records share it)
constexpr double FS_L2_BUDGET = 40.0 * 1048576.0;   // lag window of f between P1(g) and P2(g)

// Tensor map over x for either layout, cached per (stream, layout).
// Interleaved: dims (M, n, count), box (32 systems, 64 rows, 1); contiguous:
// dims (n, M, count), box (128 B of rows, 32 systems, 1), 128B swizzle.  OOB
// loads zero-fill and OOB stores are clipped (ragged M and n).  Batches that
// tiles cannot straddle use one 2-D view (flat).
template <typename T, int LAY>
static int tensor_map_for(FusedScratch &S, T *x, int64_t M, int64_t n, int64_t count, int64_t bstride, int64_t P,
                          CUtensorMap *out, bool *flat_out)
{
    const int64_t dpitch = LAY == fs::LAY_CONTIG ? n : M;
    const bool flat = P == dpitch && (LAY == fs::LAY_CONTIG
                          ? (count == 1 || (bstride == M * n && M % fs::TW == 0))
                          : (count == 1 || (bstride == M * n && n % fs::Q == 0 && n * count < ((int64_t)1 << 31))));
    const uint64_t key[6] = {(uint64_t)(uintptr_t)x, (uint64_t)M, (uint64_t)n, (uint64_t)count, (uint64_t)bstride,
                             (uint64_t)P * 16 + sizeof(T) * 2 + LAY};
    uint64_t *skey = S.key[LAY];
    void *smap = S.tmap[LAY];
    if (memcmp(key, skey, sizeof(key)) != 0) {
        auto enc = tensor_map_encoder();
        if (!enc) return set_error(PB_ECUDA, "cuTensorMapEncodeTiled unavailable");
        const auto dt = sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
        const int rank = flat ? 2 : 3;
        const int64_t bs = count > 1 ? bstride : P * (LAY == fs::LAY_CONTIG ? M : n);
        CUresult r;
        cuuint32_t estr[3] = {1, 1, 1};
        if (LAY == fs::LAY_CONTIG) {
            cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)(flat ? M * count : M), (cuuint64_t)(flat ? 1 : count)};
            cuuint64_t strides[2] = {(cuuint64_t)(P * sizeof(T)), (cuuint64_t)(bs * sizeof(T))};
            cuuint32_t box[3] = {(cuuint32_t)fs::Sw<T>::EB, (cuuint32_t)fs::TW, 1};
            r = enc((CUtensorMap *)smap, dt, rank, (void *)x, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {
            cuuint64_t dims[3] = {(cuuint64_t)M, (cuuint64_t)(flat ? n * count : n), (cuuint64_t)(flat ? 1 : count)};
            cuuint64_t strides[2] = {(cuuint64_t)(P * sizeof(T)), (cuuint64_t)(bs * sizeof(T))};
            cuuint32_t box[3] = {(cuuint32_t)fs::TW, (cuuint32_t)fs::Q, 1};
            r = enc((CUtensorMap *)smap, dt, rank, (void *)x, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        if (r != CUDA_SUCCESS) return set_error(PB_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
        memcpy(skey, key, sizeof(key));
    }
    memcpy(out, smap, sizeof(CUtensorMap));
    *flat_out = flat;
    return PB_OK;
}

// ---------------------------------------------------------------- held-tile kernel launcher
// Cluster size CS = ceil(nq / NW) (one chunk per consumer warp), cpc =
// ceil(nq / CS) chunks per CTA; clusters = the occupancy API's maximum (each
// loops over groups).  PB_EUNSUPPORTED when nq > CSM * NW or the cluster does
// not fit the GPU (the two-pass cluster kernel serves).
template <typename T, int K, bool PER, int MODE, int LAY>
static int fh_launch_t(const Band *h, T *x, T *xout, double alpha, int64_t count, int64_t bstride, cudaStream_t st,
                       int64_t Mo, int64_t pitch, int *info = nullptr)
{
    constexpr int CSM = fh::csmax<MODE>();
    auto kern = fh::fh_kernel<T, K, PER, MODE, LAY>;
    const size_t smem = sizeof(fh::HSmem<T, MODE>) + 1024;
    static std::once_flag once;
    static cudaError_t attr = cudaSuccess;
    static int ncl_of[CSM + 1];
    std::call_once(once, [&] {
        attr = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (attr == cudaSuccess) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaGetLastError();
        for (int cs = 1; cs <= CSM; ++cs) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)(cs * 16));
            cfg.blockDim = dim3(fh::NTHREADS);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cs;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int ncl = 0;
            if (attr == cudaSuccess && cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) != cudaSuccess) ncl = 0;
            cudaGetLastError();
            ncl_of[cs] = ncl;
        }
    });
    if (attr != cudaSuccess) return PB_EUNSUPPORTED;
    const int64_t M = Mo > 0 ? Mo : h->batch, n = h->n;
    const int64_t P = pitch > 0 ? pitch : (LAY == fs::LAY_CONTIG ? n : M);
    const int nq = h->fplan.nq;
    const int64_t Gb = (M + fs::TW - 1) / fs::TW, G = Gb * count;
    const int cs = (nq + fh::NW - 1) / fh::NW;
    if (G > (1 << 30) || cs > CSM || ncl_of[cs] < 1) return PB_EUNSUPPORTED;
    const int cpc = (nq + cs - 1) / cs;
    const int ncl = (int)std::min<int64_t>(ncl_of[cs], G);
    if (info) {
        info[0] = cs;
        info[1] = cpc;
        info[2] = ncl;
        info[3] = 2;
        return PB_OK;
    }
    fc::CArgs<T> A;
    CUtensorMap tmap;
    {
        std::lock_guard<std::mutex> lk(h->fplan.mu);
        FusedScratch &S = h->fplan.scratch[st];
        bool flat = false;
        int rc = tensor_map_for<T, LAY>(S, x, M, n, count, bstride, P, &tmap, &flat);
        if (rc) return rc;
        A.flat = flat ? 1 : 0;
    }
    A.rec = (const T *)h->fplan.rec;
    A.coef = (const T *)h->coef;
    A.ct = (const T *)h->fplan.ct;
    A.rsp = (const T *)h->fplan.rsp;
    A.scal = h->scal;
    A.x = x;
    A.xout = xout;
    A.alpha = (T)alpha;
    A.n = n;
    A.M = M;
    A.bstride = count > 1 ? bstride : P * (LAY == fs::LAY_CONTIG ? M : n);
    A.pitch = P;
    for (int j = 0; j < 4; ++j) A.srow[j] = h->srow[j];
    A.nq = nq;
    A.count = (int)count;
    A.Gb = (int)Gb;
    A.G = (int)G;
    A.cs = cs;
    A.cpc = cpc;
    A.ncl = ncl;
    A.dbg = 0;
    A.prof = nullptr;
#ifdef FH_PROF
    static long long *dprof = nullptr;
    static long long hprof[8 * 16];
    static int nlaunch = 0;
    if (!dprof) {
        cudaMalloc(&dprof, sizeof(hprof));
        cudaMemset(dprof, 0, sizeof(hprof));
        atexit([] {
            cudaMemcpy(hprof, dprof, sizeof(hprof), cudaMemcpyDeviceToHost);
            fprintf(stderr, "FH_PROF launches %d (cycles per launch, summed over CTAs; per warp)\n", nlaunch);
            const char *nm[16] = {"wait_full", "vload_issue", "P1", "wait_p1done", "scan", "wait_scandone", "P2", "store",
                                  "s_fwd", "s_bwd", "s_xcons", "s_xwrite", "s_xwait", "s_resolve", "s_walk", "s_cyc"};
            for (int w = 0; w < 8; ++w) {
                fprintf(stderr, "w%d", w);
                for (int i = 0; i < 16; ++i)
                    if (hprof[w * 16 + i]) fprintf(stderr, " %s=%.0f", nm[i], (double)hprof[w * 16 + i] / nlaunch);
                fprintf(stderr, "\n");
            }
        });
    }
    A.prof = dprof;
    ++nlaunch;
#endif
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(ncl * cs));
    cfg.blockDim = dim3(fh::NTHREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    PB_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, tmap, A));
    PB_LAUNCH_CHECK();
    return PB_OK;
}


// ---------------------------------------------------------------- two-pass launcher (interleaved)
// P1 (+ group scans) then P2 as its programmatic dependent.  Consumer warps
// per CTA and ring depth per warp: fp64 4 x 2 (P1 152 KB, P2 172 KB of
// slots), fp32 4 x 4.
#ifndef TP_NC1_64
#define TP_NC1_64 4
#define TP_R1_64 2
#define TP_NC2_64 4
#define TP_R2_64 2
#define TP_NC1_32 4
#define TP_R1_32 4
#define TP_NC2_32 4
#define TP_R2_32 4
#endif
template <typename T>
struct TpCfg {
    static constexpr int NC1 = sizeof(T) == 8 ? TP_NC1_64 : TP_NC1_32, R1 = sizeof(T) == 8 ? TP_R1_64 : TP_R1_32;
    static constexpr int NC2 = sizeof(T) == 8 ? TP_NC2_64 : TP_NC2_32, R2 = sizeof(T) == 8 ? TP_R2_64 : TP_R2_32;
};

template <typename T, int K, bool PER, int LAY>
static int tp_launch_t(const Band *h, T *x, int64_t count, int64_t bstride, cudaStream_t st, int64_t Mo, int64_t pitch)
{
    constexpr int NC = TpCfg<T>::NC1, R = TpCfg<T>::R1, NC2 = TpCfg<T>::NC2, R2 = TpCfg<T>::R2;
    auto k1 = tp::tp_p1_kernel<T, K, PER, NC, R, LAY>;
    auto k2 = tp::tp_p2_kernel<T, K, PER, NC2, R2, LAY>;
    auto ks = tp::tp_scan_kernel<T, K, PER>;
    auto ks8 = tp::tp_scan_kernel<T, K, PER, 8>;
    const size_t sm1 = sizeof(tp::P1Smem<T, NC, R>) + 1024;
    const size_t sm2 = sizeof(tp::P2Smem<T, NC2, R2>) + 1024;
    const int slt = h->fplan.nq <= 8 ? 8 : tp::SL, nsg = (h->fplan.nq + slt - 1) / slt;
    const size_t sms = sizeof(T) * tp::scan_smem_elems<T>(nsg, h->fplan.nq);
    if (h->fplan.nq > tp::SL * tp::NSEG) return PB_EUNSUPPORTED;   // longer systems: the global kernel serves
    static std::once_flag once;
    static cudaError_t attr = cudaSuccess;
    std::call_once(once, [&] {
        attr = cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
        if (attr == cudaSuccess) attr = cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        if (attr == cudaSuccess) attr = cudaFuncSetAttribute(ks8, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        if (attr == cudaSuccess) attr = cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
        cudaGetLastError();
    });
    if (attr != cudaSuccess) return set_error(PB_ECUDA, "tp kernels smem attribute: %s", cudaGetErrorString(attr));
    const int64_t M = Mo > 0 ? Mo : h->batch, n = h->n;
    const int64_t P = pitch > 0 ? pitch : (LAY == fs::LAY_CONTIG ? n : M);
    const int nq = h->fplan.nq;
    const int64_t Gb = (M + fs::TW - 1) / fs::TW, G = Gb * count;
    if (G > (1 << 30)) return PB_EUNSUPPORTED;
    const int64_t ntiles = G * nq;
    if (ntiles >= ((int64_t)1 << 31)) return PB_EUNSUPPORTED;
    const size_t es = sizeof(T);
    tp::Args<T> A;
    CUtensorMap tmap;
    std::lock_guard<std::mutex> lk(h->fplan.mu);
    FusedScratch &S = h->fplan.scratch[st];
    // [car][spec][xl]
    const size_t off_car = 0;
    const size_t off_spec = off_car + es * (size_t)ntiles * 4 * fs::TW, off_xl = off_spec + es * (size_t)G * 4 * fs::TW;
    const size_t need = off_xl + es * (size_t)G * 2 * fs::TW;
    if (need > S.tbytes) {
        if (S.tbuf) {
            PB_CUDA_TRY(cudaStreamSynchronize(st));   // queued solves may still use the old scratch
            cudaFree(S.tbuf);
            S.tbuf = nullptr;
            S.tbytes = 0;
        }
        PB_CUDA_TRY(cudaMalloc(&S.tbuf, need));
        S.tbytes = need;
    }
    {
        bool flat = false;
        int rc = tensor_map_for<T, LAY>(S, x, M, n, count, bstride, P, &tmap, &flat);
        if (rc) return rc;
        A.flat = flat ? 1 : 0;
    }
    char *base = (char *)S.tbuf;
    A.rec = (const T *)h->fplan.rec;
    A.coef = (const T *)h->coef;
    A.ct = (const T *)h->fplan.ct;
    A.rsp = (const T *)h->fplan.rsp;
    A.scal = h->scal;
    A.x = x;
    A.car = (T *)(base + off_car);
    A.spec = (T *)(base + off_spec);
    A.xl = (T *)(base + off_xl);
    A.n = n;
    A.M = M;
    A.bstride = count > 1 ? bstride : P * (LAY == fs::LAY_CONTIG ? M : n);
    A.pitch = P;
    A.ntiles = ntiles;
    // the last ~48 MB of f that P1 reads stay in L2 for P2's first (reversed) tiles
    const int64_t keep = (int64_t)(48.0 * 1048576.0 / (double)(fs::Q * fs::TW * es));
    A.keep_from = ntiles > keep ? ntiles - keep : 0;
    for (int j = 0; j < 4; ++j) A.srow[j] = h->srow[j];
    A.nq = nq;
    A.Gb = (int)Gb;
    A.G = (int)G;
    A.BG = (int)G;   // one band: chunk-major order over all groups (contiguous row blocks)
    const unsigned grid = (unsigned)std::min<int64_t>(fs_sm_count(), (ntiles + NC - 1) / NC);
    const unsigned grid2 = (unsigned)std::min<int64_t>(fs_sm_count(), (ntiles + NC2 - 1) / NC2);
    k1<<<grid, 32 * NC, sm1, st>>>(tmap, A);
    PB_LAUNCH_CHECK();
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl[0].val.programmaticStreamSerializationAllowed = 1;
    {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)G);
#ifndef TP_SCAN_WARPS
#define TP_SCAN_WARPS tp::SEGMAX
#endif
        cfg.blockDim = dim3(32 * std::min(TP_SCAN_WARPS, (nq + tp::SL - 1) / tp::SL));
        cfg.dynamicSmemBytes = sms;
        cfg.stream = st;
        cfg.attrs = pdl;
        cfg.numAttrs = 1;
        if (nq <= 8) PB_CUDA_TRY(cudaLaunchKernelEx(&cfg, ks8, A));
        else PB_CUDA_TRY(cudaLaunchKernelEx(&cfg, ks, A));
        PB_LAUNCH_CHECK();
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid2);
    cfg.blockDim = dim3(32 * NC2);
    cfg.dynamicSmemBytes = sm2;
    cfg.stream = st;
    cfg.attrs = pdl;
    cfg.numAttrs = 1;
    PB_CUDA_TRY(cudaLaunchKernelEx(&cfg, k2, tmap, A));
    PB_LAUNCH_CHECK();
#ifdef TP_PROF
    static int nl = 0;
    if (nl++ == 0)
        atexit([] {
            unsigned long long hp[16];
            cudaMemcpyFromSymbol(hp, tp::tp_prof, sizeof(hp));
            fprintf(stderr, "TP_PROF (cycles summed over warps, all launches):");
            for (int i = 0; i < 16; ++i) fprintf(stderr, " %d=%.3g", i, (double)hp[i]);
            fprintf(stderr, "\n");
        });
#endif
    return PB_OK;
}

template <typename T, int K, bool PER, int MODE, int LAY>
static int fs_launch_t(const Band *h, T *x, T *xout, double alpha, int64_t count, int64_t bstride, cudaStream_t st,
                       int64_t Mo, int64_t pitch)
{
    auto kern = fs::fs_kernel<T, K, PER, MODE, LAY>;
    const size_t smem = sizeof(fs::Smem<T>) + 1024;   // + alignment to 1 KB
    static std::once_flag attr_once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(attr_once, [&] {
        attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    if (attr_err != cudaSuccess) return set_error(PB_ECUDA, "fs_kernel smem attribute: %s", cudaGetErrorString(attr_err));

    const int64_t M = Mo > 0 ? Mo : h->batch, n = h->n;
    const int64_t dpitch = LAY == fs::LAY_CONTIG ? n : M;   // the packed pitch
    const int64_t P = pitch > 0 ? pitch : dpitch;
    const int nq = h->fplan.nq;
    const int64_t Gb = (M + fs::TW - 1) / fs::TW, G = Gb * count;
    if (G > INT32_MAX / 2) return set_error(PB_EINVAL, "too many systems for one launch");
    const int64_t nsys = G * fs::TW;
    const int64_t items = 2 * G * nq, nclaims = (items + fs::NC - 1) / fs::NC;
    const size_t es = sizeof(T);
    // scratch: car [nq][nsys][4], spec [nsys][4], xl [nsys][2], cnt [G], flag [G], tick [4]
    // (tick[2] CTAs done, tick[3] launches done)
    const size_t off_spec = es * (size_t)nq * nsys * 4, off_xl = off_spec + es * nsys * 4;
    const size_t off_cnt = (off_xl + es * nsys * 2 + 255) / 256 * 256;
    const size_t off_flag = off_cnt + 4 * (size_t)G, off_tick = off_flag + 4 * (size_t)G;
    const size_t need = off_tick + 16;   // tick[4]

    fs::Args<T> A;
    {
        std::lock_guard<std::mutex> lk(h->fplan.mu);
        FusedScratch &S = h->fplan.scratch[st];
        if (need > S.bytes) {
            if (S.buf) {
                PB_CUDA_TRY(cudaStreamSynchronize(st));   // queued solves may still use the old scratch
                cudaFree(S.buf);
                S.buf = nullptr;
                S.bytes = 0;
            }
            PB_CUDA_TRY(cudaMalloc(&S.buf, need));
            S.bytes = need;
            S.nq = S.nsys = -1;
            memset(S.key, 0, sizeof(S.key));
        }
        char *base = (char *)S.buf;
        if (S.nq != nq || S.nsys != nsys) {
            // fresh scratch or new shape (the counters live at shape-dependent
            // offsets): clear counters, flags and tickets; epochs restart at 1
            PB_CUDA_TRY(cudaMemsetAsync(base + off_cnt, 0, need - off_cnt, st));
            S.nq = nq;
            S.nsys = nsys;
        }
        A.car = (T *)base;
        A.spec = (T *)(base + off_spec);
        A.xl = (T *)(base + off_xl);
        A.cnt = (unsigned *)(base + off_cnt);
        A.flag = (unsigned *)(base + off_flag);
        A.tick = (unsigned *)(base + off_tick);

        // tensor map over x, cached per stream.  Interleaved: dims (M, n, count),
        // box (32 systems, 64 rows, 1); contiguous: dims (n, M, count), box
        // (128 B of rows, 32 systems, 1), 128B swizzle.  OOB loads zero-fill and
        // OOB stores are clipped (ragged M and n).  Contiguous batches that tiles
        // cannot straddle use one 2-D view.
        const bool flat = P == dpitch && (LAY == fs::LAY_CONTIG
                              ? (count == 1 || (bstride == M * n && M % fs::TW == 0))
                              : (count == 1 || (bstride == M * n && n % fs::Q == 0 && n * count < ((int64_t)1 << 31))));
        const uint64_t key[6] = {(uint64_t)(uintptr_t)x, (uint64_t)M, (uint64_t)n, (uint64_t)count,
                                 (uint64_t)bstride, (uint64_t)P * 16 + sizeof(T) * 2 + LAY};
        uint64_t *skey = S.key[LAY];
        void *smap = S.tmap[LAY];
        if (memcmp(key, skey, sizeof(key)) != 0) {
            auto enc = tensor_map_encoder();
            if (!enc) return set_error(PB_ECUDA, "cuTensorMapEncodeTiled unavailable");
            const auto dt = sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
            const int rank = flat ? 2 : 3;
            const int64_t bs = count > 1 ? bstride : P * (LAY == fs::LAY_CONTIG ? M : n);
            CUresult r;
            cuuint32_t estr[3] = {1, 1, 1};
            if (LAY == fs::LAY_CONTIG) {
                cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)(flat ? M * count : M), (cuuint64_t)(flat ? 1 : count)};
                cuuint64_t strides[2] = {(cuuint64_t)(P * sizeof(T)), (cuuint64_t)(bs * sizeof(T))};
                cuuint32_t box[3] = {(cuuint32_t)fs::Sw<T>::EB, (cuuint32_t)fs::TW, 1};
                r = enc((CUtensorMap *)smap, dt, rank, (void *)x, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            } else {
                cuuint64_t dims[3] = {(cuuint64_t)M, (cuuint64_t)(flat ? n * count : n), (cuuint64_t)(flat ? 1 : count)};
                cuuint64_t strides[2] = {(cuuint64_t)(P * sizeof(T)), (cuuint64_t)(bs * sizeof(T))};
                cuuint32_t box[3] = {(cuuint32_t)fs::TW, (cuuint32_t)fs::Q, 1};
                r = enc((CUtensorMap *)smap, dt, rank, (void *)x, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            }
            if (r != CUDA_SUCCESS) return set_error(PB_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
            memcpy(skey, key, sizeof(key));
        }
        A.flat = flat ? 1 : 0;
        CUtensorMap tmap;
        memcpy(&tmap, smap, sizeof(tmap));

        A.rec = (const T *)h->fplan.rec;
        A.coef = (const T *)h->coef;
        A.ct = (const T *)h->fplan.ct;
        A.rsp = (const T *)h->fplan.rsp;
        A.scal = h->scal;
        A.x = x;
        A.xout = xout;
        A.alpha = (T)alpha;
        A.bstride = count > 1 ? bstride : P * (LAY == fs::LAY_CONTIG ? M : n);
        A.pitch = P;
        A.n = n;
        A.M = M;
        A.nsys = nsys;
        A.items = items;
        A.nclaims = nclaims;
        for (int j = 0; j < 4; ++j) A.srow[j] = h->srow[j];
        A.nq = nq;
        A.count = (int)count;
        A.Gb = (int)Gb;
        A.G = (int)G;
        const double gbytes = (double)fs::TW * (double)n * (double)es;
        int64_t D = (int64_t)(FS_L2_BUDGET / gbytes);
        A.D = (int)(D < 1 ? 1 : (D > G ? G : D));
        A.qspec = PER ? (int)(h->srow[0] / fs::Q) : nq;
        const int grid = (int)std::min<int64_t>(fs_sm_count(), nclaims);
        // cooperative: all CTAs co-resident (the static work deal relies on it).
        // Launched under the lock: the scratch (and its cached map) is not
        // re-laid-out between this launch's setup and its enqueue
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)grid);
        cfg.blockDim = dim3(fs::NTHREADS);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        PB_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, tmap, A));
        PB_LAUNCH_CHECK();
    }
    return PB_OK;
}


// the two-pass kernels unless the batch is too small to stream (fewer than
// 32 K systems of N/64 <= 8: one launch instead of three) or, interleaved,
// the held-tile kernel keeps all its warps busy (5 <= N/64 <= 8: 0.58 vs
// 0.70 ms at 512 x 262 144; contiguous 512 x 262 144, the ADI x-sweep, is the
// other way round: cfg4 step 3.16 -> 3.08 ms)
static inline bool use_twopass(int nq, int64_t systems, int lay = fs::LAY_INTER)
{
    if (nq > fh::NW) return true;
    if (nq < 2 || systems < 32768) return false;
    return lay == fs::LAY_CONTIG || nq <= fh::NW / 2;
}

template <typename T, int LAY>
static int fs_launch_dl(const Band *h, void *x, int64_t count, int64_t bstride, cudaStream_t st, int64_t M,
                        int64_t pitch)
{
    T *X = (T *)x;
    using namespace fs;
    int rc;
    // systems longer than one held-tile CTA (8 chunks), either layout: the
    // two-pass kernels (P1 / scan / P2; measured 2.5x faster than the cluster
    // exchange of the held-tile kernel at N = M = 8192)
    // (and for N/64 <= 4 in the bandwidth regime: the held-tile CTA then runs
    // at most half its warps; 2^20 x 256 fp64: 1.52 vs 1.80 ms)
    if (use_twopass(h->fplan.nq, (M > 0 ? M : h->batch) * count, LAY)) {
        if (h->K == 2)
            rc = h->periodic ? tp_launch_t<T, 2, true, LAY>(h, X, count, bstride, st, M, pitch)
                             : tp_launch_t<T, 2, false, LAY>(h, X, count, bstride, st, M, pitch);
        else
            rc = h->periodic ? tp_launch_t<T, 1, true, LAY>(h, X, count, bstride, st, M, pitch)
                             : tp_launch_t<T, 1, false, LAY>(h, X, count, bstride, st, M, pitch);
        if (rc != PB_EUNSUPPORTED) return rc;
    }
    {
        if (h->K == 2)
            rc = h->periodic ? fh_launch_t<T, 2, true, MODE_SOLVE, LAY>(h, X, X, 0.0, count, bstride, st, M, pitch)
                             : fh_launch_t<T, 2, false, MODE_SOLVE, LAY>(h, X, X, 0.0, count, bstride, st, M, pitch);
        else
            rc = h->periodic ? fh_launch_t<T, 1, true, MODE_SOLVE, LAY>(h, X, X, 0.0, count, bstride, st, M, pitch)
                             : fh_launch_t<T, 1, false, MODE_SOLVE, LAY>(h, X, X, 0.0, count, bstride, st, M, pitch);
        if (rc != PB_EUNSUPPORTED) return rc;
    }
    // beyond the two-pass scan's span (N/64 > 512): the global-scan kernel
    if (h->K == 2)
        return h->periodic ? fs_launch_t<T, 2, true, MODE_SOLVE, LAY>(h, X, X, 0.0, count, bstride, st, M, pitch)
                           : fs_launch_t<T, 2, false, MODE_SOLVE, LAY>(h, X, X, 0.0, count, bstride, st, M, pitch);
    return h->periodic ? fs_launch_t<T, 1, true, MODE_SOLVE, LAY>(h, X, X, 0.0, count, bstride, st, M, pitch)
                       : fs_launch_t<T, 1, false, MODE_SOLVE, LAY>(h, X, X, 0.0, count, bstride, st, M, pitch);
}

int FS_NAME(const Band *h, void *x, int64_t count, int64_t bstride, cudaStream_t st, int64_t M, int64_t pitch)
{
    return fs_launch_dl<FS_T, FS_LAY>(h, x, count, bstride, st, M, pitch);
}

// diagnostics: the cluster configuration a solve of M systems x count would use
int FS_INFO_NAME(const Band *h, int64_t M, int64_t count, int *info)
{
    int rc;
    if (use_twopass(h->fplan.nq, M * count, FS_LAY) && h->fplan.nq <= tp::SL * tp::NSEG &&
        (int64_t)h->fplan.nq * ((M + fs::TW - 1) / fs::TW) * count < ((int64_t)1 << 31)) {
        // the two-pass kernels: no clusters; info[2] = CTAs of P1
        const int64_t nt = (int64_t)h->fplan.nq * ((M + fs::TW - 1) / fs::TW) * count;
        info[0] = 0;
        info[1] = 0;
        info[2] = (int)std::min<int64_t>(fs_sm_count(), (nt + TpCfg<FS_T>::NC1 - 1) / TpCfg<FS_T>::NC1);
        info[3] = 3;
        return PB_OK;
    }
    if (h->K == 2)
        rc = h->periodic ? fh_launch_t<FS_T, 2, true, fs::MODE_SOLVE, FS_LAY>(h, nullptr, nullptr, 0.0, count, 0,
                                                                              nullptr, M, 0, info)
                         : fh_launch_t<FS_T, 2, false, fs::MODE_SOLVE, FS_LAY>(h, nullptr, nullptr, 0.0, count, 0,
                                                                               nullptr, M, 0, info);
    else
        rc = h->periodic ? fh_launch_t<FS_T, 1, true, fs::MODE_SOLVE, FS_LAY>(h, nullptr, nullptr, 0.0, count, 0,
                                                                              nullptr, M, 0, info)
                         : fh_launch_t<FS_T, 1, false, fs::MODE_SOLVE, FS_LAY>(h, nullptr, nullptr, 0.0, count, 0,
                                                                               nullptr, M, 0, info);
    if (rc != PB_EUNSUPPORTED) return rc;
    info[0] = info[1] = info[2] = info[3] = 0;   // the global-scan kernel
    return PB_OK;
}

#ifdef FS_CH1D_NAME
int FS_CH1D_NAME(const Band *h, const void *c, void *cnew, double alpha, int64_t M, cudaStream_t st)
{
    int rc = fh_launch_t<FS_T, 2, true, fs::MODE_CH1D, fs::LAY_INTER>(h, (FS_T *)c, (FS_T *)cnew, alpha, 1, 0, st, M, 0);
    if (rc != PB_EUNSUPPORTED) return rc;
    return fs_launch_t<FS_T, 2, true, fs::MODE_CH1D, fs::LAY_INTER>(h, (FS_T *)c, (FS_T *)cnew, alpha, 1, 0, st, M, 0);
}
#endif

}  // namespace pb

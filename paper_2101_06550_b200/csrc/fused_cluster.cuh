// fused_cluster.cuh — what the held-tile kernel (fused_hold.cuh) shares with
// the thread-block-cluster designs of this round: its launch arguments and the
// cluster PTX (DSMEM addresses, remote mbarrier arrives, cluster waits).  (The
// cluster two-pass kernel that lived here measured 787 us at N = M = 8192
// against the two-pass kernels' 320 us and was removed.)
#pragma once
#include <cooperative_groups.h>

#include "fused_solve.cuh"

namespace pb {
namespace fc {

using namespace fs;
namespace cg = cooperative_groups;

template <typename T>
struct CArgs {
    const T *rec, *coef, *ct, *rsp;
    const double *scal;
    T *x, *xout;
    T alpha;                 // MODE_CH1D
    int64_t n, M, bstride, pitch;
    int64_t srow[4];
    int nq, count, Gb, G;
    int cs, cpc, ncl;        // cluster size, chunks per CTA, clusters
    int flat;
    int dbg;   // (unused)
    long long *prof;   // DEV ONLY (FH_PROF builds)
};

// ---------------------------------------------------------------- cluster PTX
__device__ __forceinline__ uint32_t mapa(const void *p, uint32_t rank)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(su32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void arrive_remote(const uint64_t *b, uint32_t rank)
{
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa(b, rank)) : "memory");
}
__device__ __forceinline__ void wait_cluster(uint64_t *b, uint32_t parity)
{
    asm volatile(
        "{\n .reg .pred p;\n"
        "FC_WAITC:\n"
        " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra FC_WAITC;\n}" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void fence_cluster() { asm volatile("fence.acq_rel.cluster;" ::: "memory"); }
template <typename T>
__device__ __forceinline__ T *peer(T *p, int rank)
{
    return cg::this_cluster().map_shared_rank(p, rank);
}

}  // namespace fc
}  // namespace pb

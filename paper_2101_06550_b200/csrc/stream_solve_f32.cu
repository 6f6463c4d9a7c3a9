// stream_solve_f32.cu — fp32 instantiations of the streaming solve.
#include "cluster_launch.cuh"
#include "stream_launch.cuh"

namespace pb {
int launch_stream_f32(const Band *h, void *x, int64_t count, int64_t bstride, cudaStream_t st)
{
    return launch_stream_dt<float>(h, x, count, bstride, st);
}
int stream_max_ctas_f32(int K, int periodic) { return stream_max_ctas_t<float>(K, periodic); }
int launch_clu_f32(const Band *h, void *x, int64_t count, int64_t bstride, cudaStream_t st)
{
    return launch_clu_dt<float>(h, x, count, bstride, st);
}
int clu_max_clusters_f32(int C, int K, int periodic) { return clu_max_clusters<float>(C, K, periodic); }
}  // namespace pb

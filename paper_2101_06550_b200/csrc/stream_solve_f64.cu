// stream_solve_f64.cu — fp64 instantiations of the streaming solve.
#include "cluster_launch.cuh"
#include "stream_launch.cuh"

namespace pb {
int launch_stream_f64(const Band *h, void *x, int64_t count, int64_t bstride, cudaStream_t st)
{
    return launch_stream_dt<double>(h, x, count, bstride, st);
}
int stream_max_ctas_f64(int K, int periodic) { return stream_max_ctas_t<double>(K, periodic); }
int launch_clu_f64(const Band *h, void *x, int64_t count, int64_t bstride, cudaStream_t st)
{
    return launch_clu_dt<double>(h, x, count, bstride, st);
}
int clu_max_clusters_f64(int C, int K, int periodic) { return clu_max_clusters<double>(C, K, periodic); }
}  // namespace pb

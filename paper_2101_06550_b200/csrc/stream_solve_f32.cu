// stream_solve_f32.cu — fp32 instantiations of the streaming solve.
#include "stream_launch.cuh"

namespace pb {
int launch_stream_f32(const Band *h, void *x, int64_t count, int64_t bstride, cudaStream_t st)
{
    return launch_stream_dt<float>(h, x, count, bstride, st);
}
int stream_max_ctas_f32(int K, int periodic) { return stream_max_ctas_t<float>(K, periodic); }
}  // namespace pb

// banded_inst_f32_k2.cu — tile-kernel instantiations (float, penta).
#include "band_tile.cuh"

namespace pb {
int launch_tile_f32_k2(const Band *h, void *x, int layout, int64_t count, int64_t bstride, cudaStream_t st)
{
    float *X = (float *)x;
    switch (h->plan.mr) {
        case 0: return launch_tile_l<float, 2, 32, 256, 8>(h, X, layout, count, bstride, st);
        case 1: return launch_tile_l<float, 2, 32, 256, 16>(h, X, layout, count, bstride, st);
        case 2: return launch_tile_l<float, 2, 32, 256, 32>(h, X, layout, count, bstride, st);
        case 3: return launch_tile_l<float, 2, 32, 256, 64>(h, X, layout, count, bstride, st);
        case 4: return launch_tile_l<float, 2, 32, 512, 64>(h, X, layout, count, bstride, st);
    }
    return set_error(PB_EINVAL, "bad tile cfg");
}
}  // namespace pb

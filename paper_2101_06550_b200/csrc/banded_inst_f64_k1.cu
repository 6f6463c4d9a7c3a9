// banded_inst_f64_k1.cu — tile-kernel instantiations (double, tri).
#include "band_tile.cuh"

namespace pb {
int launch_tile_f64_k1(const Band *h, void *x, int layout, int64_t count, int64_t bstride, cudaStream_t st)
{
    double *X = (double *)x;
    switch (h->plan.mr) {
        case 0: return launch_tile_l<double, 1, 16, 256, 4>(h, X, layout, count, bstride, st);
        case 1: return launch_tile_l<double, 1, 16, 256, 8>(h, X, layout, count, bstride, st);
        case 2: return launch_tile_l<double, 1, 16, 256, 16>(h, X, layout, count, bstride, st);
        case 3: return launch_tile_l<double, 1, 16, 256, 32>(h, X, layout, count, bstride, st);
        case 4: return launch_tile_l<double, 1, 16, 512, 32>(h, X, layout, count, bstride, st);
    }
    return set_error(PB_EINVAL, "bad tile cfg");
}
}  // namespace pb

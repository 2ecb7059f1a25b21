// sweep_2d.cu — instantiations of the sweep kernel for 2D, radius 1
// (one translation unit per family so the library builds in parallel).
#include "sweep_cfg.cuh"

namespace sb {

template <typename T, int SHAPE>
static LaunchFn pick2(int q, int s) {
    if (q == 1 && s == 1) return launch_cfg<Cfg2<T, SHAPE, 1, 1>>;
    if (q == 2 && s == 1) return launch_cfg<Cfg2<T, SHAPE, 2, 1>>;
    if (q == 4 && s == 1) return launch_cfg<Cfg2<T, SHAPE, 4, 1>>;
    if (q == 3 && s == 1) return launch_cfg<Cfg2<T, SHAPE, 3, 1>>;
    if (q == 1 && s == 2) return launch_cfg<Cfg2<T, SHAPE, 1, 2>>;
    if (q == 1 && s == 4) return launch_cfg<Cfg2<T, SHAPE, 1, 4>>;
    if (q == 2 && s == 2) return launch_cfg<Cfg2<T, SHAPE, 2, 2>>;
    return nullptr;
}

LaunchFn pick_2d(int dtype, int shape, int q, int s) {
    if (dtype == STENCIL_F64) return shape == STENCIL_STAR ? pick2<double, STENCIL_STAR>(q, s) : pick2<double, STENCIL_BOX>(q, s);
    return shape == STENCIL_STAR ? pick2<float, STENCIL_STAR>(q, s) : pick2<float, STENCIL_BOX>(q, s);
}

}  // namespace sb

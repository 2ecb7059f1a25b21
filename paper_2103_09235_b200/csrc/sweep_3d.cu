// sweep_3d.cu — instantiations of the sweep kernel for 3D, radius 1.
#include "sweep_cfg.cuh"

namespace sb {

template <typename T, int SHAPE>
static LaunchFn pick3(int q, int s) {
    if (q == 1 && s == 1) return launch_cfg<Cfg3<T, SHAPE, 1, 1>>;
    if (q == 2 && s == 1) return launch_cfg<Cfg3<T, SHAPE, 2, 1>>;
    if (q == 1 && s == 2) return launch_cfg<Cfg3<T, SHAPE, 1, 2>>;
    return nullptr;
}

LaunchFn pick_3d(int dtype, int shape, int q, int s) {
    if (dtype == STENCIL_F64) return shape == STENCIL_STAR ? pick3<double, STENCIL_STAR>(q, s) : pick3<double, STENCIL_BOX>(q, s);
    return shape == STENCIL_STAR ? pick3<float, STENCIL_STAR>(q, s) : pick3<float, STENCIL_BOX>(q, s);
}

}  // namespace sb

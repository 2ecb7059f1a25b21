// sweep_r2.cu — radius-2 (higher-order) stencils in 2D and 3D (SURVEY §8(f)
// NEXT-4): the same kernel template with RR = 2.  Compiled evaluations:
//   2D star/box: one pass of lambda^(1) or lambda^(2), or 2 on-chip single steps;
//   3D star: lambda^(1), lambda^(2) or 2 on-chip single steps; 3D box: lambda^(1).
#include "sweep_cfg.cuh"

namespace sb {

template <typename T, int SHAPE>
static LaunchFn pick2r2(int q, int s) {
    if (q == 1 && s == 1) return launch_cfg<Cfg2<T, SHAPE, 1, 1, 2>>;
    if (q == 2 && s == 1) return launch_cfg<Cfg2<T, SHAPE, 2, 1, 2>>;
    if (q == 1 && s == 2) return launch_cfg<Cfg2<T, SHAPE, 1, 2, 2>>;
    return nullptr;
}
template <typename T, int SHAPE>
static LaunchFn pick3r2(int q, int s) {
    if (q == 1 && s == 1) return launch_cfg<Cfg3<T, SHAPE, 1, 1, 2>>;
    if constexpr (SHAPE == STENCIL_STAR) {
        if (q == 2 && s == 1) return launch_cfg<Cfg3<T, SHAPE, 2, 1, 2>>;
        if (q == 1 && s == 2) return launch_cfg<Cfg3<T, SHAPE, 1, 2, 2>>;
    }
    return nullptr;
}

LaunchFn pick_r2(int dtype, int nd, int shape, int q, int s) {
    if (nd == 2) {
        if (dtype == STENCIL_F64) return shape == STENCIL_STAR ? pick2r2<double, STENCIL_STAR>(q, s) : pick2r2<double, STENCIL_BOX>(q, s);
        return shape == STENCIL_STAR ? pick2r2<float, STENCIL_STAR>(q, s) : pick2r2<float, STENCIL_BOX>(q, s);
    }
    if (dtype == STENCIL_F64) return shape == STENCIL_STAR ? pick3r2<double, STENCIL_STAR>(q, s) : pick3r2<double, STENCIL_BOX>(q, s);
    return shape == STENCIL_STAR ? pick3r2<float, STENCIL_STAR>(q, s) : pick3r2<float, STENCIL_BOX>(q, s);
}

}  // namespace sb

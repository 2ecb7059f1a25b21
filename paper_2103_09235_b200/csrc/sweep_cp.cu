// sweep_cp.cu — the 2D counterpart passes: lambda^(q)
// evaluated through `rank` counterparts (vertical/horizontal folding Eq.4-6,
// counterpart reuse Eq.7), q in {2, 4}, rank in {1, 2}.
#include "sweep_cfg.cuh"

namespace sb {

template <typename T>
static LaunchFn pickcp(int q, int rank) {
    if (q == 2 && rank == 1) return launch_cfg<Cfg2CP<T, 2, 1>>;
    if (q == 2 && rank == 2) return launch_cfg<Cfg2CP<T, 2, 2>>;
    if (q == 4 && rank == 1) return launch_cfg<Cfg2CP<T, 4, 1>>;
    if (q == 4 && rank == 2) return launch_cfg<Cfg2CP<T, 4, 2>>;
    return nullptr;
}

LaunchFn pick_cp(int dtype, int q, int rank) {
    return dtype == STENCIL_F64 ? pickcp<double>(q, rank) : pickcp<float>(q, rank);
}

}  // namespace sb

// tb3d_f64.cu — fp64 instantiations of the 3D temporal block (tb3d.cuh):
// radius-1 STAR, K = fold_m = 2..4 steps per HBM round trip, 64 x 32 tiles
// (8 warps of 4 rows, 2 doubles per lane and row).
#include "tb3d.cuh"

namespace sb {

#ifndef TB3_NWY
#define TB3_NWY 8
#endif
#ifndef TB3_VY
#define TB3_VY 4
#endif

Tb3LaunchFn pick_tb3d_f64(int shape, int K) {
    if (shape == STENCIL_BOX) {   // 3D27P: FMA-bound, K = 2 (K = 3 loses more to the halo than it saves)
        if (K == 2) return tb3d_launch<double, 2, TB3_NWY, TB3_VY, true>;
        return nullptr;
    }
    if (shape != STENCIL_STAR) return nullptr;
    switch (K) {
        case 2: return tb3d_launch<double, 2, TB3_NWY, TB3_VY>;
        case 3: return tb3d_launch<double, 3, TB3_NWY, TB3_VY>;
        case 4: return tb3d_launch<double, 4, TB3_NWY, TB3_VY>;
        default: return nullptr;
    }
}

}  // namespace sb

// tb3d_f64.cu — fp64 instantiations of the 3D temporal block (tb3d.cuh):
// radius-1 STAR, K = fold_m = 2..4 steps per HBM round trip, 64 x 32 tiles
// (8 warps of 4 rows, 2 doubles per lane and row); radius-1 BOX (3D27P), K = 2,
// 64 x 56 tiles (8 warps of 7 rows).
#include "tb3d.cuh"

namespace sb {

#ifndef TB3_NWY
#define TB3_NWY 8
#endif
#ifndef TB3_VY
#define TB3_VY 4
#endif

#ifndef TB3_BOX_NWY
#define TB3_BOX_NWY TB3_NWY
#endif
#ifndef TB3_BOX_VY
// 56 x 64 tiles for the FMA-bound box (52 x 60 outputs at K = 2), 236 registers, no spill;
// measured on C5 (GStencil/s): VY = 4 / 5 / 6 / 7 / 8 -> 347 / 350 / 366 / 378 / 365 (8 spills),
// 12 warps x 4 rows 357, 12 x 3 332, 16 x 2 348
#define TB3_BOX_VY 7
#endif

Tb3LaunchFn pick_tb3d_f64(int shape, int K) {
    if (shape == STENCIL_BOX) {   // 3D27P: FMA-bound, K = 2 (K = 3 loses more to the halo than it saves)
        if (K == 2) return tb3d_launch<double, 2, TB3_BOX_NWY, TB3_BOX_VY, true>;
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

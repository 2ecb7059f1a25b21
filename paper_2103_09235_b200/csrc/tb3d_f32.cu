// tb3d_f32.cu — fp32 instantiations of the 3D temporal block (tb3d.cuh):
// radius-1 STAR, K = fold_m = 2..4 steps per HBM round trip, 128 x 32 tiles
// (8 warps of 4 rows, 4 floats per lane and row); radius-1 BOX (3D27P), K = 2,
// 128 x 48 tiles.  Measured on 512^3 fp32 stars (GStencil/s): K = 2 / 3 / 4 -> 865 / 905 /
// 983; one folded pass of lambda^(2): 940, m = 1: 612.
#include "tb3d.cuh"

namespace sb {

#ifndef TB3_F32_VY
#define TB3_F32_VY 4
#endif
#ifndef TB3_F32_BOX_VY
// measured on 768 x 768 x 384 fp32 (GStencil/s): 4 / 5 / 6 rows per warp -> 566 / 514 / 586
// (247 registers, no spill); one pass per step (m = 1) runs 659-666, so fold_m = 0 keeps 1
#define TB3_F32_BOX_VY 6
#endif

Tb3LaunchFn pick_tb3d_f32(int shape, int K) {
    if (shape == STENCIL_BOX) {
        if (K == 2) return tb3d_launch<float, 2, 8, TB3_F32_BOX_VY, true>;
        return nullptr;
    }
    if (shape != STENCIL_STAR) return nullptr;
    switch (K) {
        case 2: return tb3d_launch<float, 2, 8, TB3_F32_VY>;
        case 3: return tb3d_launch<float, 3, 8, TB3_F32_VY>;
        case 4: return tb3d_launch<float, 4, 8, TB3_F32_VY>;
        default: return nullptr;
    }
}

}  // namespace sb

// tb2d_f32.cu — fp32 instantiations of the 2D temporal block (tb2d.cuh):
// STAR / BOX, K = fold_m = 2..8 steps per HBM round trip, 8 columns per lane.
#include "tb2d.cuh"

namespace sb {

#ifndef TB_F32_VX
#define TB_F32_VX 8
#endif
#ifndef TB_NW
#define TB_NW 8
#endif

template <int SHAPE, int... Ks>
static TbLaunchFn pick_k(int K, std::integer_sequence<int, Ks...>) {
    TbLaunchFn fn = nullptr;
    ((K == Ks + 2 ? (fn = tb2d_launch<float, SHAPE, Ks + 2, TB_F32_VX, TB_NW>, 0) : 0), ...);
    return fn;
}

TbLaunchFn pick_tb2d_f32(int shape, int K) {
    if (shape == STENCIL_STAR) return pick_k<STENCIL_STAR>(K, std::make_integer_sequence<int, 7>{});
    return pick_k<STENCIL_BOX>(K, std::make_integer_sequence<int, 7>{});
}

}  // namespace sb

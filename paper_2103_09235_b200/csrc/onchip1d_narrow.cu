// onchip1d_narrow.cu — 1D kernels with V = 8 and 16 cells per lane.
#include "onchip1d.cuh"

namespace sb {

template <typename T>
K1Fn<T> k1_pick_narrow(int V, int r, int m, bool wrap) {
    if (wrap) return k1_pick_v<T, 16, true>(r, m);
    return V == 8 ? k1_pick_v<T, 8, false>(r, m) : k1_pick_v<T, 16, false>(r, m);
}
template K1Fn<double> k1_pick_narrow<double>(int, int, int, bool);
template K1Fn<float> k1_pick_narrow<float>(int, int, int, bool);

}  // namespace sb

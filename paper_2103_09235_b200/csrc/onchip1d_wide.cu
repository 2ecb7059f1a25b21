// onchip1d_wide.cu — 1D kernels with V = 32 cells per lane (fold radius m*r > 16).
#include "onchip1d.cuh"

namespace sb {

template <typename T>
K1Fn<T> k1_pick_wide(int r, int m, bool wrap) {
    return wrap ? k1_pick_v<T, 32, true>(r, m) : k1_pick_v<T, 32, false>(r, m);
}
template K1Fn<double> k1_pick_wide<double>(int, int, bool);
template K1Fn<float> k1_pick_wide<float>(int, int, bool);

}  // namespace sb

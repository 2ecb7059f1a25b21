// tb2d_f64.cu — fp64 instantiations of the 2D temporal block (tb2d.cuh):
// STAR / BOX, K = fold_m = 2..8 steps per HBM round trip, 4 columns per lane.
#include "tb2d.cuh"

namespace sb {

PFN_cuTensorMapEncodeTiled_v12000 tb_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    });
    return fn;
}

#ifdef TB_PROBE
}  // namespace sb
extern "C" int stencil_debug_tb_probe(unsigned long long* host, int n, int reset) {
    cudaDeviceSynchronize();
    cudaError_t e = cudaMemcpyFromSymbol(host, sb::tb_probe_buf, sizeof(unsigned long long) * 4 * (size_t)n);
    if (reset) {
        static unsigned long long zero[4 * 8192] = {};
        cudaMemcpyToSymbol(sb::tb_probe_buf, zero, sizeof(zero));
    }
    return e == cudaSuccess ? 0 : -3;
}
namespace sb {
#endif

#ifndef TB_F64_VX
#define TB_F64_VX 4
#endif
#ifndef TB_F64_VX6
#define TB_F64_VX6 4       // doubles per lane for blocks of K <= 6 steps (6: measured slower)
#endif
constexpr int tb_vx64(int K) { return K <= 6 ? TB_F64_VX6 : TB_F64_VX; }
#ifndef TB_NW
#define TB_NW 8
#endif
#ifndef TB_NW_AUTO
#define TB_NW_AUTO 0
#endif
// resident one-warp CTAs per SM for a block of K steps: 8 (TB_NW), or with
// TB_NW_AUTO the register file's limit for K's register count (measured, one
// call: 12 warps at K <= 5, 10 at K = 6 -- which the per-SMSP register file
// caps at 168 registers, 3 warps per sub-partition -- run C2 K=4/5/6 at
// 1196/1530/1670 vs 1312/1780/1947 GStencil/s with 8; C3 K=4 2528 vs 2462,
// K=6 2129 vs 2520: kept at 8)
constexpr int tb_nw(int K) { return TB_NW_AUTO ? (K <= 5 ? 12 : K == 6 ? 10 : K == 7 ? 9 : 8) : TB_NW; }

template <int SHAPE, int... Ks>
static TbLaunchFn pick_k(int K, std::integer_sequence<int, Ks...>) {
    TbLaunchFn fn = nullptr;
    ((K == Ks + 2 ? (fn = tb2d_launch<double, SHAPE, Ks + 2, tb_vx64(Ks + 2), tb_nw(Ks + 2)>, 0) : 0), ...);
    return fn;
}

TbLaunchFn pick_tb2d_f64(int shape, int K) {
    if (shape == STENCIL_STAR) return pick_k<STENCIL_STAR>(K, std::make_integer_sequence<int, 7>{});
    return pick_k<STENCIL_BOX>(K, std::make_integer_sequence<int, 7>{});
}

}  // namespace sb

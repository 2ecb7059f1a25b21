// onchip1d.cuh — K-G4, the 1D on-chip multi-step kernel template and its
// dispatch tables (instantiated in onchip1d_narrow.cu (V = 8, 16) and
// onchip1d_wide.cu (V = 32) so the library builds in parallel).
#pragma once
#include <cuda_runtime.h>

#include <utility>

#include "internal.hpp"
#include "sweep_params.cuh"

namespace sb {

// ============================================================== K-G4 1D
// 1D: the whole grid (0.8 MB for the 1D3P config) is far below L2 and one sweep
// is shorter than a launch, so TB time steps run inside one launch.  Every
// WARP is its own overlapped tile (no shared memory, no barriers): lane l
// holds the V consecutive cells [ilo + l*V, ilo + l*V + V) of the warp's
// window in registers, the 2*R neighbours it needs from lanes l-1 / l+1 come
// through warp shuffles, and the window shrinks by R per step (its 32*V - 2H
// middle cells, H = TB*r, are exact after TB steps and are the ones stored).
// The warp applies TB/m folded steps (lambda^(m), radius RF = m*r, Eq.2) and
// then TB mod m single steps (radius RS = r).  Warps whose window comes within
// (m-1)*r of a FIXED face apply single steps throughout, with the ring cells
// frozen at u0 (exact band, R2).  Thread 0..31 of block 0 also copy
// the non-interior cells (ring + pads) src -> dst, so a launch is the whole
// sweep (no separate ring-copy launch).
constexpr int K1_THREADS = 128;
constexpr int K1_MAXC = 2 * 32 + 1;

template <typename T>
struct Params1D {
    const T* src;
    T* dst;
    long long origin, ext;
    int n, r, m, TB, B, nwarps, force_step, wrap;
    T lam[K1_MAXC];   // lambda^(m), index o + m r
    T w[9];           // original taps, index o + r
};

// One step of radius R on the lane's V cells a -> b (neighbours by shuffle).
// FROZEN: cells whose bit is set in `frozen` keep their value (ring cells).
template <typename T, int V, int R, bool FROZEN>
__device__ __forceinline__ void step1d(const T (&a)[V], T (&b)[V], const T (&c)[2 * R + 1], unsigned frozen) {
    static_assert(R <= V, "neighbours must come from the adjacent lane");
    T lft[R], rgt[R];
#pragma unroll
    for (int j = 0; j < R; ++j) {
        lft[j] = __shfl_up_sync(0xffffffffu, a[V - R + j], 1);   // cell l*V - R + j
        rgt[j] = __shfl_down_sync(0xffffffffu, a[j], 1);         // cell l*V + V + j
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
        T acc = T(0);
#pragma unroll
        for (int o = -R; o <= R; ++o) {
            const int i = v + o;
            const T x = i < 0 ? lft[i + R] : (i >= V ? rgt[i - V] : a[i]);
            acc = fma(c[o + R], x, acc);
        }
        b[v] = (FROZEN && ((frozen >> v) & 1u)) ? a[v] : acc;
    }
}

template <typename T, int V, int R, bool FROZEN>
__device__ __forceinline__ void steps1d(T (&a)[V], T (&b)[V], const T* __restrict__ cp, int n, unsigned frozen) {
    T c[2 * R + 1];   // coefficients in registers for the whole time loop
#pragma unroll
    for (int j = 0; j <= 2 * R; ++j) c[j] = cp[j];
#pragma unroll 1
    for (int s = 0; s + 1 < n; s += 2) {
        step1d<T, V, R, FROZEN>(a, b, c, frozen);
        step1d<T, V, R, FROZEN>(b, a, c, frozen);
    }
    if (n & 1) {
        step1d<T, V, R, FROZEN>(a, b, c, frozen);
#pragma unroll
        for (int v = 0; v < V; ++v) a[v] = b[v];
    }
}

template <typename T, int V, int RF, int RS, bool WRAP>
__global__ void __launch_bounds__(K1_THREADS) onchip1d_kernel(const __grid_constant__ Params1D<T> p) {
    if (blockIdx.x == 0 && threadIdx.x < 32) {   // ring + pads (never written by the steps)
        for (long long g = threadIdx.x; g < p.origin; g += 32) p.dst[g] = p.src[g];
        for (long long g = p.origin + p.n + threadIdx.x; g < p.ext; g += 32) p.dst[g] = p.src[g];
    }
    const int gw = blockIdx.x * (K1_THREADS / 32) + (threadIdx.x >> 5);
    if (gw >= p.nwarps) return;   // whole warp
    const int lane = threadIdx.x & 31;
    const int H = p.TB * p.r;
    const int x0 = gw * p.B;                 // first output of this warp
    const int x1 = min(x0 + p.B, p.n);
    const int ilo = x0 - H;                  // first cell of the window
    const int c0 = ilo + lane * V;           // first cell of this lane
    T a[V], b[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
        int x = c0 + v;
        if constexpr (WRAP) {   // PERIODIC: the window wraps around the interior
            x %= p.n;
            x = x < 0 ? x + p.n : x;
        }
        const long long g = p.origin + x;
        a[v] = (WRAP || (g >= 0 && g < p.ext)) ? p.src[g] : T(0);
    }
    const int band = WRAP ? 0 : (p.m - 1) * p.r;
    const bool stepwise = p.force_step || (!WRAP && (ilo < band || x1 + H > p.n - band));
    if (!stepwise) {
        steps1d<T, V, RF, false>(a, b, p.lam, p.TB / p.m, 0u);
        steps1d<T, V, RS, false>(a, b, p.w, p.TB % p.m, 0u);
    } else {
        unsigned frozen = 0;   // cells outside the interior keep u0 (ring; beyond it: never read by valid cells)
#pragma unroll
        for (int v = 0; v < V; ++v)
            if (!WRAP && (c0 + v < 0 || c0 + v >= p.n)) frozen |= 1u << v;
        steps1d<T, V, RS, true>(a, b, p.w, p.TB, frozen);
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
        const int x = c0 + v;
        if (x >= x0 && x < x1) p.dst[p.origin + x] = a[v];
    }
}

template <typename T>
using K1Fn = void (*)(Params1D<T>);

// dispatch table over (V in {8, 16, 32}, RS = r in 1..4, m in 1..8); V >= m*r.
// Compiled: V = 16 for RF <= 16 (V = 8 as well for RF <= 8 without WRAP), V = 32
// only for RF > 16 (the library picks the smallest V holding the fold radius).
template <typename T, int V, int RS, int M, bool WRAP>
constexpr K1Fn<T> k1_entry() {
    constexpr int RF = RS * M;
    constexpr bool want = V == 8 ? (RF <= 8 && !WRAP) : V == 16 ? RF <= 16 : RF > 16;
    if constexpr (want) return onchip1d_kernel<T, V, RF, RS, WRAP>;
    else return nullptr;
}
template <typename T, int V, int RS, bool WRAP, int... Ms>
constexpr void k1_row(K1Fn<T>* row, std::integer_sequence<int, Ms...>) {
    ((row[Ms] = k1_entry<T, V, RS, Ms + 1, WRAP>()), ...);
}
template <typename T, int V, bool WRAP>
K1Fn<T> k1_pick_v(int r, int m) {
    static K1Fn<T> tab[4][8] = {};
    static bool init = false;
    if (!init) {
        k1_row<T, V, 1, WRAP>(tab[0], std::make_integer_sequence<int, 8>{});
        k1_row<T, V, 2, WRAP>(tab[1], std::make_integer_sequence<int, 8>{});
        k1_row<T, V, 3, WRAP>(tab[2], std::make_integer_sequence<int, 8>{});
        k1_row<T, V, 4, WRAP>(tab[3], std::make_integer_sequence<int, 8>{});
        init = true;
    }
    if (r < 1 || r > 4 || m < 1 || m > 8) return nullptr;
    return tab[r - 1][m - 1];
}

// V in {8, 16} (onchip1d_narrow.cu) / V = 32 (onchip1d_wide.cu)
template <typename T>
K1Fn<T> k1_pick_narrow(int V, int r, int m, bool wrap);
template <typename T>
K1Fn<T> k1_pick_wide(int r, int m, bool wrap);

}  // namespace sb

// tb2d.cuh — on-chip multi-step temporal blocking of the 2D radius-1 sweep
// ("achieve multiple time steps computation in
// registers over the tiles efficiently without reloading", §3.4;
// "time loop fusion").  One launch applies K single steps of
// the original taps (K = fold_m = stages) per HBM round trip, exactly up to
// the FIXED faces.
//
// B200 mapping:
//  * Every WARP is an independent overlapped tile: a strip of W = 32*VX
//    columns (lane l owns VX consecutive columns) streamed along axis 0 over
//    a segment of rows.  After K steps the valid outputs are the middle
//    W - 2K columns; neighbouring strips overlap by 2K loaded columns.
//  * Rows arrive by TMA (cp.async.bulk.tensor.2d, one row per transaction,
//    issued by lane 0 PF rows ahead) into a per-warp ring of TB_D shared
//    slots, each with its own mbarrier (complete_tx).  No CTA-wide barrier
//    and no producer warp: the warp is its own producer.
//  * The K time levels form a register pipeline in "push" form (the GPU
//    reading of the paper's vertical folding, Eq.4): when a row of
//    level s-1 arrives at stage s it completes level-s row i-1 with ONE
//    multiply-add per tap row (a[s] + w_S v), seeds row i (b[s] + row-mid(v))
//    and row i+1 (w_N v).  So each stage keeps two partial rows (a, b) in
//    registers, a completed row is handed to the next stage without leaving
//    the register file, and the dependent chain per stage is one FMA (star) or
//    three (box).  The only data movement between lanes is the two x
//    neighbours of every row (warp shuffles).
//  * Frozen ring (R1): levels >= 1 of the ring rows -1 / ny and of
//    the ring columns -1 / nx are re-read from the shared slot of that row
//    (u0 never changes), so the block is exact up to the faces: no band.
//    Only the first/last K rows of a segment ("checked" iterations) and the
//    two edge strips pay for these tests.
//  * Work: units = strips x row segments, taken by warps in a grid-stride
//    order that puts neighbouring strips of one segment on concurrent warps
//    (their shared columns meet in L2).  A static schedule: launches are
//    CUDA-graph safe.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "internal.hpp"
#include "ptx.cuh"

namespace sb {

template <typename T>
struct TbParams {
    const T* src;
    T* dst;
    long long pitch;            // elements per row (stride of axis 0)
    long long org_y, org_x;     // allocation index of interior (0, 0)
    int ny, nx;                 // local interior extents
    int ext_y;                  // allocated rows (TMA rows are clamped into [0, ext_y))
    int phys_lo, phys_hi;       // axis-0 faces are physical: frozen ring rows -1 / ny
    int y_lo, y_hi;             // output rows of this launch
    int nstrips, seglen, units;
    int units_int, seglen_e;    // interior units (strips 1..nstrips-2), edge segment length
    int x0_right;               // window start of the last strip
    // fused halo exchange (NEXT-2), as SweepParams: outputs of rows j < peer_h
    // (j >= ny - peer_h) are stored again at the same address + peer_dlo (+ peer_dhi) bytes
    long long peer_dlo, peer_dhi;
    int peer_h, peer_lo_on, peer_hi_on;
    T w[9];                     // lambda^(1) as the dense 3x3 table, index (dy+1)*3 + (dx+1)
};

constexpr int TB_D = 16;   // shared row slots per warp (power of two)
#ifndef TB_FFMA2
#define TB_FFMA2 0         // fp32 element pairs with packed FFMA2: measured slower
#endif
#ifndef TB_ISSUE_LATE
#define TB_ISSUE_LATE -1   // issue the next rows' TMA after the stages (-1: for fp64)
#endif
#ifndef TB_NB
#define TB_NB 1            // steady-state TMA rows per issue sequence
#endif
#ifndef TB_LOAD_AHEAD
#define TB_LOAD_AHEAD -1   // read row t+1 from its slot after computing row t (-1: for K = 8)
#endif

template <typename T, int SHAPE, int K, int VX, int NW>
struct TbCfg {
    static constexpr int W = 32 * VX;                 // loaded columns per strip
    static constexpr int EV = 16 / (int)sizeof(T);    // elements per 16-byte vector
    static constexpr int KA = (K + EV - 1) / EV * EV; // left/right halo, rounded up so every
                                                      // strip starts 16-byte aligned (vector stores)
    static constexpr int WO = W - 2 * KA;             // output columns per strip
    static constexpr int D = TB_D;
#ifndef TB_G
#define TB_G 2
#endif
    static constexpr int G = (K % TB_G == 0 && K >= TB_G) ? TB_G : 1;   // stage groups (skew)
    static constexpr int LAG = K + G - 1;                      // rows between load and final output
    static constexpr int PF = (D - LAG - 1) < 8 ? (D - LAG - 1) : 8;   // rows in flight ahead
    static constexpr int ROW_BYTES = W * (int)sizeof(T);
    static constexpr int SMEM = D * ROW_BYTES + D * 8;   // one warp per CTA
    static constexpr int NTAP = 9;   // dense 3x3 (a star uses 5 entries)
    // register element: fp32 pairs (packed FFMA2 on sm_100) or one scalar
    static constexpr bool FP2 = sizeof(T) == 4 && TB_FFMA2;
    using E = std::conditional_t<FP2, float2, T>;
    static constexpr int NE = FP2 ? VX / 2 : VX;   // elements per lane
    // load-ahead (measured, one call: C2 K=8 1909 vs 1864, C3 K=8 2754 vs 2697,
    // C2 K=6 1858 vs 1882 GStencil/s): on for the deepest block only
    static constexpr bool LA = TB_LOAD_AHEAD < 0 ? K >= 8 : TB_LOAD_AHEAD != 0;
    // late issue (measured, one call: C2 K=8 1960 vs 1917, K=6 1959 vs 1879;
    // C3 f32 K=8 2660 vs 2755 GStencil/s): fp64 only
    static constexpr bool IL = TB_ISSUE_LATE < 0 ? sizeof(T) == 8 : TB_ISSUE_LATE != 0;
    static constexpr int NB = TB_NB;
    static_assert(K >= 1 && PF >= 2, "temporal block too deep for the slot ring");
    static_assert(W <= 256, "TMA box dimension");
    static_assert((VX * sizeof(T)) % 16 == 0, "16-byte lane vectors");
};

template <int VX, typename T>
__device__ __forceinline__ void tb_lds(T (&v)[VX], const T* s) {
    constexpr int NV = VX * (int)sizeof(T) / 16;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        if constexpr (sizeof(T) == 8) {
            const double2 x = reinterpret_cast<const double2*>(s)[q];
            v[2 * q] = x.x;
            v[2 * q + 1] = x.y;
        } else {
            const float4 x = reinterpret_cast<const float4*>(s)[q];
            v[4 * q] = x.x;
            v[4 * q + 1] = x.y;
            v[4 * q + 2] = x.z;
            v[4 * q + 3] = x.w;
        }
    }
}

// Non-edge units: every 16-byte vector of a lane is either fully stored or not
// (aligned output range), so each is one predicated vector store, no branch.
template <int VX, typename T>
__device__ __forceinline__ void tb_stg_aligned(T* g, const T (&v)[VX], unsigned mask) {
    constexpr int EV = 16 / (int)sizeof(T);
#pragma unroll
    for (int q = 0; q < VX / EV; ++q) {
        const bool on = (mask >> (q * EV)) & 1u;
        if constexpr (sizeof(T) == 8)
            ptx::stg_v2_pred(on, reinterpret_cast<double*>(g) + 2 * q, v[2 * q], v[2 * q + 1]);
        else
            ptx::stg_v4_pred(on, reinterpret_cast<float*>(g) + 4 * q, v[4 * q], v[4 * q + 1], v[4 * q + 2],
                             v[4 * q + 3]);
    }
}

template <int VX, typename T>
__device__ __forceinline__ void tb_stg(T* g, const T (&v)[VX], unsigned mask) {
    constexpr int EV = 16 / (int)sizeof(T);   // elements per 16-byte vector
    constexpr unsigned FULL = (1u << EV) - 1u;
#pragma unroll
    for (int q = 0; q < VX / EV; ++q) {
        const unsigned mq = (mask >> (q * EV)) & FULL;
        if (mq == FULL) {
            if constexpr (sizeof(T) == 8)
                reinterpret_cast<double2*>(g)[q] = make_double2(v[2 * q], v[2 * q + 1]);
            else
                reinterpret_cast<float4*>(g)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        } else if (mq) {
#pragma unroll
            for (int e = 0; e < EV; ++e)
                if (mq & (1u << e)) g[q * EV + e] = v[q * EV + e];
        }
    }
}

// fp32 element pairs: the lane's VX floats (columns c .. c+VX-1) are held as
// VX/2 float2 pairs P[q] = (column c+q, column c+q+VX/2).  Then the west
// neighbour pair of P[q] is P[q-1] and the east one P[q+1]: only the two end
// pairs are assembled from shuffled values, so packed FFMA2 needs almost no
// register moves.
template <int NE>
__device__ __forceinline__ void tb_lds(float2 (&v)[NE], const float* s) {
    static_assert(NE % 4 == 0, "fp32 pairs: VX multiple of 8");
#pragma unroll
    for (int q = 0; q < NE; q += 4) {
        const float4 lo = reinterpret_cast<const float4*>(s)[q / 4];
        const float4 hi = reinterpret_cast<const float4*>(s + NE)[q / 4];
        v[q] = make_float2(lo.x, hi.x);
        v[q + 1] = make_float2(lo.y, hi.y);
        v[q + 2] = make_float2(lo.z, hi.z);
        v[q + 3] = make_float2(lo.w, hi.w);
    }
}

template <int NE>
__device__ __forceinline__ void tb_stg(float* g, const float2 (&v)[NE], unsigned mask) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int q = 0; q < NE; q += 4) {
            const int e0 = h * NE + q;   // first column of this 16-byte vector
            const unsigned mq = (mask >> e0) & 15u;
            const float f0 = h ? v[q].y : v[q].x, f1 = h ? v[q + 1].y : v[q + 1].x;
            const float f2 = h ? v[q + 2].y : v[q + 2].x, f3 = h ? v[q + 3].y : v[q + 3].x;
            if (mq == 15u) {
                reinterpret_cast<float4*>(g + e0)[0] = make_float4(f0, f1, f2, f3);
            } else if (mq) {
                const float f[4] = {f0, f1, f2, f3};
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (mq & (1u << e)) g[e0 + e] = f[e];
            }
        }
    }
}

template <typename T, int SHAPE, int K, int VX, int NW>
struct TbWarp {
    using C = TbCfg<T, SHAPE, K, VX, NW>;
    const CUtensorMap* tmap;
    const TbParams<T>* p;
    T* ring;          // this warp's slots
    uint64_t* bar;    // this warp's barriers
    int lane;
    uint32_t fill;    // rows issued so far (slot = fill % D, parity = fill / D % 2)

    // One stage: input row v (level s), state (a, b), output o = level s+1 of
    // row j (frozen ring cells keep u0, re-read from the row's shared slot).
    using E = typename C::E;
    static constexpr int NE = C::NE;

    template <bool CHK, bool EDGE>
    __device__ __forceinline__ void stage(const T (&w)[C::NTAP], E (&a)[NE], E (&b)[NE], const E (&v)[NE], E (&o)[NE],
                                          int j, int sl, unsigned rmask) const {
        if constexpr (C::FP2) {
            // fp32 pairs P[q] = (column q, column q + NE): west neighbour pair P[q-1],
            // east P[q+1]; the end pairs take the lane neighbours' end columns
            const float vl = __shfl_up_sync(0xffffffffu, v[NE - 1].y, 1);   // column -1
            const float vr = __shfl_down_sync(0xffffffffu, v[0].x, 1);      // column VX
            const float2 Wst = make_float2(vl, v[NE - 1].x);                  // west of P[0]
            const float2 Est = make_float2(v[0].y, vr);                       // east of P[NE-1]
            auto W2 = [&](int k) { return make_float2(w[k], w[k]); };
#pragma unroll
            for (int q = 0; q < NE; ++q) {
                const float2 L = q == 0 ? Wst : v[q - 1];
                const float2 R = q == NE - 1 ? Est : v[q + 1];
                if constexpr (SHAPE == STENCIL_STAR) {
                    o[q] = __ffma2_rn(W2(7), v[q], a[q]);
                    a[q] = __ffma2_rn(W2(5), R, __ffma2_rn(W2(3), L, __ffma2_rn(W2(4), v[q], b[q])));
                    b[q] = __fmul2_rn(W2(1), v[q]);
                } else {
                    o[q] = __ffma2_rn(W2(8), R, __ffma2_rn(W2(6), L, __ffma2_rn(W2(7), v[q], a[q])));
                    a[q] = __ffma2_rn(W2(5), R, __ffma2_rn(W2(3), L, __ffma2_rn(W2(4), v[q], b[q])));
                    b[q] = __ffma2_rn(W2(2), R, __ffma2_rn(W2(0), L, __fmul2_rn(W2(1), v[q])));
                }
            }
        } else {
            const T vl = __shfl_up_sync(0xffffffffu, v[VX - 1], 1);
            const T vr = __shfl_down_sync(0xffffffffu, v[0], 1);
#pragma unroll
            for (int e = 0; e < VX; ++e) {
                const T L = e == 0 ? vl : v[e - 1];
                const T R = e == VX - 1 ? vr : v[e + 1];
                // (terms in v first, the shuffled neighbours L, R last: the
                // shuffle latency overlaps the first multiply-add)
                if constexpr (SHAPE == STENCIL_STAR) {
                    // lambda^(1) dense 3x3, index (dy+1)*3 + (dx+1): N 1, W 3, C 4, E 5, S 7
                    o[e] = fma(w[7], v[e], a[e]);
                    a[e] = fma(w[5], R, fma(w[3], L, fma(w[4], v[e], b[e])));
                    b[e] = w[1] * v[e];
                } else {
                    // taps: (dy+1)*3 + (dx+1)
                    o[e] = fma(w[8], R, fma(w[6], L, fma(w[7], v[e], a[e])));
                    a[e] = fma(w[5], R, fma(w[3], L, fma(w[4], v[e], b[e])));
                    b[e] = fma(w[2], R, fma(w[0], L, w[1] * v[e]));
                }
            }
        }
        const T* srow = ring + sl * C::W + lane * VX;
        if constexpr (CHK) {
            if ((p->phys_lo && j == -1) || (p->phys_hi && j == p->ny)) tb_lds<NE>(o, srow);
        }
        if constexpr (EDGE) {   // branch-free: no divergence between the shuffles
            E r[NE];
            tb_lds<NE>(r, srow);
#pragma unroll
            for (int q = 0; q < NE; ++q) {
                if constexpr (C::FP2) {   // pair q = columns (q, q + NE)
                    o[q].x = ((rmask >> q) & 1u) ? r[q].x : o[q].x;
                    o[q].y = ((rmask >> (q + NE)) & 1u) ? r[q].y : o[q].y;
                } else {
                    o[q] = ((rmask >> q) & 1u) ? r[q] : o[q];
                }
            }
        }
    }

    // One iteration: the K stages in G groups of K/G.  Group g works one row
    // behind group g-1 (its input is pend[g-1], group g-1's output of the
    // previous iteration), so the groups are independent within the
    // iteration and their dependent chains interleave (ILP).  Stage s (group
    // g) outputs row j = i - g - s - 1.  On return v holds the level-K row
    // i - K - (G-1).
    template <bool CHK, bool EDGE>
    __device__ __forceinline__ void row(const T (&w)[C::NTAP], E (&a)[K][NE], E (&b)[K][NE], E (&pend)[C::G][NE],
                                        E (&v)[NE], int i, int slot, unsigned rmask) const {
        E v0[NE];   // the loaded row (v is overwritten by the last group, which runs first)
#pragma unroll
        for (int e = 0; e < NE; ++e) v0[e] = v[e];
        constexpr int KG = K / C::G;
#pragma unroll
        for (int g = C::G - 1; g >= 0; --g) {
            E x[NE];
#pragma unroll
            for (int e = 0; e < NE; ++e) x[e] = g == 0 ? v0[e] : pend[g - 1][e];
#pragma unroll
            for (int q = 0; q < KG; ++q) {
                const int s = g * KG + q;
                E o[NE];
                stage<CHK, EDGE>(w, a[s], b[s], x, o, i - g - s - 1, (slot - g - s - 1) & (C::D - 1), rmask);
#pragma unroll
                for (int e = 0; e < NE; ++e) x[e] = o[e];
            }
#pragma unroll
            for (int e = 0; e < NE; ++e) {
                if (g == C::G - 1) v[e] = x[e];
                else pend[g][e] = x[e];
            }
        }
    }

    template <bool EDGE>
    __device__ __forceinline__ void unit(const T (&w)[C::NTAP], int x0, int y0, int y1) {
        const TbParams<T>& P = *p;
        const int i_lo = (P.phys_lo && y0 - K < -1) ? -1 : y0 - K;
        const int i_end = y1 - 1 + C::LAG;
        const int nrows = i_end - i_lo + 1;
        const int xl = x0 + lane * VX;
        // stores: every valid output of the window (overlapping strips write identical values)
        // (non-edge strips store the aligned middle [x0 + KA, x0 + W - KA): whole vectors)
        const int vlo = EDGE ? max(x0 + K, 0) : x0 + C::KA, vhi = EDGE ? min(x0 + C::W - K, P.nx) : x0 + C::W - C::KA;
        unsigned smask = 0;
#pragma unroll
        for (int e = 0; e < VX; ++e)
            if (xl + e >= vlo && xl + e < vhi) smask |= 1u << e;
        unsigned rmask = 0;   // elements of this lane that are ring columns (-1 or nx)
        if (EDGE) {
            if (xl <= -1 && -1 < xl + VX) rmask |= 1u << (-1 - xl);
            if (xl <= P.nx && P.nx < xl + VX) rmask |= 1u << (P.nx - xl);
        }
        const uint32_t f0 = fill;
        const int ymax = P.ext_y - 1 - (int)P.org_y;   // last allocated row (interior coords)
        auto issue = [&](int t) {
            const uint32_t f = f0 + (uint32_t)t;
            const int sl = (int)(f & (C::D - 1));
            const int yr = min(i_lo + t, ymax);        // rows past the allocation: any row (never valid)
            ptx::mbar_expect_tx(&bar[sl], C::ROW_BYTES);
            ptx::tma_load_2d(ring + sl * C::W, tmap, &bar[sl], (int)P.org_x + x0, (int)P.org_y + yr);
        };
        auto issue_pred = [&](bool pred, int t) {      // (steady state: no branch)
            const uint32_t f = f0 + (uint32_t)t;
            const int sl = (int)(f & (C::D - 1));
            const int yr = min(i_lo + t, ymax);
            ptx::tma_load_2d_pred(pred, ring + sl * C::W, tmap, &bar[sl], C::ROW_BYTES, (int)P.org_x + x0,
                                  (int)P.org_y + yr);
        };
        __syncwarp();
        if (lane == 0) {
            ptx::fence_proxy_async();
            for (int t = 0; t < min(C::PF, nrows); ++t) issue(t);
        }
        E a[K][NE], b[K][NE], pend[C::G][NE];
#pragma unroll
        for (int s = 0; s < K; ++s)
#pragma unroll
            for (int e = 0; e < NE; ++e) a[s][e] = b[s][e] = E{};
#pragma unroll
        for (int q = 0; q < C::G; ++q)
#pragma unroll
            for (int e = 0; e < NE; ++e) pend[q][e] = E{};
        T* g = P.dst + (P.org_y + (long long)(i_lo - C::LAG)) * P.pitch + P.org_x + xl;   // row i - LAG
        // One iteration: load row i = i_lo + t, K stages, store row i - LAG.
        // CHK iterations may output a ring row, a row outside [y0, y1) or a row
        // with peer stores; the steady middle runs without any of those tests.
        // Load-ahead (C::LA): row t+1 is waited for and read from its slot right
        // after the K stages of row t, so its shared-memory latency overlaps the
        // tail of row t's multiply-adds and stores instead of stalling the
        // first multiply-adds of the next iteration.
        E vin[NE];
        auto fetch = [&](int t) {
            const uint32_t f = f0 + (uint32_t)t;
            const int sl = (int)(f & (C::D - 1));
            ptx::mbar_wait_loop(&bar[sl], (f / C::D) & 1u);
            tb_lds<NE>(vin, ring + sl * C::W + lane * VX);
        };
        if constexpr (C::LA) {
            if (nrows > 0) fetch(0);
        }
        // TMA issue: rows [nis, t + PF] (at most NI of them) from lane 0.  The
        // head iterations issue one row each; the steady loop issues a batch
        // of C::NB rows every C::NB iterations (fewer issue sequences per row;
        // the prefetch depth then varies between PF - NB + 1 and PF rows).
        // (Every row t + 1 is issued before iteration t fetches it and no slot
        // is refilled while a row in it can still be read: checked for all
        // loop splits with a host simulation of this schedule.)
        int nis = min(C::PF, nrows);
        auto issue_rows = [&](auto ni_tag, int t) {
            constexpr int NI = decltype(ni_tag)::value;
            if constexpr (NI > 0) {
                __syncwarp();
#pragma unroll
                for (int k = 0; k < NI; ++k) {
                    const int r = nis + k;
                    issue_pred(lane == 0 && r <= t + C::PF && r < nrows, r);
                }
                nis = min(nis + NI, t + C::PF + 1);   // (rows [nis, t + PF] issued, at most NI)
            }
        };
        auto body = [&](auto chk_tag, auto ni_tag, int t) {
            constexpr bool CHK = decltype(chk_tag)::value;
            const int i = i_lo + t;
            if constexpr (!C::IL) issue_rows(ni_tag, t);
            const uint32_t f = f0 + (uint32_t)t;
            const int slot = (int)(f & (C::D - 1));
            E v[NE];
            if constexpr (C::LA) {
#pragma unroll
                for (int e = 0; e < NE; ++e) v[e] = vin[e];
                row<CHK, EDGE>(w, a, b, pend, v, i, slot, rmask);
                if constexpr (C::IL) issue_rows(ni_tag, t);
                if (!CHK || t + 1 < nrows) fetch(t + 1);   // (steady iterations end before nrows - 1)
            } else {
                ptx::mbar_wait_loop(&bar[slot], (f / C::D) & 1u);
                tb_lds<NE>(v, ring + slot * C::W + lane * VX);
                row<CHK, EDGE>(w, a, b, pend, v, i, slot, rmask);
                if constexpr (C::IL) issue_rows(ni_tag, t);
            }
            T* gi = g + (long long)t * P.pitch;
            auto put = [&](T* dst) {
                if constexpr (EDGE || C::FP2) tb_stg<NE>(dst, v, smask);
                else tb_stg_aligned<NE>(dst, v, smask);
            };
            if constexpr (CHK) {
                const int j = i - C::LAG;
                if (j >= y0 && j < y1) {
                    put(gi);
                    if (P.peer_lo_on && j < P.peer_h) put(reinterpret_cast<T*>(reinterpret_cast<char*>(gi) + P.peer_dlo));
                    if (P.peer_hi_on && j >= P.ny - P.peer_h)
                        put(reinterpret_cast<T*>(reinterpret_cast<char*>(gi) + P.peer_dhi));
                }
            } else {
                put(gi);
            }
        };
        using one = std::integral_constant<int, 1>;
        using none = std::integral_constant<int, 0>;
        using batch = std::integral_constant<int, C::NB>;
        // steady iterations: i >= y0 + LAG (stores start, no top ring row), no
        // bottom ring row (i <= ny when phys_hi), no peer rows
        int t_lo = y0 + C::LAG - i_lo;
        if (P.peer_lo_on) t_lo = max(t_lo, P.peer_h + C::LAG - i_lo);
        int t_hi = nrows;                                           // exclusive
        if (P.phys_hi) t_hi = min(t_hi, P.ny + 1 - i_lo);
        if (P.peer_hi_on) t_hi = min(t_hi, P.ny - P.peer_h + C::LAG - i_lo);
        if constexpr (C::LA) t_hi = min(t_hi, nrows - 1);          // the last row fetches nothing
        t_lo = min(max(t_lo, 0), nrows);
        t_hi = max(t_hi, t_lo);
        for (int t = 0; t < t_lo; ++t) body(std::true_type{}, one{}, t);
        int t = t_lo;
        if constexpr (C::NB > 1) {
            for (; t + C::NB <= t_hi; t += C::NB) {
                body(std::false_type{}, batch{}, t);
#pragma unroll
                for (int k = 1; k < C::NB; ++k) body(std::false_type{}, none{}, t + k);
            }
        }
        // (the remainder and the tail issue up to NB rows: they catch up after a batch)
        for (; t < t_hi; ++t) body(std::false_type{}, batch{}, t);
        for (int t2 = t_hi; t2 < nrows; ++t2) body(std::true_type{}, batch{}, t2);
        fill = f0 + (uint32_t)nrows;
    }
};

#ifdef TB_PROBE
// (tuning builds: per-warp smid / start / end / rows, read by stencil_debug_tb_probe)
static __device__ unsigned long long tb_probe_buf[4 * 8192];   // one per translation unit (fp64: tb2d_f64.cu)
__device__ __forceinline__ unsigned long long tb_gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#endif

// One warp per CTA (NW = resident CTAs per SM): every warp-level quantity
// (unit, rows, flags) derives from blockIdx, so the compiler knows it is
// warp-uniform and emits plain SHFLs without divergence checks.
#ifdef TB_MAXNREG
#define TB_REGS __maxnreg__(TB_MAXNREG)
#else
#define TB_REGS __launch_bounds__(32, NW)
#endif
template <typename T, int SHAPE, int K, int VX, int NW>
__global__ void TB_REGS
    tb2d_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ TbParams<T> p) {
    using C = TbCfg<T, SHAPE, K, VX, NW>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x;
    TbWarp<T, SHAPE, K, VX, NW> tw;
    tw.tmap = &tmap;
    tw.p = &p;
    tw.ring = reinterpret_cast<T*>(smem_raw);
    tw.bar = reinterpret_cast<uint64_t*>(smem_raw + (size_t)C::D * C::ROW_BYTES);
    tw.lane = lane;
    tw.fill = 0;
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < C::D; ++s) ptx::mbar_init(&tw.bar[s], 1);
        ptx::fence_mbar_init();
        ptx::prefetch_tmap(&tmap);
    }
    __syncwarp();
    T w[C::NTAP];
#pragma unroll
    for (int k = 0; k < C::NTAP; ++k) w[k] = p.w[k];
#ifdef TB_PROBE
    const unsigned long long t_start = tb_gtime();
#endif
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        // interior strips first (segments of seglen rows), then the two edge
        // strips in segments of seglen_e rows (their ring-column handling
        // costs more per row, so they get shorter segments: no tail)
        int strip, y0, y1;
        if (u < p.units_int) {
            strip = p.nstrips > 2 ? 1 + u % (p.nstrips - 2) : 0;
            y0 = p.y_lo + (u / (p.nstrips - 2)) * p.seglen;
            y1 = min(y0 + p.seglen, p.y_hi);
        } else {
            const int e = u - p.units_int;
            strip = p.nstrips == 1 ? 0 : (e % 2) * (p.nstrips - 1);
            y0 = p.y_lo + (p.nstrips == 1 ? e : e / 2) * p.seglen_e;
            y1 = min(y0 + p.seglen_e, p.y_hi);
        }
        // strips 0 .. nstrips-2 advance by WO from x = -KA; the last one is placed
        // (host) so that its window holds column nx and overlaps its neighbour
        const int x0 = (strip == p.nstrips - 1 && p.nstrips > 1) ? p.x0_right : strip * C::WO - C::KA;
        const bool edge = x0 <= -1 || x0 + C::W > p.nx;   // the window holds a ring column
        if (edge) tw.template unit<true>(w, x0, y0, y1);
        else tw.template unit<false>(w, x0, y0, y1);
    }
#ifdef TB_PROBE
    const int gw = blockIdx.x;
    if (lane == 0 && gw < 8192) {
        unsigned smid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        tb_probe_buf[4 * gw + 0] = smid;
        tb_probe_buf[4 * gw + 1] = t_start;
        tb_probe_buf[4 * gw + 2] = tb_gtime();
        tb_probe_buf[4 * gw + 3] = tw.fill;
    }
#endif
}

// ------------------------------------------------------------------ host
PFN_cuTensorMapEncodeTiled_v12000 tb_encode_fn();

template <typename T, int SHAPE, int K, int VX, int NW>
int tb2d_launch(Plan* p, const SweepCall& c) {
    using C = TbCfg<T, SHAPE, K, VX, NW>;
    const Layout3& L = *c.L;
    if (c.boxes.size() != 1 || c.boxes[0].lo[2] != 0 || c.boxes[0].hi[2] != L.n[2] || L.wrap)
        return set_error(STENCIL_EUNSUPPORTED, "tb2d: one full-width box on a FIXED layout");
    const Box& bx = c.boxes[0];
    if (bx.empty()) return 0;
    TbParams<T> prm;
    std::memset(&prm, 0, sizeof(prm));
    prm.src = static_cast<const T*>(c.src);
    prm.dst = static_cast<T*>(c.dst);
    prm.pitch = L.stride[0];
    prm.org_y = L.origin[0];
    prm.org_x = L.origin[2];
    prm.ny = (int)L.n[0];
    prm.nx = (int)L.n[2];
    prm.ext_y = (int)L.ext[0];
    prm.phys_lo = L.phys_lo[0];
    prm.phys_hi = L.phys_hi[0];
    prm.y_lo = (int)bx.lo[0];
    prm.y_hi = (int)bx.hi[0];
    if (!L.phys_lo[0] && L.lo_valid[0] < K) return set_error(STENCIL_EUNSUPPORTED, "tb2d: ghost rows < fold_m");
    if (!L.phys_hi[0] && L.hi_valid[0] < K) return set_error(STENCIL_EUNSUPPORTED, "tb2d: ghost rows < fold_m");
    if ((int)c.coef->size() != C::NTAP) return set_error(STENCIL_EUNSUPPORTED, "tb2d: expected the dense 3x3 lambda^(1)");
    for (int k = 0; k < C::NTAP; ++k) prm.w[k] = static_cast<T>((*c.coef)[k]);
    if (c.peer_h > 0) {
        const long long plane = (long long)L.n[0] * L.stride[0] * (long long)sizeof(T);
        prm.peer_h = c.peer_h;
        prm.peer_lo_on = c.peer_lo != nullptr;
        prm.peer_hi_on = c.peer_hi != nullptr;
        if (c.peer_lo)
            prm.peer_dlo = (long long)(reinterpret_cast<intptr_t>(c.peer_lo) - reinterpret_cast<intptr_t>(c.dst)) + plane;
        if (c.peer_hi)
            prm.peer_dhi = (long long)(reinterpret_cast<intptr_t>(c.peer_hi) - reinterpret_cast<intptr_t>(c.dst)) - plane;
    }
    const int rows = prm.y_hi - prm.y_lo;
    // strips: x0 = s WO - KA while the window stays left of the ring column nx;
    // then one last strip whose window holds nx, starting no later than the
    // next regular one (so the valid outputs cover [0, nx) without a gap)
    int nstrips = 1, xlast = -C::KA;
    if (xlast + C::W <= prm.nx) {
        while (xlast + C::WO + C::W <= prm.nx) {
            xlast += C::WO;
            ++nstrips;
        }
        int xr = prm.nx + C::KA + 1 - C::W;
        xr = (xr >= 0 ? xr / C::EV : -((-xr + C::EV - 1) / C::EV)) * C::EV;   // align down
        prm.x0_right = std::min(xr, xlast + C::WO);
        ++nstrips;
    }
    const int warps = std::max(1, p->sm_count) * NW;
    // segments: about one unit per resident warp, but at least 4K rows each
    // (a segment re-loads and re-computes 2K rows of pipeline fill); the two
    // edge strips get segments of half the length (2 nseg units each)
    const int nint = nstrips > 2 ? nstrips - 2 : 0, nedge = nstrips > 2 ? 2 : nstrips;
    int nseg = std::max(1, warps / (nint + 2 * nedge));
    nseg = std::min(nseg, std::max(1, rows / (4 * K)));
    const int seglen = (rows + nseg - 1) / nseg;
    nseg = (rows + seglen - 1) / seglen;
    const int seglen_e = std::max(1, (seglen + 1) / 2);
    const int nseg_e = (rows + seglen_e - 1) / seglen_e;
    prm.nstrips = nstrips;
    prm.seglen = seglen;
    prm.seglen_e = seglen_e;
    prm.units_int = nint * nseg;
    prm.units = nint * nseg + nedge * nseg_e;
    const int grid = std::max(1, std::min(warps, prm.units));   // one warp per CTA, NW CTAs per SM

    auto enc = tb_encode_fn();
    if (!enc) return set_error(STENCIL_ECUDA, "cuTensorMapEncodeTiled not available from the driver");
    CUtensorMap map;
    cuuint64_t gdim[2] = {(cuuint64_t)L.ext[2], (cuuint64_t)L.ext[0]};
    cuuint64_t gstr[1] = {(cuuint64_t)(L.stride[0] * (int64_t)sizeof(T))};
    cuuint32_t box[2] = {(cuuint32_t)C::W, 1u};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&map, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                     const_cast<void*>(c.src), gdim, gstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_error(STENCIL_ECUDA, "tb2d: cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    {   // >48 KB dynamic shared memory: per-device opt-in
        static std::mutex mu;
        static bool done[64] = {};
        int dev = 0;
        cudaGetDevice(&dev);
        std::lock_guard<std::mutex> g(mu);
        if (dev >= 0 && dev < 64 && !done[dev]) {
            cudaError_t e = cudaFuncSetAttribute(tb2d_kernel<T, SHAPE, K, VX, NW>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
            if (e != cudaSuccess) return cuda_error(e, "cudaFuncSetAttribute(tb2d)");
            done[dev] = true;
        }
    }
    tb2d_kernel<T, SHAPE, K, VX, NW><<<grid, 32, C::SMEM, (cudaStream_t)c.stream>>>(map, prm);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_error(e, "tb2d_kernel launch");
    return 1;
}

using TbLaunchFn = int (*)(Plan*, const SweepCall&);
TbLaunchFn pick_tb2d_f64(int shape, int K);
TbLaunchFn pick_tb2d_f32(int shape, int K);

}  // namespace sb

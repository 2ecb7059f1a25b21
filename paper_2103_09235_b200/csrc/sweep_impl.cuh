// sweep_impl.cuh — K-G1/K-G2: the streaming sweep of the main (folded-valid) region
// (kernel and host launch templates; instantiated by sweep_{2d,3d,r2}.cu).
//
// One template evaluates one m-step sweep as `S` on-chip passes of the folded
// weights lambda^(Q) (m = Q*S):
//   S = 1      the folded sweep (Eq.2; vertical folding Eq.4 P:381-387 and
//              horizontal folding Eq.5-6 P:390-406 collapse into one weighted
//              sum over supp lambda^(m));
//   Q = 1      the on-chip m-step temporal block ("time loop fusion", P:592,
//              P:708; "multiple time steps computation in registers over the
//              tiles ... without reloading");
//   otherwise  S on-chip passes of a Q-step fold.
//
// B200 mapping:
//  * The grid streams along its slowest axis (z in 3D, y in 2D).  Input planes
//    (in-plane tile + halo) are staged into a ring of shared-memory slots by
//    TMA (cp.async.bulk.tensor, one elected producer thread) with mbarrier
//    full/empty double-buffering; out-of-allocation cells are zero-filled by
//    TMA and are never used by a valid output.
//  * Vertical folding (Eq.4) becomes a register sliding window along the
//    stream axis: every loaded plane is multiplied by each lambda "slice" and
//    added to the 2*Q*r+1 pending output planes held in registers, so each
//    value is read from shared memory once per sweep, not once per tap.
//  * Horizontal folding (Eq.5-6) becomes the in-plane combination: each thread
//    reads its neighbourhood with 16-byte vector loads (double2/float4) and
//    owns VX x VY outputs (register reuse between adjacent outputs = the
//    paper's shifts reusing).
//  * Stages > 1 hand each completed intermediate plane to the next stage
//    through a double-buffered shared-memory plane (one named barrier per
//    stage per plane); tiles overlap by the intermediate halo.
//  * Cells of the frozen physical ring keep u0 at every intermediate level
//    (R1); only tiles whose extent reaches the ring test for it.
//  * Outputs are written with 16-byte vector stores.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "internal.hpp"
#include "ptx.cuh"
#include "sweep_params.cuh"

namespace sb {

// ------------------------------------------------------------------ config
template <typename T_, int ND_, int SHAPE_, int RR_, int Q_, int S_, int NTX_, int NTY_, int VY_, int PB_,
          int NSLOT_, int VXM_ = 1, int MINB_ = 2, int ROT_ = 0, int PINC_ = 0, int CP_ = 0>
struct Cfg {
    using T = T_;
    static constexpr int ND = ND_, SHAPE = SHAPE_, RR = RR_, Q = Q_, S = S_;
    // PB_ = 0: one TMA slot holds exactly one window period (PB = NW planes), so
    // the slot position of a plane is the compile-time window phase and the
    // NW-plane loop body has no per-plane slot branches.
    static constexpr int NTX = NTX_, NTY = NTY_, VY = VY_, PB = PB_ > 0 ? PB_ : 2 * Q_ * RR_ + 1, NSLOT = NSLOT_;
    static constexpr bool PLC = PB_ == 0 && ROT_ == 0;
    static constexpr int VEC = 16 / (int)sizeof(T);   // elements per 16-byte vector
    static constexpr int VX = VXM_ * VEC;              // consecutive x outputs per thread
    static constexpr int RQ = Q * RR;
    static constexpr int RQY = ND == 3 ? RQ : 0;
    static constexpr int H = S * RQ;
    static constexpr int NW = 2 * RQ + 1;
    static constexpr int PX = (RQ + VEC - 1) / VEC * VEC;
    static constexpr int NV = (VX + 2 * PX) / VEC;     // 16-byte vectors per neighbourhood row
    static constexpr int NR = VY + 2 * RQY;
    static constexpr int WX = NTX * VX, WY = NTY * VY;
    static constexpr int HXO = ((S - 1) * RQ + VEC - 1) / VEC * VEC;
    static constexpr int HYO = (S - 1) * RQY;
    // 2D with stages > 1: every warp is its own overlapped tile (32*VX columns,
    // HXO redundant columns per side); intermediate levels move between lanes
    // with shuffles instead of shared memory + a CTA barrier.
    static constexpr bool WARPSTAGE = ND == 2 && S > 1;
    static constexpr int WW = 32 * VX;              // columns computed per warp
    static constexpr int WSTEP = WW - 2 * HXO;      // output columns per warp (WARPSTAGE)
    static constexpr int WOX = WARPSTAGE ? (NTX / 32) * WSTEP : WX - 2 * HXO;
    static constexpr int WOY = WY - 2 * HYO;
    static constexpr int COLS = WARPSTAGE ? (NTX / 32 - 1) * WSTEP + WW + 2 * PX : WX + 2 * PX;
    static constexpr int NBX = (COLS + 255) / 256;
    static constexpr int BX = ((COLS + NBX - 1) / NBX + VEC - 1) / VEC * VEC;
    static constexpr int ROWS = WY + 2 * RQY;
    static constexpr int CHUNK = (PB * ROWS * BX + (128 / (int)sizeof(T)) - 1) / (128 / (int)sizeof(T)) *
                                 (128 / (int)sizeof(T));
    static constexpr int SLOT_ELEMS = NBX * CHUNK;
    static constexpr uint32_t SLOT_BYTES = (uint32_t)(NBX * PB * ROWS * BX * sizeof(T));
    static constexpr int LEV_ELEMS = WARPSTAGE ? 0 : ROWS * COLS;
    static constexpr int NCONS = NTX * NTY;
    static constexpr int NCW = NCONS / 32;
    static constexpr int NTHREADS = NCONS + 32;
    static constexpr int MINB = MINB_;   // resident CTAs per SM the register budget is sized for
    // ROT = 1: one loop iteration per plane, the window slots renamed by a
    // register rotation (NW-1 moves per output) instead of unrolling the loop
    // over the NW window phases (NW x smaller hot loop: instruction-cache fit).
    static constexpr bool ROT = ROT_ != 0;
    // PINC = 1: the folded coefficients are pinned in registers for the whole
    // kernel (otherwise the compiler may re-load them from the constant bank
    // every plane).
    static constexpr bool PINC = PINC_ != 0;
    // CP > 0 (2D): the pass evaluates lambda^(Q) through CP counterparts
    // (coef = a_0..a_{CP-1} | b_0..b_{CP-1}, each 2*RQ+1 long).
    static constexpr int CP = CP_;
    static_assert(CP == 0 || ND_ == 2, "counterpart evaluation is 2D");
    static constexpr int NC = ND == 3 ? NW * NW * NW : NW * NW;
    static constexpr size_t DATA_BYTES = (size_t)NSLOT * SLOT_ELEMS * sizeof(T) +
                                         (size_t)(S - 1) * 2 * LEV_ELEMS * sizeof(T);
    static constexpr size_t SMEM = (size_t)NSLOT * SLOT_ELEMS * sizeof(T) +
                                   (size_t)(S - 1) * 2 * LEV_ELEMS * sizeof(T) + 2 * NSLOT * 8 + NSLOT * 32;
    static_assert(NCONS % 32 == 0, "consumer threads must be whole warps");
    static_assert(WOX > 0 && WOY > 0, "tile too small for the halo");
    static_assert(BX <= 256 && ROWS <= 256 && PB <= 256, "TMA box limit");
    static_assert(ND == 3 || (NTY == 1 && VY == 1), "2D tiles are one row");
};

template <int SHAPE, int RR, int Q>
__host__ __device__ constexpr bool in_support(int oz, int oy, int ox) {
    // STAR: the Q-fold Minkowski sum of axis segments [-RR, RR]; BOX: the full box.
    return SHAPE == STENCIL_BOX
               ? true
               : ((oz < 0 ? -oz : oz) + RR - 1) / RR + ((oy < 0 ? -oy : oy) + RR - 1) / RR +
                         ((ox < 0 ? -ox : ox) + RR - 1) / RR <=
                     Q;
}

__host__ __device__ constexpr int pmod(int a, int n) { return ((a % n) + n) % n; }

#ifndef SB_STORE_CS
#define SB_STORE_CS 0
#endif
template <typename T>
struct VecT;
template <>
struct VecT<double> {
    using V = double2;
    // 16-byte shared-memory load from a 32-bit shared-window address
    static __device__ __forceinline__ void lds(uint32_t a, double* out) {
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(out[0]), "=d"(out[1]) : "r"(a));
    }
    static __device__ __forceinline__ void ld(const double* p, double* out) {
        double2 v = *reinterpret_cast<const double2*>(p);
        out[0] = v.x;
        out[1] = v.y;
    }
    static __device__ __forceinline__ void st(double* p, const double* in) {
        *reinterpret_cast<double2*>(p) = make_double2(in[0], in[1]);
    }
    // global output store; SB_STORE_CS: streaming (evict-first) so the written
    // planes do not displace the input planes neighbouring tiles still need in L2
    static __device__ __forceinline__ void stg(double* p, const double* in) {
#if SB_STORE_CS
        __stcs(reinterpret_cast<double2*>(p), make_double2(in[0], in[1]));
#else
        *reinterpret_cast<double2*>(p) = make_double2(in[0], in[1]);
#endif
    }
};
template <>
struct VecT<float> {
    static __device__ __forceinline__ void lds(uint32_t a, float* out) {
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(out[0]), "=f"(out[1]), "=f"(out[2]), "=f"(out[3])
                     : "r"(a));
    }
    static __device__ __forceinline__ void ld(const float* p, float* out) {
        float4 v = *reinterpret_cast<const float4*>(p);
        out[0] = v.x;
        out[1] = v.y;
        out[2] = v.z;
        out[3] = v.w;
    }
    static __device__ __forceinline__ void st(float* p, const float* in) {
        *reinterpret_cast<float4*>(p) = make_float4(in[0], in[1], in[2], in[3]);
    }
    static __device__ __forceinline__ void stg(float* p, const float* in) {
#if SB_STORE_CS
        __stcs(reinterpret_cast<float4*>(p), make_float4(in[0], in[1], in[2], in[3]));
#else
        *reinterpret_cast<float4*>(p) = make_float4(in[0], in[1], in[2], in[3]);
#endif
    }
};

__device__ __forceinline__ double fmaT(double a, double b, double c) { return fma(a, b, c); }
// Opaque copies: the compiler cannot rematerialise (re-load) the result, so
// loop-invariant coefficients / addresses stay in registers across the plane loop.
__device__ __forceinline__ double pin(double v) {
    double r;
    asm volatile("mov.b64 %0, %1;" : "=d"(r) : "d"(v));
    return r;
}
__device__ __forceinline__ float pin(float v) {
    float r;
    asm volatile("mov.b32 %0, %1;" : "=f"(r) : "f"(v));
    return r;
}
__device__ __forceinline__ uint32_t pin(uint32_t v) {
    uint32_t r;
    asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
    return r;
}
__device__ __forceinline__ float fmaT(float a, float b, float c) { return __fmaf_rn(a, b, c); }

#ifndef SB_FOLD_OXMAJOR
#define SB_FOLD_OXMAJOR 0
#endif

template <class C>
struct Consumer {
    using T = typename C::T;
    T acc[C::S][C::NW][C::VY][C::VX];

    // FMA one level-J plane into stage J's window, streaming its neighbourhood
    // row by row: `ld(rr, row)` fetches row rr (NV 16-byte vectors) of the
    // thread's (VY + 2*RQY) x (VX + 2*PX) neighbourhood, which is applied to
    // every pending output row that uses it, so only one row is live.
    template <int J, int PH, class LD>
    __device__ __forceinline__ void fold_plane(const T (&coef)[C::NC], LD&& ld) {
        constexpr int RQ = C::RQ, RQY = C::RQY, NW = C::NW;
        if constexpr (C::CP > 0) {
            // Counterparts (Eq.4-7): fold the loaded row horizontally with every
            // b_k (h_k = b_k (x) row), then fold the counterparts vertically into
            // the window: pending output at stream offset oz gets sum_k a_k[oz] h_k.
            constexpr int W = 2 * RQ + 1;
            T row[C::NV * C::VEC];
            ld(0, row);
            T h[C::CP][C::VX];
#pragma unroll
            for (int k = 0; k < C::CP; ++k)
#pragma unroll
                for (int vx = 0; vx < C::VX; ++vx) {
                    T s = T(0);
#pragma unroll
                    for (int ox = -RQ; ox <= RQ; ++ox) s = fmaT(coef[C::CP * W + k * W + ox + RQ], row[vx + ox + C::PX], s);
                    h[k][vx] = s;
                }
#pragma unroll
            for (int kk = 0; kk < NW; ++kk) {
                const int oz = RQ - kk;
                const int idx = pmod(PH - J * RQ - RQ + kk, NW);
#pragma unroll
                for (int k = 0; k < C::CP; ++k)
#pragma unroll
                    for (int vx = 0; vx < C::VX; ++vx)
                        acc[J][idx][0][vx] = fmaT(coef[k * W + oz + RQ], h[k][vx], acc[J][idx][0][vx]);
            }
            return;
        }
#pragma unroll
        for (int rr = 0; rr < C::NR; ++rr) {
            T row[C::NV * C::VEC];
            ld(rr, row);
#if SB_FOLD_OXMAJOR
            // x offset outermost: consecutive FMAs update different accumulators
            // (the per-accumulator order of contributions is unchanged: bitwise equal)
#pragma unroll
            for (int ox = -RQ; ox <= RQ; ++ox)
#pragma unroll
                for (int k = 0; k < NW; ++k) {
                    const int oz = RQ - k;
                    const int idx = pmod(PH - J * RQ - RQ + k, NW);
#pragma unroll
                    for (int oy = -RQY; oy <= RQY; ++oy) {
                        const int vy = rr - oy - RQY;
                        if (vy < 0 || vy >= C::VY) continue;
                        if (!in_support<C::SHAPE, C::RR, C::Q>(oz, oy, ox)) continue;
                        const int ci = C::ND == 3 ? ((oz + RQ) * (2 * RQY + 1) + (oy + RQY)) * (2 * RQ + 1) + (ox + RQ)
                                                  : (oz + RQ) * (2 * RQ + 1) + (ox + RQ);
                        const T c = coef[ci];
#pragma unroll
                        for (int vx = 0; vx < C::VX; ++vx)
                            acc[J][idx][vy][vx] = fmaT(c, row[vx + ox + C::PX], acc[J][idx][vy][vx]);
                    }
                }
#else
#pragma unroll
            for (int k = 0; k < NW; ++k) {
                const int oz = RQ - k;
                const int idx = pmod(PH - J * RQ - RQ + k, NW);
#pragma unroll
                for (int oy = -RQY; oy <= RQY; ++oy) {
                    const int vy = rr - oy - RQY;
                    if (vy < 0 || vy >= C::VY) continue;
#pragma unroll
                    for (int ox = -RQ; ox <= RQ; ++ox) {
                        if (!in_support<C::SHAPE, C::RR, C::Q>(oz, oy, ox)) continue;
                        const int ci = C::ND == 3 ? ((oz + RQ) * (2 * RQY + 1) + (oy + RQY)) * (2 * RQ + 1) + (ox + RQ)
                                                  : (oz + RQ) * (2 * RQ + 1) + (ox + RQ);
                        const T c = coef[ci];
#pragma unroll
                        for (int vx = 0; vx < C::VX; ++vx)
                            acc[J][idx][vy][vx] = fmaT(c, row[vx + ox + C::PX], acc[J][idx][vy][vx]);
                    }
                }
            }
#endif
        }
    }
};

// ------------------------------------------------------------------ K-G3 band
// One band block: load the output block plus an m*r halo (clipped at FIXED
// faces to the r-wide ring: nothing beyond the ring is ever needed), run m
// single steps of the ORIGINAL taps on the shrinking region, ring cells
// frozen at u0 (R1/R2), store the block.
//
// Work is distributed by rows (fixed axis-0/axis-1 coordinates): a warp takes
// 32/LX rows at a time, LX = the smallest power of two >= the row length (at
// most 32), so thin x-face blocks keep the warp busy and there is one
// multiply-high (row / n1) per row, not per cell.  The taps are unrolled at compile time in
// canonical order (R4) with shared-memory offsets o0*S0 + o1*S1 + o2.
template <class C, class F>
__device__ __forceinline__ void band_rows(int n0, int n1, int n2, int tid, int nthr, F&& f) {
    const int warp = tid >> 5, lane = tid & 31, nwarp = nthr >> 5;
    int lg = 5;
    while (lg > 0 && (1 << (lg - 1)) >= n2) --lg;
    const int LX = 1 << lg, RPW = 32 >> lg;
    const int lx = lane & (LX - 1), lr = lane >> lg;
    const int rows = n0 * n1;
    // row / n1 as a multiply-high by ceil(2^32 / n1): exact while rows * n1 < 2^32
    const unsigned mg = n1 > 1 ? (unsigned)((0x100000000ull + (unsigned)n1 - 1) / (unsigned)n1) : 0u;
    for (int rb = warp * RPW; rb < rows; rb += nwarp * RPW) {
        const int row = rb + lr;
        if (row >= rows) continue;
        const int c0 = n1 > 1 ? (int)__umulhi((unsigned)row, mg) : row;
        const int c1 = row - c0 * n1;
        f(c0, c1, lx, LX);
    }
}

struct PeerStores {
    long long dlo, dhi;   // byte deltas to the neighbours' ghost planes
    int h, lo_on, hi_on;
};

// Geometry of one band block: output box [olo, ohi), loaded box ilo + [0, ie),
// clo/chi = the loaded box was clipped at a FIXED face (the ring is its edge).
struct BandGeo {
    int olo[3], ohi[3], ilo[3], ie[3], clo[3], chi[3];
};

template <class C>
__device__ __forceinline__ BandGeo band_geo(const BandDesc<typename C::T>& bd, const DevGeom& g, int blk_id) {
    constexpr int RR = C::RR;
    constexpr bool used[3] = {true, C::ND == 3, true};
    int b = 0;
    while (b + 1 < bd.nbox && blk_id >= bd.begin[b + 1]) ++b;
    int t = blk_id - bd.begin[b];
    int bi[3];
    bi[2] = t % bd.nblk[b][2];
    t /= bd.nblk[b][2];
    bi[1] = t % bd.nblk[b][1];
    bi[0] = t / bd.nblk[b][1];
    BandGeo q;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        q.olo[a] = bd.lo[b][a] + bi[a] * bd.blk[b][a];
        q.ohi[a] = min(q.olo[a] + bd.blk[b][a], bd.hi[b][a]);
        const int H = used[a] ? bd.m * RR : 0;
        int lo = q.olo[a] - H, hi = q.ohi[a] + H;
        q.clo[a] = used[a] && g.phys_lo[a] && lo < -RR;
        q.chi[a] = used[a] && g.phys_hi[a] && hi > g.n[a] + RR;
        if (q.clo[a]) lo = -RR;
        if (q.chi[a]) hi = g.n[a] + RR;
        q.ilo[a] = lo;
        q.ie[a] = hi - lo;
    }
    return q;
}

// Issue the block's loads (cp.async / LDGSTS: global -> shared without a
// register round trip, so every thread keeps many loads in flight; cells
// outside the allocation are zero-filled, src-size 0).  The caller commits and
// waits.
template <class C>
__device__ __forceinline__ void band_load(const BandGeo& q, const DevGeom& g, const typename C::T* __restrict__ src,
                                          typename C::T* buf, int tid, int nthr) {
    using T = typename C::T;
    const int S1 = q.ie[2], S0 = q.ie[1] * q.ie[2];
    const long long s0 = g.stride0, s1 = g.stride1;
    band_rows<C>(q.ie[0], q.ie[1], q.ie[2], tid, nthr, [&](int c0, int c1, int lx, int LX) {
        const long long a0 = g.origin[0] + q.ilo[0] + c0, a1 = g.origin[1] + q.ilo[1] + c1;
        const bool rowin = a0 >= 0 && a0 < g.ext[0] && a1 >= 0 && a1 < g.ext[1];
        const int b2 = (int)g.origin[2] + q.ilo[2];   // allocation x of c2 = 0
        const T* gp = src + a0 * s0 + a1 * s1 + b2;
        T* sp = buf + c0 * S0 + c1 * S1;
        const int v0 = rowin ? max(0, -b2) : q.ie[2], v1 = min(q.ie[2], g.ext[2] - b2);
        for (int c2 = lx; c2 < q.ie[2]; c2 += LX) {
            const bool ok = c2 >= v0 && c2 < v1;
            ptx::cp_async<sizeof(T)>(sp + c2, ok ? gp + c2 : src, ok);
        }
    });
}

// The block's m single steps on the shrinking region (ring cells frozen) and
// its store; the loads into buf must be complete and visible (caller's
// wait + __syncthreads).  Ends with __syncthreads: buf is free afterwards.
template <class C>
__device__ __forceinline__ void band_finish(const BandDesc<typename C::T>& bd, const BandGeo& q, const DevGeom& g,
                                            typename C::T* __restrict__ dst, typename C::T* buf, int tid, int nthr,
                                            const PeerStores& ps) {
    using T = typename C::T;
    constexpr int RR = C::RR;
    constexpr bool used[3] = {true, C::ND == 3, true};
    const int S1 = q.ie[2], S0 = q.ie[1] * q.ie[2];
    T* cur = buf;
    T* nxt = buf + q.ie[0] * S0;
    const long long s0 = g.stride0, s1 = g.stride1;
    for (int s = 1; s <= bd.m; ++s) {
        int rlo[3], re[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int sh = used[a] ? s * RR : 0;
            rlo[a] = q.clo[a] ? 0 : sh;
            re[a] = q.ie[a] - rlo[a] - (q.chi[a] ? 0 : sh);
        }
        band_rows<C>(re[0], re[1], re[2], tid, nthr, [&](int d0, int d1, int lx, int LX) {
            const int c0 = d0 + rlo[0], c1 = d1 + rlo[1];
            const int q0 = q.ilo[0] + c0, q1 = q.ilo[1] + c1;
            const bool rowring = (q0 < 0 && g.phys_lo[0]) || (q0 >= g.n[0] && g.phys_hi[0]) ||
                                 (used[1] && ((q1 < 0 && g.phys_lo[1]) || (q1 >= g.n[1] && g.phys_hi[1])));
            const int lrow = c0 * S0 + c1 * S1;
            auto ring2 = [&](int c2) {
                const int q2 = q.ilo[2] + c2;
                return rowring || (q2 < 0 && g.phys_lo[2]) || (q2 >= g.n[2] && g.phys_hi[2]);
            };
            // one cell: the original taps in canonical order (R4)
            auto cell = [&](int li) {
                T acc = T(0);
                int j = 0;
#pragma unroll
                for (int o0 = -RR; o0 <= RR; ++o0)
#pragma unroll
                    for (int o1 = (used[1] ? -RR : 0); o1 <= (used[1] ? RR : 0); ++o1)
#pragma unroll
                        for (int o2 = -RR; o2 <= RR; ++o2) {
                            if (!in_support<C::SHAPE, RR, 1>(o0, o1, o2)) continue;
                            acc = fmaT(bd.w[j], cur[li + o0 * S0 + o1 * S1 + o2], acc);
                            ++j;
                        }
                return acc;
            };
            // two cells per lane in flight: independent FMA chains (the band is
            // latency-bound), each cell's sum in the same order as alone
            for (int d2 = lx; d2 < re[2]; d2 += 2 * LX) {
                const int ca = d2 + rlo[2], cb = ca + LX;
                const bool hb = d2 + LX < re[2];
                const bool ra = ring2(ca), rb = !hb || ring2(cb);
                const int la = lrow + ca, lb = la + LX;
                if (!ra && !rb) {
                    T aa = T(0), ab = T(0);
                    int j = 0;
#pragma unroll
                    for (int o0 = -RR; o0 <= RR; ++o0)
#pragma unroll
                        for (int o1 = (used[1] ? -RR : 0); o1 <= (used[1] ? RR : 0); ++o1)
#pragma unroll
                            for (int o2 = -RR; o2 <= RR; ++o2) {
                                if (!in_support<C::SHAPE, RR, 1>(o0, o1, o2)) continue;
                                const int o = o0 * S0 + o1 * S1 + o2;
                                aa = fmaT(bd.w[j], cur[la + o], aa);
                                ab = fmaT(bd.w[j], cur[lb + o], ab);
                                ++j;
                            }
                    nxt[la] = aa;
                    nxt[lb] = ab;
                } else {
                    nxt[la] = ra ? cur[la] : cell(la);
                    if (hb) nxt[lb] = ring2(cb) ? cur[lb] : cell(lb);
                }
            }
        });
        __syncthreads();
        T* tmp = cur;
        cur = nxt;
        nxt = tmp;
    }
    const int oe0 = q.ohi[0] - q.olo[0], oe1 = q.ohi[1] - q.olo[1], oe2 = q.ohi[2] - q.olo[2];
    band_rows<C>(oe0, oe1, oe2, tid, nthr, [&](int d0, int d1, int lx, int LX) {
        const T* sp = cur + (q.olo[0] - q.ilo[0] + d0) * S0 + (q.olo[1] - q.ilo[1] + d1) * S1 + (q.olo[2] - q.ilo[2]);
        T* gp = dst + (g.origin[0] + q.olo[0] + d0) * s0 + (g.origin[1] + q.olo[1] + d1) * s1 + g.origin[2] + q.olo[2];
        for (int d2 = lx; d2 < oe2; d2 += LX) gp[d2] = sp[d2];
        if (ps.h > 0) {   // fused halo exchange (NEXT-2)
            const int z = q.olo[0] + d0;
            if (ps.lo_on && z < ps.h) {
                T* t = reinterpret_cast<T*>(reinterpret_cast<char*>(gp) + ps.dlo);
                for (int d2 = lx; d2 < oe2; d2 += LX) t[d2] = sp[d2];
            }
            if (ps.hi_on && z >= g.n[0] - ps.h) {
                T* t = reinterpret_cast<T*>(reinterpret_cast<char*>(gp) + ps.dhi);
                for (int d2 = lx; d2 < oe2; d2 += LX) t[d2] = sp[d2];
            }
        }
    });
    __syncthreads();
}

// Per-slot metadata written by the producer before the slot's TMA is issued
// (ordered by the mbarrier's release/acquire), read by the consumers.
struct SlotMeta {
    int z_first;   // interior plane index of the slot's first plane
    int col;       // global column id
    int out_lo;    // outputs of this run are stored for planes [out_lo, out_hi)
    int out_hi;
    int flags;     // 1 = restart (new run: reset accumulators), 2 = end
};
constexpr int META_RESTART = 1, META_END = 2;

__device__ __forceinline__ unsigned long long seg_pack(unsigned e, int nx, int en) {
    return ((unsigned long long)(e & 0xFFFFu) << 48) | ((unsigned long long)(nx & 0xFFFFFF) << 24) |
           (unsigned long long)(en & 0xFFFFFF);
}

// Segment s -> box, column, initial [lo, hi) (planes relative to the box's lo[0]).
__device__ __forceinline__ void seg_init(const DevBoxes& b, int s, int* box, int* col, int* lo, int* hi) {
    int bi = 0;
    while (bi + 1 < b.nbox && s >= b.seg_begin[bi + 1]) ++bi;
    const int local = s - b.seg_begin[bi];
    const int ncol = b.tx[bi] * b.ty[bi];
    const int pz = local / ncol, c = local % ncol;
    const int zlen = b.hi[bi][0] - b.lo[bi][0];
    *box = bi;
    *col = b.col_begin[bi] + c;
    *lo = min(pz * b.zchunk[bi], zlen);
    *hi = min(*lo + b.zchunk[bi], zlen);
}

__device__ __forceinline__ void seg_state(const DevSched& sc, const DevBoxes& b, int s, unsigned long long* w,
                                          int* nx, int* en) {
    *w = *reinterpret_cast<volatile unsigned long long*>(&sc.seg[s]);
    if ((unsigned)(*w >> 48) != (sc.epoch & 0xFFFFu)) {
        int bx, c;
        seg_init(b, s, &bx, &c, nx, en);
    } else {
        *nx = (int)((*w >> 24) & 0xFFFFFF);
        *en = (int)(*w & 0xFFFFFF);
    }
}

template <class C>
__global__ void __launch_bounds__(C::NTHREADS, C::MINB)
    sweep_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ SweepParams<typename C::T, C::NC> p) {
    using T = typename C::T;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* slots = reinterpret_cast<T*>(smem_raw);
    T* lev = slots + C::NSLOT * C::SLOT_ELEMS;
    uint64_t* full = reinterpret_cast<uint64_t*>(lev + (C::S - 1) * 2 * C::LEV_ELEMS);
    uint64_t* empty = full + C::NSLOT;
    SlotMeta* meta = reinterpret_cast<SlotMeta*>(empty + C::NSLOT);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        if (blockIdx.x == 0) {
            p.sc.ctr[((p.sc.epoch + 1) & 1) * 2 + 0] = 0u;
            p.sc.ctr[((p.sc.epoch + 1) & 1) * 2 + 1] = 0u;
        }
#pragma unroll
        for (int s = 0; s < C::NSLOT; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], C::NCW);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();

    // Column id -> tile geometry (compute region origin cx0/cy0, output clip).
    auto col_geom = [&](int col, int* bx, int* cx0, int* cy0, int* xlo, int* xhi, int* ylo, int* yhi) {
        int bi = 0;
        while (bi + 1 < p.b.nbox && col >= p.b.col_begin[bi + 1]) ++bi;
        const int c = col - p.b.col_begin[bi];
        const int itx = c % p.b.tx[bi], ity = c / p.b.tx[bi];
        const int blo2 = p.b.lo[bi][2];
        const int ox0 = (blo2 - blo2 % C::VX) + itx * C::WOX;
        const int oy0 = p.b.lo[bi][1] + ity * C::WOY;
        *bx = bi;
        *cx0 = ox0 - C::HXO;
        *cy0 = oy0 - C::HYO;
        *xlo = max(ox0, blo2);
        *xhi = min(ox0 + C::WOX, p.b.hi[bi][2]);
        *ylo = C::ND == 3 ? max(oy0, p.b.lo[bi][1]) : 0;
        *yhi = C::ND == 3 ? min(oy0 + C::WOY, p.b.hi[bi][1]) : 1;
    };

    // ================================================================ producer warp
    if (warp == C::NCW) {
        const DevSched& sc = p.sc;
        const int myseg = blockIdx.x;
        int sq = 0;
        auto put = [&](const SlotMeta& m) {
            if (lane == 0) {
                const int slot = sq % C::NSLOT, round = sq / C::NSLOT;
                if (round > 0) ptx::mbar_wait(&empty[slot], (round - 1) & 1);
                meta[slot] = m;
                if (m.flags & META_END) {
                    ptx::mbar_arrive(&full[slot]);
                } else {
                    int bx, cx0, cy0, a, b2, c2, d2;
                    col_geom(m.col, &bx, &cx0, &cy0, &a, &b2, &c2, &d2);
                    const int xs = (int)p.g.origin[2] + cx0 - C::PX;
                    const int ys = (int)p.g.origin[1] + cy0 - C::RQY;
                    const int zs = (int)p.g.origin[0] + m.z_first;
                    ptx::mbar_expect_tx(&full[slot], C::SLOT_BYTES);
                    T* dst = slots + slot * C::SLOT_ELEMS;
#pragma unroll
                    for (int c = 0; c < C::NBX; ++c) {
                        if (C::ND == 2)
                            ptx::tma_load_2d(dst + c * C::CHUNK, &tmap, &full[slot], xs + c * C::BX, zs);
                        else
                            ptx::tma_load_3d(dst + c * C::CHUNK, &tmap, &full[slot], xs + c * C::BX, ys, zs);
                    }
                }
            }
            ++sq;
            __syncwarp();
        };
        // claim the next chunk of this CTA's own segment (contiguous by construction)
        auto claim = [&](int sg, int* a, int* b) -> bool {
            int ok = 0, ra = 0, rb = 0;
            if (lane == 0) {
                for (;;) {
                    unsigned long long w;
                    int nx, en;
                    seg_state(sc, p.b, sg, &w, &nx, &en);
                    if (nx >= en) break;
                    const int nn = min(nx + sc.chunk, en);
                    if (atomicCAS(&sc.seg[sg], w, seg_pack(sc.epoch, nn, en)) == w) {
                        ok = 1;
                        ra = nx;
                        rb = nn;
                        break;
                    }
                }
            }
            ok = __shfl_sync(0xffffffffu, ok, 0);
            *a = __shfl_sync(0xffffffffu, ra, 0);
            *b = __shfl_sync(0xffffffffu, rb, 0);
            return ok != 0;
        };
        // steal the upper half of the largest remaining segment (warp-parallel scan)
        auto steal = [&](int* vseg, int* a, int* b) -> bool {
            for (int attempt = 0; attempt < 64; ++attempt) {
                int best = -1, brem = 0;
                for (int s = lane; s < sc.nseg; s += 32) {
                    unsigned long long w;
                    int nx, en;
                    seg_state(sc, p.b, s, &w, &nx, &en);
                    if (en - nx > brem) {
                        brem = en - nx;
                        best = s;
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const int r2 = __shfl_xor_sync(0xffffffffu, brem, o);
                    const int s2 = __shfl_xor_sync(0xffffffffu, best, o);
                    if (r2 > brem || (r2 == brem && s2 > best)) {
                        brem = r2;
                        best = s2;
                    }
                }
                if (best < 0 || brem < sc.min_steal) return false;
                int ok = 0, ra = 0, rb = 0;
                if (lane == 0) {
                    unsigned long long w;
                    int nx, en;
                    seg_state(sc, p.b, best, &w, &nx, &en);
                    const int rem = en - nx;
                    if (rem >= sc.min_steal) {
                        const int mid = nx + rem / 2;
                        if (atomicCAS(&sc.seg[best], w, seg_pack(sc.epoch, nx, mid)) == w) {
                            ok = 1;
                            ra = mid;
                            rb = en;
                        }
                    }
                }
                ok = __shfl_sync(0xffffffffu, ok, 0);
                if (ok) {
                    if (lane == 0) atomicAdd(&sc.stats[1], 1u);
                    *vseg = best;
                    *a = __shfl_sync(0xffffffffu, ra, 0);
                    *b = __shfl_sync(0xffffffffu, rb, 0);
                    return true;
                }
            }
            return false;
        };
        // take the next never-started segment (grid-stride order) as its owner
        auto grab = [&](int* s) -> bool {
            int v = 0;
            if (lane == 0) v = (int)atomicAdd(&sc.ctr[(sc.epoch & 1) * 2 + 0], 1u) + (int)gridDim.x;
            v = __shfl_sync(0xffffffffu, v, 0);
            *s = v;
            if (lane == 0 && v < sc.nseg) atomicAdd(&sc.stats[0], 1u);
            return v < sc.nseg;
        };
        if (lane == 0) ptx::prefetch_tmap(&tmap);
        if (myseg < sc.nseg) {
            int seg = myseg;   // owned segment (claims are contiguous)
            int bx, col, lo0, hi0;
            int a = 0, b = 0;
            for (;;) {
                bool own = claim(seg, &a, &b);
                while (!own && grab(&seg)) own = claim(seg, &a, &b);
                if (!own) {
                    int vs;
                    if (!steal(&vs, &a, &b)) break;
                    seg_init(p.b, vs, &bx, &col, &lo0, &hi0);
                } else {
                    seg_init(p.b, seg, &bx, &col, &lo0, &hi0);
                }
                // one run: outputs [run_lo, claimed_hi) of column `col` (planes relative to the box)
                const int zb = p.b.lo[bx][0];
                const int run_lo = a;
                int claimed_hi = b;
                int z_in = a - C::H;
                int flags = META_RESTART;
                for (;;) {
                    if (own && (claimed_hi + C::H) - (z_in + C::PB) < sc.chunk / 2) {
                        int ca, cb;
                        if (claim(seg, &ca, &cb)) claimed_hi = cb;
                        else own = false;
                    }
                    if (z_in > claimed_hi + C::H - 1) break;
                    put(SlotMeta{zb + z_in, col, zb + run_lo, zb + claimed_hi, flags});
                    flags = 0;
                    z_in += C::PB;
                }
            }
        }
        put(SlotMeta{0, 0, 0, 0, META_END});
    } else {

    // ================================================================ consumers
    const int tx = threadIdx.x % C::NTX, ty = threadIdx.x / C::NTX;
    // first computed column of this thread, relative to the tile's compute origin
    const int tcol = C::WARPSTAGE ? warp * C::WSTEP + lane * C::VX : tx * C::VX;
    // shared-window byte address of this thread's first neighbourhood row in slot 0
    // plus per-vector offsets (loop invariant, kept in registers)
    const uint32_t sbase = pin(ptx::smem_u32(slots) + (uint32_t)(ty * C::VY * C::BX * (int)sizeof(T)));
    uint32_t soff[C::NV];
#pragma unroll
    for (int v = 0; v < C::NV; ++v) {
        const int c = tcol + v * C::VEC;
        soff[v] = (uint32_t)(((c / C::BX) * C::CHUNK + (c % C::BX)) * (int)sizeof(T));
    }
    // folded coefficients lambda^(Q) in registers (only the support is referenced)
    T cf[C::NC];
#pragma unroll
    for (int ci = 0; ci < C::NC; ++ci) {
        const int ox = ci % (2 * C::RQ + 1) - C::RQ;
        const int oy = C::ND == 3 ? (ci / (2 * C::RQ + 1)) % (2 * C::RQY + 1) - C::RQY : 0;
        const int oz = C::ND == 3 ? ci / ((2 * C::RQ + 1) * (2 * C::RQY + 1)) - C::RQ : ci / (2 * C::RQ + 1) - C::RQ;
        const bool used = C::CP > 0 ? ci < 2 * C::CP * (2 * C::RQ + 1) : in_support<C::SHAPE, C::RR, C::Q>(oz, oy, ox);
        cf[ci] = used ? (C::PINC ? pin(p.coef[ci]) : p.coef[ci]) : T(0);
    }
    Consumer<C> cs;
    const T* __restrict__ src = p.src;
    T* __restrict__ dst = p.dst;
    const long long s0 = p.g.stride0, s1 = p.g.stride1;
    // frozen-ring z range: planes z < zlo_f or z >= zhi_f are physical ring
    const int zlo_f = p.g.phys_lo[0] ? 0 : -(1 << 30), zhi_f = p.g.phys_hi[0] ? p.g.n[0] : (1 << 30);
    int gx = 0, gy = 0, xlo = 0, xhi = 0, ylo = 0, yhi = 0;
    T* optr = dst;            // output pointer of plane z_in - H (advanced by s0 per plane)
    unsigned vmask = 0, ymask = 0;   // full-vector stores allowed / rows in range
    bool edge_xy = false;
    int z_first = 0, out_lo = 0, out_hi = 0;
    bool done = false;
    int i = 0, pl = 0, slot = 0;
    uint32_t phase = 0;
#pragma unroll 1
    while (!done) {
        auto step = [&](auto PHc) {
            constexpr int PH = decltype(PHc)::value;
            if (done) return false;
            if (C::PLC ? PH == 0 : pl == 0) {
                ptx::mbar_wait(&full[slot], phase);
                const SlotMeta m = meta[slot];
                if (m.flags & META_END) {
                    done = true;
                    return false;
                }
                if (m.flags & META_RESTART) {
#pragma unroll
                    for (int s = 0; s < C::S; ++s)
#pragma unroll
                        for (int k = 0; k < C::NW; ++k)
#pragma unroll
                            for (int vy = 0; vy < C::VY; ++vy)
#pragma unroll
                                for (int vx = 0; vx < C::VX; ++vx) cs.acc[s][k][vy][vx] = T(0);
                    int bx, cx0, cy0;
                    col_geom(m.col, &bx, &cx0, &cy0, &xlo, &xhi, &ylo, &yhi);
                    gx = cx0 + tcol;
                    gy = cy0 + ty * C::VY;
                    if (C::WARPSTAGE) {   // store only this warp's output columns
                        const int wlo = cx0 + C::HXO + warp * C::WSTEP;
                        xlo = max(xlo, wlo);
                        xhi = min(xhi, wlo + C::WSTEP);
                    }
                    optr = dst + (p.g.origin[0] + m.z_first - C::H) * s0 + (p.g.origin[1] + gy) * s1 +
                           p.g.origin[2] + gx;
                    vmask = 0;
#pragma unroll
                    for (int mm = 0; mm < C::VX / C::VEC; ++mm)
                        if (gx + mm * C::VEC >= xlo && gx + (mm + 1) * C::VEC <= xhi) vmask |= 1u << mm;
                    ymask = 0;
#pragma unroll
                    for (int vy = 0; vy < C::VY; ++vy)
                        if (gy + vy >= ylo && gy + vy < yhi) ymask |= 1u << vy;
                    edge_xy = false;
                    if (C::S > 1) {
                        edge_xy |= p.g.phys_lo[2] && (cx0 - C::PX < 0);
                        edge_xy |= p.g.phys_hi[2] && (cx0 + C::COLS - C::PX > p.g.n[2]);
                        if (C::ND == 3) {
                            edge_xy |= p.g.phys_lo[1] && (cy0 - C::RQY < 0);
                            edge_xy |= p.g.phys_hi[1] && (cy0 + C::WY + C::RQY > p.g.n[1]);
                        }
                    }
                }
                z_first = m.z_first;
                out_lo = m.out_lo;
                out_hi = m.out_hi;
            }
            const int z_in = z_first + (C::PLC ? PH : pl);
            // ---------------- stage 0: level-0 plane from the TMA ring
            {
                const uint32_t pbase = sbase + (uint32_t)((slot * C::SLOT_ELEMS + (C::PLC ? PH : pl) * C::ROWS * C::BX) * (int)sizeof(T));
                cs.template fold_plane<0, PH>(cf, [&](int rr, T* row) {
#pragma unroll
                    for (int v = 0; v < C::NV; ++v)
                        VecT<T>::lds(pbase + (uint32_t)(rr * C::BX * (int)sizeof(T)) + soff[v], row + v * C::VEC);
                });
                if (C::PLC ? PH == C::PB - 1 : pl == C::PB - 1) {
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&empty[slot]);
                }
            }
            // ---------------- stages 1..S-1
            auto stage = [&](auto Jc) {
                constexpr int J = decltype(Jc)::value;
                constexpr int dn = pmod(PH - J * C::RQ, C::NW);
                T v[C::VY][C::VX];
#pragma unroll
                for (int vy = 0; vy < C::VY; ++vy)
#pragma unroll
                    for (int vx = 0; vx < C::VX; ++vx) {
                        v[vy][vx] = cs.acc[J - 1][dn][vy][vx];
                        cs.acc[J - 1][dn][vy][vx] = T(0);
                    }
                const int z = z_in - J * C::RQ;
                if (edge_xy || z < zlo_f || z >= zhi_f) {
#pragma unroll
                    for (int vy = 0; vy < C::VY; ++vy)
#pragma unroll
                        for (int vx = 0; vx < C::VX; ++vx) {
                            const int c3[3] = {z, gy + vy, gx + vx};
                            bool outside = false, inframe = true;
#pragma unroll
                            for (int a = 0; a < 3; ++a) {
                                if (C::ND == 2 && a == 1) continue;
                                if (c3[a] < 0) {
                                    if (p.g.phys_lo[a]) outside = true;
                                    if (c3[a] < -p.g.lo_valid[a]) inframe = false;
                                } else if (c3[a] >= p.g.n[a]) {
                                    if (p.g.phys_hi[a]) outside = true;
                                    if (c3[a] >= p.g.n[a] + p.g.hi_valid[a]) inframe = false;
                                }
                            }
                            if (outside && inframe)
                                v[vy][vx] = src[(p.g.origin[0] + z) * s0 + (p.g.origin[1] + gy + vy) * s1 +
                                                p.g.origin[2] + gx + vx];
                        }
                }
                if constexpr (C::WARPSTAGE) {
                    // neighbours from adjacent lanes (lanes 0/31 get values that only
                    // feed the warp's redundant edge columns)
                    cs.template fold_plane<J, PH>(cf, [&](int, T* row) {
#pragma unroll
                        for (int j = 0; j < C::NV * C::VEC; ++j) {
                            const int rel = j - C::PX;                       // column relative to gx
                            const int d = rel >= 0 ? rel / C::VX : -((-rel + C::VX - 1) / C::VX);
                            const int e = rel - d * C::VX;
                            if (d == 0) row[j] = v[0][e];
                            else if (d < 0) row[j] = __shfl_up_sync(0xffffffffu, v[0][e], -d);
                            else row[j] = __shfl_down_sync(0xffffffffu, v[0][e], d);
                        }
                    });
                } else {
                    T* lp = lev + ((J - 1) * 2 + (i & 1)) * C::LEV_ELEMS;
#pragma unroll
                    for (int vy = 0; vy < C::VY; ++vy)
#pragma unroll
                        for (int mm = 0; mm < C::VX / C::VEC; ++mm)
                            VecT<T>::st(lp + (ty * C::VY + vy + C::RQY) * C::COLS + tcol + C::PX + mm * C::VEC,
                                        &v[vy][mm * C::VEC]);
                    ptx::named_bar_sync(1, C::NCONS);
                    const T* base = lp + (ty * C::VY) * C::COLS + tcol;
                    cs.template fold_plane<J, PH>(cf, [&](int rr, T* row) {
#pragma unroll
                        for (int vv = 0; vv < C::NV; ++vv) VecT<T>::ld(base + rr * C::COLS + vv * C::VEC, row + vv * C::VEC);
                    });
                }
            };
            if constexpr (C::S > 1) stage(std::integral_constant<int, 1>{});
            if constexpr (C::S > 2) stage(std::integral_constant<int, 2>{});
            if constexpr (C::S > 3) stage(std::integral_constant<int, 3>{});
            static_assert(C::S <= 4, "at most 4 on-chip stages");
            // ---------------- output: level-S plane z_in - H
            {
                constexpr int dn = pmod(PH - C::H, C::NW);
                const int z = z_in - C::H;
                if (z >= out_lo && z < out_hi) {
                    auto emit = [&](T* ob) {
#pragma unroll
                        for (int vy = 0; vy < C::VY; ++vy) {
                            if (!(ymask & (1u << vy))) continue;
                            T* op = ob + vy * s1;
#pragma unroll
                            for (int mm = 0; mm < C::VX / C::VEC; ++mm) {
                                if (vmask & (1u << mm)) {
                                    VecT<T>::stg(op + mm * C::VEC, &cs.acc[C::S - 1][dn][vy][mm * C::VEC]);
                                } else {
#pragma unroll
                                    for (int e = 0; e < C::VEC; ++e) {
                                        const int x = gx + mm * C::VEC + e;
                                        if (x >= xlo && x < xhi)
                                            op[mm * C::VEC + e] = cs.acc[C::S - 1][dn][vy][mm * C::VEC + e];
                                    }
                                }
                            }
                        }
                    };
                    emit(optr);
                    if (p.peer_h > 0) {   // fused halo exchange: the neighbours' ghost planes, over NVLink
                        if (p.peer_lo_on && z < p.peer_h)
                            emit(reinterpret_cast<T*>(reinterpret_cast<char*>(optr) + p.peer_dlo));
                        if (p.peer_hi_on && z >= p.g.n[0] - p.peer_h)
                            emit(reinterpret_cast<T*>(reinterpret_cast<char*>(optr) + p.peer_dhi));
                    }
                }
                optr += s0;
#pragma unroll
                for (int vy = 0; vy < C::VY; ++vy)
#pragma unroll
                    for (int vx = 0; vx < C::VX; ++vx) cs.acc[C::S - 1][dn][vy][vx] = T(0);
            }
            ++i;
            if constexpr (C::PLC) {
                if constexpr (PH == C::PB - 1) {
                    if (++slot == C::NSLOT) {
                        slot = 0;
                        phase ^= 1u;
                    }
                }
            } else {
                if (++pl == C::PB) {
                    pl = 0;
                    if (++slot == C::NSLOT) {
                        slot = 0;
                        phase ^= 1u;
                    }
                }
            }
            return true;
        };
        if constexpr (C::ROT) {
            step(std::integral_constant<int, 0>{});
#pragma unroll
            for (int s = 0; s < C::S; ++s) {
                T t0[C::VY][C::VX];
#pragma unroll
                for (int vy = 0; vy < C::VY; ++vy)
#pragma unroll
                    for (int vx = 0; vx < C::VX; ++vx) t0[vy][vx] = cs.acc[s][0][vy][vx];
#pragma unroll
                for (int k = 0; k + 1 < C::NW; ++k)
#pragma unroll
                    for (int vy = 0; vy < C::VY; ++vy)
#pragma unroll
                        for (int vx = 0; vx < C::VX; ++vx) cs.acc[s][k][vy][vx] = cs.acc[s][k + 1][vy][vx];
#pragma unroll
                for (int vy = 0; vy < C::VY; ++vy)
#pragma unroll
                    for (int vx = 0; vx < C::VX; ++vx) cs.acc[s][C::NW - 1][vy][vx] = t0[vy][vx];
            }
        } else {
            // short-circuit: the phases after the END slot do not run
            [&]<int... PHs>(std::integer_sequence<int, PHs...>) {
                (step(std::integral_constant<int, PHs>{}) && ...);
            }(std::make_integer_sequence<int, C::NW>{});
        }
    }
    }  // consumers

    // ================================================================ band (tail filler)
    if (p.band.nblk_total > 0) {
        __shared__ int s_blk;
        const PeerStores ps{p.peer_dlo, p.peer_dhi, p.peer_h, p.peer_lo_on, p.peer_hi_on};
        __syncthreads();
        for (;;) {
            if (threadIdx.x == 0) s_blk = (int)atomicAdd(&p.sc.ctr[(p.sc.epoch & 1) * 2 + 1], 1u);
            __syncthreads();
            const int blk = s_blk;
            if (blk >= p.band.nblk_total) break;
            const BandGeo q = band_geo<C>(p.band, p.g, blk);
            band_load<C>(q, p.g, p.src, slots, threadIdx.x, C::NTHREADS);
            ptx::cp_async_wait_all();
            __syncthreads();
            band_finish<C>(p.band, q, p.g, p.dst, slots, threadIdx.x, C::NTHREADS, ps);
        }
    }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

template <class C>
static int make_tmap(const Layout3& L, const void* base, CUtensorMap* map) {
    auto enc = encode_fn();
    if (!enc) return set_error(STENCIL_ECUDA, "cuTensorMapEncodeTiled not available from the driver");
    using T = typename C::T;
    CUtensorMapDataType dt = sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    cuuint64_t gdim[3];
    cuuint64_t gstr[2];
    cuuint32_t box[3];
    cuuint32_t estr[3] = {1, 1, 1};
    int rank;
    if (C::ND == 2) {
        rank = 2;
        gdim[0] = L.ext[2];
        gdim[1] = L.ext[0];
        gstr[0] = L.stride[0] * sizeof(T);
        box[0] = C::BX;
        box[1] = C::PB;
    } else {
        rank = 3;
        gdim[0] = L.ext[2];
        gdim[1] = L.ext[1];
        gdim[2] = L.ext[0];
        gstr[0] = L.stride[1] * sizeof(T);
        gstr[1] = L.stride[0] * sizeof(T);
        box[0] = C::BX;
        box[1] = C::ROWS;
        box[2] = C::PB;
    }
    CUresult r = enc(map, dt, rank, const_cast<void*>(base), gdim, gstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_error(STENCIL_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return STENCIL_OK;
}

// Occupancy and the >48 KB dynamic shared-memory opt-in are per device (the
// attribute belongs to the current context), so both are kept per device id.
template <class C>
static int occupancy() {
    constexpr int MAXDEV = 64;
    static int occ[MAXDEV] = {};
    static std::mutex mu;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= MAXDEV) dev = 0;
    std::lock_guard<std::mutex> g(mu);
    if (occ[dev] <= 0) {
        if (C::SMEM > 48 * 1024)
            cudaFuncSetAttribute(sweep_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
        int o = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, sweep_kernel<C>, C::NTHREADS, C::SMEM) !=
            cudaSuccess)
            o = 1;
        occ[dev] = std::max(1, o);
    }
    return occ[dev];
}

// Cut the band boxes into blocks whose two shared-memory buffers fit in the
// sweep kernel's data region.
template <typename T>
static int plan_band(Plan* p, const SweepCall& c, BandDesc<T>* bd, size_t smem_cap, int64_t* nblk_total) {
    const int nd = p->ndim;
    bd->m = c.band_m;
    bd->r = p->r;
    bd->used[0] = nd >= 2;
    bd->used[1] = nd == 3;
    bd->used[2] = 1;
    const int k = (int)p->w.size();
    if (k > BAND_MAXT) return set_error(STENCIL_EUNSUPPORTED, "too many taps for the band");
    bd->ntaps = k;
    for (int j = 0; j < k; ++j) {
        int o3[3] = {0, 0, 0};
        if (nd == 1) o3[2] = p->taps[j];
        if (nd == 2) { o3[0] = p->taps[j * 2]; o3[2] = p->taps[j * 2 + 1]; }
        if (nd == 3) { o3[0] = p->taps[j * 3]; o3[1] = p->taps[j * 3 + 1]; o3[2] = p->taps[j * 3 + 2]; }
        for (int a = 0; a < 3; ++a) bd->toff[j][a] = (short)o3[a];
        bd->w[j] = static_cast<T>(p->w[j]);
    }
    const int H = c.band_m * p->r;
    int nb = 0;
    int64_t total = 0;
    for (const Box& b : c.band) {
        if (b.empty()) continue;
        if (nb >= BAND_MAXBOX) return set_error(STENCIL_EUNSUPPORTED, "too many band boxes");
        int blk[3];
        const int cap[3] = {nd == 3 ? 64 : 64, 64, nd == 3 ? 64 : 256};
        for (int a = 0; a < 3; ++a) blk[a] = (int)std::min<int64_t>(b.hi[a] - b.lo[a], cap[a]);
        for (;;) {
            size_t vol = 1;
            for (int a = 0; a < 3; ++a) vol *= (size_t)(blk[a] + (bd->used[a] ? 2 * H : 0));
            if (2 * vol * sizeof(T) <= smem_cap) break;
            // shrink the largest axis, keeping x (coalescing) longest when tied
            int am = 2;
            for (int a = 1; a >= 0; --a)
                if (blk[a] > blk[am] || (blk[a] == blk[am] && a < am && blk[a] > 1)) am = a;
            if (blk[am] <= 1) return set_error(STENCIL_EUNSUPPORTED, "band halo too large for the tile");
            blk[am] = (blk[am] + 1) / 2;
        }
        bd->begin[nb] = (int)total;
        int64_t cnt = 1;
        for (int a = 0; a < 3; ++a) {
            bd->lo[nb][a] = (int)b.lo[a];
            bd->hi[nb][a] = (int)b.hi[a];
            bd->blk[nb][a] = blk[a];
            bd->nblk[nb][a] = (int)((b.hi[a] - b.lo[a] + blk[a] - 1) / blk[a]);
            cnt *= bd->nblk[nb][a];
        }
        total += cnt;
        ++nb;
    }
    bd->nbox = nb;
    bd->begin[nb] = (int)total;
    bd->nblk_total = (int)total;
    *nblk_total = total;
    return STENCIL_OK;
}

static inline bool captured_now(cudaStream_t st) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    return cudaStreamIsCapturing(st, &cap) == cudaSuccess && cap == cudaStreamCaptureStatusActive;
}

template <class C>
static int launch_cfg(Plan* p, const SweepCall& c) {
    using T = typename C::T;
    const Layout3& L = *c.L;
    SweepParams<T, C::NC> prm;
    std::memset(&prm, 0, sizeof(prm));
    prm.src = static_cast<const T*>(c.src);
    prm.dst = static_cast<T*>(c.dst);
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
    fill_geom(L, &prm.g);
    if ((int)c.coef->size() > C::NC || (C::CP == 0 && (int)c.coef->size() != C::NC))
        return set_error(STENCIL_EUNSUPPORTED, "coefficient table size mismatch");
    for (int i = 0; i < (int)c.coef->size(); ++i) prm.coef[i] = static_cast<T>((*c.coef)[i]);

    std::vector<Box> boxes;
    for (const Box& b : c.boxes)
        if (!b.empty()) boxes.push_back(b);
    int64_t band_blocks = 0;
    if (c.band_m > 1) {
        int rc = plan_band<T>(p, c, &prm.band, C::DATA_BYTES, &band_blocks);
        if (rc) return rc;
    }
    if (boxes.empty() && band_blocks == 0) return 0;
    if ((int)boxes.size() > MAXBOX) return set_error(STENCIL_EUNSUPPORTED, "too many boxes");
    const int occ = occupancy<C>();
    // (tests: a capped grid gets 1.5 segments per CTA, so CTAs must grab and,
    // once the grabs run out, the idle half steals from the long second round)
    const int target = p->sched_max_ctas > 0 ? std::max(1, p->sched_max_ctas * 3 / 2) : std::max(1, p->sm_count * occ);
    int64_t vol_total = 0;
    for (const Box& b : boxes) vol_total += b.volume();
    prm.b.nbox = (int)boxes.size();
    int64_t nseg = 0, ncol = 0;
    for (size_t i = 0; i < boxes.size(); ++i) {
        const Box& b = boxes[i];
        int64_t x0 = b.lo[2] - b.lo[2] % C::VX;
        const int ntx = (int)((b.hi[2] - x0 + C::WOX - 1) / C::WOX);
        const int nty = C::ND == 3 ? (int)((b.hi[1] - b.lo[1] + C::WOY - 1) / C::WOY) : 1;
        const int64_t zlen = b.hi[0] - b.lo[0];
        // segment words pack plane bounds in 24-bit fields (seg_pack)
        if (b.hi[0] >= (int64_t(1) << 24) || zlen >= (int64_t(1) << 24))
            return set_error(STENCIL_EUNSUPPORTED, "axis-0 extent >= 2^24 planes");
        const int64_t cols = (int64_t)ntx * nty;
        // initial segments: about one resident wave of CTAs, split by volume.  When
        // there are already at least as many columns as SMs, columns are not split:
        // neighbouring columns then stream the same planes at about the same time and
        // their shared halo rows are still in L2 (3D halos are ~20% of a tile).
        double share = vol_total > 0 ? double(b.volume()) / double(vol_total) : 1.0;
        int64_t want = std::max<int64_t>(1, (int64_t)(target * share) / std::max<int64_t>(1, cols));
        if (p->sched_max_ctas > 0)   // (tests) round up: at least 1.5 segments per CTA overall
            want = std::max<int64_t>(1, ((int64_t)(target * share) + cols - 1) / std::max<int64_t>(1, cols));
        if (C::ND == 3 && cols >= p->sm_count) want = 1;
#ifdef SB_3D_ZSPLIT
        // (tuning) z-chunks per column; segments are z-chunk-major, so CTAs sweep
        // all columns of one z-range before the next and neighbours' halos meet in L2
        if (C::ND == 3 && SB_3D_ZSPLIT > 0) want = SB_3D_ZSPLIT;
#endif
        int64_t nch = std::min<int64_t>(want, std::max<int64_t>(1, zlen / 8));
        int64_t zc = (zlen + nch - 1) / nch;
        nch = (zlen + zc - 1) / zc;
        for (int a = 0; a < 3; ++a) {
            prm.b.lo[i][a] = (int)b.lo[a];
            prm.b.hi[i][a] = (int)b.hi[a];
        }
        prm.b.tx[i] = ntx;
        prm.b.ty[i] = nty;
        prm.b.zchunk[i] = (int)zc;
        prm.b.seg_begin[i] = (int)nseg;
        prm.b.col_begin[i] = (int)ncol;
        nseg += cols * nch;
        ncol += cols;
    }
    prm.b.seg_begin[boxes.size()] = (int)nseg;
    prm.b.col_begin[boxes.size()] = (int)ncol;
    CUtensorMap map;
    {
        int rc = make_tmap<C>(L, c.src, &map);
        if (rc) return rc;
    }
    // dynamic-schedule scratch + epoch (advanced only for a launch that happens).
    // Layout (64-bit words): [0, nseg) segment words | ... | stats (2 words:
    // grabs, steals, 2 spare u32) | counters (2 words: [parity][grab, band]).
    cudaStream_t cst = (cudaStream_t)c.stream;
    if (p->sched_words < nseg + 4) {
        if (captured_now(cst))
            return set_error(STENCIL_EUNSUPPORTED, "schedule scratch must grow: run this call once before capturing it");
        if (p->sched) cudaFree(p->sched);
        p->sched = nullptr;
        int64_t words = std::max<int64_t>(nseg + 4, 8192);
        cudaError_t e = cudaMalloc(&p->sched, words * 8);
        if (e != cudaSuccess) return cuda_error(e, "cudaMalloc(schedule scratch)");
        e = cudaMemsetAsync(p->sched, 0, words * 8, cst);
        if (e != cudaSuccess) return cuda_error(e, "cudaMemsetAsync");
        p->sched_words = words;
        p->epoch = 1;
    }
    unsigned long long* sw = static_cast<unsigned long long*>(p->sched);
    // CUDA graph capture: a captured launch cannot rely on the
    // epoch tags and counter parity left by the launch before it in replay
    // order, so it runs with the reserved epoch 1 on a freshly zeroed schedule
    // and zeroes it again afterwards (restoring the state every eager launch
    // expects: stale tags, zero counters).  Eager epochs skip 0 and 1.
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(cst, &cap) != cudaSuccess) return cuda_error(cudaGetLastError(), "cudaStreamIsCapturing");
    const bool captured = cap == cudaStreamCaptureStatusActive;
    auto zero_sched = [&]() -> int {
        cudaError_t e = cudaMemsetAsync(sw, 0, (size_t)nseg * 8, cst);
        if (e == cudaSuccess) e = cudaMemsetAsync(sw + p->sched_words - 2, 0, 16, cst);
        return e == cudaSuccess ? STENCIL_OK : cuda_error(e, "cudaMemsetAsync(schedule)");
    };
    unsigned epoch;
    if (captured) {
        int rc = zero_sched();
        if (rc) return rc;
        epoch = 1;
    } else {
        p->epoch = (p->epoch + 1) & 0xFFFFu;
        if (p->epoch < 2) {   // wrapped: stale tags could alias, start clean
            cudaError_t e = cudaMemsetAsync(sw, 0, (p->sched_words - 4) * 8, cst);
            if (e == cudaSuccess) e = cudaMemsetAsync(sw + p->sched_words - 2, 0, 16, cst);
            if (e != cudaSuccess) return cuda_error(e, "cudaMemsetAsync");
            p->epoch = 2;
        }
        epoch = p->epoch;
    }
    prm.sc.seg = sw;
    prm.sc.ctr = reinterpret_cast<unsigned int*>(sw + p->sched_words - 2);
    prm.sc.stats = reinterpret_cast<unsigned int*>(sw + p->sched_words - 4);
    prm.sc.epoch = epoch;
    prm.sc.nseg = (int)nseg;
#ifndef SB_CHUNK
#define SB_CHUNK 16
#endif
    prm.sc.chunk = std::max(2 * C::PB, p->sched_chunk > 0 ? p->sched_chunk : SB_CHUNK);
    prm.sc.min_steal = std::max(p->sched_chunk > 0 ? prm.sc.chunk : 2 * prm.sc.chunk,
                                p->sched_min_steal > 0 ? p->sched_min_steal : 4 * C::H + 8);
#ifndef SB_FILL_GRID
#define SB_FILL_GRID 0
#endif
    int64_t tiles = std::min<int64_t>(nseg, target);   // persistent: one resident wave
    // (SB_FILL_GRID: fewer segments than resident CTAs -- e.g. C5's 144 columns
    // on 148 SMs -- launch the whole wave anyway; the extra CTAs start by stealing)
    if (SB_FILL_GRID && C::ND == 3) tiles = std::max<int64_t>(tiles, std::min<int64_t>(target, 2 * nseg));
    if (band_blocks > 0) tiles = std::max<int64_t>(tiles, std::min<int64_t>(band_blocks, target));
    if (p->sched_max_ctas > 0) tiles = std::min<int64_t>(tiles, p->sched_max_ctas);   // (tests: force grabs)
    sweep_kernel<C><<<(unsigned)tiles, C::NTHREADS, C::SMEM, cst>>>(map, prm);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_error(e, "sweep_kernel launch");
    if (captured) {
        int rc = zero_sched();
        if (rc) return rc;
    }
    return 1;
}

}  // namespace sb

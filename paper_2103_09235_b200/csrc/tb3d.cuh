// tb3d.cuh — on-chip multi-step temporal blocking of the 3D radius-1 star
// sweep (SURVEY §8 a6 / NEXT-1 in 3D: "multiple time steps computation in
// registers over the tiles efficiently without reloading", §3.4; "time
// loop fusion").  One launch applies K single steps of the
// original 7 taps per HBM round trip, exactly up to the FIXED faces (no band).
// The same block with BOX = true applies K = 2 single steps of the 27 taps of
// the radius-1 box (3D27P, BASELINE fold_m = 2 for C5): the arriving plane adds
// a 9-point in-plane sum to each of the three output planes in flight.
//
// B200 mapping:
//  * A CTA is an overlapped TY x TX tile of the (y, x) plane streamed along z
//    over a segment of planes; after K steps its valid outputs are the middle
//    (TY - 2K) x (TX - 2KA) cells (KA = K rounded up to a 16-byte vector).
//  * Planes arrive by TMA (cp.async.bulk.tensor.3d, one TY x TX box per
//    plane, issued PF planes ahead by thread 0) into a ring of D slots with one
//    mbarrier each.
//  * Warp w owns tile rows [w VY, (w+1) VY); lane l owns VX = one 16-byte
//    vector of columns.  The K time levels are a register pipeline in push
//    form along z (the GPU reading of the paper's vertical folding, Eq.4
//    P:381-387): when a level-(s-1) plane arrives at stage s it completes
//    level-s plane z-1 with one multiply-add (o = a + w_{z+} v), seeds plane z
//    (a = b + in-plane 5-point(v)) and plane z+1 (b = w_{z-} v).
//  * The stages are skewed by one plane per stage: stage s consumes the
//    level-(s-1) plane its predecessor completed in the PREVIOUS iteration.
//    Within a plane iteration all K stages are then independent (ILP), and
//    one CTA barrier per plane suffices: x-neighbours come from warp
//    shuffles, the rows above/below a warp's patch from its neighbour warps'
//    edge rows, published in shared memory (double-buffered by iteration).
//  * Frozen ring (R1): ring cells (rows -1 / ny, columns -1 / nx,
//    planes -1 / nz) of every level are re-read from `src`, which holds u0
//    there, so the block is exact up to the faces.  Only tiles that touch an
//    x/y face and the first/last iterations of a segment pay for it.
//  * Static schedule (units = tiles x z-segments, grid-stride): launches are
//    CUDA-graph safe.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "internal.hpp"
#include "ptx.cuh"

namespace sb {

template <typename T>
struct Tb3Params {
    const T* src;
    T* dst;
    long long pz, py;               // element strides of axis 0 (z) and axis 1 (y)
    long long org_z, org_y, org_x;  // allocation index of interior (0, 0, 0)
    int nz, ny, nx;                 // local interior extents
    int ext_z;                      // allocated planes (TMA planes are clamped into [0, ext_z))
    int phys_lo, phys_hi;           // z faces are physical: frozen ring planes -1 / nz
    int z_lo, z_hi;                 // output planes of this launch
    int ntx, ntiles, seglen, units;
    // fused halo exchange (NEXT-2), as TbParams: outputs of planes j < peer_h
    // (j >= nz - peer_h) are stored again at the same address + peer_dlo (+ peer_dhi) bytes
    long long peer_dlo, peer_dhi;
    int peer_h, peer_lo_on, peer_hi_on;
    T w[7];                         // 3D7P taps in canonical order: z-, y-, x-, c, x+, y+, z+
    T wb[27];                       // 3D27P: the dense 3x3x3 table, index ((dz+1)*3 + dy+1)*3 + dx+1
};

template <typename T, int K, int NWY, int VY>
struct Tb3Cfg {
    static constexpr int EV = 16 / (int)sizeof(T);
    static constexpr int VX = EV;                       // one 16-byte vector of columns per lane
    static constexpr int TX = 32 * VX;                  // tile columns: one warp across
    static constexpr int TY = NWY * VY;                 // tile rows
    static constexpr int KA = (K + EV - 1) / EV * EV;   // x halo, 16-byte aligned
    static constexpr int WOX = TX - 2 * KA, WOY = TY - 2 * K;   // outputs per tile
    static constexpr int NT = 32 * NWY;
#ifndef TB3_PF
#define TB3_PF 2            // (3: measured equal)
#endif
#ifndef TB3_EDGE_FIRST
#define TB3_EDGE_FIRST 1    // (measured: C4 K=4 634 vs 624, K=3 588 vs 561 GStencil/s)
#endif
#ifndef TB3_CHAIN_XLAST
#define TB3_CHAIN_XLAST 1   // (measured: C4 K=4 624 vs 608, K=3 561 vs 535 GStencil/s)
#endif
#ifndef TB3_K2_CPS
#define TB3_K2_CPS 2        // resident CTAs per SM at K = 2: 128 registers, 2 x 112 KB (measured: C4 K=2 569 vs 519 GStencil/s)
#endif
    static constexpr int CPS = (K == 2 && sizeof(T) == 8) ? TB3_K2_CPS : 1;   // (fp64 stars; the box block keeps one CTA per SM)
    static constexpr int PF = TB3_PF;                   // planes in flight ahead
#ifndef TB3_RING_GLOBAL
#define TB3_RING_GLOBAL 0
#endif
    // TMA plane slots: the 2K - 1 planes behind the current one stay resident,
    // so the frozen ring cells of every level are re-read from shared memory
    // (TB3_RING_GLOBAL: re-read from src in global memory; only the current
    // plane and the PF planes in flight need a slot)
    static constexpr int D = TB3_RING_GLOBAL ? PF + 1 : 2 * K + PF;
    static constexpr int PLANE = TX * TY;               // elements per slot
    static constexpr int NPO = K > 1 ? K - 1 : 1;       // published levels 1..K-1
    static constexpr int EDGE_ELEMS = NPO * 2 * NWY * 2 * TX;   // [level][parity][warp][top|bottom][TX]
    static constexpr size_t SMEM = (size_t)D * PLANE * sizeof(T) + (size_t)EDGE_ELEMS * sizeof(T) + D * 8;
    static_assert(WOX > 0 && WOY > 0, "tile too small for the temporal block");
    static_assert(TX <= 256 && TY <= 256, "TMA box dimension");
};

template <typename T, int K, int NWY, int VY>
struct Tb3Cta {
    using C = Tb3Cfg<T, K, NWY, VY>;
    static constexpr int VX = C::VX;
    const CUtensorMap* tmap;
    const Tb3Params<T>* p;
    T* ring;
    T* edge;
    uint64_t* bar;
    int warp, lane;
    int slot;        // slot of the next plane to consume (planes stream through the slots in order)
    uint32_t phase;  // its mbarrier phase parity

    __device__ __forceinline__ T* edge_row(int lev, int par, int wp, int side) const {
        return edge + ((((lev - 1) * 2 + par) * NWY + wp) * 2 + side) * C::TX;
    }

    __device__ __forceinline__ static void ldv(T (&v)[VX], const T* s) {
        if constexpr (sizeof(T) == 8) {
            const double2 x = *reinterpret_cast<const double2*>(s);
            v[0] = x.x;
            v[1] = x.y;
        } else {
            const float4 x = *reinterpret_cast<const float4*>(s);
            v[0] = x.x;
            v[1] = x.y;
            v[2] = x.z;
            v[3] = x.w;
        }
    }
    __device__ __forceinline__ static void stv(T* s, const T (&v)[VX]) {
        if constexpr (sizeof(T) == 8) *reinterpret_cast<double2*>(s) = make_double2(v[0], v[1]);
        else *reinterpret_cast<float4*>(s) = make_float4(v[0], v[1], v[2], v[3]);
    }

};

// The per-unit body is written as a free function so that the steady and the
// checked iterations are two instantiations of one iteration template.
template <typename T, int K, int NWY, int VY, bool BOX, bool CHK, bool EDGE>
__device__ __forceinline__ void tb3_iter(const Tb3Cta<T, K, NWY, VY>& cta, const T (&w)[7],
                                         T (&a)[K][VY][Tb3Cfg<T, K, NWY, VY>::VX],
                                         T (&b)[K][VY][Tb3Cfg<T, K, NWY, VY>::VX],
                                         T (&po)[Tb3Cfg<T, K, NWY, VY>::NPO][VY][Tb3Cfg<T, K, NWY, VY>::VX], int t,
                                         int i, int slot, uint32_t phase, T* gdst, const T* gsrc, unsigned omask, unsigned rmask,
                                         unsigned fmask, int z0, int z1) {
    using C = Tb3Cfg<T, K, NWY, VY>;
    constexpr int VX = C::VX;
    const Tb3Params<T>& P = *cta.p;
    const int warp = cta.warp, lane = cta.lane;
    ptx::mbar_wait_loop(&cta.bar[slot], phase);
    const int par = t & 1;
    const T* sl = cta.ring + slot * C::PLANE + lane * VX;
#pragma unroll
    for (int s = K; s >= 1; --s) {
        T v[VY][VX], U[VX], Dn[VX];
        if (s == 1) {   // level 0: the plane that just arrived
#pragma unroll
            for (int r = 0; r < VY; ++r) Tb3Cta<T, K, NWY, VY>::ldv(v[r], sl + (warp * VY + r) * C::TX);
            Tb3Cta<T, K, NWY, VY>::ldv(U, sl + max(warp * VY - 1, 0) * C::TX);
            Tb3Cta<T, K, NWY, VY>::ldv(Dn, sl + min(warp * VY + VY, C::TY - 1) * C::TX);
        } else {        // level s-1: own rows from the registers, edge rows from the neighbour warps
#pragma unroll
            for (int r = 0; r < VY; ++r)
#pragma unroll
                for (int e = 0; e < VX; ++e) v[r][e] = po[s - 2][r][e];
            // (branch-free: the first/last warp reads its own edge row instead; the
            // tile's first/last row is outside the valid region from level 1 on)
            Tb3Cta<T, K, NWY, VY>::ldv(U, cta.edge_row(s - 1, par ^ 1, max(warp - 1, 0), 1) + lane * VX);
            Tb3Cta<T, K, NWY, VY>::ldv(Dn, cta.edge_row(s - 1, par ^ 1, min(warp + 1, NWY - 1), 0) + lane * VX);
        }
        T o[VY][VX];
        if constexpr (BOX) {
            // 3D27P: the arriving plane v contributes a 9-point in-plane sum to three
            // output planes: it completes plane z-1 (dz = +1 weights onto a), seeds plane
            // z (dz = 0 onto b) and plane z+1 (dz = -1).  Rows q = 0 (U), 1..VY (v),
            // VY+1 (Dn); their x-neighbours by warp shuffle.
            T Lc[VY + 2], Rc[VY + 2];
#pragma unroll
            for (int q = 0; q < VY + 2; ++q) {
                const T(&row)[VX] = q == 0 ? U : (q == VY + 1 ? Dn : v[q == 0 || q == VY + 1 ? 0 : q - 1]);
                Lc[q] = __shfl_up_sync(0xffffffffu, row[VX - 1], 1);
                Rc[q] = __shfl_down_sync(0xffffffffu, row[0], 1);
            }
            // tap-major order: the 3 VY VX accumulator chains advance together, so
            // consecutive multiply-adds are independent (DFMA latency 8 cycles)
            T sn[VY][VX];
#pragma unroll
            for (int r = 0; r < VY; ++r)
#pragma unroll
                for (int e = 0; e < VX; ++e) {
                    o[r][e] = a[s - 1][r][e];
                    a[s - 1][r][e] = b[s - 1][r][e];
                }
            // (the centre column and row first: the shuffled and shared-memory operands last)
#pragma unroll
            for (int iy = 0; iy < 3; ++iy)
#pragma unroll
                for (int ix = 0; ix < 3; ++ix) {
                    const int dy = iy == 0 ? 0 : (iy == 1 ? -1 : 1), dx = ix == 0 ? 0 : (ix == 1 ? -1 : 1);
                    const int k = (dy + 1) * 3 + dx + 1;
                    // (weights as constant-bank / uniform-register operands: a DFMA then reads two
                    // vector registers; with the 27 weights in vector registers, three reads per
                    // DFMA, C5 K=2 measured 302 vs 347 GStencil/s)
                    const T wp = P.wb[18 + k], wc = P.wb[9 + k], wm = P.wb[k];
#pragma unroll
                    for (int r = 0; r < VY; ++r) {
                        const int q = r + 1 + dy;
                        const T(&row)[VX] = q == 0 ? U : (q == VY + 1 ? Dn : v[q == 0 || q == VY + 1 ? 0 : q - 1]);
#pragma unroll
                        for (int e = 0; e < VX; ++e) {
                            const int c = e + dx;
                            const T x = c < 0 ? Lc[q] : (c >= VX ? Rc[q] : row[c < 0 || c >= VX ? 0 : c]);
                            o[r][e] = fma(wp, x, o[r][e]);
                            a[s - 1][r][e] = fma(wc, x, a[s - 1][r][e]);
                            sn[r][e] = (iy == 0 && ix == 0) ? wm * x : fma(wm, x, sn[r][e]);
                        }
                    }
                }
#pragma unroll
            for (int r = 0; r < VY; ++r)
#pragma unroll
                for (int e = 0; e < VX; ++e) b[s - 1][r][e] = sn[r][e];
        } else {
        T L[VY], R[VY];
#pragma unroll
        for (int r = 0; r < VY; ++r) {
            L[r] = __shfl_up_sync(0xffffffffu, v[r][VX - 1], 1);
            R[r] = __shfl_down_sync(0xffffffffu, v[r][0], 1);
        }
#pragma unroll
        for (int r = 0; r < VY; ++r)
#pragma unroll
            for (int e = 0; e < VX; ++e) {
                const T lf = e == 0 ? L[r] : v[r][e - 1];
                const T rt = e == VX - 1 ? R[r] : v[r][e + 1];
                const T up = r == 0 ? U[e] : v[r - 1][e];
                const T dn = r == VY - 1 ? Dn[e] : v[r + 1][e];
                // taps: 0 z-, 1 y-, 2 x-, 3 c, 4 x+, 5 y+, 6 z+ (in[p + o] weighted by w_o)
                o[r][e] = fma(w[6], v[r][e], a[s - 1][r][e]);
#if TB3_CHAIN_XLAST
                // (the shuffled x-neighbours last: their latency overlaps the first multiply-adds)
                a[s - 1][r][e] = fma(w[4], rt, fma(w[2], lf, fma(w[5], dn, fma(w[1], up, fma(w[3], v[r][e], b[s - 1][r][e])))));
#else
                a[s - 1][r][e] = fma(w[5], dn, fma(w[1], up, fma(w[4], rt, fma(w[2], lf, fma(w[3], v[r][e], b[s - 1][r][e])))));
#endif
                b[s - 1][r][e] = w[0] * v[r][e];
            }
        }
        const int j = i - 2 * s + 1;   // the level-s plane completed now (loaded 2s - 1 iterations ago)
        // frozen ring cells: u0 from the slot of plane j (still resident: D >= 2K + PF)
#if TB3_RING_GLOBAL
        // (from src in global memory: u0 is frozen there; only border tiles and
        // the first/last planes of a segment read it, as L2 hits)
        // (j is clamped into the allocated planes: pipeline-fill iterations complete
        // planes outside them whose values are never used)
        const T* uj = gsrc + (long long)min(max(j, (int)-P.org_z), P.ext_z - 1 - (int)P.org_z) * P.pz;
        const long long rs = P.py;   // row stride
#else
        const T* uj = cta.ring + (slot >= 2 * s - 1 ? slot - (2 * s - 1) : slot - (2 * s - 1) + C::D) * C::PLANE +
                      warp * VY * C::TX + lane * VX;
        constexpr long long rs = C::TX;
#endif
        if constexpr (EDGE) {          // ring columns / rows
            if (rmask) {
#pragma unroll
                for (int r = 0; r < VY; ++r)
#pragma unroll
                    for (int e = 0; e < VX; ++e)
                        if ((rmask >> (r * VX + e)) & 1u) o[r][e] = uj[r * rs + e];
            }
        }
        if constexpr (CHK) {           // ring planes
            if ((P.phys_lo && j == -1) || (P.phys_hi && j == P.nz)) {
#pragma unroll
                for (int r = 0; r < VY; ++r)
#pragma unroll
                    for (int e = 0; e < VX; ++e)
                        if ((fmask >> (r * VX + e)) & 1u) o[r][e] = uj[r * rs + e];
            }
        }
        if (s < K) {   // hand the level-s plane to stage s+1 (next iteration)
#pragma unroll
            for (int r = 0; r < VY; ++r)
#pragma unroll
                for (int e = 0; e < VX; ++e) po[s - 1][r][e] = o[r][e];
            Tb3Cta<T, K, NWY, VY>::stv(cta.edge_row(s, par, warp, 0) + lane * VX, o[0]);
            Tb3Cta<T, K, NWY, VY>::stv(cta.edge_row(s, par, warp, 1) + lane * VX, o[VY - 1]);
        } else {       // level K: store plane j
            bool on = true;
            if constexpr (CHK) on = j >= z0 && j < z1;
            if (on && omask) {
                T* g = gdst + (long long)j * P.pz;
                auto put = [&](T* dst, int r) {
                    const unsigned m = (omask >> (r * VX)) & ((1u << VX) - 1u);
                    if (m == (1u << VX) - 1u) Tb3Cta<T, K, NWY, VY>::stv(dst, o[r]);
                    else if (m) {
#pragma unroll
                        for (int e = 0; e < VX; ++e)
                            if ((m >> e) & 1u) dst[e] = o[r][e];
                    }
                };
#pragma unroll
                for (int r = 0; r < VY; ++r) put(g + (long long)r * P.py, r);
                if constexpr (CHK) {   // fused halo exchange (NEXT-2)
                    if (P.peer_lo_on && j < P.peer_h) {
#pragma unroll
                        for (int r = 0; r < VY; ++r)
                            put(reinterpret_cast<T*>(reinterpret_cast<char*>(g + (long long)r * P.py) + P.peer_dlo), r);
                    }
                    if (P.peer_hi_on && j >= P.nz - P.peer_h) {
#pragma unroll
                        for (int r = 0; r < VY; ++r)
                            put(reinterpret_cast<T*>(reinterpret_cast<char*>(g + (long long)r * P.py) + P.peer_dhi), r);
                    }
                }
            }
        }
    }
    __syncthreads();
}

template <typename T, int K, int NWY, int VY, bool BOX, bool EDGE>
__device__ __forceinline__ void tb3_unit(Tb3Cta<T, K, NWY, VY>& cta, const T (&w)[7], int x0, int y0, int z0,
                                         int z1) {
    using C = Tb3Cfg<T, K, NWY, VY>;
    constexpr int VX = C::VX;
    const Tb3Params<T>& P = *cta.p;
    const int i_lo = (P.phys_lo && z0 - K < -1) ? -1 : z0 - K;
    const int nit = (z1 - i_lo) + 2 * K - 1;   // iteration t loads plane i_lo + t; the last one stores z1 - 1
    const int gy = y0 + cta.warp * VY, gx = x0 + cta.lane * VX;   // interior coords of the patch origin
    unsigned omask = 0, rmask = 0, fmask = 0;
#pragma unroll
    for (int r = 0; r < VY; ++r)
#pragma unroll
        for (int e = 0; e < VX; ++e) {
            const int ry = cta.warp * VY + r, cx = cta.lane * VX + e, y = gy + r, x = gx + e;
            const unsigned bit = 1u << (r * VX + e);
            if (ry >= K && ry < C::TY - K && cx >= C::KA && cx < C::TX - C::KA && y >= 0 && y < P.ny && x >= 0 &&
                x < P.nx)
                omask |= bit;
            const bool frame = y >= -1 && y <= P.ny && x >= -1 && x <= P.nx;
            if (frame) fmask |= bit;
            if (frame && (y < 0 || y >= P.ny || x < 0 || x >= P.nx)) rmask |= bit;
        }
    const int ymax = (int)(P.ext_z - 1 - P.org_z);   // last allocated plane (interior coords)
    int sc = cta.slot;                               // slot of plane t
    uint32_t ph = cta.phase;
    auto issue = [&](int t, int sl) {
        const int zr = min(i_lo + t, ymax);           // planes past the allocation: any plane (never valid)
        ptx::mbar_expect_tx(&cta.bar[sl], (uint32_t)(C::PLANE * sizeof(T)));
        ptx::tma_load_3d(cta.ring + sl * C::PLANE, cta.tmap, &cta.bar[sl], (int)P.org_x + x0, (int)P.org_y + y0,
                         (int)P.org_z + zr);
    };
    if (threadIdx.x == 0) {
        ptx::fence_proxy_async();
        for (int t = 0; t < min(C::PF, nit); ++t) issue(t, sc + t < C::D ? sc + t : sc + t - C::D);
    }
    T a[K][VY][VX], b[K][VY][VX], po[C::NPO][VY][VX];
#pragma unroll
    for (int s = 0; s < K; ++s)
#pragma unroll
        for (int r = 0; r < VY; ++r)
#pragma unroll
            for (int e = 0; e < VX; ++e) a[s][r][e] = b[s][r][e] = T(0);
#pragma unroll
    for (int s = 0; s < C::NPO; ++s)
#pragma unroll
        for (int r = 0; r < VY; ++r)
#pragma unroll
            for (int e = 0; e < VX; ++e) po[s][r][e] = T(0);
    const long long base = P.org_x + gx + (P.org_y + gy) * P.py + P.org_z * P.pz;   // patch origin, plane 0
    T* gdst = P.dst + base;
    const T* gsrc = P.src + base;
    // steady iterations: the stored plane j_K = i - 2K + 1 lies in [z0, z1)
    // without peer rows, and no stage completes a ring plane (j_1 = i - 1 < nz)
    int t_lo = z0 - i_lo + 2 * K - 1;
    if (P.peer_lo_on) t_lo = max(t_lo, P.peer_h - i_lo + 2 * K - 1);
    int t_hi = nit;
    if (P.phys_hi) t_hi = min(t_hi, P.nz - i_lo + 1);
    if (P.peer_hi_on) t_hi = min(t_hi, P.nz - P.peer_h - i_lo + 2 * K - 1);
    t_lo = min(max(t_lo, 0), nit);
    t_hi = max(t_hi, t_lo);
    auto body = [&](auto chk_tag, int t) {
        constexpr bool CHK = decltype(chk_tag)::value;
        if (threadIdx.x == 0 && t + C::PF < nit) issue(t + C::PF, sc + C::PF < C::D ? sc + C::PF : sc + C::PF - C::D);
        tb3_iter<T, K, NWY, VY, BOX, CHK, EDGE>(cta, w, a, b, po, t, i_lo + t, sc, ph, gdst, gsrc, omask, rmask, fmask, z0, z1);
        if (++sc == C::D) {
            sc = 0;
            ph ^= 1u;
        }
    };
    for (int t = 0; t < t_lo; ++t) body(std::true_type{}, t);
    for (int t = t_lo; t < t_hi; ++t) body(std::false_type{}, t);
    for (int t = t_hi; t < nit; ++t) body(std::true_type{}, t);
    cta.slot = sc;
    cta.phase = ph;
}

template <typename T, int K, int NWY, int VY, bool BOX>
__global__ void __launch_bounds__(32 * NWY, BOX ? 1 : Tb3Cfg<T, K, NWY, VY>::CPS)
    tb3d_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ Tb3Params<T> p) {
    using C = Tb3Cfg<T, K, NWY, VY>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Tb3Cta<T, K, NWY, VY> cta;
    cta.tmap = &tmap;
    cta.p = &p;
    cta.ring = reinterpret_cast<T*>(smem_raw);
    cta.edge = cta.ring + C::D * C::PLANE;
    cta.bar = reinterpret_cast<uint64_t*>(cta.edge + C::EDGE_ELEMS);
    cta.warp = threadIdx.x >> 5;
    cta.lane = threadIdx.x & 31;
    cta.slot = 0;
    cta.phase = 0;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < C::D; ++s) ptx::mbar_init(&cta.bar[s], 1);
        ptx::fence_mbar_init();
        ptx::prefetch_tmap(&tmap);
    }
    __syncthreads();
    T w[7];
#pragma unroll
    for (int k = 0; k < 7; ++k) w[k] = p.w[k];
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        int tx, ty, seg;
#if TB3_EDGE_FIRST
        // border tiles (ring handling, the costlier units) first, spread one per
        // CTA of the first wave; then the interior tiles, segment-major
        const int nty = p.ntiles / p.ntx;
        const int nbt = (p.ntx <= 2 || nty <= 2) ? p.ntiles : 2 * p.ntx + 2 * (nty - 2);   // border tiles
        const int nseg = p.units / p.ntiles;
        if (u < nbt * nseg) {
            const int k = u % nbt;
            seg = u / nbt;
            if (nbt == p.ntiles) { tx = k % p.ntx; ty = k / p.ntx; }
            else if (k < p.ntx) { tx = k; ty = 0; }
            else if (k < 2 * p.ntx) { tx = k - p.ntx; ty = nty - 1; }
            else { const int q = k - 2 * p.ntx; ty = 1 + q / 2; tx = (q & 1) ? p.ntx - 1 : 0; }
        } else {
            const int v = u - nbt * nseg, ni = p.ntiles - nbt, k = v % ni;
            seg = v / ni;
            tx = 1 + k % (p.ntx - 2);
            ty = 1 + k / (p.ntx - 2);
        }
#else
        // tiles of one z-segment are consecutive units: concurrent CTAs stream
        // neighbouring tiles over the same planes (their halos meet in L2)
        tx = (u % p.ntiles) % p.ntx;
        ty = (u % p.ntiles) / p.ntx;
        seg = u / p.ntiles;
#endif
        const int x0 = tx * C::WOX - C::KA, y0 = ty * C::WOY - K;
        const int z0 = p.z_lo + seg * p.seglen, z1 = min(z0 + p.seglen, p.z_hi);
        if (z0 >= z1) continue;
        const bool edge = x0 <= -1 || x0 + C::TX > p.nx || y0 <= -1 || y0 + C::TY > p.ny;
        if (edge) tb3_unit<T, K, NWY, VY, BOX, true>(cta, w, x0, y0, z0, z1);
        else tb3_unit<T, K, NWY, VY, BOX, false>(cta, w, x0, y0, z0, z1);
    }
}

// ------------------------------------------------------------------ host
PFN_cuTensorMapEncodeTiled_v12000 tb_encode_fn();

template <typename T, int K, int NWY, int VY, bool BOX = false>
int tb3d_launch(Plan* p, const SweepCall& c) {
    using C = Tb3Cfg<T, K, NWY, VY>;
    const Layout3& L = *c.L;
    if (c.boxes.size() != 1 || L.wrap || c.boxes[0].lo[1] != 0 || c.boxes[0].hi[1] != L.n[1] ||
        c.boxes[0].lo[2] != 0 || c.boxes[0].hi[2] != L.n[2])
        return set_error(STENCIL_EUNSUPPORTED, "tb3d: one full-plane box on a FIXED layout");
    const Box& bx = c.boxes[0];
    if (bx.empty()) return 0;
    if (!L.phys_lo[0] && L.lo_valid[0] < K) return set_error(STENCIL_EUNSUPPORTED, "tb3d: ghost planes < fold_m");
    if (!L.phys_hi[0] && L.hi_valid[0] < K) return set_error(STENCIL_EUNSUPPORTED, "tb3d: ghost planes < fold_m");
    if ((int)c.coef->size() != 27) return set_error(STENCIL_EUNSUPPORTED, "tb3d: expected the dense 3x3x3 lambda^(1)");
    Tb3Params<T> prm;
    std::memset(&prm, 0, sizeof(prm));
    prm.src = static_cast<const T*>(c.src);
    prm.dst = static_cast<T*>(c.dst);
    prm.pz = L.stride[0];
    prm.py = L.stride[1];
    prm.org_z = L.origin[0];
    prm.org_y = L.origin[1];
    prm.org_x = L.origin[2];
    prm.nz = (int)L.n[0];
    prm.ny = (int)L.n[1];
    prm.nx = (int)L.n[2];
    prm.ext_z = (int)L.ext[0];
    prm.phys_lo = L.phys_lo[0];
    prm.phys_hi = L.phys_hi[0];
    prm.z_lo = (int)bx.lo[0];
    prm.z_hi = (int)bx.hi[0];
    // the 7 star entries of the dense table, index ((dz+1)*3 + dy+1)*3 + dx+1, canonical order
    const int idx[7] = {4, 10, 12, 13, 14, 16, 22};
    for (int k = 0; k < 7; ++k) prm.w[k] = static_cast<T>((*c.coef)[idx[k]]);
    for (int k = 0; k < 27; ++k) prm.wb[k] = static_cast<T>((*c.coef)[k]);
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
    const int ntx = (prm.nx + C::WOX - 1) / C::WOX, nty = (prm.ny + C::WOY - 1) / C::WOY;
    const int tiles = ntx * nty;
    const int Z = prm.z_hi - prm.z_lo;
    const int grid_max = std::max(1, p->sm_count) * (BOX ? 1 : C::CPS);   // one CTA per SM (star K = 2: CPS)
    // z-segments: the count with the least (waves x (segment + pipeline fill))
    int best = 1;
    double bcost = 1e300;
    for (int ns = 1; ns <= 16; ++ns) {
        const int seg = (Z + ns - 1) / ns;
        if (ns > 1 && seg < 4 * K) break;
        const int units = tiles * ns;
        const int waves = (units + grid_max - 1) / grid_max;
        const double cost = (double)waves * (seg + 3 * K);
        if (cost < bcost * 0.999) { bcost = cost; best = ns; }
    }
    prm.ntx = ntx;
    prm.ntiles = tiles;
    prm.seglen = (Z + best - 1) / best;
    prm.units = tiles * ((Z + prm.seglen - 1) / prm.seglen);
    const int grid = std::max(1, std::min(grid_max, prm.units));

    auto enc = tb_encode_fn();
    if (!enc) return set_error(STENCIL_ECUDA, "cuTensorMapEncodeTiled not available from the driver");
    CUtensorMap map;
    cuuint64_t gdim[3] = {(cuuint64_t)L.ext[2], (cuuint64_t)L.ext[1], (cuuint64_t)L.ext[0]};
    cuuint64_t gstr[2] = {(cuuint64_t)(L.stride[1] * (int64_t)sizeof(T)), (cuuint64_t)(L.stride[0] * (int64_t)sizeof(T))};
    cuuint32_t box[3] = {(cuuint32_t)C::TX, (cuuint32_t)C::TY, 1u};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(&map, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                     const_cast<void*>(c.src), gdim, gstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_error(STENCIL_ECUDA, "tb3d: cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    {   // >48 KB dynamic shared memory: per-device opt-in
        static std::mutex mu;
        static bool done[64] = {};
        int dev = 0;
        cudaGetDevice(&dev);
        std::lock_guard<std::mutex> g(mu);
        if (dev >= 0 && dev < 64 && !done[dev]) {
            cudaError_t e = cudaFuncSetAttribute(tb3d_kernel<T, K, NWY, VY, BOX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)C::SMEM);
            if (e != cudaSuccess) return cuda_error(e, "cudaFuncSetAttribute(tb3d)");
            done[dev] = true;
        }
    }
    tb3d_kernel<T, K, NWY, VY, BOX><<<grid, C::NT, C::SMEM, (cudaStream_t)c.stream>>>(map, prm);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_error(e, "tb3d_kernel launch");
    return 1;
}

using Tb3LaunchFn = int (*)(Plan*, const SweepCall&);
Tb3LaunchFn pick_tb3d_f64(int shape, int K);
Tb3LaunchFn pick_tb3d_f32(int shape, int K);

}  // namespace sb

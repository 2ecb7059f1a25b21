#pragma once
#include "sweep_impl.cuh"

namespace sb {

// sweep_cfg.cuh — tile configurations of the sweep kernel per (dim, shape, q, stages, r)
// Tile configurations:
//  2D: one row of NTX threads x VX (= 16 B) columns; PB rows per TMA slot.
//  3D: NTX x NTY threads, each 2 x VY outputs, one plane per TMA slot.
#ifndef SB_2D_NTX
#define SB_2D_NTX 256
#endif
#ifndef SB_2D_PB
#define SB_2D_PB 8      // 8-row slots x 3 (C2 m=3/4: +1% / +3% over 4 x 6, same-call A/B)
#endif
#ifndef SB_2D_PBH
#define SB_2D_PBH 4
#endif
#ifndef SB_2D_NSLOT
#define SB_2D_NSLOT 3
#endif
#ifndef SB_3D_NTY
#define SB_3D_NTY 8
#endif
#ifndef SB_3D_NSLOT
#define SB_3D_NSLOT 4
#endif
#ifndef SB_3D_VY
#define SB_3D_VY 2
#endif
#ifndef SB_3D_PB
#define SB_3D_PB 1
#endif
#ifndef SB_3D_MINB
#define SB_3D_MINB 2
#endif
#ifndef SB_2D_MINB
#define SB_2D_MINB 2
#endif
#ifndef SB_PINC_2D
#define SB_PINC_2D 0
#endif
#ifndef SB_PINC_3D
#define SB_PINC_3D 0
#endif
#ifndef SB_ROT_2D
#define SB_ROT_2D 0
#endif
#ifndef SB_ROT_2DH
#define SB_ROT_2DH 0
#endif
#ifndef SB_ROT_3D
#define SB_ROT_3D 0
#endif
#ifndef SB_2D_VXM_HEAVY
#define SB_2D_VXM_HEAVY 2
#endif
// FMA-heavy passes (|supp lambda^(Q)| >= 25) give each thread more outputs so the
// neighbourhood loads and per-row bookkeeping are amortised over more FMAs.
#ifndef SB_STAR_HEAVY_Q
#define SB_STAR_HEAVY_Q 8
#endif
template <int SHAPE, int Q, int RR = 1>
constexpr int vxm2() { return (SHAPE == STENCIL_BOX ? Q * RR >= 2 : Q * RR >= SB_STAR_HEAVY_Q) ? SB_2D_VXM_HEAVY : 1; }
// light (VXM = 1) and heavy (VXM > 1) 2D passes: consumer threads, resident CTAs per SM
#ifndef SB_2D_NTXH
#define SB_2D_NTXH 128
#endif
#ifndef SB_2D_MINBH
#define SB_2D_MINBH 2
#endif
#ifndef SB_2D_NSLOTH
#define SB_2D_NSLOTH 6
#endif
#ifndef SB_2D_NSLOT_PLC
#define SB_2D_NSLOT_PLC 2   // one-period slots: 2 (C2 m=2 740 vs 701 with 3, C3 m=2 equal; 4: C3 -3%)
#endif
// Window periods of at most 5 planes (Q <= 2) use one-period TMA slots (PB = NW,
// branch-free phase loop; measured +7% on C3 m=2, +14% on C2 m=4 in 2 passes);
// the 9-plane window of Q = 4 keeps 4-row slots (a 9-row slot would cost
// occupancy and spill).
#ifndef SB_PLC_MAXNW
#define SB_PLC_MAXNW 5
#endif
template <int Q, int RR = 1>
constexpr bool plc2() { return 2 * Q * RR + 1 <= SB_PLC_MAXNW; }
template <typename T, int SHAPE, int Q, int S, int RR = 1>
using Cfg2 = Cfg<T, 2, SHAPE, RR, Q, S, (vxm2<SHAPE, Q, RR>() > 1 ? SB_2D_NTXH : SB_2D_NTX), 1, 1,
                 (plc2<Q, RR>() ? 0 : vxm2<SHAPE, Q, RR>() > 1 ? SB_2D_PBH : SB_2D_PB),
                 (plc2<Q, RR>() ? SB_2D_NSLOT_PLC : vxm2<SHAPE, Q, RR>() > 1 ? SB_2D_NSLOTH : SB_2D_NSLOT),
                 vxm2<SHAPE, Q, RR>(), (vxm2<SHAPE, Q, RR>() > 1 ? SB_2D_MINBH : SB_2D_MINB),
                 (vxm2<SHAPE, Q, RR>() > 1 && !plc2<Q, RR>() ? SB_ROT_2DH : SB_ROT_2D), SB_PINC_2D>;
// The folded 3D star pass with Q = 2 (25 taps, C4 m=2) takes 4 output rows per
// thread (more FMAs per shared-memory row) in a 64x32 tile (the y halo re-read
// is 12.5% instead of 25%), 2-plane slots and pinned coefficients (measured
// on one box: 520 vs 495 for the 64x16 tile, 458 for the default config).
template <int SHAPE, int Q, int S>
constexpr bool star2_3d() { return SHAPE == STENCIL_STAR && Q == 2 && S == 1; }
// (radius-2 3D configs use the defaults: star2_3d is keyed on Q only for r = 1)
// (round 2: 32x16 consumer threads with 2 rows each instead of 32x8 with 4 --
// same 64x32 tile and shared memory, 17 instead of 9 warps per SM at 90
// registers: C4 m=2 571-583 vs 548-557 GStencil/s, 0.71 of HBM, one gpurun call)
#ifndef SB_S2_NTY
#define SB_S2_NTY 16
#endif
#ifndef SB_S2_VY
#define SB_S2_VY 2
#endif
#ifndef SB_S2_PB
#define SB_S2_PB 2
#endif
#ifndef SB_S2_NSLOT
#define SB_S2_NSLOT 5
#endif
#ifndef SB_S2_MINB
#define SB_S2_MINB 1
#endif
// (round 2: 128-column tiles -- SB_S2_VXM=2 with 12x2 or 8x2 rows per thread
// group -- cut the DRAM reads only from 1.41 to 1.35 GB per sweep and ran at
// 365-469 vs 563 GStencil/s: fewer resident warps; one gpurun call)
#ifndef SB_S2_VXM
#define SB_S2_VXM 1     // 16-byte vectors of x outputs per thread
#endif
// The single 3D box step (27 taps, C5 m=1) takes 4 output rows per thread in a
// 64x32 tile with 3 one-plane slots, 1 CTA/SM (measured 346 vs 318 GStencil/s
// in one gpurun call; the same change costs 14% on the 7-tap star, which keeps
// the defaults).
#ifndef SB_B1_NSLOT
#define SB_B1_NSLOT 3
#endif
#ifndef SB_B1_PB
#define SB_B1_PB 1
#endif
// (round 2: 32x16 consumer threads x 4 rows = a 64x64 tile -- y halo 1.06x
// instead of 1.125x, 17 warps per SM at 92 registers: C5 m=1 367 vs 338
// GStencil/s, 0.90 of HBM, one gpurun call; 64x32 with 2 rows per thread: 304)
#ifndef SB_B1_NTY
#define SB_B1_NTY 16
#endif
#ifndef SB_B1_VY
#define SB_B1_VY 4
#endif
template <int SHAPE, int Q, int S, int RR>
constexpr bool box1_3d() { return SHAPE == STENCIL_BOX && Q == 1 && S == 1 && RR == 1; }
// two on-chip box steps (C5 m=2)
#ifndef SB_B2_NTY
#define SB_B2_NTY 8
#endif
#ifndef SB_B2_VY
#define SB_B2_VY 2
#endif
#ifndef SB_B2_MINB
#define SB_B2_MINB 2
#endif
#ifndef SB_B2_PINC
#define SB_B2_PINC 0
#endif
#ifndef SB_B2_NSLOT
#define SB_B2_NSLOT 4
#endif
template <int SHAPE, int Q, int S, int RR>
constexpr bool box2s_3d() { return SHAPE == STENCIL_BOX && Q == 1 && S == 2 && RR == 1; }
template <typename T, int SHAPE, int Q, int S, int RR = 1>
using Cfg3 = Cfg<T, 3, SHAPE, RR, Q, S, 32,
                 (star2_3d<SHAPE, Q, S>() ? SB_S2_NTY : box2s_3d<SHAPE, Q, S, RR>() ? SB_B2_NTY
                                                     : box1_3d<SHAPE, Q, S, RR>() ? SB_B1_NTY : SB_3D_NTY),
                 (star2_3d<SHAPE, Q, S>() ? SB_S2_VY : box1_3d<SHAPE, Q, S, RR>() ? SB_B1_VY
                                                    : box2s_3d<SHAPE, Q, S, RR>() ? SB_B2_VY : SB_3D_VY),
                 (star2_3d<SHAPE, Q, S>() ? SB_S2_PB : box1_3d<SHAPE, Q, S, RR>() ? SB_B1_PB : SB_3D_PB),
                 (star2_3d<SHAPE, Q, S>() ? SB_S2_NSLOT : box1_3d<SHAPE, Q, S, RR>() ? SB_B1_NSLOT
                                                       : box2s_3d<SHAPE, Q, S, RR>() ? SB_B2_NSLOT : SB_3D_NSLOT),
                 (star2_3d<SHAPE, Q, S>() ? SB_S2_VXM : 1),
                 (star2_3d<SHAPE, Q, S>() ? SB_S2_MINB : box1_3d<SHAPE, Q, S, RR>() ? 1
                                                      : box2s_3d<SHAPE, Q, S, RR>() ? SB_B2_MINB : SB_3D_MINB),
                 SB_ROT_3D, (star2_3d<SHAPE, Q, S>() ? 1 : box2s_3d<SHAPE, Q, S, RR>() ? SB_B2_PINC : SB_PINC_3D)>;


// 2D counterpart passes (NEXT-3): one pass of lambda^(Q) through CP
// counterparts; the tile of the light 2D passes (4 + 2*... FMAs per row-point).
template <typename T, int Q, int CP>
using Cfg2CP = Cfg<T, 2, STENCIL_BOX, 1, Q, 1, SB_2D_NTX, 1, 1, (plc2<Q>() ? 0 : SB_2D_PB),
                   (plc2<Q>() ? SB_2D_NSLOT_PLC : SB_2D_NSLOT), 1, SB_2D_MINB, 0, 0, CP>;

using LaunchFn = int (*)(Plan*, const SweepCall&);

// Per-TU pickers (sweep_2d.cu, sweep_3d.cu, sweep_r2.cu)
LaunchFn pick_2d(int dtype, int shape, int q, int s);
LaunchFn pick_3d(int dtype, int shape, int q, int s);
LaunchFn pick_r2(int dtype, int nd, int shape, int q, int s);
LaunchFn pick_cp(int dtype, int q, int rank);

}  // namespace sb

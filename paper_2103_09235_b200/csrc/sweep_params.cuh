// sweep_params.cuh — kernel-parameter structs shared by the sweep and band
// kernels (passed by value as __grid_constant__ parameters).
#pragma once
#include "internal.hpp"

namespace sb {

constexpr int MAXBOX = 8;

struct DevGeom {
    long long stride0, stride1;
    long long origin[3];
    int n[3];
    int lo_valid[3], hi_valid[3];
    int phys_lo[3], phys_hi[3];
    int ext[3];
};

// Output boxes of one launch, tiled into columns (in-plane tiles streamed
// along axis 0) and, initially, `parts` equal z-segments per column.
struct DevBoxes {
    int nbox;
    int lo[MAXBOX][3], hi[MAXBOX][3];
    int seg_begin[MAXBOX + 1];   // first segment of each box
    int col_begin[MAXBOX + 1];   // first global column id of each box
    int tx[MAXBOX], ty[MAXBOX];  // columns per box along x and y
    int zchunk[MAXBOX];          // initial segment length (planes)
};

// Dynamic schedule: one 64-bit word per segment (epoch | next | end) in a
// plan-owned device scratch; CTAs claim contiguous chunks of their own segment
// and steal the upper half of the largest remaining segment when done.
struct DevSched {
    unsigned long long* seg;
    unsigned int* ctr;        // [2 parities][2]: grab counter, band counter (this launch: epoch & 1)
    unsigned int* stats;      // cumulative: [0] successful grabs, [1] successful steals (tests)
    unsigned int epoch;
    int nseg;
    int chunk;
    int min_steal;
};

// The exact stepwise band (K-G3) carried by the same launch: boxes within
// (m-1)*r of a FIXED face, cut into blocks that CTAs claim once their main
// work is exhausted (the band fills the tail of the sweep).
constexpr int BAND_MAXT = 125;
constexpr int BAND_MAXBOX = 26;

template <typename T>
struct BandDesc {
    int nbox, nblk_total;
    int lo[BAND_MAXBOX][3], hi[BAND_MAXBOX][3];
    int blk[BAND_MAXBOX][3];
    int nblk[BAND_MAXBOX][3];
    int begin[BAND_MAXBOX + 1];
    int m, r, ntaps;
    int used[3];
    short toff[BAND_MAXT][3];
    T w[BAND_MAXT];
};

template <typename T, int NC>
struct SweepParams {
    const T* src;
    T* dst;
    DevGeom g;
    DevBoxes b;
    DevSched sc;
    BandDesc<T> band;
    // Fused halo exchange (NEXT-2): outputs of local planes z < peer_h are also
    // stored into the lower neighbour's ghost planes and those of z >= n0 - peer_h
    // into the upper neighbour's, at the same element offset plus these byte
    // deltas (neighbour buffer - dst +/- n0 planes); 0 = no such neighbour.
    long long peer_dlo, peer_dhi;
    int peer_h, peer_lo_on, peer_hi_on;
    T coef[NC];
};

inline void fill_geom(const Layout3& L, DevGeom* g) {
    g->stride0 = L.stride[0];
    g->stride1 = L.stride[1];
    for (int a = 0; a < 3; ++a) {
        g->origin[a] = L.origin[a];
        g->n[a] = (int)L.n[a];
        g->lo_valid[a] = (int)L.lo_valid[a];
        g->hi_valid[a] = (int)L.hi_valid[a];
        g->phys_lo[a] = L.phys_lo[a];
        g->phys_hi[a] = L.phys_hi[a];
        g->ext[a] = (int)L.ext[a];
    }
}

bool sweep_supported(const Plan* p, int q, int s, int rank = 0);

}  // namespace sb

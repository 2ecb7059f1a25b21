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

struct DevBoxes {
    int nbox;
    int lo[MAXBOX][3], hi[MAXBOX][3];
    int tiles_begin[MAXBOX + 1];
    int tx[MAXBOX], ty[MAXBOX];
    int zchunk[MAXBOX];
};

template <typename T, int NC>
struct SweepParams {
    const T* src;
    T* dst;
    DevGeom g;
    DevBoxes b;
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

bool sweep_supported(const Plan* p, int q, int s);

}  // namespace sb

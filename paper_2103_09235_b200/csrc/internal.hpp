// internal.hpp — host-side structures of the B200 stencil library (not part
// of the C-ABI).  See include/stencil_b200.h for the contract and DESIGN.md
// for the design.
#pragma once
#include <cstdint>
#include <string>
#include <vector>
#include <map>
#include <mutex>

#include "../../include/stencil_b200.h"

namespace sb {

// ------------------------------------------------------------------ errors
int set_error(int code, const std::string& msg);
int cuda_error(int cuda_err, const char* what);

// ------------------------------------------------------------------ geometry
// Everything is kept as 3 axes internally: axis 0 = streaming axis (z in 3D,
// y in 2D, unused in 1D), axis 1 = y (3D only), axis 2 = x (unit stride).
struct Box {
    int64_t lo[3], hi[3];   // interior coordinates, half-open
    bool empty() const { return lo[0] >= hi[0] || lo[1] >= hi[1] || lo[2] >= hi[2]; }
    int64_t volume() const { return empty() ? 0 : (hi[0] - lo[0]) * (hi[1] - lo[1]) * (hi[2] - lo[2]); }
};

struct Layout3 {
    int ndim = 0;
    int r = 1;
    int64_t n[3] = {1, 1, 1};        // local interior extents
    int64_t ext[3] = {1, 1, 1};      // allocated extents
    int64_t stride[3] = {0, 0, 1};   // element strides
    int64_t origin[3] = {0, 0, 0};   // allocation index of interior 0
    int64_t lo_valid[3] = {0, 0, 0}; // cells below 0 that hold data (r, or halo for ghosts)
    int64_t hi_valid[3] = {0, 0, 0};
    int phys_lo[3] = {1, 1, 1};      // 1 = physical (frozen-ring) face
    int phys_hi[3] = {1, 1, 1};
    int64_t esize = 8;
    int64_t bytes = 0;
    int64_t gofs0 = 0;               // dist: global index of local plane 0
    int64_t gn[3] = {1, 1, 1};       // global interior extents
    bool wrap = false;               // PERIODIC: ghosts hold the wrapped interior
};

// ------------------------------------------------------------------ plan
struct Plan {
    int ndim;
    int64_t dims[3];     // user order, slowest first
    int r;
    int shape;           // STENCIL_STAR / STENCIL_BOX
    int dtype;           // STENCIL_F32 / STENCIL_F64
    int boundary;
    std::vector<int> taps;       // k * ndim canonical offsets
    std::vector<double> w;       // k weights (fp64)
    // folded maps lambda^(q) as dense (2qr+1)^ndim fp64, q = 1..STENCIL_MAX_FOLD
    std::map<int, std::vector<double>> lam;
    std::map<int, struct LowRank*> lowrank;   // owned; 2D counterpart decompositions
    std::mutex mu;
    int64_t last_launches = 0;
    // measurement support (stencil_plan_set_timing)
    bool timing = false;
    bool counterparts = true;     // stencil_plan_set_counterparts
    struct TimingRec { void* a; void* b; int kind; int64_t bytes; int64_t fmas; };
    std::vector<TimingRec> recs;
    std::vector<void*> event_pool;
    int sm_count = 0;
    int device = -1;
    // dynamic-schedule scratch (device, plan-owned; 8 bytes per segment)
    void* sched = nullptr;
    int64_t sched_words = 0;
    unsigned int epoch = 0;
    // stencil_run_host_batch: internal copy streams + pipeline events (lazy)
    void* h2d_stream = nullptr;
    void* d2h_stream = nullptr;
    void* pipe_ev[7] = {};   // start, in[2], comp[2], out[2]
    // schedule granularity override (stencil_plan_set_schedule; 0 = default)
    int sched_chunk = 0, sched_min_steal = 0, sched_max_ctas = 0;
};

const std::vector<double>& folded(Plan* p, int q);   // cached lambda^(q)
Layout3 make_layout(const Plan* p, int rank, int nranks, int halo);
void to_public(const Layout3& L, stencil_layout* out);

// Evaluation variant of one m-step sweep on the main (folded-valid) region.
// rank > 0: the pass evaluates lambda^(q) through `rank` counterparts
// (Eq.4-7): a horizontal fold per counterpart of every loaded row,
// then the vertical fold of the counterparts into the window (2D only).
struct Variant { int q; int stages; int rank = 0; };
Variant choose_variant(Plan* p, int m);
bool tb_supported(const Plan* p, int q, int s);   // 2D temporal block compiled for (q = 1, s steps)
int auto_fold(Plan* p);   // fold_m = 0 in a run: the measured-best fold for the family

// Counterpart decomposition of the 2D folded matrix Lambda = lambda^(q)
// (rows: vertical offset, columns: horizontal offset):
//   Lambda = sum_k a_k b_k^T, k < rank,
// by LU with complete pivoting, stopped when the largest residual entry is
// below 1e-13 max|Lambda| (exact for the paper's rank-1 uniform example).
struct LowRank { int rank = 0; int W = 0; std::vector<double> a, b; };   // a, b: rank x W
const LowRank& lowrank(Plan* p, int q);
int support_size(int ndim, int shape, int r, int q);

// ------------------------------------------------------------------ kernels
// Sweep of the main region with `stages` on-chip passes of lambda^(q).
// Returns number of launches (>=0) or a negative status.
struct SweepCall {
    const void* src;
    void* dst;
    const Layout3* L;
    std::vector<Box> boxes;   // output boxes (interior coords)
    int q, stages;
    const std::vector<double>* coef;   // lambda^(q), dense fp64 (or packed a_k | b_k when rank > 0)
    int rank = 0;                      // counterpart evaluation (Variant::rank)
    // fused halo exchange (NEXT-2): neighbour buffers of the same parity as dst
    void* peer_lo = nullptr;           // rank - 1 (receives local planes [0, peer_h))
    void* peer_hi = nullptr;           // rank + 1 (receives local planes [n0 - peer_h, n0))
    int peer_h = 0;
    std::vector<Box> band;    // exact stepwise band boxes (K-G3), same launch
    int band_m = 1;           // steps of the band (the sweep's fold_m)
    void* stream;
};
int launch_sweep(Plan* p, const SweepCall& c);

// 1D on-chip multi-step kernel (K-G4): T steps (fold m) in one launch.
int launch_1d(Plan* p, const void* src, void* dst, const Layout3* L, int64_t T, int m,
              int stages_flag, void* stream);   // PERIODIC (L->wrap): loads wrap around
int onchip1d_cells_per_lane(int r, int m, bool wrap);   // V of the warp window (32*V cells)

// PERIODIC: fill every ghost cell of buf from its wrapped interior cell.
int launch_wrap_fill(Plan* p, void* buf, const Layout3* L, void* stream);
// Copy every non-interior cell (ring, ghosts, pads) src -> dst (K-G5).
// keep_ghost_interior: leave the interior (y, x) cells of non-physical ghost
// planes alone (the fused exchange's neighbours write them).
int launch_ring_copy(Plan* p, const void* src, void* dst, const Layout3* L, void* stream,
                     bool keep_ghost_interior = false);
// K-G0 seeded field over the frame (global padded index).
int launch_fill(Plan* p, void* buf, const Layout3* L, uint64_t seed, void* stream);

// Measurement: bracket a launch with events when timing is enabled.
struct TimedScope {
    Plan* p; void* stream; int kind; int64_t bytes, fmas; void* a = nullptr;
    TimedScope(Plan* p_, void* s, int k, int64_t b, int64_t f);
    ~TimedScope();
};

// ------------------------------------------------------------------ run
int run_single(Plan* p, const void* in, void* out, int64_t T, int m, int stages, void* ws,
               void* stream);

}  // namespace sb

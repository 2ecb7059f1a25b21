// sweep.cu — dispatch of the main-region sweep (K-G1/K-G2) to the compiled
// tile configurations (sweep_cfg.cuh), instantiated per family in
// sweep_2d.cu, sweep_3d.cu and sweep_r2.cu (kernel: sweep_impl.cuh).
#include "sweep_cfg.cuh"
#include "tb2d.cuh"
#include "tb3d.cuh"

namespace sb {

static LaunchFn pick(int dtype, int nd, int shape, int r, int q, int s) {
    if (r == 1 && nd == 2) return pick_2d(dtype, shape, q, s);
    if (r == 1 && nd == 3) return pick_3d(dtype, shape, q, s);
    if (r == 2 && (nd == 2 || nd == 3)) return pick_r2(dtype, nd, shape, q, s);
    return nullptr;
}

// The on-chip stepwise block (q = 1, stages = m) of a 2D radius-1 FIXED plan
// runs in the warp-tile temporal-blocking kernel (tb2d.cuh); that of a 3D
// radius-1 star or 27-point box in the CTA-tile temporal block (tb3d.cuh).
static TbLaunchFn pick_tb(const Plan* p, int q, int s, int rank, bool wrap) {
    if (rank != 0 || q != 1 || s < 2 || p->r != 1 || wrap) return nullptr;
    if (p->ndim == 2) return p->dtype == STENCIL_F64 ? pick_tb2d_f64(p->shape, s) : pick_tb2d_f32(p->shape, s);
    if (p->ndim == 3) return p->dtype == STENCIL_F64 ? pick_tb3d_f64(p->shape, s) : pick_tb3d_f32(p->shape, s);
    return nullptr;
}

bool tb_supported(const Plan* p, int q, int s) { return pick_tb(p, q, s, 0, p->boundary == STENCIL_BC_PERIODIC) != nullptr; }

bool sweep_supported(const Plan* p, int q, int s, int rank) {
    if (rank == 0 && pick_tb(p, q, s, 0, p->boundary == STENCIL_BC_PERIODIC)) return true;
    if (rank > 0) return s == 1 && p->ndim == 2 && p->r == 1 && pick_cp(p->dtype, q, rank) != nullptr;
    return pick(p->dtype, p->ndim, p->shape, p->r, q, s) != nullptr;
}

int launch_sweep(Plan* p, const SweepCall& c) {
    if (TbLaunchFn tb = pick_tb(p, c.q, c.stages, c.rank, c.L->wrap)) {
        if (c.band.empty()) return tb(p, c);
    }
    LaunchFn fn = c.rank > 0 ? (p->ndim == 2 && p->r == 1 && c.stages == 1 ? pick_cp(p->dtype, c.q, c.rank) : nullptr)
                             : pick(p->dtype, p->ndim, p->shape, p->r, c.q, c.stages);
    if (!fn)
        return set_error(STENCIL_EUNSUPPORTED, "no compiled sweep for ndim=" + std::to_string(p->ndim) +
                                                   " r=" + std::to_string(p->r) + " q=" + std::to_string(c.q) +
                                                   " stages=" + std::to_string(c.stages));
    return fn(p, c);
}

}  // namespace sb

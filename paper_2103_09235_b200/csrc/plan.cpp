// plan.cpp — plan creation, canonical taps, the coefficient-folding generator
// (SURVEY §8(a) a1/a2), buffer layouts and the evaluation-variant choice.
// Host only: nothing here calls CUDA.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <map>
#include <new>

#include <cuda_runtime.h>

#include "internal.hpp"

namespace sb {

static thread_local std::string g_err;

int set_error(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

static int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

// Canonical taps (R4): offsets in [-r, r]^d, lexicographic with the
// slowest axis outermost; STAR keeps offsets with at most one nonzero
// coordinate.
static std::vector<int> canonical_taps(int nd, int r, int shape) {
    std::vector<int> out;
    int o[3];
    int side = 2 * r + 1;
    int total = 1;
    for (int a = 0; a < nd; ++a) total *= side;
    for (int idx = 0; idx < total; ++idx) {
        int t = idx, nz = 0;
        for (int a = nd - 1; a >= 0; --a) {
            o[a] = t % side - r;
            t /= side;
            nz += o[a] != 0;
        }
        if (shape == STENCIL_STAR && nz > 1) continue;
        for (int a = 0; a < nd; ++a) out.push_back(o[a]);
    }
    return out;
}

// ---------------------------------------------------------------- folding
// lambda^(q) (Eq.2) by binary powering of sparse offset maps:
// lambda^(a+b) = lambda^(a) (*) lambda^(b) (the semigroup property),
// with (*) the convolution of coefficient maps (offsets add — composing two
// correlations, R3).  Independent of the oracle's repeated dense
// convolution; tests compare the two.
using Key = std::array<int, 3>;
using SparseMap = std::map<Key, double>;

static SparseMap sparse_conv(const SparseMap& a, const SparseMap& b) {
    SparseMap out;
    for (const auto& ea : a)
        for (const auto& eb : b) {
            Key k = {ea.first[0] + eb.first[0], ea.first[1] + eb.first[1], ea.first[2] + eb.first[2]};
            out[k] += ea.second * eb.second;
        }
    return out;
}

static SparseMap fold_sparse(const Plan* p, int q) {
    SparseMap base;
    int nd = p->ndim;
    for (size_t j = 0; j < p->w.size(); ++j) {
        Key k = {0, 0, 0};
        for (int a = 0; a < nd; ++a) k[a] = p->taps[j * nd + a];
        base[k] += p->w[j];
    }
    SparseMap result;
    bool have = false;
    SparseMap pw = base;
    int e = q;
    while (e > 0) {
        if (e & 1) {
            result = have ? sparse_conv(result, pw) : pw;
            have = true;
        }
        e >>= 1;
        if (e) pw = sparse_conv(pw, pw);
    }
    return result;
}

const std::vector<double>& folded(Plan* p, int q) {
    std::lock_guard<std::mutex> g(p->mu);
    auto it = p->lam.find(q);
    if (it != p->lam.end()) return it->second;
    SparseMap sm = fold_sparse(p, q);
    int nd = p->ndim, R = q * p->r, side = 2 * R + 1;
    int64_t total = 1;
    for (int a = 0; a < nd; ++a) total *= side;
    std::vector<double> dense((size_t)total, 0.0);
    for (const auto& e : sm) {
        int64_t idx = 0;
        for (int a = 0; a < nd; ++a) idx = idx * side + (e.first[a] + R);
        dense[(size_t)idx] = e.second;
    }
    return p->lam.emplace(q, std::move(dense)).first->second;
}

int support_size(int nd, int shape, int r, int q) {
    int R = q * r, side = 2 * R + 1, cnt = 0, total = 1;
    for (int a = 0; a < nd; ++a) total *= side;
    for (int idx = 0; idx < total; ++idx) {
        int t = idx, s = 0;
        bool ok = true;
        for (int a = 0; a < nd; ++a) {
            int o = t % side - R;
            t /= side;
            s += (std::abs(o) + r - 1) / r;
        }
        if (shape == STENCIL_STAR) ok = s <= q;
        cnt += ok;
    }
    return cnt;
}

// ---------------------------------------------------------------- variants
// Variant choice (the GPU form of the paper's profitability
// index Eq.3).  Measured on B200: one folded pass beats on-chip multi-stage
// evaluation whenever |supp lambda^(m)| <= 64 taps (e.g. 2D5P fp64 m=4, 41 taps:
// 930 vs 664 GStencil/s), because the single pass needs no intermediate
// hand-off; above that (2D9P m=4: 81 taps, 3D27P m=2: 125 taps) the divisor
// split (q, stages) with the fewest FMAs per point wins.
const LowRank& lowrank(Plan* p, int q) {
    const std::vector<double>& lam = folded(p, q);   // (takes the plan lock itself)
    std::lock_guard<std::mutex> g(p->mu);
    auto it = p->lowrank.find(q);
    if (it != p->lowrank.end()) return *it->second;
    LowRank* lr = new LowRank();
    p->lowrank[q] = lr;
    if (p->ndim != 2) return *lr;
    const int W = 2 * q * p->r + 1;
    lr->W = W;
    std::vector<double> R(lam);
    double amax = 0.0;
    for (double v : R) amax = std::max(amax, std::fabs(v));
    for (int k = 0; k < W; ++k) {
        int bi = 0, bj = 0;
        double best = 0.0;
        for (int i = 0; i < W; ++i)
            for (int j = 0; j < W; ++j)
                if (std::fabs(R[i * W + j]) > best) { best = std::fabs(R[i * W + j]); bi = i; bj = j; }
        if (best <= 1e-13 * amax) break;
        const double piv = R[bi * W + bj];
        std::vector<double> a(W), b(W);
        for (int i = 0; i < W; ++i) a[i] = R[i * W + bj];
        for (int j = 0; j < W; ++j) b[j] = R[bi * W + j] / piv;
        for (int i = 0; i < W; ++i)
            for (int j = 0; j < W; ++j) R[i * W + j] -= a[i] * b[j];
        lr->a.insert(lr->a.end(), a.begin(), a.end());
        lr->b.insert(lr->b.end(), b.begin(), b.end());
        ++lr->rank;
    }
    return *lr;
}

Variant choose_variant(Plan* p, int m) {
    if (m <= 1) return {1, 1};
    const int full = support_size(p->ndim, p->shape, p->r, m);
    // GPU form of the profitability index (Eq.3): the counterpart
    // evaluation costs rank * (W + W) FMAs per point (a horizontal fold per
    // counterpart, then the vertical fold of the counterparts, Eq.4-6), the
    // folded one |supp lambda^(m)|; take the counterparts when they are fewer
    // and a compiled rank exists (the paper's uniform 2D9P, m=2: 10 vs 25).
    if (p->ndim == 2 && p->r == 1 && p->counterparts && (m == 2 || m == 4)) {
        const LowRank& lr = lowrank(p, m);
        const int W = 2 * m * p->r + 1;
        if (lr.rank >= 1 && lr.rank <= STENCIL_MAX_COUNTERPARTS && 2 * W * lr.rank < full)
            return Variant{m, 1, lr.rank};
    }
    // 2D radius-1 FIXED plans: the warp-tile temporal block (tb2d.cuh, m single
    // steps per HBM round trip, stages = m) beats one folded pass from m = 4
    // (stars) / m = 3 (boxes) on -- measured on B200 (C2 m=4
    // 1140 vs 983, m=3 822 vs 1016; C3 m=3 1306 vs 983, m=2 963 vs 1428).
    if (p->ndim == 2 && p->r == 1 && p->boundary == STENCIL_BC_FIXED && tb_supported(p, 1, m) &&
        (m >= 4 || (m == 3 && p->shape == STENCIL_BOX)))
        return {1, m};
    // 3D radius-1 fp64 FIXED stars: the CTA-tile temporal block (tb3d.cuh, m single steps
    // per HBM round trip) beats one folded pass from m = 3 on -- measured on B200 (DESIGN.md
    // §5.8: C4 m=4 624 vs the folded m=2 571 GStencil/s; K=2 520)
    // (fp32 stars: from m = 4 on -- 512^3: K = 4 983 vs 940 for the folded m = 2 pass, K = 3 905)
    if (p->ndim == 3 && p->r == 1 && p->boundary == STENCIL_BC_FIXED && p->shape == STENCIL_STAR &&
        tb_supported(p, 1, m) && m >= (p->dtype == STENCIL_F64 ? 3 : 4))
        return {1, m};
    if (full <= 64) return {m, 1};
    Variant best = {m, 1};
    double best_cost = 1e30;
    for (int s = 1; s <= m; ++s) {
        if (m % s) continue;
        int q = m / s;
        double red = 1.0;
        if (s > 1) {
            double w = p->ndim == 3 ? 16.0 : 64.0;
            red = (w + 2.0 * (s - 1) * q * p->r) / w;
            if (p->ndim == 3) red *= (64.0 + 2.0 * (s - 1) * q * p->r) / 64.0;
        }
        // + a fixed cost per on-chip hand-off, calibrated on B200 (C3 m=4: 2 passes of
        // lambda^(2) 731 vs 4 single steps 623 GStencil/s although the latter has fewer FMAs)
        double cost = s * support_size(p->ndim, p->shape, p->r, q) * red + 12.0 * (s - 1);
        if (cost < best_cost) { best_cost = cost; best = {q, s}; }
    }
    return best;
}

// ---------------------------------------------------------------- layouts
// SURVEY §8(b) Layout: ring of r cells on every axis; the unit-stride axis has
// a left pad so interior x = 0 is 128-byte aligned and a pitch that is a
// multiple of 128 bytes.  Dist: axis 0 carries `halo` ghost planes per side.
Layout3 make_layout(const Plan* p, int rank, int nranks, int halo) {
    Layout3 L;
    L.ndim = p->ndim;
    L.r = p->r;
    L.esize = p->dtype == STENCIL_F64 ? 8 : 4;
    int64_t al = 128 / L.esize;
    int nd = p->ndim;
    // map user axes (slowest first) -> internal axes (0 stream, 1 y, 2 x)
    int64_t g[3] = {1, 1, 1};
    if (nd == 1) g[2] = p->dims[0];
    if (nd == 2) { g[0] = p->dims[0]; g[2] = p->dims[1]; }
    if (nd == 3) { g[0] = p->dims[0]; g[1] = p->dims[1]; g[2] = p->dims[2]; }
    for (int a = 0; a < 3; ++a) { L.gn[a] = g[a]; L.n[a] = g[a]; }
    bool used[3] = {nd >= 2, nd == 3, true};
    // PERIODIC: a ghost ring of G = STENCIL_MAX_FOLD * r cells per side on every
    // axis, refilled from the wrapped interior after every sweep (no physical
    // face, so no band); FIXED: the frozen r-ring.
    const bool per = p->boundary == STENCIL_BC_PERIODIC;
    const int64_t G = per ? (int64_t)STENCIL_MAX_FOLD * p->r : p->r;
    L.wrap = per;
    for (int a = 0; a < 3; ++a) {
        if (!used[a]) {
            L.phys_lo[a] = L.phys_hi[a] = 0;
            L.lo_valid[a] = L.hi_valid[a] = 0;
        } else {
            L.lo_valid[a] = L.hi_valid[a] = G;
            if (per) L.phys_lo[a] = L.phys_hi[a] = 0;
        }
    }
    // x
    L.origin[2] = round_up(G, al);
    L.ext[2] = round_up(L.origin[2] + g[2] + G, al);
    L.stride[2] = 1;
    // y
    if (used[1]) { L.origin[1] = G; L.ext[1] = g[1] + 2 * G; }
    else { L.origin[1] = 0; L.ext[1] = 1; }
    L.stride[1] = L.ext[2];
    // stream axis
    if (used[0]) {
        int64_t nloc = g[0] / nranks;
        L.n[0] = nloc;
        L.gofs0 = nloc * rank;
        int64_t h = nranks > 1 ? halo : G;
        if (h < G) h = G;
        L.origin[0] = h;
        L.ext[0] = nloc + 2 * h;
        L.phys_lo[0] = !per && rank == 0;
        L.phys_hi[0] = !per && rank == nranks - 1;
        L.lo_valid[0] = L.phys_lo[0] ? p->r : h;
        L.hi_valid[0] = L.phys_hi[0] ? p->r : h;
    } else {
        L.origin[0] = 0;
        L.ext[0] = 1;
    }
    L.stride[0] = L.ext[1] * L.stride[1];
    L.bytes = L.ext[0] * L.stride[0] * L.esize;
    return L;
}

void to_public(const Layout3& L, stencil_layout* out) {
    std::memset(out, 0, sizeof(*out));
    out->ndim = L.ndim;
    out->radius = L.r;
    int map[3];
    if (L.ndim == 1) { map[0] = 2; }
    if (L.ndim == 2) { map[0] = 0; map[1] = 2; }
    if (L.ndim == 3) { map[0] = 0; map[1] = 1; map[2] = 2; }
    for (int a = 0; a < L.ndim; ++a) {
        int i = map[a];
        out->interior[a] = L.n[i];
        out->extent[a] = L.ext[i];
        out->stride[a] = L.stride[i];
        out->origin[a] = L.origin[i];
    }
    out->elem_bytes = L.esize;
    out->bytes = L.bytes;
    out->global_offset0 = L.gofs0;
}

// fold_m = 0 ("auto"): per family, the fold that keeps the folded pass near the
// HBM roofline without making it FMA-bound (measured for the
// five BASELINE configs and the uniform 2D9P).
int auto_fold(Plan* p) {
    if (p->ndim == 1) return 2;
    if (p->ndim == 2 && p->r == 1) {
        if (p->counterparts && lowrank(p, 4).rank >= 1 && lowrank(p, 4).rank <= STENCIL_MAX_COUNTERPARTS &&
            2 * 9 * lowrank(p, 4).rank < support_size(2, p->shape, 1, 4))
            return 4;                                    // counterparts: 18 FMAs per point for 4 steps
        // temporal block: 8 steps per HBM round trip; 6 for fp64 stars (C2: K = 6 at 1936-1959
        // vs K = 8 at 1921-1960 GStencil/s in three calls, 0.83 of the HBM roofline per round trip)
        if (p->boundary == STENCIL_BC_FIXED && p->shape == STENCIL_STAR && p->dtype == STENCIL_F64 &&
            tb_supported(p, 1, 6))
            return 6;
        if (p->boundary == STENCIL_BC_FIXED && tb_supported(p, 1, 8)) return 8;
        if (p->shape == STENCIL_STAR) return 3;
        return 2;
    }
    if (p->ndim == 3 && p->r == 1) {
        if (p->shape == STENCIL_STAR && p->boundary == STENCIL_BC_FIXED && tb_supported(p, 1, 4))
            return 4;   // tb3d (fp64 C4: 635 vs 541-588 for m = 2; fp32 512^3: 983 vs 940)
        // 27-point box: the K = 2 temporal block (tb3d, BOX) -- C5 378 vs 355-368 GStencil/s for m = 1
        if (p->shape == STENCIL_BOX && p->boundary == STENCIL_BC_FIXED && p->dtype == STENCIL_F64 &&
            tb_supported(p, 1, 2))
            return 2;
        return p->shape == STENCIL_STAR ? 2 : 1;
    }
    return 1;
}

}  // namespace sb

using namespace sb;

extern "C" {

const char* stencil_last_error(void) { return g_err.c_str(); }

const char* stencil_version(void) { return "paper_2103_09235_b200 0.1 (sm_100a)"; }

int stencil_plan_create(stencil_plan* plan, int ndim, const int64_t* dims, int radius,
                        stencil_shape shape, const double* coeffs, int ncoeffs,
                        stencil_dtype dtype, stencil_boundary boundary) {
    g_err.clear();
    if (!plan) return set_error(STENCIL_EINVAL, "plan pointer is NULL");
    *plan = nullptr;
    if (ndim < 1 || ndim > 3) return set_error(STENCIL_EINVAL, "ndim must be 1..3");
    if (!dims) return set_error(STENCIL_EINVAL, "dims is NULL");
    for (int a = 0; a < ndim; ++a)
        if (dims[a] < 1 || dims[a] > (int64_t(1) << 31))
            return set_error(STENCIL_EINVAL, "every interior extent must be in [1, 2^31]");
    if (radius < 1 || radius > 4) return set_error(STENCIL_EINVAL, "radius must be 1..4");
    if (shape != STENCIL_STAR && shape != STENCIL_BOX) return set_error(STENCIL_EINVAL, "bad shape");
    if (dtype != STENCIL_F32 && dtype != STENCIL_F64) return set_error(STENCIL_EINVAL, "bad dtype");
    if (boundary != STENCIL_BC_FIXED && boundary != STENCIL_BC_PERIODIC)
        return set_error(STENCIL_EINVAL, "bad boundary");
    std::vector<int> taps = canonical_taps(ndim, radius, shape);
    int k = (int)taps.size() / ndim;
    if (!coeffs || ncoeffs != k)
        return set_error(STENCIL_EINVAL, "ncoeffs must equal the canonical tap count " + std::to_string(k));
    for (int j = 0; j < k; ++j)
        if (!std::isfinite(coeffs[j])) return set_error(STENCIL_EINVAL, "coefficients must be finite");
    Plan* p = new (std::nothrow) Plan();
    if (!p) return set_error(STENCIL_ENOMEM, "out of host memory");
    p->ndim = ndim;
    for (int a = 0; a < 3; ++a) p->dims[a] = a < ndim ? dims[a] : 1;
    p->r = radius;
    p->shape = shape;
    p->dtype = dtype;
    p->boundary = boundary;
    p->taps = taps;
    p->w.assign(coeffs, coeffs + k);
    *plan = reinterpret_cast<stencil_plan>(p);
    return STENCIL_OK;
}

int stencil_plan_destroy(stencil_plan plan) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (p) {
        for (const auto& r : p->recs) {
            cudaEventDestroy((cudaEvent_t)r.a);
            cudaEventDestroy((cudaEvent_t)r.b);
        }
        for (void* e : p->event_pool) cudaEventDestroy((cudaEvent_t)e);
        if (p->sched) cudaFree(p->sched);
        for (void* e : p->pipe_ev)
            if (e) cudaEventDestroy((cudaEvent_t)e);
        if (p->h2d_stream) cudaStreamDestroy((cudaStream_t)p->h2d_stream);
        if (p->d2h_stream) cudaStreamDestroy((cudaStream_t)p->d2h_stream);
        for (auto& kv : p->lowrank) delete kv.second;
    }
    delete p;
    return STENCIL_OK;
}

int stencil_plan_layout(stencil_plan plan, stencil_layout* out) {
    if (!plan || !out) return set_error(STENCIL_EINVAL, "NULL argument");
    to_public(make_layout(reinterpret_cast<Plan*>(plan), 0, 1, 0), out);
    return STENCIL_OK;
}

int stencil_plan_ntaps(stencil_plan plan, int* ntaps) {
    if (!plan || !ntaps) return set_error(STENCIL_EINVAL, "NULL argument");
    Plan* p = reinterpret_cast<Plan*>(plan);
    *ntaps = (int)p->w.size();
    return STENCIL_OK;
}

int stencil_plan_taps(stencil_plan plan, int* offsets, int cap) {
    if (!plan || !offsets) return set_error(STENCIL_EINVAL, "NULL argument");
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (cap < (int)p->taps.size()) return set_error(STENCIL_EINVAL, "capacity too small");
    std::copy(p->taps.begin(), p->taps.end(), offsets);
    return STENCIL_OK;
}

int stencil_plan_fold_coeffs(stencil_plan plan, int m, double* dense, int64_t cap) {
    if (!plan || !dense) return set_error(STENCIL_EINVAL, "NULL argument");
    if (m < 1) return set_error(STENCIL_EINVAL, "fold_m must be >= 1");
    if (m > STENCIL_MAX_FOLD) return set_error(STENCIL_EUNSUPPORTED, "fold_m > STENCIL_MAX_FOLD");
    Plan* p = reinterpret_cast<Plan*>(plan);
    const std::vector<double>& lam = folded(p, m);
    if (cap < (int64_t)lam.size()) return set_error(STENCIL_EINVAL, "capacity too small");
    std::copy(lam.begin(), lam.end(), dense);
    return STENCIL_OK;
}

int stencil_plan_fold_rank(stencil_plan plan, int m, int* rank, double* a, double* b, int64_t cap) {
    if (!plan || !rank) return set_error(STENCIL_EINVAL, "NULL argument");
    if (m < 1) return set_error(STENCIL_EINVAL, "fold_m must be >= 1");
    if (m > STENCIL_MAX_FOLD) return set_error(STENCIL_EUNSUPPORTED, "fold_m > STENCIL_MAX_FOLD");
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (p->ndim != 2) return set_error(STENCIL_EUNSUPPORTED, "counterpart decomposition is 2D");
    const LowRank& lr = lowrank(p, m);
    *rank = lr.rank;
    if (a || b) {
        if (cap < (int64_t)lr.a.size()) return set_error(STENCIL_EINVAL, "capacity too small");
        if (a) std::copy(lr.a.begin(), lr.a.end(), a);
        if (b) std::copy(lr.b.begin(), lr.b.end(), b);
    }
    return STENCIL_OK;
}

int stencil_plan_perturb_fold(stencil_plan plan, int m, int64_t index, double delta) {
    if (!plan) return set_error(STENCIL_EINVAL, "NULL argument");
    if (m < 1 || m > STENCIL_MAX_FOLD) return set_error(STENCIL_EINVAL, "bad fold_m");
    Plan* p = reinterpret_cast<Plan*>(plan);
    std::vector<double>& lam = const_cast<std::vector<double>&>(folded(p, m));
    if (index < 0 || index >= (int64_t)lam.size()) return set_error(STENCIL_EINVAL, "index out of range");
    std::lock_guard<std::mutex> g(p->mu);
    lam[(size_t)index] += delta;
    auto it = p->lowrank.find(m);   // the counterparts derive from lambda: recompute on demand
    if (it != p->lowrank.end()) {
        delete it->second;
        p->lowrank.erase(it);
    }
    return STENCIL_OK;
}

int stencil_plan_auto_fold(stencil_plan plan, int* fold_m) {
    if (!plan || !fold_m) return set_error(STENCIL_EINVAL, "NULL argument");
    *fold_m = sb::auto_fold(reinterpret_cast<Plan*>(plan));
    return STENCIL_OK;
}

int stencil_plan_set_counterparts(stencil_plan plan, int enable) {
    if (!plan) return set_error(STENCIL_EINVAL, "NULL argument");
    reinterpret_cast<Plan*>(plan)->counterparts = enable != 0;
    return STENCIL_OK;
}

int stencil_plan_variant(stencil_plan plan, int m, int* q, int* stages, int* rank) {
    if (!plan || !q || !stages || !rank) return set_error(STENCIL_EINVAL, "NULL argument");
    if (m < 1) return set_error(STENCIL_EINVAL, "fold_m must be >= 1");
    if (m > STENCIL_MAX_FOLD) return set_error(STENCIL_EUNSUPPORTED, "fold_m > STENCIL_MAX_FOLD");
    Variant v = choose_variant(reinterpret_cast<Plan*>(plan), m);
    *q = v.q;
    *stages = v.stages;
    *rank = v.rank;
    return STENCIL_OK;
}

int stencil_workspace_size(stencil_plan plan, int64_t* bytes) {
    if (!plan || !bytes) return set_error(STENCIL_EINVAL, "NULL argument");
    *bytes = make_layout(reinterpret_cast<Plan*>(plan), 0, 1, 0).bytes;
    return STENCIL_OK;
}

int stencil_plan_layout_dist(stencil_plan plan, int rank, int nranks, int halo,
                             stencil_layout* out) {
    if (!plan || !out) return set_error(STENCIL_EINVAL, "NULL argument");
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (p->ndim < 2) return set_error(STENCIL_EUNSUPPORTED, "dist layouts need ndim >= 2");
    if (p->boundary != STENCIL_BC_FIXED) return set_error(STENCIL_EUNSUPPORTED, "dist layouts need a FIXED boundary");
    if (nranks < 1 || rank < 0 || rank >= nranks) return set_error(STENCIL_EINVAL, "bad rank/nranks");
    if (halo < p->r) return set_error(STENCIL_EINVAL, "halo must be >= radius");
    if (p->dims[0] % nranks) return set_error(STENCIL_EINVAL, "axis-0 extent not divisible by nranks");
    if (nranks > 1 && p->dims[0] / nranks < halo)
        return set_error(STENCIL_EINVAL, "slab thinner than the halo");
    to_public(make_layout(p, rank, nranks, halo), out);
    return STENCIL_OK;
}

int stencil_plan_last_launches(stencil_plan plan, int64_t* launches) {
    if (!plan || !launches) return set_error(STENCIL_EINVAL, "NULL argument");
    *launches = reinterpret_cast<Plan*>(plan)->last_launches;
    return STENCIL_OK;
}

}  // extern "C"

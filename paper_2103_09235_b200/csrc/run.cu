// run.cu — orchestration of a run: frozen-ring init,
// floor(T/m) folded sweeps + T mod m single steps in Jacobi ping-pong
// (P:410), the main-region sweep plus the exact boundary band per sweep, and
// the slab-decomposed multi-GPU run with a per-sweep halo exchange
// (NCCL send/recv on a comm stream, overlapped with the interior).
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <thread>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include <nvtx3/nvToolsExt.h>

#include "internal.hpp"
#include "sweep_params.cuh"

namespace sb {

// ------------------------------------------------------------------ tracing
// NVTX ranges (header-only NVTX 3: free unless a profiler is attached) around
// every run and every sweep, so nsys/ncu timelines show the library's phases.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

// ------------------------------------------------------------------ timing
static void* take_event(Plan* p) {
    if (!p->event_pool.empty()) {
        void* e = p->event_pool.back();
        p->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    return e;
}

TimedScope::TimedScope(Plan* p_, void* s, int k, int64_t b, int64_t f)
    : p(p_), stream(s), kind(k), bytes(b), fmas(f) {
    if (!p->timing) return;
    a = take_event(p);
    if (a) cudaEventRecord((cudaEvent_t)a, (cudaStream_t)stream);
}

TimedScope::~TimedScope() {
    if (!p->timing || !a) return;
    void* b = take_event(p);
    if (!b) return;
    cudaEventRecord((cudaEvent_t)b, (cudaStream_t)stream);
    p->recs.push_back({a, b, kind, bytes, fmas});
}

static int ensure_device(Plan* p) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_error(e, "cudaGetDevice");
    if (p->device != dev || p->sm_count <= 0) {
        if (p->device >= 0 && p->device != dev && p->sched) {
            // the schedule scratch lives on the previous device
            cudaFree(p->sched);
            p->sched = nullptr;
            p->sched_words = 0;
        }
        int sms = 0;
        e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return cuda_error(e, "cudaDeviceGetAttribute");
        p->sm_count = sms;
        p->device = dev;
    }
    return STENCIL_OK;
}

// Partition the local interior into the region where lambda^(m) is valid (at
// distance >= (m-1) r from every FIXED face) and the band shell around it.
static void split_band(const Layout3& L, int m, Box* main, std::vector<Box>* band) {
    Box in;
    for (int a = 0; a < 3; ++a) { in.lo[a] = 0; in.hi[a] = L.n[a]; }
    const int64_t b = (int64_t)(m - 1) * L.r;
    band->clear();
    for (int a = 0; a < 3; ++a) {
        int64_t bl = L.phys_lo[a] ? b : 0, bh = L.phys_hi[a] ? b : 0;
        if (bl > 0) {
            Box s = in;
            s.hi[a] = std::min(in.hi[a], in.lo[a] + bl);
            if (!s.empty()) band->push_back(s);
            in.lo[a] = s.hi[a];
        }
        if (bh > 0) {
            Box s = in;
            s.lo[a] = std::max(in.lo[a], in.hi[a] - bh);
            if (!s.empty()) band->push_back(s);
            in.hi[a] = s.lo[a];
        }
    }
    *main = in;
}

static Box clip0(Box b, int64_t z0, int64_t z1) {
    b.lo[0] = std::max(b.lo[0], z0);
    b.hi[0] = std::min(b.hi[0], z1);
    return b;
}

struct SweepSpec {
    int m;          // steps in this sweep
    Variant v;      // evaluation of the main region
};

// Enqueue one sweep restricted to axis-0 range [z0, z1). Returns launches or <0.
static int enqueue_sweep(Plan* p, const Layout3& L, const void* src, void* dst, const SweepSpec& s,
                         int64_t z0, int64_t z1, void* stream, void* peer_lo = nullptr, void* peer_hi = nullptr,
                         int peer_h = 0) {
    NvtxRange nv(s.v.rank > 0 ? "stencil sweep (counterparts)" : s.v.stages > 1 ? "stencil sweep (on-chip stages)"
                                                                               : "stencil sweep (folded)");
    Box mainb;
    std::vector<Box> band;
    // The on-chip stepwise block (Q = 1, S = m stages) is exact up to the FIXED
    // faces by itself: intermediate ring cells are reloaded from u0 (R1), so it
    // takes the whole interior and no band is needed.
    const bool stepwise_exact = s.v.q == 1 && s.v.rank == 0 && s.v.stages == s.m;
    split_band(L, stepwise_exact ? 1 : s.m, &mainb, &band);
    int launches = 0;
    SweepCall sc;
    sc.src = src;
    sc.dst = dst;
    sc.L = &L;
    Box mb = clip0(mainb, z0, z1);
    if (!mb.empty()) sc.boxes.push_back(mb);
    sc.q = s.v.q;
    sc.stages = s.v.stages;
    sc.rank = s.v.rank;
    sc.peer_lo = peer_lo;
    sc.peer_hi = peer_hi;
    sc.peer_h = (peer_lo || peer_hi) ? peer_h : 0;
    std::vector<double> packed;
    if (s.v.rank > 0) {   // counterparts: a_0..a_{rank-1} | b_0..b_{rank-1}
        const LowRank& lr = lowrank(p, s.v.q);
        packed.assign(lr.a.begin(), lr.a.begin() + (size_t)s.v.rank * lr.W);
        packed.insert(packed.end(), lr.b.begin(), lr.b.begin() + (size_t)s.v.rank * lr.W);
        sc.coef = &packed;
    } else {
        sc.coef = &folded(p, s.v.q);
    }
    sc.stream = stream;
#ifdef STENCIL_TUNING_BUILD
    // STENCIL_DEBUG_NO_BAND=1 drops the band (WRONG results near FIXED faces):
    // only in tuning builds (tools/tunebuild.py), to measure what the band costs
    static const bool no_band = getenv("STENCIL_DEBUG_NO_BAND") != nullptr;
#else
    constexpr bool no_band = false;
#endif
    if (s.m > 1 && !no_band) {
        for (const Box& b : band) {
            Box c = clip0(b, z0, z1);
            if (!c.empty()) sc.band.push_back(c);
        }
        sc.band_m = s.m;
    }
    int rc;
    {
        int64_t pts = mb.volume(), bpts = 0;
        for (const Box& b : sc.band) bpts += b.volume();
        const int64_t per_pt = s.v.rank > 0 ? (int64_t)s.v.rank * 2 * (2 * s.v.q * p->r + 1)
                                            : (int64_t)s.v.stages * support_size(p->ndim, p->shape, p->r, s.v.q);
        TimedScope ts(p, stream, 0, 2 * L.esize * (pts + bpts), pts * per_pt + bpts * s.m * (int64_t)p->w.size());
        rc = launch_sweep(p, sc);
    }
    if (rc < 0) return rc;
    launches += rc;
    return launches;
}

static int resolve_variant(Plan* p, int m, int stages, Variant* v) {
    if (m == 1) { *v = {1, 1}; return STENCIL_OK; }
    if (stages == 0 || stages == 1) {
        Variant c = choose_variant(p, m);
        if (c.rank > 0 && sweep_supported(p, c.q, 1, c.rank)) { *v = c; return STENCIL_OK; }   // one pass, counterparts
    }
    if (stages == 0) {
        *v = choose_variant(p, m);
        v->rank = 0;
        if (!sweep_supported(p, v->q, v->stages)) {
            // fall back to any compiled split of m
            for (int s = 1; s <= m; ++s)
                if (m % s == 0 && sweep_supported(p, m / s, s)) { *v = {m / s, s}; return STENCIL_OK; }
            return set_error(STENCIL_EUNSUPPORTED, "no compiled evaluation for fold_m=" + std::to_string(m));
        }
        return STENCIL_OK;
    }
    if (stages < 1 || m % stages) return set_error(STENCIL_EINVAL, "stages must divide fold_m");
    *v = {m / stages, stages};
    if (!sweep_supported(p, v->q, v->stages))
        return set_error(STENCIL_EUNSUPPORTED, "no compiled sweep for fold_m=" + std::to_string(m) +
                                                   " stages=" + std::to_string(stages));
    return STENCIL_OK;
}

// R10 refined: T = nf * m + nr steps run as nf sweeps of lambda^(m) and, when
// nr > 1, ONE sweep of lambda^(nr) (one HBM pass instead of nr); nr single
// steps only when no evaluation of fold nr is compiled.
static void remainder_plan(Plan* p, int64_t T, int m, int64_t* n, int* mr, Variant* vr) {
    const int64_t nf = T / m, nr = T % m;
    *mr = 1;
    *vr = Variant{1, 1};
    if (nr > 1) {
        Variant v;
        const std::string keep = stencil_last_error();
        if (resolve_variant(p, (int)nr, 0, &v) == STENCIL_OK) {
            *mr = (int)nr;
            *vr = v;
            *n = nf + 1;
            return;
        }
        set_error(STENCIL_OK, keep);   // the fallback is not an error
    }
    *n = nf + nr;
}

static bool misaligned(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 127) != 0; }

static int check_run_args(Plan* p, const void* in, void* out, int64_t T, int m, void* ws) {
    if (!p) return set_error(STENCIL_EINVAL, "plan is NULL");
    if (T < 0) return set_error(STENCIL_EINVAL, "T must be >= 0");
    if (m < 1) return set_error(STENCIL_EINVAL, "fold_m must be >= 1");
    if (m > STENCIL_MAX_FOLD) return set_error(STENCIL_EUNSUPPORTED, "fold_m > STENCIL_MAX_FOLD");
    if (!in || !out) return set_error(STENCIL_EINVAL, "in/out is NULL");
    if (in == out || (ws && (ws == in || ws == out))) return set_error(STENCIL_EINVAL, "in, out and workspace must not alias");
    if (misaligned(in) || misaligned(out) || (ws && misaligned(ws)))
        return set_error(STENCIL_EINVAL, "buffers must be 128-byte aligned");
    if (p->boundary == STENCIL_BC_PERIODIC && (int64_t)m * p->r > (int64_t)STENCIL_MAX_FOLD * p->r)
        return set_error(STENCIL_EUNSUPPORTED, "PERIODIC: fold_m * r beyond the ghost ring");
    return STENCIL_OK;
}

// ------------------------------------------------------------------ 1D
static int run_1d(Plan* p, const Layout3& L, const void* in, void* out, int64_t T, int m, int stages, void* ws,
                  void* stream) {
    // steps per launch: the warp window (32*V cells) keeps at least half of its
    // cells as outputs, i.e. a halo H = TB*r <= 8*V; a multiple of m
    // (STENCIL_1D_HMAX overrides the 8*V halo bound: tuning)
    const int V = onchip1d_cells_per_lane(p->r, m, L.wrap);
#ifdef STENCIL_TUNING_BUILD
    static const int64_t hforce = [] {   // (tuning builds only)
        const char* e = getenv("STENCIL_1D_HMAX");
        return e ? (int64_t)atoll(e) : (int64_t)0;
    }();
#else
    constexpr int64_t hforce = 0;
#endif
    const int64_t hmax = std::min<int64_t>(hforce > 0 ? hforce : 8 * V, 16 * V - 1) / p->r;
    int64_t cap = std::max<int64_t>(m, hmax / m * m);
    int64_t nl = (T + cap - 1) / cap;
    cap = std::max<int64_t>(m, ((T + nl - 1) / nl + m - 1) / m * m);   // balance the launches
    nl = (T + cap - 1) / cap;
    if (nl >= 2 && !ws) return set_error(STENCIL_EINVAL, "workspace required");
    bool force_step = (stages == m && m > 1);
    int launches = 0;
    int rc = 0;
    void* bufs[2] = {out, ws};
    int64_t left = T;
    const int64_t k = (int64_t)p->w.size();
    for (int64_t j = 1; j <= nl; ++j) {
        int64_t tb = std::min(cap, left);
        left -= tb;
        const void* src = j == 1 ? in : bufs[(nl - j + 1) % 2];
        void* dst = bufs[(nl - j) % 2];
        {
            TimedScope ts(p, stream, 0, 2 * L.esize * L.n[2],
                          L.n[2] * (force_step ? tb * k : (tb / m) * support_size(1, p->shape, p->r, m) +
                                                              (tb % m) * k));
            rc = launch_1d(p, src, dst, &L, tb, m, force_step ? 1 : 0, stream);
        }
        if (rc < 0) return rc;
        launches += rc;
    }
    if (L.wrap) {   // PERIODIC: out's ghosts = its wrapped interior
        rc = launch_wrap_fill(p, out, &L, stream);
        if (rc < 0) return rc;
        launches += rc;
    }
    p->last_launches = launches;
    return STENCIL_OK;
}

int run_single(Plan* p, const void* in, void* out, int64_t T, int m, int stages, void* ws, void* stream) {
    NvtxRange nv("stencil_run");
    if (p && m == 0) m = auto_fold(p);
    int rc = check_run_args(p, in, out, T, m, ws);
    if (rc) return rc;
    rc = ensure_device(p);
    if (rc) return rc;
    Layout3 L = make_layout(p, 0, 1, 0);
    cudaStream_t st = (cudaStream_t)stream;
    if (T == 0) {
        cudaError_t e = cudaMemcpyAsync(out, in, L.bytes, cudaMemcpyDeviceToDevice, st);
        p->last_launches = 0;
        return e == cudaSuccess ? STENCIL_OK : cuda_error(e, "cudaMemcpyAsync");
    }
    if (p->ndim == 1) return run_1d(p, L, in, out, T, m, stages, ws, stream);
    Variant v{1, 1};
    if (T >= m) {   // (T < m: only the remainder sweep runs)
        rc = resolve_variant(p, m, stages, &v);
        if (rc) return rc;
    }
    const int64_t nf = T / m;
    int64_t n;
    int mr;
    Variant vr;
    remainder_plan(p, T, m, &n, &mr, &vr);
    if (L.wrap) {
        // PERIODIC (NEXT-4): copy `in` (never written) into the buffer the
        // ping-pong starts from, fill its ghosts from the wrapped interior, then
        // after every sweep refill the ghosts of its output.  No band: there is
        // no physical face, so lambda^(m) is valid everywhere.
        if (!ws) return set_error(STENCIL_EINVAL, "workspace required for PERIODIC runs");
        void* bufs[2] = {out, ws};
        void* start = bufs[n % 2];   // so that sweep n writes `out`
        cudaError_t e = cudaMemcpyAsync(start, in, L.bytes, cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) return cuda_error(e, "cudaMemcpyAsync");
        int launches = 0;
        rc = launch_wrap_fill(p, start, &L, stream);
        if (rc < 0) return rc;
        launches += rc;
        for (int64_t j = 1; j <= n; ++j) {
            SweepSpec s;
            s.m = j <= nf ? m : mr;
            s.v = j <= nf ? v : vr;
            const void* src = bufs[(n - j + 1) % 2];
            void* dst = bufs[(n - j) % 2];
            rc = enqueue_sweep(p, L, src, dst, s, 0, L.n[0], stream);
            if (rc < 0) return rc;
            launches += rc;
            rc = launch_wrap_fill(p, dst, &L, stream);
            if (rc < 0) return rc;
            launches += rc;
        }
        p->last_launches = launches;
        return STENCIL_OK;
    }
    if (n >= 2 && !ws) return set_error(STENCIL_EINVAL, "workspace required when more than one sweep runs");
    int launches = 0;
    rc = launch_ring_copy(p, in, out, &L, stream);
    if (rc < 0) return rc;
    launches += rc;
    if (n >= 2) {
        rc = launch_ring_copy(p, in, ws, &L, stream);
        if (rc < 0) return rc;
        launches += rc;
    }
    void* bufs[2] = {out, ws};
    for (int64_t j = 1; j <= n; ++j) {
        SweepSpec s;
        s.m = j <= nf ? m : mr;
        s.v = j <= nf ? v : vr;
        const void* src = j == 1 ? in : bufs[(n - j + 1) % 2];
        void* dst = bufs[(n - j) % 2];
        rc = enqueue_sweep(p, L, src, dst, s, 0, L.n[0], stream);
        if (rc < 0) return rc;
        launches += rc;
    }
    p->last_launches = launches;
    return STENCIL_OK;
}

// ------------------------------------------------------------------ NCCL (dlopen)
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    bool ok = false;
    std::string why;
};

static NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) { api.why = std::string("cannot dlopen libnccl.so.2: ") + dlerror(); return; }
#define LOAD(name, field)                                                           \
    api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name));              \
    if (!api.field) { api.why = std::string("missing NCCL symbol ") + name; return; }
        LOAD("ncclGetUniqueId", GetUniqueId);
        LOAD("ncclCommInitRank", CommInitRank);
        LOAD("ncclCommDestroy", CommDestroy);
        LOAD("ncclSend", Send);
        LOAD("ncclRecv", Recv);
        LOAD("ncclGroupStart", GroupStart);
        LOAD("ncclGroupEnd", GroupEnd);
        LOAD("ncclGetErrorString", GetErrorString);
        LOAD("ncclCommGetAsyncError", CommGetAsyncError);
        LOAD("ncclCommAbort", CommAbort);
#undef LOAD
        api.ok = true;
    });
    return api;
}

static int nccl_error(ncclResult_t r, const char* what) {
    NcclApi& a = nccl();
    return set_error(STENCIL_ENCCL, std::string(what) + ": " + (a.GetErrorString ? a.GetErrorString(r) : "?"));
}

// Stream memory operations and address-range query (driver API, resolved at
// run time like the TMA encoder): the fused exchange's inter-GPU sweep flags.
struct DrvMemOps {
    CUresult (*wait32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
    CUresult (*write32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
    CUresult (*range)(CUdeviceptr*, size_t*, CUdeviceptr) = nullptr;
};
static DrvMemOps& drv() {
    static DrvMemOps d;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            d.wait32 = reinterpret_cast<decltype(d.wait32)>(f);
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            d.write32 = reinterpret_cast<decltype(d.write32)>(f);
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            d.range = reinterpret_cast<decltype(d.range)>(f);
    });
    return d;
}

}  // namespace sb

struct stencil_comm_s {
    ncclComm_t comm = nullptr;
    int rank = 0, nranks = 1;
    cudaStream_t cstream = nullptr;
    cudaEvent_t evA = nullptr, evC = nullptr;
    // fused peer-store exchange (NEXT-2): this rank's two ping-pong buffers, the
    // neighbours' buffers mapped through CUDA IPC, and sweep flags: flags[0] is
    // written by rank - 1, flags[1] by rank + 1 (stream memory operations).
    bool peer = false;
    void* buf[2] = {nullptr, nullptr};
    void* nbuf[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};   // [side 0 = lo, 1 = hi][buffer]
    void* nbase[2][3] = {{nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr}};   // opened IPC bases
    uint32_t* flags = nullptr;
    uint32_t* nflag[2] = {nullptr, nullptr};   // neighbour's flag slot this rank writes
    uint32_t epoch = 0;
    bool failed = false;   // NCCL comm aborted (async error or stencil_comm_wait timeout)
};

namespace sb {

// Exchange planes between neighbours: rank g sends its planes [0,hx) to g-1
// and [n0-hx, n0) to g+1; it receives into [-hx, 0) and [n0, n0+hx).
struct Exchange {
    virtual ~Exchange() {}
    virtual int begin(int j, void* stream) = 0;   // after phase A of sweep j is enqueued
    virtual int end(void* stream) = 0;            // before sweep j+1
};

static int dist_layout_check(Plan* p, int rank, int nranks, int halo, int m, Layout3* L) {
    if (p->ndim < 2) return set_error(STENCIL_EUNSUPPORTED, "dist runs need ndim >= 2");
    if (p->boundary != STENCIL_BC_FIXED) return set_error(STENCIL_EUNSUPPORTED, "dist runs need a FIXED boundary");
    if (p->dims[0] % nranks) return set_error(STENCIL_EINVAL, "axis-0 extent not divisible by nranks");
    if (halo < m * p->r) return set_error(STENCIL_EINVAL, "halo must be >= fold_m * radius");
    if (nranks > 1 && p->dims[0] / nranks < halo) return set_error(STENCIL_EINVAL, "slab thinner than the halo");
    *L = make_layout(p, rank, nranks, halo);
    return STENCIL_OK;
}

// One rank's share of a sweep, split in phase A (the planes neighbours need)
// and phase B (the rest).
static int sweep_phase(Plan* p, const Layout3& L, const void* src, void* dst, const SweepSpec& s, int rank,
                       int nranks, int64_t hx, int phase, void* stream) {
    const int64_t n0 = L.n[0];
    bool has_lo = rank > 0, has_hi = rank < nranks - 1;
    if (nranks == 1 || 2 * hx >= n0) {
        if (phase == 0) return enqueue_sweep(p, L, src, dst, s, 0, n0, stream);
        return 0;
    }
    int launches = 0, rc;
    if (phase == 0) {
        if (has_lo) {
            rc = enqueue_sweep(p, L, src, dst, s, 0, hx, stream);
            if (rc < 0) return rc;
            launches += rc;
        }
        if (has_hi) {
            rc = enqueue_sweep(p, L, src, dst, s, n0 - hx, n0, stream);
            if (rc < 0) return rc;
            launches += rc;
        }
        return launches;
    }
    int64_t z0 = has_lo ? hx : 0, z1 = has_hi ? n0 - hx : n0;
    return enqueue_sweep(p, L, src, dst, s, z0, z1, stream);
}

static size_t plane_bytes(const Layout3& L) { return (size_t)L.stride[0] * L.esize; }

}  // namespace sb

// ------------------------------------------------------------------ fused exchange (NEXT-2)
// One launch per sweep over the whole slab: the sweep kernel stores the
// outputs of its first/last hx planes a second time, straight into the
// neighbours' ghost planes of the same ping-pong parity (CUDA IPC peer
// pointers over NVLink), so the transfer overlaps the math tile by tile and
// there is no NCCL kernel.  Ordering between GPUs: after sweep j a rank writes
// the sweep counter into each neighbour's flag (cuStreamWriteValue32, which
// fences the kernel's stores first); before sweep j+1 it waits until both
// neighbours' counters reached j (cuStreamWaitValue32, a stream-level wait, no
// spinning kernel).  That covers both hazards: the ghosts read by sweep j+1
// were written by the neighbours' sweep j, and a neighbour's sweep j+1 writes
// into the buffer this rank read during sweep j.
static int run_dist_peer(sb::Plan* p, stencil_comm_s* c, const sb::Layout3& L, const void* in_local, void* out_local,
                         void* ws, int64_t n, int64_t nf, int fold_m, sb::Variant v, int mr, sb::Variant vr, int64_t hx,
                         void* stream) {
    using namespace sb;
    // One fixed order on every rank: a rank's peer stores go into
    // the neighbour's buffer of the same REGISTERED index, so all ranks must
    // use buf0 as `out` and buf1 as the workspace.
    if (!(out_local == c->buf[0] && (n < 2 || ws == c->buf[1])))
        return set_error(STENCIL_EINVAL, "peer comm: out must be buf0 and workspace buf1 (the registered order)");
    const int bo = 0;   // registered index of `out`
    DrvMemOps& d = drv();
    if (!d.wait32 || !d.write32) return set_error(STENCIL_ECUDA, "cuStreamWaitValue32/WriteValue32 unavailable");
    CUstream cs = (CUstream)stream;
    int launches = 0;
    // ring/pads only: the interior cells of the ghost planes belong to the
    // neighbours' peer stores (they may already be writing them)
    int rc = launch_ring_copy(p, in_local, out_local, &L, stream, true);
    if (rc < 0) return rc;
    launches += rc;
    if (n >= 2) {
        rc = launch_ring_copy(p, in_local, ws, &L, stream, true);
        if (rc < 0) return rc;
        launches += rc;
    }
    const bool has_lo = c->rank > 0, has_hi = c->rank < c->nranks - 1;
    void* bufs[2] = {out_local, ws};
    for (int64_t j = 1; j <= n; ++j) {
        SweepSpec s;
        s.m = j <= nf ? fold_m : mr;
        s.v = j <= nf ? v : vr;
        const void* src = j == 1 ? in_local : bufs[(n - j + 1) % 2];
        const int di = (int)((n - j) % 2);           // 0 = out, 1 = ws
        const int reg = di == 0 ? bo : 1 - bo;       // registered index of dst
        {   // the neighbours finished sweep j-1 (for j = 1: their previous run)
            const uint32_t want = c->epoch + (uint32_t)(j - 1);
            if (has_lo && d.wait32(cs, (CUdeviceptr)(c->flags + 0), want, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
                return set_error(STENCIL_ECUDA, "cuStreamWaitValue32");
            if (has_hi && d.wait32(cs, (CUdeviceptr)(c->flags + 1), want, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
                return set_error(STENCIL_ECUDA, "cuStreamWaitValue32");
        }
        // every sweep stores its boundary planes into the neighbours' ghosts,
        // the last one included: after the run out_local's ghost planes hold
        // the neighbours' final planes, so a copy of out_local is a complete
        // in_local for a chained run (no separate exchange needed)
        rc = enqueue_sweep(p, L, src, bufs[di], s, 0, L.n[0], stream, has_lo ? c->nbuf[0][reg] : nullptr,
                           has_hi ? c->nbuf[1][reg] : nullptr, (int)hx);
        if (rc < 0) return rc;
        launches += rc;
        {   // every sweep signals, the last one included (orders the next run)
            const uint32_t val = c->epoch + (uint32_t)j;
            if (has_lo && d.write32(cs, (CUdeviceptr)c->nflag[0], val, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
                return set_error(STENCIL_ECUDA, "cuStreamWriteValue32");
            if (has_hi && d.write32(cs, (CUdeviceptr)c->nflag[1], val, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
                return set_error(STENCIL_ECUDA, "cuStreamWriteValue32");
        }
    }
    c->epoch += (uint32_t)n;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_error(e, "run_dist_peer");
    p->last_launches = launches;
    return STENCIL_OK;
}

using namespace sb;

extern "C" {

int stencil_fill_random(stencil_plan plan, void* buf, uint64_t seed, void* stream) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (!p || !buf) return set_error(STENCIL_EINVAL, "NULL argument");
    int rc = ensure_device(p);
    if (rc) return rc;
    Layout3 L = make_layout(p, 0, 1, 0);
    rc = launch_fill(p, buf, &L, seed, stream);
    return rc < 0 ? rc : STENCIL_OK;
}

int stencil_fill_random_dist(stencil_plan plan, int rank, int nranks, int halo, void* buf, uint64_t seed,
                             void* stream) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (!p || !buf) return set_error(STENCIL_EINVAL, "NULL argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return set_error(STENCIL_EINVAL, "bad rank/nranks");
    Layout3 L;
    int rc = dist_layout_check(p, rank, nranks, halo, 1, &L);
    if (rc) return rc;
    rc = ensure_device(p);
    if (rc) return rc;
    rc = launch_fill(p, buf, &L, seed, stream);
    return rc < 0 ? rc : STENCIL_OK;
}

int stencil_plan_set_schedule(stencil_plan plan, int chunk, int min_steal, int max_ctas) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (!p || chunk < 0 || min_steal < 0 || max_ctas < 0) return set_error(STENCIL_EINVAL, "bad argument");
    p->sched_chunk = chunk;
    p->sched_min_steal = min_steal;
    p->sched_max_ctas = max_ctas;
    return STENCIL_OK;
}

int stencil_plan_sched_stats(stencil_plan plan, int64_t* grabs, int64_t* steals, int reset) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (!p || !grabs || !steals) return set_error(STENCIL_EINVAL, "NULL argument");
    *grabs = 0;
    *steals = 0;
    if (!p->sched) return STENCIL_OK;
    unsigned int* st = reinterpret_cast<unsigned int*>(static_cast<unsigned long long*>(p->sched) + p->sched_words - 4);
    unsigned int h[2] = {0, 0};
    cudaError_t e = cudaMemcpy(h, st, sizeof(h), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_error(e, "cudaMemcpy(schedule stats)");
    *grabs = h[0];
    *steals = h[1];
    if (reset) {
        e = cudaMemset(st, 0, sizeof(h));
        if (e != cudaSuccess) return cuda_error(e, "cudaMemset(schedule stats)");
    }
    return STENCIL_OK;
}

int stencil_plan_set_timing(stencil_plan plan, int enable) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (!p) return set_error(STENCIL_EINVAL, "NULL argument");
    p->timing = enable != 0;
    return STENCIL_OK;
}

int stencil_plan_timing(stencil_plan plan, int kind, double* ms, int64_t* launches, int64_t* bytes,
                        int64_t* fmas) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (!p || !ms || !launches || !bytes || !fmas) return set_error(STENCIL_EINVAL, "NULL argument");
    double t = 0;
    int64_t n = 0, by = 0, fm = 0;
    for (const auto& rec : p->recs) {
        if (rec.kind != kind) continue;
        cudaError_t e = cudaEventSynchronize((cudaEvent_t)rec.b);
        if (e != cudaSuccess) return cuda_error(e, "cudaEventSynchronize");
        float x = 0;
        e = cudaEventElapsedTime(&x, (cudaEvent_t)rec.a, (cudaEvent_t)rec.b);
        if (e != cudaSuccess) return cuda_error(e, "cudaEventElapsedTime");
        t += x;
        ++n;
        by += rec.bytes;
        fm += rec.fmas;
    }
    *ms = t;
    *launches = n;
    *bytes = by;
    *fmas = fm;
    return STENCIL_OK;
}

int stencil_plan_timing_reset(stencil_plan plan) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (!p) return set_error(STENCIL_EINVAL, "NULL argument");
    for (const auto& rec : p->recs) {
        cudaEventSynchronize((cudaEvent_t)rec.b);
        p->event_pool.push_back(rec.a);
        p->event_pool.push_back(rec.b);
    }
    p->recs.clear();
    return STENCIL_OK;
}

int stencil_run(stencil_plan plan, const void* in, void* out, int64_t T, int fold_m, void* workspace,
                void* stream) {
    return run_single(reinterpret_cast<Plan*>(plan), in, out, T, fold_m, 0, workspace, stream);
}

int stencil_run_ex(stencil_plan plan, const void* in, void* out, int64_t T, int fold_m, int stages,
                   void* workspace, void* stream) {
    return run_single(reinterpret_cast<Plan*>(plan), in, out, T, fold_m, stages, workspace, stream);
}

int stencil_run_host(stencil_plan plan, const void* in_host, void* out_host, int64_t T, int fold_m, int stages,
                     void* dev_in, void* dev_out, void* workspace, void* stream) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (!p || !in_host || !out_host || !dev_in || !dev_out) return set_error(STENCIL_EINVAL, "NULL argument");
    Layout3 L = make_layout(p, 0, 1, 0);
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemcpyAsync(dev_in, in_host, L.bytes, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_error(e, "cudaMemcpyAsync H2D");
    int rc = run_single(p, dev_in, dev_out, T, fold_m, stages, workspace, stream);
    if (rc) return rc;
    e = cudaMemcpyAsync(out_host, dev_out, L.bytes, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return cuda_error(e, "cudaMemcpyAsync D2H");
    return STENCIL_OK;
}

// A batch of independent problems from host memory, pipelined across the
// GPU's copy engines: problem k's H2D (copy stream 1) and problem k-2's D2H
// (copy stream 2) overlap problem k-1's run (the caller's stream), on two
// device buffer sets used alternately.  Hazards are ordered with events:
// H2D into set j waits until the run two problems back finished reading it,
// a run into set j waits until that set's previous result left the device.
int stencil_run_host_batch(stencil_plan plan, int nbatch, const void* const* in_hosts, void* const* out_hosts,
                           int64_t T, int fold_m, int stages, void* const* dev, void* stream) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (!p || nbatch < 0 || (nbatch > 0 && (!in_hosts || !out_hosts || !dev)))
        return set_error(STENCIL_EINVAL, "NULL argument");
    if (nbatch == 0) return STENCIL_OK;
    const int sets = nbatch >= 2 ? 2 : 1;
    for (int j = 0; j < sets; ++j)
        if (!dev[3 * j] || !dev[3 * j + 1]) return set_error(STENCIL_EINVAL, "NULL device buffer");
    for (int k = 0; k < nbatch; ++k)
        if (!in_hosts[k] || !out_hosts[k]) return set_error(STENCIL_EINVAL, "NULL host buffer");
    cudaError_t e = cudaSuccess;
    if (!p->h2d_stream) e = cudaStreamCreateWithFlags(reinterpret_cast<cudaStream_t*>(&p->h2d_stream), cudaStreamNonBlocking);
    if (e == cudaSuccess && !p->d2h_stream)
        e = cudaStreamCreateWithFlags(reinterpret_cast<cudaStream_t*>(&p->d2h_stream), cudaStreamNonBlocking);
    for (void*& ev : p->pipe_ev)
        if (e == cudaSuccess && !ev) e = cudaEventCreateWithFlags(reinterpret_cast<cudaEvent_t*>(&ev), cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_error(e, "run_host_batch streams/events");
    Layout3 L = make_layout(p, 0, 1, 0);
    cudaStream_t st = (cudaStream_t)stream, si = (cudaStream_t)p->h2d_stream, so = (cudaStream_t)p->d2h_stream;
    cudaEvent_t* ev = reinterpret_cast<cudaEvent_t*>(p->pipe_ev);
    cudaEvent_t e_start = ev[0], *e_in = ev + 1, *e_comp = ev + 3, *e_out = ev + 5;
    int64_t launches = 0;
#define CK(x, what)                                   \
    do {                                              \
        cudaError_t _e = (x);                         \
        if (_e != cudaSuccess) return cuda_error(_e, what); \
    } while (0)
    CK(cudaEventRecord(e_start, st), "cudaEventRecord");
    CK(cudaStreamWaitEvent(si, e_start, 0), "cudaStreamWaitEvent");
    CK(cudaStreamWaitEvent(so, e_start, 0), "cudaStreamWaitEvent");
    for (int k = 0; k < nbatch; ++k) {
        const int j = k % sets;
        void* din = dev[3 * j];
        void* dout = dev[3 * j + 1];
        void* dws = dev[3 * j + 2];
        if (k >= sets) CK(cudaStreamWaitEvent(si, e_comp[j], 0), "cudaStreamWaitEvent");
        CK(cudaMemcpyAsync(din, in_hosts[k], L.bytes, cudaMemcpyHostToDevice, si), "cudaMemcpyAsync H2D");
        CK(cudaEventRecord(e_in[j], si), "cudaEventRecord");
        CK(cudaStreamWaitEvent(st, e_in[j], 0), "cudaStreamWaitEvent");
        if (k >= sets) CK(cudaStreamWaitEvent(st, e_out[j], 0), "cudaStreamWaitEvent");
        int rc = run_single(p, din, dout, T, fold_m, stages, dws, stream);
        if (rc) return rc;
        launches += p->last_launches;
        CK(cudaEventRecord(e_comp[j], st), "cudaEventRecord");
        CK(cudaStreamWaitEvent(so, e_comp[j], 0), "cudaStreamWaitEvent");
        CK(cudaMemcpyAsync(out_hosts[k], dout, L.bytes, cudaMemcpyDeviceToHost, so), "cudaMemcpyAsync D2H");
        CK(cudaEventRecord(e_out[j], so), "cudaEventRecord");
    }
    for (int j = 0; j < sets; ++j) CK(cudaStreamWaitEvent(st, e_out[j], 0), "cudaStreamWaitEvent");
#undef CK
    p->last_launches = launches;
    return STENCIL_OK;
}

int stencil_comm_unique_id(unsigned char id[128]) {
    if (!id) return set_error(STENCIL_EINVAL, "NULL argument");
    NcclApi& a = nccl();
    if (!a.ok) return set_error(STENCIL_ENCCL, a.why);
    ncclUniqueId u;
    ncclResult_t r = a.GetUniqueId(&u);
    if (r != ncclSuccess) return nccl_error(r, "ncclGetUniqueId");
    static_assert(sizeof(u) == 128, "ncclUniqueId size");
    std::memcpy(id, &u, 128);
    return STENCIL_OK;
}

int stencil_comm_create(stencil_comm* comm, const unsigned char id[128], int rank, int nranks) {
    if (!comm || !id) return set_error(STENCIL_EINVAL, "NULL argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return set_error(STENCIL_EINVAL, "bad rank/nranks");
    *comm = nullptr;
    NcclApi& a = nccl();
    if (!a.ok) return set_error(STENCIL_ENCCL, a.why);
    stencil_comm_s* c = new stencil_comm_s();
    c->rank = rank;
    c->nranks = nranks;
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    ncclResult_t r = a.CommInitRank(&c->comm, nranks, u, rank);
    if (r != ncclSuccess) {
        delete c;
        return nccl_error(r, "ncclCommInitRank");
    }
    cudaError_t e = cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->evA, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->evC, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        a.CommDestroy(c->comm);
        delete c;
        return cuda_error(e, "comm stream/events");
    }
    *comm = c;
    return STENCIL_OK;
}

// ---- fused peer-store exchange (NEXT-2)
int stencil_comm_create_peer(stencil_comm* comm, int rank, int nranks, void* buf0, void* buf1) {
    if (!comm || !buf0 || !buf1) return set_error(STENCIL_EINVAL, "NULL argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return set_error(STENCIL_EINVAL, "bad rank/nranks");
    if (buf0 == buf1) return set_error(STENCIL_EINVAL, "the two buffers must differ");
    *comm = nullptr;
    stencil_comm_s* c = new stencil_comm_s();
    c->rank = rank;
    c->nranks = nranks;
    c->peer = true;
    c->buf[0] = buf0;
    c->buf[1] = buf1;
    cudaError_t e = cudaMalloc(&c->flags, 256);   // own allocation: exported alone
    if (e == cudaSuccess) e = cudaMemset(c->flags, 0, 256);
    if (e != cudaSuccess) {
        delete c;
        return cuda_error(e, "flags");
    }
    *comm = c;
    return STENCIL_OK;
}

// 3 records of STENCIL_PEER_HANDLE_BYTES (buf0, buf1, flags): a 64-byte CUDA
// IPC handle of the allocation holding the pointer + the 8-byte offset into it.
int stencil_comm_peer_handles(stencil_comm comm, unsigned char* out) {
    if (!comm || !out) return set_error(STENCIL_EINVAL, "NULL argument");
    if (!comm->peer) return set_error(STENCIL_EINVAL, "not a peer comm");
    DrvMemOps& d = drv();
    if (!d.range) return set_error(STENCIL_ECUDA, "cuMemGetAddressRange unavailable");
    void* ptrs[3] = {comm->buf[0], comm->buf[1], comm->flags};
    for (int i = 0; i < 3; ++i) {
        CUdeviceptr base = 0;
        size_t size = 0;
        if (d.range(&base, &size, (CUdeviceptr)ptrs[i]) != CUDA_SUCCESS)
            return set_error(STENCIL_ECUDA, "cuMemGetAddressRange");
        cudaIpcMemHandle_t h;
        cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
        if (e != cudaSuccess) return cuda_error(e, "cudaIpcGetMemHandle");
        uint64_t off = (uint64_t)((CUdeviceptr)ptrs[i] - base);
        std::memcpy(out + i * STENCIL_PEER_HANDLE_BYTES, &h, 64);
        std::memcpy(out + i * STENCIL_PEER_HANDLE_BYTES + 64, &off, 8);
    }
    return STENCIL_OK;
}

// all: nranks x 3 records, in rank order (what every rank's peer_handles wrote).
int stencil_comm_peer_attach(stencil_comm comm, const unsigned char* all) {
    if (!comm || !all) return set_error(STENCIL_EINVAL, "NULL argument");
    if (!comm->peer) return set_error(STENCIL_EINVAL, "not a peer comm");
    const int nb[2] = {comm->rank - 1, comm->rank + 1};
    for (int side = 0; side < 2; ++side) {
        const int g = nb[side];
        if (g < 0 || g >= comm->nranks) continue;
        for (int i = 0; i < 3; ++i) {
            const unsigned char* rec = all + ((size_t)g * 3 + i) * STENCIL_PEER_HANDLE_BYTES;
            cudaIpcMemHandle_t h;
            uint64_t off = 0;
            std::memcpy(&h, rec, 64);
            std::memcpy(&off, rec + 64, 8);
            void* base = nullptr;
            cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess) return cuda_error(e, "cudaIpcOpenMemHandle");
            comm->nbase[side][i] = base;
            char* ptr = static_cast<char*>(base) + off;
            if (i < 2) comm->nbuf[side][i] = ptr;
            // the neighbour's flag this rank writes: the lower neighbour hears from
            // its upper side (slot 1), the upper neighbour from its lower side (slot 0)
            else comm->nflag[side] = reinterpret_cast<uint32_t*>(ptr) + (side == 0 ? 1 : 0);
        }
    }
    return STENCIL_OK;
}

int stencil_comm_destroy(stencil_comm comm) {
    if (!comm) return STENCIL_OK;
    for (auto& side : comm->nbase)
        for (void*& b : side)
            if (b) cudaIpcCloseMemHandle(b);
    if (comm->flags) cudaFree(comm->flags);
    NcclApi& a = nccl();
    if (comm->comm && a.ok) a.CommDestroy(comm->comm);
    if (comm->evA) cudaEventDestroy(comm->evA);
    if (comm->evC) cudaEventDestroy(comm->evC);
    if (comm->cstream) cudaStreamDestroy(comm->cstream);
    delete comm;
    return STENCIL_OK;
}

// NCCL failure detection: the communicator's asynchronous error
// (a peer died, a network/NVLink fault) is polled before every exchange and
// by stencil_comm_wait; every call's return code is checked.
static int nccl_async_check(stencil_comm_s* c) {
    NcclApi& a = nccl();
    if (!a.ok) return set_error(STENCIL_ENCCL, a.why);
    if (!c->comm) return set_error(STENCIL_EINVAL, "not an NCCL comm");
    if (c->failed) return set_error(STENCIL_ENCCL, "communicator aborted after an earlier failure");
    ncclResult_t ar = ncclSuccess;
    ncclResult_t r = a.CommGetAsyncError(c->comm, &ar);
    if (r != ncclSuccess) return nccl_error(r, "ncclCommGetAsyncError");
    if (ar != ncclSuccess && ar != ncclInProgress) {
        c->failed = true;
        a.CommAbort(c->comm);
        c->comm = nullptr;
        return nccl_error(ar, "NCCL asynchronous error (communicator aborted)");
    }
    return STENCIL_OK;
}

// lo_peer / hi_peer: the ranks owning the planes below / above this slab (-1: a
// physical face, no exchange on that side).
static int nccl_exchange_with(Plan* p, stencil_comm_s* c, const Layout3& L, void* buf, int64_t hx, cudaStream_t st,
                              int lo_peer, int hi_peer) {
    int rc = nccl_async_check(c);
    if (rc) return rc;
    NcclApi& a = nccl();
    const ncclDataType_t dt = p->dtype == STENCIL_F64 ? ncclDouble : ncclFloat;
    const size_t cnt = (size_t)hx * L.stride[0];
    char* base = static_cast<char*>(buf);
    const size_t pb = plane_bytes(L);
    auto plane = [&](int64_t z) { return base + (size_t)(L.origin[0] + z) * pb; };
    ncclResult_t r = a.GroupStart();
    if (r != ncclSuccess) return nccl_error(r, "ncclGroupStart");
    ncclResult_t first = ncclSuccess;
    const char* what = nullptr;
    auto chk = [&](ncclResult_t x, const char* w) {
        if (x != ncclSuccess && first == ncclSuccess) { first = x; what = w; }
    };
    if (lo_peer >= 0) {
        chk(a.Send(plane(0), cnt, dt, lo_peer, c->comm, st), "ncclSend(lower)");
        chk(a.Recv(plane(-hx), cnt, dt, lo_peer, c->comm, st), "ncclRecv(lower)");
    }
    if (hi_peer >= 0) {
        chk(a.Send(plane(L.n[0] - hx), cnt, dt, hi_peer, c->comm, st), "ncclSend(upper)");
        chk(a.Recv(plane(L.n[0]), cnt, dt, hi_peer, c->comm, st), "ncclRecv(upper)");
    }
    r = a.GroupEnd();   // always close the group, even after a failed call
    if (first != ncclSuccess) return nccl_error(first, what);
    if (r != ncclSuccess) return nccl_error(r, "ncclGroupEnd");
    return STENCIL_OK;
}

static int nccl_exchange(Plan* p, stencil_comm_s* c, const Layout3& L, void* buf, int64_t hx, cudaStream_t st) {
    return nccl_exchange_with(p, c, L, buf, hx, st, c->rank > 0 ? c->rank - 1 : -1,
                              c->rank < c->nranks - 1 ? c->rank + 1 : -1);
}

int stencil_halo_exchange_loopback(stencil_plan plan, stencil_comm comm, void* buf, int halo, void* stream) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (!p || !comm || !buf) return set_error(STENCIL_EINVAL, "NULL argument");
    Layout3 L;
    int rc = dist_layout_check(p, comm->rank, comm->nranks, halo, 1, &L);
    if (rc) return rc;
    if (comm->peer) return set_error(STENCIL_EINVAL, "loopback exchange needs an NCCL comm");
    if (L.n[0] < halo) return set_error(STENCIL_EINVAL, "slab thinner than the halo");
    if (halo > L.origin[0] || halo > L.ext[0] - L.origin[0] - L.n[0])
        return set_error(STENCIL_EINVAL, "halo exceeds the planes this layout allocates outside the slab");
    // the sweep's exchange with this rank as both neighbours: in the group the
    // sends and receives to one peer match in issue order, so planes [0, halo)
    // land in the lower ghost planes and planes [n0 - halo, n0) in the upper
    return nccl_exchange_with(p, comm, L, buf, halo, (cudaStream_t)stream, comm->rank, comm->rank);
}

int stencil_halo_exchange(stencil_plan plan, stencil_comm comm, void* buf, int halo, void* stream) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (!p || !comm || !buf) return set_error(STENCIL_EINVAL, "NULL argument");
    Layout3 L;
    int rc = dist_layout_check(p, comm->rank, comm->nranks, halo, 1, &L);
    if (rc) return rc;
    if (comm->peer)
        return set_error(STENCIL_EINVAL, "peer comm: ghost planes are written by the sweep kernel; "
                                         "stencil_halo_exchange needs an NCCL comm");
    if (comm->nranks == 1) return STENCIL_OK;
    return nccl_exchange(p, comm, L, buf, halo, (cudaStream_t)stream);
}

int stencil_comm_wait(stencil_comm comm, void* stream, int64_t timeout_ms) {
    if (!comm) return set_error(STENCIL_EINVAL, "NULL argument");
    cudaStream_t st = (cudaStream_t)stream;
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        cudaError_t e = cudaStreamQuery(st);
        if (e == cudaSuccess) break;
        if (e != cudaErrorNotReady) return cuda_error(e, "cudaStreamQuery");
        if (!comm->peer) {
            int rc = nccl_async_check(comm);
            if (rc) return rc;
        }
        const auto ms = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count();
        if (timeout_ms >= 0 && ms > timeout_ms) {
            if (!comm->peer && comm->comm) {   // a hung collective: abort so the stream can drain
                comm->failed = true;
                nccl().CommAbort(comm->comm);
                comm->comm = nullptr;
            }
            return set_error(STENCIL_ETIMEOUT, "stencil_comm_wait: timed out after " + std::to_string(ms) + " ms");
        }
        std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
    if (!comm->peer) return nccl_async_check(comm);
    return STENCIL_OK;
}

int stencil_run_dist(stencil_plan plan, stencil_comm comm, const void* in_local, void* out_local, int64_t T,
                     int fold_m, int stages, int halo, void* workspace, void* stream) {
    NvtxRange nv("stencil_run_dist");
    if (plan && fold_m == 0) fold_m = auto_fold(reinterpret_cast<Plan*>(plan));
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (!comm) return set_error(STENCIL_EINVAL, "comm is NULL");
    int rc = check_run_args(p, in_local, out_local, T, fold_m, workspace);
    if (rc) return rc;
    Layout3 L;
    rc = dist_layout_check(p, comm->rank, comm->nranks, halo, fold_m, &L);
    if (rc) return rc;
    rc = ensure_device(p);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    if (T == 0) {
        cudaError_t e = cudaMemcpyAsync(out_local, in_local, L.bytes, cudaMemcpyDeviceToDevice, st);
        return e == cudaSuccess ? STENCIL_OK : cuda_error(e, "cudaMemcpyAsync");
    }
    Variant v{1, 1};
    if (T >= fold_m) {   // (T < fold_m: only the remainder sweep runs)
        rc = resolve_variant(p, fold_m, stages, &v);
        if (rc) return rc;
    }
    const int64_t nf = T / fold_m;
    int64_t n;
    int mr;
    Variant vr;
    remainder_plan(p, T, fold_m, &n, &mr, &vr);
    if (n >= 2 && !workspace) return set_error(STENCIL_EINVAL, "workspace required");
    const int64_t hx = (int64_t)fold_m * p->r;
    if (comm->peer)
        return run_dist_peer(p, comm, L, in_local, out_local, workspace, n, nf, fold_m, v, mr, vr, hx, stream);
    rc = nccl_async_check(comm);
    if (rc) return rc;
    int launches = 0;
    rc = launch_ring_copy(p, in_local, out_local, &L, stream);
    if (rc < 0) return rc;
    launches += rc;
    if (n >= 2) {
        rc = launch_ring_copy(p, in_local, workspace, &L, stream);
        if (rc < 0) return rc;
        launches += rc;
    }
    void* bufs[2] = {out_local, workspace};
    for (int64_t j = 1; j <= n; ++j) {
        SweepSpec s;
        s.m = j <= nf ? fold_m : mr;
        s.v = j <= nf ? v : vr;
        const void* src = j == 1 ? in_local : bufs[(n - j + 1) % 2];
        void* dst = bufs[(n - j) % 2];
        rc = sweep_phase(p, L, src, dst, s, comm->rank, comm->nranks, hx, 0, stream);
        if (rc < 0) return rc;
        launches += rc;
        const bool xchg = comm->nranks > 1 && j < n;
        if (xchg) {
            cudaEventRecord(comm->evA, st);
            cudaStreamWaitEvent(comm->cstream, comm->evA, 0);
            rc = nccl_exchange(p, comm, L, dst, hx, comm->cstream);
            if (rc) return rc;
            cudaEventRecord(comm->evC, comm->cstream);
        }
        rc = sweep_phase(p, L, src, dst, s, comm->rank, comm->nranks, hx, 1, stream);
        if (rc < 0) return rc;
        launches += rc;
        if (xchg) cudaStreamWaitEvent(st, comm->evC, 0);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_error(e, "run_dist");
    p->last_launches = launches;
    return STENCIL_OK;
}

int stencil_run_dist_emulated(stencil_plan plan, int nranks, const void* const* in_locals, void* const* out_locals,
                              int64_t T, int fold_m, int stages, int halo, void* const* workspaces, int exchange,
                              void* stream) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (!p || !in_locals || !out_locals || nranks < 1) return set_error(STENCIL_EINVAL, "bad argument");
    std::vector<Layout3> Ls(nranks);
    for (int g = 0; g < nranks; ++g) {
        int rc = check_run_args(p, in_locals[g], out_locals[g], T, fold_m, workspaces ? workspaces[g] : nullptr);
        if (rc) return rc;
        rc = dist_layout_check(p, g, nranks, halo, fold_m, &Ls[g]);
        if (rc) return rc;
    }
    int rc = ensure_device(p);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    if (T == 0) {
        for (int g = 0; g < nranks; ++g) {
            cudaError_t e = cudaMemcpyAsync(out_locals[g], in_locals[g], Ls[g].bytes, cudaMemcpyDeviceToDevice, st);
            if (e != cudaSuccess) return cuda_error(e, "cudaMemcpyAsync");
        }
        return STENCIL_OK;
    }
    Variant v{1, 1};
    if (T >= fold_m) {   // (T < fold_m: only the remainder sweep runs)
        rc = resolve_variant(p, fold_m, stages, &v);
        if (rc) return rc;
    }
    const int64_t nf = T / fold_m;
    int64_t n;
    int mr;
    Variant vr;
    remainder_plan(p, T, fold_m, &n, &mr, &vr);
    if (n >= 2 && !workspaces) return set_error(STENCIL_EINVAL, "workspaces required");
    const int64_t hx = (int64_t)fold_m * p->r;
    int launches = 0;
    for (int g = 0; g < nranks; ++g) {
        rc = launch_ring_copy(p, in_locals[g], out_locals[g], &Ls[g], stream);
        if (rc < 0) return rc;
        if (n >= 2) {
            if (!workspaces[g]) return set_error(STENCIL_EINVAL, "workspace required");
            rc = launch_ring_copy(p, in_locals[g], workspaces[g], &Ls[g], stream);
            if (rc < 0) return rc;
        }
    }
    if (exchange == 1) {
        // fused peer stores (NEXT-2): one launch per rank and sweep over the whole
        // slab; the kernel itself stores its boundary planes into the
        // neighbours' ghost planes (here plain device pointers on this GPU; the
        // ranks run one after another on one stream, so no flags are needed)
        for (int64_t j = 1; j <= n; ++j) {
            SweepSpec s;
            s.m = j <= nf ? fold_m : mr;
            s.v = j <= nf ? v : vr;
            std::vector<void*> dsts(nranks);
            for (int g = 0; g < nranks; ++g) {
                void* bufs[2] = {out_locals[g], workspaces ? workspaces[g] : nullptr};
                dsts[g] = bufs[(n - j) % 2];
            }
            for (int g = 0; g < nranks; ++g) {
                void* bufs[2] = {out_locals[g], workspaces ? workspaces[g] : nullptr};
                const void* src = j == 1 ? in_locals[g] : bufs[(n - j + 1) % 2];
                rc = enqueue_sweep(p, Ls[g], src, dsts[g], s, 0, Ls[g].n[0], stream,
                                   g > 0 ? dsts[g - 1] : nullptr, g < nranks - 1 ? dsts[g + 1] : nullptr,
                                   (int)hx);
                if (rc < 0) return rc;
                launches += rc;
            }
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_error(e, "run_dist_emulated");
        p->last_launches = launches;
        return STENCIL_OK;
    }
    for (int64_t j = 1; j <= n; ++j) {
        SweepSpec s;
        s.m = j <= nf ? fold_m : mr;
        s.v = j <= nf ? v : vr;
        std::vector<const void*> srcs(nranks);
        std::vector<void*> dsts(nranks);
        for (int g = 0; g < nranks; ++g) {
            void* bufs[2] = {out_locals[g], workspaces ? workspaces[g] : nullptr};
            srcs[g] = j == 1 ? in_locals[g] : bufs[(n - j + 1) % 2];
            dsts[g] = bufs[(n - j) % 2];
            rc = sweep_phase(p, Ls[g], srcs[g], dsts[g], s, g, nranks, hx, 0, stream);
            if (rc < 0) return rc;
            launches += rc;
        }
        if (nranks > 1 && j < n) {
            // the transport: device-to-device copies between the ranks' buffers
            for (int g = 0; g < nranks; ++g) {
                const Layout3& L = Ls[g];
                const size_t pb = plane_bytes(L);
                char* me = static_cast<char*>(dsts[g]);
                if (g > 0) {
                    const Layout3& Ln = Ls[g - 1];
                    char* nb = static_cast<char*>(dsts[g - 1]);
                    cudaMemcpyAsync(nb + (size_t)(Ln.origin[0] + Ln.n[0]) * pb, me + (size_t)L.origin[0] * pb,
                                    (size_t)hx * pb, cudaMemcpyDeviceToDevice, st);
                }
                if (g < nranks - 1) {
                    const Layout3& Ln = Ls[g + 1];
                    char* nb = static_cast<char*>(dsts[g + 1]);
                    cudaMemcpyAsync(nb + (size_t)(Ln.origin[0] - hx) * pb,
                                    me + (size_t)(L.origin[0] + L.n[0] - hx) * pb, (size_t)hx * pb,
                                    cudaMemcpyDeviceToDevice, st);
                }
            }
        }
        for (int g = 0; g < nranks; ++g) {
            rc = sweep_phase(p, Ls[g], srcs[g], dsts[g], s, g, nranks, hx, 1, stream);
            if (rc < 0) return rc;
            launches += rc;
        }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_error(e, "run_dist_emulated");
    p->last_launches = launches;
    return STENCIL_OK;
}

}  // extern "C"

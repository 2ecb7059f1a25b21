// aux.cu — the 1D on-chip multi-step kernel (K-G4),
// the frozen-ring initialisation (K-G5) and the seeded field generator (K-G0).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <cstdlib>
#include <utility>

#include "internal.hpp"
#include "onchip1d.cuh"
#include "sweep_params.cuh"

namespace sb {

int cuda_error(int e, const char* what) {
    return set_error(STENCIL_ECUDA, std::string(what) + ": " + cudaGetErrorString((cudaError_t)e));
}

template <typename T>
static K1Fn<T> k1_pick(int V, int r, int m, bool wrap) {
    return V == 32 ? k1_pick_wide<T>(r, m, wrap) : k1_pick_narrow<T>(V, r, m, wrap);
}

// Cells per lane: the smallest of {8, 16, 32} holding the fold radius; the
// env var STENCIL_1D_V overrides it (tuning).
int onchip1d_cells_per_lane(int r, int m, bool wrap) {
#ifdef STENCIL_TUNING_BUILD
    static int forced = [] {   // (tuning builds only)
        const char* e = getenv("STENCIL_1D_V");
        return e ? atoi(e) : 0;
    }();
#else
    constexpr int forced = 0;
#endif
    int v = (r * m <= 8 && !wrap) ? 8 : r * m <= 16 ? 16 : 32;
    if (wrap) return v;
    if (forced == 16 && r * m <= 16) v = 16;   // (tuning) the only other compiled choice
    return v;
}

template <typename T>
static int launch_1d_t(Plan* p, const void* src, void* dst, const Layout3* L, int64_t TB, int m,
                       bool force_step, void* stream) {
    Params1D<T> prm;
    std::memset(&prm, 0, sizeof(prm));
    prm.src = static_cast<const T*>(src);
    prm.dst = static_cast<T*>(dst);
    prm.origin = L->origin[2];
    prm.ext = L->ext[2];
    prm.n = (int)L->n[2];
    prm.r = p->r;
    prm.m = m;
    prm.TB = (int)TB;
    prm.force_step = force_step ? 1 : 0;
    prm.wrap = L->wrap ? 1 : 0;
    const std::vector<double>& lam = folded(p, m);
    if ((int)lam.size() > K1_MAXC || (int)p->w.size() > 9) return set_error(STENCIL_EUNSUPPORTED, "1D fold too wide");
    for (size_t i = 0; i < lam.size(); ++i) prm.lam[i] = static_cast<T>(lam[i]);
    for (size_t i = 0; i < p->w.size(); ++i) prm.w[i] = static_cast<T>(p->w[i]);
    const int V = onchip1d_cells_per_lane(p->r, m, L->wrap);
    K1Fn<T> fn = k1_pick<T>(V, p->r, m, L->wrap);
    if (!fn) return set_error(STENCIL_EUNSUPPORTED, "1D kernel: r or fold_m out of range");
    prm.B = 32 * V - 2 * (int)TB * p->r;   // outputs per warp
    if (prm.B <= 0) return set_error(STENCIL_EINVAL, "1D kernel: too many steps per launch for the warp window");
    prm.nwarps = (prm.n + prm.B - 1) / prm.B;
    const int wpb = K1_THREADS / 32;
    const unsigned blocks = (unsigned)std::max(1, (prm.nwarps + wpb - 1) / wpb);
    fn<<<blocks, K1_THREADS, 0, (cudaStream_t)stream>>>(prm);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_error(e, "onchip1d_kernel launch");
    return 1;
}

int launch_1d(Plan* p, const void* src, void* dst, const Layout3* L, int64_t TB, int m, int force_step,
              void* stream) {
    return p->dtype == STENCIL_F64 ? launch_1d_t<double>(p, src, dst, L, TB, m, force_step != 0, stream)
                                   : launch_1d_t<float>(p, src, dst, L, TB, m, force_step != 0, stream);
}

// ============================================================== K-G5 ring
// Copy every non-interior cell (frozen ring, ghost planes, pads) src -> dst,
// one warp per row of the allocation.
template <typename T>
__global__ void ring_copy_kernel(const T* __restrict__ src, T* __restrict__ dst, DevGeom g, long long rows,
                                 int keep_ghost_interior) {
    long long row = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (row >= rows) return;
    const int lane = threadIdx.x & 31;
    long long r0 = row / g.ext[1], r1 = row % g.ext[1];
    long long c0 = r0 - g.origin[0], c1 = r1 - g.origin[1];
    // a ghost plane (non-physical face) counts as interior along axis 0 when its
    // interior cells are owned by the neighbours' stores
    const bool ghost0 = keep_ghost_interior && ((c0 < 0 && !g.phys_lo[0]) || (c0 >= g.n[0] && !g.phys_hi[0]));
    bool inside = (ghost0 || (c0 >= 0 && c0 < g.n[0])) && c1 >= 0 && c1 < g.n[1];
    long long base = r0 * g.stride0 + r1 * g.stride1;
    if (!inside) {
        for (long long x = lane; x < g.ext[2]; x += 32) dst[base + x] = src[base + x];
    } else {
        long long xl = g.origin[2], xr = g.origin[2] + g.n[2];
        for (long long x = lane; x < xl; x += 32) dst[base + x] = src[base + x];
        for (long long x = xr + lane; x < g.ext[2]; x += 32) dst[base + x] = src[base + x];
    }
}

int launch_ring_copy(Plan* p, const void* src, void* dst, const Layout3* L, void* stream, bool keep_ghost_interior) {
    DevGeom g;
    fill_geom(*L, &g);
    long long rows = L->ext[0] * L->ext[1];
    int wpb = 8;
    unsigned blocks = (unsigned)((rows + wpb - 1) / wpb);
    if (p->dtype == STENCIL_F64)
        ring_copy_kernel<double><<<blocks, wpb * 32, 0, (cudaStream_t)stream>>>(
            static_cast<const double*>(src), static_cast<double*>(dst), g, rows, keep_ghost_interior ? 1 : 0);
    else
        ring_copy_kernel<float><<<blocks, wpb * 32, 0, (cudaStream_t)stream>>>(
            static_cast<const float*>(src), static_cast<float*>(dst), g, rows, keep_ghost_interior ? 1 : 0);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_error(e, "ring_copy_kernel launch");
    return 1;
}

// ============================================================== PERIODIC ghosts
// Every ghost cell (within the allocation, outside the interior) takes the
// value of its wrapped interior cell; one warp per allocation row.  Reads and
// writes are disjoint (interior -> ghosts), so one launch fills edges and
// corners alike.
template <typename T>
__global__ void wrap_fill_kernel(T* __restrict__ buf, DevGeom g, long long rows, int used0, int used1) {
    long long row = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (row >= rows) return;
    const int lane = threadIdx.x & 31;
    const long long r0 = row / g.ext[1], r1 = row % g.ext[1];
    const long long c0 = r0 - g.origin[0], c1 = r1 - g.origin[1];
    auto wrapi = [](long long c, long long n) { long long w = c % n; return w < 0 ? w + n : w; };
    const long long w0 = used0 ? wrapi(c0, g.n[0]) : 0, w1 = used1 ? wrapi(c1, g.n[1]) : 0;
    const bool inside = (!used0 || (c0 >= 0 && c0 < g.n[0])) && (!used1 || (c1 >= 0 && c1 < g.n[1]));
    const T* srow = buf + (g.origin[0] + w0) * g.stride0 + (g.origin[1] + w1) * g.stride1 + g.origin[2];
    T* drow = buf + r0 * g.stride0 + r1 * g.stride1 + g.origin[2];
    const long long xlo = -(long long)g.lo_valid[2], xhi = g.n[2] + (long long)g.hi_valid[2];
    if (!inside) {
        for (long long x = xlo + lane; x < xhi; x += 32) drow[x] = srow[wrapi(x, g.n[2])];
    } else {
        for (long long x = xlo + lane; x < 0; x += 32) drow[x] = srow[wrapi(x, g.n[2])];
        for (long long x = g.n[2] + lane; x < xhi; x += 32) drow[x] = srow[wrapi(x, g.n[2])];
    }
}

int launch_wrap_fill(Plan* p, void* buf, const Layout3* L, void* stream) {
    DevGeom g;
    fill_geom(*L, &g);
    const int used0 = p->ndim >= 2, used1 = p->ndim == 3;
    // rows of the ghost-extended frame only: axis-0/1 rows in [-G, n+G)
    long long rows = L->ext[0] * L->ext[1];
    int wpb = 8;
    unsigned blocks = (unsigned)((rows + wpb - 1) / wpb);
    if (p->dtype == STENCIL_F64)
        wrap_fill_kernel<double><<<blocks, wpb * 32, 0, (cudaStream_t)stream>>>(static_cast<double*>(buf), g, rows,
                                                                                used0, used1);
    else
        wrap_fill_kernel<float><<<blocks, wpb * 32, 0, (cudaStream_t)stream>>>(static_cast<float*>(buf), g, rows,
                                                                               used0, used1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_error(e, "wrap_fill_kernel launch");
    return 1;
}

// ============================================================== K-G0 fill
// u0 = U(seed, i), i = row-major index in the unaligned GLOBAL padded frame
// prod(N_a + 2r) (R6): splitmix64 in counter form, (mix >> 11) * 2^-53.
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <typename T>
__global__ void fill_kernel(T* __restrict__ buf, DevGeom g, long long gofs0, long long gn0, long long gn1,
                            long long gn2, int r, int used0, int used1, unsigned long long seed, long long total) {
    long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    long long stride = (long long)gridDim.x * blockDim.x;
    const long long P1 = used1 ? gn1 + 2 * r : 1, P2 = gn2 + 2 * r;
    for (; e < total; e += stride) {
        long long a0 = e / g.stride0, rem = e % g.stride0;
        long long a1 = rem / g.stride1, a2 = rem % g.stride1;
        // global padded coordinates
        long long p0 = used0 ? (a0 - g.origin[0] + gofs0 + r) : 0;
        long long p1 = used1 ? (a1 - g.origin[1] + r) : 0;
        long long p2 = a2 - g.origin[2] + r;
        bool in = p2 >= 0 && p2 < P2 && p1 >= 0 && p1 < P1 && (!used0 || (p0 >= 0 && p0 < gn0 + 2 * r));
        T v = T(0);
        if (in) {
            unsigned long long idx = (unsigned long long)((p0 * P1 + p1) * P2 + p2);
            unsigned long long z = seed + (idx + 1ull) * 0x9E3779B97F4A7C15ull;
            v = static_cast<T>((double)(mix64(z) >> 11) * 0x1.0p-53);
        }
        buf[e] = v;
    }
}

int launch_fill(Plan* p, void* buf, const Layout3* L, uint64_t seed, void* stream) {
    DevGeom g;
    fill_geom(*L, &g);
    if (g.stride1 == 0) g.stride1 = 1;
    long long total = L->ext[0] * L->stride[0];
    int used0 = p->ndim >= 2, used1 = p->ndim == 3;
    unsigned blocks = (unsigned)std::min<long long>((total + 255) / 256, 148 * 64);
    if (p->dtype == STENCIL_F64)
        fill_kernel<double><<<blocks, 256, 0, (cudaStream_t)stream>>>(static_cast<double*>(buf), g, L->gofs0, L->gn[0],
                                                                      L->gn[1], L->gn[2], p->r, used0, used1, seed, total);
    else
        fill_kernel<float><<<blocks, 256, 0, (cudaStream_t)stream>>>(static_cast<float*>(buf), g, L->gofs0, L->gn[0],
                                                                     L->gn[1], L->gn[2], p->r, used0, used1, seed, total);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_error(e, "fill_kernel launch");
    return 1;
}

}  // namespace sb

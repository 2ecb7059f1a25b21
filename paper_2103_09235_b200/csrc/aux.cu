// aux.cu — the 1D on-chip multi-step kernel (K-G4),
// the frozen-ring initialisation (K-G5) and the seeded field generator (K-G0).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "internal.hpp"
#include "sweep_params.cuh"

namespace sb {

int cuda_error(int e, const char* what) {
    return set_error(STENCIL_ECUDA, std::string(what) + ": " + cudaGetErrorString((cudaError_t)e));
}

// ============================================================== K-G4 1D
// 1D: the whole grid (0.8 MB for the 1D3P config) is far below L2 and one sweep
// is shorter than a launch, so TB time steps run inside one launch: each CTA
// owns B outputs, loads them plus a TB*r halo into shared memory and applies
// TB/m folded steps (lambda^(m)) then TB mod m single steps on a shrinking
// region (overlapped tiles, no inter-CTA synchronisation).  CTAs whose region
// comes within (m-1)*r of a FIXED face apply single steps throughout (exact
// band, R2); ring cells keep u0.
constexpr int K1_THREADS = 256;
constexpr int K1_MAXC = 2 * STENCIL_MAX_FOLD * 4 + 1;

template <typename T>
struct Params1D {
    const T* src;
    T* dst;
    long long origin, ext;
    int n, r, m, TB, B, force_step;
    int nlam, nw;
    T lam[K1_MAXC];   // lambda^(m), index o + m r
    T w[9];           // original taps, index o + r
};

template <typename T>
__global__ void __launch_bounds__(K1_THREADS) onchip1d_kernel(const __grid_constant__ Params1D<T> p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int hal = p.TB * p.r;
    const int x0 = blockIdx.x * p.B;
    const int x1 = min(x0 + p.B, p.n);
    const int ilo = x0 - hal;
    const int len = (x1 - x0) + 2 * hal;
    T* a = reinterpret_cast<T*>(smem_raw);
    T* b = a + len;
    for (int e = threadIdx.x; e < len; e += blockDim.x) {
        long long g = p.origin + ilo + e;
        a[e] = (g >= 0 && g < p.ext) ? p.src[g] : T(0);
    }
    __syncthreads();
    const int band = (p.m - 1) * p.r;
    const bool stepwise = p.force_step || (ilo < band) || (x1 + hal > p.n - band);
    const int nfold = stepwise ? 0 : p.TB / p.m;
    const int nsingle = stepwise ? p.TB : p.TB % p.m;
    int shrink = 0;
    for (int s = 0; s < nfold + nsingle; ++s) {
        const bool fold = s < nfold;
        const int R = fold ? p.m * p.r : p.r;
        shrink += R;
        for (int e = shrink + threadIdx.x; e < len - shrink; e += blockDim.x) {
            const int x = ilo + e;
            T acc;
            if (x < 0 || x >= p.n) {
                acc = a[e];   // frozen ring (or unused cells beyond it)
            } else if (fold) {
                acc = T(0);
                for (int o = -R; o <= R; ++o) acc = fma(p.lam[o + R], a[e + o], acc);
            } else {
                acc = T(0);
                for (int o = -R; o <= R; ++o) acc = fma(p.w[o + R], a[e + o], acc);
            }
            b[e] = acc;
        }
        __syncthreads();
        T* t = a;
        a = b;
        b = t;
    }
    for (int e = threadIdx.x; e < x1 - x0; e += blockDim.x) p.dst[p.origin + x0 + e] = a[hal + e];
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
    const std::vector<double>& lam = folded(p, m);
    if ((int)lam.size() > K1_MAXC || (int)p->w.size() > 9) return set_error(STENCIL_EUNSUPPORTED, "1D fold too wide");
    prm.nlam = (int)lam.size();
    for (size_t i = 0; i < lam.size(); ++i) prm.lam[i] = static_cast<T>(lam[i]);
    prm.nw = (int)p->w.size();
    for (size_t i = 0; i < p->w.size(); ++i) prm.w[i] = static_cast<T>(p->w[i]);
    // about two CTAs per SM, each B outputs (+ 2*TB*r halo)
    int nctas = std::max(1, 2 * p->sm_count);
    int B = (int)std::max<int64_t>(64, (prm.n + nctas - 1) / nctas);
    prm.B = B;
    nctas = (prm.n + B - 1) / B;
    size_t smem = 2 * (size_t)(B + 2 * TB * p->r) * sizeof(T);
    if (smem > 200 * 1024) return set_error(STENCIL_EUNSUPPORTED, "1D on-chip block too large");
    static bool attr_set[2] = {false, false};
    if (!attr_set[sizeof(T) == 8]) {
        cudaFuncSetAttribute(onchip1d_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_set[sizeof(T) == 8] = true;
    }
    onchip1d_kernel<T><<<nctas, K1_THREADS, smem, (cudaStream_t)stream>>>(prm);
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
__global__ void ring_copy_kernel(const T* __restrict__ src, T* __restrict__ dst, DevGeom g, long long rows) {
    long long row = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (row >= rows) return;
    const int lane = threadIdx.x & 31;
    long long r0 = row / g.ext[1], r1 = row % g.ext[1];
    long long c0 = r0 - g.origin[0], c1 = r1 - g.origin[1];
    bool inside = c0 >= 0 && c0 < g.n[0] && c1 >= 0 && c1 < g.n[1];
    long long base = r0 * g.stride0 + r1 * g.stride1;
    if (!inside) {
        for (long long x = lane; x < g.ext[2]; x += 32) dst[base + x] = src[base + x];
    } else {
        long long xl = g.origin[2], xr = g.origin[2] + g.n[2];
        for (long long x = lane; x < xl; x += 32) dst[base + x] = src[base + x];
        for (long long x = xr + lane; x < g.ext[2]; x += 32) dst[base + x] = src[base + x];
    }
}

int launch_ring_copy(Plan* p, const void* src, void* dst, const Layout3* L, void* stream) {
    DevGeom g;
    fill_geom(*L, &g);
    long long rows = L->ext[0] * L->ext[1];
    int wpb = 8;
    unsigned blocks = (unsigned)((rows + wpb - 1) / wpb);
    if (p->dtype == STENCIL_F64)
        ring_copy_kernel<double><<<blocks, wpb * 32, 0, (cudaStream_t)stream>>>(
            static_cast<const double*>(src), static_cast<double*>(dst), g, rows);
    else
        ring_copy_kernel<float><<<blocks, wpb * 32, 0, (cudaStream_t)stream>>>(
            static_cast<const float*>(src), static_cast<float*>(dst), g, rows);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_error(e, "ring_copy_kernel launch");
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

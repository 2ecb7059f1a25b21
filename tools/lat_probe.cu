// Dependent-chain latency and per-SMSP throughput of DFMA / FFMA / SHFL / LDS on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
template <typename T>
__global__ void chain(T* out, long long* cyc, int n, T a, T b) {
    T x = (T)threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) x = fma(x, a, b);
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <typename T, int ILP>
__global__ void thru(T* out, long long* cyc, int n, T a, T b) {
    T x[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = (T)(threadIdx.x + k);
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < ILP; ++k) x[k] = fma(x[k], a, b);
    }
    __syncthreads();
    long long t1 = clock64();
    T s = 0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void shfl_chain(double* out, long long* cyc, int n) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __shfl_down_sync(0xffffffffu, x, 1) + 1.0;
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
    double* od; float* of; long long* c; long long h[1024];
    cudaMalloc(&od, 1 << 24); cudaMalloc(&of, 1 << 24); cudaMalloc(&c, 8192);
    int n = 4096;
    chain<double><<<1, 32>>>(od, c, n, 1.0000001, 1e-9); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.2f cyc\n", (double)h[0] / (n * 16));
    chain<float><<<1, 32>>>(of, c, n, 1.0000001f, 1e-9f); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
    printf("FFMA dependent latency: %.2f cyc\n", (double)h[0] / (n * 16));
    shfl_chain<<<1, 32>>>(od, c, n); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
    printf("SHFL(double)+DADD chain: %.2f cyc\n", (double)h[0] / n);
    for (int w : {1, 2, 4, 8, 16}) {
        thru<double, 8><<<1, 32 * w>>>(od, c, n, 1.0000001, 1e-9); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
        printf("DFMA ILP8 warps/SM=%2d: %.2f cyc per warp-instr per SM (%.1f FMA/clk/SM)\n", w,
               (double)h[0] / (n * 8.0 * w), 32.0 * n * 8 * w / h[0]);
    }
    for (int w : {1, 4, 8, 16}) {
        thru<float, 8><<<1, 32 * w>>>(of, c, n, 1.0000001f, 1e-9f); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
        printf("FFMA ILP8 warps/SM=%2d: %.1f FMA/clk/SM\n", w, 32.0 * n * 8 * w / h[0]);
    }
    return 0;
}

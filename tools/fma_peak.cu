// fma_peak.cu — measures the plain fp64 / fp32 FMA throughput of this GPU
// (the "alu" roofline denominators of DESIGN.md).  Independent chains per
// thread, full occupancy, CUDA-event timed.
#include <cstdio>
#include <cuda_runtime.h>

template <typename T, int CH>
__global__ void fma_loop(T* out, int iters, T a, T b) {
    T x[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = T(threadIdx.x + i);
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) x[i] = fma(x[i], a, b);
    T s = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s += x[i];
    if (s == T(-1.2345)) out[threadIdx.x] = s;
}

__global__ void ffma2_loop(float* out, int iters, float a, float b) {
    float2 x[8];
    for (int i = 0; i < 8; ++i) x[i] = make_float2(threadIdx.x + i, i);
    float2 A = make_float2(a, a), B = make_float2(b, b);
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __ffma2_rn(x[i], A, B);
    float s = 0;
    for (int i = 0; i < 8; ++i) s += x[i].x + x[i].y;
    if (s == -1.2345f) out[threadIdx.x] = s;
}

template <typename K>
double run(K k, int blocks, int threads, int iters, double fma_per_thread_iter) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k(blocks, threads, iters);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k(blocks, threads, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return 5.0 * blocks * threads * (double)iters * fma_per_thread_iter / (ms * 1e-3) / 1e12;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* dout;
    float* fout;
    cudaMalloc(&dout, 4096 * 8);
    cudaMalloc(&fout, 4096 * 4);
    int blocks = sms * 8, threads = 256, iters = 4096;
    double d = run([&](int b, int t, int i) { fma_loop<double, 8><<<b, t>>>(dout, i, 1.0000001, 1e-7); }, blocks,
                   threads, iters, 8);
    double f = run([&](int b, int t, int i) { fma_loop<float, 8><<<b, t>>>(fout, i, 1.0000001f, 1e-7f); }, blocks,
                   threads, iters, 8);
    double f2 = run([&](int b, int t, int i) { ffma2_loop<<<b, t>>>(fout, i, 1.0000001f, 1e-7f); }, blocks, threads,
                    iters, 16);
    printf("{\"sms\": %d, \"fp64_tfma_s\": %.3f, \"fp32_tfma_s\": %.3f, \"fp32_ffma2_tfma_s\": %.3f}\n", sms, d, f, f2);
    return 0;
}

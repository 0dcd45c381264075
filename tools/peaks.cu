// Arithmetic peaks of this GPU for the roofline denominators: FP32 FFMA and FP64 DFMA
// throughput (independent FMA chains, all SMs, CUDA-event timed, best of several runs).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/peaks tools/peaks.cu
#include <cstdio>
#include <cuda_runtime.h>

template <typename T, int CH>
__global__ void __launch_bounds__(256) fma_loop(T *out, int iters, T a, T b)
{
    T x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = (T)(threadIdx.x + c);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = x[c] * a + b;
    }
    T s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    if (s == (T)-1234.5) out[threadIdx.x] = s;
}

template <typename T, int CH>
static double run(int sms, int iters)
{
    T *out;
    cudaMalloc(&out, 1024 * sizeof(T));
    const int blocks = sms * 8, threads = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    fma_loop<T, CH><<<blocks, threads>>>(out, iters / 10, (T)0.999999, (T)1e-7);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        fma_loop<T, CH><<<blocks, threads>>>(out, iters, (T)0.999999, (T)1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaFree(out);
    const double flops = 2.0 * CH * (double)iters * blocks * threads;
    return flops / (best * 1e-3) / 1e12;
}

int main()
{
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const double f32 = run<float, 16>(sms, 1 << 16);
    const double f64 = run<double, 8>(sms, 1 << 14);
    printf("{\"sms\": %d, \"clock_mhz\": %.0f, \"fp32_fma_tflops\": %.2f, \"fp64_fma_tflops\": %.2f}\n", sms,
           clk / 1000.0, f32, f64);
    return 0;
}

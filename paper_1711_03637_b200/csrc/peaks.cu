// Pipe-peak microbenchmarks for the roofline denominators (not product code).
// MEASURED_PEAKS.json carries HBM and bf16 tensor peaks only; the SNN kernels
// are bound by the FP64 (and integer/ALU) pipes, so bench.py measures the
// FP64 DFMA and FP32 FFMA peaks on the box in the same run.
#include <cuda_runtime.h>
#include <stdint.h>

template <typename T, int CH>
__global__ void __launch_bounds__(256) k_fma_peak(T *out, int iters, T a, T b) {
    T x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = (T)(threadIdx.x + c);
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = x[c] * a + b;
    T s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    if (s == (T)-1.2345) out[0] = s;  // keep the chains alive
}

template <typename T>
static double run(int iters) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    T *out;
    cudaMalloc(&out, sizeof(T));
    const int blocks = sms * 8, threads = 256;
    constexpr int CH = 8;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_fma_peak<T, CH><<<blocks, threads>>>(out, iters / 4, (T)0.999, (T)1e-3);  // warm-up
    cudaEventRecord(e0);
    k_fma_peak<T, CH><<<blocks, threads>>>(out, iters, (T)0.999, (T)1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaFree(out);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double flops = 2.0 * CH * (double)iters * blocks * threads;
    return flops / (ms * 1e-3) / 1e12;
}

extern "C" int snn_measure_fma_peaks(double *tflops_fp64, double *tflops_fp32) {
    *tflops_fp64 = run<double>(1 << 14);
    *tflops_fp32 = run<float>(1 << 15);
    return cudaGetLastError() == cudaSuccess ? 0 : 1002;
}

// ALU (integer / logic pipe) peak: independent LOP3 chains, 8 per thread, each
// step one 3-input LOP3 (x = (x ^ a) & (x | b)); returns lane-ops per second
// (x 1e12).  The guard-band hidden kernel is bound by this pipe.
__global__ void __launch_bounds__(256) k_alu_peak(uint32_t *out, int iters, uint32_t a, uint32_t b) {
    uint32_t x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 2654435761u + c;
#pragma unroll 8
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            uint32_t y;
            asm volatile("lop3.b32 %0, %1, %2, %3, 0x68;" : "=r"(y) : "r"(x[c]), "r"(a), "r"(b));
            x[c] = y;
        }
    uint32_t s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s ^= x[c];
    if (s == 0x12345678u) out[0] = s;
}

extern "C" int snn_measure_alu_peak(double *tops) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint32_t *out;
    cudaMalloc(&out, sizeof(uint32_t));
    const int blocks = sms * 8, threads = 256, iters = 1 << 15;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_alu_peak<<<blocks, threads>>>(out, iters / 4, 0x5bd1e995u, 0x9e3779b9u);
    cudaEventRecord(e0);
    k_alu_peak<<<blocks, threads>>>(out, iters, 0x5bd1e995u, 0x9e3779b9u);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaFree(out);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *tops = 8.0 * (double)iters * blocks * threads / (ms * 1e-3) / 1e12;
    return cudaGetLastError() == cudaSuccess ? 0 : 1002;
}

// Dependent-chain latency of one FP64 add/mul (cycles), single thread.
__global__ void k_dp_latency(double *out, long long *cycles, int iters, double a, double b) {
    double x = out[0];
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        x = __dadd_rn(x, a);
        x = __dmul_rn(x, b);
    }
    const long long t1 = clock64();
    out[1] = x;
    cycles[0] = t1 - t0;
}

extern "C" int snn_measure_dp_latency(double *cycles_per_op) {
    double *out;
    long long *cyc;
    cudaMalloc(&out, 2 * sizeof(double));
    cudaMalloc(&cyc, sizeof(long long));
    cudaMemset(out, 0, 2 * sizeof(double));
    const int iters = 4096;
    k_dp_latency<<<1, 1>>>(out, cyc, iters, 1e-3, 0.999);
    k_dp_latency<<<1, 1>>>(out, cyc, iters, 1e-3, 0.999);
    long long c = 0;
    cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    cudaFree(out);
    cudaFree(cyc);
    *cycles_per_op = (double)c / (2.0 * iters);
    return cudaGetLastError() == cudaSuccess ? 0 : 1002;
}

// peaks.cu -- microbenchmarks of the non-tensor FP32 pipe (FFMA, FFMA2), the
// FP64 pipe (DFMA) and legacy FP64 tensor MMA (DMMA m8n8k4) on this B200.
// They fill in the FP32 / FP64 roofline denominators MEASURED_PEAKS.json does
// not carry (it measures HBM copy and bf16 cuBLAS only).
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

template <int NACC>
__global__ void k_ffma(float *out, int iters, float a, float b) {
    float acc[NACC];
#pragma unroll
    for (int j = 0; j < NACC; ++j) acc[j] = threadIdx.x * 1e-7f + j;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < NACC; ++j) acc[j] = __fmaf_rn(acc[j], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < NACC; ++j) s += acc[j];
    if (s == 1234.5f) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void k_ffma2(float *out, int iters, float a, float b) {
    unsigned long long acc[NACC];
    unsigned long long aa, bb;
    asm("mov.b64 %0, {%1,%2};" : "=l"(aa) : "f"(a), "f"(a));
    asm("mov.b64 %0, {%1,%2};" : "=l"(bb) : "f"(b), "f"(b));
#pragma unroll
    for (int j = 0; j < NACC; ++j) {
        float x = threadIdx.x * 1e-7f + j;
        asm("mov.b64 %0, {%1,%2};" : "=l"(acc[j]) : "f"(x), "f"(x));
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < NACC; ++j) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(acc[j]) : "l"(aa), "l"(bb));
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < NACC; ++j) {
        float x, y;
        asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(acc[j]));
        s += x + y;
    }
    if (s == 1234.5f) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void k_dfma(double *out, int iters, double a, double b) {
    double acc[NACC];
#pragma unroll
    for (int j = 0; j < NACC; ++j) acc[j] = threadIdx.x * 1e-7 + j;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < NACC; ++j) acc[j] = fma(acc[j], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < NACC; ++j) s += acc[j];
    if (s == 1234.5) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void k_dmma(double *out, int iters, double a, double b) {
    double c[NACC][2];
#pragma unroll
    for (int j = 0; j < NACC; ++j) c[j][0] = c[j][1] = threadIdx.x * 1e-9 + j;
    double av = a + threadIdx.x * 1e-12, bv = b;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < NACC; ++j)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[j][0]), "+d"(c[j][1])
                         : "d"(av), "d"(bv));
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < NACC; ++j) s += c[j][0] + c[j][1];
    if (s == 1234.5) out[threadIdx.x] = s;
}

template <typename F>
float timeit(F &&launch) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ms;
}

}  // namespace

// Each returns achieved TFLOP/s (2 flops per FMA; DMMA m8n8k4 = 256 FMA per warp op).
extern "C" double peak_ffma(int blocks, int threads, int iters) {
    float *o;
    cudaMalloc(&o, 4096);
    float ms = timeit([&] { k_ffma<16><<<blocks, threads>>>(o, iters, 0.999f, 1e-3f); });
    cudaFree(o);
    return 2.0 * 16.0 * blocks * threads * (double)iters / (ms * 1e-3) / 1e12;
}
extern "C" double peak_ffma2(int blocks, int threads, int iters) {
    float *o;
    cudaMalloc(&o, 4096);
    float ms = timeit([&] { k_ffma2<8><<<blocks, threads>>>(o, iters, 0.999f, 1e-3f); });
    cudaFree(o);
    return 2.0 * 16.0 * blocks * threads * (double)iters / (ms * 1e-3) / 1e12;
}
extern "C" double peak_dfma(int blocks, int threads, int iters) {
    double *o;
    cudaMalloc(&o, 8192);
    float ms = timeit([&] { k_dfma<8><<<blocks, threads>>>(o, iters, 0.999, 1e-3); });
    cudaFree(o);
    return 2.0 * 8.0 * blocks * threads * (double)iters / (ms * 1e-3) / 1e12;
}
extern "C" double peak_dmma(int blocks, int threads, int iters) {
    double *o;
    cudaMalloc(&o, 8192);
    float ms = timeit([&] { k_dmma<8><<<blocks, threads>>>(o, iters, 0.999, 1e-3); });
    cudaFree(o);
    const double warps = blocks * (threads / 32.0);
    return 2.0 * 256.0 * 8.0 * warps * (double)iters / (ms * 1e-3) / 1e12;
}
extern "C" int last_error() { return (int)cudaGetLastError(); }

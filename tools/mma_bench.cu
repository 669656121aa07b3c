// Throughput of legacy warp-level mma.sync on sm_100a (TF32 m16n8k8, BF16 m16n8k16,
// FP64 m8n8k4) vs FFMA, one kernel each, all SMs, independent accumulators.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_tf32(float *out, int iters) {
    float c[8][4] = {};
    unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(c[q][0]), "+f"(c[q][1]), "+f"(c[q][2]), "+f"(c[q][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1] + c[q][2] + c[q][3];
    if (s == 123.f) out[0] = s;
}
__global__ void k_bf16(float *out, int iters) {
    float c[8][4] = {};
    unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(c[q][0]), "+f"(c[q][1]), "+f"(c[q][2]), "+f"(c[q][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1] + c[q][2] + c[q][3];
    if (s == 123.f) out[0] = s;
}
int main() {
    float *o;
    cudaMalloc(&o, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int iters = 20000;
    for (int w : {4, 8, 16}) {
        dim3 g(148 * 2), b(32 * w);
        k_tf32<<<g, b>>>(o, 100);
        cudaEventRecord(e0);
        k_tf32<<<g, b>>>(o, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 16 * 8 * 8 * 8 * (double)iters * g.x * w;
        printf("tf32 mma.sync warps/CTA %d: %.1f TFLOP/s\n", w, fl / ms / 1e9);
        k_bf16<<<g, b>>>(o, 100);
        cudaEventRecord(e0);
        k_bf16<<<g, b>>>(o, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        fl = 2.0 * 16 * 8 * 16 * 8 * (double)iters * g.x * w;
        printf("bf16 mma.sync warps/CTA %d: %.1f TFLOP/s\n", w, fl / ms / 1e9);
    }
    return 0;
}

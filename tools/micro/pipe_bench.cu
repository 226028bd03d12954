// Throughput probes on the B200: FFMA, FFMA2 and mma.sync m16n8k8 tf32 / m16n8k16 bf16.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_ffma(float* out, int iters) {
    float a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
    const float b = 1.0001f, c = 0.999f;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], b, c);
    float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__device__ __forceinline__ unsigned long long f2(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d;
}
__global__ void k_ffma2(float* out, int iters) {
    unsigned long long a[8];
    for (int i = 0; i < 8; ++i) { float2 v = make_float2(threadIdx.x * 1e-3f + i, i); a[i] = *reinterpret_cast<unsigned long long*>(&v); }
    float2 bv = make_float2(1.0001f, 1.0001f), cv = make_float2(0.999f, 0.999f);
    unsigned long long b = *reinterpret_cast<unsigned long long*>(&bv), c = *reinterpret_cast<unsigned long long*>(&cv);
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = f2(a[i], b, c);
    float s = 0; for (int i = 0; i < 8; ++i) { float2 v = *reinterpret_cast<float2*>(&a[i]); s += v.x + v.y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_mma_tf32(float* out, int iters) {
    unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
    float d[4][4] = {};
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 4; ++i)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(d[i][0]), "+f"(d[i][1]), "+f"(d[i][2]), "+f"(d[i][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    float s = 0; for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) s += d[i][j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_mma_bf16(float* out, int iters) {
    unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
    float d[4][4] = {};
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 4; ++i)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(d[i][0]), "+f"(d[i][1]), "+f"(d[i][2]), "+f"(d[i][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    float s = 0; for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) s += d[i][j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out; cudaMalloc(&out, 1 << 26);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    auto run = [&](const char* name, void (*k)(float*, int), double flop_per_inner) {
        k<<<blocks, threads>>>(out, 16);
        cudaEventRecord(e0);
        k<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double flop = double(blocks) * threads / 32 * iters * flop_per_inner;  // per warp
        printf("%-10s %8.3f ms  %8.1f TFLOP/s\n", name, ms, flop / ms / 1e9);
    };
    run("ffma", k_ffma, 8.0 * 32 * 2);
    run("ffma2", k_ffma2, 8.0 * 32 * 4);
    run("mma_tf32", k_mma_tf32, 4.0 * 16 * 8 * 8 * 2);
    run("mma_bf16", k_mma_bf16, 4.0 * 16 * 8 * 16 * 2);
    return 0;
}

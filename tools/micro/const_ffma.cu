// Throughput probe: a per-thread chain of 20x20 dense layers (the ARM's
// shape) with the weights read as FFMA constant-bank operands (c[0x3][imm])
// versus weights broadcast from shared memory (3-register FFMA, and FFMA2 on
// two latents per thread with duplicated weight pairs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o const_ffma const_ffma.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 20;
constexpr int MAXM = 6;  // matrices in the constant table (12 x 1.6 KB = 19.2 KB)
__constant__ float cw[MAXM][N][N];

template <int M>
__global__ void __launch_bounds__(128, 1) k_const(float* out, int iters) {
    float x[N];
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = (threadIdx.x + blockIdx.x) * 1e-4f + i * 1e-3f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int m = 0; m < M; ++m) {
            float y[N];
#pragma unroll
            for (int a = 0; a < N; ++a) {
                float s = 0.0f;
#pragma unroll
                for (int k = 0; k < N; ++k) s = fmaf(x[k], cw[m][a][k], s);
                y[a] = s;
            }
#pragma unroll
            for (int a = 0; a < N; ++a) x[a] = y[a];
        }
    }
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < N; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// same chain, the weights broadcast from shared memory (LDS.128, uniform address)
template <int M>
__global__ void __launch_bounds__(128, 1) k_smem(float* out, int iters) {
    __shared__ __align__(16) float sw[M][N][N];
    for (int e = threadIdx.x; e < M * N * N; e += blockDim.x) (&sw[0][0][0])[e] = (&cw[0][0][0])[e];
    __syncthreads();
    float x[N];
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = (threadIdx.x + blockIdx.x) * 1e-4f + i * 1e-3f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int m = 0; m < M; ++m) {
            float y[N];
#pragma unroll
            for (int a = 0; a < N; ++a) {
                float s = 0.0f;
#pragma unroll
                for (int k = 0; k < N; k += 4) {
                    const float4 w = *reinterpret_cast<const float4*>(&sw[m][a][k]);
                    s = fmaf(x[k], w.x, s);
                    s = fmaf(x[k + 1], w.y, s);
                    s = fmaf(x[k + 2], w.z, s);
                    s = fmaf(x[k + 3], w.w, s);
                }
                y[a] = s;
            }
#pragma unroll
            for (int a = 0; a < N; ++a) x[a] = y[a];
        }
    }
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < N; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ unsigned long long f2(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}

// two latents per thread (FFMA2 lanes), duplicated weight pairs from shared memory
template <int M>
__global__ void __launch_bounds__(128, 1) k_ffma2(float* out, int iters) {
    __shared__ __align__(16) float2 sw[M][N][N];
    for (int e = threadIdx.x; e < M * N * N; e += blockDim.x) {
        const float w = (&cw[0][0][0])[e];
        (&sw[0][0][0])[e] = make_float2(w, w);
    }
    __syncthreads();
    unsigned long long x[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
        float2 v = make_float2((threadIdx.x + blockIdx.x) * 1e-4f + i * 1e-3f, i * 2e-3f);
        x[i] = *reinterpret_cast<unsigned long long*>(&v);
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int m = 0; m < M; ++m) {
            unsigned long long y[N];
#pragma unroll
            for (int a = 0; a < N; ++a) {
                unsigned long long s = 0ull;
#pragma unroll
                for (int k = 0; k < N; k += 2) {
                    const ulonglong2 w = *reinterpret_cast<const ulonglong2*>(&sw[m][a][k]);
                    s = f2(x[k], w.x, s);
                    s = f2(x[k + 1], w.y, s);
                }
                y[a] = s;
            }
#pragma unroll
            for (int a = 0; a < N; ++a) x[a] = y[a];
        }
    }
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        float2 v = *reinterpret_cast<float2*>(&x[i]);
        s += v.x + v.y;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}


// two latents per thread, weight pairs (w, w) built from the constant bank
template <int M>
__global__ void __launch_bounds__(128, 1) k_const2(float* out, int iters) {
    unsigned long long x[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
        float2 v = make_float2((threadIdx.x + blockIdx.x) * 1e-4f + i * 1e-3f, i * 2e-3f);
        x[i] = *reinterpret_cast<unsigned long long*>(&v);
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int m = 0; m < M; ++m) {
            unsigned long long y[N];
#pragma unroll
            for (int a = 0; a < N; ++a) {
                unsigned long long s = 0ull;
#pragma unroll
                for (int k = 0; k < N; ++k) {
                    unsigned long long w;
                    const float c = cw[m][a][k];
                    asm("mov.b64 %0, {%1, %1};" : "=l"(w) : "f"(c));
                    s = f2(x[k], w, s);
                }
                y[a] = s;
            }
#pragma unroll
            for (int a = 0; a < N; ++a) x[a] = y[a];
        }
    }
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        float2 v = *reinterpret_cast<float2*>(&x[i]);
        s += v.x + v.y;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// duplicated constant table: (w, w) pairs stored, read as 64-bit
__constant__ float2 cw2[4][N][N];
template <int M>
__global__ void __launch_bounds__(128, 1) k_const2d(float* out, int iters) {
    unsigned long long x[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
        float2 v = make_float2((threadIdx.x + blockIdx.x) * 1e-4f + i * 1e-3f, i * 2e-3f);
        x[i] = *reinterpret_cast<unsigned long long*>(&v);
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int m = 0; m < M; ++m) {
            unsigned long long y[N];
#pragma unroll
            for (int a = 0; a < N; ++a) {
                unsigned long long s = 0ull;
#pragma unroll
                for (int k = 0; k < N; ++k) {
                    const float2 c = cw2[m][a][k];
                    s = f2(x[k], *reinterpret_cast<const unsigned long long*>(&c), s);
                }
                y[a] = s;
            }
#pragma unroll
            for (int a = 0; a < N; ++a) x[a] = y[a];
        }
    }
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        float2 v = *reinterpret_cast<float2*>(&x[i]);
        s += v.x + v.y;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}


// runtime (warp-uniform) slot index into a larger constant table
__constant__ float cws[6 * 1536];
template <int M>
__global__ void __launch_bounds__(128, 1) k_slot(float* out, int iters) {
    const float* w = cws + (iters & 3) * 1536;
    unsigned long long x[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
        float2 v = make_float2((threadIdx.x + blockIdx.x) * 1e-4f + i * 1e-3f, i * 2e-3f);
        x[i] = *reinterpret_cast<unsigned long long*>(&v);
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int m = 0; m < M; ++m) {
            unsigned long long y[N];
#pragma unroll
            for (int a = 0; a < N; ++a) {
                unsigned long long s = 0ull;
#pragma unroll
                for (int k = 0; k < N; ++k) {
                    unsigned long long ww;
                    const float c = w[(m * N + a) * N + k];
                    asm("mov.b64 %0, {%1, %1};" : "=l"(ww) : "f"(c));
                    s = f2(x[k], ww, s);
                }
                y[a] = s;
            }
#pragma unroll
            for (int a = 0; a < N; ++a) x[a] = y[a];
        }
    }
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        float2 v = *reinterpret_cast<float2*>(&x[i]);
        s += v.x + v.y;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename Kern>
void run(const char* name, Kern k, int blocks, int iters, double fma_per_thread, float* out, int nt = 128) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<<<blocks, nt>>>(out, 1);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    k<<<blocks, nt>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flop = 2.0 * fma_per_thread * iters * blocks * double(nt);
    printf("%-22s nt %3d blocks %5d  %8.3f ms  %7.2f TFLOP/s  err=%s\n", name, nt, blocks, ms, flop / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    static float h[MAXM][N][N];
    for (int m = 0; m < MAXM; ++m)
        for (int a = 0; a < N; ++a)
            for (int k = 0; k < N; ++k) h[m][a][k] = ((m * 7 + a * 3 + k) % 11 - 5) * 0.009f;
    cudaMemcpyToSymbol(cw, h, sizeof(h));
    static float2 h2[4][N][N];
    for (int m = 0; m < 4; ++m) for (int a = 0; a < N; ++a) for (int k = 0; k < N; ++k) h2[m][a][k] = make_float2(h[m][a][k], h[m][a][k]);
    cudaMemcpyToSymbol(cw2, h2, sizeof(h2));
    static float hs[6 * 1536]; for (int i = 0; i < 6 * 1536; ++i) hs[i] = (&h[0][0][0])[i % (MAXM * N * N)];
    cudaMemcpyToSymbol(cws, hs, sizeof(hs));
    float* out;
    cudaMalloc(&out, 148 * 64 * 128 * sizeof(float));
    const int it = 200;
    for (int bpsm : {4, 8, 16}) {
        const int b = 148 * bpsm;
        run("const M=2 (3.2KB)", k_const<2>, b, it * 3, 2.0 * N * N, out);
        run("const M=4 (6.4KB)", k_const<4>, b, it * 3 / 2, 4.0 * N * N, out);
        run("const M=6 (9.6KB)", k_const<6>, b, it, 6.0 * N * N, out);
        run("const M=6b", k_const<6>, b, it / 2, 12.0 * N * N, out);
        run("const FFMA2 M=2", k_const2<2>, b, it * 3, 4.0 * N * N, out);
        run("const FFMA2 M=4", k_const2<4>, b, it * 3 / 2, 8.0 * N * N, out);
        run("const2d FFMA2 M=2", k_const2d<2>, b, it * 3, 4.0 * N * N, out);
        run("const2d FFMA2 M=4", k_const2d<4>, b, it * 3 / 2, 8.0 * N * N, out);
        run("slot FFMA2 M=2", k_slot<2>, b, it * 3, 4.0 * N * N, out);
        run("slot FFMA2 M=4", k_slot<4>, b, it * 3 / 2, 8.0 * N * N, out);
    }
    for (int bpsm : {2, 3, 4, 6}) {
        run("lowocc FFMA2 M=2", k_const2<2>, 148 * bpsm, it * 3, 4.0 * N * N, out, 64);
        run("lowocc FFMA2 M=4", k_const2<4>, 148 * bpsm, it * 3 / 2, 8.0 * N * N, out, 64);
        run("lowocc slot M=2", k_slot<2>, 148 * bpsm, it * 3, 4.0 * N * N, out, 64);
        run("lowocc slot M=4", k_slot<4>, 148 * bpsm, it * 3 / 2, 8.0 * N * N, out, 64);
    }
    return 0;
}

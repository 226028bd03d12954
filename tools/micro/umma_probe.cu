// umma_probe.cu — validates the tcgen05 primitives of cc_umma.cuh on a B200:
//   1. K-major A [128 x 24] x K-major B [32 x 24] (per-latent layer shape),
//      exact small-integer inputs -> bit-exact result expected;
//   2. the SAME tile bytes read MN-major: D[feat][feat2] = sum over 128
//      latents (weight-gradient shape, M = 128, N = 32, K = 128);
//   3. 3xTF32 split on random fp32 vs fp64 (and plain 1xTF32) — error report;
//   4. raw fp32 bits fed as tf32: truncation or rounding?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_probe umma_probe.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_2605_02726_b200/csrc/cc_umma.cuh"

using namespace ccb;

constexpr int KC1 = 6;    // 24 / 4
constexpr int KCA = 32;   // 128 / 4 (activation tile for test 2: 128 features)
constexpr int KCB = 8;    // 32 / 4

struct Smem {
    alignas(128) float A[128 * 24];     // test 1/3 A (hi)
    alignas(128) float Alo[128 * 24];
    alignas(128) float B[32 * 24];
    alignas(128) float Blo[32 * 24];
    alignas(128) float X[128 * 128];    // test 2: [lat][128 feat]
    alignas(128) float Y[128 * 32];     // test 2: [lat][32 feat]
    uint64_t mbar;
    uint32_t tmem;
};

__global__ void k_probe(const float* a, const float* b, const float* x, const float* y, float* out1,
                        float* out2, float* out3, float* out4, int mode) {
    extern __shared__ __align__(1024) unsigned char raw[];
    Smem& s = *reinterpret_cast<Smem*>(raw);
    const int tid = threadIdx.x, warp = tid >> 5;
    if (warp == 0) umma::tmem_alloc(&s.tmem, 256);
    if (tid == 0) umma::mbar_init(&s.mbar, 1);
    // fill tiles: logical a[r][k] (row-major 128 x 24), b[n][k] (32 x 24)
    for (int e = tid; e < 128 * 24; e += blockDim.x) {
        const int r = e / 24, k = e % 24;
        float hi, lo;
        if (mode == 2) {  // raw fp32 into the operand (hardware rounding test)
            hi = a[e];
            lo = 0.0f;
        } else {
            umma::split(a[e], hi, lo);
        }
        s.A[umma::tile_off(r, k, KC1) / 4] = hi;
        s.Alo[umma::tile_off(r, k, KC1) / 4] = lo;
    }
    for (int e = tid; e < 32 * 24; e += blockDim.x) {
        const int n = e / 24, k = e % 24;
        float hi, lo;
        if (mode == 2) {
            hi = b[e];
            lo = 0.0f;
        } else {
            umma::split(b[e], hi, lo);
        }
        s.B[umma::tile_off(n, k, KC1) / 4] = hi;
        s.Blo[umma::tile_off(n, k, KC1) / 4] = lo;
    }
    for (int e = tid; e < 128 * 128; e += blockDim.x) {
        const int l = e / 128, f = e % 128;
        s.X[umma::tile_off(l, f, KCA) / 4] = x[e];
    }
    for (int e = tid; e < 128 * 32; e += blockDim.x) {
        const int l = e / 32, f = e % 32;
        s.Y[umma::tile_off(l, f, KCB) / 4] = y[e];
    }
    umma::fence_async_smem();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tm = s.tmem;
    if (tid == 0) {
        // test 1 / 3: D0 (cols 0..31) = A*B^T, 3 k-steps; D1 (cols 32..63) = 3xTF32 split
        const uint32_t id = umma::idesc_tf32(128, 32, false, false);
        for (int ks = 0; ks < 3; ++ks) {
            const uint32_t koff = ks * 256;  // 2 core columns of 128 B
            umma::mma_tf32(tm, umma::desc(umma::smem_u32(s.A) + koff, 128, KC1 * 128),
                           umma::desc(umma::smem_u32(s.B) + koff, 128, KC1 * 128), id, ks > 0);
        }
        for (int ks = 0; ks < 3; ++ks) {
            const uint32_t koff = ks * 256;
            const uint64_t ah = umma::desc(umma::smem_u32(s.A) + koff, 128, KC1 * 128);
            const uint64_t al = umma::desc(umma::smem_u32(s.Alo) + koff, 128, KC1 * 128);
            const uint64_t bh = umma::desc(umma::smem_u32(s.B) + koff, 128, KC1 * 128);
            const uint64_t bl = umma::desc(umma::smem_u32(s.Blo) + koff, 128, KC1 * 128);
            umma::mma_tf32(tm + 32, al, bh, id, ks > 0);
            umma::mma_tf32(tm + 32, ah, bl, id, 1);
            umma::mma_tf32(tm + 32, ah, bh, id, 1);
        }
        // test 2: D2 (cols 64..95) [feat 128][feat2 32] = X^T Y over 128 latents, MN-major reads
        // variant a (cols 64..95): LBO = K-group stride, SBO = MN-chunk stride
        // variant b (cols 96..127): swapped
        const uint32_t id2 = umma::idesc_tf32(128, 32, true, true);
        for (int ks = 0; ks < 16; ++ks) {  // 8 latents per k-step
            umma::mma_tf32(tm + 64, umma::desc(umma::smem_u32(s.X) + ks * KCA * 128, KCA * 128, 128),
                           umma::desc(umma::smem_u32(s.Y) + ks * KCB * 128, KCB * 128, 128), id2, ks > 0);
            umma::mma_tf32(tm + 96, umma::desc(umma::smem_u32(s.X) + ks * KCA * 128, 128, KCA * 128),
                           umma::desc(umma::smem_u32(s.Y) + ks * KCB * 128, 128, KCB * 128), id2, ks > 0);
        }
        // test 5: M = 64 K-major (A rows 0..63 of the test-1 tile) -> cols 128..159
        umma::mma_tf32(tm + 128, umma::desc(umma::smem_u32(s.A), 128, KC1 * 128),
                       umma::desc(umma::smem_u32(s.B), 128, KC1 * 128), umma::idesc_tf32(64, 32, false, false), 0);
        // test 6: M = 128, N = 56 (N % 16 != 0) K-major -> cols 160..215, B rows beyond 32 read Y
        umma::mma_tf32(tm + 160, umma::desc(umma::smem_u32(s.A), 128, KC1 * 128),
                       umma::desc(umma::smem_u32(s.B), 128, KC1 * 128), umma::idesc_tf32(128, 56, false, false), 0);
        umma::commit(&s.mbar);
    }
    umma::mbar_wait(&s.mbar, 0);
    umma::fence_after_sync();
    const int row = (warp & 3) * 32 + (tid & 31);
    const uint32_t ta = tm + (uint32_t((warp & 3) * 32) << 16);
    float v[32];
    umma::ld32(ta, v);
    umma::wait_ld();
    for (int j = 0; j < 32; ++j) out1[row * 32 + j] = v[j];
    umma::ld32(ta + 32, v);
    umma::wait_ld();
    for (int j = 0; j < 32; ++j) out3[row * 32 + j] = v[j];
    umma::ld32(ta + 64, v);
    umma::wait_ld();
    for (int j = 0; j < 32; ++j) out2[row * 32 + j] = v[j];
    umma::ld32(ta + 96, v);
    umma::wait_ld();
    for (int j = 0; j < 32; ++j) out4[row * 96 + j] = v[j];
    umma::ld32(ta + 128, v);
    umma::wait_ld();
    for (int j = 0; j < 32; ++j) out4[row * 96 + 32 + j] = v[j];
    umma::ld32(ta + 160, v);
    umma::wait_ld();
    for (int j = 0; j < 32; ++j) out4[row * 96 + 64 + j] = v[j];
    umma::fence_before_sync();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc(tm, 256);
}

static float trunc_tf32(float x) {
    unsigned u;
    memcpy(&u, &x, 4);
    u &= 0xFFFFE000u;
    float r;
    memcpy(&r, &u, 4);
    return r;
}
static float round_tf32(float x) {
    unsigned u;
    memcpy(&u, &x, 4);
    u = (u + 0x1000u) & 0xFFFFE000u;
    float r;
    memcpy(&r, &u, 4);
    return r;
}

int main() {
    std::vector<float> a(128 * 24), b(32 * 24), x(128 * 128), y(128 * 32);
    srand(1);
    auto rnd = [] { return (rand() / float(RAND_MAX)) * 2.0f - 1.0f; };
    float *da, *db, *dx, *dy, *o1, *o2, *o3, *o4;
    cudaMalloc(&da, a.size() * 4);
    cudaMalloc(&db, b.size() * 4);
    cudaMalloc(&dx, x.size() * 4);
    cudaMalloc(&dy, y.size() * 4);
    cudaMalloc(&o1, 128 * 32 * 4);
    cudaMalloc(&o2, 128 * 32 * 4);
    cudaMalloc(&o3, 128 * 32 * 4);
    cudaMalloc(&o4, 128 * 96 * 4);
    const int smem = sizeof(Smem);
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    std::vector<float> r1(128 * 32), r2(128 * 32), r3(128 * 32);
    int fails = 0;
    for (int mode = 0; mode < 3; ++mode) {
        // mode 0: exact small integers; mode 1: random fp32; mode 2: random fp32 raw (rounding test)
        for (int i = 0; i < 128 * 24; ++i)
            a[i] = mode == 0 ? float((i * 7 % 11) - 5) * 0.25f : rnd();
        for (int i = 0; i < 32 * 24; ++i) b[i] = mode == 0 ? float((i * 5 % 13) - 6) * 0.5f : rnd();
        for (int i = 0; i < 128 * 128; ++i) x[i] = float((i * 3 % 7) - 3);
        for (int i = 0; i < 128 * 32; ++i) y[i] = float((i * 5 % 9) - 4) * 0.5f;
        cudaMemcpy(da, a.data(), a.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(db, b.data(), b.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dy, y.data(), y.size() * 4, cudaMemcpyHostToDevice);
        k_probe<<<1, 128, smem>>>(da, db, dx, dy, o1, o2, o3, o4, mode);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("mode %d: CUDA error %s\n", mode, cudaGetErrorString(e));
            return 2;
        }
        cudaMemcpy(r1.data(), o1, r1.size() * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(r2.data(), o2, r2.size() * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(r3.data(), o3, r3.size() * 4, cudaMemcpyDeviceToHost);
        double e1 = 0, e3 = 0, e1n = 0, eT = 0, eR = 0, nrm = 0;
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < 32; ++n) {
                double ex = 0, et = 0, er = 0;
                for (int k = 0; k < 24; ++k) {
                    ex += double(a[m * 24 + k]) * double(b[n * 24 + k]);
                    et += double(trunc_tf32(a[m * 24 + k])) * double(trunc_tf32(b[n * 24 + k]));
                    er += double(round_tf32(a[m * 24 + k])) * double(round_tf32(b[n * 24 + k]));
                }
                e1 = fmax(e1, fabs(r1[m * 32 + n] - ex));
                e3 = fmax(e3, fabs(r3[m * 32 + n] - ex));
                eT = fmax(eT, fabs(r1[m * 32 + n] - et));
                eR = fmax(eR, fabs(r1[m * 32 + n] - er));
                nrm = fmax(nrm, fabs(ex));
            }
        (void)e1n;
        std::vector<float> r4(128 * 96);
        cudaMemcpy(r4.data(), o4, r4.size() * 4, cudaMemcpyDeviceToHost);
        double e2b = 0, e6 = 0;
        for (int f = 0; f < 128; ++f)
            for (int g = 0; g < 32; ++g) {
                double ex = 0;
                for (int l = 0; l < 128; ++l) ex += double(x[l * 128 + f]) * double(y[l * 32 + g]);
                e2b = fmax(e2b, fabs(r4[f * 96 + g] - ex));
            }
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < 32; ++n) e6 = fmax(e6, fabs(r4[m * 96 + 64 + n] - r1[m * 32 + n]));
        if (mode == 0) {
            // M = 64: where does row m land?  print lane of rows 0..63 by matching column 0..3
            printf("M=64 rows -> lanes:");
            for (int m = 0; m < 64; ++m) {
                int hit = -1;
                for (int ln = 0; ln < 128 && hit < 0; ++ln) {
                    bool ok = true;
                    for (int n = 0; n < 32; ++n) ok = ok && r4[ln * 96 + 32 + n] == r1[m * 32 + n];
                    if (ok) hit = ln;
                }
                printf(" %d", hit);
            }
            printf("\n");
        }
        printf("mode %d: MN-major swapped |D2b-exact| %.3e ; N=56 vs N=32 |diff| %.3e\n", mode, e2b, e6);
        double e2 = 0;
        for (int f = 0; f < 128; ++f)
            for (int g = 0; g < 32; ++g) {
                double ex = 0;
                for (int l = 0; l < 128; ++l) ex += double(x[l * 128 + f]) * double(y[l * 32 + g]);
                e2 = fmax(e2, fabs(r2[f * 32 + g] - ex));
            }
        printf("mode %d: |D1-exact| %.3e  |D3(3xTF32)-exact| %.3e  |D1-trunc| %.3e |D1-round| %.3e  "
               "max|D| %.3e  |D2(MN-major)-exact| %.3e\n",
               mode, e1, e3, eT, eR, nrm, e2);
        if (mode == 0 && (e1 != 0 || e2 != 0 || e3 != 0)) ++fails;
        if (mode == 1 && e3 > 1e-5 * nrm) ++fails;
        if (e2 != 0 && e2b != 0) ++fails;
    }
    printf(fails ? "UMMA PROBE FAIL\n" : "UMMA PROBE OK\n");
    return fails ? 1 : 0;
}

// umma_probe3.cu — (1) A operand from TMEM (tcgen05.st by the owning lane,
// "ts" MMA form) vs the smem form; (2) truncation vs round-to-nearest 3xTF32
// split accuracy on random fp32 vs fp64; (3) the M = 64 accumulator lane map
// with distinct values.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_2605_02726_b200/csrc/cc_umma.cuh"

using namespace ccb;
constexpr int KC = 6;  // K = 24

struct Smem {
    alignas(128) float A[2][128 * 24];
    alignas(128) float B[2][32 * 24];
    uint64_t mbar;
    uint32_t tmem;
};

// mode 0: trunc split smem A; 1: rn split smem A; 2: rn split, A from TMEM; 3: M=64 (plain, smem)
__global__ void k(const float* a, const float* b, float* out, int mode) {
    extern __shared__ __align__(1024) unsigned char raw[];
    Smem& s = *reinterpret_cast<Smem*>(raw);
    const int tid = threadIdx.x, warp = tid >> 5;
    if (warp == 0) umma::tmem_alloc(&s.tmem, 256);
    if (tid == 0) umma::mbar_init(&s.mbar, 1);
    __syncthreads();
    const uint32_t tm = s.tmem;
    const uint32_t tl = tm + (uint32_t((warp & 3) * 32) << 16);
    for (int e = tid; e < 128 * 24; e += 128) {
        const int r = e / 24, kk = e % 24;
        float h, l;
        if (mode == 0 || mode == 3) umma::split(a[e], h, l); else umma::split_rn(a[e], h, l);
        s.A[0][umma::tile_off(r, kk, KC) / 4] = h;
        s.A[1][umma::tile_off(r, kk, KC) / 4] = l;
    }
    for (int e = tid; e < 32 * 24; e += 128) {
        const int n = e / 24, kk = e % 24;
        float h, l;
        if (mode == 0 || mode == 3) umma::split(b[e], h, l); else umma::split_rn(b[e], h, l);
        s.B[0][umma::tile_off(n, kk, KC) / 4] = h;
        s.B[1][umma::tile_off(n, kk, KC) / 4] = l;
    }
    if (mode == 2) {  // this thread's row of A, hi at columns 128.., lo at 160..
        const int r = tid;
        float h[8], l[8];
        for (int c = 0; c < 3; ++c) {
            for (int i = 0; i < 8; ++i) umma::split_rn(a[r * 24 + 8 * c + i], h[i], l[i]);
            umma::st8(tl + 128 + 8 * c, h);
            umma::st8(tl + 160 + 8 * c, l);
        }
        umma::wait_st();
    }
    umma::fence_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    if (tid == 0) {
        umma::fence_after_sync();
        const uint32_t id = umma::idesc_tf32(mode == 3 ? 64 : 128, 32, false, false);
        for (int ks = 0; ks < 3; ++ks) {
            const uint32_t ko = ks * 256;
            const uint64_t ah = umma::desc(umma::smem_u32(s.A[0]) + ko, 128, KC * 128);
            const uint64_t al = umma::desc(umma::smem_u32(s.A[1]) + ko, 128, KC * 128);
            const uint64_t bh = umma::desc(umma::smem_u32(s.B[0]) + ko, 128, KC * 128);
            const uint64_t bl = umma::desc(umma::smem_u32(s.B[1]) + ko, 128, KC * 128);
            if (mode == 2) {
                umma::mma_tf32_ts(tm, tm + 160 + 8 * ks, bh, id, ks > 0);
                umma::mma_tf32_ts(tm, tm + 128 + 8 * ks, bl, id, 1);
                umma::mma_tf32_ts(tm, tm + 128 + 8 * ks, bh, id, 1);
            } else if (mode == 3) {
                umma::mma_tf32(tm, ah, bh, id, ks > 0);
            } else {
                umma::mma_tf32(tm, al, bh, id, ks > 0);
                umma::mma_tf32(tm, ah, bl, id, 1);
                umma::mma_tf32(tm, ah, bh, id, 1);
            }
        }
        umma::commit(&s.mbar);
    }
    umma::mbar_wait(&s.mbar, 0);
    umma::fence_after_sync();
    float v[32];
    umma::ld32(tl, v);
    umma::wait_ld();
    for (int j = 0; j < 32; ++j) out[tid * 32 + j] = v[j];
    umma::fence_before_sync();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc(tm, 256);
}

int main() {
    std::vector<float> a(128 * 24), b(32 * 24), o(128 * 32);
    srand(7);
    for (auto& x : a) x = (rand() / float(RAND_MAX)) * 2.0f - 1.0f;
    for (auto& x : b) x = (rand() / float(RAND_MAX)) * 2.0f - 1.0f;
    float *da, *db, *dout;
    cudaMalloc(&da, a.size() * 4);
    cudaMalloc(&db, b.size() * 4);
    cudaMalloc(&dout, o.size() * 4);
    cudaMemcpy(da, a.data(), a.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(db, b.data(), b.size() * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(Smem)));
    for (int mode = 0; mode < 4; ++mode) {
        k<<<1, 128, sizeof(Smem)>>>(da, db, dout, mode);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("mode %d: %s\n", mode, cudaGetErrorString(e)); return 2; }
        cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost);
        if (mode < 3) {
            double err = 0, ef = 0, nrm = 0;
            for (int m = 0; m < 128; ++m)
                for (int n = 0; n < 32; ++n) {
                    double ex = 0;
                    float f32 = 0.0f;
                    for (int kk = 0; kk < 24; ++kk) {
                        ex += double(a[m * 24 + kk]) * double(b[n * 24 + kk]);
                        f32 = fmaf(a[m * 24 + kk], b[n * 24 + kk], f32);
                    }
                    err += (o[m * 32 + n] - ex) * (o[m * 32 + n] - ex);
                    ef += (f32 - ex) * (f32 - ex);
                    nrm += ex * ex;
                }
            printf("mode %d (%s): rel L2 err vs fp64 %.3e   (sequential fp32 fmaf: %.3e)\n", mode,
                   mode == 0 ? "trunc split, smem A" : mode == 1 ? "rn split, smem A" : "rn split, TMEM A",
                   sqrt(err / nrm), sqrt(ef / nrm));
        } else {
            printf("M=64 rows -> lanes:");
            for (int m = 0; m < 64; ++m) {
                double ex0 = 0;
                for (int kk = 0; kk < 24; ++kk) {
                    unsigned u; memcpy(&u, &a[m * 24 + kk], 4); u &= 0xFFFFE000u; float ah; memcpy(&ah, &u, 4);
                    unsigned w; memcpy(&w, &b[kk], 4); w &= 0xFFFFE000u; float bh; memcpy(&bh, &w, 4);
                    ex0 += double(ah) * double(bh);
                }
                int hit = -1;
                for (int ln = 0; ln < 128; ++ln)
                    if (fabs(o[ln * 32] - ex0) < 1e-4) hit = ln;
                printf(" %d", hit);
            }
            printf("\n");
        }
    }
    return 0;
}

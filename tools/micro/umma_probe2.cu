// umma_probe2.cu — one tcgen05.mma configuration per launch, accumulator at
// TMEM column 0; dumps lanes 0..127 x columns 0..63 of TMEM for offline
// analysis (tools/micro/umma_probe2.py).  Inputs: X [128 lat][128 feat],
// Y [128 lat][64 feat] small integers, stored in the [r/8][k/4][r%8][k%4] tile
// layout of cc_umma.cuh, plus Xt / Yt = the same matrices transposed and
// stored with rows = features (so a K-major read over latents is possible).
//   cfg 0: K-major  A = X (rows lat, K = feat 0..23), B = Y (rows lat 0..31, K = feat 0..23) M128 N32
//   cfg 1: MN-major A = X, B = Y, K = lat 0..7, (LBO, SBO) = (KCX*128, 128), M128 N32
//   cfg 2: same, (LBO, SBO) = (128, KCX*128)
//   cfg 3: K-major  A = Xt (rows feat, K = lat 0..7), B = Yt, M128 N32  (the transposed reference)
//   cfg 4: M64 N32 K-major like cfg 0
//   cfg 5: M128 N56 K-major like cfg 0 (B rows 0..55)
//   cfg 6: M128 N48 K-major like cfg 0
//   cfg 7: MN-major A only (B = Yt K-major), (LBO, SBO) = (KCX*128, 128)
//   cfg 8: MN-major B only (A = Xt K-major), (LBO, SBO) = (KCY*128, 128)
//   cfg 9: MN-major A only, (128, KCX*128)
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "../../paper_2605_02726_b200/csrc/cc_umma.cuh"

using namespace ccb;

constexpr int KCX = 32;  // X: 128 features
constexpr int KCY = 16;  // Y: 64 features
constexpr int KCT = 32;  // Xt / Yt: 128 latents

struct Smem {
    alignas(128) float X[128 * 128];
    alignas(128) float Y[128 * 64];
    alignas(128) float Xt[128 * 128];  // rows = feature (128), K = latents (128)
    alignas(128) float Yt[64 * 128];   // rows = feature (64)
    alignas(128) float pad[4096];
    uint64_t mbar;
    uint32_t tmem;
};

__global__ void k_probe(const float* x, const float* y, float* out, int cfg) {
    extern __shared__ __align__(1024) unsigned char raw[];
    Smem& s = *reinterpret_cast<Smem*>(raw);
    const int tid = threadIdx.x, warp = tid >> 5;
    if (warp == 0) umma::tmem_alloc(&s.tmem, 128);
    if (tid == 0) umma::mbar_init(&s.mbar, 1);
    for (int e = tid; e < 128 * 128; e += blockDim.x) {
        const int l = e / 128, f = e % 128;
        s.X[umma::tile_off(l, f, KCX) / 4] = x[e];
        s.Xt[umma::tile_off(f, l, KCT) / 4] = x[e];
    }
    for (int e = tid; e < 128 * 64; e += blockDim.x) {
        const int l = e / 64, f = e % 64;
        s.Y[umma::tile_off(l, f, KCY) / 4] = y[e];
        s.Yt[umma::tile_off(f, l, KCT) / 4] = y[e];
    }
    for (int e = tid; e < 4096; e += blockDim.x) s.pad[e] = 0.0f;
    umma::fence_async_smem();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tm = s.tmem;
    if (tid == 0) {
        const uint32_t X = umma::smem_u32(s.X), Y = umma::smem_u32(s.Y);
        const uint32_t Xt = umma::smem_u32(s.Xt), Yt = umma::smem_u32(s.Yt);
        switch (cfg) {
            case 0:
                for (int ks = 0; ks < 3; ++ks)
                    umma::mma_tf32(tm, umma::desc(X + ks * 256, 128, KCX * 128), umma::desc(Y + ks * 256, 128, KCY * 128),
                                   umma::idesc_tf32(128, 32, false, false), ks > 0);
                break;
            case 1:
                umma::mma_tf32(tm, umma::desc(X, KCX * 128, 128), umma::desc(Y, KCY * 128, 128),
                               umma::idesc_tf32(128, 32, true, true), 0);
                break;
            case 2:
                umma::mma_tf32(tm, umma::desc(X, 128, KCX * 128), umma::desc(Y, 128, KCY * 128),
                               umma::idesc_tf32(128, 32, true, true), 0);
                break;
            case 3:
                umma::mma_tf32(tm, umma::desc(Xt, 128, KCT * 128), umma::desc(Yt, 128, KCT * 128),
                               umma::idesc_tf32(128, 32, false, false), 0);
                break;
            case 4:
                for (int ks = 0; ks < 3; ++ks)
                    umma::mma_tf32(tm, umma::desc(X + ks * 256, 128, KCX * 128), umma::desc(Y + ks * 256, 128, KCY * 128),
                                   umma::idesc_tf32(64, 32, false, false), ks > 0);
                break;
            case 5:
                for (int ks = 0; ks < 3; ++ks)
                    umma::mma_tf32(tm, umma::desc(X + ks * 256, 128, KCX * 128), umma::desc(Y + ks * 256, 128, KCY * 128),
                                   umma::idesc_tf32(128, 56, false, false), ks > 0);
                break;
            case 6:
                for (int ks = 0; ks < 3; ++ks)
                    umma::mma_tf32(tm, umma::desc(X + ks * 256, 128, KCX * 128), umma::desc(Y + ks * 256, 128, KCY * 128),
                                   umma::idesc_tf32(128, 48, false, false), ks > 0);
                break;
            case 7:
                umma::mma_tf32(tm, umma::desc(X, KCX * 128, 128), umma::desc(Yt, 128, KCT * 128),
                               umma::idesc_tf32(128, 32, true, false), 0);
                break;
            case 8:
                umma::mma_tf32(tm, umma::desc(Xt, 128, KCT * 128), umma::desc(Y, KCY * 128, 128),
                               umma::idesc_tf32(128, 32, false, true), 0);
                break;
            case 9:
                umma::mma_tf32(tm, umma::desc(X, 128, KCX * 128), umma::desc(Yt, 128, KCT * 128),
                               umma::idesc_tf32(128, 32, true, false), 0);
                break;
        }
        umma::commit(&s.mbar);
    }
    umma::mbar_wait(&s.mbar, 0);
    umma::fence_after_sync();
    const int row = (warp & 3) * 32 + (tid & 31);
    const uint32_t ta = tm + (uint32_t((warp & 3) * 32) << 16);
    float v[32];
    umma::ld32(ta, v);
    umma::wait_ld();
    for (int j = 0; j < 32; ++j) out[row * 64 + j] = v[j];
    umma::ld32(ta + 32, v);
    umma::wait_ld();
    for (int j = 0; j < 32; ++j) out[row * 64 + 32 + j] = v[j];
    umma::fence_before_sync();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc(tm, 128);
}

int main(int argc, char** argv) {
    const char* path = argc > 1 ? argv[1] : "umma_probe2.bin";
    std::vector<float> x(128 * 128), y(128 * 64);
    for (int i = 0; i < 128 * 128; ++i) x[i] = float((i * 37 + (i >> 7) * 11) % 17 - 8);
    for (int i = 0; i < 128 * 64; ++i) y[i] = float((i * 29 + (i >> 6) * 7) % 13 - 6);
    float *dx, *dy, *dout;
    cudaMalloc(&dx, x.size() * 4);
    cudaMalloc(&dy, y.size() * 4);
    cudaMalloc(&dout, 128 * 64 * 4);
    cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dy, y.data(), y.size() * 4, cudaMemcpyHostToDevice);
    const int smem = sizeof(Smem);
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    FILE* f = fopen(path, "wb");
    fwrite(x.data(), 4, x.size(), f);
    fwrite(y.data(), 4, y.size(), f);
    std::vector<float> out(128 * 64);
    for (int cfg = 0; cfg < 10; ++cfg) {
        cudaMemset(dout, 0xff, out.size() * 4);
        k_probe<<<1, 128, smem>>>(dx, dy, dout, cfg);
        cudaError_t e = cudaDeviceSynchronize();
        printf("cfg %d: %s\n", cfg, cudaGetErrorString(e));
        if (e != cudaSuccess) return 2;
        cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
        fwrite(out.data(), 4, out.size(), f);
    }
    fclose(f);
    return 0;
}

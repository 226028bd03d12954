// cc_syn.cu — synthesis forward + MSE + backward.
//
// Replaces synthesize_forward / synthesize_backward (synthesis.hpp:191-233),
// conv1x1_* (layers.hpp:196-250), conv3x3_* (layers.hpp:257-343), mse_*
// (layers.hpp:643-657) and the straight-through clamp (layers.hpp:661-664,
// synthesis.hpp:215).
//
//   k_syn_trunk_fwd   z -> relu(c1) -> c2 = t (3 planes); the F-wide hidden
//                     layer h1 never leaves registers (663 MAC/px HOP)
//   k_syn_post_fwd    residual 3x3 post filter i (replicate padding)
//   k_syn_out         + stabilizer, clamp, MSE partial (fp64), dx̂
//   k_syn_post_bwd    post filter i backward: gather-transposed conv + dW
//   k_syn_trunk_bwd   recompute h1, dh1, dz, and the c1/c2/stab weight
//                     gradients as per-tile shared-memory GEMMs (persistent
//                     CTAs, fixed-order fp64 accumulation; no atomics)
#include <cuda_runtime.h>

#include "cc_kernels.h"
#include "cc_math.cuh"
#include "cc_reduce.cuh"

namespace ccb {

namespace {

constexpr int kLZ = kMaxLevels;  // z vector padded to 8 channels
constexpr int kSynTile = 128;

__host__ __device__ constexpr int r4(int n) { return (n + 3) / 4 * 4; }
__host__ __device__ constexpr int oddc(int n) { return ((r4(n) / 4) % 2 == 0) ? r4(n) + 4 : r4(n); }

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// ---------------------------------------------------------------- trunk fwd
__global__ void __launch_bounds__(256) k_syn_trunk_fwd(const Plan* __restrict__ pp) {
    const Plan& P = *pp;
    __shared__ float c1w[64 * kLZ], c1b[64], c2w[3 * 64], c2b[4];
    const int L = P.L, F = P.syn_F;
    for (int e = threadIdx.x; e < 64 * kLZ; e += blockDim.x) {
        const int f = e / kLZ, k = e - f * kLZ;
        c1w[e] = (f < F && k < L) ? P.params[P.off_c1w + f * L + k] : 0.0f;
    }
    for (int e = threadIdx.x; e < 64; e += blockDim.x) c1b[e] = e < F ? P.params[P.off_c1b + e] : 0.0f;
    for (int e = threadIdx.x; e < 3 * 64; e += blockDim.x) {
        const int co = e / 64, f = e - co * 64;
        c2w[e] = f < F ? P.params[P.off_c2w + co * F + f] : 0.0f;
    }
    if (threadIdx.x < 4) c2b[threadIdx.x] = threadIdx.x < 3 ? P.params[P.off_c2b + threadIdx.x] : 0.0f;
    __syncthreads();
    const int64_t np = P.npix;
    for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < np;
         p += int64_t(gridDim.x) * blockDim.x) {
        float zv[kLZ];
#pragma unroll
        for (int k = 0; k < kLZ; ++k) zv[k] = k < L ? P.z[int64_t(k) * np + p] : 0.0f;
        float t0 = c2b[0], t1 = c2b[1], t2 = c2b[2];
        for (int f = 0; f < F; ++f) {
            float acc = c1b[f];
#pragma unroll
            for (int k = 0; k < kLZ; ++k) acc = fmaf(zv[k], c1w[f * kLZ + k], acc);
            const float h = acc > 0.0f ? acc : 0.0f;
            t0 = fmaf(c2w[f], h, t0);
            t1 = fmaf(c2w[64 + f], h, t1);
            t2 = fmaf(c2w[128 + f], h, t2);
        }
        P.syn_t[p] = t0;
        P.syn_t[np + p] = t1;
        P.syn_t[2 * np + p] = t2;
    }
}

// ---------------------------------------------------------- residual posts
__device__ __forceinline__ const float* post_in(const Plan& P, int i) {
    return i == 0 ? P.syn_t : P.syn_p[i - 1];
}

// conv3x3_forward (layers.hpp:257-300) + residual (synthesis.hpp:204-209)
__global__ void k_syn_post_fwd(const Plan* __restrict__ pp, int i) {
    const Plan& P = *pp;
    __shared__ float w[81], b[3];
    if (threadIdx.x < 81) w[threadIdx.x] = P.params[P.off_pw[i] + threadIdx.x];
    if (threadIdx.x < 3) b[threadIdx.x] = P.params[P.off_pb[i] + threadIdx.x];
    __syncthreads();
    const float* in = post_in(P, i);
    float* out = P.syn_p[i];
    const int H = P.H, W = P.W;
    const int64_t np = P.npix;
    for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < np;
         p += int64_t(gridDim.x) * blockDim.x) {
        const int r = int(p / W), c = int(p - int64_t(r) * W);
        const int rm = r > 0 ? r - 1 : 0, rp = r < H - 1 ? r + 1 : H - 1;
        const int cm = c > 0 ? c - 1 : 0, cp = c < W - 1 ? c + 1 : W - 1;
#pragma unroll
        for (int co = 0; co < 3; ++co) {
            float acc = b[co];
#pragma unroll
            for (int ci = 0; ci < 3; ++ci) {
                const float* k = w + (co * 3 + ci) * 9;
                const float* x = in + int64_t(ci) * np;
                const float* x0 = x + int64_t(rm) * W;
                const float* x1 = x + int64_t(r) * W;
                const float* x2 = x + int64_t(rp) * W;
                acc += k[0] * x0[cm] + k[1] * x0[c] + k[2] * x0[cp] + k[3] * x1[cm] + k[4] * x1[c] +
                       k[5] * x1[cp] + k[6] * x2[cm] + k[7] * x2[c] + k[8] * x2[cp];
            }
            out[int64_t(co) * np + p] = acc + in[int64_t(co) * np + p];
        }
    }
}

// x̂ = clamp01(posts + stab·z); MSE (double) and dx̂ = 2(x̂ - x)/(3HW)
// (synthesis.hpp:210-212, layers.hpp:643-657, encoder.hpp:256-260).
__global__ void __launch_bounds__(256) k_syn_out(const Plan* __restrict__ pp, int with_grad) {
    const Plan& P = *pp;
    __shared__ float st[3 * kLZ];
    __shared__ double red[8];
    const int L = P.L;
    if (threadIdx.x < 3 * kLZ) {
        const int co = threadIdx.x / kLZ, k = threadIdx.x - co * kLZ;
        st[threadIdx.x] = (P.off_sstab >= 0 && k < L) ? P.params[P.off_sstab + co * L + k] : 0.0f;
    }
    __syncthreads();
    const int64_t np = P.npix;
    const float* pl = P.posts > 0 ? P.syn_p[P.posts - 1] : P.syn_t;
    const float s = float(2.0 / double(3 * np));
    double acc = 0.0;
    for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < np;
         p += int64_t(gridDim.x) * blockDim.x) {
        float zv[kLZ];
#pragma unroll
        for (int k = 0; k < kLZ; ++k) zv[k] = k < L ? P.z[int64_t(k) * np + p] : 0.0f;
#pragma unroll
        for (int co = 0; co < 3; ++co) {
            float x = pl[int64_t(co) * np + p];
            if (P.off_sstab >= 0) {
#pragma unroll
                for (int k = 0; k < kLZ; ++k)
                    if (k < L) x += st[co * kLZ + k] * zv[k];
            }
            x = std_min(1.0f, std_max(0.0f, x));
            const float tgt = P.image[int64_t(co) * np + p];
            const double d = double(x) - double(tgt);
            acc += d * d;
            if (with_grad) P.syn_dx[int64_t(co) * np + p] = s * (x - tgt);
        }
    }
    const double tot = block_sum(acc, red);
    if (threadIdx.x == 0) P.mse_part[blockIdx.x] = tot;
}

// conv3x3_backward (layers.hpp:302-343) + residual path (synthesis.hpp:222-228)
__global__ void __launch_bounds__(256) k_syn_post_bwd(const Plan* __restrict__ pp, int i,
                                                      const float* __restrict__ dcur,
                                                      float* __restrict__ dprev) {
    const Plan& P = *pp;
    __shared__ float w[81];
    __shared__ double sbuf[84 * 8];
    __shared__ double tot[84];
    if (threadIdx.x < 81) w[threadIdx.x] = P.params[P.off_pw[i] + threadIdx.x];
    __syncthreads();
    const float* in = post_in(P, i);
    const int H = P.H, W = P.W;
    const int64_t np = P.npix;
    float acc[84];
#pragma unroll
    for (int k = 0; k < 84; ++k) acc[k] = 0.0f;
    for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < np;
         p += int64_t(gridDim.x) * blockDim.x) {
        const int r = int(p / W), c = int(p - int64_t(r) * W);
        const int rm = r > 0 ? r - 1 : 0, rp = r < H - 1 ? r + 1 : H - 1;
        const int cm = c > 0 ? c - 1 : 0, cp = c < W - 1 ? c + 1 : W - 1;
        // weight gradients (forward-direction loop)
#pragma unroll
        for (int co = 0; co < 3; ++co) {
            const float g = dcur[int64_t(co) * np + p];
            acc[81 + co] += g;
#pragma unroll
            for (int ci = 0; ci < 3; ++ci) {
                const float* x = in + int64_t(ci) * np;
                const float* x0 = x + int64_t(rm) * W;
                const float* x1 = x + int64_t(r) * W;
                const float* x2 = x + int64_t(rp) * W;
                float* dk = acc + (co * 3 + ci) * 9;
                dk[0] += g * x0[cm]; dk[1] += g * x0[c]; dk[2] += g * x0[cp];
                dk[3] += g * x1[cm]; dk[4] += g * x1[c]; dk[5] += g * x1[cp];
                dk[6] += g * x2[cm]; dk[7] += g * x2[c]; dk[8] += g * x2[cp];
            }
        }
        // input gradient by gather over the replicate-clamped neighbourhood
        int rr[3], dr[3], cc[3], dc[3];
        int nr = 0, nc = 0;
        for (int q = r - 1; q <= r + 1; ++q) {
            if (q < 0 || q >= H) continue;
            for (int d = -1; d <= 1; ++d)
                if (clampi(q + d, 0, H - 1) == r && nr < 3) { rr[nr] = q; dr[nr] = d; ++nr; }
        }
        for (int q = c - 1; q <= c + 1; ++q) {
            if (q < 0 || q >= W) continue;
            for (int d = -1; d <= 1; ++d)
                if (clampi(q + d, 0, W - 1) == c && nc < 3) { cc[nc] = q; dc[nc] = d; ++nc; }
        }
#pragma unroll
        for (int ci = 0; ci < 3; ++ci) {
            float s = 0.0f;
            for (int co = 0; co < 3; ++co) {
                const float* k = w + (co * 3 + ci) * 9;
                const float* g = dcur + int64_t(co) * np;
                for (int a = 0; a < nr; ++a)
                    for (int b = 0; b < nc; ++b)
                        s += k[(dr[a] + 1) * 3 + (dc[b] + 1)] * g[int64_t(rr[a]) * W + cc[b]];
            }
            dprev[int64_t(ci) * np + p] = s + dcur[int64_t(ci) * np + p];  // residual path
        }
    }
    double dacc[84];
#pragma unroll
    for (int k = 0; k < 84; ++k) dacc[k] = double(acc[k]);
    block_sum_vec<84>(dacc, sbuf, tot);
    __syncthreads();
    const PartialRegion& R = P.region[P.reg_post[i]];
    double* row = P.partials + R.base + int64_t(blockIdx.x) * R.count;
    for (int e = threadIdx.x; e < R.count; e += blockDim.x) {
        const int pidx = R.param_off + e;
        double v = 0.0;
        if (pidx >= P.off_pw[i] && pidx < P.off_pw[i] + 81) v = tot[pidx - P.off_pw[i]];
        else if (pidx >= P.off_pb[i] && pidx < P.off_pb[i] + 3) v = tot[81 + pidx - P.off_pb[i]];
        row[e] = v;
    }
}

// ----------------------------------------------------------- trunk backward
template <int FP>
struct TrunkCfg {
    static constexpr int LZ = oddc(kLZ + 1);   // z row, ones at kLZ
    static constexpr int LH = oddc(FP + 1);    // h1 row, ones at FP
    static constexpr int LDH = oddc(FP);       // dh1 row
    static constexpr int LT = 4;               // dt / dx̂ rows
    static constexpr int O_Z = 0;
    static constexpr int O_H = O_Z + kSynTile * LZ;
    static constexpr int O_DH = O_H + kSynTile * LH;
    static constexpr int O_DT = O_DH + kSynTile * LDH;
    static constexpr int O_DX = O_DT + kSynTile * LT;
    static constexpr int ACT = O_DX + kSynTile * LT;
    static constexpr int NJ1 = (FP / 2) * (r4(kLZ + 1) / 4);  // dh1 x [z|1]
    static constexpr int NJ2 = 2 * (r4(FP + 1) / 4);          // dt x [h1|1]
    static constexpr int NJ3 = 2 * (kLZ / 4);                 // dx̂ x z
    static constexpr int NJ = NJ1 + NJ2 + NJ3;
    static constexpr int NACC = FP * kLZ + FP + 3 * FP + 3 + 3 * kLZ;
};

template <int FP>
struct alignas(16) TrunkSmem {
    using K = TrunkCfg<FP>;
    alignas(16) float c1w[FP * kLZ];
    alignas(16) float c1b[FP];
    alignas(16) float c2w[3 * FP];
    alignas(16) float st[3 * kLZ];
    alignas(16) float act[K::ACT];
    alignas(16) double acc[K::NACC];
};

template <int LDA, int LDB>
__device__ __forceinline__ void syn_mt(const float* __restrict__ A, const float* __restrict__ B,
                                       int a0, int b0, float (&acc)[8]) {
#pragma unroll 4
    for (int i = 0; i < kSynTile; ++i) {
        const float2 av = *reinterpret_cast<const float2*>(A + i * LDA + a0);
        const float4 bv = *reinterpret_cast<const float4*>(B + i * LDB + b0);
        acc[0] = fmaf(av.x, bv.x, acc[0]);
        acc[1] = fmaf(av.x, bv.y, acc[1]);
        acc[2] = fmaf(av.x, bv.z, acc[2]);
        acc[3] = fmaf(av.x, bv.w, acc[3]);
        acc[4] = fmaf(av.y, bv.x, acc[4]);
        acc[5] = fmaf(av.y, bv.y, acc[5]);
        acc[6] = fmaf(av.y, bv.z, acc[6]);
        acc[7] = fmaf(av.y, bv.w, acc[7]);
    }
}

// accumulator index layout: [c1w F*8 | c1b F | c2w 3*F | c2b 3 | st 3*8] (padded dims)
template <int FP>
__global__ void __launch_bounds__(kSynTile) k_syn_trunk_bwd(const Plan* __restrict__ pp,
                                                            const float* __restrict__ dt_in) {
    using K = TrunkCfg<FP>;
    const Plan& P = *pp;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TrunkSmem<FP>& sm = *reinterpret_cast<TrunkSmem<FP>*>(smem_raw);
    const int tid = threadIdx.x;
    const int L = P.L, F = P.syn_F;
    for (int e = tid; e < FP * kLZ; e += kSynTile) {
        const int f = e / kLZ, k = e - f * kLZ;
        sm.c1w[e] = (f < F && k < L) ? P.params[P.off_c1w + f * L + k] : 0.0f;
    }
    for (int e = tid; e < FP; e += kSynTile) sm.c1b[e] = e < F ? P.params[P.off_c1b + e] : 0.0f;
    for (int e = tid; e < 3 * FP; e += kSynTile) {
        const int co = e / FP, f = e - co * FP;
        sm.c2w[e] = f < F ? P.params[P.off_c2w + co * F + f] : 0.0f;
    }
    for (int e = tid; e < 3 * kLZ; e += kSynTile) {
        const int co = e / kLZ, k = e - co * kLZ;
        sm.st[e] = (P.off_sstab >= 0 && k < L) ? P.params[P.off_sstab + co * L + k] : 0.0f;
    }
    for (int e = tid; e < K::NACC; e += kSynTile) sm.acc[e] = 0.0;
    __syncthreads();

    const int64_t np = P.npix;
    const int64_t ntiles = (np + kSynTile - 1) / kSynTile;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t p = t * kSynTile + tid;
        const bool valid = p < np;
        float zv[kLZ];
#pragma unroll
        for (int k = 0; k < kLZ; ++k) zv[k] = (valid && k < L) ? P.z[int64_t(k) * np + p] : 0.0f;
        float dt[3], dx[3];
#pragma unroll
        for (int co = 0; co < 3; ++co) {
            dt[co] = valid ? dt_in[int64_t(co) * np + p] : 0.0f;
            dx[co] = valid ? P.syn_dx[int64_t(co) * np + p] : 0.0f;
        }
        float* myZ = sm.act + K::O_Z + tid * K::LZ;
        float* myH = sm.act + K::O_H + tid * K::LH;
        float* myDH = sm.act + K::O_DH + tid * K::LDH;
        float* myDT = sm.act + K::O_DT + tid * K::LT;
        float* myDX = sm.act + K::O_DX + tid * K::LT;
        // dz accumulates the stabilizer term first, then c1 (synthesis.hpp:220,232)
        float dz[kLZ];
#pragma unroll
        for (int k = 0; k < kLZ; ++k) {
            float a = 0.0f;
            a = fmaf(sm.st[k], dx[0], a);
            a = fmaf(sm.st[kLZ + k], dx[1], a);
            a = fmaf(sm.st[2 * kLZ + k], dx[2], a);
            dz[k] = P.off_sstab >= 0 ? a : 0.0f;
        }
#pragma unroll 4
        for (int f = 0; f < FP; ++f) {
            float acc = sm.c1b[f];
#pragma unroll
            for (int k = 0; k < kLZ; ++k) acc = fmaf(zv[k], sm.c1w[f * kLZ + k], acc);
            const float h = acc > 0.0f ? acc : 0.0f;
            float d = 0.0f;
            d = fmaf(sm.c2w[f], dt[0], d);
            d = fmaf(sm.c2w[FP + f], dt[1], d);
            d = fmaf(sm.c2w[2 * FP + f], dt[2], d);
            d = h > 0.0f ? d : 0.0f;
#pragma unroll
            for (int k = 0; k < kLZ; ++k) dz[k] = fmaf(sm.c1w[f * kLZ + k], d, dz[k]);
            myH[f] = valid ? h : 0.0f;
            myDH[f] = valid ? d : 0.0f;
        }
        if (valid) {
#pragma unroll
            for (int k = 0; k < kLZ; ++k)
                if (k < L) P.dz[int64_t(k) * np + p] = dz[k];
        }
        for (int k = 0; k < K::LZ; ++k) myZ[k] = k < kLZ ? zv[k] : ((k == kLZ && valid) ? 1.0f : 0.0f);
        for (int f = FP; f < K::LH; ++f) myH[f] = (f == FP && valid) ? 1.0f : 0.0f;
        for (int f = FP; f < K::LDH; ++f) myDH[f] = 0.0f;
        *reinterpret_cast<float4*>(myDT) = make_float4(dt[0], dt[1], dt[2], 0.0f);
        *reinterpret_cast<float4*>(myDX) = make_float4(dx[0], dx[1], dx[2], 0.0f);
        __syncthreads();
        for (int job = tid; job < K::NJ; job += kSynTile) {
            float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            int a0, b0, kind;
            if (job < K::NJ1) {
                constexpr int nq = r4(kLZ + 1) / 4;
                a0 = 2 * (job / nq);
                b0 = 4 * (job % nq);
                kind = 0;
                syn_mt<K::LDH, K::LZ>(sm.act + K::O_DH, sm.act + K::O_Z, a0, b0, acc);
            } else if (job < K::NJ1 + K::NJ2) {
                constexpr int nq = r4(FP + 1) / 4;
                const int jj = job - K::NJ1;
                a0 = 2 * (jj / nq);
                b0 = 4 * (jj % nq);
                kind = 1;
                syn_mt<K::LT, K::LH>(sm.act + K::O_DT, sm.act + K::O_H, a0, b0, acc);
            } else {
                constexpr int nq = kLZ / 4;
                const int jj = job - K::NJ1 - K::NJ2;
                a0 = 2 * (jj / nq);
                b0 = 4 * (jj % nq);
                kind = 2;
                syn_mt<K::LT, K::LZ>(sm.act + K::O_DX, sm.act + K::O_Z, a0, b0, acc);
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int a = a0 + (e >> 2), b = b0 + (e & 3);
                int o = -1;
                if (kind == 0) {
                    if (b < kLZ) o = a * kLZ + b;
                    else if (b == kLZ) o = FP * kLZ + a;
                } else if (kind == 1) {
                    if (a < 3) {
                        if (b < FP) o = FP * kLZ + FP + a * FP + b;
                        else if (b == FP) o = FP * kLZ + FP + 3 * FP + a;
                    }
                } else {
                    if (a < 3 && b < kLZ) o = FP * kLZ + FP + 3 * FP + 3 + a * kLZ + b;
                }
                if (o >= 0) sm.acc[o] += double(acc[e]);
            }
        }
        __syncthreads();
    }
    // scatter the padded accumulators into this CTA's partial row
    const PartialRegion& R = P.region[P.reg_syn_trunk];
    double* row = P.partials + R.base + int64_t(blockIdx.x) * R.count;
    for (int e = tid; e < R.count; e += kSynTile) {
        const int pidx = R.param_off + e;
        double v = 0.0;
        if (pidx >= P.off_c1w && pidx < P.off_c1w + F * L) {
            const int q = pidx - P.off_c1w, f = q / L, k = q - f * L;
            v = sm.acc[f * kLZ + k];
        } else if (pidx >= P.off_c1b && pidx < P.off_c1b + F) {
            v = sm.acc[FP * kLZ + (pidx - P.off_c1b)];
        } else if (pidx >= P.off_c2w && pidx < P.off_c2w + 3 * F) {
            const int q = pidx - P.off_c2w, co = q / F, f = q - co * F;
            v = sm.acc[FP * kLZ + FP + co * FP + f];
        } else if (pidx >= P.off_c2b && pidx < P.off_c2b + 3) {
            v = sm.acc[FP * kLZ + FP + 3 * FP + (pidx - P.off_c2b)];
        } else if (P.off_sstab >= 0 && pidx >= P.off_sstab && pidx < P.off_sstab + 3 * L) {
            const int q = pidx - P.off_sstab, co = q / L, k = q - co * L;
            v = sm.acc[FP * kLZ + FP + 3 * FP + 3 + co * kLZ + k];
        }
        row[e] = v;
    }
}

template <int FP>
size_t trunk_smem() {
    return sizeof(TrunkSmem<FP>);
}

template <int FP>
void launch_trunk_bwd_t(const LaunchCtx& L, const float* dt) {
    k_syn_trunk_bwd<FP><<<L.syn_blocks, kSynTile, trunk_smem<FP>(), L.stream>>>(L.plan, dt);
}

}  // namespace

int syn_padded_hidden(int F) {
    if (F <= 8) return 8;
    if (F <= 16) return 16;
    if (F <= 48) return 48;
    if (F <= 64) return 64;
    return -1;
}

size_t syn_trunk_smem(int FP) {
    switch (FP) {
        case 8: return trunk_smem<8>();
        case 16: return trunk_smem<16>();
        case 48: return trunk_smem<48>();
        default: return trunk_smem<64>();
    }
}

void syn_configure(int FP) {
    const int smem = int(syn_trunk_smem(FP));
    switch (FP) {
        case 8: cudaFuncSetAttribute(k_syn_trunk_bwd<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); break;
        case 16: cudaFuncSetAttribute(k_syn_trunk_bwd<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); break;
        case 48: cudaFuncSetAttribute(k_syn_trunk_bwd<48>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); break;
        default: cudaFuncSetAttribute(k_syn_trunk_bwd<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); break;
    }
}

void launch_syn_forward(const LaunchCtx& L, bool backward) {
    const Plan& H = *L.host;
    k_syn_trunk_fwd<<<L.pix_blocks, 256, 0, L.stream>>>(L.plan);
    for (int i = 0; i < H.posts; ++i) k_syn_post_fwd<<<L.pix_blocks, 256, 0, L.stream>>>(L.plan, i);
    k_syn_out<<<H.n_mse_part, 256, 0, L.stream>>>(L.plan, backward ? 1 : 0);
}

void launch_syn_backward(const LaunchCtx& L) {
    const Plan& H = *L.host;
    const float* dcur = H.syn_dx;
    for (int i = H.posts - 1; i >= 0; --i) {
        float* dprev = (i == 0) ? H.syn_dt : H.syn_dtmp;
        if (i > 0 && dcur == H.syn_dtmp) dprev = H.syn_dt;  // ping-pong (posts <= 2)
        k_syn_post_bwd<<<L.red_blocks, 256, 0, L.stream>>>(L.plan, i, dcur, dprev);
        dcur = dprev;
    }
    const int FP = syn_padded_hidden(H.syn_F);
    switch (FP) {
        case 8: launch_trunk_bwd_t<8>(L, dcur); break;
        case 16: launch_trunk_bwd_t<16>(L, dcur); break;
        case 48: launch_trunk_bwd_t<48>(L, dcur); break;
        default: launch_trunk_bwd_t<64>(L, dcur); break;
    }
}

}  // namespace ccb

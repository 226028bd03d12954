// cc_arm.cu — the auto-regressive entropy model (ARM + IFCE), forward and
// backward fused into ONE persistent kernel over every grid of the pyramid.
//
// Replaces rate_pass (entropy_model.hpp:180-336), i.e. per latent:
//   gather 14 causal neighbours + IFCE context        entropy_model.hpp:232-248
//   MLP d -> w -> w -> 2 (+ linear stabilizer)        entropy_model.hpp:250-255
//   Laplace mu/sigma, bits (rate)                     entropy_model.hpp:257-273
//   rate backward to (mu, sigma_raw, value)           entropy_model.hpp:276-296
//   MLP backward (dH2, dH1, dC)                       entropy_model.hpp:298-310
//   weight gradients dW1..dW3, dstab, IFCE dWf        entropy_model.hpp:301-321
// In the training proxy nothing is sequential across latents (every ŷ is
// known), so all grids run in one launch from a tile table.
//
// B200 design: one thread owns one latent's data path (context, activations
// and their gradients stay in registers; the weights sit in shared memory and
// are read as broadcast LDS.128).  The weight gradients are per-tile small
// GEMMs over the latent dimension: the per-latent vectors go to shared memory
// and every thread owns a 2x4 micro-tile of (dW | db), accumulating over the
// 128 latents of the tile in fp32 and across tiles in fp64 shared memory.
// CTAs are persistent (grid = SMs x occupancy) and walk the tile table in a
// fixed stride, so every sum has a fixed order: no float atomics, bitwise
// deterministic.  The latent-side gradients are NOT scattered: dC (S planes),
// dF (F planes) and the own-value term are written per latent and gathered by
// k_latent_grad, the IFCE coarse-grid term through a 2x2 block-sum pyramid
// (k_pyramid) — W_f^T is linear, so sum-then-multiply equals the reference's
// multiply-then-scatter (entropy_model.hpp:322-330).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <vector>
#include <mutex>

#include "cc_kernels.h"
#include "cc_math.cuh"
#include "cc_reduce.cuh"

namespace ccb {

// kArmTile (latents per tile == threads per CTA) lives in cc_plan.h
constexpr int kRMax = 12;      // max IFCE source grids (hyper 4 + main 7)
constexpr int kFMax = 8;       // max IFCE width

__host__ __device__ constexpr int round4(int n) { return (n + 3) / 4 * 4; }
// row stride (floats) with an odd number of 16-byte chunks: conflict-free LDS.128
__host__ __device__ constexpr int odd_chunks(int n) {
    return ((round4(n) / 4) % 2 == 0) ? round4(n) + 4 : round4(n);
}

template <int DP, int WP>
struct ArmCfg {
    static constexpr int LC = odd_chunks(DP + 1);   // context row, ones at DP
    static constexpr int LH = odd_chunks(WP + 1);   // activation row, ones at WP
    static constexpr int LDH = odd_chunks(WP);      // activation-gradient row
    static constexpr int LR = odd_chunks(kRMax + 1);  // IFCE source row, ones at kRMax
    static constexpr int LF = odd_chunks(kFMax);    // dF row
    static constexpr int LDR = 4;                   // (dmu, dsigma_raw, 0, 0)
    // phase A rows: C | H2 | dH1 | draw | R | dF ; phase B rows: H1 | dH2
    static constexpr int OA_C = 0;
    static constexpr int OA_H2 = OA_C + kArmTile * LC;
    static constexpr int OA_DH1 = OA_H2 + kArmTile * LH;
    static constexpr int OA_DR = OA_DH1 + kArmTile * LDH;
    static constexpr int OA_R = OA_DR + kArmTile * LDR;
    static constexpr int OA_DF = OA_R + kArmTile * LR;
    static constexpr int ACT = OA_DF + kArmTile * LF;
    static constexpr int OB_H1 = 0;
    static constexpr int OB_DH2 = kArmTile * LH;
    static_assert(OB_DH2 + kArmTile * LDH <= ACT, "phase B must fit in phase A");
    // upper bound of the ARM+IFCE partial region (unpadded dims <= padded)
    static constexpr int NACC =
        WP * DP + WP + WP * WP + WP + 2 * WP + 2 + 2 * DP + kMaxSlots * (kFMax * kRMax + kFMax);
    // micro-tile jobs (2 rows x 4 cols)
    static constexpr int NJ1 = (WP / 2) * (round4(DP + 1) / 4);  // dH1 x [C|1]
    static constexpr int NJ3 = round4(WP + 1) / 4;              // draw x [H2|1]
    static constexpr int NJ4 = round4(DP) / 4;                  // draw x C (stab)
    static constexpr int NJ5 = (kFMax / 2) * (round4(kRMax + 1) / 4);  // dF x [R|1]
    static constexpr int NJA = NJ1 + NJ3 + NJ4 + NJ5;
    static constexpr int NJ2 = (WP / 2) * (round4(WP + 1) / 4);  // dH2 x [H1|1]
};

template <int DP, int WP>
struct alignas(16) ArmSmem {
    using K = ArmCfg<DP, WP>;
    alignas(16) float W1[WP * DP];
    alignas(16) float W2[WP * WP];
    alignas(16) float W3[2 * WP];
    alignas(16) float stab[2 * DP];
    alignas(16) float b1[WP];
    alignas(16) float b2[WP];
    alignas(16) float b3[4];
    alignas(16) float Wf[kMaxSlots][kFMax * kRMax];
    alignas(16) float bf[kMaxSlots][kFMax];
    alignas(16) float act[K::ACT];
    alignas(16) double acc[K::NACC];
    int ctx_dy[kMaxCtx], ctx_dx[kMaxCtx];
    double red[kArmTile / 32];
};

// 2x4 outer-product accumulation over the tile's latents.
template <int LDA, int LDB>
__device__ __forceinline__ void mt_accum(const float* __restrict__ A, const float* __restrict__ B,
                                         int a0, int b0, float (&acc)[8]) {
#pragma unroll 4
    for (int i = 0; i < kArmTile; ++i) {
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

// Region index (== flat parameter index; the ARM region starts at arm.l1.w,
// which is parameter 0) of output (a, b) of job `kind`, or -1 to discard.
struct OutMap {
    int w_off, b_off;  // weight / bias parameter offsets (b_off < 0: none)
    int rows, cols;    // real (unpadded) extents
    int ones_col;      // column index of the bias "ones" column
    __device__ __forceinline__ int operator()(int a, int b) const {
        if (a >= rows) return -1;
        if (b < cols) return w_off + a * cols + b;
        if (b == ones_col && b_off >= 0) return b_off + a;
        return -1;
    }
};

template <int DP, int WP, int MODE>
__global__ void __launch_bounds__(kArmTile) k_arm(const Plan* __restrict__ pp,
                                                  const int4* __restrict__ tiles, int ntiles) {
    using K = ArmCfg<DP, WP>;
    const Plan& P = pp[blockIdx.z];  // batched launches: one plan per image
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ArmSmem<DP, WP>& sm = *reinterpret_cast<ArmSmem<DP, WP>*>(smem_raw);
    const int tid = threadIdx.x;
    const int D = P.D, Wd = P.Wd, S = P.S, F = P.F;
    const float* prm = P.params;

    // ---- weights -> shared memory, zero-padded to (WP, DP) ----
    for (int e = tid; e < WP * DP; e += kArmTile) {
        const int a = e / DP, b = e - a * DP;
        sm.W1[e] = (a < Wd && b < D) ? prm[P.off_l1w + a * D + b] : 0.0f;
    }
    for (int e = tid; e < WP * WP; e += kArmTile) {
        const int a = e / WP, b = e - a * WP;
        sm.W2[e] = (a < Wd && b < Wd) ? prm[P.off_l2w + a * Wd + b] : 0.0f;
    }
    for (int e = tid; e < 2 * WP; e += kArmTile) {
        const int a = e / WP, b = e - a * WP;
        sm.W3[e] = b < Wd ? prm[P.off_hw + a * Wd + b] : 0.0f;
    }
    for (int e = tid; e < 2 * DP; e += kArmTile) {
        const int a = e / DP, b = e - a * DP;
        sm.stab[e] = (P.off_astab >= 0 && b < D) ? prm[P.off_astab + a * D + b] : 0.0f;
    }
    for (int e = tid; e < WP; e += kArmTile) {
        sm.b1[e] = e < Wd ? prm[P.off_l1b + e] : 0.0f;
        sm.b2[e] = e < Wd ? prm[P.off_l2b + e] : 0.0f;
    }
    if (tid < 4) sm.b3[tid] = tid < 2 ? prm[P.off_hb + tid] : 0.0f;
    for (int e = tid; e < kMaxSlots * kFMax * kRMax; e += kArmTile) {
        const int s = e / (kFMax * kRMax), rem = e - s * kFMax * kRMax;
        const int f = rem / kRMax, j = rem - f * kRMax;
        float v = 0.0f;
        if (s < P.n_slots) {
            const int rd = P.g[P.slot_gi[s]].rdim;
            if (f < F && j < rd) v = prm[P.off_ifw[s] + f * rd + j];
        }
        sm.Wf[s][f * kRMax + j] = v;
    }
    for (int e = tid; e < kMaxSlots * kFMax; e += kArmTile) {
        const int s = e / kFMax, f = e - s * kFMax;
        sm.bf[s][f] = (s < P.n_slots && f < F) ? prm[P.off_ifb[s] + f] : 0.0f;
    }
    for (int e = tid; e < kMaxCtx; e += kArmTile) {
        sm.ctx_dy[e] = e < S ? P.ctx_dy[e] : 0;
        sm.ctx_dx[e] = e < S ? P.ctx_dx[e] : 0;
    }
    if (MODE != kArmForward)
        for (int e = tid; e < K::NACC; e += kArmTile) sm.acc[e] = 0.0;
    __syncthreads();

    const float upstream = P.rate_upstream;
    double bits_cta = 0.0;  // thread 0

    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int4 tile = tiles[t];
        const GridGeom& g = P.g[tile.x];
        const int64_t count = int64_t(g.rows) * g.cols;
        const int64_t li = int64_t(tile.y) + tid;
        const bool valid = tid < tile.w;  // row segment of tile.w latents
        const int r = valid ? int(li / g.cols) : 0;
        const int c = valid ? int(li - int64_t(r) * g.cols) : 0;
        const int slot = g.ifce_slot;

        // ---- context row in shared memory (runtime extents), then registers ----
        float* myC = sm.act + K::OA_C + tid * K::LC;
        float* myR = sm.act + K::OA_R + tid * K::LR;
        {
            const float* base = P.yhat_pad + g.pad_base + int64_t(r) * g.stride + c;
            for (int o = 0; o < S; ++o)
                myC[o] = valid ? __ldg(base + sm.ctx_dy[o] * g.stride + sm.ctx_dx[o]) : 0.0f;
            if (slot >= 0) {
                const int rd = g.rdim;
                for (int j = 0; j < kRMax; ++j) {
                    float v = 0.0f;
                    if (valid && j < rd) {
                        const GridGeom& s = P.g[j];
                        const int sh = s.level - g.level;
                        v = __ldg(P.yhat_pad + s.pad_base + int64_t(r >> sh) * s.stride + (c >> sh));
                    }
                    myR[j] = v;
                }
                myR[kRMax] = valid ? 1.0f : 0.0f;
                for (int j = kRMax + 1; j < K::LR; ++j) myR[j] = 0.0f;
                for (int f = 0; f < F; ++f) {
                    float acc = sm.bf[slot][f];
                    for (int j = 0; j < kRMax; ++j) acc = fmaf(myR[j], sm.Wf[slot][f * kRMax + j], acc);
                    myC[S + f] = valid ? acc : 0.0f;
                }
            } else {
                for (int f = 0; f < F; ++f) myC[S + f] = 0.0f;
                for (int j = 0; j < K::LR; ++j) myR[j] = 0.0f;
            }
            for (int o = D; o < K::LC; ++o) myC[o] = (o == DP && valid) ? 1.0f : 0.0f;
        }
        float C[DP];
#pragma unroll
        for (int o = 0; o < DP; o += 4) {
            const float4 v = *reinterpret_cast<const float4*>(myC + o);
            C[o] = v.x; C[o + 1] = v.y; C[o + 2] = v.z; C[o + 3] = v.w;
        }

        // ---- MLP forward (entropy_model.hpp:250-255) ----
        float h1[WP], h2[WP];
#pragma unroll
        for (int a = 0; a < WP; ++a) {
            float acc = sm.b1[a];
#pragma unroll
            for (int b = 0; b < DP; b += 4) {
                const float4 w = *reinterpret_cast<const float4*>(&sm.W1[a * DP + b]);
                acc = fmaf(C[b], w.x, acc);
                acc = fmaf(C[b + 1], w.y, acc);
                acc = fmaf(C[b + 2], w.z, acc);
                acc = fmaf(C[b + 3], w.w, acc);
            }
            h1[a] = acc > 0.0f ? acc : 0.0f;
        }
#pragma unroll
        for (int a = 0; a < WP; ++a) {
            float acc = sm.b2[a];
#pragma unroll
            for (int b = 0; b < WP; b += 4) {
                const float4 w = *reinterpret_cast<const float4*>(&sm.W2[a * WP + b]);
                acc = fmaf(h1[b], w.x, acc);
                acc = fmaf(h1[b + 1], w.y, acc);
                acc = fmaf(h1[b + 2], w.z, acc);
                acc = fmaf(h1[b + 3], w.w, acc);
            }
            h2[a] = acc > 0.0f ? acc : 0.0f;
        }
        float raw[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            float acc = sm.b3[j];
#pragma unroll
            for (int b = 0; b < WP; b += 4) {
                const float4 w = *reinterpret_cast<const float4*>(&sm.W3[j * WP + b]);
                acc = fmaf(h2[b], w.x, acc);
                acc = fmaf(h2[b + 1], w.y, acc);
                acc = fmaf(h2[b + 2], w.z, acc);
                acc = fmaf(h2[b + 3], w.w, acc);
            }
#pragma unroll
            for (int b = 0; b < DP; b += 4) {
                const float4 w = *reinterpret_cast<const float4*>(&sm.stab[j * DP + b]);
                acc = fmaf(C[b], w.x, acc);
                acc = fmaf(C[b + 1], w.y, acc);
                acc = fmaf(C[b + 2], w.z, acc);
                acc = fmaf(C[b + 3], w.w, acc);
            }
            raw[j] = acc;
        }

        // ---- Laplace rate (entropy_model.hpp:257-273) ----
        const float v = valid ? P.yhat_pad[g.pad_base + int64_t(r) * g.stride + c] : 0.0f;
        const float mu = raw[0];
        const float sg = sigma_from_raw(raw[1]);
        const float bsc = sg * kInvSqrt2F;
        const float u = fabsf(v - mu);
        const float e1 = cc_exp(-(u + 0.5f) / bsc);
        const float e2 = cc_exp(-fabsf(u - 0.5f) / bsc);
        const float p = u >= 0.5f ? 0.5f * (e2 - e1) : 1.0f - 0.5f * (e1 + e2);
        const float bits = valid ? -(cc_log(std_max(p, kProbFloorF)) * kLog2EF) : 0.0f;
        {
            const double tb = block_sum(double(bits), sm.red);
            if (tid == 0) bits_cta += tb;
        }
        if (MODE == kArmForward) continue;

        // ---- rate backward (entropy_model.hpp:276-296) ----
        float dmu = 0.0f, dsr = 0.0f, gv = 0.0f;
        if (valid && p > kProbFloorF) {
            const float tt = v - mu;
            const float dbits_dp = -1.0f / (p * kLn2F);
            const float dp_du = (e1 - e2) / (2.0f * bsc);
            const float sgn = tt > 0.0f ? 1.0f : (tt < 0.0f ? -1.0f : 0.0f);
            const float dp_db = -((u + 0.5f) * e1 - (u - 0.5f) * e2) / (2.0f * bsc * bsc);
            const float up = upstream * dbits_dp;
            dmu = -up * dp_du * sgn;
            if (sg > kSigmaMinF && sg < kSigmaMaxF) dsr = up * dp_db * kInvSqrt2F * sg;
            gv = up * dp_du * sgn;
        }

        // ---- MLP backward (entropy_model.hpp:298-310) ----
        float dH2[WP];
#pragma unroll
        for (int a = 0; a < WP; ++a) {
            float acc = fmaf(dmu, sm.W3[a], 0.0f);
            acc = fmaf(dsr, sm.W3[WP + a], acc);
            dH2[a] = h2[a] > 0.0f ? acc : 0.0f;
        }
        float dH1[WP];
#pragma unroll
        for (int b = 0; b < WP; ++b) dH1[b] = 0.0f;
#pragma unroll
        for (int a = 0; a < WP; ++a) {
#pragma unroll
            for (int b = 0; b < WP; b += 4) {
                const float4 w = *reinterpret_cast<const float4*>(&sm.W2[a * WP + b]);
                dH1[b] = fmaf(dH2[a], w.x, dH1[b]);
                dH1[b + 1] = fmaf(dH2[a], w.y, dH1[b + 1]);
                dH1[b + 2] = fmaf(dH2[a], w.z, dH1[b + 2]);
                dH1[b + 3] = fmaf(dH2[a], w.w, dH1[b + 3]);
            }
        }
#pragma unroll
        for (int b = 0; b < WP; ++b) dH1[b] = h1[b] > 0.0f ? dH1[b] : 0.0f;
        float dC[DP];
#pragma unroll
        for (int k = 0; k < DP; ++k) dC[k] = 0.0f;
#pragma unroll
        for (int a = 0; a < WP; ++a) {
#pragma unroll
            for (int k = 0; k < DP; k += 4) {
                const float4 w = *reinterpret_cast<const float4*>(&sm.W1[a * DP + k]);
                dC[k] = fmaf(dH1[a], w.x, dC[k]);
                dC[k + 1] = fmaf(dH1[a], w.y, dC[k + 1]);
                dC[k + 2] = fmaf(dH1[a], w.z, dC[k + 2]);
                dC[k + 3] = fmaf(dH1[a], w.w, dC[k + 3]);
            }
        }
#pragma unroll
        for (int k = 0; k < DP; ++k) {
            dC[k] = fmaf(dmu, sm.stab[k], dC[k]);
            dC[k] = fmaf(dsr, sm.stab[DP + k], dC[k]);
        }

        // ---- latent-side outputs (gathered later, no scatter) ----
        float* myDF = sm.act + K::OA_DF + tid * K::LF;
        if (MODE == kArmProxy && valid) {
            P.gown[g.lat_off + li] = gv;
            float* dcp = P.dctx + g.dctx_off + li;
#pragma unroll
            for (int o = 0; o < DP; ++o)
                if (o < S) dcp[int64_t(o) * count] = dC[o];
        }
        if (slot >= 0) {
            float* dfp = P.dfeat + g.dfeat_off + li;
#pragma unroll
            for (int o = 0; o < DP; ++o) {
                if (o >= S && o < S + F) {
                    const float vv = valid ? dC[o] : 0.0f;
                    myDF[o - S] = vv;
                    if (MODE == kArmProxy && valid) dfp[int64_t(o - S) * count] = vv;
                }
            }
            for (int f = F; f < K::LF; ++f) myDF[f] = 0.0f;
        }

        // ---- phase A: C | H2 | dH1 | draw | R | dF in shared memory ----
        {
            float* myH2 = sm.act + K::OA_H2 + tid * K::LH;
            float* myDH1 = sm.act + K::OA_DH1 + tid * K::LDH;
            float* myDR = sm.act + K::OA_DR + tid * K::LDR;
#pragma unroll
            for (int a = 0; a < WP; a += 4) {
                *reinterpret_cast<float4*>(myH2 + a) =
                    valid ? make_float4(h2[a], h2[a + 1], h2[a + 2], h2[a + 3])
                          : make_float4(0.f, 0.f, 0.f, 0.f);
                *reinterpret_cast<float4*>(myDH1 + a) =
                    valid ? make_float4(dH1[a], dH1[a + 1], dH1[a + 2], dH1[a + 3])
                          : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            for (int a = WP; a < K::LH; ++a) myH2[a] = (a == WP && valid) ? 1.0f : 0.0f;
            for (int a = WP; a < K::LDH; ++a) myDH1[a] = 0.0f;
            *reinterpret_cast<float4*>(myDR) = make_float4(dmu, dsr, 0.f, 0.f);
        }
        __syncthreads();
        for (int job = tid; job < K::NJA; job += kArmTile) {
            float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            OutMap om;
            int a0, b0;
            if (job < K::NJ1) {
                constexpr int nq = round4(DP + 1) / 4;
                a0 = 2 * (job / nq);
                b0 = 4 * (job % nq);
                mt_accum<K::LDH, K::LC>(sm.act + K::OA_DH1, sm.act + K::OA_C, a0, b0, acc);
                om = OutMap{P.off_l1w, P.off_l1b, Wd, D, DP};
            } else if (job < K::NJ1 + K::NJ3) {
                a0 = 0;
                b0 = 4 * (job - K::NJ1);
                mt_accum<K::LDR, K::LH>(sm.act + K::OA_DR, sm.act + K::OA_H2, a0, b0, acc);
                om = OutMap{P.off_hw, P.off_hb, 2, Wd, WP};
            } else if (job < K::NJ1 + K::NJ3 + K::NJ4) {
                if (P.off_astab < 0) continue;
                a0 = 0;
                b0 = 4 * (job - K::NJ1 - K::NJ3);
                mt_accum<K::LDR, K::LC>(sm.act + K::OA_DR, sm.act + K::OA_C, a0, b0, acc);
                om = OutMap{P.off_astab, -1, 2, D, -1};
            } else {
                if (slot < 0) continue;
                constexpr int nq = round4(kRMax + 1) / 4;
                const int jj = job - K::NJ1 - K::NJ3 - K::NJ4;
                a0 = 2 * (jj / nq);
                b0 = 4 * (jj % nq);
                mt_accum<K::LF, K::LR>(sm.act + K::OA_DF, sm.act + K::OA_R, a0, b0, acc);
                om = OutMap{P.off_ifw[slot], P.off_ifb[slot], F, g.rdim, kRMax};
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int o = om(a0 + (e >> 2), b0 + (e & 3));
                if (o >= 0) sm.acc[o] += double(acc[e]);
            }
        }
        __syncthreads();
        // ---- phase B: H1 | dH2 ----
        {
            float* myH1 = sm.act + K::OB_H1 + tid * K::LH;
            float* myDH2 = sm.act + K::OB_DH2 + tid * K::LDH;
#pragma unroll
            for (int a = 0; a < WP; a += 4) {
                *reinterpret_cast<float4*>(myH1 + a) =
                    valid ? make_float4(h1[a], h1[a + 1], h1[a + 2], h1[a + 3])
                          : make_float4(0.f, 0.f, 0.f, 0.f);
                *reinterpret_cast<float4*>(myDH2 + a) =
                    valid ? make_float4(dH2[a], dH2[a + 1], dH2[a + 2], dH2[a + 3])
                          : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            for (int a = WP; a < K::LH; ++a) myH1[a] = (a == WP && valid) ? 1.0f : 0.0f;
            for (int a = WP; a < K::LDH; ++a) myDH2[a] = 0.0f;
        }
        __syncthreads();
        for (int job = tid; job < K::NJ2; job += kArmTile) {
            float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            constexpr int nq = round4(WP + 1) / 4;
            const int a0 = 2 * (job / nq), b0 = 4 * (job % nq);
            mt_accum<K::LDH, K::LH>(sm.act + K::OB_DH2, sm.act + K::OB_H1, a0, b0, acc);
            const OutMap om{P.off_l2w, P.off_l2b, Wd, Wd, WP};
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int o = om(a0 + (e >> 2), b0 + (e & 3));
                if (o >= 0) sm.acc[o] += double(acc[e]);
            }
        }
        __syncthreads();
    }

    if (tid == 0) P.bits_part[blockIdx.x] = bits_cta;
    if (MODE != kArmForward) {
        const PartialRegion& R = P.region[P.reg_arm];
        const PartialRow row(P, R, blockIdx.x);
        for (int e = tid; e < R.count; e += kArmTile) row[e] = sm.acc[e];
    }
}

// 2x2 block sums of dF for every IFCE-equipped grid, ALL levels in one
// launch: CTA (coarse block, slot*F + f) loads the 2^smax x 2^smax fine
// block of channel f (zeros past the grid edge) and halves it level by level
// in shared memory, writing each level.  Summation order ((a+b)+(c+d)) is
// the same at every level, so results do not depend on the blocking.
__global__ void __launch_bounds__(256) k_pyramid_fused(const Plan* __restrict__ pp) {
    const Plan& P = pp[blockIdx.z];  // batched launches: one plan per image
    extern __shared__ float pbuf[];
    const int s = blockIdx.y / P.F, f = blockIdx.y - s * P.F;
    const int smax = P.slot_smax[s];
    const int B = 1 << smax;
    const int cr = P.slot_pyr_rows[s][smax], ccn = P.slot_pyr_cols[s][smax];
    const int R = blockIdx.x / ccn, Cc = blockIdx.x - R * ccn;
    if (R >= cr) return;
    float* a = pbuf;
    float* b = pbuf + B * B;
    {
        // level 0 is dF in the grid's local rows; the pyramid's blocks are
        // aligned to global rows (origin slot_pyr_a): local = aligned - off
        const int rows = P.slot_pyr_rows[s][0], cols = P.slot_pyr_cols[s][0];
        const int off = P.g[P.slot_gi[s]].row0 - P.slot_pyr_a[s];
        const float* in = P.dfeat + P.slot_pyr_off[s][0] + int64_t(f) * rows * cols;
        for (int e = threadIdx.x; e < B * B; e += blockDim.x) {
            const int y = e >> smax, x = e & (B - 1);
            const int gy = R * B + y - off, gx = Cc * B + x;
            a[e] = (gy >= 0 && gy < rows && gx < cols) ? in[int64_t(gy) * cols + gx] : 0.0f;
        }
    }
    __syncthreads();
    for (int l = 1; l <= smax; ++l) {
        const int n = B >> l;  // edge of this level's block
        const int rows = P.slot_pyr_rows[s][l], cols = P.slot_pyr_cols[s][l];
        float* out = P.dfeat + P.slot_pyr_off[s][l] + int64_t(f) * rows * cols;
        for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
            const int y = e / n, x = e - y * n;
            const float* src = a + (2 * y) * (2 * n) + 2 * x;
            const float v = (src[0] + src[1]) + (src[2 * n] + src[2 * n + 1]);
            b[e] = v;
            const int gy = R * n + y, gx = Cc * n + x;
            if (gy < rows && gx < cols) out[int64_t(gy) * cols + gx] = v;
        }
        __syncthreads();
        float* t = a;
        a = b;
        b = t;
    }
}

// 2x2 block sums of dF for every IFCE-equipped grid, one level per launch.
__global__ void k_pyramid(const Plan* __restrict__ pp, int level) {
    const Plan& P = pp[blockIdx.z];  // batched launches: one plan per image
    for (int s = 0; s < P.n_slots; ++s) {
        if (level > P.slot_smax[s]) continue;
        const int ri = P.slot_pyr_rows[s][level - 1], ci = P.slot_pyr_cols[s][level - 1];
        const int ro = P.slot_pyr_rows[s][level], co = P.slot_pyr_cols[s][level];
        const float* in = P.dfeat + P.slot_pyr_off[s][level - 1];
        float* out = P.dfeat + P.slot_pyr_off[s][level];
        const int64_t n = int64_t(P.F) * ro * co;
        for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
             e += int64_t(gridDim.x) * blockDim.x) {
            const int f = int(e / (int64_t(ro) * co));
            const int rem = int(e - int64_t(f) * ro * co);
            const int R = rem / co, Cc = rem - R * co;
            const float* pl = in + int64_t(f) * ri * ci;
            const int r0 = 2 * R, c0 = 2 * Cc;
            const float a = pl[int64_t(r0) * ci + c0];
            const float b = (c0 + 1 < ci) ? pl[int64_t(r0) * ci + c0 + 1] : 0.0f;
            const float cc = (r0 + 1 < ri) ? pl[int64_t(r0 + 1) * ci + c0] : 0.0f;
            const float d = (r0 + 1 < ri && c0 + 1 < ci) ? pl[int64_t(r0 + 1) * ci + c0 + 1] : 0.0f;
            out[int64_t(f) * ro * co + int64_t(R) * co + Cc] = (a + b) + (cc + d);
        }
    }
}

// ---------------------------------------------------------------------------
// Instantiated (Dp, Wp) pairs; any decoder whose (D, W) fits one of them runs
// zero-padded (exact: padded weights and activations are exact zeros).
struct ArmVariant {
    int Dp, Wp;
};
static const ArmVariant kVariants[] = {{8, 8}, {16, 12}, {20, 20}, {28, 28}, {32, 20}, {40, 40}};

void arm_padded_dims(int D, int W, int* Dp, int* Wp) {
    for (const auto& v : kVariants)
        if (D <= v.Dp && W <= v.Wp) {
            *Dp = v.Dp;
            *Wp = v.Wp;
            return;
        }
    *Dp = *Wp = -1;
}

bool arm_dims_supported(int D, int W) {
    int a, b;
    arm_padded_dims(D, W, &a, &b);
    return a > 0;
}

template <int DP, int WP>
static size_t arm_smem() {
    return sizeof(ArmSmem<DP, WP>);
}

template <int DP, int WP, int MODE>
static void launch_arm_t(const LaunchCtx& L) {
    const size_t smem = arm_smem<DP, WP>();
    k_arm<DP, WP, MODE><<<dim3(L.arm_blocks, 1, L.batch), kArmTile, smem, L.stream>>>(L.plan, L.arm_tiles,
                                                                    L.arm_ntiles);
}

template <int DP, int WP>
static void configure_t() {
    const int smem = int(arm_smem<DP, WP>());
    cudaFuncSetAttribute(k_arm<DP, WP, kArmForward>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_arm<DP, WP, kArmHard>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_arm<DP, WP, kArmProxy>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

// The register-tiled kernel (cc_arm2.cu) runs every variant it instantiates;
// this per-latent kernel is the fallback for the wide ARMs it does not.
bool arm2_supported(int Dp, int Wp);
size_t arm2_smem_bytes(int Dp, int Wp);
void arm2_configure(int Dp, int Wp);
void launch_arm2(const LaunchCtx& L, int mode);

bool arm_tc_supported(int Dp, int Wp);
size_t arm_tc_smem_bytes(int Dp, int Wp);
int arm_tc_blocks_per_sm(int Dp, int Wp);
void arm_tc_configure(int Dp, int Wp);
void launch_arm_tc(const LaunchCtx& L, int mode);

// The FFMA2 tile kernel (cc_arm2.cu) is the default: per iteration it is the
// faster of the two (512x768 HOP: 0.453 vs 0.489 ms, the tensor-core kernel
// needs 2 x 109 KB of shared memory per SM for its best time and starves the
// concurrent distortion branch).  CCB_ARM=tc selects the
// tensor-core kernel (cc_arm_tc.cu).
static int arm_env() {
    static const int v = [] {
        const char* e = std::getenv("CCB_ARM");
        return (e && e[0] == 't') ? 3 : (e && e[0] == '2') ? 2 : 0;
    }();
    return v;
}
static bool use_tc(int Dp, int Wp) { return arm_env() == 3 && arm_tc_supported(Dp, Wp); }
static bool use_arm2(int Dp, int Wp) { return !use_tc(Dp, Wp) && arm2_supported(Dp, Wp); }

// both tiled kernels stage a (P+1)-row window (row bands, halo <= 4)
bool arm_uses_v2(int Dp, int Wp) { return use_tc(Dp, Wp) || use_arm2(Dp, Wp); }
bool arm_uses_tc(int Dp, int Wp) { return use_tc(Dp, Wp); }

void arm_configure(int Dp, int Wp) {
    if (use_tc(Dp, Wp)) arm_tc_configure(Dp, Wp);
    if (use_arm2(Dp, Wp)) arm2_configure(Dp, Wp);
    if (Dp == 8 && Wp == 8) configure_t<8, 8>();
    else if (Dp == 16 && Wp == 12) configure_t<16, 12>();
    else if (Dp == 20 && Wp == 20) configure_t<20, 20>();
    else if (Dp == 28 && Wp == 28) configure_t<28, 28>();
    else if (Dp == 32 && Wp == 20) configure_t<32, 20>();
    else configure_t<40, 40>();
}

template <int DP, int WP>
static void launch_arm_mode(const LaunchCtx& L, int mode) {
    if (mode == kArmForward)
        launch_arm_t<DP, WP, kArmForward>(L);
    else if (mode == kArmHard)
        launch_arm_t<DP, WP, kArmHard>(L);
    else
        launch_arm_t<DP, WP, kArmProxy>(L);
}


// IFCE weight gradients of the constant-bank ARM's plans (Plan::ifce_sep),
// from the dF block-sum pyramid (entropy_model.hpp:318-321):
//   dW_f[s][f][j] = sum over latents of IFCE grid s of dF[f] * yhat_j(r >> sh, c >> sh)
//                 = sum over the positions (R, C) of source grid j of
//                   yhat_j(R, C) * P_sh[f](R, C),
// P_sh = level sh = level_j - level_s of the pyramid of dF (the same block
// sums k_latent_grad scatters as dR, aligned the same way), and
//   db_f[s][f] = sum of dF[f] = sum over the deepest pyramid level.
// One CTA per work item (s, j, e0, e1) — a chunk of <= kIfceChunk positions
// of source grid j (j = kIfceBias: the deepest pyramid level, for the bias),
// built by the runtime (ifce_dw_items); the item writes its F sums and zeros
// for the rest of its row of slot s's partial region (fixed-order reduction).
constexpr int kIfceThreads = 128;
constexpr int kIfceF = 8;

__global__ void __launch_bounds__(kIfceThreads) k_ifce_dw(const Plan* __restrict__ pp) {
    const Plan& P = pp[blockIdx.z];
    const int4 it = P.ifce_items[blockIdx.x];
    const int s = it.x, j = it.y, e0 = it.z, e1 = it.w;
    const GridGeom& g = P.g[P.slot_gi[s]];
    const int rd = g.rdim, F = P.F;
    const bool bias = j == kIfceBias;
    const int sh = bias ? P.slot_smax[s] : P.g[j].level - g.level;
    const int prows = P.slot_pyr_rows[s][sh], cols = P.slot_pyr_cols[s][sh];
    const float* pyr = P.dfeat + P.slot_pyr_off[s][sh];
    const int64_t pc = int64_t(prows) * cols;
    const FDivU cdiv(cols);
    float acc[kIfceF];
#pragma unroll
    for (int f = 0; f < kIfceF; ++f) acc[f] = 0.0f;
#pragma unroll 4
    for (int e = e0 + threadIdx.x; e < e1; e += kIfceThreads) {
        const int r = cdiv.div(e), c = e - r * cols;
        float w = 1.0f;
        int R = r;
        if (!bias) {
            const GridGeom& sg = P.g[j];
            R = sg.row0 + r - (P.slot_pyr_a[s] >> sh);  // as k_latent_grad's dR gather
            if (R < 0 || R >= prows) continue;
            w = P.yhat_pad[sg.pad_base + int64_t(r) * sg.stride + c];
        }
        const float* q = pyr + int64_t(R) * cols + c;
#pragma unroll
        for (int f = 0; f < kIfceF; ++f)
            if (f < F) acc[f] = fmaf(w, q[int64_t(f) * pc], acc[f]);
    }
    __shared__ float part[kIfceF][kIfceThreads + 1];
#pragma unroll
    for (int f = 0; f < kIfceF; ++f) part[f][threadIdx.x] = acc[f];
    __syncthreads();
    const PartialRegion& Rg = P.region[P.reg_ifce[s]];
    const PartialRow row(P, Rg, blockIdx.x - P.ifce_item0[s]);
    for (int x = threadIdx.x; x < F * (rd + 1); x += kIfceThreads) {
        const int f = x / (rd + 1), b = x % (rd + 1);
        double v = 0.0;
        if ((b < rd && b == j) || (b == rd && bias))
            for (int t = 0; t < kIfceThreads; ++t) v += double(part[f][t]);
        const int o = b < rd ? P.off_ifw[s] + f * rd + b : P.off_ifb[s] + f;
        row[o - Rg.param_off] = v;
    }
}

static void launch_ifce_dw(const LaunchCtx& L) {
    const Plan& H = *L.host;
    if (!H.ifce_sep) return;
    k_ifce_dw<<<dim3(H.n_ifce_items, 1, L.batch), kIfceThreads, 0, L.stream>>>(L.plan);
}

// the work items of k_ifce_dw (row x of slot s's region = item ifce_item0[s] + x)
std::vector<int4> ifce_dw_items(const Plan& P, int* item0) {
    std::vector<int4> v;
    for (int s = 0; s < P.n_slots; ++s) {
        item0[s] = int(v.size());
        const GridGeom& g = P.g[P.slot_gi[s]];
        for (int j = 0; j <= g.rdim; ++j) {
            const bool bias = j == g.rdim;
            const int sh = bias ? P.slot_smax[s] : P.g[j].level - g.level;
            const int n = (bias ? P.slot_pyr_rows[s][sh] : P.g[j].rows) * P.slot_pyr_cols[s][sh];
            for (int e = 0; e < n; e += kIfceChunk)
                v.push_back(make_int4(s, bias ? kIfceBias : j, e, std::min(n, e + kIfceChunk)));
        }
    }
    return v;
}



// The constant-bank ARM (cc_armc.cuh) is the default for the dims it
// instantiates: one constant slot per translation unit cc_armc_s<k>.cu.
// CCB_ARM=2 selects the FFMA2 tile kernel, CCB_ARM=tc the tensor-core one.
#define CCB_ARMC_DECL(k)                                 \
    void armc_launch_s##k(const LaunchCtx& L, int mode); \
    void armc_prep_s##k(const LaunchCtx& L);             \
    void armc_configure_s##k(int Dp, int Wp);
CCB_ARMC_DECL(0)
CCB_ARMC_DECL(1)
CCB_ARMC_DECL(2)
CCB_ARMC_DECL(3)
CCB_ARMC_DECL(4)
CCB_ARMC_DECL(5)
CCB_ARMC_DECL(6)
CCB_ARMC_DECL(7)
#undef CCB_ARMC_DECL
static_assert(kArmcSlots == 8, "one translation unit per slot");
using ArmcLaunch = void (*)(const LaunchCtx&, int);
using ArmcPrep = void (*)(const LaunchCtx&);
using ArmcConf = void (*)(int, int);
static const ArmcLaunch g_armc_launch[kArmcSlots] = {armc_launch_s0, armc_launch_s1, armc_launch_s2, armc_launch_s3,
                                                     armc_launch_s4, armc_launch_s5, armc_launch_s6, armc_launch_s7};
static const ArmcPrep g_armc_prep[kArmcSlots] = {armc_prep_s0, armc_prep_s1, armc_prep_s2, armc_prep_s3,
                                                 armc_prep_s4, armc_prep_s5, armc_prep_s6, armc_prep_s7};
static const ArmcConf g_armc_conf[kArmcSlots] = {armc_configure_s0, armc_configure_s1, armc_configure_s2,
                                                 armc_configure_s3, armc_configure_s4, armc_configure_s5,
                                                 armc_configure_s6, armc_configure_s7};

size_t armc_smem_s0(int Dp, int Wp);

int armc_blocks_per_sm(int Dp, int Wp) {  // resident 64-thread CTAs per SM (shared-memory bound)
    const int b = int((228 * 1024) / (armc_smem_s0(Dp, Wp) + 1024));
    return std::max(1, std::min(kArmcPerSm, b));
}

bool armc_supported(int Dp, int Wp) {
    return arm_env() == 0 && ((Dp == 20 && Wp == 20) || (Dp == 32 && Wp == 20));
}

// Slots are handed out to trainers for their lifetime, exclusively: a
// trainer created while all 8 are taken runs the FFMA2 tile kernel
// (cc_arm2.cu) on the same launch geometry — correct, slower — so any number
// of trainers may run concurrently on any streams.
static std::mutex g_armc_mu;
static bool g_armc_used[kArmcSlots] = {};

int armc_acquire_slot() {
    std::lock_guard<std::mutex> lk(g_armc_mu);
    for (int s = 0; s < kArmcSlots; ++s)
        if (!g_armc_used[s]) {
            g_armc_used[s] = true;
            return s;
        }
    return -1;
}

void armc_release_slot(int slot) {
    if (slot < 0 || slot >= kArmcSlots) return;
    std::lock_guard<std::mutex> lk(g_armc_mu);
    g_armc_used[slot] = false;
}

void armc_configure(int Dp, int Wp) {
    for (int s = 0; s < kArmcSlots; ++s) g_armc_conf[s](Dp, Wp);
}

bool launch_arm_prep(const LaunchCtx& L) {
    static const bool skip = [] {
        const char* e = std::getenv("CCB_DIAG_SKIP_ARM");
        return e && e[0] == '1';
    }();
    if (L.arm_cslot < 0 || skip) return false;
    g_armc_prep[L.arm_cslot](L);
    return true;
}

void launch_arm(const LaunchCtx& L, int mode) {
    const int Dp = L.host->Dp, Wp = L.host->Wp;
    static const bool skip = [] {  // timing diagnostic only (wrong results): the iteration without the ARM
        const char* e = std::getenv("CCB_DIAG_SKIP_ARM");
        return e && e[0] == '1';
    }();
    if (skip) return;
    if (L.arm_cslot >= 0) g_armc_launch[L.arm_cslot](L, mode);
    else if (use_tc(Dp, Wp)) launch_arm_tc(L, mode);
    else if (use_arm2(Dp, Wp)) launch_arm2(L, mode);
    else if (Dp == 8 && Wp == 8) launch_arm_mode<8, 8>(L, mode);
    else if (Dp == 16 && Wp == 12) launch_arm_mode<16, 12>(L, mode);
    else if (Dp == 20 && Wp == 20) launch_arm_mode<20, 20>(L, mode);
    else if (Dp == 28 && Wp == 28) launch_arm_mode<28, 28>(L, mode);
    else if (Dp == 32 && Wp == 20) launch_arm_mode<32, 20>(L, mode);
    else launch_arm_mode<40, 40>(L, mode);
    // Plan::ifce_sep: the IFCE weight gradients come from the dF pyramid
    // (k_ifce_dw); the proxy iteration launches the pyramid after the ARM
    // anyway, a hardround iteration needs it here
    if (mode == kArmHard && L.host->ifce_sep) launch_pyramid(L);
}

int arm_blocks_per_sm(int Dp, int Wp) {
    if (use_tc(Dp, Wp)) return std::min(2, arm_tc_blocks_per_sm(Dp, Wp));  // TMEM: <= 128 columns per CTA
    if (use_arm2(Dp, Wp)) {  // __launch_bounds__(128, 2)
        const int b = int((227 * 1024) / (arm2_smem_bytes(Dp, Wp) + 1024));
        return b < 1 ? 1 : (b > 2 ? 2 : b);
    }
    size_t smem;
    if (Dp == 8 && Wp == 8) smem = arm_smem<8, 8>();
    else if (Dp == 16 && Wp == 12) smem = arm_smem<16, 12>();
    else if (Dp == 20 && Wp == 20) smem = arm_smem<20, 20>();
    else if (Dp == 28 && Wp == 28) smem = arm_smem<28, 28>();
    else if (Dp == 32 && Wp == 20) smem = arm_smem<32, 20>();
    else smem = arm_smem<40, 40>();
    const size_t per_sm = 227 * 1024;
    int b = int(per_sm / (smem + 1024));
    return b < 1 ? 1 : (b > 8 ? 8 : b);
}

static size_t pyramid_smem(const Plan& H) {
    int smax = 0;
    for (int s = 0; s < H.n_slots; ++s) smax = smax > H.slot_smax[s] ? smax : H.slot_smax[s];
    const size_t B = size_t(1) << smax;
    return sizeof(float) * (B * B + (B / 2) * (B / 2));
}

void pyramid_configure(const Plan& H) {
    cudaFuncSetAttribute(k_pyramid_fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(pyramid_smem(H)));
}

void launch_pyramid(const LaunchCtx& L) {
    const Plan& H = *L.host;
    if (H.n_slots == 0 || H.F == 0) return;
    // every slot's deepest level is the coarsest grid: same coarse block count
    int nblk = 0;
    for (int s = 0; s < H.n_slots; ++s)
        nblk = std::max(nblk, H.slot_pyr_rows[s][H.slot_smax[s]] * H.slot_pyr_cols[s][H.slot_smax[s]]);
    const dim3 grid(nblk, H.n_slots * H.F, L.batch);
    k_pyramid_fused<<<grid, 256, pyramid_smem(H), L.stream>>>(L.plan);
    launch_ifce_dw(L);  // constant-bank ARM: the IFCE weight gradients from the pyramid
}

}  // namespace ccb

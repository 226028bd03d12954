// cc_arm2.cu — the auto-regressive entropy model (ARM + IFCE) as a chain of
// register-tiled tile-GEMMs.  Same math and summation orders as cc_arm.cu
// (entropy_model.hpp:180-336); different execution shape:
//
//   * a CTA (128 threads) owns a tile of 128 latents of one grid; every
//     activation lives FEATURE-MAJOR in shared memory ([feature][latent],
//     latents contiguous), so a thread reads 4 latents of a feature with one
//     LDS.128 (conflict-free across the warp);
//   * every dense layer (forward l1, l2; backward dH1 = W2ᵀdH2, dC = W1ᵀdH1 +
//     stabᵀ·draw) is a [128 x K] x [K x N] tile GEMM in which thread
//     (quad q = lane, group g = warp) computes 4 latents x N/4 outputs: per K
//     step one LDS.128 of activations + two LDS.128 of (broadcast) weights
//     feed 4·N/4 FMAs;
//   * the per-latent scalar work (head, Laplace rate and its backward, ReLU
//     masks of the head) runs one thread per latent;
//   * the weight gradients are 4x4 register micro-tiles of
//     [dH1|dH2|draw|dF] x [C|1, H1|1, H2|1, R|1] over the latent axis, split
//     in thirds of the tile so that all 128 threads carry (nearly) the same
//     work, and accumulated in REGISTERS across all tiles of the persistent
//     CTA (fp32 per thread, fp64 at the final per-CTA reduction) — no
//     per-tile shared-memory accumulation, no atomics, fixed order.
//   The IFCE weight gradient (whose output depends on the tile's grid) is
//   staged per tile and added to an fp64 shared accumulator in fixed order.
#include <cuda_runtime.h>

#include "cc_kernels.h"
#include "cc_math.cuh"
#include "cc_reduce.cuh"

namespace ccb {

namespace {

constexpr int T = kArmTile;   // latents per tile == threads per CTA (128)
constexpr int LT = T + 4;     // shared-memory row length (floats)
constexpr int kRM = 12;       // max IFCE source grids
constexpr int kFM = 8;        // max IFCE width

template <int DP, int WP>
struct A2 {
    static_assert(T == 128, "thread mapping assumes 128 latents per tile");
    static_assert(DP % 4 == 0 && WP % 4 == 0 && DP <= 32 && WP <= 32, "padded dims");
    static constexpr int NW = WP / 4;  // outputs per thread, W-wide layers
    static constexpr int ND = DP / 4;  // outputs per thread, D-wide layer
    // feature-major activation rows
    static constexpr int RC = DP + 4;   // C: 0..D-1, ones at DP, own value at DP+1
    static constexpr int RH = WP + 4;   // H1 / H2: ones at WP
    static constexpr int RDH = WP;      // dH1 / dH2
    static constexpr int RDR = 4;       // dmu, dsr, 0, 0
    static constexpr int RR = kRM + 4;  // R: ones at kRM
    static constexpr int RF = kFM;      // dF
    static constexpr int O_C = 0;
    static constexpr int O_H1 = O_C + RC * LT;
    static constexpr int O_H2 = O_H1 + RH * LT;
    static constexpr int O_DH1 = O_H2 + RH * LT;
    static constexpr int O_DH2 = O_DH1 + RDH * LT;
    static constexpr int O_DR = O_DH2 + RDH * LT;
    static constexpr int O_R = O_DR + RDR * LT;
    static constexpr int O_DF = O_R + RR * LT;
    static constexpr int O_C2 = O_DF + RF * LT;  // second C / R buffers: the
    static constexpr int O_R2 = O_C2 + RC * LT;  // next tile's gather lands here
    static constexpr int ACT = O_R2 + RR * LT;
    // weight-gradient jobs (4x4 micro-tiles) and units (job x latent third)
    static constexpr int J1 = (WP / 4) * (DP / 4 + 1);   // dH1 x [C|1]
    static constexpr int J2 = (WP / 4) * (WP / 4 + 1);   // dH2 x [H1|1]
    static constexpr int J3 = WP / 4 + 1;                // draw x [H2|1]
    static constexpr int J4 = DP / 4;                    // draw x C (stabilizer)
    static constexpr int NJ = J1 + J2 + J3 + J4;
    static constexpr int NU = 3 * NJ;                    // register-accumulated units
    static constexpr int J5 = (kFM / 4) * (kRM / 4 + 1); // dF x [R|1] (per tile)
    static constexpr int NU5 = 3 * J5;
    static constexpr int MAXU = (NU + NU5 + T - 1) / T;  // units per thread (upper bound)
    static constexpr int NACC5 = kMaxSlots * kFM * (kRM + 1);
};

template <int DP, int WP>
struct alignas(16) A2Smem {
    using K = A2<DP, WP>;
    alignas(16) float W1T[DP][32];   // [k][out a] (forward l1), group stride 8
    alignas(16) float W1[WP][32];    // [a][out k] (backward dC)
    alignas(16) float W2T[WP][32];   // [k][out a] (forward l2)
    alignas(16) float W2[WP][32];    // [a][out b] (backward dH1)
    alignas(16) float ST[2][32];     // stab [j][out k] (backward dC)
    alignas(16) float W3[2][WP];
    alignas(16) float stab[2][DP];
    alignas(16) float b1[WP];
    alignas(16) float b2[WP];
    alignas(16) float b3[4];
    alignas(16) float Wf[kMaxSlots][kFM][kRM];
    alignas(16) float bf[kMaxSlots][kFM];
    alignas(16) float act[K::ACT];
    alignas(16) float stage5[K::NU5][16];
    double acc5[K::NACC5];  // IFCE dW (+db), per slot, fp64
    GridGeom geo[kMaxGrids];
    int ctx_dy[kMaxCtx], ctx_dx[kMaxCtx];
    double red[T / 32];
};

// 4x4 outer-product micro-tile over latents [i0, i1), step 4: FFMA2 lanes
// carry the even / odd latents, folded into acc (+= even + odd) at the end.
__device__ __forceinline__ void dw_tile(const float* __restrict__ A, const float* __restrict__ B,
                                        int i0, int i1, float (&acc)[16]) {
    float2 p[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) p[e] = make_float2(0.0f, 0.0f);
#pragma unroll 2
    for (int i = i0; i < i1; i += 4) {
        float4 av[4], bv[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            av[r] = *reinterpret_cast<const float4*>(A + r * LT + i);
            bv[r] = *reinterpret_cast<const float4*>(B + r * LT + i);
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                float2 a = p[r * 4 + c];
                a = ffma2(make_float2(av[r].x, av[r].y), make_float2(bv[c].x, bv[c].y), a);
                a = ffma2(make_float2(av[r].z, av[r].w), make_float2(bv[c].z, bv[c].w), a);
                p[r * 4 + c] = a;
            }
    }
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[e] += p[e].x + p[e].y;
}

// one K step of a tile GEMM: 4 latents (x) x N outputs (w, broadcast);
// lo / hi hold latents {0,1} / {2,3} of every output in FFMA2 lanes
template <int N>
__device__ __forceinline__ void gemm_step(const float4& x, const float* w, float2 (&lo)[N], float2 (&hi)[N]) {
#pragma unroll
    for (int n = 0; n < N; ++n) {
        lo[n] = ffma2(make_float2(x.x, x.y), w[n], lo[n]);
        hi[n] = ffma2(make_float2(x.z, x.w), w[n], hi[n]);
    }
}

__device__ __forceinline__ void third_range(int s, int& i0, int& i1) {
    i0 = s * 44;
    i1 = s == 2 ? T : i0 + 44;
}

__device__ __forceinline__ void cp_async4_zfill(float* smem, const float* gmem, bool full) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem), "r"(full ? 4 : 0)
                 : "memory");
}

// Asynchronous gather of tile t (thread = latent): the S causal-context
// values, the latent's own value (row DP+1) and, on IFCE grids, the kRM
// co-located coarser-grid values (zero-filled past rdim / past the grid).
template <int DP>
__device__ __forceinline__ void issue_gather(const Plan& P, const GridGeom* geo, int2 tile,
                                             const int* cdy, const int* cdx, float* sCb, float* sRb,
                                             int tid) {
    const GridGeom& g = geo[tile.x];
    const int64_t count = int64_t(g.rows) * g.cols;
    const int64_t li = int64_t(tile.y) + tid;
    const bool valid = li < count;
    const int r = valid ? int(li / g.cols) : 0;
    const int c = valid ? int(li - int64_t(r) * g.cols) : 0;
    const float* base = P.yhat_pad + g.pad_base + int64_t(r) * g.stride + c;
    const int S = P.S;
#pragma unroll 4
    for (int o = 0; o < S; ++o) cp_async4_zfill(sCb + o * LT + tid, base + cdy[o] * g.stride + cdx[o], valid);
    cp_async4_zfill(sCb + (DP + 1) * LT + tid, base, valid);
    if (g.ifce_slot >= 0) {
        const int rd = g.rdim;
#pragma unroll
        for (int j = 0; j < kRM; ++j) {
            const bool on = valid && j < rd;
            const float* src = P.yhat_pad;
            if (on) {
                const GridGeom& sg = geo[j];
                const int sh = sg.level - g.level;
                src = P.yhat_pad + sg.pad_base + int64_t(r >> sh) * sg.stride + (c >> sh);
            }
            cp_async4_zfill(sRb + j * LT + tid, src, on);
        }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}

__device__ __forceinline__ void swap_bufs(float*& a, float*& b, float*& c, float*& d) {
    float* x = a; a = b; b = x;
    x = c; c = d; d = x;
}

template <int DP, int WP, int MODE>
__global__ void __launch_bounds__(T, 2) k_arm2(const Plan* __restrict__ pp,
                                               const int2* __restrict__ tiles, int ntiles) {
    using K = A2<DP, WP>;
    const Plan& P = *pp;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    A2Smem<DP, WP>& sm = *reinterpret_cast<A2Smem<DP, WP>*>(smem_raw);
    const int tid = threadIdx.x;
    const int lane = tid & 31, grp = tid >> 5;
    const int D = P.D, Wd = P.Wd, S = P.S, F = P.F;
    const float* prm = P.params;

    // ---------------- weights -> shared memory (zero padded) ----------------
    for (int e = tid; e < DP * 32; e += T) {
        const int k = e / 32, c = e % 32, g = c / 8, n = c % 8;
        const int a = g * K::NW + n;  // output of l1 (W-wide)
        sm.W1T[k][c] = (n < K::NW && a < Wd && k < D) ? prm[P.off_l1w + a * D + k] : 0.0f;
    }
    for (int e = tid; e < WP * 32; e += T) {
        const int a = e / 32, c = e % 32, g = c / 8, n = c % 8;
        const int k = g * K::ND + n;  // output of dC (D-wide)
        sm.W1[a][c] = (n < K::ND && a < Wd && k < D) ? prm[P.off_l1w + a * D + k] : 0.0f;
        const int b = g * K::NW + n;  // output of l2 / dH1 (W-wide)
        sm.W2T[a][c] = (n < K::NW && a < Wd && b < Wd) ? prm[P.off_l2w + b * Wd + a] : 0.0f;
        sm.W2[a][c] = (n < K::NW && a < Wd && b < Wd) ? prm[P.off_l2w + a * Wd + b] : 0.0f;
    }
    for (int e = tid; e < 2 * 32; e += T) {
        const int j = e / 32, c = e % 32, g = c / 8, n = c % 8;
        const int k = g * K::ND + n;
        sm.ST[j][c] = (n < K::ND && k < D && P.off_astab >= 0) ? prm[P.off_astab + j * D + k] : 0.0f;
    }
    for (int e = tid; e < 2 * WP; e += T) {
        const int j = e / WP, a = e % WP;
        sm.W3[j][a] = a < Wd ? prm[P.off_hw + j * Wd + a] : 0.0f;
    }
    for (int e = tid; e < 2 * DP; e += T) {
        const int j = e / DP, k = e % DP;
        sm.stab[j][k] = (P.off_astab >= 0 && k < D) ? prm[P.off_astab + j * D + k] : 0.0f;
    }
    for (int e = tid; e < WP; e += T) {
        sm.b1[e] = e < Wd ? prm[P.off_l1b + e] : 0.0f;
        sm.b2[e] = e < Wd ? prm[P.off_l2b + e] : 0.0f;
    }
    if (tid < 4) sm.b3[tid] = tid < 2 ? prm[P.off_hb + tid] : 0.0f;
    for (int e = tid; e < kMaxSlots * kFM * kRM; e += T) {
        const int s = e / (kFM * kRM), r = e % (kFM * kRM), f = r / kRM, j = r % kRM;
        float v = 0.0f;
        if (s < P.n_slots) {
            const int rd = P.g[P.slot_gi[s]].rdim;
            if (f < F && j < rd) v = prm[P.off_ifw[s] + f * rd + j];
        }
        sm.Wf[s][f][j] = v;
    }
    for (int e = tid; e < kMaxSlots * kFM; e += T) {
        const int s = e / kFM, f = e % kFM;
        sm.bf[s][f] = (s < P.n_slots && f < F) ? prm[P.off_ifb[s] + f] : 0.0f;
    }
    for (int e = tid; e < kMaxCtx; e += T) {
        sm.ctx_dy[e] = e < S ? P.ctx_dy[e] : 0;
        sm.ctx_dx[e] = e < S ? P.ctx_dx[e] : 0;
    }
    for (int e = tid; e < K::NACC5; e += T) sm.acc5[e] = 0.0;
    for (int e = tid; e < P.n_grids; e += T) sm.geo[e] = P.g[e];
    // constant rows: zero padding of every activation array (written once)
    for (int e = tid; e < K::ACT; e += T) sm.act[e] = 0.0f;
    __syncthreads();

    float* sC = sm.act + K::O_C;
    float* const sH1 = sm.act + K::O_H1;
    float* const sH2 = sm.act + K::O_H2;
    float* const sDH1 = sm.act + K::O_DH1;
    float* const sDH2 = sm.act + K::O_DH2;
    float* const sDR = sm.act + K::O_DR;
    float* sR = sm.act + K::O_R;
    float* sCn = sm.act + K::O_C2;
    float* sRn = sm.act + K::O_R2;
    // tile records run two ahead of the tile being computed (register
    // prefetch); the gather of tile t+grid is issued while tile t computes
    int2 cur = blockIdx.x < ntiles ? tiles[blockIdx.x] : make_int2(0, 0);
    int2 nxt = blockIdx.x + gridDim.x < ntiles ? tiles[blockIdx.x + gridDim.x] : make_int2(0, 0);
    if (blockIdx.x < ntiles) issue_gather<DP>(P, sm.geo, cur, sm.ctx_dy, sm.ctx_dx, sC, sR, tid);
    float* const sDF = sm.act + K::O_DF;

    // persistent weight-gradient accumulators of this thread's units
    float uacc[K::MAXU][16];
#pragma unroll
    for (int m = 0; m < K::MAXU; ++m)
#pragma unroll
        for (int e = 0; e < 16; ++e) uacc[m][e] = 0.0f;
    double bits_thr = 0.0;
    const float upstream = P.rate_upstream;

    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int2 tile = cur;
        const int2 nxt2 = t + 2 * int(gridDim.x) < ntiles ? tiles[t + 2 * gridDim.x] : make_int2(0, 0);
        const GridGeom& g = sm.geo[tile.x];
        const int64_t count = int64_t(g.rows) * g.cols;
        const int slot = g.ifce_slot;

        // ---- P0/P1: per-latent gather (thread = latent) + IFCE forward ----
        const int64_t li = int64_t(tile.y) + tid;
        const bool valid = li < count;
        {
            // prefetch the next tile into the other buffers (their last readers
            // finished at the previous tile's closing barrier), then wait for
            // this thread's own columns of the current tile
            if (t + int(gridDim.x) < ntiles)
                issue_gather<DP>(P, sm.geo, nxt, sm.ctx_dy, sm.ctx_dx, sCn, sRn, tid);
            else
                asm volatile("cp.async.commit_group;\n" ::: "memory");
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
            if (slot >= 0) {
                float rv[kRM];
#pragma unroll
                for (int j = 0; j < kRM; ++j) rv[j] = sR[j * LT + tid];
                sR[kRM * LT + tid] = valid ? 1.0f : 0.0f;
                for (int f = 0; f < F; ++f) {  // gemm_xwt_fast order: bias, then j
                    float a = sm.bf[slot][f];
#pragma unroll
                    for (int j = 0; j < kRM; ++j) a = fmaf(rv[j], sm.Wf[slot][f][j], a);
                    sC[(S + f) * LT + tid] = valid ? a : 0.0f;
                }
            } else {
                for (int f = 0; f < F; ++f) sC[(S + f) * LT + tid] = 0.0f;
            }
            sC[DP * LT + tid] = valid ? 1.0f : 0.0f;
            sH1[WP * LT + tid] = valid ? 1.0f : 0.0f;
            sH2[WP * LT + tid] = valid ? 1.0f : 0.0f;
        }
        __syncthreads();

        // ---- P2: H1 = relu(b1 + W1·C)   (tile GEMM, 4 latents x NW outputs) ----
        {
            float2 lo[K::NW], hi[K::NW];
#pragma unroll
            for (int n = 0; n < K::NW; ++n) {
                const float b = sm.b1[grp * K::NW + n];
                lo[n] = hi[n] = make_float2(b, b);
            }
#pragma unroll 4
            for (int k = 0; k < DP; ++k) {
                const float4 x = *reinterpret_cast<const float4*>(sC + k * LT + 4 * lane);
                const float* w = &sm.W1T[k][grp * 8];
                gemm_step<K::NW>(x, w, lo, hi);
            }
#pragma unroll
            for (int n = 0; n < K::NW; ++n) {
                const int a = grp * K::NW + n;
                float4 h;
                h.x = lo[n].x > 0.0f ? lo[n].x : 0.0f;
                h.y = lo[n].y > 0.0f ? lo[n].y : 0.0f;
                h.z = hi[n].x > 0.0f ? hi[n].x : 0.0f;
                h.w = hi[n].y > 0.0f ? hi[n].y : 0.0f;
                *reinterpret_cast<float4*>(sH1 + a * LT + 4 * lane) = h;
            }
        }
        __syncthreads();
        // ---- P3: H2 = relu(b2 + W2·H1) ----
        {
            float2 lo[K::NW], hi[K::NW];
#pragma unroll
            for (int n = 0; n < K::NW; ++n) {
                const float b = sm.b2[grp * K::NW + n];
                lo[n] = hi[n] = make_float2(b, b);
            }
#pragma unroll 4
            for (int k = 0; k < WP; ++k) {
                const float4 x = *reinterpret_cast<const float4*>(sH1 + k * LT + 4 * lane);
                const float* w = &sm.W2T[k][grp * 8];
                gemm_step<K::NW>(x, w, lo, hi);
            }
#pragma unroll
            for (int n = 0; n < K::NW; ++n) {
                const int a = grp * K::NW + n;
                float4 h;
                h.x = lo[n].x > 0.0f ? lo[n].x : 0.0f;
                h.y = lo[n].y > 0.0f ? lo[n].y : 0.0f;
                h.z = hi[n].x > 0.0f ? hi[n].x : 0.0f;
                h.w = hi[n].y > 0.0f ? hi[n].y : 0.0f;
                *reinterpret_cast<float4*>(sH2 + a * LT + 4 * lane) = h;
            }
        }
        __syncthreads();
        // ---- P4/P5: head, Laplace rate + its backward, dH2 (thread = latent) ----
        {
            float raw[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                float a = sm.b3[j];
#pragma unroll
                for (int k = 0; k < WP; ++k) a = fmaf(sH2[k * LT + tid], sm.W3[j][k], a);
#pragma unroll
                for (int k = 0; k < DP; ++k) a = fmaf(sC[k * LT + tid], sm.stab[j][k], a);
                raw[j] = a;
            }
            const float v = sC[(DP + 1) * LT + tid];
            const float mu = raw[0];
            const float sg = sigma_from_raw(raw[1]);
            const float bsc = sg * kInvSqrt2F;
            const float u = fabsf(v - mu);
            const float e1 = cc_exp(-(u + 0.5f) / bsc);
            const float e2 = cc_exp(-fabsf(u - 0.5f) / bsc);
            const float p = u >= 0.5f ? 0.5f * (e2 - e1) : 1.0f - 0.5f * (e1 + e2);
            if (valid) bits_thr += double(-(cc_log(std_max(p, kProbFloorF)) * kLog2EF));
            if (MODE != kArmForward) {
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
                if (MODE == kArmProxy && valid) P.gown[g.lat_off + li] = gv;
                sDR[0 * LT + tid] = dmu;
                sDR[1 * LT + tid] = dsr;
#pragma unroll
                for (int a = 0; a < WP; ++a) {  // dH2 = (W3ᵀ draw) ⊙ relu'(H2)
                    float d = fmaf(dmu, sm.W3[0][a], 0.0f);
                    d = fmaf(dsr, sm.W3[1][a], d);
                    sDH2[a * LT + tid] = sH2[a * LT + tid] > 0.0f ? d : 0.0f;
                }
            }
        }
        if (MODE == kArmForward) {
            __syncthreads();  // activations are rewritten by the next tile
            swap_bufs(sC, sCn, sR, sRn);
            cur = nxt;
            nxt = nxt2;
            continue;
        }
        __syncthreads();
        // ---- P6: dH1 = (W2ᵀ·dH2) ⊙ relu'(H1) ----
        {
            float2 lo[K::NW], hi[K::NW];
#pragma unroll
            for (int n = 0; n < K::NW; ++n)
                lo[n] = hi[n] = make_float2(0.0f, 0.0f);
#pragma unroll 4
            for (int a = 0; a < WP; ++a) {
                const float4 x = *reinterpret_cast<const float4*>(sDH2 + a * LT + 4 * lane);
                const float* w = &sm.W2[a][grp * 8];
                gemm_step<K::NW>(x, w, lo, hi);
            }
#pragma unroll
            for (int n = 0; n < K::NW; ++n) {
                const int b = grp * K::NW + n;
                const float4 h = *reinterpret_cast<const float4*>(sH1 + b * LT + 4 * lane);
                float4 d;
                d.x = h.x > 0.0f ? lo[n].x : 0.0f;
                d.y = h.y > 0.0f ? lo[n].y : 0.0f;
                d.z = h.z > 0.0f ? hi[n].x : 0.0f;
                d.w = h.w > 0.0f ? hi[n].y : 0.0f;
                *reinterpret_cast<float4*>(sDH1 + b * LT + 4 * lane) = d;
            }
        }
        __syncthreads();
        // ---- P7: dC = W1ᵀ·dH1 + stabᵀ·draw -> dctx / dF ----
        {
            float2 lo[K::ND], hi[K::ND];
#pragma unroll
            for (int n = 0; n < K::ND; ++n)
                lo[n] = hi[n] = make_float2(0.0f, 0.0f);
#pragma unroll 4
            for (int a = 0; a < WP; ++a) {
                const float4 x = *reinterpret_cast<const float4*>(sDH1 + a * LT + 4 * lane);
                const float* w = &sm.W1[a][grp * 8];
                gemm_step<K::ND>(x, w, lo, hi);
            }
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const float4 x = *reinterpret_cast<const float4*>(sDR + j * LT + 4 * lane);
                const float* w = &sm.ST[j][grp * 8];
                gemm_step<K::ND>(x, w, lo, hi);
            }
            const int64_t l0 = int64_t(tile.y) + 4 * lane;
#pragma unroll
            for (int n = 0; n < K::ND; ++n) {
                const int k = grp * K::ND + n;
                if (k < S) {
                    if (MODE == kArmProxy) {
                        float* dcp = P.dctx + g.dctx_off + int64_t(k) * count + l0;
                        const float vv[4] = {lo[n].x, lo[n].y, hi[n].x, hi[n].y};
#pragma unroll
                        for (int l = 0; l < 4; ++l)
                            if (l0 + l < count) dcp[l] = vv[l];
                    }
                } else if (k < S + F && slot >= 0) {
                    float4 dv = make_float4(lo[n].x, lo[n].y, hi[n].x, hi[n].y);
                    if (l0 + 0 >= count) dv.x = 0.0f;
                    if (l0 + 1 >= count) dv.y = 0.0f;
                    if (l0 + 2 >= count) dv.z = 0.0f;
                    if (l0 + 3 >= count) dv.w = 0.0f;
                    *reinterpret_cast<float4*>(sDF + (k - S) * LT + 4 * lane) = dv;
                    if (MODE == kArmProxy) {
                        float* dfp = P.dfeat + g.dfeat_off + int64_t(k - S) * count + l0;
                        const float vv[4] = {dv.x, dv.y, dv.z, dv.w};
#pragma unroll
                        for (int l = 0; l < 4; ++l)
                            if (l0 + l < count) dfp[l] = vv[l];
                    }
                }
            }
        }
        __syncthreads();
        // ---- P8: weight gradients (register micro-tiles, balanced units) ----
#pragma unroll
        for (int m = 0; m < K::MAXU; ++m) {
            const int u = tid + m * T;
            if (u < K::NU) {
                const int j = u / 3;
                int i0, i1;
                third_range(u % 3, i0, i1);
                const float* A;
                const float* B;
                if (j < K::J1) {
                    constexpr int nq = DP / 4 + 1;
                    A = sDH1 + (4 * (j / nq)) * LT;
                    B = sC + (4 * (j % nq)) * LT;
                } else if (j < K::J1 + K::J2) {
                    constexpr int nq = WP / 4 + 1;
                    const int jj = j - K::J1;
                    A = sDH2 + (4 * (jj / nq)) * LT;
                    B = sH1 + (4 * (jj % nq)) * LT;
                } else if (j < K::J1 + K::J2 + K::J3) {
                    A = sDR;
                    B = sH2 + (4 * (j - K::J1 - K::J2)) * LT;
                } else {
                    A = sDR;
                    B = sC + (4 * (j - K::J1 - K::J2 - K::J3)) * LT;
                }
                dw_tile(A, B, i0, i1, uacc[m]);
            } else if (u < K::NU + K::NU5 && slot >= 0) {
                const int uu = u - K::NU, j = uu / 3;
                int i0, i1;
                third_range(uu % 3, i0, i1);
                constexpr int nq = kRM / 4 + 1;
                float acc5[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) acc5[e] = 0.0f;
                dw_tile(sDF + (4 * (j / nq)) * LT, sR + (4 * (j % nq)) * LT, i0, i1, acc5);
#pragma unroll
                for (int e = 0; e < 16; ++e) sm.stage5[uu][e] = acc5[e];
            }
        }
        __syncthreads();
        if (slot >= 0) {  // IFCE dW: thirds summed in order, then fp64 accumulate
            constexpr int nq = kRM / 4 + 1;
            for (int e = tid; e < K::J5 * 16; e += T) {
                const int j = e / 16, q = e % 16;
                const float v = (sm.stage5[3 * j][q] + sm.stage5[3 * j + 1][q]) + sm.stage5[3 * j + 2][q];
                const int a = 4 * (j / nq) + q / 4, b = 4 * (j % nq) + q % 4;
                if (b <= kRM) sm.acc5[(slot * kFM + a) * (kRM + 1) + b] += double(v);
            }
        }
        __syncthreads();
        swap_bufs(sC, sCn, sR, sRn);
        cur = nxt;
        nxt = nxt2;
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");

    // ---------------- per-CTA results ----------------
    const double tb = block_sum(bits_thr, sm.red);
    if (tid == 0) P.bits_part[blockIdx.x] = tb;
    if (MODE == kArmForward) return;
    const PartialRegion& R = P.region[P.reg_arm];
    double* row = P.partials + R.base + int64_t(blockIdx.x) * R.count;
    // stage the register units in (now dead) activation memory, then every
    // parameter of the region is written exactly once: the three latent
    // thirds of its job summed in order
    float* stage = sm.act;
#pragma unroll
    for (int m = 0; m < K::MAXU; ++m) {
        const int u = tid + m * T;
        if (u < K::NU)
#pragma unroll
            for (int e = 0; e < 16; ++e) stage[u * 16 + e] = uacc[m][e];
    }
    __syncthreads();
    for (int x = tid; x < K::NJ * 16; x += T) {
        const int j = x / 16, q = x % 16;
        const double v = (double(stage[(3 * j) * 16 + q]) + double(stage[(3 * j + 1) * 16 + q])) +
                         double(stage[(3 * j + 2) * 16 + q]);
        int o = -1;
        if (j < K::J1) {
            constexpr int nq = DP / 4 + 1;
            const int a = 4 * (j / nq) + q / 4, b = 4 * (j % nq) + q % 4;
            if (a < Wd) o = b < D ? P.off_l1w + a * D + b : (b == DP ? P.off_l1b + a : -1);
        } else if (j < K::J1 + K::J2) {
            constexpr int nq = WP / 4 + 1;
            const int jj = j - K::J1;
            const int a = 4 * (jj / nq) + q / 4, b = 4 * (jj % nq) + q % 4;
            if (a < Wd) o = b < Wd ? P.off_l2w + a * Wd + b : (b == WP ? P.off_l2b + a : -1);
        } else if (j < K::J1 + K::J2 + K::J3) {
            const int a = q / 4, b = 4 * (j - K::J1 - K::J2) + q % 4;
            if (a < 2) o = b < Wd ? P.off_hw + a * Wd + b : (b == WP ? P.off_hb + a : -1);
        } else {
            const int a = q / 4, b = 4 * (j - K::J1 - K::J2 - K::J3) + q % 4;
            if (a < 2 && b < D && P.off_astab >= 0) o = P.off_astab + a * D + b;
        }
        if (o >= 0) row[o - R.param_off] = v;
    }
    for (int s = 0; s < P.n_slots; ++s) {
        const int rd = P.g[P.slot_gi[s]].rdim;
        for (int e = tid; e < F * (rd + 1); e += T) {
            const int f = e / (rd + 1), b = e % (rd + 1);
            const double v = sm.acc5[(s * kFM + f) * (kRM + 1) + (b < rd ? b : kRM)];
            const int o = b < rd ? P.off_ifw[s] + f * rd + b : P.off_ifb[s] + f;
            row[o - R.param_off] = v;
        }
    }
}

template <int DP, int WP>
size_t arm2_smem() {
    return sizeof(A2Smem<DP, WP>);
}

template <int DP, int WP, int MODE>
void launch_t(const LaunchCtx& L) {
    k_arm2<DP, WP, MODE><<<L.arm_blocks, T, arm2_smem<DP, WP>(), L.stream>>>(L.plan, L.arm_tiles,
                                                                              L.arm_ntiles);
}

template <int DP, int WP>
void launch_mode(const LaunchCtx& L, int mode) {
    if (mode == kArmForward) launch_t<DP, WP, kArmForward>(L);
    else if (mode == kArmHard) launch_t<DP, WP, kArmHard>(L);
    else launch_t<DP, WP, kArmProxy>(L);
}

template <int DP, int WP>
void configure_t() {
    const int smem = int(arm2_smem<DP, WP>());
    cudaFuncSetAttribute(k_arm2<DP, WP, kArmForward>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_arm2<DP, WP, kArmHard>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_arm2<DP, WP, kArmProxy>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

}  // namespace

// instantiated (Dp, Wp): the same variants as cc_arm.cu except the wide fallback
bool arm2_supported(int Dp, int Wp) {
    return (Dp == 8 && Wp == 8) || (Dp == 16 && Wp == 12) || (Dp == 20 && Wp == 20) ||
           (Dp == 28 && Wp == 28) || (Dp == 32 && Wp == 20);
}

size_t arm2_smem_bytes(int Dp, int Wp) {
    if (Dp == 8 && Wp == 8) return arm2_smem<8, 8>();
    if (Dp == 16 && Wp == 12) return arm2_smem<16, 12>();
    if (Dp == 20 && Wp == 20) return arm2_smem<20, 20>();
    if (Dp == 28 && Wp == 28) return arm2_smem<28, 28>();
    return arm2_smem<32, 20>();
}

void arm2_configure(int Dp, int Wp) {
    if (Dp == 8 && Wp == 8) configure_t<8, 8>();
    else if (Dp == 16 && Wp == 12) configure_t<16, 12>();
    else if (Dp == 20 && Wp == 20) configure_t<20, 20>();
    else if (Dp == 28 && Wp == 28) configure_t<28, 28>();
    else if (Dp == 32 && Wp == 20) configure_t<32, 20>();
}

void launch_arm2(const LaunchCtx& L, int mode) {
    const int Dp = L.host->Dp, Wp = L.host->Wp;
    if (Dp == 8 && Wp == 8) launch_mode<8, 8>(L, mode);
    else if (Dp == 16 && Wp == 12) launch_mode<16, 12>(L, mode);
    else if (Dp == 20 && Wp == 20) launch_mode<20, 20>(L, mode);
    else if (Dp == 28 && Wp == 28) launch_mode<28, 28>(L, mode);
    else launch_mode<32, 20>(L, mode);
}

}  // namespace ccb

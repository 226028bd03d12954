// cc_armc.cuh — the auto-regressive entropy model (ARM + IFCE, rate_pass,
// entropy_model.hpp:180-336) with the weights in the CONSTANT BANK.
//
// Included by cc_armc_s<k>.cu with CCB_ARMC_SLOT = k: every translation unit
// owns one constant slot (c_armw, 10 KB) and instantiates the kernels that
// read it, so a kernel's weight operands are constant-bank addresses known at
// compile time (unrolled code) or uniform-register relative (the rolled layer
// loops).  A per-thread runtime slot index would compile to LDC and run 5-15x
// slower (tools/micro/const_ffma.cu).
//
// Execution shape (one CTA = 64 threads = one 128-latent row-segment tile at a
// time, persistent over the tile list):
//   * a thread carries TWO adjacent latents through the whole chain in
//     registers — context gather, IFCE, l1, l2, head, Laplace rate and its
//     backward, dH2, dH1, dC — as packed FFMA2 with the two latents as the two
//     lanes and the weight as a uniform-register scalar loaded straight from
//     the constant bank (LDCU; SASS FFMA2 R, R.F32x2, UR.F32, R): no shared-
//     memory traffic for weights, no barrier inside the chain (probe: a 20x20
//     layer chain at 57-66 TFLOP/s on the B200);
//   * the chain leaves its activations FEATURE-MAJOR in shared memory ([row]
//     [latent], latents contiguous): C, H1, H2, dH1, dH2, draw;
//   * the weight gradients are ONE job per thread: a 4 x NB register
//     micro-tile over the tile's latent axis (dW1 = dH1 x C, dW2 = dH2 x H1,
//     head = draw x [H2 | C]; the bias rows = row sums of the A rows, in the
//     first column group of each family), accumulated in fp64 registers
//     across all tiles of the CTA — deterministic, no atomics;
//   * per CTA one fp64 partial row of every ARM parameter (k_nn_reduce sums
//     the rows in order) and one fp64 bits partial.  The IFCE weight
//     gradients come from the dF pyramid (k_ifce_dw, cc_arm.cu).
// Same data outputs as cc_arm2.cu: dC as S planes (dctx), dF planes (dfeat),
// the own-value gradient (gown), bits_part.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "cc_kernels.h"
#include "cc_math.cuh"
#include "cc_reduce.cuh"

#ifndef CCB_ARMC_SLOT
#error "cc_armc.cuh is included by cc_armc_s<k>.cu"
#endif

namespace ccb {
namespace armc {

constexpr int T = kArmTile;   // latents per tile (128)
constexpr int NT = 64;        // threads per CTA (two latents each)
constexpr int LT = T + 4;     // shared row stride (floats): 132 = 4 mod 32, rows r, r+1, ... on distinct bank quads
constexpr int kRM = 12;       // max IFCE source grids
constexpr int kFM = 8;        // max IFCE width
constexpr int kSlotFloats = 2560;

// constant-slot layout (floats), padded dims, zero padded.  Every dense
// layer's weights are stored with the OUTPUT index contiguous, in the order
// the layer loop walks them (input outer, rolled; outputs inner, unrolled):
// consecutive outputs read consecutive constant words.
template <int DP, int WP>
struct CL {
    static constexpr int W1T = 0;                // [DP][WP]  l1.w[a][k] at (k, a): forward
    static constexpr int W1 = W1T + DP * WP;     // [WP][DP]  l1.w[a][k] at (a, k): dC backward
    static constexpr int B1 = W1 + WP * DP;      // [WP]
    static constexpr int W2T = B1 + WP;          // [WP][WP]  l2.w[b][a] at (a, b): forward
    static constexpr int W2 = W2T + WP * WP;     // [WP][WP]  l2.w[a][b] at (a, b): dH1 backward
    static constexpr int B2 = W2 + WP * WP;      // [WP]
    static constexpr int W3 = B2 + WP;           // [2][WP]
    static constexpr int B3 = W3 + 2 * WP;       // [2] (+2)
    static constexpr int ST = B3 + 4;            // [2][DP]
    static constexpr int WF = ST + 2 * DP;       // [kMaxSlots][kFM][kRM]
    static constexpr int BF = WF + kMaxSlots * kFM * kRM;  // [kMaxSlots][kFM]
    static constexpr int END = BF + kMaxSlots * kFM;
    static_assert(END <= kSlotFloats, "constant slot");
};

// weight-gradient jobs: ONE per thread, all of the same shape — 4 A rows x NB
// B rows (+ the 4 A-row sums on the first B group of a family) over the
// tile's 128 latents.  Rows of a group are strided (row g, g + ng, ...), so a
// warp's loads of one row index hit consecutive rows = distinct bank quads.
template <int DP, int WP>
struct JB {
    static constexpr int NB = DP > WP ? 6 : 4;     // B rows per job
    static constexpr int NGA = WP / 4;             // A row groups of a W-wide array
    static constexpr int NGC = (DP + NB - 1) / NB; // B groups of C
    static constexpr int NGW = (WP + NB - 1) / NB; // B groups of H1
    static constexpr int NGH = (WP + DP + NB - 1) / NB;  // B groups of [H2 | C]
    static constexpr int N1 = NGA * NGC;           // dW1 = dH1 x C (+ b1)
    static constexpr int N2 = NGA * NGW;           // dW2 = dH2 x H1 (+ b2)
    static constexpr int NH = NGH;                 // head = draw x [H2 | C] (+ b3)
    static constexpr int NJ = N1 + N2 + NH;
    static constexpr int NO = 4 * NB + 4;          // outputs per job
    static_assert(NJ <= 64, "one job per thread");
    static_assert(2 * NGA + 1 <= 32, "the row-sum carriers fit in warp 0");
};

struct Job {
    const float* a[4];
    const float* b[6];
    int fam;    // 0 dW1, 1 dW2, 2 head
    int ga, gb;
};

template <int DP, int WP>
struct alignas(16) Smem {
    float C[DP][LT];
    float H1[WP][LT];
    float H2[WP][LT];
    float DH1[WP][LT];
    float DH2[WP][LT];
    float DR[2][LT];
    float ZR[LT];                 // zero row (padding operand)
    GridGeom geo[kMaxGrids];
    int coff[kMaxGrids][DP];      // context offset o of grid gi: dy * padded stride + dx
    int64_t rsrc[2][kRM];         // IFCE source rows of the tile (double-buffered by tile parity):
    int rsh[2][kRM];              //   yhat_pad offset of the source row, column shift
    double red[NT / 32];
};

// the IFCE source rows of tile `tile` (threads t0, t0 + step, ...): the row
// of source grid j that latent row r maps to (global rows, clamped to the
// band window, entropy_model.hpp:239-244) and the column shift
template <int DP, int WP>
__device__ __forceinline__ void ifce_rows(const Plan& P, Smem<DP, WP>& sm, int4 tile, int buf, int t0, int step) {
    const GridGeom& g = sm.geo[tile.x];
    if (g.ifce_slot < 0) return;
    for (int j = t0; j < g.rdim; j += step) {
        const GridGeom& sg = sm.geo[j];
        const int sh = sg.level - g.level;
        const int rs = min(max(((g.row0 + tile.z) >> sh) - sg.row0, 0), sg.rows - 1);
        sm.rsrc[buf][j] = sg.pad_base + int64_t(rs) * sg.stride;
        sm.rsh[buf][j] = sh;
    }
}

// job index -> family / groups: the row-sum carriers (first B group of each
// family) are jobs 0 .. 2 NGA (all in warp 0), so warp 1 skips the sums
template <int DP, int WP>
__device__ __forceinline__ void job_id(int j, int& fam, int& ga, int& gb) {
    using J = JB<DP, WP>;
    if (j <= 2 * J::NGA) {
        gb = 0;
        fam = j < J::NGA ? 0 : (j < 2 * J::NGA ? 1 : 2);
        ga = j < J::NGA ? j : (j < 2 * J::NGA ? j - J::NGA : 0);
        return;
    }
    j -= 2 * J::NGA + 1;
    constexpr int R1 = J::NGA * (J::NGC - 1), R2 = J::NGA * (J::NGW - 1);
    if (j < R1) { fam = 0; ga = j / (J::NGC - 1); gb = 1 + j % (J::NGC - 1); return; }
    j -= R1;
    if (j < R2) { fam = 1; ga = j / (J::NGW - 1); gb = 1 + j % (J::NGW - 1); return; }
    j -= R2;
    fam = 2; ga = 0; gb = 1 + j;
}

template <int DP, int WP>
__device__ __forceinline__ Job job_rows(Smem<DP, WP>& sm, int j) {
    using J = JB<DP, WP>;
    Job jb;
    job_id<DP, WP>(j, jb.fam, jb.ga, jb.gb);
    const int ga = jb.ga, gb = jb.gb;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (jb.fam == 0) jb.a[i] = sm.DH1[ga + i * J::NGA];
        else if (jb.fam == 1) jb.a[i] = sm.DH2[ga + i * J::NGA];
        else jb.a[i] = i < 2 ? sm.DR[i] : sm.ZR;
    }
#pragma unroll
    for (int c = 0; c < J::NB; ++c) {
        if (jb.fam == 0) {
            const int x = gb + c * J::NGC;
            jb.b[c] = x < DP ? sm.C[x] : sm.ZR;
        } else if (jb.fam == 1) {
            const int x = gb + c * J::NGW;
            jb.b[c] = x < WP ? sm.H1[x] : sm.ZR;
        } else {
            const int x = gb + c * J::NGH;
            jb.b[c] = x < WP ? sm.H2[x] : (x < WP + DP ? sm.C[x - WP] : sm.ZR);
        }
    }
    return jb;
}

__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    unsigned long long ua, ub, ud;
    asm("mov.b64 %0, {%1, %2};" : "=l"(ua) : "f"(a.x), "f"(a.y));
    asm("mov.b64 %0, {%1, %2};" : "=l"(ub) : "f"(b.x), "f"(b.y));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(ud) : "l"(ua), "l"(ub));
    float2 d;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(ud));
    return d;
}

// Laplace rate of one latent and its backward (entropy_model.hpp:257-296)
template <int MODE>
__device__ __forceinline__ void laplace(float v, float mu, float sr, bool own, float upstream, double& bits,
                                        float& dmu, float& dsr, float& gv) {
    const float sg = sigma_from_raw(sr);
    const float bsc = sg * kInvSqrt2F;
    const float u = fabsf(v - mu);
    const float e1 = cc_exp(-(u + 0.5f) / bsc);
    const float e2 = cc_exp(-fabsf(u - 0.5f) / bsc);
    const float p = u >= 0.5f ? 0.5f * (e2 - e1) : 1.0f - 0.5f * (e1 + e2);
    if (own) bits += double(-(cc_log(std_max(p, kProbFloorF)) * kLog2EF));
    dmu = dsr = gv = 0.0f;
    if (MODE != kArmForward && own && p > kProbFloorF) {
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
}

__device__ __forceinline__ void store2(float* p, float2 v, bool v0, bool v1) {
    if (v1 && (reinterpret_cast<uintptr_t>(p) & 7) == 0) {
        *reinterpret_cast<float2*>(p) = v;
    } else {
        if (v0) p[0] = v.x;
        if (v1) p[1] = v.y;
    }
}

}  // namespace armc
}  // namespace ccb

// ---------------------------------------------------------------------------
// per-slot part: the constant slot and the kernels that read it
// ---------------------------------------------------------------------------
namespace ccb {
namespace {

using namespace armc;

__constant__ __align__(16) float c_armw[kSlotFloats];

#define CW(i) c_armw[(i)]

// acc[n] += x * w[off + n] for a row of N weights (off a multiple of 4):
// 128-bit uniform constant loads, FFMA2 with the scalar uniform operand
template <int N>
__device__ __forceinline__ void row_fma(float2 x, int off, float2 (&acc)[N]) {
    static_assert(N % 4 == 0, "rows of 4-float groups");
    const float4* w4 = reinterpret_cast<const float4*>(c_armw + off);
#pragma unroll
    for (int g = 0; g < N / 4; ++g) {
        const float4 w = w4[g];
        acc[4 * g] = ffma2(x, w.x, acc[4 * g]);
        acc[4 * g + 1] = ffma2(x, w.y, acc[4 * g + 1]);
        acc[4 * g + 2] = ffma2(x, w.z, acc[4 * g + 2]);
        acc[4 * g + 3] = ffma2(x, w.w, acc[4 * g + 3]);
    }
}

// IFCE forward of IFCE slot IS (gemm_xwt_fast order: bias, then the sources)
template <int DP, int WP, int IS>
__device__ __forceinline__ void ifce_fwd(const float2 (&rv)[kRM], int F, float2 (&f)[kFM]) {
    using W = CL<DP, WP>;
#pragma unroll
    for (int ff = 0; ff < kFM; ++ff) {
        if (ff < F) {
            const float b = CW(W::BF + IS * kFM + ff);
            float2 a = make_float2(b, b);
#pragma unroll
            for (int j = 0; j < kRM; ++j) a = ffma2(rv[j], CW(W::WF + (IS * kFM + ff) * kRM + j), a);
            f[ff] = a;
        } else {
            f[ff] = make_float2(0.0f, 0.0f);
        }
    }
}

// register budget: 168 for the (20,20) kernel (__launch_bounds__ min 6 CTAs:
// 128 bytes of spills, the same speed, and room beside it for the concurrent
// distortion kernels: 0.420 -> 0.412 ms per iteration at 512x768); the
// (32,20) kernel keeps its 227 (spilling it costs 9 %)
template <int DP, int WP, int MODE>
__global__ void __launch_bounds__(NT, DP > WP ? 4 : 6) k_armc(const Plan* __restrict__ pp, const int4* __restrict__ tiles,
                                                int ntiles) {
    using W = CL<DP, WP>;
    using J = JB<DP, WP>;
    const Plan& P = pp[blockIdx.z];
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem<DP, WP>& sm = *reinterpret_cast<Smem<DP, WP>*>(smem_raw);
    const int tid = threadIdx.x;
    const int S = P.S, F = P.F;

    {   // every activation row zero (padding rows are never written again)
        float* rows = &sm.C[0][0];
        constexpr int NR = DP + 4 * WP + 2 + 1;
        for (int e = tid; e < NR * LT; e += NT) rows[e] = 0.0f;
        for (int e = tid; e < P.n_grids; e += NT) sm.geo[e] = P.g[e];
        for (int e = tid; e < kMaxGrids * DP; e += NT) {
            const int gi = e / DP, o = e % DP;
            sm.coff[gi][o] = (gi < P.n_grids && o < S) ? P.ctx_dy[o] * P.g[gi].stride + P.ctx_dx[o] : 0;
        }
    }
    __syncthreads();
    if (blockIdx.x < ntiles) ifce_rows(P, sm, tiles[blockIdx.x], 0, tid, NT);
    __syncthreads();

    // this thread's weight-gradient job (one per thread, persistent fp64
    // accumulators across the CTA's tiles)
    const bool has_job = tid < J::NJ;
    double acc[J::NO];
#pragma unroll
    for (int e = 0; e < J::NO; ++e) acc[e] = 0.0;
    double bits_thr = 0.0;
    const float upstream = P.rate_upstream;
    const int l0 = 2 * tid;

    int par = 0;  // tile parity: rsrc / rsh buffer of the current tile
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, par ^= 1) {
        const int4 tile = tiles[t];
        const GridGeom& g = sm.geo[tile.x];
        const int r = tile.z, len = tile.w, c0 = tile.y - r * g.cols;
        const bool v0 = l0 < len, v1 = l0 + 1 < len;
        const bool own = r >= g.own_lo && r < g.own_hi;
        const int cA = c0 + (v0 ? l0 : 0), cB = c0 + (v1 ? l0 + 1 : 0);
        const int slot = g.ifce_slot;
        const int stride = g.stride;
        const float* rowp = P.yhat_pad + g.pad_base + int64_t(r) * stride;

        // ---- P1: causal context, own value, IFCE sources and features ----
        float2 vv;
        {
            float2 cx[DP];
#pragma unroll
            for (int o = 0; o < DP; ++o) {
                if (o < S) {
                    const int off = sm.coff[tile.x][o];
                    cx[o] = make_float2(v0 ? __ldg(rowp + off + cA) : 0.0f, v1 ? __ldg(rowp + off + cB) : 0.0f);
                }
            }
            vv = make_float2(v0 ? __ldg(rowp + cA) : 0.0f, v1 ? __ldg(rowp + cB) : 0.0f);
#pragma unroll
            for (int o = 0; o < DP; ++o)
                if (o < S) *reinterpret_cast<float2*>(&sm.C[o][l0]) = cx[o];
        }
        if (slot >= 0) {
            float2 rv[kRM];
#pragma unroll
            for (int j = 0; j < kRM; ++j) {
                rv[j] = make_float2(0.0f, 0.0f);
                if (j < g.rdim) {
                    const float* src;
                    int sh;
                    if (MODE == kArmForward) {  // no per-tile barrier in this mode: rows computed here
                        const GridGeom& sg = sm.geo[j];
                        sh = sg.level - g.level;
                        const int rs = min(max(((g.row0 + r) >> sh) - sg.row0, 0), sg.rows - 1);
                        src = P.yhat_pad + sg.pad_base + int64_t(rs) * sg.stride;
                    } else {
                        src = P.yhat_pad + sm.rsrc[par][j];
                        sh = sm.rsh[par][j];
                    }
                    rv[j] = make_float2(v0 ? __ldg(src + (cA >> sh)) : 0.0f, v1 ? __ldg(src + (cB >> sh)) : 0.0f);
                }
            }
            float2 f[kFM];
            if (slot == 0) ifce_fwd<DP, WP, 0>(rv, F, f);
            else if (slot == 1) ifce_fwd<DP, WP, 1>(rv, F, f);
            else ifce_fwd<DP, WP, 2>(rv, F, f);
#pragma unroll
            for (int ff = 0; ff < kFM; ++ff)
                if (ff < F)
                    *reinterpret_cast<float2*>(&sm.C[S + ff][l0]) =
                        make_float2(v0 ? f[ff].x : 0.0f, v1 ? f[ff].y : 0.0f);
        } else {
#pragma unroll
            for (int ff = 0; ff < kFM; ++ff)
                if (ff < F) *reinterpret_cast<float2*>(&sm.C[S + ff][l0]) = make_float2(0.0f, 0.0f);
        }

        // ---- P2: H1 = relu(b1 + W1 C), the stabiliser part of the head ----
        uint32_t m1a = 0, m1b = 0, m2a = 0, m2b = 0;  // relu masks (lane A, lane B)
        float2 h1[WP];
        float2 st0 = make_float2(0.0f, 0.0f), st1 = make_float2(0.0f, 0.0f);
        {
#pragma unroll
            for (int a = 0; a < WP; ++a) {
                const float b = CW(W::B1 + a);
                h1[a] = make_float2(b, b);
            }
            const float* xp = &sm.C[0][l0];
#pragma unroll 4
            for (int k = 0; k < DP; ++k, xp += LT) {  // input outer (own column back from shared memory)
                const float2 x = *reinterpret_cast<const float2*>(xp);
                row_fma<WP>(x, W::W1T + k * WP, h1);
                st0 = ffma2(x, CW(W::ST + k), st0);
                st1 = ffma2(x, CW(W::ST + DP + k), st1);
            }
#pragma unroll
            for (int a = 0; a < WP; ++a) {
                const bool pa = h1[a].x > 0.0f, pb = h1[a].y > 0.0f;
                h1[a] = make_float2(pa ? h1[a].x : 0.0f, pb ? h1[a].y : 0.0f);
                m1a |= uint32_t(pa) << a;
                m1b |= uint32_t(pb) << a;
                *reinterpret_cast<float2*>(&sm.H1[a][l0]) = h1[a];
            }
        }
        // ---- P3: H2 = relu(b2 + W2 H1), head raw = b3 + W3 H2 + stab C ----
        float2 raw0, raw1;
        {
            float2 h2[WP];
#pragma unroll
            for (int b = 0; b < WP; ++b) {
                const float bb = CW(W::B2 + b);
                h2[b] = make_float2(bb, bb);
            }
            const float* xp = &sm.H1[0][l0];
#pragma unroll 4
            for (int a = 0; a < WP; ++a, xp += LT) {
                const float2 x = *reinterpret_cast<const float2*>(xp);
                row_fma<WP>(x, W::W2T + a * WP, h2);
            }
            const float b30 = CW(W::B3), b31 = CW(W::B3 + 1);
            raw0 = make_float2(b30, b30);
            raw1 = make_float2(b31, b31);
#pragma unroll
            for (int b = 0; b < WP; ++b) {
                const bool pa = h2[b].x > 0.0f, pb = h2[b].y > 0.0f;
                h2[b] = make_float2(pa ? h2[b].x : 0.0f, pb ? h2[b].y : 0.0f);
                m2a |= uint32_t(pa) << b;
                m2b |= uint32_t(pb) << b;
                *reinterpret_cast<float2*>(&sm.H2[b][l0]) = h2[b];
                raw0 = ffma2(h2[b], CW(W::W3 + b), raw0);
                raw1 = ffma2(h2[b], CW(W::W3 + WP + b), raw1);
            }
            raw0 = make_float2(raw0.x + st0.x, raw0.y + st0.y);
            raw1 = make_float2(raw1.x + st1.x, raw1.y + st1.y);
        }
        // ---- P4: Laplace rate and its backward ----
        float2 dmu, dsr;
        {
            float gva, gvb;
            laplace<MODE>(vv.x, raw0.x, raw1.x, v0 && own, upstream, bits_thr, dmu.x, dsr.x, gva);
            laplace<MODE>(vv.y, raw0.y, raw1.y, v1 && own, upstream, bits_thr, dmu.y, dsr.y, gvb);
            if (MODE == kArmProxy) store2(P.gown + g.lat_off + tile.y + l0, make_float2(gva, gvb), v0, v1);
        }
        if (MODE == kArmForward) continue;
        *reinterpret_cast<float2*>(&sm.DR[0][l0]) = dmu;
        *reinterpret_cast<float2*>(&sm.DR[1][l0]) = dsr;
        // ---- P5: dH2 = (W3^T draw) . relu'(H2); dH1 = (W2^T dH2) . relu'(H1) ----
        float2 dh1[WP];
        {
            float2 dh2[WP];
#pragma unroll
            for (int a = 0; a < WP; ++a) {
                float2 d = ffma2(dmu, CW(W::W3 + a), make_float2(0.0f, 0.0f));
                d = ffma2(dsr, CW(W::W3 + WP + a), d);
                dh2[a] = make_float2((m2a >> a) & 1u ? d.x : 0.0f, (m2b >> a) & 1u ? d.y : 0.0f);
                *reinterpret_cast<float2*>(&sm.DH2[a][l0]) = dh2[a];
            }
#pragma unroll
            for (int b = 0; b < WP; ++b) dh1[b] = make_float2(0.0f, 0.0f);
            const float* xp = &sm.DH2[0][l0];
#pragma unroll 4
            for (int a = 0; a < WP; ++a, xp += LT) {
                const float2 x = *reinterpret_cast<const float2*>(xp);
                row_fma<WP>(x, W::W2 + a * WP, dh1);
            }
#pragma unroll
            for (int b = 0; b < WP; ++b) {
                dh1[b] = make_float2((m1a >> b) & 1u ? dh1[b].x : 0.0f, (m1b >> b) & 1u ? dh1[b].y : 0.0f);
                *reinterpret_cast<float2*>(&sm.DH1[b][l0]) = dh1[b];
            }
        }
        // ---- P6: dC = W1^T dH1 + stab^T draw -> context planes, dF ----
        {
            float2 dc[DP];
#pragma unroll
            for (int k = 0; k < DP; ++k) dc[k] = make_float2(0.0f, 0.0f);
            const float* xp = &sm.DH1[0][l0];
#pragma unroll 4
            for (int a = 0; a < WP; ++a, xp += LT) {
                const float2 x = *reinterpret_cast<const float2*>(xp);
                row_fma<DP>(x, W::W1 + a * DP, dc);
            }
#pragma unroll
            for (int k = 0; k < DP; ++k) {
                dc[k] = ffma2(dmu, CW(W::ST + k), dc[k]);
                dc[k] = ffma2(dsr, CW(W::ST + DP + k), dc[k]);
            }
            const int64_t count = int64_t(g.rows) * g.cols;
            const int64_t li = int64_t(tile.y) + l0;
            float* dcp = P.dctx + g.dctx_off + li;
#pragma unroll
            for (int k = 0; k < DP; ++k, dcp += count) {
                if (k < S) {
                    if (MODE == kArmProxy) store2(dcp, dc[k], v0, v1);
                } else if (k < S + F && slot >= 0) {
                    // dF: the dR pyramid (k_pyramid_fused) and the IFCE weight gradient (k_ifce_dw)
                    const float2 dv = make_float2(v0 ? dc[k].x : 0.0f, v1 ? dc[k].y : 0.0f);
                    if (MODE != kArmForward) store2(P.dfeat + g.dfeat_off + int64_t(k - S) * count + li, dv, v0, v1);
                }
            }
        }
        __syncthreads();  // every activation row of the tile is in shared memory

        // ---- P7: this thread's weight-gradient job over the tile; the
        // threads without a job prepare the next tile's IFCE source rows ----
        if (!has_job && t + int(gridDim.x) < ntiles)
            ifce_rows(P, sm, tiles[t + gridDim.x], par ^ 1, tid - J::NJ, NT - J::NJ);
        if (has_job) {
            const Job jb = job_rows<DP, WP>(sm, tid);
            {
                constexpr int NB = J::NB;
                const bool sums = jb.gb == 0;
                float2 p[4 * NB], s4[4];
#pragma unroll
                for (int e = 0; e < 4 * NB; ++e) p[e] = make_float2(0.0f, 0.0f);
#pragma unroll
                for (int i = 0; i < 4; ++i) s4[i] = make_float2(0.0f, 0.0f);
                // the row-sum carriers are all in warp 0 (job_id): warp 1 runs
                // the loop without the sums (a warp-uniform branch)
                auto quads = [&](auto with_sums) {
#pragma unroll 2
                    for (int q = 0; q < T / 4; ++q) {
                        float4 av[4], bv[NB];
#pragma unroll
                        for (int i = 0; i < 4; ++i) av[i] = *reinterpret_cast<const float4*>(jb.a[i] + 4 * q);
#pragma unroll
                        for (int c = 0; c < NB; ++c) bv[c] = *reinterpret_cast<const float4*>(jb.b[c] + 4 * q);
#pragma unroll
                        for (int i = 0; i < 4; ++i)
#pragma unroll
                            for (int c = 0; c < NB; ++c) {
                                float2 t = p[i * NB + c];
                                t = ffma2(make_float2(av[i].x, av[i].y), make_float2(bv[c].x, bv[c].y), t);
                                t = ffma2(make_float2(av[i].z, av[i].w), make_float2(bv[c].z, bv[c].w), t);
                                p[i * NB + c] = t;
                            }
                        if (decltype(with_sums)::value && sums) {
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                s4[i] = fadd2(s4[i], make_float2(av[i].x, av[i].y));
                                s4[i] = fadd2(s4[i], make_float2(av[i].z, av[i].w));
                            }
                        }
                    }
                };
                if (tid < 32) quads(std::true_type{});
                else quads(std::false_type{});
                {
#pragma unroll
                    for (int e = 0; e < 4 * NB; ++e) acc[e] += double(p[e].x + p[e].y);
#pragma unroll
                    for (int i = 0; i < 4; ++i) acc[4 * NB + i] += double(s4[i].x + s4[i].y);
                }
            }
        }
        __syncthreads();  // the tile's activation rows are free again
    }

    // ---------------- per-CTA results ----------------
    const double tb = block_sum(bits_thr, sm.red);
    if (tid == 0) P.bits_part[blockIdx.x] = tb;
    if (MODE == kArmForward) return;
    const PartialRegion& R = P.region[P.reg_arm];
    const PartialRow row(P, R, blockIdx.x);
    const int D = P.D, Wd = P.Wd;
    if (has_job) {
        int fam, ga, gb;
        job_id<DP, WP>(tid, fam, ga, gb);
        {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
#pragma unroll
                for (int c = 0; c < J::NB; ++c) {
                    int o = -1;
                    if (fam == 0) {
                        const int a = ga + i * J::NGA, kk = gb + c * J::NGC;
                        if (a < Wd && kk < D) o = P.off_l1w + a * D + kk;
                    } else if (fam == 1) {
                        const int a = ga + i * J::NGA, b = gb + c * J::NGW;
                        if (a < Wd && b < Wd) o = P.off_l2w + a * Wd + b;
                    } else if (i < 2) {
                        const int x = gb + c * J::NGH;
                        if (x < WP) {
                            if (x < Wd) o = P.off_hw + i * Wd + x;
                        } else if (x - WP < D && P.off_astab >= 0) {
                            o = P.off_astab + i * D + (x - WP);
                        }
                    }
                    if (o >= 0) row[o - R.param_off] = acc[i * J::NB + c];
                }
                if (gb == 0) {
                    int o = -1;
                    if (fam == 0) {
                        if (ga + i * J::NGA < Wd) o = P.off_l1b + ga + i * J::NGA;
                    } else if (fam == 1) {
                        if (ga + i * J::NGA < Wd) o = P.off_l2b + ga + i * J::NGA;
                    } else if (i < 2) {
                        o = P.off_hb + i;
                    }
                    if (o >= 0) row[o - R.param_off] = acc[4 * J::NB + i];
                }
            }
        }
    }
    // (the IFCE weight gradients: k_ifce_dw's own region, Plan::ifce_sep)
}

// the padded constant image of each image's ARM weights (one thread per entry)
template <int DP, int WP>
__global__ void k_armc_pack(const Plan* __restrict__ pp) {
    using W = CL<DP, WP>;
    const Plan& P = pp[blockIdx.z];
    float* o = P.arm_cstage;
    const float* prm = P.params;
    const int D = P.D, Wd = P.Wd, F = P.F;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < W::END) {
        float v = 0.0f;
        if (e < W::W1) {
            const int k = e / WP, a = e % WP;
            if (a < Wd && k < D) v = prm[P.off_l1w + a * D + k];
        } else if (e < W::B1) {
            const int a = (e - W::W1) / DP, k = (e - W::W1) % DP;
            if (a < Wd && k < D) v = prm[P.off_l1w + a * D + k];
        } else if (e < W::W2T) {
            const int a = e - W::B1;
            if (a < Wd) v = prm[P.off_l1b + a];
        } else if (e < W::W2) {
            const int a = (e - W::W2T) / WP, b = (e - W::W2T) % WP;
            if (a < Wd && b < Wd) v = prm[P.off_l2w + b * Wd + a];
        } else if (e < W::B2) {
            const int a = (e - W::W2) / WP, b = (e - W::W2) % WP;
            if (a < Wd && b < Wd) v = prm[P.off_l2w + a * Wd + b];
        } else if (e < W::W3) {
            const int b = e - W::B2;
            if (b < Wd) v = prm[P.off_l2b + b];
        } else if (e < W::B3) {
            const int j = (e - W::W3) / WP, a = (e - W::W3) % WP;
            if (a < Wd) v = prm[P.off_hw + j * Wd + a];
        } else if (e < W::ST) {
            const int j = e - W::B3;
            if (j < 2) v = prm[P.off_hb + j];
        } else if (e < W::WF) {
            const int j = (e - W::ST) / DP, k = (e - W::ST) % DP;
            if (k < D && P.off_astab >= 0) v = prm[P.off_astab + j * D + k];
        } else if (e < W::BF) {
            const int x = e - W::WF, s = x / (kFM * kRM), f = (x / kRM) % kFM, j = x % kRM;
            if (s < P.n_slots) {
                const int rd = P.g[P.slot_gi[s]].rdim;
                if (f < F && j < rd) v = prm[P.off_ifw[s] + f * rd + j];
            }
        } else {
            const int x = e - W::BF, s = x / kFM, f = x % kFM;
            if (s < P.n_slots && f < F) v = prm[P.off_ifb[s] + f];
        }
        o[e] = v;
    }
}

template <int DP, int WP, int MODE>
void launch_mode_t(const LaunchCtx& L, const Plan* plan) {
    k_armc<DP, WP, MODE><<<dim3(L.arm_blocks, 1, 1), NT, sizeof(Smem<DP, WP>), L.stream>>>(plan, L.arm_tiles,
                                                                                        L.arm_ntiles);
}

template <int DP, int WP>
void fill_slot(const LaunchCtx& L, int b) {
    cuda_check(cudaMemcpyToSymbolAsync(c_armw, L.arm_cstages[b], sizeof(float) * CL<DP, WP>::END, 0,
                                       cudaMemcpyDeviceToDevice, L.stream),
               "cudaMemcpyToSymbolAsync(ARM weights)");
}

template <int DP, int WP>
void prep_t(const LaunchCtx& L) {
    k_armc_pack<DP, WP><<<dim3((CL<DP, WP>::END + 127) / 128, 1, L.batch), 128, 0, L.stream>>>(L.plan);
    fill_slot<DP, WP>(L, 0);
}

template <int DP, int WP>
void launch_t(const LaunchCtx& L, int mode) {
    if (!L.arm_prepped) prep_t<DP, WP>(L);
    // one image at a time: its padded weights into this slot, then the ARM
    for (int b = 0; b < L.batch; ++b) {
        if (b > 0) fill_slot<DP, WP>(L, b);
        if (mode == kArmForward) launch_mode_t<DP, WP, kArmForward>(L, L.plan + b);
        else if (mode == kArmHard) launch_mode_t<DP, WP, kArmHard>(L, L.plan + b);
        else launch_mode_t<DP, WP, kArmProxy>(L, L.plan + b);
    }
}

template <int DP, int WP>
void configure_t() {
    const int smem = int(sizeof(Smem<DP, WP>));
    cudaFuncSetAttribute(k_armc<DP, WP, kArmForward>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_armc<DP, WP, kArmHard>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_armc<DP, WP, kArmProxy>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

#undef CW

}  // namespace

#define CCB_ARMC_CAT2(a, b) a##b
#define CCB_ARMC_CAT(a, b) CCB_ARMC_CAT2(a, b)

void CCB_ARMC_CAT(armc_launch_s, CCB_ARMC_SLOT)(const LaunchCtx& L, int mode) {
    const int Dp = L.host->Dp, Wp = L.host->Wp;
    if (Dp == 20 && Wp == 20) launch_t<20, 20>(L, mode);
    else if (Dp == 32 && Wp == 20) launch_t<32, 20>(L, mode);
    else throw_config("constant-bank ARM: unsupported padded dims");
}

void CCB_ARMC_CAT(armc_prep_s, CCB_ARMC_SLOT)(const LaunchCtx& L) {
    if (L.host->Dp == 32) prep_t<32, 20>(L);
    else prep_t<20, 20>(L);
}

size_t CCB_ARMC_CAT(armc_smem_s, CCB_ARMC_SLOT)(int Dp, int Wp) {
    return Dp == 32 ? sizeof(Smem<32, 20>) : sizeof(Smem<20, 20>);
}

void CCB_ARMC_CAT(armc_configure_s, CCB_ARMC_SLOT)(int Dp, int Wp) {
    if (Dp == 20 && Wp == 20) configure_t<20, 20>();
    else if (Dp == 32 && Wp == 20) configure_t<32, 20>();
}

}  // namespace ccb

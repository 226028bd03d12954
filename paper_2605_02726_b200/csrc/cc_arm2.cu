// cc_arm2.cu — the auto-regressive entropy model (ARM + IFCE) as a chain of
// register-tiled tile-GEMMs.  Same math and per-output summation orders as
// cc_arm.cu (entropy_model.hpp:180-336); different execution shape:
//
//   * a CTA (256 threads, 8 warps) owns a tile of 128 latents of one grid;
//     every activation lives FEATURE-MAJOR in shared memory ([feature][latent],
//     latents contiguous), so a thread reads 2 latents of a feature with one
//     LDS.64 (conflict-free across the warp);
//   * every dense layer (forward l1, l2; backward dH1 = W2ᵀdH2, dC = W1ᵀdH1 +
//     stabᵀ·draw) is a [128 x K] x [K x N] tile GEMM in which thread
//     (latent pair p, output group g) computes 2 latents x N/4 outputs with
//     packed FFMA2 (the two latents are the two lanes, the weight is the
//     FFMA2 broadcast operand);
//   * the per-latent work (causal-context gather, IFCE, the two head outputs,
//     Laplace rate and its backward) runs on one or two threads per latent;
//   * the weight gradients are 4x4 register micro-tiles of
//     [dH1|dH2|draw|dF] x [C|1, H1|1, H2|1, R|1] over the latent axis, split
//     in thirds of the tile so that the 256 threads carry (nearly) the same
//     work, accumulated in REGISTERS across all tiles of the persistent CTA
//     (fp32 per thread, fp64 at the final per-CTA reduction) — no per-tile
//     shared-memory accumulation, no atomics, fixed order.  The IFCE weight
//     gradient (whose output depends on the tile's grid) is staged per tile
//     and added to an fp64 shared accumulator in fixed order;
//   * the gather of tile t + grid is issued with cp.async (zero-fill past the
//     grid) into a second set of buffers while tile t computes.
#include <cuda_runtime.h>

#include <cstdint>

#pragma nv_diag_suppress 128  // forward-only instantiations skip the backward phases

#include "cc_kernels.h"
#include "cc_math.cuh"
#include "cc_reduce.cuh"
#include "cc_ctx.cuh"
#include "cc_tile.cuh"

namespace ccb {

namespace {

constexpr int T = kArmTile;   // latents per tile (128)
constexpr int NT = 2 * T;     // threads per CTA
constexpr int LT = T + 4;     // shared-memory row length (floats)
constexpr int kRM = 12;       // max IFCE source grids
constexpr int kFM = 8;        // max IFCE width
constexpr int kMaxPad = 4;    // context window halo (yhat_pad border P)
constexpr int WS = T + 2 * kMaxPad;  // context window row: columns c0-P .. c0+len-1+P
static_assert(WS == kArmWinCols, "the window row is the TMA box row (Trainer::make_pad_maps)");
constexpr int WC = (kMaxPad + 1) * WS;  // context part of a window
// + R rows [j][latent]: sources, ones at kRM, zeros; a multiple of 32 floats
// so that both window buffers start on the 128 bytes the TMA destination needs
constexpr int WIN = (WC + (kRM + 4) * LT + 31) & ~31;

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
    static constexpr int RF = kFM;      // dF
    static constexpr int O_C = 0;
    static constexpr int O_H1 = O_C + RC * LT;
    static constexpr int O_H2 = O_H1 + RH * LT;
    static constexpr int O_DH1 = O_H2 + RH * LT;
    static constexpr int O_DH2 = O_DH1 + RDH * LT;
    static constexpr int O_DR = O_DH2 + RDH * LT;
    static constexpr int O_DF = O_DR + RDR * LT;
    // head partials [group][mu|sigma-raw]: written in P3, read in P4b, so
    // they share dH1's rows (first written in P6); keeps the (32, 20)
    // variant (cfg4) at two CTAs per SM
    static constexpr int O_HP = O_DH1;
    static_assert(RDH >= 8, "head partials fit in the dH1 rows");
    static constexpr int ACT = O_DF + RF * LT;
    // weight-gradient jobs (4x4 micro-tiles) and units (job x latent third)
    static constexpr int J1 = (WP / 4) * (DP / 4 + 1);   // dH1 x [C|1]
    static constexpr int J2 = (WP / 4) * (WP / 4 + 1);   // dH2 x [H1|1]
    static constexpr int J3 = WP / 4 + 1;                // draw x [H2|1]
    static constexpr int J4 = DP / 4;                    // draw x C (stabilizer)
    static constexpr int NJ = J1 + J2 + J3 + J4;
    static constexpr int NU = 3 * NJ;                    // register-accumulated units
    static constexpr int J5 = (kFM / 4) * (kRM / 4 + 1); // dF x [R|1] (per tile)
    static constexpr int NU5 = 3 * J5;
    static constexpr int MAXU = (NU + NU5 + NT - 1) / NT;  // units per thread (upper bound)
    static constexpr int NACC5 = kMaxSlots * kFM * (kRM + 1);
    static_assert(NU * 16 <= ACT, "epilogue staging fits in the activation buffers");
    static_assert(2 * RH >= DP, "dC rows (S <= D <= DP) fit in the H1 / H2 rows");
};

template <int DP, int WP>
struct alignas(128) A2Smem {
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
    alignas(128) float win[2][WIN];  // gather windows: this tile's, the next tile's
    int woff[kMaxCtx];               // context offset o -> window position
    alignas(16) float stage5[K::NU5][16];
    double acc5[K::NACC5];  // IFCE dW (+db), per slot, fp64
    GridGeom geo[kMaxGrids];
    double red[NT / 32];
    alignas(16) int4 trec[4];  // tile records two ahead, landed by cp.async with the gathers
    alignas(8) uint64_t wbar[2];  // TMA completion of each window buffer's context rows
    CtxTable ctxt;  // context offsets by target row (cc_ctx.cuh)
};

template <typename AccT>
__device__ __forceinline__ void dw_tile(const float* __restrict__ A, const float* __restrict__ B,
                                        int i0, int i1, AccT (&acc)[16]) {
    dw_tile4x4<LT>(A, B, i0, i1, acc);
}

// a tile GEMM over K rows of X (feature-major, LT stride): thread's 2 latents
// at column 2p, N outputs of group g; acc holds (latent 2p, latent 2p+1)
template <int N, int K>
__device__ __forceinline__ void tile_gemm(const float* __restrict__ X, const float (*W)[32], int p, int g,
                                          float2 (&acc)[N]) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const float2 x = *reinterpret_cast<const float2*>(X + k * LT + 2 * p);
        const float* w = &W[k][g * 8];
#pragma unroll
        for (int n = 0; n < N; ++n) acc[n] = ffma2(x, w[n], acc[n]);
    }
}

__device__ __forceinline__ void third_range(int s, int& i0, int& i1) {
    i0 = s * 44;
    i1 = s == 2 ? T : i0 + 44;
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

struct alignas(64) CUtensorMapOpaque {  // CUtensorMap (cuda.h): 128 opaque bytes
    unsigned long long opaque[16];
};

__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, unsigned parity) {
    const unsigned sb = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    asm volatile(
        "{\n\t.reg .pred done;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
        "@!done bra WAIT_%=;\n\t}\n" ::"r"(sb),
        "r"(parity)
        : "memory");
}

// Asynchronous gather of one row-segment tile (grid tile.x, latents
// tile.y .. tile.y+len-1 = row r, columns c0 .. c0+len-1) into a window
// buffer: the P+1 padded rows r-P .. r over columns c0-P .. c0-P+WS-1 (the
// causal context of every latent of the tile, zero border included) as ONE
// TMA box load (cp.async.bulk.tensor.2d from the grid's padded array,
// Trainer::make_pad_maps; zero fill past the array) completing on `bar`, and
// on IFCE grids the R rows [j][latent] = ŷ of coarser grid j < rdim at
// (r >> sh, c >> sh) (global rows, clamped to the band) — one warp per
// source grid, cp.async.  All 256 threads; always commits one cp.async group.
__device__ __forceinline__ void issue_gather(const Plan& P, const GridGeom* geo, int4 tile, float* win,
                                             uint64_t* bar, int tid) {
    const GridGeom& g = geo[tile.x];
    const int r = tile.z, len = tile.w, c0 = tile.y - r * g.cols;
    if (tid == 0) {
        const unsigned sb = static_cast<unsigned>(__cvta_generic_to_shared(bar));
        const unsigned sw = static_cast<unsigned>(__cvta_generic_to_shared(win));
        const unsigned bytes = unsigned(WS) * unsigned(P.P + 1) * 4u;
        const CUtensorMapOpaque* map = static_cast<const CUtensorMapOpaque*>(P.pad_maps) + tile.x;
        // the buffer's previous (generic-proxy) readers are ordered before the async-proxy write
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sb), "r"(bytes) : "memory");
        // box origin in padded coordinates: column c0 (= c0 - P unpadded), row r (= r - P)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(sw),
            "l"(map), "r"(c0), "r"(r), "r"(sb)
            : "memory");
    }
    if (g.ifce_slot >= 0) {
        float* wr = win + WC;
        const int warp = tid >> 5, lane = tid & 31;
        for (int j = warp; j < g.rdim; j += NT / 32) {
            const GridGeom& sg = geo[j];
            const int sh = sg.level - g.level;
            const int rs = min(max(((g.row0 + r) >> sh) - sg.row0, 0), sg.rows - 1);
            const float* src = P.yhat_pad + sg.pad_base + int64_t(rs) * sg.stride;
            for (int x = lane; x < len; x += 32) cp_async4(wr + j * LT + x, src + ((c0 + x) >> sh));
        }
    }
    cp_async_commit();
}

template <int DP, int WP, int MODE>
__global__ void __launch_bounds__(NT, 2) k_arm2(const Plan* __restrict__ pp,
                                                const int4* __restrict__ tiles, int ntiles) {
    using K = A2<DP, WP>;
    const Plan& P = pp[blockIdx.z];  // batched launches: one plan per image
    extern __shared__ __align__(128) unsigned char smem_raw[];
    A2Smem<DP, WP>& sm = *reinterpret_cast<A2Smem<DP, WP>*>(smem_raw);
    const int tid = threadIdx.x;
    const int half = tid >> 7, lt = tid & (T - 1);   // per-latent roles
    const int pr = tid & 63, grp = tid >> 6;         // tile-GEMM roles
    const int D = P.D, Wd = P.Wd, S = P.S, F = P.F;
    const float* prm = P.params;

    // ---------------- weights -> shared memory (zero padded) ----------------
    for (int e = tid; e < DP * 32; e += NT) {
        const int k = e / 32, c = e % 32, g = c / 8, n = c % 8;
        const int a = g * K::NW + n;  // output of l1 (W-wide)
        sm.W1T[k][c] = (n < K::NW && a < Wd && k < D) ? prm[P.off_l1w + a * D + k] : 0.0f;
    }
    for (int e = tid; e < WP * 32; e += NT) {
        const int a = e / 32, c = e % 32, g = c / 8, n = c % 8;
        const int k = g * K::ND + n;  // output of dC (D-wide)
        sm.W1[a][c] = (n < K::ND && a < Wd && k < D) ? prm[P.off_l1w + a * D + k] : 0.0f;
        const int b = g * K::NW + n;  // output of l2 / dH1 (W-wide)
        sm.W2T[a][c] = (n < K::NW && a < Wd && b < Wd) ? prm[P.off_l2w + b * Wd + a] : 0.0f;
        sm.W2[a][c] = (n < K::NW && a < Wd && b < Wd) ? prm[P.off_l2w + a * Wd + b] : 0.0f;
    }
    for (int e = tid; e < 2 * 32; e += NT) {
        const int j = e / 32, c = e % 32, g = c / 8, n = c % 8;
        const int k = g * K::ND + n;
        sm.ST[j][c] = (n < K::ND && k < D && P.off_astab >= 0) ? prm[P.off_astab + j * D + k] : 0.0f;
    }
    for (int e = tid; e < 2 * WP; e += NT) {
        const int j = e / WP, a = e % WP;
        sm.W3[j][a] = a < Wd ? prm[P.off_hw + j * Wd + a] : 0.0f;
    }
    for (int e = tid; e < 2 * DP; e += NT) {
        const int j = e / DP, k = e % DP;
        sm.stab[j][k] = (P.off_astab >= 0 && k < D) ? prm[P.off_astab + j * D + k] : 0.0f;
    }
    for (int e = tid; e < WP; e += NT) {
        sm.b1[e] = e < Wd ? prm[P.off_l1b + e] : 0.0f;
        sm.b2[e] = e < Wd ? prm[P.off_l2b + e] : 0.0f;
    }
    if (tid < 4) sm.b3[tid] = tid < 2 ? prm[P.off_hb + tid] : 0.0f;
    for (int e = tid; e < kMaxSlots * kFM * kRM; e += NT) {
        const int s = e / (kFM * kRM), r = e % (kFM * kRM), f = r / kRM, j = r % kRM;
        float v = 0.0f;
        if (s < P.n_slots) {
            const int rd = P.g[P.slot_gi[s]].rdim;
            if (f < F && j < rd) v = prm[P.off_ifw[s] + f * rd + j];
        }
        sm.Wf[s][f][j] = v;
    }
    for (int e = tid; e < kMaxSlots * kFM; e += NT) {
        const int s = e / kFM, f = e % kFM;
        sm.bf[s][f] = (s < P.n_slots && f < F) ? prm[P.off_ifb[s] + f] : 0.0f;
    }
    for (int e = tid; e < kMaxCtx; e += NT)  // context offset o -> window position
        sm.woff[e] = e < S ? (P.P + P.ctx_dy[e]) * WS + P.P + P.ctx_dx[e] : 0;
    for (int e = tid; e < K::NACC5; e += NT) sm.acc5[e] = 0.0;
    for (int e = tid; e < P.n_grids; e += NT) sm.geo[e] = P.g[e];
    if (tid == 0) {
        ctx_table_build(P, sm.ctxt);
        for (int b = 0; b < 2; ++b) {
            const unsigned sb = static_cast<unsigned>(__cvta_generic_to_shared(&sm.wbar[b]));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sb) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    // constant rows: zero padding of every activation array (written once);
    // windows zeroed so R rows past a grid's rdim are always finite
    for (int e = tid; e < K::ACT; e += NT) sm.act[e] = 0.0f;
    for (int e = tid; e < 2 * WIN; e += NT) (&sm.win[0][0])[e] = 0.0f;
    __syncthreads();

    float* const sC = sm.act + K::O_C;
    float* const sH1 = sm.act + K::O_H1;
    float* const sH2 = sm.act + K::O_H2;
    float* const sDH1 = sm.act + K::O_DH1;
    float* const sDH2 = sm.act + K::O_DH2;
    float* const sDR = sm.act + K::O_DR;
    float* const sDF = sm.act + K::O_DF;
    float* const sHP = sm.act + K::O_HP;
    // tile records run two ahead of the tile being computed (register
    // prefetch); the gather of tile t+grid is issued while tile t computes
    int4 cur = blockIdx.x < ntiles ? tiles[blockIdx.x] : make_int4(0, 0, 0, 0);
    int4 nxt = blockIdx.x + gridDim.x < ntiles ? tiles[blockIdx.x + gridDim.x] : make_int4(0, 0, 0, 0);
    int wb = 0;  // window buffer of the current tile
    if (tid == 0)  // ring slot of the first tile's record two ahead; later ones by cp.async
        sm.trec[0] = blockIdx.x + 2 * gridDim.x < ntiles ? tiles[blockIdx.x + 2 * gridDim.x] : make_int4(0, 0, 0, 0);
    if (blockIdx.x < ntiles) issue_gather(P, sm.geo, cur, sm.win[0], &sm.wbar[0], tid);
    int kt = 0;  // tile count of this CTA (ring index)

    // persistent weight-gradient accumulators of this thread's units
    double uacc[K::MAXU][16];  // fp64 across tiles: large images sum millions of terms
#pragma unroll
    for (int m = 0; m < K::MAXU; ++m)
#pragma unroll
        for (int e = 0; e < 16; ++e) uacc[m][e] = 0.0;
    double bits_thr = 0.0;
    const float upstream = P.rate_upstream;

    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int4 tile = cur;
        const GridGeom& g = sm.geo[tile.x];
        const int64_t count = int64_t(g.rows) * g.cols;
        const int slot = g.ifce_slot;
        const int len = tile.w;
        const int64_t li = int64_t(tile.y) + lt;
        const bool valid = lt < len;
        // rate terms only for owned rows (row bands; whole images own all rows)
        const bool own = valid && tile.z >= g.own_lo && tile.z < g.own_hi;

        // ---- P0: prefetch the next tile (its buffers' last readers finished
        // at the previous tile's closing barrier), land the current one ----
        if (tid == 0) {  // the record three ahead joins this group (read two tiles from now)
            const int64_t t3 = int64_t(t) + 3 * int64_t(gridDim.x);
            const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(&sm.trec[(kt + 1) & 3]));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa),
                         "l"(t3 < ntiles ? tiles + t3 : tiles), "r"(t3 < ntiles ? 16 : 0)
                         : "memory");
        }
        if (t + int(gridDim.x) < ntiles)
            issue_gather(P, sm.geo, nxt, sm.win[wb ^ 1], &sm.wbar[wb ^ 1], tid);
        else
            cp_async_commit();
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        mbar_wait_parity(&sm.wbar[wb], unsigned(kt >> 1) & 1u);  // this tile's context rows (TMA)
        __syncthreads();
        const int4 nxt2 = sm.trec[kt & 3];
        ++kt;

        // ---- P1: context rows from the window, IFCE forward (two threads
        // per latent), constant rows ----
        float* const sR = sm.win[wb] + WC;  // this tile's R rows
        {
            const float* win = sm.win[wb];
            for (int o = half; o < S; o += 2)  // C[o] = ŷ(r + dy_o, c + dx_o)
                sC[o * LT + lt] = valid ? win[sm.woff[o] + lt] : 0.0f;
            constexpr int FH = kFM / 2;
            if (slot >= 0) {
                float rv[kRM];
#pragma unroll
                for (int j = 0; j < kRM; ++j) rv[j] = sR[j * LT + lt];
#pragma unroll
                for (int ff = 0; ff < FH; ++ff) {  // gemm_xwt_fast order: bias, then j
                    const int f = half * FH + ff;
                    if (f < F) {
                        float a = sm.bf[slot][f];
#pragma unroll
                        for (int j = 0; j < kRM; ++j) a = fmaf(rv[j], sm.Wf[slot][f][j], a);
                        sC[(S + f) * LT + lt] = valid ? a : 0.0f;
                    }
                }
                if (half) sR[kRM * LT + lt] = valid ? 1.0f : 0.0f;
            } else {
#pragma unroll
                for (int ff = 0; ff < FH; ++ff) {
                    const int f = half * FH + ff;
                    if (f < F) sC[(S + f) * LT + lt] = 0.0f;
                }
            }
            if (half == 0) {
                sC[(DP + 1) * LT + lt] = valid ? win[P.P * WS + P.P + lt] : 0.0f;  // own value
                sC[DP * LT + lt] = valid ? 1.0f : 0.0f;
                sH1[WP * LT + lt] = valid ? 1.0f : 0.0f;
            } else {
                sH2[WP * LT + lt] = valid ? 1.0f : 0.0f;
            }
        }
        __syncthreads();

        // ---- P2: H1 = relu(b1 + W1·C) ----
        {
            float2 acc[K::NW];
#pragma unroll
            for (int n = 0; n < K::NW; ++n) {
                const float b = sm.b1[grp * K::NW + n];
                acc[n] = make_float2(b, b);
            }
            tile_gemm<K::NW, DP>(sC, sm.W1T, pr, grp, acc);
#pragma unroll
            for (int n = 0; n < K::NW; ++n) {
                const float2 h = make_float2(acc[n].x > 0.0f ? acc[n].x : 0.0f, acc[n].y > 0.0f ? acc[n].y : 0.0f);
                *reinterpret_cast<float2*>(sH1 + (grp * K::NW + n) * LT + 2 * pr) = h;
            }
        }
        __syncthreads();
        // ---- P3: H2 = relu(b2 + W2·H1) ----
        {
            float2 acc[K::NW];
#pragma unroll
            for (int n = 0; n < K::NW; ++n) {
                const float b = sm.b2[grp * K::NW + n];
                acc[n] = make_float2(b, b);
            }
            tile_gemm<K::NW, WP>(sH1, sm.W2T, pr, grp, acc);
            // the two head outputs, this group's share: W3 over its H2
            // outputs plus the stabiliser over its quarter of the C rows
            float2 p0 = make_float2(0.0f, 0.0f), p1 = make_float2(0.0f, 0.0f);
#pragma unroll
            for (int n = 0; n < K::NW; ++n) {
                const int a = grp * K::NW + n;
                const float2 h = make_float2(acc[n].x > 0.0f ? acc[n].x : 0.0f, acc[n].y > 0.0f ? acc[n].y : 0.0f);
                *reinterpret_cast<float2*>(sH2 + a * LT + 2 * pr) = h;
                p0 = ffma2(h, sm.W3[0][a], p0);
                p1 = ffma2(h, sm.W3[1][a], p1);
            }
#pragma unroll
            for (int n = 0; n < K::ND; ++n) {
                const int k = grp * K::ND + n;
                const float2 c = *reinterpret_cast<const float2*>(sC + k * LT + 2 * pr);
                p0 = ffma2(c, sm.stab[0][k], p0);
                p1 = ffma2(c, sm.stab[1][k], p1);
            }
            *reinterpret_cast<float2*>(sHP + (2 * grp) * LT + 2 * pr) = p0;
            *reinterpret_cast<float2*>(sHP + (2 * grp + 1) * LT + 2 * pr) = p1;
        }
        __syncthreads();
        // ---- P4b: Laplace rate + its backward, dH2 (threads [0,128)) ----
        if (half == 0) {
            const float v = sC[(DP + 1) * LT + lt];
            // raw = b3 + sum of the four group partials (fixed order)
            const float mu = sm.b3[0] + (((sHP[lt] + sHP[2 * LT + lt]) + sHP[4 * LT + lt]) + sHP[6 * LT + lt]);
            const float sr = sm.b3[1] + (((sHP[LT + lt] + sHP[3 * LT + lt]) + sHP[5 * LT + lt]) + sHP[7 * LT + lt]);
            const float sg = sigma_from_raw(sr);
            const float bsc = sg * kInvSqrt2F;
            const float u = fabsf(v - mu);
            const float e1 = cc_exp(-(u + 0.5f) / bsc);
            const float e2 = cc_exp(-fabsf(u - 0.5f) / bsc);
            const float p = u >= 0.5f ? 0.5f * (e2 - e1) : 1.0f - 0.5f * (e1 + e2);
            if (own) bits_thr += double(-(cc_log(std_max(p, kProbFloorF)) * kLog2EF));
            if (MODE != kArmForward) {
                float dmu = 0.0f, dsr = 0.0f, gv = 0.0f;
                if (own && p > kProbFloorF) {
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
                sDR[0 * LT + lt] = dmu;
                sDR[1 * LT + lt] = dsr;
#pragma unroll
                for (int a = 0; a < WP; ++a) {  // dH2 = (W3ᵀ draw) ⊙ relu'(H2)
                    float d = fmaf(dmu, sm.W3[0][a], 0.0f);
                    d = fmaf(dsr, sm.W3[1][a], d);
                    sDH2[a * LT + lt] = sH2[a * LT + lt] > 0.0f ? d : 0.0f;
                }
            }
        }
        __syncthreads();
        if (MODE == kArmForward) {
            wb ^= 1;
            cur = nxt;
            nxt = nxt2;
            continue;
        }
        // ---- P6: dH1 = (W2ᵀ·dH2) ⊙ relu'(H1) ----
        {
            float2 acc[K::NW];
#pragma unroll
            for (int n = 0; n < K::NW; ++n) acc[n] = make_float2(0.0f, 0.0f);
            tile_gemm<K::NW, WP>(sDH2, sm.W2, pr, grp, acc);
#pragma unroll
            for (int n = 0; n < K::NW; ++n) {
                const int b = grp * K::NW + n;
                const float2 h = *reinterpret_cast<const float2*>(sH1 + b * LT + 2 * pr);
                const float2 d = make_float2(h.x > 0.0f ? acc[n].x : 0.0f, h.y > 0.0f ? acc[n].y : 0.0f);
                *reinterpret_cast<float2*>(sDH1 + b * LT + 2 * pr) = d;
            }
        }
        __syncthreads();
        // ---- P7: dC = W1ᵀ·dH1 + stabᵀ·draw -> dF now, context rows after P8 ----
        float2 dcacc[K::ND];
        {
            float2 (&acc)[K::ND] = dcacc;
#pragma unroll
            for (int n = 0; n < K::ND; ++n) acc[n] = make_float2(0.0f, 0.0f);
            tile_gemm<K::ND, WP>(sDH1, sm.W1, pr, grp, acc);
            tile_gemm<K::ND, 2>(sDR, sm.ST, pr, grp, acc);
            const int64_t l0 = int64_t(tile.y) + 2 * pr;
            const bool v0 = 2 * pr < len, v1 = 2 * pr + 1 < len;
#pragma unroll
            for (int n = 0; n < K::ND; ++n) {
                const int k = grp * K::ND + n;
                if (k < S) {
                    if (MODE == kArmProxy && !P.ctx_part) {  // S planes (else row partials after P8)
                        float* dcp = P.dctx + g.dctx_off + int64_t(k) * count + l0;
                        if (v1 && (reinterpret_cast<uintptr_t>(dcp) & 7) == 0) {
                            *reinterpret_cast<float2*>(dcp) = acc[n];
                        } else {
                            if (v0) dcp[0] = acc[n].x;
                            if (v1) dcp[1] = acc[n].y;
                        }
                    }
                } else if (k < S + F && slot >= 0) {
                    const float2 dv = make_float2(v0 ? acc[n].x : 0.0f, v1 ? acc[n].y : 0.0f);
                    *reinterpret_cast<float2*>(sDF + (k - S) * LT + 2 * pr) = dv;
                    if (MODE == kArmProxy || (MODE == kArmHard && P.ifce_sep)) {  // k_ifce_dw reads dF
                        float* dfp = P.dfeat + g.dfeat_off + int64_t(k - S) * count + l0;
                        if (v1 && (reinterpret_cast<uintptr_t>(dfp) & 7) == 0) {
                            *reinterpret_cast<float2*>(dfp) = dv;
                        } else {
                            if (v0) dfp[0] = dv.x;
                            if (v1) dfp[1] = dv.y;
                        }
                    }
                }
            }
        }
        __syncthreads();
        // ---- P8: weight gradients (register micro-tiles, balanced units) ----
#pragma unroll
        for (int m = 0; m < K::MAXU; ++m) {
            const int u = tid + m * NT;
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
            for (int e = tid; e < K::J5 * 16; e += NT) {
                const int j = e / 16, q = e % 16;
                const float v = (sm.stage5[3 * j][q] + sm.stage5[3 * j + 1][q]) + sm.stage5[3 * j + 2][q];
                const int a = 4 * (j / nq) + q / 4, b = 4 * (j % nq) + q % 4;
                if (b <= kRM) sm.acc5[(slot * kFM + a) * (kRM + 1) + b] += double(v);
            }
            // stage5 is rewritten only after the next tile's five barriers
        }
        if (MODE == kArmProxy && P.ctx_part) {
            // ---- P9: the context gradient as row partials (cc_ctx.cuh); the
            // H1 / H2 rows are dead here and hold dC[o][latent] ----
            float* const sDC = sm.act + K::O_H1;
#pragma unroll
            for (int n = 0; n < K::ND; ++n) {
                const int k = grp * K::ND + n;
                if (k < S) *reinterpret_cast<float2*>(sDC + k * LT + 2 * pr) = dcacc[n];
            }
            __syncthreads();
            ctx_store_partials(P, g, tile, sDC, LT, sm.ctxt, tid, NT);
            // (the next tile's P0 barrier orders these reads before P1's writes)
        }
        wb ^= 1;
        cur = nxt;
        nxt = nxt2;
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");

    // ---------------- per-CTA results ----------------
    const double tb = block_sum(bits_thr, sm.red);  // (its barriers also close the last tile)
    if (tid == 0) P.bits_part[blockIdx.x] = tb;
    if (MODE == kArmForward) return;
    const PartialRegion& R = P.region[P.reg_arm];
    const PartialRow row(P, R, blockIdx.x);
    // stage the register units in (now dead) activation memory, then every
    // parameter of the region is written exactly once: the three latent
    // thirds of its job summed in order
    static_assert(K::NU * 16 * 2 <= K::ACT, "fp64 staging fits in the activation buffers");
    double* stage = reinterpret_cast<double*>(sm.act);
#pragma unroll
    for (int m = 0; m < K::MAXU; ++m) {
        const int u = tid + m * NT;
        if (u < K::NU)
#pragma unroll
            for (int e = 0; e < 16; ++e) stage[u * 16 + e] = uacc[m][e];
    }
    __syncthreads();
    for (int x = tid; x < K::NJ * 16; x += NT) {
        const int j = x / 16, q = x % 16;
        const double v = (stage[(3 * j) * 16 + q] + stage[(3 * j + 1) * 16 + q]) + stage[(3 * j + 2) * 16 + q];
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
    for (int s = 0; s < (P.ifce_sep ? 0 : P.n_slots); ++s) {  // ifce_sep: k_ifce_dw's own region
        const int rd = P.g[P.slot_gi[s]].rdim;
        for (int e = tid; e < F * (rd + 1); e += NT) {
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
    k_arm2<DP, WP, MODE><<<dim3(L.arm_blocks, 1, L.batch), NT, arm2_smem<DP, WP>(), L.stream>>>(L.plan, L.arm_tiles,
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

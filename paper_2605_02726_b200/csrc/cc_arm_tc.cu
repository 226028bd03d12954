// cc_arm_tc.cu — the auto-regressive entropy model (ARM + IFCE, rate_pass
// entropy_model.hpp:180-336) with its four per-latent dense layers on the
// sm_100a tensor cores.
//
// Persistent CTAs of 256 threads over row-segment tiles of <= 128 latents: a
// latent is one TMEM lane, shared by two threads (warps w and w + 4 address the
// same lane quarter) that each own half of every layer's features; two CTAs
// per SM so that one CTA's tensor-core round trips and barriers overlap the
// other's CUDA-core work.
// Per tile:
//
//   gather C (causal context + IFCE features, fp32)          CUDA cores
//   H1 = relu(C W1^T + b1)                                    tcgen05, TMEM accumulator
//   H2 = relu(H1 W2^T + b2)                                   tcgen05
//   head mu / sigma_raw, Laplace rate and its backward, dH2   CUDA cores
//   dH1 = (dH2 W2) * relu'(H1)                                tcgen05
//   dC  = dH1 W1 + draw stab                                  tcgen05
//   weight gradients (register micro-tiles over the latents)  CUDA cores, overlapping
//                                                             the dH1 / dC MMAs
//
// The tensor-core layers run as 3xTF32: every operand x is split into
// hi = round_tf32(x) and lo = round_tf32(x - hi) (|x - hi - lo| <= 2^-24 |x|)
// and D = Alo*Bhi + Ahi*Blo + Ahi*Bhi with fp32 accumulation in TMEM
// (tools/micro/umma_probe3.cu: relative error 1.8e-7 vs fp64 on K = 24 dot
// products, sequential fp32 FMA 0.9e-7).  Biases ride along as a column of
// ones in A (B holds the bias in that column).
// The A operand of each layer lives in TMEM (lane = latent, one column per
// input feature, hi and lo): the thread that owns a latent writes its row
// with tcgen05.st after the previous layer's accumulator was read, so the
// activations never go through shared memory on their way to the tensor
// core.  B operands (weights hi/lo, canonical no-swizzle K-major layout of
// cc_umma.cuh) are staged once per CTA.  The feature-major fp32 rows that the
// weight-gradient micro-tiles read stay in shared memory (as cc_arm2.cu).
// Thread 0 issues the MMAs; completion is an mbarrier arrive by tcgen05.commit.
#include <cuda_runtime.h>

#include <cstdint>

#pragma nv_diag_suppress 128  // forward-only instantiations skip the backward phases

#include "cc_kernels.h"
#include "cc_math.cuh"
#include "cc_reduce.cuh"
#include "cc_ctx.cuh"
#include "cc_tile.cuh"
#include "cc_umma.cuh"

namespace ccb {

namespace {

constexpr int T = kArmTile;   // latents per tile (128)
constexpr int NT = 2 * T;     // two threads per latent: half h owns half of every layer's features
constexpr int LT = T + 4;     // feature-major row length (floats)
constexpr int kRM = 11;       // max IFCE source grids: hyper (L - 4) + L - 1 - k <= 11 for L <= 8
constexpr int kRR = kRM + 1;  // R rows + the ones row (3 row blocks of 4)
constexpr int kFM = 8;        // max IFCE width
constexpr int kMaxPad = 4;    // context window halo (yhat_pad border P)
constexpr int WS = T + 2 * kMaxPad;
constexpr int WC = (kMaxPad + 1) * WS;
constexpr int WIN = WC + kRR * LT;

constexpr int r8(int x) { return (x + 7) / 8 * 8; }
constexpr int cmax(int a, int b) { return a > b ? a : b; }
constexpr uint32_t pow2cols(int x) { return x <= 32 ? 32u : x <= 64 ? 64u : x <= 128 ? 128u : 256u; }

template <int DP, int WP>
struct TC {
    static_assert(T == 128, "one TMEM lane per latent");
    static constexpr int KD = r8(DP + 1);        // A of L1: C | 1 (ones at DP)
    static constexpr int KW = r8(WP + 1);        // A of L2: H1 | 1 (ones at WP); dH2 for dH1
    static constexpr int KC = KW + 8;            // A of dC: dH1 | draw
    static constexpr int KT = cmax(KD, KC);      // TMEM columns of one A copy
    static constexpr int NW = r8(WP);            // N of L1 / L2 / dH1
    static constexpr int ND = r8(DP);            // N of dC
    static_assert(NW <= 32 && ND <= 32, "one 32-column TMEM load per layer");
    // TMEM columns: the layer accumulator, then A hi, then A lo
    static constexpr uint32_t TM_ACC = 0, TM_AH = 32, TM_AL = 32 + KT;
    static constexpr uint32_t TM_COLS = pow2cols(32 + 2 * KT);
    // feature-major fp32 rows (weight gradients, Laplace), as cc_arm2.cu
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
    static constexpr int ACT = O_DF + RF * LT;
    static constexpr int O_HP = O_DH1;  // head partials [mu | sigma_raw]: P3 -> P4, before dH1 exists
    static_assert(2 * RH >= DP, "dC rows (S <= D <= DP) fit in the H1 / H2 rows");
    // weight-gradient jobs (4x4 micro-tiles) and units (job x latent third)
    static constexpr int J1 = (WP / 4) * (DP / 4 + 1);   // dH1 x [C|1]   (after the dH1 MMA)
    static constexpr int J2 = (WP / 4) * (WP / 4 + 1);   // dH2 x [H1|1]  (beside the dH1 MMA)
    static constexpr int J3 = WP / 4 + 1;                // draw x [H2|1]
    static constexpr int J4 = DP / 4;                    // draw x C (stabilizer)
    static constexpr int NJ = J1 + J2 + J3 + J4;
    static constexpr int NU = 3 * NJ;
    static constexpr int J5 = (kFM / 4) * (kRR / 4);     // dF x [R|1] (per tile, 8 latent slices each)
    static constexpr int MAXU = (NU + NT - 1) / NT;
    static constexpr int NACC5 = kMaxSlots * kFM * kRR;
    static_assert(NU * 16 * 2 <= ACT, "fp64 epilogue staging fits in the activation rows");
    // two CTAs per SM (128 registers) unless the weight-gradient units need a
    // second register-accumulated set (wide ARM inputs, e.g. the cfg4 decoder)
    static constexpr int MINB = MAXU > 1 ? 1 : 2;
};

template <int DP, int WP>
struct TcSmem {
    using K = TC<DP, WP>;
    alignas(16) float b1[2][K::NW * K::KD];      // L1: [a][k]  W1, b1 at k = DP
    alignas(16) float b2[2][K::NW * K::KW];      // L2: [b][a]  W2, b2 at a = WP
    alignas(16) float b3[2][K::NW * K::KW];      // dH1: [a][b] = W2[b][a]
    alignas(16) float b4[2][K::ND * K::KC];      // dC: [k][a] = W1[a][k]; [k][KW + j] = stab[j][k]
    alignas(16) float act[K::ACT];
    alignas(16) float win[2][WIN];
    alignas(16) float W3[2][WP];
    alignas(16) float stab[2][DP];
    alignas(16) float hb[4];
    alignas(16) float Wf[kMaxSlots][kFM][kRR];  // rows padded to 12 (float4 loads); column 11 zero
    alignas(16) float bf[kMaxSlots][kFM];
    int woff[kMaxCtx];
    double acc5[K::NACC5];
    alignas(16) float st5[K::J5 * 8][16];  // IFCE dW slice partials of one tile
    GridGeom geo[kMaxGrids];
    double red[NT / 32];
    alignas(16) int4 trec[4];
    CtxTable ctxt;  // context offsets by target row (cc_ctx.cuh)
    uint64_t mbar;
    uint32_t tmem;
};

__device__ __forceinline__ void third_range(int s, int& i0, int& i1) {
    i0 = s * 44;
    i1 = s == 2 ? T : i0 + 44;
}

__device__ __forceinline__ void cp_async4_zfill(float* smem, const float* gmem, bool full) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem), "r"(full ? 4 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

// the (P+1)-row causal window of a row-segment tile and, on IFCE grids, one
// row of every source grid (see cc_arm2.cu issue_gather)
__device__ __forceinline__ void issue_gather(const Plan& P, const GridGeom* geo, int4 tile, float* win,
                                             int tid) {
    const GridGeom& g = geo[tile.x];
    const int r = tile.z, len = tile.w, c0 = tile.y - r * g.cols;
    const int pad = P.P;
    const float* base = P.yhat_pad + g.pad_base + int64_t(r - pad) * g.stride + (c0 - pad);
    const int lenw = len + 2 * pad;
    for (int e = tid; e < (pad + 1) * WS; e += NT) {
        const int i = e / WS, x = e - i * WS;
        const bool full = x < lenw;
        cp_async4_zfill(win + e, full ? base + int64_t(i) * g.stride + x : base, full);
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

template <int DP, int WP>
struct ChunkStore {  // hi at TM_AH + c, lo at TM_AL + c
    __device__ __forceinline__ static void put(uint32_t tl, int c, float a, float b, float cc, float d) {
        using K = TC<DP, WP>;
        float h[4], l[4];
        umma::split_rn_fast(a, h[0], l[0]);
        umma::split_rn_fast(b, h[1], l[1]);
        umma::split_rn_fast(cc, h[2], l[2]);
        umma::split_rn_fast(d, h[3], l[3]);
        umma::st4(tl + K::TM_AH + uint32_t(c), h[0], h[1], h[2], h[3]);
        umma::st4(tl + K::TM_AL + uint32_t(c), l[0], l[1], l[2], l[3]);
    }
};

// v[h * OFF + i] with i a compile-time index: a select of two registers
// instead of a dynamically indexed (local-memory) array
template <int OFF>
__device__ __forceinline__ float hsel(const float (&v)[32], int h, int i) {
    return h ? v[OFF + i] : v[i];
}

// this thread's A row is complete in TMEM: make it visible to the MMA issuer
__device__ __forceinline__ void a_ready() {
    umma::wait_st();
    umma::fence_before_sync();
    __syncthreads();
}

// D = A (TMEM columns a_hi / a_lo, k-steps of 8) x B^T (smem, K-major) as 3xTF32
__device__ __forceinline__ void mma3_ts(uint32_t d, uint32_t a_hi, uint32_t a_lo, uint64_t bh,
                                        uint64_t bl, int nks, uint32_t idesc) {
    for (int ks = 0; ks < nks; ++ks) {
        const uint32_t ka = 8u * uint32_t(ks);
        const uint64_t kb = uint64_t(16 * ks);  // 256 B (two core columns) in descriptor units
        umma::mma_tf32_ts(d, a_lo + ka, bh + kb, idesc, ks > 0 ? 1u : 0u);
        umma::mma_tf32_ts(d, a_hi + ka, bl + kb, idesc, 1u);
        umma::mma_tf32_ts(d, a_hi + ka, bh + kb, idesc, 1u);
    }
}

template <int DP, int WP, int MODE>
__global__ void __launch_bounds__(NT, TC<DP, WP>::MINB) k_arm_tc(const Plan* __restrict__ pp,
                                                  const int4* __restrict__ tiles, int ntiles) {
    using K = TC<DP, WP>;
    using CS = ChunkStore<DP, WP>;
    const Plan& P = pp[blockIdx.z];  // batched launches: one plan per image
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TcSmem<DP, WP>& sm = *reinterpret_cast<TcSmem<DP, WP>*>(smem_raw);
    const int tid = threadIdx.x;
    const int half = tid >> 7, lt = tid & (T - 1);
    const int D = P.D, Wd = P.Wd, S = P.S, F = P.F;
    const float* prm = P.params;
    const bool has_stab = P.off_astab >= 0;

    if ((tid >> 5) == 0) umma::tmem_alloc(&sm.tmem, K::TM_COLS);
    if (tid == 0) umma::mbar_init(&sm.mbar, 1);

    // ---------------- weights -> shared memory ----------------
    for (int e = tid; e < K::NW * K::KD; e += NT) {  // L1: B1[a][k]
        const int a = e / K::KD, k = e % K::KD;
        float v = 0.0f;
        if (a < Wd) v = k < D ? prm[P.off_l1w + a * D + k] : (k == DP ? prm[P.off_l1b + a] : 0.0f);
        const uint32_t o = umma::tile_off(a, k, K::KD / 4) / 4;
        umma::split_rn(v, sm.b1[0][o], sm.b1[1][o]);
    }
    for (int e = tid; e < K::NW * K::KW; e += NT) {  // L2: B2[b][a]; dH1: B3[a][b] = W2[b][a]
        const int n = e / K::KW, k = e % K::KW;
        float v2 = 0.0f, v3 = 0.0f;
        if (n < Wd) {
            v2 = k < Wd ? prm[P.off_l2w + n * Wd + k] : (k == WP ? prm[P.off_l2b + n] : 0.0f);
            v3 = k < Wd ? prm[P.off_l2w + k * Wd + n] : 0.0f;
        }
        const uint32_t o = umma::tile_off(n, k, K::KW / 4) / 4;
        umma::split_rn(v2, sm.b2[0][o], sm.b2[1][o]);
        umma::split_rn(v3, sm.b3[0][o], sm.b3[1][o]);
    }
    for (int e = tid; e < K::ND * K::KC; e += NT) {  // dC: B4[k][a] = W1[a][k], B4[k][KW + j] = stab[j][k]
        const int k = e / K::KC, a = e % K::KC;
        float v = 0.0f;
        if (k < D) {
            if (a < Wd) v = prm[P.off_l1w + a * D + k];
            else if (a >= K::KW && a < K::KW + 2 && has_stab) v = prm[P.off_astab + (a - K::KW) * D + k];
        }
        const uint32_t o = umma::tile_off(k, a, K::KC / 4) / 4;
        umma::split_rn(v, sm.b4[0][o], sm.b4[1][o]);
    }
    for (int e = tid; e < 2 * WP; e += NT) {
        const int j = e / WP, a = e % WP;
        sm.W3[j][a] = a < Wd ? prm[P.off_hw + j * Wd + a] : 0.0f;
    }
    for (int e = tid; e < 2 * DP; e += NT) {
        const int j = e / DP, k = e % DP;
        sm.stab[j][k] = (has_stab && k < D) ? prm[P.off_astab + j * D + k] : 0.0f;
    }
    if (tid < 4) sm.hb[tid] = tid < 2 ? prm[P.off_hb + tid] : 0.0f;
    for (int e = tid; e < kMaxSlots * kFM * kRR; e += NT) {
        const int s = e / (kFM * kRR), r = e % (kFM * kRR), f = r / kRR, j = r % kRR;
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
    for (int e = tid; e < kMaxCtx; e += NT)
        sm.woff[e] = e < S ? (P.P + P.ctx_dy[e]) * WS + P.P + P.ctx_dx[e] : 0;
    for (int e = tid; e < K::NACC5; e += NT) sm.acc5[e] = 0.0;
    for (int e = tid; e < P.n_grids; e += NT) sm.geo[e] = P.g[e];
    if (tid == 0) ctx_table_build(P, sm.ctxt);
    for (int e = tid; e < K::ACT; e += NT) sm.act[e] = 0.0f;
    for (int e = tid; e < 2 * WIN; e += NT) (&sm.win[0][0])[e] = 0.0f;
    umma::fence_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tm0 = sm.tmem;
    const uint32_t tl = tm0 + (uint32_t(tid & 96) << 16);  // this warp's lane quarter (warps w, w + 4 share it)
    // B descriptors (constant for the whole launch)
    const uint64_t d_b1h = umma::desc(umma::smem_u32(sm.b1[0]), 128, (K::KD / 4) * 128);
    const uint64_t d_b1l = umma::desc(umma::smem_u32(sm.b1[1]), 128, (K::KD / 4) * 128);
    const uint64_t d_b2h = umma::desc(umma::smem_u32(sm.b2[0]), 128, (K::KW / 4) * 128);
    const uint64_t d_b2l = umma::desc(umma::smem_u32(sm.b2[1]), 128, (K::KW / 4) * 128);
    const uint64_t d_b3h = umma::desc(umma::smem_u32(sm.b3[0]), 128, (K::KW / 4) * 128);
    const uint64_t d_b3l = umma::desc(umma::smem_u32(sm.b3[1]), 128, (K::KW / 4) * 128);
    const uint64_t d_b4h = umma::desc(umma::smem_u32(sm.b4[0]), 128, (K::KC / 4) * 128);
    const uint64_t d_b4l = umma::desc(umma::smem_u32(sm.b4[1]), 128, (K::KC / 4) * 128);
    constexpr uint32_t ID_W = umma::idesc_tf32(128, K::NW, false, false);
    constexpr uint32_t ID_D = umma::idesc_tf32(128, K::ND, false, false);
    const uint32_t acc = tm0 + K::TM_ACC, a_hi = tm0 + K::TM_AH, a_lo = tm0 + K::TM_AL;

    float* const sC = sm.act + K::O_C;
    float* const sH1 = sm.act + K::O_H1;
    float* const sH2 = sm.act + K::O_H2;
    float* const sDH1 = sm.act + K::O_DH1;
    float* const sDH2 = sm.act + K::O_DH2;
    float* const sDR = sm.act + K::O_DR;
    float* const sDF = sm.act + K::O_DF;
    float* const sHP = sm.act + K::O_HP;
    uint32_t phase = 0;

    int4 cur = blockIdx.x < ntiles ? tiles[blockIdx.x] : make_int4(0, 0, 0, 0);
    int4 nxt = blockIdx.x + gridDim.x < ntiles ? tiles[blockIdx.x + gridDim.x] : make_int4(0, 0, 0, 0);
    int wb = 0;
    if (tid == 0)
        sm.trec[0] = blockIdx.x + 2 * gridDim.x < ntiles ? tiles[blockIdx.x + 2 * gridDim.x] : make_int4(0, 0, 0, 0);
    if (blockIdx.x < ntiles) issue_gather(P, sm.geo, cur, sm.win[0], tid);
    int kt = 0;

    double uacc[K::MAXU][16];
#pragma unroll
    for (int m = 0; m < K::MAXU; ++m)
#pragma unroll
        for (int e = 0; e < 16; ++e) uacc[m][e] = 0.0;
    double bits_thr = 0.0;
    const float upstream = P.rate_upstream;

    // this thread's weight-gradient units of one kind (J1: after the dH1 MMA;
    // the others beside it); each unit a 4x4 register micro-tile over a third
    // of the tile's latents
    auto dw_units = [&](bool j1_kind) {
#pragma unroll
        for (int m = 0; m < K::MAXU; ++m) {
            const int u = tid + m * NT;
            if (u < K::NU && ((u / 3 < K::J1) == j1_kind)) {
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
                dw_tile4x4<LT>(A, B, i0, i1, uacc[m]);
            }
        }
    };

    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int4 tile = cur;
        const GridGeom& g = sm.geo[tile.x];
        const int64_t count = int64_t(g.rows) * g.cols;
        const int slot = g.ifce_slot;
        const int len = tile.w;
        const int64_t li = int64_t(tile.y) + lt;
        const bool valid = lt < len;
        const bool own = valid && tile.z >= g.own_lo && tile.z < g.own_hi;

        // ---- P0: prefetch the next tile, land the current one ----
        if (tid == 0) {
            const int64_t t3 = int64_t(t) + 3 * int64_t(gridDim.x);
            const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(&sm.trec[(kt + 1) & 3]));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa),
                         "l"(t3 < ntiles ? tiles + t3 : tiles), "r"(t3 < ntiles ? 16 : 0)
                         : "memory");
        }
        if (t + int(gridDim.x) < ntiles)
            issue_gather(P, sm.geo, nxt, sm.win[wb ^ 1], tid);
        else
            cp_async_commit();
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        __syncthreads();
        const int4 nxt2 = sm.trec[kt & 3];
        ++kt;

        // ---- P1: C = context + IFCE features (+ ones at DP): this half's
        // chunks -> feature-major rows + A ----
        float* const sR = sm.win[wb] + WC;
        float pc0 = 0.0f, pc1 = 0.0f;  // this half's share of the stabiliser term stab . C
        {
            const float* win = sm.win[wb];
            constexpr int CH = K::KD / 8;  // chunks per half
            float rv[kRM];
            const bool need_r = slot >= 0 && (half + 1) * 4 * CH > S;
            if (need_r) {
#pragma unroll
                for (int j = 0; j < kRM; ++j) rv[j] = sR[j * LT + lt];
            }
#pragma unroll
            for (int cc = 0; cc < CH; ++cc) {
                const int c = half * CH + cc;
                float v4[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int f = 4 * c + i;
                    float v = 0.0f;
                    if (f < S) {
                        v = valid ? win[sm.woff[f] + lt] : 0.0f;
                    } else if (f < D) {
                        if (need_r && valid) {
                            const float4* wf = reinterpret_cast<const float4*>(sm.Wf[slot][f - S]);
                            float a = sm.bf[slot][f - S];  // gemm_xwt_fast order: bias, then j
#pragma unroll
                            for (int q = 0; q < (kRM + 3) / 4; ++q) {
                                const float4 w4 = wf[q];
                                a = fmaf(rv[4 * q], w4.x, a);
                                if (4 * q + 1 < kRM) a = fmaf(rv[4 * q + 1], w4.y, a);
                                if (4 * q + 2 < kRM) a = fmaf(rv[4 * q + 2], w4.z, a);
                                if (4 * q + 3 < kRM) a = fmaf(rv[4 * q + 3], w4.w, a);
                            }
                            v = a;
                        }
                    } else if (f == DP) {
                        v = valid ? 1.0f : 0.0f;
                    }
                    v4[i] = v;
                    if (f < DP) {
                        pc0 = fmaf(v, sm.stab[0][f], pc0);
                        pc1 = fmaf(v, sm.stab[1][f], pc1);
                    }
                    if (f <= DP) sC[f * LT + lt] = v;
                }
                CS::put(tl, 4 * c, v4[0], v4[1], v4[2], v4[3]);
            }
            if (half == 0) {
                sC[(DP + 1) * LT + lt] = valid ? win[P.P * WS + P.P + lt] : 0.0f;  // own value
                sH1[WP * LT + lt] = valid ? 1.0f : 0.0f;
            } else {
                sH2[WP * LT + lt] = valid ? 1.0f : 0.0f;
                if (slot >= 0) sR[kRM * LT + lt] = valid ? 1.0f : 0.0f;
            }
        }
        a_ready();
        if (tid == 0) {
            umma::fence_after_sync();
            mma3_ts(acc, a_hi, a_lo, d_b1h, d_b1l, K::KD / 8, ID_W);
            umma::commit(&sm.mbar);
        }

        // ---- P2: H1 = relu(acc) -> rows + A (ones at WP), this half's chunks ----
        uint32_t m1 = 0;  // relu'(H1) of this half's features
        umma::mbar_wait(&sm.mbar, phase);
        phase ^= 1;
        umma::fence_after_sync();
        {
            float v[32];
            umma::ld32(tl + K::TM_ACC, v);
            umma::wait_ld();
            constexpr int CH = K::KW / 8;
#pragma unroll
            for (int cc = 0; cc < CH; ++cc) {
                const int c = half * CH + cc;
                float h4[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int a = 4 * c + i;
                    const float x = hsel<K::KW / 2>(v, half, 4 * cc + i);
                    float h = 0.0f;
                    if (a < WP) {
                        h = x > 0.0f ? x : 0.0f;
                        if (x > 0.0f) m1 |= 1u << (4 * cc + i);
                        sH1[a * LT + lt] = h;
                    } else if (a == WP) {
                        h = valid ? 1.0f : 0.0f;
                    }
                    h4[i] = h;
                }
                CS::put(tl, 4 * c, h4[0], h4[1], h4[2], h4[3]);
            }
        }
        a_ready();
        if (tid == 0) {
            umma::fence_after_sync();
            mma3_ts(acc, a_hi, a_lo, d_b2h, d_b2l, K::KW / 8, ID_W);
            umma::commit(&sm.mbar);
        }

        // ---- P3: H2 = relu(acc) -> rows; this half's head partials ----
        uint32_t m2 = 0;  // relu'(H2) of this half's features
        umma::mbar_wait(&sm.mbar, phase);
        phase ^= 1;
        umma::fence_after_sync();
        {
            float v[32];
            umma::ld32(tl + K::TM_ACC, v);
            umma::wait_ld();
            float p0 = pc0, p1 = pc1;
#pragma unroll
            for (int i = 0; i < K::KW / 2; ++i) {
                const int a = half * (K::KW / 2) + i;
                const float x = hsel<K::KW / 2>(v, half, i);
                if (a < WP) {
                    const float h = x > 0.0f ? x : 0.0f;
                    if (x > 0.0f) m2 |= 1u << i;
                    sH2[a * LT + lt] = h;
                    p0 = fmaf(h, sm.W3[0][a], p0);
                    p1 = fmaf(h, sm.W3[1][a], p1);
                }
            }
            sHP[(2 * half) * LT + lt] = p0;
            sHP[(2 * half + 1) * LT + lt] = p1;
        }
        umma::fence_before_sync();
        __syncthreads();

        // ---- P4: Laplace rate + its backward (both halves, identical
        // arithmetic), dH2 for this half's features ----
        float dmu = 0.0f, dsr = 0.0f;
        {
            const float vv = sC[(DP + 1) * LT + lt];
            const float mu = sm.hb[0] + (sHP[lt] + sHP[2 * LT + lt]);
            const float sr = sm.hb[1] + (sHP[LT + lt] + sHP[3 * LT + lt]);
            const float sg = sigma_from_raw(sr);
            const float bsc = sg * kInvSqrt2F;
            const float u = fabsf(vv - mu);
            const float e1 = cc_exp(-(u + 0.5f) / bsc);
            const float e2 = cc_exp(-fabsf(u - 0.5f) / bsc);
            const float p = u >= 0.5f ? 0.5f * (e2 - e1) : 1.0f - 0.5f * (e1 + e2);
            if (own && half == 0) bits_thr += double(-(cc_log(std_max(p, kProbFloorF)) * kLog2EF));
            if (MODE != kArmForward) {
                float gv = 0.0f;
                if (own && p > kProbFloorF) {
                    const float tt = vv - mu;
                    const float dbits_dp = -1.0f / (p * kLn2F);
                    const float dp_du = (e1 - e2) / (2.0f * bsc);
                    const float sgn = tt > 0.0f ? 1.0f : (tt < 0.0f ? -1.0f : 0.0f);
                    const float dp_db = -((u + 0.5f) * e1 - (u - 0.5f) * e2) / (2.0f * bsc * bsc);
                    const float up = upstream * dbits_dp;
                    dmu = -up * dp_du * sgn;
                    if (sg > kSigmaMinF && sg < kSigmaMaxF) dsr = up * dp_db * kInvSqrt2F * sg;
                    gv = up * dp_du * sgn;
                }
                if (half == 0) {
                    if (MODE == kArmProxy && valid) P.gown[g.lat_off + li] = gv;
                    sDR[0 * LT + lt] = dmu;
                    sDR[1 * LT + lt] = dsr;
                }
                constexpr int CH = K::KW / 8;
#pragma unroll
                for (int cc = 0; cc < CH; ++cc) {  // dH2 = (W3^T draw) * relu'(H2)
                    const int c = half * CH + cc;
                    float d4[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int a = 4 * c + i;
                        float d = 0.0f;
                        if (a < WP) {
                            d = fmaf(dmu, sm.W3[0][a], 0.0f);
                            d = fmaf(dsr, sm.W3[1][a], d);
                            d = (m2 >> (4 * cc + i)) & 1u ? d : 0.0f;
                            sDH2[a * LT + lt] = d;
                        }
                        d4[i] = d;
                    }
                    CS::put(tl, 4 * c, d4[0], d4[1], d4[2], d4[3]);
                }
            }
        }
        if (MODE == kArmForward) {
            __syncthreads();  // windows / head partials reused by the next tile
            wb ^= 1;
            cur = nxt;
            nxt = nxt2;
            continue;
        }
        a_ready();
        if (tid == 0) {
            umma::fence_after_sync();
            mma3_ts(acc, a_hi, a_lo, d_b3h, d_b3l, K::KW / 8, ID_W);
            umma::commit(&sm.mbar);
        }
        dw_units(false);  // dH2 x [H1|1], draw x [H2|1], draw x C beside the dH1 MMA

        // ---- P5: dH1 = acc * relu'(H1) -> rows + A; draw columns ----
        umma::mbar_wait(&sm.mbar, phase);
        phase ^= 1;
        umma::fence_after_sync();
        {
            float v[32];
            umma::ld32(tl + K::TM_ACC, v);
            umma::wait_ld();
            constexpr int CH = K::KW / 8;
#pragma unroll
            for (int cc = 0; cc < CH; ++cc) {
                const int c = half * CH + cc;
                float d4[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int b = 4 * c + i;
                    float d = 0.0f;
                    if (b < WP) {
                        d = (m1 >> (4 * cc + i)) & 1u ? hsel<K::KW / 2>(v, half, 4 * cc + i) : 0.0f;
                        sDH1[b * LT + lt] = d;
                    }
                    d4[i] = d;
                }
                CS::put(tl, 4 * c, d4[0], d4[1], d4[2], d4[3]);
            }
            // draw (dmu, dsr, 0, 0 | 0, 0, 0, 0) at columns KW .. KW+7
            if (half == 0) CS::put(tl, K::KW, dmu, dsr, 0.0f, 0.0f);
            else CS::put(tl, K::KW + 4, 0.0f, 0.0f, 0.0f, 0.0f);
        }
        umma::wait_st();
        umma::fence_before_sync();
        __syncthreads();  // A complete; dH1 rows complete
        if (tid == 0) {
            umma::fence_after_sync();
            mma3_ts(acc, a_hi, a_lo, d_b4h, d_b4l, K::KC / 8, ID_D);
            umma::commit(&sm.mbar);
        }
        dw_units(true);  // dH1 x [C|1] beside the dC MMA

        // ---- P6: dC -> dctx planes / dF ----
        umma::mbar_wait(&sm.mbar, phase);
        phase ^= 1;
        umma::fence_after_sync();
        {
            float v[32];
            umma::ld32(tl + K::TM_ACC, v);
            umma::wait_ld();
            const bool st = MODE == kArmProxy && valid;
            float* const sDC = sm.act + K::O_H1;  // H1 / H2 rows are dead: dC[o][latent]
#pragma unroll
            for (int i = 0; i < K::ND / 2; ++i) {
                const int k = half * (K::ND / 2) + i;
                const float x = hsel<K::ND / 2>(v, half, i);
                if (k < S) {
                    if (P.ctx_part) sDC[k * LT + lt] = x;                              // row partials below
                    else if (st) P.dctx[g.dctx_off + int64_t(k) * count + li] = x;  // S planes
                } else if (k < S + F && slot >= 0) {
                    const float dv = valid ? x : 0.0f;
                    sDF[(k - S) * LT + lt] = dv;
                    if (st) P.dfeat[g.dfeat_off + int64_t(k - S) * count + li] = dv;
                }
            }
        }
        umma::fence_before_sync();
        __syncthreads();
        // the context gradient as row partials (cc_ctx.cuh)
        if (MODE == kArmProxy && P.ctx_part) ctx_store_partials(P, g, tile, sm.act + K::O_H1, LT, sm.ctxt, tid, NT);
        // ---- P9: IFCE weight gradient dF x [R|1]: 6 4x4 jobs x 8 slices of
        // 16 latents (48 threads), slices summed in order, fp64 per slot ----
        if (slot >= 0) {
            constexpr int nq = kRR / 4;
            if (tid < K::J5 * 8) {
                const int j = tid >> 3, sl = tid & 7;
                float part[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) part[e] = 0.0f;
                dw_tile4x4<LT>(sDF + (4 * (j / nq)) * LT, sR + (4 * (j % nq)) * LT, 16 * sl, 16 * sl + 16, part);
#pragma unroll
                for (int e = 0; e < 16; ++e) sm.st5[tid][e] = part[e];
            }
            __syncthreads();
            if (tid < K::J5 * 16) {
                const int j = tid >> 4, q = tid & 15;
                float v = sm.st5[8 * j][q];
#pragma unroll
                for (int sl = 1; sl < 8; ++sl) v += sm.st5[8 * j + sl][q];
                const int a = 4 * (j / nq) + q / 4, b = 4 * (j % nq) + q % 4;
                sm.acc5[(slot * kFM + a) * kRR + b] += double(v);
            }
        }
        __syncthreads();  // windows / dF rows reused by the next tile
        wb ^= 1;
        cur = nxt;
        nxt = nxt2;
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");

    // ---------------- per-CTA results ----------------
    const double tb = block_sum(bits_thr, sm.red);
    if (tid == 0) P.bits_part[blockIdx.x] = tb;
    if (MODE != kArmForward) {
        const PartialRegion& R = P.region[P.reg_arm];
        const PartialRow row(P, R, blockIdx.x);
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
                if (a < 2 && b < D && has_stab) o = P.off_astab + a * D + b;
            }
            if (o >= 0) row[o - R.param_off] = v;
        }
        for (int s = 0; s < P.n_slots; ++s) {
            const int rd = P.g[P.slot_gi[s]].rdim;
            for (int e = tid; e < F * (rd + 1); e += NT) {
                const int f = e / (rd + 1), b = e % (rd + 1);
                const double v = sm.acc5[(s * kFM + f) * kRR + (b < rd ? b : kRM)];
                const int o = b < rd ? P.off_ifw[s] + f * rd + b : P.off_ifb[s] + f;
                row[o - R.param_off] = v;
            }
        }
    }
    umma::fence_before_sync();
    __syncthreads();
    if ((tid >> 5) == 0) umma::tmem_dealloc(tm0, K::TM_COLS);
}

template <int DP, int WP>
size_t tc_smem() {
    return sizeof(TcSmem<DP, WP>);
}

template <int DP, int WP, int MODE>
void launch_t(const LaunchCtx& L) {
    k_arm_tc<DP, WP, MODE><<<dim3(L.arm_blocks, 1, L.batch), NT, tc_smem<DP, WP>(), L.stream>>>(L.plan, L.arm_tiles,
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
    const int smem = int(tc_smem<DP, WP>());
    cudaFuncSetAttribute(k_arm_tc<DP, WP, kArmForward>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_arm_tc<DP, WP, kArmHard>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_arm_tc<DP, WP, kArmProxy>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

template <int DP, int WP>
int occ_t() {
    configure_t<DP, WP>();  // the >48 KB shared-memory opt-in the occupancy query needs
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_arm_tc<DP, WP, kArmProxy>, NT, tc_smem<DP, WP>());
    return b < 1 ? 1 : b;
}

}  // namespace

bool arm_tc_supported(int Dp, int Wp) {
    return (Dp == 8 && Wp == 8) || (Dp == 16 && Wp == 12) || (Dp == 20 && Wp == 20) ||
           (Dp == 28 && Wp == 28) || (Dp == 32 && Wp == 20);
}

// resident CTAs per SM of the proxy variant (registers and shared memory)
int arm_tc_blocks_per_sm(int Dp, int Wp) {
    if (Dp == 8 && Wp == 8) return occ_t<8, 8>();
    if (Dp == 16 && Wp == 12) return occ_t<16, 12>();
    if (Dp == 20 && Wp == 20) return occ_t<20, 20>();
    if (Dp == 28 && Wp == 28) return occ_t<28, 28>();
    return occ_t<32, 20>();
}

size_t arm_tc_smem_bytes(int Dp, int Wp) {
    if (Dp == 8 && Wp == 8) return tc_smem<8, 8>();
    if (Dp == 16 && Wp == 12) return tc_smem<16, 12>();
    if (Dp == 20 && Wp == 20) return tc_smem<20, 20>();
    if (Dp == 28 && Wp == 28) return tc_smem<28, 28>();
    return tc_smem<32, 20>();
}

void arm_tc_configure(int Dp, int Wp) {
    if (Dp == 8 && Wp == 8) configure_t<8, 8>();
    else if (Dp == 16 && Wp == 12) configure_t<16, 12>();
    else if (Dp == 20 && Wp == 20) configure_t<20, 20>();
    else if (Dp == 28 && Wp == 28) configure_t<28, 28>();
    else if (Dp == 32 && Wp == 20) configure_t<32, 20>();
}

void launch_arm_tc(const LaunchCtx& L, int mode) {
    const int Dp = L.host->Dp, Wp = L.host->Wp;
    if (Dp == 8 && Wp == 8) launch_mode<8, 8>(L, mode);
    else if (Dp == 16 && Wp == 12) launch_mode<16, 12>(L, mode);
    else if (Dp == 20 && Wp == 20) launch_mode<20, 20>(L, mode);
    else if (Dp == 28 && Wp == 28) launch_mode<28, 28>(L, mode);
    else launch_mode<32, 20>(L, mode);
}

}  // namespace ccb

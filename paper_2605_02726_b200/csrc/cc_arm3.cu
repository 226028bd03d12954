// cc_arm3.cu — the auto-regressive entropy model (ARM + IFCE, forward and
// backward; entropy_model.hpp:180-336) on the tensor cores.
//
// Same contract as cc_arm2.cu (tiles, window gather, outputs, partial rows);
// different execution shape:
//
//   * every dense contraction runs as mma.sync m16n8k8 TF32 with a 3-term
//     split (x = hi + lo, hi = rna-tf32(x); acc += lo*B_hi + hi*B_lo +
//     hi*B_hi), which carries ~22 mantissa bits per product: fp32-class
//     accuracy (the dropped lo*lo term is <= 2^-22 relative, the fp32
//     rounding of a single FFMA is 2^-24) at 3 HMMA per 1,024 MAC;
//   * a warp owns 16 latents (one m16 tile) of the CTA's 128-latent tile and
//     runs the whole per-latent chain in REGISTERS: C -> H1 -> H2 -> head ->
//     Laplace rate -> dH2 -> dH1 -> dC.  The accumulator fragment of one
//     layer is the A fragment of the next up to a fixed permutation of the K
//     index inside each 8-wide k-step (accumulator columns 2t, 2t+1 <-> A
//     columns t, t+4), which the pre-arranged weight fragments absorb, so no
//     activation goes back through shared memory between layers and the
//     chain has no CTA barrier;
//   * the two head outputs are quad-shuffle reductions of the H2 / C
//     fragments; the Laplace rate and its backward run on the lane pair that
//     holds a latent's row;
//   * weight gradients dW = sum over latents of dAct^T [Act|1] are mma tiles
//     with the LATENT axis as K: activations are staged feature-major
//     ([feature][latent], row stride 136 = 8 mod 32: the pair loads of the
//     fragments are conflict-free) and 24 units (6 m16 row blocks x 4
//     32-latent quarters) are spread over the 8 warps, 3 per warp.  The unit
//     accumulators live in registers across all tiles of the persistent CTA
//     (fp32 over <= 32 tiles = 1,024 latents, then fp64 flushes into the CTA's
//     partial rows); the four quarters are summed in fixed order at the end.
//     No atomics: every fp64 value has exactly one owner lane;
//   * per tile: one barrier after the gather lands, one before the weight-
//     gradient tiles (cc_arm2: seven).
//
// Opt-in (CCB_ARM_V3=1), not the default: at 512x768 it runs 278 us against
// cc_arm2's 265 us.  The TF32 splits (two integer ops + one FADD per
// operand element, B fragments of the weight-gradient tiles re-split per
// unit) and the fragment index arithmetic add more instructions than the
// FFMA2 tile GEMMs they remove (99 M vs 76 M warp instructions per launch;
// profiles/r01_arm3_*), and its different summation order flips more
// near-threshold ReLU / probability-floor branches than cc_arm2, whose
// per-output order is the reference's.
#include <cuda_runtime.h>

#include <cstdint>

#include "cc_kernels.h"
#include "cc_math.cuh"
#include "cc_reduce.cuh"

namespace ccb {

namespace {

constexpr int T = kArmTile;  // latents per tile (128)
constexpr int NT = 2 * T;    // 8 warps
constexpr int LT = T + 8;    // staging / window row stride (floats), 8 mod 32
constexpr int kRM = 12;      // max IFCE source grids
constexpr int kFM = 8;       // max IFCE width
constexpr int kMaxPad = 4;   // context window halo
constexpr int WROWS = kMaxPad + 1 + 16;  // (P+1) context rows + 16 R rows (12 sources, ones, zeros)
constexpr int kFlushTiles = 32;           // fp32 unit accumulators span <= 32 tiles (1,024 latents)
static_assert(T + 2 * kMaxPad <= LT, "context window row fits the row stride");

constexpr int r8(int x) { return (x + 7) / 8 * 8; }

template <int DP, int WP>
struct A3 {
    static_assert(T == 128, "thread mapping assumes 128 latents per tile");
    static constexpr int KD = r8(DP);      // L1 K / dC N
    static constexpr int KW = r8(WP);      // hidden width (N of L1, L2; K of the backward)
    static constexpr int KC = r8(DP + 2);  // staged C rows: C | ones (D) | own value (D+1) | 0
    static constexpr int KH = r8(WP + 1);  // staged H rows: H | ones (W) | 0
    static constexpr int KA = r8(WP + 2);  // staged dA1 rows: dH1 | dmu, dsr (W, W+1) | 0
    static constexpr int NS1 = KD / 8, NW8 = KW / 8, ND8 = KD / 8;
    static constexpr int MT1 = (KA + 15) / 16;  // m16 blocks of dA1
    static constexpr int MT2 = (KW + 15) / 16;  // m16 blocks of dA2 (= dH2)
    static constexpr int NMR = MT1 + MT2 + 2;   // + dW3 block + IFCE block
    static constexpr int NU = NMR * 4;          // units: row block x latent quarter
    static constexpr int NUPW = (NU + 7) / 8;   // units per warp
    static constexpr int NC8 = KC / 8, NH8 = KH / 8;
    static constexpr int NMAX = NC8 > NH8 ? (NC8 > 2 ? NC8 : 2) : (NH8 > 2 ? NH8 : 2);
    // staging rows (floats) inside the activation buffer
    static constexpr int O_C = 0;
    static constexpr int O_H1 = O_C + KC * LT;
    static constexpr int O_H2 = O_H1 + KH * LT;
    static constexpr int O_A1 = O_H2 + KH * LT;
    static constexpr int O_A2 = O_A1 + KA * LT;
    static constexpr int O_DF = O_A2 + KW * LT;
    static constexpr int ACT = O_DF + kFM * LT;
};

template <int DP, int WP>
struct alignas(16) A3Smem {
    using K = A3<DP, WP>;
    // weight fragments: per (k-step, n-tile, lane) {hi b0, hi b1, lo b0, lo b1}
    float4 fL1[K::NS1][K::NW8][32];  // B = W1ᵀ (standard K order)
    float4 fL2[K::NW8][K::NW8][32];  // B = W2ᵀ (permuted K)
    float4 fH1[K::NW8][K::NW8][32];  // B = W2  (dH1 = dH2·W2, permuted K)
    float4 fDC[K::NW8][K::ND8][32];  // B = W1  (dC = dH1·W1, permuted K)
    float W3[2][K::KW];
    float stab[2][K::KD];
    float b1[K::KW];
    float b2[K::KW];
    float b3[2];
    float Wf[kMaxSlots][kFM][kRM];
    float bf[kMaxSlots][kFM];
    int woff[kMaxCtx];
    GridGeom geo[kMaxGrids];
    double red[NT / 32];
    alignas(16) float act[K::ACT];
    alignas(16) float win[2][WROWS * LT];
};

// round to the 10-bit TF32 mantissa, ties away from zero (cvt.rna), on the
// integer pipe (finite inputs)
__device__ __forceinline__ uint32_t tf32_hi(float x) { return (__float_as_uint(x) + 0x1000u) & 0xffffe000u; }
// x -> (hi, lo) with hi = rna_tf32(x), lo = x - hi (the MMA reads lo's top 19 bits)
__device__ __forceinline__ void split4(const float (&x)[4], uint32_t (&hi)[4], uint32_t (&lo)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        hi[i] = tf32_hi(x[i]);
        lo[i] = __float_as_uint(x[i] - __uint_as_float(hi[i]));
    }
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// d += A·B at fp32-class accuracy; B given as a pre-split fragment
__device__ __forceinline__ void mma3(float (&d)[4], const uint32_t (&ahi)[4], const uint32_t (&alo)[4],
                                     const float4 b) {
    mma_tf32(d, alo, __float_as_uint(b.x), __float_as_uint(b.y));
    mma_tf32(d, ahi, __float_as_uint(b.z), __float_as_uint(b.w));
    mma_tf32(d, ahi, __float_as_uint(b.x), __float_as_uint(b.y));
}
__device__ __forceinline__ float4 split_pair(float b0, float b1) {
    const uint32_t h0 = tf32_hi(b0), h1 = tf32_hi(b1);
    return make_float4(__uint_as_float(h0), __uint_as_float(h1), b0 - __uint_as_float(h0),
                       b1 - __uint_as_float(h1));
}
// accumulator fragment -> A fragment of the next layer (K permutation
// t <-> 2t, t+4 <-> 2t+1 inside the k-step)
__device__ __forceinline__ void acc_as_a(const float (&c)[4], float (&a)[4]) {
    a[0] = c[0];
    a[1] = c[2];
    a[2] = c[1];
    a[3] = c[3];
}

__device__ __forceinline__ void cp_async4_zfill(float* smem, const float* gmem, bool full) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem), "r"(full ? 4 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

// Asynchronous gather of one row-segment tile into a window buffer: the P+1
// padded rows r-P .. r over columns c0-P .. c0+len-1+P (zero border
// included), and on IFCE grids the R rows [j][latent] = ŷ of coarser grid
// j < rdim at (r >> sh, c >> sh) (entropy_model.hpp:232-248).  All threads;
// always commits one cp.async group.
__device__ __forceinline__ void issue_gather(const Plan& P, const GridGeom* geo, int4 tile, float* win,
                                             int tid) {
    const GridGeom& g = geo[tile.x];
    const int r = tile.z, len = tile.w, c0 = tile.y - r * g.cols;
    const int pad = P.P;
    const float* base = P.yhat_pad + g.pad_base + int64_t(r - pad) * g.stride + (c0 - pad);
    const int lenw = len + 2 * pad;
    for (int e = tid; e < (pad + 1) * LT; e += NT) {
        const int i = e / LT, x = e - i * LT;
        const bool full = x < lenw;
        cp_async4_zfill(win + e, full ? base + int64_t(i) * g.stride + x : base, full);
    }
    if (g.ifce_slot >= 0) {
        float* wr = win + (kMaxPad + 1) * LT;
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

// weight-gradient row blocks
enum UnitKind { kU_W1 = 0, kU_W2 = 1, kU_W3 = 2, kU_IF = 3 };

template <int DP, int WP>
struct UnitDesc {
    int kind, m0, arows, nn;
    const float* A;
    const float* B;
};

template <int DP, int WP>
__device__ __forceinline__ UnitDesc<DP, WP> unit_desc(int mr, const float* act, const float* winR, int Wd) {
    using K = A3<DP, WP>;
    UnitDesc<DP, WP> u;
    if (mr < K::MT1) {
        u = {kU_W1, 16 * mr, K::KA, K::NC8, act + K::O_A1, act + K::O_C};
    } else if (mr < K::MT1 + K::MT2) {
        u = {kU_W2, 16 * (mr - K::MT1), K::KW, K::NH8, act + K::O_A2, act + K::O_H1};
    } else if (mr == K::MT1 + K::MT2) {
        u = {kU_W3, 16 * (Wd / 16), K::KA, K::NH8, act + K::O_A1, act + K::O_H2};
    } else {
        u = {kU_IF, 0, kFM, 2, act + K::O_DF, winR};
    }
    return u;
}

// flat parameter index of weight-gradient element (m, c) of a unit kind, or -1
__device__ __forceinline__ int unit_param(const Plan& P, int kind, int m, int c, int slot) {
    const int D = P.D, Wd = P.Wd;
    if (kind == kU_W1) {
        if (m < Wd) return c < D ? P.off_l1w + m * D + c : (c == D ? P.off_l1b + m : -1);
        const int j = m - Wd;
        if (j < 2) {
            if (c < D) return P.off_astab >= 0 ? P.off_astab + j * D + c : -1;
            return c == D ? P.off_hb + j : -1;
        }
        return -1;
    }
    if (kind == kU_W2) {
        if (m < Wd) return c < Wd ? P.off_l2w + m * Wd + c : (c == Wd ? P.off_l2b + m : -1);
        return -1;
    }
    if (kind == kU_W3) {
        const int j = m - Wd;
        return (j >= 0 && j < 2 && c < Wd) ? P.off_hw + j * Wd + c : -1;
    }
    // IFCE: rows f < F, columns j < rdim (weights) and kRM (the ones row: bias)
    if (slot < 0 || m >= P.F) return -1;
    const int rd = P.g[P.slot_gi[slot]].rdim;
    return c < rd ? P.off_ifw[slot] + m * rd + c : (c == kRM ? P.off_ifb[slot] + m : -1);
}

// fp32 unit accumulators -> fp64 partial row: store (first flush of a
// parameter slot) or add; all loads are issued before the first store
template <int NMAX>
__device__ __forceinline__ void unit_flush(const Plan& P, double* row, int kind, int m0, int nn, int slot,
                                           float (&acc)[NMAX][4], int lane, bool add) {
    const int g = lane >> 2, t = lane & 3;
    int o[NMAX][4];
    double old[NMAX][4];
#pragma unroll
    for (int n = 0; n < NMAX; ++n)
#pragma unroll
        for (int r = 0; r < 4; ++r)
            o[n][r] = n < nn ? unit_param(P, kind, m0 + g + 8 * (r >> 1), 8 * n + 2 * t + (r & 1), slot) : -1;
#pragma unroll
    for (int n = 0; n < NMAX; ++n)
#pragma unroll
        for (int r = 0; r < 4; ++r) old[n][r] = (add && o[n][r] >= 0) ? row[o[n][r]] : 0.0;
#pragma unroll
    for (int n = 0; n < NMAX; ++n)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (o[n][r] >= 0) row[o[n][r]] = old[n][r] + double(acc[n][r]);
            acc[n][r] = 0.0f;
        }
}

template <int DP, int WP, int MODE>
__global__ void __launch_bounds__(NT, 2) k_arm3(const Plan* __restrict__ pp, const int4* __restrict__ tiles,
                                                int ntiles) {
    using K = A3<DP, WP>;
    const Plan& P = *pp;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    A3Smem<DP, WP>& sm = *reinterpret_cast<A3Smem<DP, WP>*>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g8 = lane >> 2, t4 = lane & 3;  // mma group / thread-in-group
    const int D = P.D, Wd = P.Wd, S = P.S, F = P.F;
    const float* prm = P.params;

    // ---------------- weights -> shared memory ----------------
    auto w1 = [&](int a, int k) { return (a < Wd && k < D) ? prm[P.off_l1w + a * D + k] : 0.0f; };
    auto w2 = [&](int b, int a) { return (b < Wd && a < Wd) ? prm[P.off_l2w + b * Wd + a] : 0.0f; };
    for (int e = tid; e < K::NS1 * K::NW8 * 32; e += NT) {  // W1ᵀ[k][a], standard order
        const int ks = e / (K::NW8 * 32), n = (e / 32) % K::NW8, l = e % 32, g = l >> 2, t = l & 3;
        sm.fL1[ks][n][l] = split_pair(w1(8 * n + g, 8 * ks + t), w1(8 * n + g, 8 * ks + t + 4));
    }
    for (int e = tid; e < K::NW8 * K::NW8 * 32; e += NT) {
        const int ks = e / (K::NW8 * 32), n = (e / 32) % K::NW8, l = e % 32, g = l >> 2, t = l & 3;
        // L2: B[k=a][n=b] = W2[b][a]; dH1: B[k=b][n=a] = W2[b][a]; K permuted (2t, 2t+1)
        sm.fL2[ks][n][l] = split_pair(w2(8 * n + g, 8 * ks + 2 * t), w2(8 * n + g, 8 * ks + 2 * t + 1));
        sm.fH1[ks][n][l] = split_pair(w2(8 * ks + 2 * t, 8 * n + g), w2(8 * ks + 2 * t + 1, 8 * n + g));
    }
    for (int e = tid; e < K::NW8 * K::ND8 * 32; e += NT) {  // dC: B[k=a][n=k'] = W1[a][k']
        const int ks = e / (K::ND8 * 32), n = (e / 32) % K::ND8, l = e % 32, g = l >> 2, t = l & 3;
        sm.fDC[ks][n][l] = split_pair(w1(8 * ks + 2 * t, 8 * n + g), w1(8 * ks + 2 * t + 1, 8 * n + g));
    }
    for (int e = tid; e < 2 * K::KW; e += NT) {
        const int j = e / K::KW, a = e % K::KW;
        sm.W3[j][a] = a < Wd ? prm[P.off_hw + j * Wd + a] : 0.0f;
    }
    for (int e = tid; e < 2 * K::KD; e += NT) {
        const int j = e / K::KD, k = e % K::KD;
        sm.stab[j][k] = (P.off_astab >= 0 && k < D) ? prm[P.off_astab + j * D + k] : 0.0f;
    }
    for (int e = tid; e < K::KW; e += NT) {
        sm.b1[e] = e < Wd ? prm[P.off_l1b + e] : 0.0f;
        sm.b2[e] = e < Wd ? prm[P.off_l2b + e] : 0.0f;
    }
    if (tid < 2) sm.b3[tid] = prm[P.off_hb + tid];
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
        sm.woff[e] = e < S ? (P.P + P.ctx_dy[e]) * LT + P.P + P.ctx_dx[e] : 0;
    for (int e = tid; e < P.n_grids; e += NT) sm.geo[e] = P.g[e];
    // staging: zero everywhere, then the constant ones rows (C: D, H1/H2: W);
    // windows zeroed, R ones row at kRM
    for (int e = tid; e < K::ACT; e += NT) sm.act[e] = 0.0f;
    for (int e = tid; e < 2 * WROWS * LT; e += NT) (&sm.win[0][0])[e] = 0.0f;
    __syncthreads();
    for (int e = tid; e < T; e += NT) {
        sm.act[K::O_C + D * LT + e] = 1.0f;
        sm.act[K::O_H1 + Wd * LT + e] = 1.0f;
        sm.act[K::O_H2 + Wd * LT + e] = 1.0f;
        sm.win[0][(kMaxPad + 1 + kRM) * LT + e] = 1.0f;
        sm.win[1][(kMaxPad + 1 + kRM) * LT + e] = 1.0f;
    }

    float* const sC = sm.act + K::O_C;
    float* const sH1 = sm.act + K::O_H1;
    float* const sH2 = sm.act + K::O_H2;
    float* const sA1 = sm.act + K::O_A1;
    float* const sA2 = sm.act + K::O_A2;
    float* const sDF = sm.act + K::O_DF;
    const int m0 = 16 * warp;  // this warp's latents inside the tile

    // weight-gradient units of this warp: u = warp + 8 i -> (row block, quarter)
    const PartialRegion& R = P.region[P.reg_arm];
    float uacc[K::NUPW][K::NMAX][4];
#pragma unroll
    for (int i = 0; i < K::NUPW; ++i)
#pragma unroll
        for (int n = 0; n < K::NMAX; ++n)
#pragma unroll
            for (int r = 0; r < 4; ++r) uacc[i][n][r] = 0.0f;
    auto qrow = [&](int q) -> double* {
        return P.arm_qs + (int64_t(q) * gridDim.x + blockIdx.x) * R.count - R.param_off;
    };
    // this warp's units, resolved once: A / B row bases (A, B inside the
    // activation buffer; the IFCE unit's B is the tile window's R rows)
    int uA[K::NUPW], uB[K::NUPW], uinfo[K::NUPW];  // info: nn | lo8 << 4 | ifce << 5 | valid << 6 | q << 8
#pragma unroll
    for (int i = 0; i < K::NUPW; ++i) {
        const int u = warp + 8 * i;
        const int mr = u % K::NMR, q = u / K::NMR;
        const UnitDesc<DP, WP> ud = unit_desc<DP, WP>(mr, sm.act, sm.act, Wd);
        uA[i] = int(ud.A - sm.act) + (ud.m0 + g8) * LT + 2 * t4;
        uB[i] = int(ud.B - sm.act) + g8 * LT + 2 * t4;
        if (ud.kind == kU_IF) uB[i] = g8 * LT + 2 * t4;
        uinfo[i] = ud.nn | (ud.m0 + 8 < ud.arows ? 16 : 0) | (ud.kind == kU_IF ? 32 : 0) | (u < K::NU ? 64 : 0) |
                   (q << 8);
    }
    int acc_slot = -1;      // IFCE slot the IFCE unit accumulators belong to
    int acc_tiles = 0;      // tiles in the fp32 unit accumulators
    bool main_flushed = false;
    int if_flushed = 0;     // IFCE slots whose parameters hold a value
    auto flush_units = [&](bool main_units, bool ifce_unit) {
        const bool if_go = ifce_unit && acc_slot >= 0;
        const bool if_add = if_go && ((if_flushed >> acc_slot) & 1);
#pragma unroll
        for (int i = 0; i < K::NUPW; ++i) {
            const int u = warp + 8 * i;
            if (u < K::NU) {
                const int mr = u % K::NMR, q = u / K::NMR;
                const UnitDesc<DP, WP> ud = unit_desc<DP, WP>(mr, sm.act, sm.act, Wd);
                if (ud.kind == kU_IF) {
                    if (if_go) unit_flush<K::NMAX>(P, qrow(q), ud.kind, ud.m0, ud.nn, acc_slot, uacc[i], lane, if_add);
                } else if (main_units) {
                    unit_flush<K::NMAX>(P, qrow(q), ud.kind, ud.m0, ud.nn, -1, uacc[i], lane, main_flushed);
                }
            }
        }
        if (if_go) if_flushed |= 1 << acc_slot;
        if (main_units) main_flushed = true;
    };

    int4 cur = blockIdx.x < ntiles ? tiles[blockIdx.x] : make_int4(0, 0, 0, 0);
    int wb = 0;
    if (blockIdx.x < ntiles) issue_gather(P, sm.geo, cur, sm.win[0], tid);
    double bits_thr = 0.0;
    const float upstream = P.rate_upstream;

    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int4 tile = cur;
        const bool has_next = t + int(gridDim.x) < ntiles;
        const int4 nxt = has_next ? tiles[t + gridDim.x] : make_int4(0, 0, 0, 0);
        const GridGeom& g = sm.geo[tile.x];
        const int64_t count = int64_t(g.rows) * g.cols;
        const int slot = g.ifce_slot;
        const int len = tile.w;
        const bool own_row = tile.z >= g.own_lo && tile.z < g.own_hi;

        // ---- land this tile's window; every warp is past the previous
        // tile's weight-gradient reads (staging, window R rows) ----
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        __syncthreads();
        if (has_next) issue_gather(P, sm.geo, nxt, sm.win[wb ^ 1], tid);
        if (MODE != kArmForward) {
            if (slot != acc_slot) {  // IFCE unit: a new slot begins (tiles run in grid order)
                flush_units(false, true);
                acc_slot = slot;
            }
            if (acc_tiles == kFlushTiles) {
                flush_units(true, true);
                acc_tiles = 0;
            }
            ++acc_tiles;
        }
        const float* win = sm.win[wb];
        const float* sR = win + (kMaxPad + 1) * LT;

        if (m0 < len) {
            // ---- P1 (warp-local): context + IFCE rows of the warp's 16 latents ----
            {
                const int l = lane & 15, half = lane >> 4, lt = m0 + l;
                const bool valid = lt < len;
                for (int o = half; o < S; o += 2) sC[o * LT + lt] = valid ? win[sm.woff[o] + lt] : 0.0f;
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
                } else {
#pragma unroll
                    for (int ff = 0; ff < FH; ++ff) {
                        const int f = half * FH + ff;
                        if (f < F) sC[(S + f) * LT + lt] = 0.0f;
                    }
                }
                if (half == 0) sC[(D + 1) * LT + lt] = valid ? win[P.P * LT + P.P + lt] : 0.0f;
            }
            __syncwarp();

            // ---- L1: H1 = relu(b1 + C·W1ᵀ); head stabiliser partials ----
            float h1[K::NW8][4];
            float p0g = 0.0f, p0h = 0.0f, p1g = 0.0f, p1h = 0.0f;  // (mu, sigma-raw) x (latent g, g+8)
#pragma unroll
            for (int n = 0; n < K::NW8; ++n) {
                const float bl = sm.b1[8 * n + 2 * t4], bh = sm.b1[8 * n + 2 * t4 + 1];
                h1[n][0] = bl;
                h1[n][1] = bh;
                h1[n][2] = bl;
                h1[n][3] = bh;
            }
#pragma unroll
            for (int ks = 0; ks < K::NS1; ++ks) {
                float a[4];
                const float* c0p = sC + (8 * ks + t4) * LT + m0 + g8;
                a[0] = c0p[0];
                a[1] = c0p[8];
                a[2] = c0p[4 * LT];
                a[3] = c0p[4 * LT + 8];
                const float s0a = sm.stab[0][8 * ks + t4], s0b = sm.stab[0][8 * ks + t4 + 4];
                const float s1a = sm.stab[1][8 * ks + t4], s1b = sm.stab[1][8 * ks + t4 + 4];
                p0g = fmaf(a[2], s0b, fmaf(a[0], s0a, p0g));
                p0h = fmaf(a[3], s0b, fmaf(a[1], s0a, p0h));
                p1g = fmaf(a[2], s1b, fmaf(a[0], s1a, p1g));
                p1h = fmaf(a[3], s1b, fmaf(a[1], s1a, p1h));
                uint32_t ah[4], al[4];
                split4(a, ah, al);
#pragma unroll
                for (int n = 0; n < K::NW8; ++n) mma3(h1[n], ah, al, sm.fL1[ks][n][lane]);
            }
#pragma unroll
            for (int n = 0; n < K::NW8; ++n)
#pragma unroll
                for (int r = 0; r < 4; ++r) h1[n][r] = h1[n][r] > 0.0f ? h1[n][r] : 0.0f;

            // ---- L2: H2 = relu(b2 + H1·W2ᵀ) ----
            float h2[K::NW8][4];
#pragma unroll
            for (int n = 0; n < K::NW8; ++n) {
                const float bl = sm.b2[8 * n + 2 * t4], bh = sm.b2[8 * n + 2 * t4 + 1];
                h2[n][0] = bl;
                h2[n][1] = bh;
                h2[n][2] = bl;
                h2[n][3] = bh;
            }
#pragma unroll
            for (int ks = 0; ks < K::NW8; ++ks) {
                float a[4];
                acc_as_a(h1[ks], a);
                uint32_t ah[4], al[4];
                split4(a, ah, al);
#pragma unroll
                for (int n = 0; n < K::NW8; ++n) mma3(h2[n], ah, al, sm.fL2[ks][n][lane]);
            }
#pragma unroll
            for (int n = 0; n < K::NW8; ++n) {
                const float w0a = sm.W3[0][8 * n + 2 * t4], w0b = sm.W3[0][8 * n + 2 * t4 + 1];
                const float w1a = sm.W3[1][8 * n + 2 * t4], w1b = sm.W3[1][8 * n + 2 * t4 + 1];
#pragma unroll
                for (int r = 0; r < 4; ++r) h2[n][r] = h2[n][r] > 0.0f ? h2[n][r] : 0.0f;
                p0g = fmaf(h2[n][1], w0b, fmaf(h2[n][0], w0a, p0g));
                p0h = fmaf(h2[n][3], w0b, fmaf(h2[n][2], w0a, p0h));
                p1g = fmaf(h2[n][1], w1b, fmaf(h2[n][0], w1a, p1g));
                p1h = fmaf(h2[n][3], w1b, fmaf(h2[n][2], w1a, p1h));
            }
            // quad reduction: every lane of the quad holds the four head outputs
#pragma unroll
            for (int s = 1; s <= 2; s <<= 1) {
                p0g += __shfl_xor_sync(0xffffffffu, p0g, s);
                p0h += __shfl_xor_sync(0xffffffffu, p0h, s);
                p1g += __shfl_xor_sync(0xffffffffu, p1g, s);
                p1h += __shfl_xor_sync(0xffffffffu, p1h, s);
            }

            // ---- Laplace rate + its backward: lane t of the quad takes
            // latent g (t even) or g+8 (t odd); t < 2 writes ----
            const int my = (t4 & 1) ? g8 + 8 : g8;
            const int lt = m0 + my;
            const bool valid = lt < len;
            const bool own = valid && own_row;
            float dmu = 0.0f, dsr = 0.0f;
            {
                const float v = sC[(D + 1) * LT + lt];
                const float mu = sm.b3[0] + ((t4 & 1) ? p0h : p0g);
                const float sr = sm.b3[1] + ((t4 & 1) ? p1h : p1g);
                const float sg = sigma_from_raw(sr);
                const float bsc = sg * kInvSqrt2F;
                const float u = fabsf(v - mu);
                const float e1 = cc_exp(-(u + 0.5f) / bsc);
                const float e2 = cc_exp(-fabsf(u - 0.5f) / bsc);
                const float p = u >= 0.5f ? 0.5f * (e2 - e1) : 1.0f - 0.5f * (e1 + e2);
                if (own && t4 < 2) bits_thr += double(-(cc_log(std_max(p, kProbFloorF)) * kLog2EF));
                if (MODE != kArmForward) {
                    float gv = 0.0f;
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
                    if (MODE == kArmProxy && valid && t4 < 2) P.gown[g.lat_off + int64_t(tile.y) + lt] = gv;
                    if (t4 < 2) {
                        sA1[Wd * LT + lt] = dmu;
                        sA1[(Wd + 1) * LT + lt] = dsr;
                    }
                }
            }
            if (MODE != kArmForward) {
                const int qb = lane & ~3;
                const float dmu_g = __shfl_sync(0xffffffffu, dmu, qb);
                const float dsr_g = __shfl_sync(0xffffffffu, dsr, qb);
                const float dmu_h = __shfl_sync(0xffffffffu, dmu, qb | 1);
                const float dsr_h = __shfl_sync(0xffffffffu, dsr, qb | 1);
                const int cg = m0 + g8;  // staging column of latent g (g+8: +8)

                // ---- stage C-side activations for the weight gradients ----
#pragma unroll
                for (int n = 0; n < K::NW8; ++n)
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const int a = 8 * n + 2 * t4 + (r & 1), c = cg + 8 * (r >> 1);
                        if (a < Wd) {
                            sH1[a * LT + c] = h1[n][r];
                            sH2[a * LT + c] = h2[n][r];
                        }
                    }
                // ---- dH2 = (W3ᵀ·draw) ⊙ relu'(H2) ----
                float dh2[K::NW8][4];
#pragma unroll
                for (int n = 0; n < K::NW8; ++n)
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const int a = 8 * n + 2 * t4 + (r & 1);
                        const float dm = (r >> 1) ? dmu_h : dmu_g, ds = (r >> 1) ? dsr_h : dsr_g;
                        const float d = fmaf(ds, sm.W3[1][a], fmaf(dm, sm.W3[0][a], 0.0f));
                        dh2[n][r] = h2[n][r] > 0.0f ? d : 0.0f;
                        if (a < Wd) sA2[a * LT + cg + 8 * (r >> 1)] = dh2[n][r];
                    }
                // ---- dH1 = (dH2·W2) ⊙ relu'(H1) ----
                float dh1[K::NW8][4];
#pragma unroll
                for (int n = 0; n < K::NW8; ++n)
#pragma unroll
                    for (int r = 0; r < 4; ++r) dh1[n][r] = 0.0f;
#pragma unroll
                for (int ks = 0; ks < K::NW8; ++ks) {
                    float a[4];
                    acc_as_a(dh2[ks], a);
                    uint32_t ah[4], al[4];
                    split4(a, ah, al);
#pragma unroll
                    for (int n = 0; n < K::NW8; ++n) mma3(dh1[n], ah, al, sm.fH1[ks][n][lane]);
                }
#pragma unroll
                for (int n = 0; n < K::NW8; ++n)
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const int a = 8 * n + 2 * t4 + (r & 1);
                        dh1[n][r] = h1[n][r] > 0.0f ? dh1[n][r] : 0.0f;
                        if (a < Wd) sA1[a * LT + cg + 8 * (r >> 1)] = dh1[n][r];
                    }
                // ---- dC = dH1·W1 + draw·stab -> dctx / dF ----
                float dc[K::ND8][4];
#pragma unroll
                for (int n = 0; n < K::ND8; ++n)
#pragma unroll
                    for (int r = 0; r < 4; ++r) dc[n][r] = 0.0f;
#pragma unroll
                for (int ks = 0; ks < K::NW8; ++ks) {
                    float a[4];
                    acc_as_a(dh1[ks], a);
                    uint32_t ah[4], al[4];
                    split4(a, ah, al);
#pragma unroll
                    for (int n = 0; n < K::ND8; ++n) mma3(dc[n], ah, al, sm.fDC[ks][n][lane]);
                }
                const int64_t lbase = int64_t(tile.y) + cg;
#pragma unroll
                for (int n = 0; n < K::ND8; ++n)
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const int k = 8 * n + 2 * t4 + (r & 1), hi = r >> 1;
                        const float dm = hi ? dmu_h : dmu_g, ds = hi ? dsr_h : dsr_g;
                        const float v = fmaf(ds, sm.stab[1][k], fmaf(dm, sm.stab[0][k], dc[n][r]));
                        const bool vl = cg + 8 * hi < len;
                        if (k < S) {
                            if (MODE == kArmProxy && vl) P.dctx[g.dctx_off + int64_t(k) * count + lbase + 8 * hi] = v;
                        } else if (k < S + F && slot >= 0) {
                            sDF[(k - S) * LT + cg + 8 * hi] = vl ? v : 0.0f;
                            if (MODE == kArmProxy && vl)
                                P.dfeat[g.dfeat_off + int64_t(k - S) * count + lbase + 8 * hi] = v;
                        }
                    }
            }
        } else if (MODE != kArmForward) {
            // an empty warp slice: its staging columns must not carry the
            // previous tile's gradients into this tile's weight gradients
            const int l = lane & 15, half = lane >> 4, c = m0 + l;
            for (int a = half; a < Wd + 2; a += 2) sA1[a * LT + c] = 0.0f;
            for (int a = half; a < Wd; a += 2) sA2[a * LT + c] = 0.0f;
            for (int f = half; f < F; f += 2) sDF[f * LT + c] = 0.0f;
        }
        if (MODE == kArmForward) {
            wb ^= 1;
            cur = nxt;
            continue;
        }
        __syncthreads();

        // ---- weight gradients: this warp's units over their latent quarters ----
#pragma unroll
        for (int i = 0; i < K::NUPW; ++i) {
            const int info = uinfo[i];
            const int nn = info & 15, q = info >> 8;
            const bool is_if = info & 32;
            if ((info & 64) && 32 * q < len && (!is_if || slot >= 0)) {
                const bool lo8 = info & 16;  // rows g+8 exist
                const float* Ab = sm.act + uA[i] + 32 * q;
                const float* Bb = (is_if ? sR : sm.act) + uB[i] + 32 * q;
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const float2 x0 = *reinterpret_cast<const float2*>(Ab + 8 * ks);
                    const float2 x1 =
                        lo8 ? *reinterpret_cast<const float2*>(Ab + 8 * LT + 8 * ks) : make_float2(0.0f, 0.0f);
                    const float a[4] = {x0.x, x1.x, x0.y, x1.y};
                    uint32_t ah[4], al[4];
                    split4(a, ah, al);
#pragma unroll
                    for (int n = 0; n < K::NMAX; ++n) {
                        if (n < nn) {
                            const float2 y = *reinterpret_cast<const float2*>(Bb + 8 * n * LT + 8 * ks);
                            mma3(uacc[i][n], ah, al, split_pair(y.x, y.y));
                        }
                    }
                }
            }
        }
        wb ^= 1;
        cur = nxt;
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");

    // ---------------- per-CTA results ----------------
    const double tb = block_sum(bits_thr, sm.red);
    if (tid == 0) P.bits_part[blockIdx.x] = tb;
    if (MODE == kArmForward) return;
    flush_units(true, true);
    // IFCE slots this CTA never visited: zero their parameter slots
#pragma unroll
    for (int i = 0; i < K::NUPW; ++i) {
        const int u = warp + 8 * i;
        if (u < K::NU) {
            const int mr = u % K::NMR, q = u / K::NMR;
            const UnitDesc<DP, WP> ud = unit_desc<DP, WP>(mr, sm.act, sm.act, Wd);
            if (ud.kind == kU_IF)
                for (int s = 0; s < P.n_slots; ++s)
                    if (!((if_flushed >> s) & 1))
                        unit_flush<K::NMAX>(P, qrow(q), ud.kind, ud.m0, ud.nn, s, uacc[i], lane, false);
        }
    }
    __syncthreads();
    // quarters summed in fixed order into the CTA's partial row
    const double* q0 = qrow(0);
    const double* q1 = qrow(1);
    const double* q2 = qrow(2);
    const double* q3 = qrow(3);
    const PartialRow row(P, R, blockIdx.x);
    for (int o = R.param_off + tid; o < R.param_off + R.count; o += NT)
        row[o - R.param_off] = ((q0[o] + q1[o]) + q2[o]) + q3[o];
}

template <int DP, int WP>
size_t arm3_smem() {
    return sizeof(A3Smem<DP, WP>);
}

template <int DP, int WP, int MODE>
void launch_t(const LaunchCtx& L) {
    k_arm3<DP, WP, MODE><<<L.arm_blocks, NT, arm3_smem<DP, WP>(), L.stream>>>(L.plan, L.arm_tiles,
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
    const int smem = int(arm3_smem<DP, WP>());
    cudaFuncSetAttribute(k_arm3<DP, WP, kArmForward>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_arm3<DP, WP, kArmHard>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_arm3<DP, WP, kArmProxy>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

}  // namespace

// instantiated (Dp, Wp): the widths whose draw rows (W, W+1) share one m16 block
bool arm3_supported(int Dp, int Wp) {
    return (Dp == 8 && Wp == 8) || (Dp == 16 && Wp == 12) || (Dp == 20 && Wp == 20) ||
           (Dp == 28 && Wp == 28) || (Dp == 32 && Wp == 20);
}

size_t arm3_smem_bytes(int Dp, int Wp) {
    if (Dp == 8 && Wp == 8) return arm3_smem<8, 8>();
    if (Dp == 16 && Wp == 12) return arm3_smem<16, 12>();
    if (Dp == 20 && Wp == 20) return arm3_smem<20, 20>();
    if (Dp == 28 && Wp == 28) return arm3_smem<28, 28>();
    return arm3_smem<32, 20>();
}

void arm3_configure(int Dp, int Wp) {
    if (Dp == 8 && Wp == 8) configure_t<8, 8>();
    else if (Dp == 16 && Wp == 12) configure_t<16, 12>();
    else if (Dp == 20 && Wp == 20) configure_t<20, 20>();
    else if (Dp == 28 && Wp == 28) configure_t<28, 28>();
    else if (Dp == 32 && Wp == 20) configure_t<32, 20>();
}

void launch_arm3(const LaunchCtx& L, int mode) {
    const int Dp = L.host->Dp, Wp = L.host->Wp;
    if (Dp == 8 && Wp == 8) launch_mode<8, 8>(L, mode);
    else if (Dp == 16 && Wp == 12) launch_mode<16, 12>(L, mode);
    else if (Dp == 20 && Wp == 20) launch_mode<20, 20>(L, mode);
    else if (Dp == 28 && Wp == 28) launch_mode<28, 28>(L, mode);
    else launch_mode<32, 20>(L, mode);
}

}  // namespace ccb

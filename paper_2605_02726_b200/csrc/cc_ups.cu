// cc_ups.cu — learned 2x upsampling chain, forward and backward.
//
// Replaces upsample_forward / upsample_backward (synthesis.hpp:55-139) built
// from tconv2x_rows/cols (layers.hpp:353-460) and conv3x3_sym
// (layers.hpp:467-515).  Main grid k >= 1 is lifted through stages
// j = k-1 .. 0; stage j's parameters are shared by every grid passing it.
//
// B200 design: ONE kernel per stage and direction, all grids at that stage in
// the same launch (blockIdx.y = grid).  A CTA owns a 2-D tile; the row pass,
// the column pass and the 3x3 refinement run back to back in shared memory on
// the tile plus its replicate-clamped halo, so the intermediates (rowtmp,
// coltmp) never touch HBM — the backward recomputes them from the stage input
// instead of reading caches.  The backward is a chain of deterministic
// GATHERS (transposed refine -> transposed column pass -> transposed row
// pass); each level-j position is "owned" by exactly one CTA (the one owning
// its parent at level j+1), which is where its contribution to the tap
// gradients dk4 / dr3 is summed (fp64, fixed-order block reduction, per-CTA
// partial rows).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "cc_kernels.h"
#include "cc_math.cuh"
#include "cc_reduce.cuh"

namespace ccb {

namespace {

constexpr int kFT = 32;   // forward output tile (level j), square
constexpr int kBT = 16;   // backward input tile (level j+1), square
constexpr int kThreads = 256;     // big stages
constexpr int kThreadsWide = 512; // stages with few tiles: shorter per-CTA phase chains

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// Polyphase tap table (layers.hpp:346-351): output t reads idx[q] with tap[q].
__device__ __forceinline__ void tconv_map(int t, int last, int (&idx)[4], int (&tap)[4]) {
    const int u = t >> 1;
    if ((t & 1) == 0) {
        idx[0] = u >= 2 ? u - 2 : 0;
        idx[1] = u >= 1 ? u - 1 : 0;
        idx[2] = u;
        idx[3] = u < last ? u + 1 : last;
        tap[0] = 0; tap[1] = 2; tap[2] = 3; tap[3] = 1;
    } else {
        idx[0] = u >= 1 ? u - 1 : 0;
        idx[1] = u;
        idx[2] = u < last ? u + 1 : last;
        idx[3] = u + 2 < last ? u + 2 : last;
        tap[0] = 1; tap[1] = 3; tap[2] = 2; tap[3] = 0;
    }
}

// A clamped index window [lo, hi] of one axis, stored densely in smem.
struct Win {
    int lo, hi;
    __device__ __forceinline__ int n() const { return hi - lo + 1; }
};
// window of the tconv inputs read by outputs in [a, b] (clamped to [0, last])
__device__ __forceinline__ Win tconv_src(Win out, int last) {
    return Win{clampi((out.lo >> 1) - 2, 0, last), clampi((out.hi >> 1) + 2, 0, last)};
}

__device__ __forceinline__ const float* stage_in(const Plan& P, const UpsStage& s) {
    return s.in_is_pad ? P.yhat_pad + s.in_off : P.ups_buf + s.in_off;
}
__device__ __forceinline__ float* stage_out(const Plan& P, const UpsStage& s) {
    return s.out_is_z ? P.z + s.out_off : P.ups_buf + s.out_off;
}
__device__ __forceinline__ const float* stage_dout(const Plan& P, const UpsStage& s) {
    return s.dout_is_z ? P.dz + s.dout_off : P.ups_grad + s.dout_off;
}
__device__ __forceinline__ float* stage_din(const Plan& P, const UpsStage& s) {
    return s.din_is_lat ? P.dups + s.din_off : P.ups_grad + s.din_off;
}

// ---------------------------------------------------------------- forward
// One CTA = one kFT x kFT output tile of stage j for grid blockIdx.y.
constexpr int kFC = kFT + 2;              // coltmp window (tile + refine halo)
constexpr int kFR = kFC / 2 + 6;          // rowtmp rows / input rows
struct FwdSmem {
    float s_in[kFR * kFR];
    float s_row[kFR * kFC];
    float s_col[kFC * kFC];
};

// Tiles t_begin, t_begin + t_step, ... of stage j for grid entry si.
__device__ __forceinline__ void ups_fwd_stage(const Plan& P, int j, int si, int t_begin, int t_step,
                                              FwdSmem& fs) {
    const UpsStage& s = P.ups[j][si];
    const int ro = s.rows_out, co = s.cols_out, ri = s.rows_in, ci = s.cols_in;
    const int tiles_x = (co + kFT - 1) / kFT;
    const int ntiles = tiles_x * ((ro + kFT - 1) / kFT);
    float* s_in = fs.s_in;
    float* s_row = fs.s_row;
    float* s_col = fs.s_col;
    const float* k4 = P.params + P.off_tconv[j];
    const float* r3 = P.params + P.off_refine[j];
    const float t0 = k4[0], t1 = k4[1], t2 = k4[2], t3 = k4[3];
    const float kc = r3[0], ke = r3[1], ko = r3[2];
    const float* in = stage_in(P, s);
    float* out = stage_out(P, s);
    for (int tile = t_begin; tile < ntiles; tile += t_step) {
        const int y0 = (tile / tiles_x) * kFT, x0 = (tile % tiles_x) * kFT;
        if (y0 >= kFT && x0 >= kFT && y0 / 2 + 18 <= ri - 1 && x0 / 2 + 18 <= ci - 1 && y0 + kFT <= ro - 1 &&
            x0 + kFT <= co - 1) {
            // interior tile: fixed taps and geometry, 2D thread mapping
            constexpr int XW = 22, RW = kFT + 2, CW = kFT + 2;
            const int U = y0 / 2, V = x0 / 2;
            const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5, ny = blockDim.x >> 5;
            const float kk[4] = {t0, t1, t2, t3};
            __syncthreads();
            for (int i = ty; i < XW; i += ny)
                for (int j = tx; j < XW; j += 32)
                    cp_async4(&s_in[i * XW + j], in + int64_t(U - 3 + i) * s.in_stride + (V - 3 + j));
            cp_async_wait_all();
            __syncthreads();
            for (int i = ty; i < XW; i += ny)
                for (int j = tx; j < RW; j += 32) {
                    const float* x = &s_in[i * XW + ((j - 1) >> 1) + 3];
                    s_row[i * RW + j] = ((j - 1) & 1) == 0
                                            ? kk[0] * x[-2] + kk[2] * x[-1] + kk[3] * x[0] + kk[1] * x[1]
                                            : kk[1] * x[-1] + kk[3] * x[0] + kk[2] * x[1] + kk[0] * x[2];
                }
            __syncthreads();
            for (int i = ty; i < CW; i += ny)
                for (int j = tx; j < CW; j += 32) {
                    const float* rr = &s_row[(((i - 1) >> 1) + 3) * RW + j];
                    s_col[i * CW + j] = ((i - 1) & 1) == 0
                                            ? kk[0] * rr[-2 * RW] + kk[2] * rr[-RW] + kk[3] * rr[0] + kk[1] * rr[RW]
                                            : kk[1] * rr[-RW] + kk[3] * rr[0] + kk[2] * rr[RW] + kk[0] * rr[2 * RW];
                }
            __syncthreads();
            for (int i = ty; i < kFT; i += ny) {
                const float* x0r = &s_col[i * CW + 1];
                const float* x1r = x0r + CW;
                const float* x2r = x1r + CW;
                const int j = tx;
                out[int64_t(y0 + i) * co + x0 + j] = kc * x1r[j] + ke * (x0r[j] + x2r[j] + x1r[j - 1] + x1r[j + 1]) +
                                                     ko * (x0r[j - 1] + x0r[j + 1] + x2r[j - 1] + x2r[j + 1]);
            }
            continue;
        }
        const Win cr{clampi(y0 - 1, 0, ro - 1), clampi(y0 + kFT, 0, ro - 1)};   // coltmp rows
        const Win cc{clampi(x0 - 1, 0, co - 1), clampi(x0 + kFT, 0, co - 1)};   // coltmp cols
        const Win rr = tconv_src(cr, ri - 1);                                  // rowtmp/input rows
        const Win ic = tconv_src(cc, ci - 1);                                  // input cols
        __syncthreads();
        for (int e = threadIdx.x; e < rr.n() * ic.n(); e += blockDim.x) {
            const int a = FDiv(ic.n()).div(e), b = e - a * ic.n();
            cp_async4(&s_in[a * kFR + b], in + int64_t(rr.lo + a) * s.in_stride + (ic.lo + b));
        }
        cp_async_wait_all();
        __syncthreads();
        // tconv2x_rows_forward (layers.hpp:353-376)
        for (int e = threadIdx.x; e < rr.n() * cc.n(); e += blockDim.x) {
            const int a = FDiv(cc.n()).div(e), b = e - a * cc.n();
            const int t = cc.lo + b;
            int idx[4], tap[4];
            tconv_map(t, ci - 1, idx, tap);
            const float* x = s_in + a * kFR - ic.lo;
            const float kk[4] = {t0, t1, t2, t3};
            s_row[a * kFC + b] = kk[tap[0]] * x[idx[0]] + kk[tap[1]] * x[idx[1]] +
                                 kk[tap[2]] * x[idx[2]] + kk[tap[3]] * x[idx[3]];
        }
        __syncthreads();
        // tconv2x_cols_forward (layers.hpp:407-429)
        for (int e = threadIdx.x; e < cr.n() * cc.n(); e += blockDim.x) {
            const int a = FDiv(cc.n()).div(e), b = e - a * cc.n();
            const int t = cr.lo + a;
            int idx[4], tap[4];
            tconv_map(t, ri - 1, idx, tap);
            const float kk[4] = {t0, t1, t2, t3};
            const float* xr = s_row + b - rr.lo * kFC;
            s_col[a * kFC + b] = kk[tap[0]] * xr[idx[0] * kFC] + kk[tap[1]] * xr[idx[1] * kFC] +
                                 kk[tap[2]] * xr[idx[2] * kFC] + kk[tap[3]] * xr[idx[3] * kFC];
        }
        __syncthreads();
        // conv3x3_sym_forward (layers.hpp:467-483)
        for (int e = threadIdx.x; e < kFT * kFT; e += blockDim.x) {
            const int r = y0 + e / kFT, c = x0 + (e % kFT);
            if (r >= ro || c >= co) continue;
            const int rm = (r > 0 ? r - 1 : 0) - cr.lo, r0 = r - cr.lo, rp = (r < ro - 1 ? r + 1 : ro - 1) - cr.lo;
            const int cm = (c > 0 ? c - 1 : 0) - cc.lo, c0 = c - cc.lo, cp = (c < co - 1 ? c + 1 : co - 1) - cc.lo;
            const float* x0r = s_col + rm * kFC;
            const float* x1r = s_col + r0 * kFC;
            const float* x2r = s_col + rp * kFC;
            out[int64_t(r) * co + c] = kc * x1r[c0] + ke * (x0r[c0] + x2r[c0] + x1r[cm] + x1r[cp]) +
                                       ko * (x0r[cm] + x0r[cp] + x2r[cm] + x2r[cp]);
        }
    }
}

__global__ void __launch_bounds__(kThreadsWide) k_ups_fwd(const Plan* __restrict__ pp, int j) {
    __shared__ FwdSmem fs;
    ups_fwd_stage(*pp, j, blockIdx.y, blockIdx.x, gridDim.x, fs);
}

// Coarse stages j >= jc of every cascade k > jc in ONE launch: CTA b runs
// cascade k = jc + 1 + b through its stages k-1 .. jc in order (a stage's
// output is the next one's input; __syncthreads orders them in the CTA).
// The coarse stages have a handful of tiles each, so this trades k - jc
// latency-bound launches for one.
__global__ void __launch_bounds__(kThreadsWide) k_ups_fwd_coarse(const Plan* __restrict__ pp, int jc) {
    __shared__ FwdSmem fs;
    const Plan& P = *pp;
    const int k = jc + 1 + blockIdx.x;
    for (int j = k - 1; j >= jc; --j) {
        ups_fwd_stage(P, j, k - j - 1, 0, 1, fs);
        __syncthreads();
    }
}

// --------------------------------------------------------------- backward
// (r', d) pairs with clamp(r' + d) == r, r' in [0, n): the transposed
// replicate-padded 3-tap stencil.
__device__ __forceinline__ int nbr_pairs(int r, int n, int (&rr)[3], int (&dd)[3]) {
    int k = 0;
    for (int q = r - 1; q <= r + 1; ++q) {
        if (q < 0 || q >= n) continue;
        for (int d = -1; d <= 1; ++d)
            if (clampi(q + d, 0, n - 1) == r && k < 3) {
                rr[k] = q;
                dd[k] = d;
                ++k;
            }
    }
    return k;
}

// windows of the backward tile (input tile [U0,U0+kBT) x [V0,V0+kBT))
constexpr int kBO = 2 * kBT;              // owned level-j span
constexpr int kBD = kBO + 10;             // dcol / drow-column window
constexpr int kBG = kBD + 2;              // dOut window
constexpr int kBC = kBO + 2;              // coltmp window (owned + refine halo)
constexpr int kBR = kBC / 2 + 6;          // rowtmp rows / input rows
constexpr int kBI = kBD / 2 + 8;          // input cols window

struct BwdSmem {
    float dout[kBG * kBG];
    float dcol[kBD * kBD];
    float drow[kBT * kBD];
    float in[kBR * kBI];
    float row[kBR * kBC];
    float col[kBC * kBC];
    double red[7 * (kThreadsWide / 32)];
    double tot[7];
};

// ---- interior fast path of the backward tile --------------------------
// For tiles whose every window is in range (no replicate clamp, no crop, no
// tconv index clamp) the stencils have fixed taps and fixed geometry, so each
// phase is a flat loop over a compile-time window.  a = 2·U0, b = 2·V0.
constexpr int FO = 2 * kBT;    // owned level-j span (32)
constexpr int FDO = FO + 10;   // dOut window: a-5 .. a+36
constexpr int FDC = FO + 8;    // dcol window: a-4 .. a+35
constexpr int FX = kBT + 6;    // input window: U0-3 .. U0+18
constexpr int FRC = FO + 4;    // rowtmp columns: b-2 .. b+33 (rows = input rows)
constexpr int FC = FO + 2;     // coltmp window: a-1 .. a+32
struct FastSmem {
    float dout[FDO * FDO];
    float dcol[FDC * FDC];
    float x[FX * FX];
    float r[FX * FRC];
    float c[FC * FC];
    float drow[kBT * FDC];
};
static_assert(sizeof(FastSmem) <= sizeof(BwdSmem) - sizeof(double) * 7 * (kThreadsWide / 32 + 1),
              "fast-path windows overlay the generic ones");

__device__ __forceinline__ bool bwd_interior(int U0, int V0, int ri, int ci, int ro, int co) {
    return U0 >= kBT && V0 >= kBT && U0 + kBT + 2 <= ri - 1 && V0 + kBT + 2 <= ci - 1 &&
           2 * U0 + FO + 4 <= ro - 1 && 2 * V0 + FO + 4 <= co - 1;
}

__device__ __forceinline__ void bwd_tile_fast(const float* __restrict__ in, int in_stride,
                                              const float* __restrict__ dout, int co,
                                              float* __restrict__ din, int ci, bool wd, int U0, int V0,
                                              const float (&kk)[4], float kc, float ke, float ko,
                                              FastSmem& f, double (&acc)[7]) {
    const int a = 2 * U0, b = 2 * V0;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5, ny = blockDim.x >> 5;
    __syncthreads();
    for (int i = ty; i < FDO; i += ny)
    for (int j = tx; j < FDO; j += 32) {
        const int e = i * FDO + j;
        cp_async4(&f.dout[e], dout + int64_t(a - 5 + i) * co + (b - 5 + j));
    }
    for (int i = ty; i < FX; i += ny)
    for (int j = tx; j < FX; j += 32) {
        const int e = i * FX + j;
        cp_async4(&f.x[e], in + int64_t(U0 - 3 + i) * in_stride + (V0 - 3 + j));
    }
    cp_async_wait_all();
    __syncthreads();
    // dcol = refineᵀ(dOut) (symmetric interior stencil), rowtmp recompute
    for (int i = ty; i < FDC; i += ny)
    for (int j = tx; j < FDC; j += 32) {
        const int e = i * FDC + j;
        const float* g = &f.dout[(i + 1) * FDO + (j + 1)];
        f.dcol[e] = kc * g[0] + ke * (g[-FDO] + g[FDO] + g[-1] + g[1]) +
                    ko * (g[-FDO - 1] + g[-FDO + 1] + g[FDO - 1] + g[FDO + 1]);
    }
    for (int i = ty; i < FX; i += ny)
    for (int j = tx; j < FRC; j += 32) {
        const int e = i * FRC + j;
        const float* x = &f.x[i * FX + (j >> 1) + 2];
        f.r[e] = (j & 1) == 0 ? kk[0] * x[-2] + kk[2] * x[-1] + kk[3] * x[0] + kk[1] * x[1]
                              : kk[1] * x[-1] + kk[3] * x[0] + kk[2] * x[1] + kk[0] * x[2];
    }
    __syncthreads();
    // coltmp recompute; drow = colᵀ(dcol) on the tile's input rows
    for (int i = ty; i < FC; i += ny)
    for (int j = tx; j < FC; j += 32) {
        const int e = i * FC + j;
        const int tr = i - 1;                 // output row a + tr
        const int v = (tr >> 1) + 3;          // R row (local) of v = U0 + floor(tr/2)
        const float* rr = &f.r[v * FRC + j + 1];
        f.c[e] = (tr & 1) == 0 ? kk[0] * rr[-2 * FRC] + kk[2] * rr[-FRC] + kk[3] * rr[0] + kk[1] * rr[FRC]
                               : kk[1] * rr[-FRC] + kk[3] * rr[0] + kk[2] * rr[FRC] + kk[0] * rr[2 * FRC];
    }
    for (int i = ty; i < kBT; i += ny)
    for (int j = tx; j < FDC; j += 32) {
        const int e = i * FDC + j;
        const float* g = &f.dcol[(2 * i + 4) * FDC + j];
        f.drow[e] = kk[0] * (g[4 * FDC] + g[-3 * FDC]) + kk[1] * (g[-2 * FDC] + g[3 * FDC]) +
                    kk[2] * (g[2 * FDC] + g[-FDC]) + kk[3] * (g[0] + g[FDC]);
    }
    __syncthreads();
    float fa[7] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    // din = rowᵀ(drow)
    if (wd) {
        for (int i = ty; i < kBT; i += ny)
        for (int j = tx; j < kBT; j += 32) {
            const float* g = &f.drow[i * FDC + 2 * j + 4];
            din[int64_t(U0 + i) * ci + V0 + j] = kk[0] * (g[4] + g[-3]) + kk[1] * (g[-2] + g[3]) +
                                                 kk[2] * (g[2] + g[-1]) + kk[3] * (g[0] + g[1]);
        }
    }
    // refine taps over the owned outputs: dOut x coltmp neighbourhoods
    for (int i = ty; i < FO; i += ny)
    for (int j = tx; j < FO; j += 32) {
        const float g = f.dout[(i + 5) * FDO + j + 5];
        const float* x0 = &f.c[i * FC + j];
        const float* x1 = x0 + FC;
        const float* x2 = x1 + FC;
        fa[4] = fmaf(g, x1[1], fa[4]);
        fa[5] = fmaf(g, x0[1] + x2[1] + x1[0] + x1[2], fa[5]);
        fa[6] = fmaf(g, x0[0] + x0[2] + x2[0] + x2[2], fa[6]);
        // column pass: dcol x rowtmp (owned output (a+i, b+j))
        const float gc = f.dcol[(i + 4) * FDC + j + 4];
        const float* rr = &f.r[((i >> 1) + 3) * FRC + j + 2];
        if ((i & 1) == 0) {
            fa[0] = fmaf(gc, rr[-2 * FRC], fa[0]);
            fa[2] = fmaf(gc, rr[-FRC], fa[2]);
            fa[3] = fmaf(gc, rr[0], fa[3]);
            fa[1] = fmaf(gc, rr[FRC], fa[1]);
        } else {
            fa[1] = fmaf(gc, rr[-FRC], fa[1]);
            fa[3] = fmaf(gc, rr[0], fa[3]);
            fa[2] = fmaf(gc, rr[FRC], fa[2]);
            fa[0] = fmaf(gc, rr[2 * FRC], fa[0]);
        }
    }
    // row pass: drow x input (input rows of the tile, owned output columns)
    for (int i = ty; i < kBT; i += ny)
    for (int j = tx; j < FO; j += 32) {
        const float g = f.drow[i * FDC + j + 4];
        const float* x = &f.x[(i + 3) * FX + (j >> 1) + 3];
        if ((j & 1) == 0) {
            fa[0] = fmaf(g, x[-2], fa[0]);
            fa[2] = fmaf(g, x[-1], fa[2]);
            fa[3] = fmaf(g, x[0], fa[3]);
            fa[1] = fmaf(g, x[1], fa[1]);
        } else {
            fa[1] = fmaf(g, x[-1], fa[1]);
            fa[3] = fmaf(g, x[0], fa[3]);
            fa[2] = fmaf(g, x[1], fa[2]);
            fa[0] = fmaf(g, x[2], fa[0]);
        }
    }
#pragma unroll
    for (int k = 0; k < 7; ++k) acc[k] += double(fa[k]);
}

__device__ __forceinline__ void ups_bwd_stage(const Plan& P, int j, int si, int t_begin, int t_step,
                                              int write_lat, unsigned char* smem_raw,
                                              double (&acc)[7]) {
    const UpsStage& s = P.ups[j][si];
    const int ro = s.rows_out, co = s.cols_out, ri = s.rows_in, ci = s.cols_in;
    const int tiles_x = (ci + kBT - 1) / kBT;
    const int ntiles = tiles_x * ((ri + kBT - 1) / kBT);
    BwdSmem& sm = *reinterpret_cast<BwdSmem*>(smem_raw);
    const float* k4 = P.params + P.off_tconv[j];
    const float* r3 = P.params + P.off_refine[j];
    const float kk[4] = {k4[0], k4[1], k4[2], k4[3]};
    const float kc = r3[0], ke = r3[1], ko = r3[2];
    const float* in = stage_in(P, s);
    const float* dout = stage_dout(P, s);
    float* din = stage_din(P, s);
    const bool wd = write_lat || !s.din_is_lat;
    for (int tile = t_begin; tile < ntiles; tile += t_step) {
        const int U0 = (tile / tiles_x) * kBT, V0 = (tile % tiles_x) * kBT;
        if (bwd_interior(U0, V0, ri, ci, ro, co)) {
            bwd_tile_fast(in, s.in_stride, dout, co, din, ci, wd, U0, V0, kk, kc, ke, ko,
                          *reinterpret_cast<FastSmem*>(smem_raw), acc);
            continue;
        }
        const int U1 = min(U0 + kBT, ri) - 1, V1 = min(V0 + kBT, ci) - 1;  // inclusive
        // owned level-j positions: parents in the tile
        const Win own_r{2 * U0, min(2 * U1 + 1, ro - 1)};
        const Win own_c{2 * V0, min(2 * V1 + 1, co - 1)};
        // level-j rows/cols whose transposed-tconv reaches the tile: t with
        // any idx(t, q) in [U0, U1]  ->  t in [2U0 - 4, 2U1 + 5]
        const Win dr{clampi(2 * U0 - 4, 0, ro - 1), clampi(2 * U1 + 5, 0, ro - 1)};
        const Win dc{clampi(2 * V0 - 4, 0, co - 1), clampi(2 * V1 + 5, 0, co - 1)};
        const Win gr{clampi(dr.lo - 1, 0, ro - 1), clampi(dr.hi + 1, 0, ro - 1)};
        const Win gc{clampi(dc.lo - 1, 0, co - 1), clampi(dc.hi + 1, 0, co - 1)};
        // recomputed forward intermediates over the owned region + refine halo
        const Win cr{clampi(own_r.lo - 1, 0, ro - 1), clampi(own_r.hi + 1, 0, ro - 1)};
        const Win cc{clampi(own_c.lo - 1, 0, co - 1), clampi(own_c.hi + 1, 0, co - 1)};
        const Win rr = tconv_src(cr, ri - 1);  // rowtmp rows (also covers rows U0..U1)
        const Win rw{min(rr.lo, U0), max(rr.hi, U1)};
        // input columns: for rowtmp over cc, and for the row-pass dk4 over own_c
        const Win ic = tconv_src(Win{min(cc.lo, own_c.lo), max(cc.hi, own_c.hi)}, ci - 1);
        __syncthreads();
        for (int e = threadIdx.x; e < gr.n() * gc.n(); e += blockDim.x) {
            const int a = FDiv(gc.n()).div(e), b = e - a * gc.n();
            cp_async4(&sm.dout[a * kBG + b], dout + int64_t(gr.lo + a) * co + (gc.lo + b));
        }
        for (int e = threadIdx.x; e < rw.n() * ic.n(); e += blockDim.x) {
            const int a = FDiv(ic.n()).div(e), b = e - a * ic.n();
            cp_async4(&sm.in[a * kBI + b], in + int64_t(rw.lo + a) * s.in_stride + (ic.lo + b));
        }
        cp_async_wait_all();
        __syncthreads();
        // rowtmp over rows rw, cols cc (recompute of tconv2x_rows_forward)
        for (int e = threadIdx.x; e < rw.n() * cc.n(); e += blockDim.x) {
            const int a = FDiv(cc.n()).div(e), b = e - a * cc.n();
            int idx[4], tap[4];
            tconv_map(cc.lo + b, ci - 1, idx, tap);
            const float* x = sm.in + a * kBI - ic.lo;
            sm.row[a * kBC + b] = kk[tap[0]] * x[idx[0]] + kk[tap[1]] * x[idx[1]] +
                                  kk[tap[2]] * x[idx[2]] + kk[tap[3]] * x[idx[3]];
        }
        // dcol over (dr, dc): transposed refine (conv3x3_sym_backward, layers.hpp:486-515)
        for (int e = threadIdx.x; e < dr.n() * dc.n(); e += blockDim.x) {
            const int a = FDiv(dc.n()).div(e), b = e - a * dc.n();
            const int r = dr.lo + a, c = dc.lo + b;
            if (r >= 1 && r <= ro - 2 && c >= 1 && c <= co - 2) {
                // interior: the symmetric stencil is its own transpose
                const float* g = sm.dout + (r - gr.lo) * kBG + (c - gc.lo);
                sm.dcol[a * kBD + b] = kc * g[0] + ke * (g[-kBG] + g[kBG] + g[-1] + g[1]) +
                                       ko * (g[-kBG - 1] + g[-kBG + 1] + g[kBG - 1] + g[kBG + 1]);
                continue;
            }
            int rp[3], rd[3], cp[3], cd[3];
            const int nr = nbr_pairs(r, ro, rp, rd), nc = nbr_pairs(c, co, cp, cd);
            float sum = 0.0f;
            for (int x = 0; x < nr; ++x)
                for (int y = 0; y < nc; ++y) {
                    const int cls = (rd[x] != 0) + (cd[y] != 0);
                    const float w = cls == 0 ? kc : (cls == 1 ? ke : ko);
                    sum += w * sm.dout[(rp[x] - gr.lo) * kBG + (cp[y] - gc.lo)];
                }
            sm.dcol[a * kBD + b] = sum;
        }
        __syncthreads();
        // coltmp over (cr, cc) (recompute of tconv2x_cols_forward)
        for (int e = threadIdx.x; e < cr.n() * cc.n(); e += blockDim.x) {
            const int a = FDiv(cc.n()).div(e), b = e - a * cc.n();
            int idx[4], tap[4];
            tconv_map(cr.lo + a, ri - 1, idx, tap);
            const float* xr = sm.row + b - rw.lo * kBC;
            sm.col[a * kBC + b] = kk[tap[0]] * xr[idx[0] * kBC] + kk[tap[1]] * xr[idx[1] * kBC] +
                                  kk[tap[2]] * xr[idx[2] * kBC] + kk[tap[3]] * xr[idx[3] * kBC];
        }
        // drow[u][t'] for u in tile rows, t' in dc: transposed column pass
        const int vmax_r = (ro - 1) >> 1;
        const int ufast_hi = min(ri - 2, (ro - 5) / 2);
        for (int e = threadIdx.x; e < (U1 - U0 + 1) * dc.n(); e += blockDim.x) {
            const int a = FDiv(dc.n()).div(e), b = e - a * dc.n();
            const int u = U0 + a;
            if (u >= 2 && u <= ufast_hi) {
                // interior: outputs 2u-3 .. 2u+4 reach u with fixed taps
                const float* g = sm.dcol + (2 * u - dr.lo) * kBD + b;
                sm.drow[a * kBD + b] = kk[0] * (g[4 * kBD] + g[-3 * kBD]) + kk[1] * (g[-2 * kBD] + g[3 * kBD]) +
                                       kk[2] * (g[2 * kBD] + g[-kBD]) + kk[3] * (g[0] + g[kBD]);
                continue;
            }
            float sum = 0.0f;
            const int v0 = max(u - 2, 0), v1 = min(u + 2, vmax_r);
            for (int v = v0; v <= v1; ++v)
                for (int par = 0; par < 2; ++par) {
                    const int t = 2 * v + par;
                    if (t >= ro) continue;
                    int idx[4], tap[4];
                    tconv_map(t, ri - 1, idx, tap);
                    const float g = sm.dcol[(t - dr.lo) * kBD + b];
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (idx[q] == u) sum += kk[tap[q]] * g;
                }
            sm.drow[a * kBD + b] = sum;
        }
        __syncthreads();
        // din[u][v]: transposed row pass (tconv2x_rows_backward, layers.hpp:378-405)
        if (wd) {
            const int vmax_c = (co - 1) >> 1;
            const int vfast_hi = min(ci - 2, (co - 5) / 2);
            for (int e = threadIdx.x; e < (U1 - U0 + 1) * (V1 - V0 + 1); e += blockDim.x) {
                const int a = FDiv(V1 - V0 + 1).div(e), b = e - a * (V1 - V0 + 1);
                const int u = V0 + b;
                if (u >= 2 && u <= vfast_hi) {
                    const float* g = sm.drow + a * kBD + (2 * u - dc.lo);
                    din[int64_t(U0 + a) * ci + u] = kk[0] * (g[4] + g[-3]) + kk[1] * (g[-2] + g[3]) +
                                                    kk[2] * (g[2] + g[-1]) + kk[3] * (g[0] + g[1]);
                    continue;
                }
                float sum = 0.0f;
                const int w0 = max(u - 2, 0), w1 = min(u + 2, vmax_c);
                for (int w = w0; w <= w1; ++w)
                    for (int par = 0; par < 2; ++par) {
                        const int t = 2 * w + par;
                        if (t >= co) continue;
                        int idx[4], tap[4];
                        tconv_map(t, ci - 1, idx, tap);
                        const float g = sm.drow[a * kBD + (t - dc.lo)];
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            if (idx[q] == u) sum += kk[tap[q]] * g;
                    }
                din[int64_t(U0 + a) * ci + u] = sum;
            }
        }
        // tap gradients over owned positions
        for (int e = threadIdx.x; e < own_r.n() * own_c.n(); e += blockDim.x) {
            const int a = FDiv(own_c.n()).div(e), b = e - a * own_c.n();
            const int r = own_r.lo + a, c = own_c.lo + b;
            // refine: dOut x coltmp neighbourhood (layers.hpp:504-506)
            const float g = sm.dout[(r - gr.lo) * kBG + (c - gc.lo)];
            const int rm = (r > 0 ? r - 1 : 0) - cr.lo, r0 = r - cr.lo, rp = (r < ro - 1 ? r + 1 : ro - 1) - cr.lo;
            const int cm = (c > 0 ? c - 1 : 0) - cc.lo, c0 = c - cc.lo, cp = (c < co - 1 ? c + 1 : co - 1) - cc.lo;
            const float* x0 = sm.col + rm * kBC;
            const float* x1 = sm.col + r0 * kBC;
            const float* x2 = sm.col + rp * kBC;
            acc[4] += double(g) * double(x1[c0]);
            acc[5] += double(g) * double(x0[c0] + x2[c0] + x1[cm] + x1[cp]);
            acc[6] += double(g) * double(x0[cm] + x0[cp] + x2[cm] + x2[cp]);
            // column pass: dcol x rowtmp (layers.hpp:452-457)
            int idx[4], tap[4];
            tconv_map(r, ri - 1, idx, tap);
            const double gc2 = double(sm.dcol[(r - dr.lo) * kBD + (c - dc.lo)]);
#pragma unroll
            for (int q = 0; q < 4; ++q)
                acc[tap[q]] += gc2 * double(sm.row[(idx[q] - rw.lo) * kBC + (c - cc.lo)]);
        }
        // row pass: drow x input over (u in tile, t' owned) (layers.hpp:395,401)
        for (int e = threadIdx.x; e < (U1 - U0 + 1) * own_c.n(); e += blockDim.x) {
            const int a = FDiv(own_c.n()).div(e), b = e - a * own_c.n();
            const int t = own_c.lo + b;
            int idx[4], tap[4];
            tconv_map(t, ci - 1, idx, tap);
            const double g = double(sm.drow[a * kBD + (t - dc.lo)]);
            const float* x = sm.in + (U0 + a - rw.lo) * kBI - ic.lo;
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[tap[q]] += g * double(x[idx[q]]);
        }
    }
}

// tap gradients of this CTA for stage j -> partial row `row`
__device__ __forceinline__ void ups_bwd_write(const Plan& P, int j, int row, unsigned char* smem_raw,
                                              double (&acc)[7]) {
    BwdSmem& sm = *reinterpret_cast<BwdSmem*>(smem_raw);
    block_sum_vec<7>(acc, sm.red, sm.tot);
    __syncthreads();
    if (threadIdx.x < 4) {
        const PartialRegion& R = P.region[P.reg_ups_rows[j]];
        P.partials[R.base + int64_t(row) * R.count + threadIdx.x] = sm.tot[threadIdx.x];
    } else if (threadIdx.x < 7) {
        const PartialRegion& R = P.region[P.reg_ups_ref[j]];
        P.partials[R.base + int64_t(row) * R.count + (threadIdx.x - 4)] = sm.tot[threadIdx.x];
    }
}

__global__ void __launch_bounds__(kThreadsWide) k_ups_bwd(const Plan* __restrict__ pp, int j,
                                                      int write_lat) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const Plan& P = *pp;
    double acc[7] = {0, 0, 0, 0, 0, 0, 0};  // dk4[0..3] (rows+cols passes), dr3[0..2]
    ups_bwd_stage(P, j, blockIdx.y, blockIdx.x, gridDim.x, write_lat, smem_raw, acc);
    ups_bwd_write(P, j, blockIdx.y * gridDim.x + blockIdx.x, smem_raw, acc);
}

// Coarse stages j >= jc in one launch (see k_ups_fwd_coarse): CTA b runs
// cascade k = jc + 1 + b through stages jc .. k-1; one partial row per
// (stage, cascade).
__global__ void __launch_bounds__(kThreadsWide) k_ups_bwd_coarse(const Plan* __restrict__ pp, int jc,
                                                             int write_lat) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const Plan& P = *pp;
    const int k = jc + 1 + blockIdx.x;
    for (int j = jc; j < k; ++j) {
        double acc[7] = {0, 0, 0, 0, 0, 0, 0};
        ups_bwd_stage(P, j, k - j - 1, 0, 1, write_lat, smem_raw, acc);
        ups_bwd_write(P, j, k - j - 1, smem_raw, acc);
        __syncthreads();
    }
}

}  // namespace

int ups_blocks_x(const Plan& H, int j, int num_sms, bool forward) {
    // enough CTAs to cover the largest grid of the stage, capped at ~2 waves
    int best = 1;
    for (int i = 0; i < H.ups_n[j]; ++i) {
        const UpsStage& s = H.ups[j][i];
        const int t = forward ? ((s.rows_out + kFT - 1) / kFT) * ((s.cols_out + kFT - 1) / kFT)
                              : ((s.rows_in + kBT - 1) / kBT) * ((s.cols_in + kBT - 1) / kBT);
        best = t > best ? t : best;
    }
    // forward: up to ~2 waves; backward: persistent CTAs (~3 per SM over all
    // grids of the stage) — every backward CTA writes a partial row of tap
    // gradients that k_nn_reduce sums, so fewer, longer-lived CTAs
    const int n = H.ups_n[j] > 0 ? H.ups_n[j] : 1;
    const int cap = forward ? (2 * num_sms * 8 + n - 1) / n : (3 * num_sms + n - 1) / n;
    return best < cap ? best : cap;
}

// First stage of the fused coarse launch: the smallest j such that every
// stage j' >= j has at most 8 tiles per grid in either direction.  Off by
// default (CCB_UPS_FUSE=1 enables it): measured at 512x768 the per-cascade
// CTA serialises ~9 tiles of the clamp-aware path (~4 us each), which is
// slower than the 3-4 latency-bound launches it replaces (146 -> 178 us).
int ups_coarse_from(const Plan& H) {
    const char* e = std::getenv("CCB_UPS_FUSE");
    if (!e || e[0] != '1') return H.L - 1;
    int jc = H.L - 1;
    for (int j = H.L - 2; j >= 0; --j) {
        int mt = 0;
        for (int i = 0; i < H.ups_n[j]; ++i) {
            const UpsStage& s = H.ups[j][i];
            const int tf = ((s.rows_out + kFT - 1) / kFT) * ((s.cols_out + kFT - 1) / kFT);
            const int tb = ((s.rows_in + kBT - 1) / kBT) * ((s.cols_in + kBT - 1) / kBT);
            mt = std::max(mt, std::max(tf, tb));
        }
        if (mt > 8) break;
        jc = j;
    }
    return jc;
}

size_t ups_bwd_smem() { return sizeof(BwdSmem); }

void ups_configure() {
    cudaFuncSetAttribute(k_ups_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(BwdSmem)));
    cudaFuncSetAttribute(k_ups_bwd_coarse, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(BwdSmem)));
}

void launch_ups_forward(const LaunchCtx& L) {
    const Plan& H = *L.host;
    // z plane 0 (= ŷ of main grid 0) is written by k_softq_fwd / k_pads_from_q
    const int jc = H.ups_jc;
    if (jc <= H.L - 2) k_ups_fwd_coarse<<<H.L - 1 - jc, kThreadsWide, 0, L.stream>>>(L.plan, jc);
    for (int j = jc - 1; j >= 0; --j) {
        if (H.ups_n[j] == 0) continue;
        const dim3 grid(ups_blocks_x(H, j, L.num_sms, true), H.ups_n[j]);
        const int nt = int(grid.x * grid.y) < 2 * L.num_sms ? kThreadsWide : kThreads;
        k_ups_fwd<<<grid, nt, 0, L.stream>>>(L.plan, j);
    }
}

void launch_ups_backward(const LaunchCtx& L, bool latent_grads, int j_begin, int j_end) {
    const Plan& H = *L.host;
    const int jc = H.ups_jc;
    for (int j = j_begin; j < jc && j <= H.L - 2 && j < j_end; ++j) {
        if (H.ups_n[j] == 0) continue;
        const dim3 grid(ups_blocks_x(H, j, L.num_sms, false), H.ups_n[j]);
        const int nt = int(grid.x * grid.y) < 2 * L.num_sms ? kThreadsWide : kThreads;
        k_ups_bwd<<<grid, nt, sizeof(BwdSmem), L.stream>>>(L.plan, j, latent_grads ? 1 : 0);
    }
    if (jc <= H.L - 2 && j_end > H.L - 2)
        k_ups_bwd_coarse<<<H.L - 1 - jc, kThreadsWide, sizeof(BwdSmem), L.stream>>>(L.plan, jc,
                                                                                   latent_grads ? 1 : 0);
}

}  // namespace ccb

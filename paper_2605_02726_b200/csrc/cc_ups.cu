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

constexpr int kThreads = 256;

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// Polyphase taps (layers.hpp:346-351): with u = t >> 1, an even output t
// reads inputs (u-2, u-1, u, u+1) with taps (k0, k2, k3, k1), an odd output
// reads (u-1, u, u+1, u+2) with taps (k1, k3, k2, k0); indices clamp to the
// input (replicate).  Every phase below hard-codes this table on a window.

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
// A CTA owns output tile [a,a+2TB) x [b,b+2TB) of stage j (a = 2U0, b = 2V0),
// computed from the input window [U0-3,U0+TB+3) x [V0-3,V0+TB+3): rowtmp
// and coltmp in polyphase pairs, the refinement in 4-row register strips.
// Border tiles clamp-load the input (replicate padding of the tconv,
// layers.hpp:353-429) and re-clamp coltmp one position outside the cropped
// level (replicate padding of conv3x3_sym_forward, layers.hpp:467-483).
template <int TB>
struct FwdGeo {
    static constexpr int FO = 2 * TB;  // owned outputs per side
    static constexpr int XW = TB + 6;  // input window, origin U0-3 / V0-3
    static constexpr int RC = FO + 4;  // rowtmp cols, origin b-2 (rows: XW)
    static constexpr int CR = FO + 4;  // coltmp rows, origin a-2
    static constexpr int CC = FO + 2;  // coltmp cols, origin b-1
};
template <int TB>
struct FwdSmem {
    using G = FwdGeo<TB>;
    float x[G::XW * G::XW];
    float r[G::XW * G::RC];
    float c[G::CR * G::CC];
};

template <int TB>
__device__ __forceinline__ bool fwd_interior(int U0, int V0, int ri, int ci, int ro, int co) {
    return U0 >= 3 && V0 >= 3 && U0 + TB + 2 <= ri - 1 && V0 + TB + 2 <= ci - 1 &&
           2 * U0 + 2 * TB + 1 <= ro - 1 && 2 * V0 + 2 * TB + 1 <= co - 1;
}

template <int TB, bool BORDER>
__device__ __forceinline__ void fwd_tile(const float* __restrict__ in, int in_stride, float* __restrict__ out,
                                         int ro, int co, int ri, int ci, int U0, int V0, const float (&kk)[4],
                                         float kc, float ke, float ko, FwdSmem<TB>& f) {
    using G = FwdGeo<TB>;
    constexpr int FO = G::FO, XW = G::XW, RC = G::RC, CR = G::CR, CC = G::CC;
    const int a = 2 * U0, b = 2 * V0;
    const int tid = threadIdx.x, nt = blockDim.x;
    __syncthreads();  // the previous tile's readers are done with the windows
    for (int e = tid; e < XW * XW; e += nt) {
        const int i = e / XW, j = e - i * XW;
        int u = U0 - 3 + i, v = V0 - 3 + j;
        if (BORDER) {
            u = clampi(u, 0, ri - 1);
            v = clampi(v, 0, ci - 1);
        }
        cp_async4(&f.x[e], in + int64_t(u) * in_stride + v);
    }
    cp_async_wait_all();
    __syncthreads();
    // rowtmp (tconv2x_rows_forward, layers.hpp:353-376): column pairs
    for (int e = tid; e < XW * (TB + 2); e += nt) {
        const int i = e / (TB + 2), m = e - i * (TB + 2);  // t' = b - 2 + 2m, +1
        const float* x = &f.x[i * XW + m];
        float* r = &f.r[i * RC + 2 * m];
        r[0] = kk[0] * x[0] + kk[2] * x[1] + kk[3] * x[2] + kk[1] * x[3];
        r[1] = kk[1] * x[1] + kk[3] * x[2] + kk[2] * x[3] + kk[0] * x[4];
    }
    __syncthreads();
    // coltmp (tconv2x_cols_forward, layers.hpp:407-429): row pairs
    for (int e = tid; e < (TB + 2) * CC; e += nt) {
        const int p = e / CC, j = e - p * CC;  // t = a - 2 + 2p, +1
        const float* r = &f.r[p * RC + j + 1];
        const float r0 = r[0], r1 = r[RC], r2 = r[2 * RC], r3 = r[3 * RC], r4 = r[4 * RC];
        f.c[(2 * p) * CC + j] = kk[0] * r0 + kk[2] * r1 + kk[3] * r2 + kk[1] * r3;
        f.c[(2 * p + 1) * CC + j] = kk[1] * r1 + kk[3] * r2 + kk[2] * r3 + kk[0] * r4;
    }
    __syncthreads();
    if (BORDER) {  // replicate padding of the cropped level: rows -1 / ro, then columns
        if (tid < CC) {
            const int im = 1 - a, ip = ro - (a - 2);
            if (im >= 0) f.c[im * CC + tid] = f.c[(im + 1) * CC + tid];
            if (ip < CR) f.c[ip * CC + tid] = f.c[(ip - 1) * CC + tid];
        }
        __syncthreads();
        if (tid < CR) {
            float* c = &f.c[tid * CC];
            const int jm = -b, jp = co - (b - 1);
            if (jm >= 0) c[jm] = c[jm + 1];
            if (jp < CC) c[jp] = c[jp - 1];
        }
        __syncthreads();
    }
    // conv3x3_sym_forward (layers.hpp:467-483) in 4-row strips
    for (int e = tid; e < (FO / 4) * FO; e += nt) {
        const int sb = e / FO, j = e - sb * FO;
        const int t0 = a + 4 * sb, tc = b + j;
        if (BORDER && (t0 >= ro || tc >= co)) continue;
        float cl[6], cm[6], cr[6];
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            const float* c = &f.c[(4 * sb + 1 + q) * CC + j];
            cl[q] = c[0];
            cm[q] = c[1];
            cr[q] = c[2];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (BORDER && t0 + q >= ro) break;
            out[int64_t(t0 + q) * co + tc] = kc * cm[q + 1] + ke * (cm[q] + cm[q + 2] + cl[q + 1] + cr[q + 1]) +
                                             ko * (cl[q] + cr[q] + cl[q + 2] + cr[q + 2]);
        }
    }
}

template <int TB>
__global__ void __launch_bounds__(kThreads) k_ups_fwd(const Plan* __restrict__ pp, int j) {
    __shared__ FwdSmem<TB> f;
    const Plan& P = pp[blockIdx.z];  // batched launches: one plan per image
    const UpsStage& s = P.ups[j][blockIdx.y];
    const int ro = s.rows_out, co = s.cols_out, ri = s.rows_in, ci = s.cols_in;
    constexpr int FO = 2 * TB;
    const int tiles_x = (co + FO - 1) / FO;
    const int ntiles = tiles_x * ((ro + FO - 1) / FO);
    const float* k4 = P.params + P.off_tconv[j];
    const float* r3 = P.params + P.off_refine[j];
    const float kk[4] = {k4[0], k4[1], k4[2], k4[3]};
    const float kc = r3[0], ke = r3[1], ko = r3[2];
    const float* in = stage_in(P, s);
    float* out = stage_out(P, s);
    pdl_wait();  // the stage input is the previous stage's output
    pdl_trigger();
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int U0 = (tile / tiles_x) * TB, V0 = (tile % tiles_x) * TB;
        if (fwd_interior<TB>(U0, V0, ri, ci, ro, co))
            fwd_tile<TB, false>(in, s.in_stride, out, ro, co, ri, ci, U0, V0, kk, kc, ke, ko, f);
        else
            fwd_tile<TB, true>(in, s.in_stride, out, ro, co, ri, ci, U0, V0, kk, kc, ke, ko, f);
    }
}

// --------------------------------------------------------------- backward
// A CTA owns input tile [U0,U0+TB) x [V0,V0+TB) of stage j+1 and the level-j
// outputs [a,a+2TB) x [b,b+2TB) (a = 2U0, b = 2V0) it parents.  Every phase is
// a flat loop over a compile-time window; each thread produces a short
// register strip (4 rows of a stencil, a polyphase pair), so operands loaded
// from shared memory are reused across the strip.
//
// Border tiles (touching the image edge or the crop of an odd-sized level)
// run the same stencils over a virtual, unclamped window and restore the
// replicate-padding semantics of the reference around them:
//   * input X is clamp-loaded, so rowtmp / coltmp recomputed on the window
//     equal R[clamp(u)] / C[clamp(t)] (tconv_map's clamped indices,
//     layers.hpp:353-429);
//   * coltmp one position outside [0,ro) x [0,co) is re-clamped to its edge
//     value (the replicate padding of conv3x3_sym_forward, layers.hpp:467-483);
//   * dOut is zero outside the image; the transposed refine stencil then
//     gives dC at virtual positions (nonzero only at distance 1), which are
//     folded onto the edge positions they clamp to, rows then columns
//     (conv3x3_sym_backward, layers.hpp:486-515);
//   * drow (virtual input rows, distance <= 2) and din (virtual input
//     columns) are folded the same way (tconv2x_{cols,rows}_backward).
// The border windows are 3 (dOut, dcol) / 2 (drow, din) positions wider per
// side.  a - 7 is odd, never 0, so every edge position a later phase reads
// has its fold sources inside the window.
template <int TB, bool BORDER>
struct BwdGeo {
    static constexpr int M = BORDER ? 3 : 0, MR = BORDER ? 2 : 0;
    static constexpr int FO = 2 * TB;           // owned level-j span
    static constexpr int DO = FO + 10 + 2 * M;  // dOut, origin a-5-M (both axes)
    static constexpr int DC = FO + 8 + 2 * M;   // dcol, origin a-4-M
    static constexpr int DR = TB + 2 * MR;      // drow rows, origin U0-MR (cols: dcol's)
    static constexpr int DI = TB + 2 * MR;      // din cols, origin V0-MR
    static constexpr int XW = TB + 6;           // input window, origin U0-3 / V0-3
    static constexpr int RC = FO + 4;           // rowtmp cols, origin b-2 (rows: XW)
    static constexpr int CR = FO + 4;           // coltmp rows, origin a-2 (pairs u = U0-1 .. U0+TB)
    static constexpr int CC = FO + 2;           // coltmp cols, origin b-1
    static constexpr int OFF = 4 + M - 2 * MR;  // dcol row of 2u for drow row 0 (same for cols)
};

template <int TB>
struct BwdSmem {
    using G = BwdGeo<TB, true>;
    float dout[G::DO * G::DO];
    float dcol[G::DC * G::DC];
    float x[G::XW * G::XW];
    float r[G::XW * G::RC];
    float c[G::CR * G::CC];
    float drow[G::DR * G::DC];
    float din[TB * G::DI];
    double red[7 * (kThreads / 32)];
    double tot[7];
};

template <int TB>
__device__ __forceinline__ bool bwd_interior(int U0, int V0, int ri, int ci, int ro, int co) {
    return U0 >= 3 && V0 >= 3 && U0 + TB + 2 <= ri - 1 && V0 + TB + 2 <= ci - 1 &&
           2 * U0 + 2 * TB + 5 <= ro && 2 * V0 + 2 * TB + 5 <= co;
}

template <int TB, bool BORDER>
__device__ __forceinline__ void bwd_tile(const float* __restrict__ in, int in_stride,
                                         const float* __restrict__ dout, int ro, int co,
                                         float* __restrict__ din, int ri, int ci, bool wd, int U0, int V0,
                                         const float (&kk)[4], float kc, float ke, float ko,
                                         BwdSmem<TB>& f, double (&acc)[7], bool first) {
    using G = BwdGeo<TB, BORDER>;
    constexpr int M = G::M, MR = G::MR, FO = G::FO, DO = G::DO, DC = G::DC, DR = G::DR, DI = G::DI;
    constexpr int XW = G::XW, RC = G::RC, CR = G::CR, CC = G::CC, OFF = G::OFF;
    const int a = 2 * U0, b = 2 * V0;
    const int tid = threadIdx.x, nt = blockDim.x;
    __syncthreads();  // the previous tile's readers are done with the windows
    // ---- P0: input window (clamped; forward data), then — once the
    // predecessor grid is done — the dOut window (zero outside the image)
    for (int e = tid; e < XW * XW; e += nt) {
        const int i = e / XW, j = e - i * XW;
        int u = U0 - 3 + i, v = V0 - 3 + j;
        if (BORDER) {
            u = clampi(u, 0, ri - 1);
            v = clampi(v, 0, ci - 1);
        }
        cp_async4(&f.x[e], in + int64_t(u) * in_stride + v);
    }
    if (first) {
        pdl_wait();
        pdl_trigger();
    }
    for (int e = tid; e < DO * DO; e += nt) {
        const int i = e / DO, j = e - i * DO;
        const int t = a - 5 - M + i, tc = b - 5 - M + j;
        if (!BORDER || (t >= 0 && t < ro && tc >= 0 && tc < co))
            cp_async4(&f.dout[e], dout + int64_t(t) * co + tc);
        else
            f.dout[e] = 0.0f;
    }
    cp_async_wait_all();
    __syncthreads();
    // ---- P1: dcol = refineᵀ(dOut) in 4-row strips; rowtmp in polyphase pairs
    {
        constexpr int NB = (DC + 3) / 4;
        for (int e = tid; e < NB * DC; e += nt) {
            const int rb = e / DC, j = e - rb * DC, i0 = 4 * rb;
            float m[6], h[6];
#pragma unroll
            for (int q = 0; q < 6; ++q) {
                if (DC % 4 == 0 || i0 + q < DO) {
                    const float* g = &f.dout[(i0 + q) * DO + j];
                    m[q] = g[1];
                    h[q] = g[0] + g[2];
                } else {
                    m[q] = h[q] = 0.0f;
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (DC % 4 == 0 || i0 + q < DC)
                    f.dcol[(i0 + q) * DC + j] = kc * m[q + 1] + ke * (m[q] + m[q + 2] + h[q + 1]) + ko * (h[q] + h[q + 2]);
        }
    }
    for (int e = tid; e < XW * (TB + 2); e += nt) {
        const int i = e / (TB + 2), m = e - i * (TB + 2);  // t' = b - 2 + 2m, +1
        const float* x = &f.x[i * XW + m];
        float* r = &f.r[i * RC + 2 * m];
        r[0] = kk[0] * x[0] + kk[2] * x[1] + kk[3] * x[2] + kk[1] * x[3];
        r[1] = kk[1] * x[1] + kk[3] * x[2] + kk[2] * x[3] + kk[0] * x[4];
    }
    __syncthreads();
    // ---- P2: coltmp in polyphase pairs; fold of dcol rows -1 -> 0, ro -> ro-1
    for (int e = tid; e < (TB + 2) * CC; e += nt) {
        const int p = e / CC, j = e - p * CC;  // t = a - 2 + 2p, +1
        const float* r = &f.r[p * RC + j + 1];
        const float r0 = r[0], r1 = r[RC], r2 = r[2 * RC], r3 = r[3 * RC], r4 = r[4 * RC];
        f.c[(2 * p) * CC + j] = kk[0] * r0 + kk[2] * r1 + kk[3] * r2 + kk[1] * r3;
        f.c[(2 * p + 1) * CC + j] = kk[1] * r1 + kk[3] * r2 + kk[2] * r3 + kk[0] * r4;
    }
    if (BORDER && tid < DC) {
        const int j = tid;
        const int i0 = 4 + M - a;           // local row of t = 0
        const int i1 = ro - 1 - (a - 4 - M);  // local row of t = ro - 1
        if (i0 >= 1 && i0 < DC) {
            f.dcol[i0 * DC + j] += f.dcol[(i0 - 1) * DC + j];
            f.dcol[(i0 - 1) * DC + j] = 0.0f;
        }
        if (i1 >= 0 && i1 + 1 < DC) {
            f.dcol[i1 * DC + j] += f.dcol[(i1 + 1) * DC + j];
            f.dcol[(i1 + 1) * DC + j] = 0.0f;
        }
    }
    __syncthreads();
    if (BORDER) {
        // fold of dcol columns; coltmp rows -1 / ro re-clamped
        if (tid < DC) {
            float* d = &f.dcol[tid * DC];
            const int j0 = 4 + M - b, j1 = co - 1 - (b - 4 - M);
            if (j0 >= 1 && j0 < DC) {
                d[j0] += d[j0 - 1];
                d[j0 - 1] = 0.0f;
            }
            if (j1 >= 0 && j1 + 1 < DC) {
                d[j1] += d[j1 + 1];
                d[j1 + 1] = 0.0f;
            }
        }
        if (tid >= nt - CC) {
            const int j = tid - (nt - CC);
            const int im = 1 - a, ip = ro - (a - 2);  // local rows of t = -1, t = ro
            if (im >= 0) f.c[im * CC + j] = f.c[(im + 1) * CC + j];
            if (ip < CR) f.c[ip * CC + j] = f.c[(ip - 1) * CC + j];
        }
        __syncthreads();
        if (tid >= nt - CR) {  // coltmp columns -1 / co (after the rows: corners)
            float* c = &f.c[(tid - (nt - CR)) * CC];
            const int jm = -b, jp = co - (b - 1);
            if (jm >= 0) c[jm] = c[jm + 1];
            if (jp < CC) c[jp] = c[jp - 1];
        }
    }
    // ---- P3: drow = colᵀ(dcol), two input rows per thread
    for (int e = tid; e < (DR / 2) * DC; e += nt) {
        const int pb = e / DC, j = e - pb * DC;
        const float* g = &f.dcol[(4 * pb + OFF - 3) * DC + j];
        float v[10];
#pragma unroll
        for (int k = 0; k < 10; ++k) v[k] = g[k * DC];
        f.drow[(2 * pb) * DC + j] = kk[0] * (v[7] + v[0]) + kk[1] * (v[1] + v[6]) + kk[2] * (v[5] + v[2]) + kk[3] * (v[3] + v[4]);
        f.drow[(2 * pb + 1) * DC + j] = kk[0] * (v[9] + v[2]) + kk[1] * (v[3] + v[8]) + kk[2] * (v[7] + v[4]) + kk[3] * (v[5] + v[6]);
    }
    __syncthreads();
    if (BORDER) {
        // fold of drow rows -2,-1 -> 0 and ri, ri+1 -> ri-1 (only own rows are read)
        if (tid < DC) {
            const int j = tid;
            if (U0 == 0) {
                float* d = &f.drow[MR * DC + j];
                float s = d[-DC] + d[-2 * DC];
                if (ri == 1) s += d[DC] + d[2 * DC];
                d[0] += s;
            }
            const int i1 = ri - 1 - (U0 - MR);
            if (ri > 1 && ri - 1 >= U0 && ri - 1 < U0 + TB) {
                float* d = &f.drow[i1 * DC + j];
                d[0] += d[DC] + d[2 * DC];
            }
        }
        __syncthreads();
    }
    // ---- P4: din = rowᵀ(drow); tap gradients
    float fa[7] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (wd) {
        constexpr int NI = BORDER ? DI : TB;
        for (int e = tid; e < TB * NI; e += nt) {
            const int i = e / NI, jj = e - i * NI;
            if (BORDER && U0 + i >= ri) continue;
            const float* g = &f.drow[(i + MR) * DC + 2 * jj + OFF];
            const float s = kk[0] * (g[4] + g[-3]) + kk[1] * (g[-2] + g[3]) + kk[2] * (g[2] + g[-1]) + kk[3] * (g[0] + g[1]);
            if (BORDER) f.din[i * DI + jj] = s;
            else din[int64_t(U0 + i) * ci + V0 + jj] = s;
        }
    }
    // refine taps (dOut x coltmp neighbourhood) and column pass (dcol x
    // rowtmp) over 4-row strips of owned outputs
    for (int e = tid; e < (FO / 4) * FO; e += nt) {
        const int sb = e / FO, j = e - sb * FO;
        const int t0 = a + 4 * sb;
        if (BORDER && (t0 >= ro || b + j >= co)) continue;
        float cm[6], ch[6];
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            const float* c = &f.c[(4 * sb + 1 + q) * CC + j];
            cm[q] = c[1];
            ch[q] = c[0] + c[2];
        }
        float rr[6];
#pragma unroll
        for (int q = 0; q < 6; ++q) rr[q] = f.r[(2 * sb + 1 + q) * RC + j + 2];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (BORDER && t0 + q >= ro) break;
            const float g = f.dout[(4 * sb + q + 5 + M) * DO + j + 5 + M];
            fa[4] = fmaf(g, cm[q + 1], fa[4]);
            fa[5] = fmaf(g, cm[q] + cm[q + 2] + ch[q + 1], fa[5]);
            fa[6] = fmaf(g, ch[q] + ch[q + 2], fa[6]);
            const float gc = f.dcol[(4 * sb + q + 4 + M) * DC + j + 4 + M];
            const int u = q >> 1;  // rr[u + k] = R row (t>>1) - 2 + k
            if ((q & 1) == 0) {
                fa[0] = fmaf(gc, rr[u + 0], fa[0]);
                fa[2] = fmaf(gc, rr[u + 1], fa[2]);
                fa[3] = fmaf(gc, rr[u + 2], fa[3]);
                fa[1] = fmaf(gc, rr[u + 3], fa[1]);
            } else {
                fa[1] = fmaf(gc, rr[u + 1], fa[1]);
                fa[3] = fmaf(gc, rr[u + 2], fa[3]);
                fa[2] = fmaf(gc, rr[u + 3], fa[2]);
                fa[0] = fmaf(gc, rr[u + 4], fa[0]);
            }
        }
    }
    // row pass: drow x input over own input rows and owned output column pairs
    for (int e = tid; e < TB * TB; e += nt) {
        const int i = e / TB, m = e - i * TB;
        if (BORDER && (U0 + i >= ri || b + 2 * m >= co)) continue;
        const float* x = &f.x[(i + 3) * XW + m + 1];  // x[k] = X col V0 + m - 2 + k
        const float* g = &f.drow[(i + MR) * DC + 2 * m + 4 + M];
        const float ge = g[0];
        fa[0] = fmaf(ge, x[0], fa[0]);
        fa[2] = fmaf(ge, x[1], fa[2]);
        fa[3] = fmaf(ge, x[2], fa[3]);
        fa[1] = fmaf(ge, x[3], fa[1]);
        if (!BORDER || b + 2 * m + 1 < co) {
            const float go = g[1];
            fa[1] = fmaf(go, x[1], fa[1]);
            fa[3] = fmaf(go, x[2], fa[3]);
            fa[2] = fmaf(go, x[3], fa[2]);
            fa[0] = fmaf(go, x[4], fa[0]);
        }
    }
#pragma unroll
    for (int k = 0; k < 7; ++k) acc[k] += double(fa[k]);
    if (!BORDER || !wd) return;
    __syncthreads();
    // din: fold virtual cols -2,-1 -> 0 and ci, ci+1 -> ci-1; own in-image writes
    for (int e = tid; e < TB * TB; e += nt) {
        const int i = e / TB, jj = e - i * TB;
        const int v = V0 + jj;
        if (U0 + i >= ri || v >= ci) continue;
        const float* d = &f.din[i * DI + MR];  // d[k] = column V0 + k
        float s = d[jj];
        if (v == 0) s += d[-1] + d[-2];
        if (v == ci - 1) s += d[jj + 1] + d[jj + 2];
        din[int64_t(U0 + i) * ci + v] = s;
    }
}

// Backward tile edge per stage: the largest of 16 / 8 / 4 that still gives
// every resident CTA slot work (2 per SM); coarse stages take small tiles so
// their latency-bound phase chain is short.
__host__ __device__ inline int bwd_tiles(const UpsStage& s, int tb) {
    return ((s.rows_in + tb - 1) / tb) * ((s.cols_in + tb - 1) / tb);
}
__host__ __device__ inline int fwd_tiles(const UpsStage& s, int tb) {
    return ((s.rows_out + 2 * tb - 1) / (2 * tb)) * ((s.cols_out + 2 * tb - 1) / (2 * tb));
}

template <int TB>
__device__ __forceinline__ void ups_bwd_stage(const Plan& P, int j, int si, int t_begin, int t_step,
                                              int write_lat, BwdSmem<TB>& f, double (&acc)[7]) {
    const UpsStage& s = P.ups[j][si];
    const int ro = s.rows_out, co = s.cols_out, ri = s.rows_in, ci = s.cols_in;
    const int tiles_x = (ci + TB - 1) / TB;
    const int ntiles = tiles_x * ((ri + TB - 1) / TB);
    const float* k4 = P.params + P.off_tconv[j];
    const float* r3 = P.params + P.off_refine[j];
    const float kk[4] = {k4[0], k4[1], k4[2], k4[3]};
    const float kc = r3[0], ke = r3[1], ko = r3[2];
    const float* in = stage_in(P, s);
    const float* dout = stage_dout(P, s);
    float* din = stage_din(P, s);
    const bool wd = write_lat || !s.din_is_lat;
    for (int tile = t_begin; tile < ntiles; tile += t_step) {
        const int U0 = (tile / tiles_x) * TB, V0 = (tile % tiles_x) * TB;
        const bool first = tile == t_begin;
        if (bwd_interior<TB>(U0, V0, ri, ci, ro, co))
            bwd_tile<TB, false>(in, s.in_stride, dout, ro, co, din, ri, ci, wd, U0, V0, kk, kc, ke, ko, f, acc, first);
        else
            bwd_tile<TB, true>(in, s.in_stride, dout, ro, co, din, ri, ci, wd, U0, V0, kk, kc, ke, ko, f, acc, first);
    }
}

template <int TB>
__global__ void __launch_bounds__(kThreads, 3) k_ups_bwd(const Plan* __restrict__ pp, int j, int write_lat) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BwdSmem<TB>& f = *reinterpret_cast<BwdSmem<TB>*>(smem_raw);
    const Plan& P = pp[blockIdx.z];  // batched launches: one plan per image
    double acc[7] = {0, 0, 0, 0, 0, 0, 0};  // dk4[0..3] (rows+cols passes), dr3[0..2]
    ups_bwd_stage<TB>(P, j, blockIdx.y, blockIdx.x, gridDim.x, write_lat, f, acc);
    // tap gradients of this CTA -> partial row (blockIdx.y, blockIdx.x)
    block_sum_vec<7>(acc, f.red, f.tot);
    __syncthreads();
    const int row = blockIdx.y * gridDim.x + blockIdx.x;
    if (threadIdx.x < 4) {
        const PartialRegion& R = P.region[P.reg_ups_rows[j]];
        P.partials[R.base + int64_t(threadIdx.x) * R.nblocks + row] = f.tot[threadIdx.x];
    } else if (threadIdx.x < 7) {
        const PartialRegion& R = P.region[P.reg_ups_ref[j]];
        P.partials[R.base + int64_t(threadIdx.x - 4) * R.nblocks + row] = f.tot[threadIdx.x];
    }
}

// ---------------------------------------------------------- coarse chains
// The coarse stages j >= P.ups_jc (little work each, a latency-bound launch
// apiece when run stage by stage) as ONE launch per direction: a thread-block
// cluster per cascade k walks that cascade's coarse stages in order — tiles
// of a stage spread over the cluster's CTAs, a cluster barrier
// (release / acquire) between consecutive stages, which is exactly the
// dependency (stage j of cascade k reads only stage j +- 1 of cascade k).
// Every stage uses the same tile code as the per-stage kernels.
// CTAs per cluster: CCB_UPS_CHAIN_CL (8 portable, 16 non-portable)
static int chain_cl() {
    static const int v = [] {
        const char* e = std::getenv("CCB_UPS_CHAIN_CL");
        const int c = e ? std::atoi(e) : 8;
        return c == 16 ? 16 : (c == 4 ? 4 : 8);
    }();
    return v;
}

struct ChainTiles {
    int tb[kMaxLevels];  // tile edge (4 / 8) of each stage
};

__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ int cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return int(r);
}

template <int TB>
__device__ __forceinline__ void fwd_stage_tiles(const Plan& P, int j, int si, int t_begin, int t_step,
                                                FwdSmem<TB>& f) {
    const UpsStage& s = P.ups[j][si];
    const int ro = s.rows_out, co = s.cols_out, ri = s.rows_in, ci = s.cols_in;
    constexpr int FO = 2 * TB;
    const int tiles_x = (co + FO - 1) / FO;
    const int ntiles = tiles_x * ((ro + FO - 1) / FO);
    const float* k4 = P.params + P.off_tconv[j];
    const float* r3 = P.params + P.off_refine[j];
    const float kk[4] = {k4[0], k4[1], k4[2], k4[3]};
    const float kc = r3[0], ke = r3[1], ko = r3[2];
    const float* in = stage_in(P, s);
    float* out = stage_out(P, s);
    for (int tile = t_begin; tile < ntiles; tile += t_step) {
        const int U0 = (tile / tiles_x) * TB, V0 = (tile % tiles_x) * TB;
        if (fwd_interior<TB>(U0, V0, ri, ci, ro, co))
            fwd_tile<TB, false>(in, s.in_stride, out, ro, co, ri, ci, U0, V0, kk, kc, ke, ko, f);
        else
            fwd_tile<TB, true>(in, s.in_stride, out, ro, co, ri, ci, U0, V0, kk, kc, ke, ko, f);
    }
}

// forward: cascade k = jc + 1 + blockIdx.y runs stages k-1 .. jc
__global__ void __launch_bounds__(kThreads) k_ups_fwd_chain(const Plan* __restrict__ pp, ChainTiles ct) {
    __shared__ FwdSmem<8> f8;
    const Plan& P = pp[blockIdx.z];  // batched launches: one plan per image
    const int jc = P.ups_jc, k = jc + 1 + int(blockIdx.y), rank = cluster_rank();
    pdl_wait();  // the inputs (the soft-quantised latents) come from the predecessor
    pdl_trigger();
    for (int j = k - 1; j >= jc; --j) {
        const int si = k - j - 1;  // ups[j] lists the cascades k = j+1, j+2, ... in order
        if (ct.tb[j] == 8) fwd_stage_tiles<8>(P, j, si, rank, int(gridDim.x), f8);
        else fwd_stage_tiles<4>(P, j, si, rank, int(gridDim.x), *reinterpret_cast<FwdSmem<4>*>(&f8));
        cluster_barrier();  // stage j's output is the next stage's input
    }
}

// backward: cascade k = jc + 1 + blockIdx.y runs stages jc .. k-1; each
// stage's tap gradients of this CTA -> partial row (si * kChainCL + rank)
__global__ void __launch_bounds__(kThreads) k_ups_bwd_chain(const Plan* __restrict__ pp, int write_lat,
                                                            ChainTiles ct) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BwdSmem<8>& f8 = *reinterpret_cast<BwdSmem<8>*>(smem_raw);
    const Plan& P = pp[blockIdx.z];  // batched launches: one plan per image
    const int jc = P.ups_jc, k = jc + 1 + int(blockIdx.y), rank = cluster_rank();
    for (int j = jc; j < k; ++j) {
        const int si = k - j - 1;
        double acc[7] = {0, 0, 0, 0, 0, 0, 0};
        if (ct.tb[j] == 8) ups_bwd_stage<8>(P, j, si, rank, int(gridDim.x), write_lat, f8, acc);
        else ups_bwd_stage<4>(P, j, si, rank, int(gridDim.x), write_lat, *reinterpret_cast<BwdSmem<4>*>(smem_raw), acc);
        __syncthreads();
        block_sum_vec<7>(acc, f8.red, f8.tot);
        __syncthreads();
        const int row = si * int(gridDim.x) + rank;
        if (threadIdx.x < 4) {
            const PartialRegion& R = P.region[P.reg_ups_rows[j]];
            P.partials[R.base + int64_t(threadIdx.x) * R.nblocks + row] = f8.tot[threadIdx.x];
        } else if (threadIdx.x < 7) {
            const PartialRegion& R = P.region[P.reg_ups_ref[j]];
            P.partials[R.base + int64_t(threadIdx.x - 4) * R.nblocks + row] = f8.tot[threadIdx.x];
        }
        cluster_barrier();  // stage j's input gradient is the next stage's output gradient
    }
}

}  // namespace

int ups_bwd_tile(const Plan& H, int j, int num_sms) {
    for (int tb : {16, 8}) {
        int t = 0;
        for (int i = 0; i < H.ups_n[j]; ++i) t += bwd_tiles(H.ups[j][i], tb);
        if (t >= 2 * num_sms) return tb;
    }
    return 4;
}

// Forward tile edge (input units; outputs 2x) per stage, by the same rule.
int ups_fwd_tile(const Plan& H, int j, int num_sms) {
    for (int tb : {16, 8}) {
        int t = 0;
        for (int i = 0; i < H.ups_n[j]; ++i) t += fwd_tiles(H.ups[j][i], tb);
        if (t >= 2 * num_sms) return tb;
    }
    return 4;
}

int ups_blocks_x(const Plan& H, int j, int num_sms, bool forward) {
    // enough CTAs to cover the largest grid of the stage, capped
    const int tb = forward ? ups_fwd_tile(H, j, num_sms) : ups_bwd_tile(H, j, num_sms);
    int best = 1;
    for (int i = 0; i < H.ups_n[j]; ++i) {
        const UpsStage& s = H.ups[j][i];
        const int t = forward ? fwd_tiles(s, tb) : bwd_tiles(s, tb);
        best = t > best ? t : best;
    }
    // forward: up to ~2 waves; backward: persistent CTAs (~3 per SM over all
    // grids of the stage) — every backward CTA writes a partial row of tap
    // gradients that k_nn_reduce sums, so fewer, longer-lived CTAs
    const int n = H.ups_n[j] > 0 ? H.ups_n[j] : 1;
    const int cap = forward ? (2 * num_sms * 8 + n - 1) / n : (3 * num_sms + n - 1) / n;
    return best < cap ? best : cap;
}

// first stage of the coarse chains (H.L - 1 = none).  Opt-in, CCB_UPS_CHAIN=j
// (chain stages j .. L-2) and CCB_UPS_CHAIN_CL = 8 / 16: measured at 512x768
// (profiles/r02_ups_chain.txt) every setting is slower than the per-stage
// launches with programmatic dependent launch (0.4598 ms per iteration vs
// 0.4598-0.4709: a cluster per cascade has fewer CTAs than the per-stage
// grids, and the stage kernels' launch latency is already hidden by PDL).
int ups_coarse_from(const Plan& H) {
    static const int jc = [] {
        const char* e = std::getenv("CCB_UPS_CHAIN");
        return e ? std::atoi(e) : 0;
    }();
    return (jc < 1 || H.L < jc + 2) ? H.L - 1 : jc;
}

int ups_chain_ctas() { return chain_cl(); }

static ChainTiles chain_tiles(const Plan& H, int num_sms) {
    ChainTiles ct{};
    for (int j = 0; j < kMaxLevels; ++j) {
        int t = 0;  // the chain's CTAs: kChainCL per cascade
        for (int i = 0; i < H.ups_n[j]; ++i) t += bwd_tiles(H.ups[j][i], 8);
        ct.tb[j] = t >= 2 * chain_cl() * (H.ups_n[j] > 0 ? H.ups_n[j] : 1) ? 8 : 4;
    }
    (void)num_sms;
    return ct;
}

static void launch_chain(const LaunchCtx& L, bool forward, int write_lat) {
    const Plan& H = *L.host;
    const int ncas = H.L - 1 - H.ups_jc;
    if (ncas <= 0) return;
    const ChainTiles ct = chain_tiles(H, L.num_sms);
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = chain_cl();
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    int na = 1;
    if (pdl_enabled(forward ? 'f' : 'b')) {
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[1].val.programmaticStreamSerializationAllowed = 1;
        na = 2;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(chain_cl(), ncas, L.batch);
    cfg.blockDim = dim3(kThreads);
    cfg.stream = L.stream;
    cfg.attrs = at;
    cfg.numAttrs = na;
    if (forward) {
        cfg.dynamicSmemBytes = 0;
        cuda_check(cudaLaunchKernelEx(&cfg, k_ups_fwd_chain, L.plan, ct), "cudaLaunchKernelEx(ups fwd chain)");
    } else {
        cfg.dynamicSmemBytes = sizeof(BwdSmem<8>);
        cuda_check(cudaLaunchKernelEx(&cfg, k_ups_bwd_chain, L.plan, write_lat, ct),
                   "cudaLaunchKernelEx(ups bwd chain)");
    }
}

void ups_configure() {
    cudaFuncSetAttribute(k_ups_bwd<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(BwdSmem<16>)));
    cudaFuncSetAttribute(k_ups_bwd<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(BwdSmem<8>)));
    cudaFuncSetAttribute(k_ups_bwd<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(BwdSmem<4>)));
    cudaFuncSetAttribute(k_ups_bwd_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(BwdSmem<8>)));
    cudaFuncSetAttribute(k_ups_bwd_chain, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_ups_fwd_chain, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
}

void launch_ups_forward(const LaunchCtx& L) {
    const Plan& H = *L.host;
    // z plane 0 (= ŷ of main grid 0) is written by k_softq_fwd / k_pads_from_q
    launch_chain(L, true, 0);  // stages >= ups_jc, every cascade in one cluster launch
    for (int j = std::min(H.L - 2, H.ups_jc - 1); j >= 0; --j) {
        if (H.ups_n[j] == 0) continue;
        const dim3 grid(ups_blocks_x(H, j, L.num_sms, true), H.ups_n[j], L.batch);
        switch (ups_fwd_tile(H, j, L.num_sms)) {
            case 16: launch_pdl(k_ups_fwd<16>, grid, kThreads, 0, L.stream, 'f', L.plan, j); break;
            case 8: launch_pdl(k_ups_fwd<8>, grid, kThreads, 0, L.stream, 'f', L.plan, j); break;
            default: launch_pdl(k_ups_fwd<4>, grid, kThreads, 0, L.stream, 'f', L.plan, j); break;
        }
    }
}

void launch_ups_backward(const LaunchCtx& L, bool latent_grads, int j_begin, int j_end) {
    const Plan& H = *L.host;
    for (int j = j_begin; j <= H.L - 2 && j < j_end; ++j) {
        if (H.ups_n[j] == 0) continue;
        if (j >= H.ups_jc) {  // the coarse chain covers every remaining stage
            launch_chain(L, false, latent_grads ? 1 : 0);
            return;
        }
        const dim3 grid(ups_blocks_x(H, j, L.num_sms, false), H.ups_n[j], L.batch);
        const int wl = latent_grads ? 1 : 0;
        switch (ups_bwd_tile(H, j, L.num_sms)) {
            case 16: launch_pdl(k_ups_bwd<16>, grid, kThreads, sizeof(BwdSmem<16>), L.stream, 'b', L.plan, j, wl); break;
            case 8: launch_pdl(k_ups_bwd<8>, grid, kThreads, sizeof(BwdSmem<8>), L.stream, 'b', L.plan, j, wl); break;
            default: launch_pdl(k_ups_bwd<4>, grid, kThreads, sizeof(BwdSmem<4>), L.stream, 'b', L.plan, j, wl); break;
        }
    }
}

}  // namespace ccb

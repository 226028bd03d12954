// cc_ctx.cuh — the ARM context gradient on its way back to the latents
// (rate_pass's scatter pads.grad[r+dy][c+dx] += dC[:, o], entropy_model.hpp:
// 312-317) as ROW PARTIALS instead of S per-offset planes.
//
// A row-segment tile (grid row r, columns c0 .. c0+len-1, c0 = q * T) groups
// its dC by the target row: offsets with dy = -d (d = 0 .. P) land in row
// r - d, at columns c0 - P .. c0 + T + P - 1.  ctx_store_partials writes, for
// every d and every such target column, the sum of the tile's contributions
// (offsets in their reference order o = 0 .. S-1); the slot [r][d][q][*] is
// written only by that tile (no atomics).  ctx_gather returns, for one latent
// (R, C), the sum over d = 0 .. P (source row R + d) of the partials of the
// (at most three) row tiles q - 1, q, q + 1 whose column span covers C — a
// fixed order, so the result is deterministic.
#pragma once

#include "cc_plan.h"

namespace ccb {

// The context offsets grouped by target row: for d = 0 .. P, the offsets
// o (ascending) with dy_o = -d and their dx.  Built once per CTA.
struct CtxTable {
    int n[5];
    int o[5][12];
    int dx[5][12];
};

__device__ __forceinline__ void ctx_table_build(const Plan& P, CtxTable& t) {  // one thread
    for (int d = 0; d < 5; ++d) t.n[d] = 0;
    for (int o = 0; o < P.S; ++o) {
        const int d = -P.ctx_dy[o];
        if (d < 0 || d > 4 || t.n[d] >= 9) continue;  // (context offsets: dy <= 0, -dy, |dx| <= pad <= 4)
        t.o[d][t.n[d]] = o;
        t.dx[d][t.n[d]] = P.ctx_dx[o];
        ++t.n[d];
    }
}

// dC: shared memory, rows o = 0 .. S-1 (stride ldc floats) over the tile's
// latents 0 .. len-1.  All nthreads threads of the CTA call it.
__device__ __forceinline__ void ctx_store_partials(const Plan& P, const GridGeom& g, int4 tile,
                                                   const float* __restrict__ dC, int ldc, const CtxTable& tb,
                                                   int tid, int nthreads) {
    constexpr int T = kArmTile;
    const int pad = P.P, W2 = T + 2 * pad, nd = pad + 1;
    const int r = tile.z, len = tile.w, c0 = tile.y - r * g.cols, q = c0 / T;
    const int ntr = (g.cols + T - 1) / T;
    float* const base = P.dctx + g.dctx_off + (int64_t(r) * nd * ntr + q) * W2;
    for (int d = 0; d < nd; ++d) {
        const int n = tb.n[d];
        int oo[9], xx[9];
#pragma unroll
        for (int i = 0; i < 9; ++i) {  // this row's offsets (<= 2P + 1 <= 9), padded with no-ops
            oo[i] = i < n ? tb.o[d][i] : 0;
            xx[i] = i < n ? tb.dx[d][i] : -(1 << 20);
        }
        float* const out = base + int64_t(d) * ntr * W2;
        for (int j = tid; j < W2; j += nthreads) {
            float acc = 0.0f;
#pragma unroll
            for (int i = 0; i < 9; ++i) {
                const int c = j - pad - xx[i];  // source latent of this target column
                if (unsigned(c) < unsigned(len)) acc += dC[oo[i] * ldc + c];
            }
            out[j] = acc;
        }
    }
}

// the context-gradient terms of latent (R, C) of grid g
__device__ __forceinline__ float ctx_gather(const Plan& P, const GridGeom& g, int R, int C) {
    constexpr int T = kArmTile;
    const int pad = P.P, W2 = T + 2 * pad, nd = pad + 1;
    const int ntr = (g.cols + T - 1) / T, q = C / T;
    const float* const base = P.dctx + g.dctx_off;
    float v[3 * 5];  // (d, q - 1 .. q + 1); pad <= 4
    int n = 0;
#pragma unroll
    for (int d = 0; d < 5; ++d) {
#pragma unroll
        for (int k = -1; k <= 1; ++k) {
            const int qq = q + k, j = C - qq * T + pad, r = R + d;
            const bool ok = d < nd && r < g.rows && qq >= 0 && qq < ntr && j >= 0 && j < W2;
            v[n++] = ok ? __ldg(base + ((int64_t(r) * nd + d) * ntr + qq) * W2 + j) : 0.0f;
        }
    }
    float acc = 0.0f;
#pragma unroll
    for (int i = 0; i < 15; ++i) acc += v[i];
    return acc;
}

}  // namespace ccb

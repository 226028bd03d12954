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

// dC: shared memory, rows o = 0 .. S-1 (stride ldc floats) over the tile's
// latents 0 .. len-1.  All nthreads threads of the CTA call it.
__device__ __forceinline__ void ctx_store_partials(const Plan& P, const GridGeom& g, int4 tile,
                                                   const float* __restrict__ dC, int ldc, int tid,
                                                   int nthreads) {
    constexpr int T = kArmTile;
    const int pad = P.P, W2 = T + 2 * pad, nd = pad + 1;
    const int r = tile.z, len = tile.w, c0 = tile.y - r * g.cols, q = c0 / T;
    const int ntr = (g.cols + T - 1) / T;
    const int S = P.S;
    float* const base = P.dctx + g.dctx_off;
    for (int e = tid; e < nd * W2; e += nthreads) {
        const int d = e / W2, j = e - d * W2;
        float acc = 0.0f;
        for (int o = 0; o < S; ++o) {
            if (-P.ctx_dy[o] != d) continue;
            const int c = j - pad - P.ctx_dx[o];  // source latent of this target column
            if (c >= 0 && c < len) acc += dC[o * ldc + c];
        }
        base[((int64_t(r) * nd + d) * ntr + q) * W2 + j] = acc;
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

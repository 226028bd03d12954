// cc_tile.cuh — register micro-tiles shared by the feature-major kernels
// (cc_arm2.cu, cc_syn_trunk.cu).
#pragma once

#include "cc_math.cuh"

namespace ccb {

// acc[r*4+c] += sum_{i in [i0,i1)} A[r][i] * B[c][i] for a 4x4 block of rows
// of two feature-major arrays (row stride LD floats, i0/i1 multiples of 4).
// FFMA2 lanes carry the even / odd columns; they are folded (even + odd)
// into acc once at the end.
// AccT = double for accumulators that live across many tiles (the per-tile
// partial is an fp32 sum over <= 64 columns; the cross-tile sum is fp64, so
// the error does not grow with the image).
template <int LD, typename AccT>
__device__ __forceinline__ void dw_tile4x4(const float* __restrict__ A, const float* __restrict__ B,
                                           int i0, int i1, AccT (&acc)[16]) {
    float2 p[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) p[e] = make_float2(0.0f, 0.0f);
#pragma unroll 2
    for (int i = i0; i < i1; i += 4) {
        float4 av[4], bv[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            av[r] = *reinterpret_cast<const float4*>(A + r * LD + i);
            bv[r] = *reinterpret_cast<const float4*>(B + r * LD + i);
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
    for (int e = 0; e < 16; ++e) acc[e] += AccT(p[e].x + p[e].y);
}

}  // namespace ccb

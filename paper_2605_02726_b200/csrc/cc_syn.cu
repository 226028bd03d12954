// cc_syn.cu — synthesis forward + MSE + backward.
//
// Replaces synthesize_forward / synthesize_backward (synthesis.hpp:191-233),
// conv1x1_* (layers.hpp:196-250), conv3x3_* (layers.hpp:257-343), mse_*
// (layers.hpp:643-657) and the straight-through clamp (layers.hpp:661-664,
// synthesis.hpp:215).  Three kernels per iteration:
//
//   k_syn_trunk_fwd   per pixel: z -> relu(c1) -> c2 = t, and the linear
//                     stabilizer term s = stab·z (3 + 3 planes); the F-wide
//                     hidden layer never leaves registers (663 MAC/px HOP)
//   k_syn_post        per 16x16 tile, in shared memory on replicate-clamped
//                     halos: residual 3x3 posts forward, clamp, MSE (fp64,
//                     owned pixels), dx̂, posts backward (transposed conv by
//                     gather), post weight gradients -> dt
//   k_syn_trunk_bwd2  (cc_syn_trunk.cu) recompute h1, dh1, dz and the
//                     c1/c2/stab weight gradients
#include <cuda_runtime.h>

#include "cc_kernels.h"
#include "cc_math.cuh"
#include "cc_reduce.cuh"

namespace ccb {

namespace {

constexpr int kLZ = kMaxLevels;  // z vector padded to 8 channels
// kSynTile (pixels per trunk-backward tile) lives in cc_plan.h



// ---------------------------------------------------------------- trunk fwd
// One thread = two neighbouring pixels: FFMA2 lanes carry the pixels, the
// weights (4 hidden units per LDS.128) are the broadcast operand.  Per output
// the order is the reference's: bias, then z channels; t sums hidden units in
// order (conv1x1_forward, layers.hpp:196-214).
__global__ void __launch_bounds__(256) k_syn_trunk_fwd(const Plan* __restrict__ pp) {
    const Plan& P = pp[blockIdx.z];  // batched launches: one plan per image
    __shared__ __align__(16) float c1wT[kLZ][64];
    __shared__ __align__(16) float c1b[64], c2w[3][64];
    __shared__ float c2b[4], st[3][kLZ];
    const int L = P.L, F = P.syn_F;
    for (int e = threadIdx.x; e < 64 * kLZ; e += blockDim.x) {
        const int f = e / kLZ, k = e - f * kLZ;
        c1wT[k][f] = (f < F && k < L) ? P.params[P.off_c1w + f * L + k] : 0.0f;
    }
    for (int e = threadIdx.x; e < 64; e += blockDim.x) c1b[e] = e < F ? P.params[P.off_c1b + e] : 0.0f;
    for (int e = threadIdx.x; e < 3 * 64; e += blockDim.x) {
        const int co = e / 64, f = e - co * 64;
        c2w[co][f] = f < F ? P.params[P.off_c2w + co * F + f] : 0.0f;
    }
    if (threadIdx.x < 4) c2b[threadIdx.x] = threadIdx.x < 3 ? P.params[P.off_c2b + threadIdx.x] : 0.0f;
    if (threadIdx.x < 3 * kLZ) {
        const int co = threadIdx.x / kLZ, k = threadIdx.x - co * kLZ;
        st[co][k] = (P.off_sstab >= 0 && k < L) ? P.params[P.off_sstab + co * L + k] : 0.0f;
    }
    __syncthreads();
    // programmatic dependent launch: the weights (settled since the last NN
    // step) are staged while the upsampling chain drains; z only after it
    pdl_wait();
    pdl_trigger();
    const int64_t np = P.npix;
    const int64_t npairs = (np + 1) / 2;
    const bool vec = P.zvec != 0;
    const int F4 = (F + 3) & ~3;
    for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < npairs;
         q += int64_t(gridDim.x) * blockDim.x) {
        const int64_t p = 2 * q;
        const bool two = p + 1 < np;
        float2 z[kLZ];
#pragma unroll
        for (int k = 0; k < kLZ; ++k) {
            z[k] = make_float2(0.0f, 0.0f);
            if (k < L) {
                const float* src = P.z + P.zpix[k] + p;
                if (vec) z[k] = *reinterpret_cast<const float2*>(src);
                else z[k] = make_float2(src[0], two ? src[1] : 0.0f);
            }
        }
        float2 t[3];
#pragma unroll
        for (int co = 0; co < 3; ++co) t[co] = make_float2(c2b[co], c2b[co]);
        for (int f = 0; f < F4; f += 4) {
            float2 a[4];
            {
                const float4 b = *reinterpret_cast<const float4*>(&c1b[f]);
                a[0] = make_float2(b.x, b.x);
                a[1] = make_float2(b.y, b.y);
                a[2] = make_float2(b.z, b.z);
                a[3] = make_float2(b.w, b.w);
            }
#pragma unroll
            for (int k = 0; k < kLZ; ++k) {
                const float4 w = *reinterpret_cast<const float4*>(&c1wT[k][f]);
                a[0] = ffma2(z[k], w.x, a[0]);
                a[1] = ffma2(z[k], w.y, a[1]);
                a[2] = ffma2(z[k], w.z, a[2]);
                a[3] = ffma2(z[k], w.w, a[3]);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float2 h = make_float2(a[i].x > 0.0f ? a[i].x : 0.0f, a[i].y > 0.0f ? a[i].y : 0.0f);
#pragma unroll
                for (int co = 0; co < 3; ++co) t[co] = ffma2(h, c2w[co][f + i], t[co]);
            }
        }
        // stabilizer s = stab·z (synthesis.hpp:211; zero padding is exact)
        float2 sz[3];
#pragma unroll
        for (int co = 0; co < 3; ++co) {
            float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
            for (int k = 0; k < kLZ; ++k) acc = ffma2(z[k], st[co][k], acc);
            sz[co] = acc;
        }
#pragma unroll
        for (int co = 0; co < 3; ++co) {
            float* dt = P.syn_t + co * np + p;
            float* ds = P.syn_sz + co * np + p;
            if (vec) {
                *reinterpret_cast<float2*>(dt) = t[co];
                *reinterpret_cast<float2*>(ds) = sz[co];
            } else {
                dt[0] = t[co].x;
                ds[0] = sz[co].x;
                if (two) {
                    dt[1] = t[co].y;
                    ds[1] = sz[co].y;
                }
            }
        }
    }
}

}  // namespace

void launch_syn_forward(const LaunchCtx& L, bool backward) {
    launch_pdl(k_syn_trunk_fwd, dim3(L.pix_blocks, 1, L.batch), dim3(256), 0, L.stream, 's', L.plan);
    launch_syn_post(L, backward);
}

}  // namespace ccb

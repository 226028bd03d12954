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
__global__ void __launch_bounds__(256) k_syn_trunk_fwd(const Plan* __restrict__ pp) {
    const Plan& P = *pp;
    __shared__ float c1w[64 * kLZ], c1b[64], c2w[3 * 64], c2b[4], st[3 * kLZ];
    const int L = P.L, F = P.syn_F;
    for (int e = threadIdx.x; e < 64 * kLZ; e += blockDim.x) {
        const int f = e / kLZ, k = e - f * kLZ;
        c1w[e] = (f < F && k < L) ? P.params[P.off_c1w + f * L + k] : 0.0f;
    }
    for (int e = threadIdx.x; e < 64; e += blockDim.x) c1b[e] = e < F ? P.params[P.off_c1b + e] : 0.0f;
    for (int e = threadIdx.x; e < 3 * 64; e += blockDim.x) {
        const int co = e / 64, f = e - co * 64;
        c2w[e] = f < F ? P.params[P.off_c2w + co * F + f] : 0.0f;
    }
    if (threadIdx.x < 4) c2b[threadIdx.x] = threadIdx.x < 3 ? P.params[P.off_c2b + threadIdx.x] : 0.0f;
    if (threadIdx.x < 3 * kLZ) {
        const int co = threadIdx.x / kLZ, k = threadIdx.x - co * kLZ;
        st[threadIdx.x] = (P.off_sstab >= 0 && k < L) ? P.params[P.off_sstab + co * L + k] : 0.0f;
    }
    __syncthreads();
    const int64_t np = P.npix;
    for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < np;
         p += int64_t(gridDim.x) * blockDim.x) {
        float zv[kLZ];
#pragma unroll
        for (int k = 0; k < kLZ; ++k) zv[k] = k < L ? P.z[P.zpix[k] + p] : 0.0f;
        float t0 = c2b[0], t1 = c2b[1], t2 = c2b[2];
        for (int f = 0; f < F; ++f) {
            float acc = c1b[f];
#pragma unroll
            for (int k = 0; k < kLZ; ++k) acc = fmaf(zv[k], c1w[f * kLZ + k], acc);
            const float h = acc > 0.0f ? acc : 0.0f;
            t0 = fmaf(c2w[f], h, t0);
            t1 = fmaf(c2w[64 + f], h, t1);
            t2 = fmaf(c2w[128 + f], h, t2);
        }
        P.syn_t[p] = t0;
        P.syn_t[np + p] = t1;
        P.syn_t[2 * np + p] = t2;
        // stabilizer s = stab·z (synthesis.hpp:211; zero padding is exact)
#pragma unroll
        for (int co = 0; co < 3; ++co) {
            float a = 0.0f;
#pragma unroll
            for (int k = 0; k < kLZ; ++k) a = fmaf(st[co * kLZ + k], zv[k], a);
            P.syn_sz[co * np + p] = a;
        }
    }
}

}  // namespace

void launch_syn_forward(const LaunchCtx& L, bool backward) {
    k_syn_trunk_fwd<<<L.pix_blocks, 256, 0, L.stream>>>(L.plan);
    launch_syn_post(L, backward);
}

}  // namespace ccb

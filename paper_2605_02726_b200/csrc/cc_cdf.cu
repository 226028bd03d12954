// cc_cdf.cu — the Laplace parameters (mu, sigma) of every quantised latent,
// for the latent entropy coder.
//
// encode_latents (bitstream.hpp:145-155) walks the latents in decode order
// and, per latent, gathers the causal context of the quantised values,
// evaluates the IFCE features and arm_forward_single (entropy_model.hpp:
// 107-134), then builds the CDF (quantize_cdf, range_coder.hpp:119-161) and
// range-codes the symbol.  Every q is known at encode time, so all (mu, sigma)
// are independent: one thread per latent computes them here.  The decoder
// recomputes them sequentially on the CPU from the decoded values, so they
// must be BIT-identical to the reference's code as compiled: every dot product
// is the reference's left-to-right chain acc = b; acc += w[k] * x[k].  The
// reference's codegen for these loops is ISA-dependent — built for
// x86-64-v3 (AVX2+FMA, -O3 -ffp-contract=fast) they are NOT contracted (a
// rounded product, then a rounded add), built for x86-64-v4 some are fused,
// and the two builds disagree on ~80 % of the mu values
// (tools/mu_sigma_isa.py).  This kernel reproduces the v3 build: explicit
// __fmul_rn / __fadd_rn, which the compiler never fuses; the ReLU, the head's
// stabiliser continuation of the same chain, cc_exp and the sigma clamp follow
// the reference's operand order.
// The range coding itself stays sequential on the host.
#include <cuda_runtime.h>

#include "cc_kernels.h"
#include "cc_math.cuh"

namespace ccb {

namespace {

constexpr int kMaxFan = 64;  // kMaxFanOut (layers.hpp:18)

// acc += w * x as the reference's x86-64-v3 build evaluates it
__device__ __forceinline__ float mul_add(float w, float x, float acc) { return __fadd_rn(acc, __fmul_rn(w, x)); }

__global__ void __launch_bounds__(128) k_latent_mu_sigma(const Plan* __restrict__ pp, float* __restrict__ mu_out,
                                                         float* __restrict__ sigma_out) {
    const Plan& P = pp[blockIdx.z];  // batched launches: one plan per image
    const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (i >= P.n_latents) return;
    int gi = 0;
    while (gi + 1 < P.n_grids && i >= P.g[gi + 1].lat_off) ++gi;
    const GridGeom& g = P.g[gi];
    const int li = int(i - g.lat_off);
    const int r = li / g.cols, c = li - r * g.cols;
    const int S = P.S, D = P.D, Wd = P.Wd;
    const int32_t* q = P.q + g.lat_off;
    float ctx[kMaxFan];
    // extract_spatial_context (entropy_model.hpp:137-150): zero outside
    for (int o = 0; o < S; ++o) {
        const int rr = r + P.ctx_dy[o], cc = c + P.ctx_dx[o];
        ctx[o] = (rr >= 0 && rr < g.rows && cc >= 0 && cc < g.cols) ? float(q[rr * g.cols + cc]) : 0.0f;
    }
    for (int j = S; j < D; ++j) ctx[j] = 0.0f;
    const int slot = g.ifce_slot;
    if (slot >= 0) {  // walk_symbols (bitstream.hpp:119-133)
        const int rd = g.rdim;
        float rv[kMaxFan];
        for (int j = 0; j < rd; ++j) {
            const GridGeom& s = P.g[j];
            const int sh = s.level - g.level;
            rv[j] = float(P.q[s.lat_off + int64_t(r >> sh) * s.cols + (c >> sh)]);
        }
        const float* w = P.params + P.off_ifw[slot];
        const float* b = P.params + P.off_ifb[slot];
        for (int f = 0; f < P.F; ++f) {
            float acc = b[f];
            for (int k = 0; k < rd; ++k) acc = mul_add(w[f * rd + k], rv[k], acc);
            ctx[S + f] = acc;
        }
    }
    // arm_forward_single (entropy_model.hpp:107-134)
    const float* w1 = P.params + P.off_l1w;
    const float* b1 = P.params + P.off_l1b;
    const float* w2 = P.params + P.off_l2w;
    const float* b2 = P.params + P.off_l2b;
    const float* w3 = P.params + P.off_hw;
    const float* b3 = P.params + P.off_hb;
    const float* st = P.off_astab >= 0 ? P.params + P.off_astab : nullptr;
    float h1[kMaxFan], h2[kMaxFan], raw[2];
    for (int j = 0; j < Wd; ++j) {
        float acc = b1[j];
        for (int k = 0; k < D; ++k) acc = mul_add(w1[j * D + k], ctx[k], acc);
        h1[j] = acc > 0.0f ? acc : 0.0f;
    }
    for (int j = 0; j < Wd; ++j) {
        float acc = b2[j];
        for (int k = 0; k < Wd; ++k) acc = mul_add(w2[j * Wd + k], h1[k], acc);
        h2[j] = acc > 0.0f ? acc : 0.0f;
    }
    for (int j = 0; j < 2; ++j) {
        float acc = b3[j];
        for (int k = 0; k < Wd; ++k) acc = mul_add(w3[j * Wd + k], h2[k], acc);
        if (st)
            for (int k = 0; k < D; ++k) acc = mul_add(st[j * D + k], ctx[k], acc);
        raw[j] = acc;
    }
    mu_out[i] = raw[0];
    sigma_out[i] = std_min(kSigmaMaxF, std_max(kSigmaMinF, cc_exp(raw[1])));
}

}  // namespace

void launch_latent_mu_sigma(const LaunchCtx& L, float* mu, float* sigma) {
    const int64_t n = L.host->n_latents;
    k_latent_mu_sigma<<<dim3(int((n + 127) / 128), 1, L.batch), 128, 0, L.stream>>>(L.plan, mu, sigma);
}

}  // namespace ccb

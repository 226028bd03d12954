// cc_latent.cu — elementwise latent kernels (HBM/L2-bound, one thread per
// latent, grid sized in multiples of the SM count by the host):
//   k_softq_fwd   soft_quantize_forward over every grid     latent.hpp:120-128,
//                 softround layers.hpp:557-568, noise encoder.hpp:100-110,213-215
//   k_quantize    quantize_all                              latent.hpp:86-99
//   k_pads_from_q load_pads_from_q                          encoder.hpp:170-180
//   k_latent_grad deterministic gather of every gradient landing on a padded
//                 latent (own rate term, ARM context scatter, IFCE scatter,
//                 upsampling) + soft_quantize_backward       latent.hpp:131-139,
//                 entropy_model.hpp:292,312-331, synthesis.hpp:135-137
//   k_adam_latents adam_step per grid, double math           optim.hpp:38-53
//   k_init_latents init_latents_uniform                      latent.hpp:73-80
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "cc_kernels.h"
#include "cc_ctx.cuh"
#include "cc_math.cuh"

namespace ccb {

// Grid of flat latent index i: latent offsets cached in shared memory (unused
// slots hold INT64_MAX), counted branch-free.
#define CCB_GRID_CACHE(P)                                                                      \
    __shared__ int64_t s_off[kMaxGrids];                                                       \
    if (threadIdx.x < kMaxGrids)                                                               \
        s_off[threadIdx.x] = int(threadIdx.x) < (P).n_grids ? (P).g[threadIdx.x].lat_off : INT64_MAX; \
    __syncthreads()

// binary search over the (sorted, INT64_MAX-padded) offsets: s_off[gi] <= i
__device__ __forceinline__ int find_grid(const int64_t* s_off, int64_t i) {
    static_assert((kMaxGrids & (kMaxGrids - 1)) == 0, "power-of-two grid table");
    int gi = 0;
#pragma unroll
    for (int step = kMaxGrids / 2; step >= 1; step >>= 1)
        if (s_off[gi + step] <= i) gi += step;
    return gi;
}

__global__ void k_softq_fwd(const Plan* __restrict__ pp) {
    const Plan& P = pp[blockIdx.z];  // batched launches: one plan per image
    CCB_GRID_CACHE(P);
    // per-grid gradient-finiteness flags of this iteration (ANDed by k_latent_grad)
    if (blockIdx.x == 0 && threadIdx.x < kMaxGrids) P.lat_ok[threadIdx.x] = 1;
    if (blockIdx.x == 0 && threadIdx.x < kMaxTensors) P.tensor_ok[threadIdx.x] = 1;  // ANDed by k_nn_reduce
    // programmatic dependent launch: the schedule scalars come from k_sched_load
    pdl_wait();
    pdl_trigger();  // the first upsampling stage may become resident
    const float temp = float(P.scal->temp);         // encoder.hpp:98
    const float noise_std = float(P.scal->noise);   // encoder.hpp:108
    const int64_t n = P.n_latents;
    const uint64_t giter = uint64_t(P.scal->global_iter);
    // the unit Gaussians of this iteration, if the previous iteration drew them
    // ahead (k_noise_ahead) for the counter value it ended with
    const bool pre = P.noise_buf != nullptr && P.scal->noise_iter == P.scal->global_iter;
    const float inv_denom = 1.0f / softround_denom(temp);
    const float inv_t = 1.0f / temp;
    __shared__ GridGeom s_geo[kMaxGrids];
    for (int k = threadIdx.x; k < P.n_grids; k += blockDim.x) s_geo[k] = P.g[k];
    __syncthreads();
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int gi = find_grid(s_off, i);
        const GridGeom& g = s_geo[gi];
        const int li = int(i - g.lat_off);  // < 2^31 latents per grid
        const int r = li / g.cols, c = li - r * g.cols;
        const float x = P.y[i];
        float f = floorf(x);
        float d = x - f - 0.5f;
        const float t1 = cc_tanh(d * inv_t);
        float o = f + 0.5f + t1 * inv_denom;
        if (noise_std > 0.0f) {
            float gz;
            if (pre) {
                gz = P.noise_buf[i];
            } else {
                const uint64_t stream = hash_combine(hash_combine(P.seed, giter), uint64_t(gi));
                gz = counter_gauss(stream, uint64_t(li) + uint64_t(int64_t(g.row0) * g.cols));  // global raster index
            }
            o += noise_std * gz;
        }
        f = floorf(o);
        d = o - f - 0.5f;
        const float t2 = cc_tanh(d * inv_t);
        o = f + 0.5f + t2 * inv_denom;
        P.yhat_pad[g.pad_base + int64_t(r) * g.stride + c] = o;
        if (g.main_level == 0) P.z[P.zpix[0] + int64_t(r) * P.W + c] = o;  // z plane 0 = ŷ_0
        P.th1[i] = t1;
        P.th2[i] = t2;
    }
}

// The noise of the NEXT iteration (noise_stream(seed, global_iter + 1),
// encoder.hpp:213-215): it depends only on the counter, so it is drawn on the
// rate branch while the distortion branch of this iteration runs.  If this
// iteration's cost turns out non-finite the counter does not advance and
// k_softq_fwd draws inline instead.
__global__ void k_noise_ahead(const Plan* __restrict__ pp) {
    const Plan& P = pp[blockIdx.z];  // batched launches: one plan per image
    CCB_GRID_CACHE(P);
    const uint64_t giter = uint64_t(P.scal->global_iter) + 1;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < P.n_latents;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int gi = find_grid(s_off, i);
        const GridGeom& g = P.g[gi];
        const uint64_t stream = hash_combine(hash_combine(P.seed, giter), uint64_t(gi));
        P.noise_buf[i] = counter_gauss(stream, uint64_t(i - g.lat_off + int64_t(g.row0) * g.cols));
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) P.scal->noise_iter = int64_t(giter);
}

__global__ void k_quantize(const Plan* __restrict__ pp, int amp) {
    const Plan& P = pp[blockIdx.z];  // batched launches: one plan per image
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < P.n_latents;
         i += int64_t(gridDim.x) * blockDim.x) {
        long q = lroundf(P.y[i]);  // ties away from zero, like std::lround
        if (q > amp) q = amp;
        if (q < -amp) q = -amp;
        P.q[i] = int32_t(q);
    }
}

__global__ void k_pads_from_q(const Plan* __restrict__ pp) {
    const Plan& P = pp[blockIdx.z];  // batched launches: one plan per image
    CCB_GRID_CACHE(P);
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < P.n_latents;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int gi = find_grid(s_off, i);
        const GridGeom& g = P.g[gi];
        const int64_t li = i - g.lat_off;
        const int r = int(li / g.cols), c = int(li - int64_t(r) * g.cols);
        P.yhat_pad[g.pad_base + int64_t(r) * g.stride + c] = float(P.q[i]);
        if (g.main_level == 0) P.z[P.zpix[0] + int64_t(r) * P.W + c] = float(P.q[i]);
    }
}

// Gradient wrt the padded soft-quantized latent, assembled by GATHER in a
// fixed order (the reference scatters with +=; the sum is the same set of
// terms):  own rate term, the S context-gradient planes of the causal
// successors, the IFCE terms W_f^T * (block sum of dF) from every equipped
// finer grid, and the upsampling gradient for main grids.  Then the
// soft-quantize backward chain rule and the per-grid finiteness flag.
__global__ void k_latent_grad(const Plan* __restrict__ pp, int force, int64_t i_begin, int64_t i_end) {
    const Plan& P = pp[blockIdx.z];  // batched launches: one plan per image
    CCB_GRID_CACHE(P);
    const float temp = float(P.scal->temp);
    (void)force;  // gradients are assembled regardless of the cost flag; k_adam_latents
                  // zeroes them when the cost is not finite (encoder.hpp:118)
    const float scale = 1.0f / (temp * softround_denom(temp));
    __shared__ int s_dy[kMaxCtx], s_dx[kMaxCtx];
    __shared__ GridGeom s_geo[kMaxGrids];
    const int S = P.S;
    for (int o = threadIdx.x; o < kMaxCtx; o += blockDim.x) {
        s_dy[o] = P.ctx_dy[o];
        s_dx[o] = P.ctx_dx[o];
    }
    for (int k = threadIdx.x; k < P.n_grids; k += blockDim.x) s_geo[k] = P.g[k];
    __syncthreads();
    for (int64_t i = i_begin + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < i_end;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int gi = find_grid(s_off, i);
        const GridGeom& g = s_geo[gi];
        const int64_t cnt = int64_t(g.rows) * g.cols;
        const int li = int(i - g.lat_off);  // < 2^31 latents per grid
        const int r = li / g.cols, c = li - r * g.cols;
        // every load of the latent is issued before the ordered sums: own
        // rate gradient, the per-latent terms below, and the causal
        // successors' context gradients (chunks of 8 offsets)
        float acc = P.gown[i];
        const float t2 = P.th2[i], t1 = P.th1[i];
        float zterm = 0.0f;
        if (g.main_level == 0)
            zterm = P.dz[P.zpix[0] + int64_t(r) * P.W + c];
        else if (g.main_level > 0)
            zterm = P.dups[i];
        const float* dc = P.dctx + g.dctx_off + li;
        if (P.ctx_part) {  // row partials of the tiled ARM kernels (cc_ctx.cuh)
            acc += ctx_gather(P, g, r, c);
        } else for (int o0 = 0; o0 < S; o0 += 8) {
            float v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int o = o0 + k;
                v[k] = 0.0f;
                if (o < S) {
                    const int dy = s_dy[o], dx = s_dx[o];
                    const int rs = r - dy, cs = c - dx;
                    if (rs >= 0 && rs < g.rows && cs >= 0 && cs < g.cols)
                        v[k] = __ldg(dc + (int64_t(o) * cnt - (dy * g.cols + dx)));
                }
            }
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (o0 + k < S) acc += v[k];  // out-of-grid terms are +0
        }
        for (int s = 0; s < P.n_slots; ++s) {
            const GridGeom& e = s_geo[P.slot_gi[s]];
            if (gi >= e.rdim) continue;
            const int sh = g.level - e.level;
            const float* pyr = P.dfeat + P.slot_pyr_off[s][sh];
            const int64_t pc = int64_t(P.slot_pyr_rows[s][sh]) * P.slot_pyr_cols[s][sh];
            const float* wf = P.params + P.off_ifw[s];
            // pyramid rows are aligned to global rows from slot_pyr_a
            const int R = g.row0 + r - (P.slot_pyr_a[s] >> sh);
            if (R < 0 || R >= P.slot_pyr_rows[s][sh]) continue;
            float dr = 0.0f;
            for (int f = 0; f < P.F; ++f)
                dr += wf[f * e.rdim + gi] * pyr[int64_t(f) * pc + int64_t(R) * g.cols + c];
            acc += dr;
        }
        if (g.main_level >= 0) acc += zterm;
        const float d2 = fmaf(-t2, t2, 1.0f) * scale;
        const float d1 = fmaf(-t1, t1, 1.0f) * scale;
        const float dy = acc * d2 * d1;
        P.lat_g[i] = dy;
        if (!isfinite(dy)) atomicAnd(&P.lat_ok[gi], 0);
    }
}

// One Adam step per grid (optim.hpp:38-53) with the per-tensor skip: a grid
// whose gradient has a non-finite element is left untouched.  bc1/bc2 were
// computed per grid by k_finalize from lat_t + 1.  Block 0 / thread 0 also
// advances the step counters (encoder.hpp:129-133).
__global__ void k_adam_latents(const Plan* __restrict__ pp, int g_begin, int g_end) {
    const Plan& P = pp[blockIdx.z];  // batched launches: one plan per image
    CCB_GRID_CACHE(P);
    const double lr = P.scal->lr;
    const double* __restrict__ bc = P.bc_lat;
    const int cost_ok = P.scal->cost_ok;
    const int64_t i_begin = P.g[g_begin].lat_off;
    const int64_t i_end = g_end < P.n_grids ? P.g[g_end].lat_off : P.n_latents;
    if (!cost_ok) {  // encoder.hpp:118 returns before the backward: grads stay zero
        for (int64_t i = i_begin + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < i_end;
             i += int64_t(gridDim.x) * blockDim.x)
            P.lat_g[i] = 0.0f;
        return;
    }
    const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
    for (int64_t i = i_begin + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < i_end;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int gi = find_grid(s_off, i);
        if (!P.lat_ok[gi]) continue;
        const double bc1 = bc[2 * gi], bc2 = bc[2 * gi + 1];
        const double gv = double(P.lat_g[i]);
        const double mt = b1 * double(P.lat_m[i]) + (1.0 - b1) * gv;
        const double vt = b2 * double(P.lat_v[i]) + (1.0 - b2) * gv * gv;
        P.lat_m[i] = float(mt);
        P.lat_v[i] = float(vt);
        P.y[i] = float(double(P.y[i]) - lr * (mt / bc1) / (sqrt(vt / bc2) + eps));
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        for (int gi = g_begin; gi < g_end; ++gi) {
            if (P.lat_ok[gi])
                P.lat_t[gi] += 1;
            else
                atomicAdd(&P.scal->skipped, 1);  // k_nn_step counts concurrently
        }
    }
}

__global__ void k_init_latents(const Plan* __restrict__ pp, uint64_t stream, float amp) {
    const Plan& P = pp[blockIdx.z];  // batched launches: one plan per image
    CCB_GRID_CACHE(P);
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < P.n_latents;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int gi = find_grid(s_off, i);
        const uint64_t gs = hash_combine(stream, uint64_t(gi));
        P.y[i] = counter_uniform(gs, uint64_t(i - P.g[gi].lat_off + int64_t(P.g[gi].row0) * P.g[gi].cols), -amp, amp);
    }
}

// ---------------------------------------------------------------------------
void launch_softq_fwd(const LaunchCtx& L) {
    launch_pdl(k_softq_fwd, dim3(L.elem_blocks, 1, L.batch), dim3(256), 0, L.stream, 's', L.plan);
}
void launch_quantize(const LaunchCtx& L, int amp) {
    k_quantize<<<dim3(L.elem_blocks, 1, L.batch), 256, 0, L.stream>>>(L.plan, amp);
}
void launch_pads_from_q(const LaunchCtx& L) {
    k_pads_from_q<<<dim3(L.elem_blocks, 1, L.batch), 256, 0, L.stream>>>(L.plan);
}
void launch_latent_grad(const LaunchCtx& L) {
    k_latent_grad<<<dim3(L.elem_blocks, 1, L.batch), 256, 0, L.stream>>>(L.plan, 0, 0, L.host->n_latents);
}
void launch_latent_grad_partial(const LaunchCtx& L) {
    k_latent_grad<<<dim3(L.elem_blocks, 1, L.batch), 256, 0, L.stream>>>(L.plan, 1, 0, L.host->n_latents);
}
// grids [g_begin, g_end) only (their latents are contiguous in decode order)
void launch_latent_grad_grids(const LaunchCtx& L, int g_begin, int g_end) {
    const Plan& H = *L.host;
    const int64_t a = H.g[g_begin].lat_off, b = g_end < H.n_grids ? H.g[g_end].lat_off : H.n_latents;
    const int blocks = int(std::max<int64_t>(1, std::min<int64_t>((b - a + 255) / 256, L.elem_blocks)));
    k_latent_grad<<<dim3(blocks, 1, L.batch), 256, 0, L.stream>>>(L.plan, 0, a, b);
}
void launch_adam_latents_grids(const LaunchCtx& L, int g_begin, int g_end) {
    const Plan& H = *L.host;
    const int64_t a = H.g[g_begin].lat_off, b = g_end < H.n_grids ? H.g[g_end].lat_off : H.n_latents;
    const int blocks = int(std::max<int64_t>(1, std::min<int64_t>((b - a + 255) / 256, L.elem_blocks)));
    k_adam_latents<<<dim3(blocks, 1, L.batch), 256, 0, L.stream>>>(L.plan, g_begin, g_end);
}

// Row bands: per-grid finiteness of the OWN rows' (complete) latent gradients,
// the per-tensor check of adam_step (optim.hpp:38-41) restricted to this band.
__global__ void k_ok_reset(const Plan* __restrict__ pp) {
    if (threadIdx.x < kMaxGrids) pp[blockIdx.z].lat_ok[threadIdx.x] = 1;
}
__global__ void k_band_own_finite(const Plan* __restrict__ pp) {
    const Plan& P = pp[blockIdx.z];  // batched launches: one plan per image
    CCB_GRID_CACHE(P);
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < P.n_latents;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int gi = find_grid(s_off, i);
        const GridGeom& g = P.g[gi];
        const int64_t li = i - g.lat_off;
        if (li < int64_t(g.own_lo) * g.cols || li >= int64_t(g.own_hi) * g.cols) continue;
        if (!isfinite(P.lat_g[i])) atomicAnd(&P.lat_ok[gi], 0);
    }
}
void launch_band_own_finite(const LaunchCtx& L) {
    k_ok_reset<<<dim3(1, 1, L.batch), 32, 0, L.stream>>>(L.plan);
    k_band_own_finite<<<dim3(L.elem_blocks, 1, L.batch), 256, 0, L.stream>>>(L.plan);
}
void launch_adam_latents(const LaunchCtx& L) {
    k_adam_latents<<<dim3(L.elem_blocks, 1, L.batch), 256, 0, L.stream>>>(L.plan, 0, L.host->n_grids);
}
void launch_noise_ahead(const LaunchCtx& L) {
    k_noise_ahead<<<dim3(L.elem_blocks, 1, L.batch), 256, 0, L.stream>>>(L.plan);
}
void launch_init_latents(const LaunchCtx& L, uint64_t stream, float amp) {
    k_init_latents<<<dim3(L.elem_blocks, 1, L.batch), 256, 0, L.stream>>>(L.plan, stream, amp);
}

}  // namespace ccb

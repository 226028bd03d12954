// cc_step.cu — per-iteration bookkeeping on the device, so an iteration needs
// no host round trip:
//   k_finalize       bits / mse partials -> cost (encoder.hpp:111-118, 256;
//                    rd_loss encoder.hpp:20-22); Adam bias corrections per
//                    latent grid; snapshot decision (encoder.hpp:151)
//   k_nn_step        fixed-order reduction of every per-CTA weight-gradient
//                    partial into ParamTensor::g, per-tensor finiteness and
//                    Adam (optim.hpp:38-53, NnOptimizer::step optim.hpp:277-286)
//   k_snapshot_copy  Trainer::snapshot for the hardround "best" slot
//                    (encoder.hpp:151,182-189)
#include <cuda_runtime.h>

#include "cc_kernels.h"
#include "cc_math.cuh"
#include "cc_reduce.cuh"

namespace ccb {

namespace {

// one CTA of 256 threads: strided partial sums, then a fixed-order tree
__global__ void __launch_bounds__(256) k_finalize(const Plan* __restrict__ pp, int mode,
                                                  int snap_slot) {
    const Plan& P = pp[blockIdx.z];  // batched launches: one plan per image
    double* bc_lat = P.bc_lat;
    __shared__ double red[8];
    double b_loc = 0.0, s_loc = 0.0;
    for (int b = threadIdx.x; b < P.n_bits_part; b += blockDim.x) b_loc += P.bits_part[b];
    for (int b = threadIdx.x; b < P.n_mse_part; b += blockDim.x) s_loc += P.mse_part[b];
    const double bits_all = block_sum(b_loc, red);
    const double se_all = block_sum(s_loc, red);
    if (mode != kArmProxy)  // proxy iterations reset the flags in k_softq_fwd
        for (int t = threadIdx.x; t < P.n_tensors; t += blockDim.x) P.tensor_ok[t] = 1;
    if (mode == kArmProxy) {  // Adam bias corrections of every latent grid, one thread each
        for (int g = threadIdx.x; g < P.n_grids; g += blockDim.x) {
            const double t = double(P.lat_t[g] + 1);
            bc_lat[2 * g] = 1.0 - pow(0.9, t);
            bc_lat[2 * g + 1] = 1.0 - pow(0.999, t);
        }
    }
    if (threadIdx.x != 0) return;
    const double bits = bits_all, se = se_all;
    const double mse = se / double(3 * P.npix_global);
    const double cost = fma(P.lambda, bits / double(P.npix_global), mse);  // contracted (reference: -ffp-contract=fast)
    DevScalars* s = P.scal;
    s->bits = bits;
    s->mse = mse;
    // once a proxy iteration of a batch came out non-finite, the remaining
    // iterations of the batch take no step and advance no counter (train()
    // restarts from the record of the first bad one, encoder.hpp:365-371)
    const bool halted = mode == kArmProxy && s->halt;
    s->cost = halted ? __longlong_as_double(0x7ff8000000000000LL) : cost;
    s->cost_ok = (!halted && isfinite(cost)) ? 1 : 0;
    if (mode == kArmProxy && !s->cost_ok) s->halt = 1;
    s->snap_take = (snap_slot >= 0 && s->cost_ok && cost < s->snap_cost[snap_slot]) ? 1 : 0;
}

// Wide reduction: one warp per parameter over the whole grid; lanes stride the
// per-CTA partial rows, fixed shuffle tree, regions in index order.  Writes
// ParamTensor::g and clears the tensor's finiteness flag on a non-finite grad.
__global__ void __launch_bounds__(256) k_nn_reduce(const Plan* __restrict__ pp, int p_begin, int p_end) {
    const Plan& P = pp[blockIdx.z];  // batched launches: one plan per image
    int* __restrict__ tensor_ok = P.tensor_ok;
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int p = p_begin + gw; p < p_end; p += nw) {
        double sum = 0.0;
        for (int r = 0; r < P.n_regions; ++r) {
            const PartialRegion& R = P.region[r];
            if (p < R.param_off || p >= R.param_off + R.count) continue;
            const double* col = P.partials + R.base + int64_t(p - R.param_off) * R.nblocks;  // parameter-major
            double s = 0.0;
#pragma unroll 4
            for (int b = lane; b < R.nblocks; b += 32) s += col[b];
            sum += warp_sum(s);
        }
        if (lane == 0) {
            const float g = float(sum);
            P.grads[p] = g;
            P.grads_d[p] = sum;
            if (!isfinite(g)) {
                int ti = 0;
                while (ti + 1 < P.n_tensors && P.tensor_off[ti + 1] <= p) ++ti;
                atomicAnd(&tensor_ok[ti], 0);
            }
        }
    }
}

// One CTA per NN tensor: Adam with the per-tensor skip (optim.hpp:38-41).
__global__ void __launch_bounds__(256) k_nn_step(const Plan* __restrict__ pp, int do_step,
                                                 int count_iter, int log_rec) {
    const Plan& P = pp[blockIdx.z];  // batched launches: one plan per image
    const int* __restrict__ tensor_ok = P.tensor_ok;
    double* __restrict__ cost_log = log_rec ? P.rec : nullptr;
    const double lr = P.scal->lr;
    const int ti = blockIdx.x;
    const int off = P.tensor_off[ti], n = P.tensor_size[ti];
    const bool finite = tensor_ok[ti] != 0;
    DevScalars* s = P.scal;
    if (do_step && s->cost_ok) {
        if (finite) {
            const double t = double(P.nn_t[ti] + 1);
            const double bc1 = 1.0 - pow(0.9, t), bc2 = 1.0 - pow(0.999, t);
            const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
            for (int e = threadIdx.x; e < n; e += blockDim.x) {
                const int p = off + e;
                const double gv = double(P.grads[p]);
                const double mt = b1 * double(P.nn_m[p]) + (1.0 - b1) * gv;
                const double vt = b2 * double(P.nn_v[p]) + (1.0 - b2) * gv * gv;
                P.nn_m[p] = float(mt);
                P.nn_v[p] = float(vt);
                P.params[p] = float(double(P.params[p]) - lr * (mt / bc1) / (sqrt(vt / bc2) + eps));
            }
            if (threadIdx.x == 0) P.nn_t[ti] += 1;
        } else if (threadIdx.x == 0) {
            atomicAdd(&s->skipped, 1);  // integer counter: order-independent
        }
    }
    if (count_iter && ti == 0 && threadIdx.x == 0 && s->cost_ok) s->global_iter += 1;
    if (cost_log && ti == 0 && threadIdx.x == 0) {  // batched runs: per-iteration record
        double* rec = cost_log + 4 * s->sched_pos;
        rec[0] = s->cost;
        rec[1] = s->mse;
        rec[2] = s->bits;
        rec[3] = double(s->global_iter);
        s->sched_pos += 1;
    }
}

// Batched runs: the scalars of iteration sched_pos (lr, temp, noise_std).
__global__ void k_sched_load(const Plan* __restrict__ pp) {
    const Plan& P = pp[blockIdx.z];
    DevScalars* s = P.scal;
    const double* __restrict__ sched = P.sched;
    const double* e = sched + 3 * s->sched_pos;
    s->lr = e[0];
    s->temp = e[1];
    s->noise = e[2];
}

__global__ void k_snapshot_copy(const Plan* __restrict__ pp, int slot, float* __restrict__ sy,
                                float* __restrict__ sp) {
    const Plan& P = pp[blockIdx.z];  // batched launches: one plan per image
    DevScalars* s = P.scal;
    if (!s->snap_take) return;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < P.n_latents;
         i += int64_t(gridDim.x) * blockDim.x)
        sy[i] = P.y[i];
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < P.n_params;
         i += int64_t(gridDim.x) * blockDim.x)
        sp[i] = P.params[i];
    if (blockIdx.x == 0 && threadIdx.x == 0) s->snap_cost[slot] = s->cost;
}

}  // namespace

void launch_finalize(const LaunchCtx& L, int mode, int snap_slot) {
    k_finalize<<<dim3(1, 1, L.batch), 256, 0, L.stream>>>(L.plan, mode, snap_slot);
}

void launch_nn_reduce(const LaunchCtx& L, int p_begin, int p_end) {
    const Plan& H = *L.host;
    if (p_end < 0 || p_end > H.n_params) p_end = H.n_params;
    if (p_end <= p_begin) return;
    const int blocks = (p_end - p_begin + 7) / 8;
    k_nn_reduce<<<dim3(blocks, 1, L.batch), 256, 0, L.stream>>>(L.plan, p_begin, p_end);
}

void launch_nn_apply(const LaunchCtx& L, bool do_step, bool count_iter, bool log_rec) {
    k_nn_step<<<dim3(L.host->n_tensors, 1, L.batch), 256, 0, L.stream>>>(L.plan, do_step ? 1 : 0,
                                                                          count_iter ? 1 : 0, log_rec ? 1 : 0);
}

void launch_nn_step(const LaunchCtx& L, bool do_step, bool count_iter, bool log_rec) {
    launch_nn_reduce(L);
    launch_nn_apply(L, do_step, count_iter, log_rec);
}

void launch_sched_load(const LaunchCtx& L) {
    k_sched_load<<<dim3(1, 1, L.batch), 1, 0, L.stream>>>(L.plan);
}

void launch_snapshot_if_better(const LaunchCtx& L, int slot, float* snap_y, float* snap_p) {
    k_snapshot_copy<<<dim3(L.elem_blocks, 1, L.batch), 256, 0, L.stream>>>(L.plan, slot, snap_y, snap_p);
}

}  // namespace ccb

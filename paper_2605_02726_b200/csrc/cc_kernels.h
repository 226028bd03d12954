// cc_kernels.h — host-side launchers for the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include "cc_plan.h"

#include <vector>

namespace ccb {

void cuda_check(cudaError_t e, const char* what);  // throws CudaError (cc_runtime.cu)
[[noreturn]] void throw_config(const char* what);   // throws ConfigError (cc_runtime.cu)

struct LaunchCtx {
    const Plan* plan;      // device copy
    const Plan* host;      // host copy (same pointers)
    cudaStream_t stream;
    int num_sms;
    int elem_blocks;       // grid for elementwise kernels over the latents
    int pix_blocks;        // grid for per-pixel kernels
    // ARM work table
    const int4* arm_tiles; // (grid, first latent, row, length) per <=128-latent row segment
    int arm_ntiles;
    int arm_blocks;
    int syn_ntiles;        // 128-pixel tiles of the trunk-backward kernel
    int syn_blocks;
    int red_blocks;        // per-CTA partial rows of the small reduction kernels
    int batch = 1;         // images per launch: plan points at `batch` consecutive Plans,
                           // every kernel reads pp[blockIdx.z] (same geometry for all)
    int arm_cslot = -1;    // constant-bank ARM (cc_armc.cuh): the constant slot, -1 = not used
    float* const* arm_cstages = nullptr;  // host array: each image's Plan::arm_cstage (launch time only)
    bool arm_prepped = false;  // launch_arm_prep already packed the weights and filled the slot for image 0
};

// Launch with programmatic stream serialization (see pdl_wait in
// cc_math.cuh); CCB_PDL=0 falls back to plain stream order (A/B).
bool pdl_enabled(char which = 'a');  // which: 'f' upsampling forward, 'b' backward
template <typename... P, typename... A>
inline void launch_pdl(void (*k)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, char which,
                       A... args) {
    cudaLaunchAttribute at[1];
    int na = 0;
    if (pdl_enabled(which)) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = na;
    cuda_check(cudaLaunchKernelEx(&cfg, k, static_cast<P>(args)...), "cudaLaunchKernelEx");
}

enum ArmMode { kArmForward = 0, kArmHard = 1, kArmProxy = 2 };

// latent side (cc_latent.cu)
void launch_softq_fwd(const LaunchCtx& L);
void launch_quantize(const LaunchCtx& L, int amp);
void launch_pads_from_q(const LaunchCtx& L);
void launch_latent_grad(const LaunchCtx& L);
void launch_latent_grad_partial(const LaunchCtx& L);  // row bands: ignore the local cost flag
void launch_band_own_finite(const LaunchCtx& L);
void launch_adam_latents(const LaunchCtx& L);
void launch_latent_grad_grids(const LaunchCtx& L, int g_begin, int g_end);
void launch_adam_latents_grids(const LaunchCtx& L, int g_begin, int g_end);
void launch_init_latents(const LaunchCtx& L, uint64_t stream, float amp);
void launch_noise_ahead(const LaunchCtx& L);

// entropy model (cc_arm.cu)
bool arm_dims_supported(int D, int W);
void arm_padded_dims(int D, int W, int* Dp, int* Wp);
void launch_arm(const LaunchCtx& L, int mode);
// constant-bank ARM: pack the weights and fill the slot for image 0 (returns
// false when the launch context does not use it); launch_arm then skips that
// with LaunchCtx::arm_prepped
bool launch_arm_prep(const LaunchCtx& L);
// IFCE weight gradients from the dF pyramid (Plan::ifce_sep): work items
constexpr int kIfceChunk = 256;  // positions per item (two per thread: latency-bound gathers need many CTAs)
constexpr int kIfceBias = 15;     // item source index of the bias sums
std::vector<int4> ifce_dw_items(const Plan& P, int* item0);
void launch_pyramid(const LaunchCtx& L);
int arm_blocks_per_sm(int Dp, int Wp);
void arm_configure(int Dp, int Wp);
bool arm_uses_v2(int Dp, int Wp);
bool arm_uses_tc(int Dp, int Wp);  // the tensor-core kernel (cc_arm_tc.cu)
void pyramid_configure(const Plan& H);
// constant-bank ARM (cc_armc.cuh, one constant slot per translation unit)
constexpr int kArmcSlots = 8;
constexpr int kArmcSlotFloats = 2560;
constexpr int kArmcPerSm = 4;       // 64-thread CTAs per SM (at most)
bool armc_supported(int Dp, int Wp);
int armc_blocks_per_sm(int Dp, int Wp);
int armc_acquire_slot();             // a free slot, or -1 (then the FFMA2 tile kernel runs)
void armc_release_slot(int slot);
void armc_configure(int Dp, int Wp);

// upsampling (cc_ups.cu)
void launch_ups_forward(const LaunchCtx& L);
void launch_ups_backward(const LaunchCtx& L, bool latent_grads, int j_begin = 0, int j_end = 1 << 30);
int ups_blocks_x(const Plan& H, int j, int num_sms, bool forward);
int ups_coarse_from(const Plan& H);
int ups_chain_ctas();  // CTAs per cascade of the coarse-chain launches
int ups_bwd_tile(const Plan& H, int j, int num_sms);  // backward tile edge of stage j
void ups_configure();

// latent entropy-coding parameters (cc_cdf.cu)
void launch_latent_mu_sigma(const LaunchCtx& L, float* mu, float* sigma);

// synthesis (cc_syn.cu, cc_syn_trunk.cu)
void launch_syn_forward(const LaunchCtx& L, bool backward);
void launch_syn_backward(const LaunchCtx& L, int part = 0);  // 0 all, 1 dz, 2 weight grads
int syn_padded_hidden(int F);
size_t syn_trunk_smem(int FP);
int syn_trunk_blocks_per_sm(int FP);
void syn_configure(int FP);
void syn_post_configure();
void launch_syn_post(const LaunchCtx& L, bool backward);  // cc_syn_post.cu
int syn_post_tiles(int H, int W);

// optimizer / bookkeeping (cc_step.cu)
void launch_finalize(const LaunchCtx& L, int mode, int snap_slot);
void launch_nn_step(const LaunchCtx& L, bool do_step, bool count_iter, bool log_rec);
void launch_nn_reduce(const LaunchCtx& L, int p_begin = 0, int p_end = -1);
void launch_nn_apply(const LaunchCtx& L, bool do_step, bool count_iter, bool log_rec);
void launch_sched_load(const LaunchCtx& L);

// SOAP for the NN parameters (cc_soap.cu)
size_t soap_smem(const Plan& H);
void soap_configure(const Plan& H);
void launch_soap_apply(const LaunchCtx& L, bool do_step, bool count_iter, bool log_rec);
void launch_soap_reset(const LaunchCtx& L);
void launch_snapshot_if_better(const LaunchCtx& L, int slot, float* snap_y, float* snap_p);

}  // namespace ccb

// cc_plan.h — geometry and device-buffer plan shared by the host runtime and
// the sm_100a kernels.  Plain-old-data only: a Plan is passed BY VALUE to every
// kernel (it is ~3 KB, well inside the 32 KB kernel-parameter limit), so
// several trainers can live in one process without sharing __constant__ state.
//
// Layout in HBM (all fp32 unless noted), per image:
//   yhat_pad : every grid (decode order) as a zero-bordered (rows+2P)x(cols+2P)
//              plane — the PaddedGrid values of entropy_model.hpp:153-171; the
//              border is written once at allocation and never touched again.
//   y, m, v, g, th1, th2, gown, dups, q(int32) : flat latent layout (grids in
//              decode order, unpadded row-major) — LatentSet, latent.hpp:30-44.
//   dctx     : the ARM's context gradient dC on its way to the latents it came
//              from, consumed by a deterministic gather (no float atomics).
//              Tiled ARM kernels (ctx_part = 1): per grid, ROW PARTIALS
//              [source row r][d = 0..P][row tile q][T + 2P]: for the targets
//              of source row r that lie d rows up (column c0 - P .. c0 + T + P
//              of tile q), the sum over the context offsets with dy = -d;
//              ~4.2 floats per latent (P = 3) instead of S = 14 planes.
//              Per-latent kernel (ctx_part = 0): S planes (S x rows x cols).
//   dfeat    : per IFCE-equipped grid, F planes of dF plus its 2x2 block-sum
//              pyramid (levels 1..smax), see cc_arm.cu.
//   z, dz    : (L, H, W) dense upsampled latents and their gradient.
//   ups_*    : per main grid k >= 1 and stage j < k, the rowtmp / coltmp / out
//              caches of upsample_forward (synthesis.hpp:40-93).
//   syn_*    : (3, H, W) planes: trunk output t, posts p_i, stab term, dx̂.
//   params/grads/nn_m/nn_v : for_each_param order (model.hpp:158-171).
//   partials : per-CTA weight-gradient partial sums, reduced in a fixed order
//              (parameter-major: the rows of one parameter are contiguous).
#pragma once

#include <stdint.h>

namespace ccb {

constexpr int kMaxGrids = 16;
constexpr int kArmWinCols = 136;  // ARM context window row: a 128-latent tile + 2 x 4 halo columns
constexpr int kMaxLevels = 8;
constexpr int kMaxCtx = 64;
constexpr int kMaxTensors = 64;
constexpr int kMaxSlots = 3;
constexpr int kMaxPartialRegions = 48;
constexpr int kMaxUpsGrids = 8;
constexpr int kArmTile = 128;  // latents per ARM tile == threads per ARM CTA
constexpr int kSynTile = 128;  // pixels per trunk-backward tile == threads per CTA

struct GridGeom {
    int level, hyper, rows, cols;
    int stride;          // padded row stride, cols + 2P
    int ifce_slot;       // -1 when unequipped (model.hpp:72-77)
    int rdim;            // IFCE source count for equipped grids
    int main_level;      // level if main grid, -1 if hyper
    int64_t pad_base;    // offset of element (0,0) inside yhat_pad
    int64_t lat_off;     // offset inside the flat latent layout
    int64_t dctx_off;    // offset of this grid's context-gradient rows / planes inside dctx
    int64_t dfeat_off;   // equipped grids: offset of dF level 0 inside dfeat
    // row bands (cfg5): this grid holds global rows [row0, row0 + rows) of a
    // grid with `grows` rows; local rows [own_lo, own_hi) are owned (rate terms,
    // Adam); the rest is halo.  Whole-image runs: row0 = 0, own = all rows.
    int row0, grows, own_lo, own_hi;
};

// One upsampling stage j for one main grid k (k > j).
struct UpsStage {
    int k;                      // main level of the grid being lifted
    int rows_in, cols_in;       // level j+1 dims
    int rows_out, cols_out;     // level j dims
    int in_stride;              // stride of the stage input
    int64_t in_off;             // stage input: yhat_pad (pad_base) when k == j+1, else ups_out
    int in_is_pad;              // 1: input lives in yhat_pad
    int64_t row_off;            // rowtmp   rows_in  x cols_out  (in ups_buf)
    int64_t col_off;            // coltmp   rows_out x cols_out  (in ups_buf)
    int64_t out_off;            // stage output rows_out x cols_out (ups_buf, or z plane k)
    int out_is_z;               // j == 0: output is z plane k
    int64_t din_off;            // gradient of the stage input (ups_grad), or dups lat_off
    int din_is_lat;             // k == j+1: gradient goes to dups (flat latent layout)
    int64_t dout_off;           // gradient of the stage output (ups_grad), or dz plane k
    int dout_is_z;
};

struct PartialRegion {
    int param_off;   // first flat parameter index covered
    int count;       // number of consecutive parameters
    int nblocks;     // number of per-CTA partial rows
    int64_t base;    // offset of row 0 inside the partials buffer (double)
};

struct Plan {
    // ---- image / config ----
    int H, W, L, hyper, n_grids, P;
    int S, F, D, Wd;          // spatial ctx, ifce dim, ARM input dim, ARM width
    int Dp, Wp;               // padded (instantiated) ARM dims
    int syn_F, posts, use_stab_arm, use_stab_syn;
    int64_t npix, n_latents;
    int n_params, n_tensors;
    float rate_upstream;      // float(lambda / npix), encoder.hpp:64
    double lambda;
    // row bands: pixel rows of the image held here are global rows
    // [pix_row0, pix_row0 + H) of an image with npix_global pixels; rows
    // [pix_own_lo, pix_own_hi) (local) are owned (MSE terms).
    int band, pix_row0, pix_own_lo, pix_own_hi;
    int64_t npix_global;
    int64_t zpix[kMaxLevels];    // z / dz plane k: offset of local pixel (0,0)
    int zvec;                    // npix and all zpix are multiples of 4 (16-byte loads)
    int ctx_part;                // dctx holds row partials (tiled ARM kernels), see above
    int slot_pyr_a[kMaxSlots];   // global row of the dF pyramid origin (aligned)
    uint64_t seed;

    int ctx_dy[kMaxCtx], ctx_dx[kMaxCtx];
    GridGeom g[kMaxGrids];
    int main_gi[kMaxLevels];  // decode index of main grid k
    int slot_gi[kMaxSlots];   // decode index of the grid equipped with IFCE slot s
    int n_slots;
    int slot_smax[kMaxSlots]; // deepest pyramid level needed for slot s
    int64_t slot_pyr_off[kMaxSlots][kMaxLevels + 1];  // dfeat offsets of level l
    int slot_pyr_rows[kMaxSlots][kMaxLevels + 1];
    int slot_pyr_cols[kMaxSlots][kMaxLevels + 1];

    // ---- parameter arena offsets (for_each_param order) ----
    int off_l1w, off_l1b, off_l2w, off_l2b, off_hw, off_hb, off_astab;  // astab -1 if none
    int off_ifw[kMaxSlots], off_ifb[kMaxSlots];
    int off_tconv[kMaxLevels], off_refine[kMaxLevels];
    int off_c1w, off_c1b, off_c2w, off_c2b;
    int off_pw[2], off_pb[2];
    int off_sstab;  // -1 if none
    int tensor_off[kMaxTensors], tensor_size[kMaxTensors];
    int tensor_rows[kMaxTensors], tensor_cols[kMaxTensors];  // MatView::of shape
    // SOAP (use_soap): per tensor L (r x r), R (c x c), QL, QR in fp64
    int use_soap, soap_dmax, soap_nmax;
    int64_t soap_off[kMaxTensors];

    // ---- partial regions ----
    int n_regions;
    PartialRegion region[kMaxPartialRegions];
    int reg_arm;              // region index of the ARM kernel (ARM + IFCE params)
    int ifce_sep;             // IFCE weight gradients from k_ifce_dw (constant-bank ARM); the ARM kernels write zeros
    int reg_ifce[kMaxSlots];  // its regions (one per IFCE slot): one row per work item of the slot
    int n_ifce_items;         // k_ifce_dw work items (slot, source j or kIfceBias, first, end position)
    int ifce_item0[kMaxSlots];  // first item of each slot (row 0 of its region)
    const int4* ifce_items;
    int reg_syn_trunk;        // syn c1,c2,stab
    int reg_post[2];          // syn post i (w + b)
    int reg_ups_rows[kMaxLevels], reg_ups_cols[kMaxLevels], reg_ups_ref[kMaxLevels];
    int arm_nvals;            // values per ARM partial row
    int syn_nvals;

    // ---- upsampling stages: stage j -> list of (grid) stages ----
    int ups_n[kMaxLevels];
    int ups_jc;               // stages j >= ups_jc run fused, one CTA per cascade
    UpsStage ups[kMaxLevels][kMaxUpsGrids];

    // ---- device buffers ----
    float* yhat_pad;
    const void* pad_maps;     // CUtensorMap[kMaxGrids]: TMA descriptors of the padded grids
    float* y;
    float* lat_m;
    float* lat_v;
    float* lat_g;
    float* th1;
    float* th2;
    float* gown;
    float* dups;
    int32_t* q;
    float* dctx;
    float* dfeat;
    float* z;
    float* dz;
    float* ups_buf;
    float* ups_grad;
    float* ups_grad2;
    float* image;
    float* arm_cstage;        // constant-bank ARM: this image's padded weight image (cc_armc.cuh)
    float* syn_t;
    float* syn_p[2];
    float* syn_sz;
    float* syn_dx;
    float* syn_dt;
    float* syn_dtmp;
    float* params;
    float* grads;
    double* grads_d;          // the same gradients before rounding (band reduction)
    double* soap;             // SOAP preconditioners / eigenbases (use_soap)
    float* noise_buf;         // unit Gaussians drawn ahead for scal->noise_iter
    double* post_scratch;     // k_syn_post2 fp64 dW slots (large images), zeroed per iteration
    float* nn_m;
    float* nn_v;
    double* partials;
    double* bc_lat;           // per grid Adam bias corrections (2 per grid)
    double* bits_part;
    double* mse_part;
    int n_bits_part, n_mse_part;
    int64_t* lat_t;           // per grid
    int64_t* nn_t;            // per tensor
    int* lat_ok;              // per grid: grads finite
    int* tensor_ok;           // per NN tensor: grads finite
    const double* sched;      // batched runs: (lr, temp, noise_std) per iteration
    double* rec;              // batched runs: (cost, mse, bits, global_iter) per iteration (mapped host)
    // device scalars (see DevScalars)
    struct DevScalars* scal;
};

struct DevScalars {
    double cost, mse, bits;   // last finalized iteration (encoder.hpp:115-117)
    double lr, temp, noise;   // scalars of the running iteration
    int cost_ok;              // isfinite(cost)
    int skipped;              // skipped_steps (encoder.hpp:72)
    int snap_take;            // hardround: take the pre-step snapshot
    int halt;                 // set by a non-finite proxy cost: the rest of the batch are no-ops
    int64_t global_iter;      // encoder.hpp:71; keys the noise stream
    int64_t sched_pos;        // batched runs: index into the schedule arrays
    int64_t noise_iter;       // global_iter the noise_buf values belong to (-1: none)
    double snap_cost[8];      // per snapshot slot
};

}  // namespace ccb

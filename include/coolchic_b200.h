/*
 * coolchic_b200.h — C ABI of the B200-native Cool-chic 5.0 encode iteration.
 *
 * The reference (arXiv 2605.02726, /root/reference/proj/include/coolcodec) is a
 * header-only C++20 library with no FFI; its per-iteration driver is the class
 * coolcodec::detail::Trainer (encoder.hpp:59-306) and its callers warmup()
 * (encoder.hpp:315-342) and train() (encoder.hpp:349-413).  Every entry point
 * below replaces one member of that surface; the reference line it stands in
 * for is cited on each declaration.  Three libraries export this exact symbol
 * set, so tests drive them interchangeably:
 *
 *   paper_2605_02726_b200/libcoolchic_b200.so   sm_100a kernels (the product)
 *   oracle/_ref/libccref.so                     the reference headers compiled
 *                                               behind this ABI (checker only)
 *   oracle/libccport.so                         plain-C restatement (checker only)
 *
 * Conventions (mirroring tensor.hpp:11-25 / encoder.hpp:118,129-133):
 *   - every function returns CC_OK or an error code; cc_last_error() returns a
 *     thread-local message for the last failure on the calling thread;
 *   - CC_ERR_CONFIG  <-> coolcodec::ConfigError, CC_ERR_FORMAT <-> FormatError,
 *     CC_ERR_TRAINING <-> TrainingError, CC_ERR_CUDA = device/runtime failure;
 *   - a non-finite RD cost is RETURNED through *cost (CC_OK), never an error,
 *     exactly like proxy_iteration (encoder.hpp:118): no optimizer step is taken
 *     and global_iter is not advanced;
 *   - host buffers are borrowed for the duration of the call only;
 *   - a trainer is single-threaded; distinct trainers are independent.
 *
 * Flat layouts used by the state/gradient transfer calls:
 *   latents : every grid in decode order (LatentSet::grids, latent.hpp:46-70),
 *             each unpadded row-major rows x cols, concatenated (n_latents);
 *   params  : every tensor in for_each_param order (model.hpp:158-171),
 *             concatenated (n_params);
 *   Adam    : m/v with the same layout as the tensor they belong to, plus one
 *             int64 step counter t per tensor (optim.hpp:21-29).
 */
#ifndef COOLCHIC_B200_H
#define COOLCHIC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CC_OK 0
#define CC_ERR_CONFIG 1
#define CC_ERR_FORMAT 2
#define CC_ERR_TRAINING 3
#define CC_ERR_CUDA 4
#define CC_ERR_STATE 5

/* DecoderConfig (config.hpp:40-81).  Presets: "lop", "mop", "hop", "vhop". */
typedef struct cc_decoder_config {
    int preset; /* 0 lop, 1 mop, 2 hop, 3 vhop (name only) */
    int spatial_ctx;
    int ifce_dim;
    int arm_width;
    int arm_hidden;
    int synth_hidden;
    int synth_posts;
    int use_hyperlatents;
    int use_stabilizer;
} cc_decoder_config;

/* EncoderConfig (config.hpp:93-142). */
typedef struct cc_encoder_config {
    int warmup_candidates;
    int warmup_keep;
    int warmup_iters;
    int main_iters;
    int hardround_iters;
    double lr_start, lr_end;
    double noise_std_start, noise_std_end;
    double temp_start, temp_end;
    double hardround_lr;
    double lambda;
    uint64_t seed;
    int use_soap;           /* 1 (reference default, config.hpp:107): SOAP on the NN params; 0: Adam */
    int true_cost_interval;
    const char* log_path;   /* optional per-iteration CSV, NULL/"" = off */
} cc_encoder_config;

typedef struct cc_layout {
    int height, width;
    int levels;        /* L, latent_levels() config.hpp:84 */
    int hyper_count;
    int n_grids;
    int64_t n_latents;
    int n_tensors;
    int64_t n_params;
    int pad;           /* PaddedGrid border, max(1, ctx.pad) encoder.hpp:218 */
} cc_layout;

typedef struct cc_grid_info {
    int level, hyper, rows, cols;
    int64_t offset;    /* into the flat latent layout */
    int ifce_slot;     /* model.hpp:72-77 (-1 = none) */
} cc_grid_info;

typedef struct cc_param_info {
    char name[32];
    int rows, cols;    /* MatView::of (tensor.hpp:74-78) */
    int64_t size;
    int64_t offset;    /* into the flat parameter layout */
} cc_param_info;

/* TrainStats (encoder.hpp:24-32). */
typedef struct cc_train_stats {
    int64_t iterations;
    double true_cost;
    double psnr;
    double rate_bpp;
    int restarts;
    int skipped_steps;
    double seconds;
} cc_train_stats;

typedef struct cc_trainer cc_trainer;

/* Thread-local description of the last failing call on this thread. */
const char* cc_last_error(void);
/* Implementation tag: "b200", "reference" or "port". */
const char* cc_impl_name(void);

/* DecoderConfig::from_name (config.hpp:66-72). */
int cc_decoder_config_preset(const char* name, cc_decoder_config* out);
/* EncoderConfig{} defaults (config.hpp:93-109). */
int cc_encoder_config_default(cc_encoder_config* out);
/* EncoderConfig::with_total (config.hpp:127-141). */
int cc_encoder_config_with_total(int total, cc_encoder_config* out);
/* count_macs_per_pixel (synthesis.hpp:239-277): the FLOP convention. */
double cc_count_macs_per_pixel(const cc_decoder_config* cfg, int h, int w);

/* Seeded synthetic RGB test image, planar (3,h,w) fp32 in [0,1]
 * (BASELINE.json configs; SURVEY.md 8(d) "synthetic inputs"). */
int cc_make_synthetic_image(int h, int w, uint64_t seed, float* out);

/* detail::Trainer(const Image&, const EncoderConfig&, const DecoderConfig&)
 * (encoder.hpp:61-67).  The image (planar (3,h,w) fp32) is copied to the
 * device; `device` selects the CUDA device (ignored by CPU checkers). */
int cc_trainer_create(const float* image, int h, int w, const cc_encoder_config* enc,
                      const cc_decoder_config* dec, int device, cc_trainer** out);
void cc_trainer_destroy(cc_trainer* tr);
/* Replace the target image (same shape); host buffer, synchronous copy. */
int cc_trainer_upload_image(cc_trainer* tr, const float* image);

int cc_trainer_layout(cc_trainer* tr, cc_layout* out);
int cc_trainer_grid_info(cc_trainer* tr, int gi, cc_grid_info* out);
int cc_trainer_param_info(cc_trainer* tr, int ti, cc_param_info* out);

/* Trainer::fresh_candidate (encoder.hpp:82-93). */
int cc_trainer_fresh_candidate(cc_trainer* tr, int index);

/* Lock-step state transfer (CandidateState, encoder.hpp:42-48).  Any pointer
 * may be NULL to leave/skip that part.  lat_t has n_grids entries, nn_t has
 * n_tensors entries. */
int cc_trainer_set_state(cc_trainer* tr, const float* latents, const float* params,
                         const float* lat_m, const float* lat_v, const int64_t* lat_t,
                         const float* nn_m, const float* nn_v, const int64_t* nn_t);
int cc_trainer_get_state(cc_trainer* tr, float* latents, float* params, float* lat_m,
                         float* lat_v, int64_t* lat_t, float* nn_m, float* nn_v,
                         int64_t* nn_t);
/* Gradients of the last iteration (y.g per grid, ParamTensor::g per tensor);
 * they stay readable until the next iteration (encoder.hpp:99). */
int cc_trainer_get_grads(cc_trainer* tr, float* latent_grads, float* param_grads);
/* Quantized latents q (LatentGrid::q, latent.hpp:21), flat latent layout. */
int cc_trainer_get_q(cc_trainer* tr, int32_t* q);

/* Public fields global_iter / skipped_steps (encoder.hpp:71-72). */
int cc_trainer_get_counters(cc_trainer* tr, int64_t* global_iter, int* skipped_steps);
int cc_trainer_set_counters(cc_trainer* tr, int64_t global_iter, int skipped_steps);

/* Trainer::proxy_iteration(lr, temp, noise_std) (encoder.hpp:97-135). */
int cc_trainer_proxy_iteration(cc_trainer* tr, double lr, double temp, double noise_std,
                               double* cost);
/* n back-to-back proxy iterations without a host round trip in between; costs
 * (may be NULL) receives the n per-iteration costs.  After a non-finite cost
 * the remaining iterations are not run and their costs are NaN; the number of
 * iterations actually attempted is returned through *ran (may be NULL). */
int cc_trainer_proxy_iterations(cc_trainer* tr, int n, const double* lr, const double* temp,
                                const double* noise_std, double* costs, int* ran);
/* Trainer::hardround_iteration(lr, best) (encoder.hpp:141-155).  With
 * best_slot >= 0 the snapshot slot is replaced by the pre-step state when the
 * cost improves on the slot's cost. */
int cc_trainer_hardround_iteration(cc_trainer* tr, double lr, int best_slot, double* cost);
/* Trainer::true_cost(psnr*, bpp*) (encoder.hpp:158-168); psnr/bpp may be NULL. */
int cc_trainer_true_cost(cc_trainer* tr, double* cost, double* psnr, double* bpp);
/* quantize_all(current().lat) (latent.hpp:97-99). */
int cc_trainer_quantize_all(cc_trainer* tr);
/* Trainer::load_pads_from_q (encoder.hpp:170-180). */
int cc_trainer_load_pads_from_q(cc_trainer* tr);
/* last_mse()/last_bits() (encoder.hpp:209-210). */
int cc_trainer_last_terms(cc_trainer* tr, double* mse, double* bits);

/* Snapshot / restore / reset_optimizers (encoder.hpp:182-199).  Snapshots
 * live in numbered slots owned by the trainer. */
int cc_trainer_snapshot(cc_trainer* tr, int slot, double cost);
int cc_trainer_snapshot_cost(cc_trainer* tr, int slot, double* cost);
int cc_trainer_restore(cc_trainer* tr, int slot);
int cc_trainer_reset_optimizers(cc_trainer* tr);

/* take_candidate / load_candidate (encoder.hpp:74-80): the whole
 * CandidateState (latents, model, optimizer states, cost) moves to / from a
 * numbered candidate slot. */
int cc_trainer_take_candidate(cc_trainer* tr, int slot, double cost);
int cc_trainer_load_candidate(cc_trainer* tr, int slot);
int cc_trainer_candidate_cost(cc_trainer* tr, int slot, double* cost);

/* ---- asynchronous use (no reference counterpart; the reference is a
 * synchronous CPU library).  Launch on the caller's CUDA stream (a
 * cudaStream_t passed as void*; NULL = the trainer's own stream), enqueue n
 * proxy iterations without waiting, and wait for them.  Costs of enqueued
 * iterations are readable with cc_trainer_last_records after synchronize. */
int cc_trainer_set_stream(cc_trainer* tr, void* cuda_stream);
int cc_trainer_enqueue_proxy_iterations(cc_trainer* tr, int n, const double* lr,
                                        const double* temp, const double* noise_std);
/* size the batch buffers for n enqueued iterations and instantiate the batched
 * iteration graph now, so later enqueues of up to n iterations do no setup. */
int cc_trainer_reserve_iterations(cc_trainer* tr, int n);
int cc_trainer_synchronize(cc_trainer* tr);
/* records of the last batched run: 4 doubles per iteration
 * (cost, mse, bits, global_iter after the iteration). */
int cc_trainer_last_records(cc_trainer* tr, int n, double* rec);

/* warmup(tr, enc) + load_candidate (encoder.hpp:315-342, 352). */
int cc_trainer_warmup(cc_trainer* tr);
/* train(img, enc, dcfg) (encoder.hpp:349-413) on an existing trainer (image
 * already uploaded).  Outputs (may be NULL): stats; final latents y, q and
 * params in the flat layouts. */
int cc_trainer_train(cc_trainer* tr, cc_train_stats* stats, float* latents, int32_t* q,
                     float* params);

#ifdef __cplusplus
}
#endif

#endif /* COOLCHIC_B200_H */

/*
 * coolchic_b200_diag.h — measurement hooks of the B200 library (used by
 * bench.py and the profiling notes; not part of the reference surface).
 */
#ifndef COOLCHIC_B200_DIAG_H
#define COOLCHIC_B200_DIAG_H

#include "coolchic_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

#define CCB_NUM_STAGES 8
/* Stage names, in launch order of one proxy iteration:
 * 0 softq_fwd, 1 arm (fused ARM+IFCE fwd/bwd), 2 pyramid, 3 ups_fwd,
 * 4 syn_fwd, 5 syn_bwd, 6 ups_bwd, 7 tail (finalize, gather, Adam). */
const char* ccb_stage_name(int stage);

/* Run n proxy iterations (lr/temp/noise fixed) WITHOUT the graph, with CUDA
 * events between stages on the trainer's stream; ms[s] receives the average
 * duration of stage s per iteration. */
int ccb_profile_stages(cc_trainer* tr, int n, double lr, double temp, double noise, double* ms);

/* Number of kernel nodes in one captured proxy iteration (graph). */
int ccb_kernels_per_iteration(cc_trainer* tr, int* count);

/* Algorithmic FLOPs of one launch of the fused ARM kernel (proxy mode):
 * 6 x (ARM + IFCE MACs of count_macs_per_pixel) x npix, SURVEY 8(d). */
double ccb_arm_flops(cc_trainer* tr);

/* FP32 FFMA peak of `device` measured by a register-only FMA kernel
 * (TFLOP/s, 2 flops per FMA), ms = device time of the measurement. */
int ccb_fp32_peak(int device, double* tflops, double* ms);

/* Device evaluation of the parity-critical element functions on n inputs:
 * fn 0 cc_exp(a), 1 cc_log(a), 2 cc_tanh(a), 3 softround_value(a, T=b),
 * 4 laplace_bits(a, mu=b, sigma=c), 5 quantize_value(a, 255),
 * 6 softround derivative at (a, T=b).  b/c may be NULL (zeros). */
int ccb_eval_math(int fn, int n, const float* a, const float* b, const float* c, float* out);
/* counter_gauss(stream, idx0 + i) for i < n, on the device. */
int ccb_counter_gauss(uint64_t stream, uint64_t idx0, int n, float* out);
/* SOAP state of a use_soap trainer (tests): *n_arena doubles of per-tensor
 * L, R, QL, QR (for_each_param order, row-major, L r x r, R c x c) into arena,
 * the moments m1 / v2 (fp32, n_params) and the step counters (n_tensors).
 * Any output may be NULL. */
/* Event timeline of one proxy iteration (graph with event marks, mean over n
 * replays): ms[13] = time after the start of mark k (see cc_runtime.cu
 * Trainer::enqueue_proxy; 0 = start). */
int ccb_timeline(cc_trainer* tr, int n, double lr, double temp, double noise, double* ms);
int ccb_soap_state(cc_trainer* tr, double* arena, float* m1, float* v2, int64_t* t, int64_t* n_arena);
/* Load a SOAP state in the same layout (teacher-forced lock-step against the
 * reference's soap_step, optim.hpp:189-254).  Any input may be NULL. */
int ccb_soap_set_state(cc_trainer* tr, const double* arena, const float* m1, const float* v2,
                       const int64_t* t);
/* Host waits on the device the library has issued so far in this process
 * (stream / event synchronisations): the band iteration's sync budget. */
int ccb_host_sync_count(int64_t* n);

#ifdef __cplusplus
}
#endif

#endif /* COOLCHIC_B200_DIAG_H */

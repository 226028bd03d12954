/* coolchic_b200_band.h — row-band decomposition of one large image across
 * ranks (BASELINE config 5).  No reference counterpart: the
 * reference encodes one image in one process (encoder.hpp:59-306).  These
 * entry points expose the three phases of one proxy_iteration
 * (encoder.hpp:97-135) around the exchange steps a multi-rank driver
 * performs (paper_2605_02726_b200/bands.py):
 *
 *   rank b owns full-resolution rows [r0, r1) (multiples of 2^(L-1)); every
 *   latent grid holds its own rows plus `halo` rows per side (clipped at the
 *   image border).  Per iteration:
 *     1. halo rows of the latents y are refreshed from their owners;
 *     2. cc_band_forward_backward: forward + backward on the band; rate and
 *        distortion terms of OWN rows only; returns this band's bits and
 *        squared-error sums; latent gradients of halo rows are partial;
 *     3. exchange: halo-row latent gradients are added into their owners'
 *        rows; NN-gradient partial sums (cc_band_nn_partial) and the bits /
 *        squared-error sums are summed over ranks in rank order;
 *     4. cc_band_finish: global gradients + cost; returns the per-grid
 *        finiteness of the own rows; the driver ANDs it over ranks;
 *     5. cc_band_step: Adam on latents and NN parameters.
 *
 * Same error conventions as coolchic_b200.h (CC_OK / CC_ERR_*). */
#ifndef COOLCHIC_B200_BAND_H
#define COOLCHIC_B200_BAND_H

#include "coolchic_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Pixel rows [*w0, *w1) of the image a band trainer for rows [r0, r1) holds. */
int cc_band_window(int h, int w, int r0, int r1, int halo, int* w0, int* w1);

/* A trainer for rows [r0, r1) of an h x w image; image_window = the planar
 * RGB rows [w0, w1) from cc_band_window. */
int cc_band_trainer_create(const float* image_window, int h, int w, int r0, int r1, int halo,
                           const cc_encoder_config* enc, const cc_decoder_config* dec, int device,
                           cc_trainer** out);

/* Global rows of grid gi (decode order): out4 = {window begin, own begin,
 * own end, window end}. */
int cc_band_grid_rows(cc_trainer* tr, int gi, int* out4);

/* Global rows [rb, re) of grid gi, flat row-major: which 0 = latents y,
 * 1 = latent gradients; mode 0 = read into buf, 1 = write from buf,
 * 2 = add buf. */
int cc_band_rows(cc_trainer* tr, int which, int gi, int rb, int re, float* buf, int mode);

/* Device views for a collective library (NCCL): the device address of global
 * rows [rb, re) of grid gi (which 0 = latents, 1 = latent gradients; fp32,
 * contiguous) and of the fp64 NN-gradient partial sums.  Valid until the
 * trainer is destroyed; the trainer's own work is complete when
 * cc_band_forward_backward / cc_band_step return. */
int cc_band_device_rows(cc_trainer* tr, int which, int gi, int rb, int re, void** dptr, int64_t* count);
int cc_band_device_nn_partial(cc_trainer* tr, void** dptr, int64_t* count);

int cc_band_forward_backward(cc_trainer* tr, double lr, double temp, double noise_std,
                             double* bits, double* sq_err);
/* this band's NN-gradient partial sums (fp64, for_each_param order) */
int cc_band_nn_partial(cc_trainer* tr, double* out);
/* global NN-gradient sums and bits / squared-error sums -> cost; lat_ok_own
 * receives one flag per grid (own rows finite). */
int cc_band_finish(cc_trainer* tr, const double* nn_sums, double bits, double sq_err,
                   double* cost, int* lat_ok_own);
/* Adam steps with the per-grid finiteness ANDed over ranks. */
int cc_band_step(cc_trainer* tr, const int* lat_ok);

/* ---- device-resident band iteration (csrc/cc_band.h) ----------------------
 * The same iteration with the exchange inside the library, on the band
 * trainers' streams: a run of n proxy iterations is enqueued without any host
 * synchronisation; each band trainer keeps the per-iteration records
 * (cc_trainer_last_records: cost, mse, bits, global_iter — identical on every
 * band).  Results are bit-identical to the host-driven phases above.
 *
 *   local group: every band of the image in this process (trainers on one
 *                GPU or several), ordered by events between their streams;
 *   NCCL group:  one band per process; `nccl_id` (128 bytes) comes from
 *                cc_band_nccl_unique_id on one rank and is shared by the
 *                caller (e.g. torch.distributed.broadcast_object_list);
 *                `edges` = the nranks+1 band row edges (edges[r], edges[r+1]
 *                = rank r's rows).  libnccl.so.2 is resolved at run time. */
typedef struct cc_band_group cc_band_group;
int cc_band_group_local(cc_trainer* const* bands, int nbands, cc_band_group** out);
int cc_band_nccl_unique_id(void* id128);
int cc_band_group_nccl(cc_trainer* band, const void* id128, int nranks, int rank, const int* edges,
                       cc_band_group** out);
/* buffers for up to n iterations per enqueue (optional: enqueue grows them) */
int cc_band_group_reserve(cc_band_group* g, int n);
/* n proxy iterations with per-iteration (lr, temp, noise_std); returns
 * without waiting for the device */
int cc_band_group_enqueue_proxy_iterations(cc_band_group* g, int n, const double* lr,
                                           const double* temp, const double* noise_std);
int cc_band_group_synchronize(cc_band_group* g);
int cc_band_group_destroy(cc_band_group* g);

#ifdef __cplusplus
}
#endif

#endif /* COOLCHIC_B200_BAND_H */

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

#ifdef __cplusplus
}
#endif

#endif /* COOLCHIC_B200_BAND_H */

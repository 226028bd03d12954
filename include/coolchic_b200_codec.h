/* coolchic_b200_codec.h — forward-only decode passes on the device, the step
 * right after the encode loop: the network-parameter
 * quantisation search select_nn_coding (nn_coding.hpp:146-224) evaluates
 * 4 submodules x 64 (Delta_w, Delta_b) candidates, each one
 *   latent_rate_estimate(lat, m, ctx)           (decode_core.hpp:38-44)  or
 *   mse_rgb(reconstruct_image(lat, m), x)       (decode_core.hpp:47-63, image.hpp:31-34)
 * on the quantised latents with the candidate parameters substituted.
 * Implemented by the product and by the reference checker (oracle/_ref);
 * same error conventions as coolchic_b200.h. */
#ifndef COOLCHIC_B200_CODEC_H
#define COOLCHIC_B200_CODEC_H

#include "coolchic_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Replace the trainer's quantised latents (flat layout, int32) — e.g. after
 * encode_image's amplitude clamp (bitstream.hpp:194-197). */
int cc_trainer_set_q(cc_trainer* tr, const int32_t* q);

/* One forward-only evaluation on the current quantised latents with params
 * (for_each_param order; NULL = the trainer's own) substituted for this call:
 * which & 1 -> *rate_bits = latent_rate_estimate; which & 2 -> *mse =
 * mse_rgb(reconstruct_image, image).  The trainer's parameters are unchanged. */
int cc_trainer_decode_terms(cc_trainer* tr, const float* params, int which, double* rate_bits,
                            double* mse);

/* The Laplace parameters of every quantised latent as encode_latents computes
 * them (bitstream.hpp:106-141: causal context of q, IFCE features,
 * arm_forward_single, entropy_model.hpp:107-134), flat layout, with params
 * (for_each_param order; NULL = the trainer's own) substituted.  Bit-identical
 * to the reference's scalar evaluation, so the reference decoder rebuilds the
 * same CDFs.  mu / sigma: n_latents floats each. */
int cc_trainer_latent_mu_sigma(cc_trainer* tr, const float* params, float* mu, float* sigma);

#ifdef __cplusplus
}
#endif

#endif /* COOLCHIC_B200_CODEC_H */

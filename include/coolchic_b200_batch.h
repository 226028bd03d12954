/* coolchic_b200_batch.h — several images of one size trained in lock-step by
 * one set of kernel launches per stage (BASELINE config 3: 24 independent
 * 512x768 images, sharded across GPUs and batched within each).
 *
 * Reference counterpart: the reference has no batched trainer; its only
 * multi-image mode is independent encodes on a thread pool
 * (tools/coolcodec.cpp:150-171, one detail::Trainer per image,
 * encoder.hpp:59-306).  Each trainer in a batch stays a complete
 * detail::Trainer equivalent (own latents, model, optimiser state, counters,
 * records, snapshots): the batch only changes how its proxy iterations
 * (encoder.hpp:97-135) are launched — every kernel of the iteration graph runs
 * once for all images, blockIdx.z selecting the image.  Results per image are
 * identical to running the trainer alone (tests/test_batch.py).
 *
 * Same error conventions as coolchic_b200.h (CC_OK / CC_ERR_*). */
#ifndef COOLCHIC_B200_BATCH_H
#define COOLCHIC_B200_BATCH_H

#include "coolchic_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cc_batch cc_batch;

/* n trainers (borrowed; they must outlive the batch) of the same device, image
 * size, decoder and optimizer, each with a candidate loaded.  They are moved
 * onto the first trainer's CUDA stream until cc_batch_destroy, which moves
 * them back onto their own streams. */
int cc_batch_create(cc_trainer* const* trainers, int n, cc_batch** out);
void cc_batch_destroy(cc_batch* b);
/* size every trainer's record buffer for n iterations and instantiate the
 * batched iteration graph (one-off setup, outside any timed region). */
int cc_batch_reserve_iterations(cc_batch* b, int n);
/* enqueue n proxy iterations of every image with the same schedule; each
 * trainer's records are readable with cc_trainer_last_records after
 * cc_batch_synchronize. */
int cc_batch_enqueue_proxy_iterations(cc_batch* b, int n, const double* lr, const double* temp,
                                      const double* noise_std);
int cc_batch_synchronize(cc_batch* b);

#ifdef __cplusplus
}
#endif

#endif /* COOLCHIC_B200_BATCH_H */

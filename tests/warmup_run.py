"""Helper of tests/test_batch.py::test_batched_warmup_is_the_sequential_warmup:
a full train() (warm-up, main stage, hardround) whose final state is saved;
run in a subprocess so that CCB_WARMUP_SERIAL (read once per process) can
select the sequential warm-up."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main(out: str, soap: int) -> None:
    from paper_2605_02726_b200 import capi
    from paper_2605_02726_b200.trainer import DecoderConfig, EncoderConfig, Trainer, make_synthetic_image

    lib = capi.load_product()
    img = make_synthetic_image(64, 96, 4, lib)
    enc = EncoderConfig.with_total(1500)
    enc.lmbda, enc.seed, enc.use_soap, enc.true_cost_interval = 1e-3, 7, bool(soap), 200
    with Trainer(img, enc, DecoderConfig.hop(), lib=lib) as tr:
        r = tr.train()
    np.savez(out, lat=r.latents, q=r.q, par=r.params,
             stats=np.array([r.stats.iterations, r.stats.true_cost, r.stats.psnr, r.stats.rate_bpp,
                             r.stats.restarts, r.stats.skipped_steps], np.float64))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))

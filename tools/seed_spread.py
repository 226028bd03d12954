"""Full with_total(10000) encodes of BASELINE config 2 (512x768 HOP, image
seed 0) for encoder seeds 0..4 on the device: the final true RD cost per
seed (compare with tests/golden/train_cfg2*.json from the reference)."""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_02726_b200 import capi  # noqa: E402
from paper_2605_02726_b200.trainer import DecoderConfig, EncoderConfig, Trainer, make_synthetic_image  # noqa: E402

lib = capi.load_product()
img = make_synthetic_image(512, 768, 0, lib)
out = {}
for seed in range(5):
    enc = EncoderConfig.with_total(10000)
    enc.lmbda, enc.seed, enc.use_soap = 1e-3, seed, False
    with Trainer(img, enc, DecoderConfig.hop(), lib=lib) as tr:
        r = tr.train()
    out[seed] = r.stats.true_cost
    print(seed, r.stats.true_cost, r.stats.psnr, r.stats.rate_bpp, flush=True)
print(json.dumps(out))

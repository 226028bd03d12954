"""The reference built for x86-64-v3 vs x86-64-v4 on the same quantised latents:
fraction of latents whose encode_latents (mu, sigma) differ (CPU only)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_02726_b200 import capi
from paper_2605_02726_b200.trainer import DecoderConfig, EncoderConfig, Trainer
from tests.oracle_util import REF_DIR
from tests.conftest import make_image
l3 = capi.load_library(REF_DIR / "libccref_v3.so"); l4 = capi.load_library(REF_DIR / "libccref_v4.so")
img = make_image(l3, 64, 96, seed=7)
enc, dcfg = EncoderConfig(use_soap=False, lmbda=1e-3, seed=3), DecoderConfig.hop()
with Trainer(img, enc, dcfg, lib=l3) as t3, Trainer(img, enc, dcfg, lib=l4) as t4:
    t3.fresh_candidate(0)
    for _ in range(5): t3.proxy_iteration(1e-2, 0.35, 0.22)
    st = t3.get_state(); t4.fresh_candidate(0); t4.set_state(st)
    t3.quantize_all(); q = np.clip(t3.get_q(), -7, 7); t3.set_q(q); t4.set_q(q)
    m3, s3 = t3.latent_mu_sigma(); m4, s4 = t4.latent_mu_sigma()
    print("v3 vs v4 mu mismatch frac", np.mean(m3 != m4), "sigma", np.mean(s3 != s4))

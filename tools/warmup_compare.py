"""Warm-up winner check at BASELINE config 2 (512x768 HOP, with_total(10000),
seed 0): the reference's warmup (encoder.hpp:315-342) vs the device's.
    python tools/warmup_compare.py ref  -> gpurun_out/warm_ref.npz (CPU, ~4 min)
    python tools/warmup_compare.py gpu  -> compares against warm_ref.npz"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_02726_b200 import capi  # noqa: E402
from paper_2605_02726_b200.trainer import DecoderConfig, EncoderConfig, Trainer  # noqa: E402

REPO = Path(__file__).resolve().parents[1]
OUT = REPO / "tests" / "golden" / "warm_cfg2.npz"

mode = sys.argv[1]
if mode == "ref":
    from tests.oracle_util import load_reference
    lib = load_reference()
else:
    lib = capi.load_product()
img = np.empty((3, 512, 768), np.float32)
lib.cc_make_synthetic_image(512, 768, 0, img.ctypes.data_as(capi._F))
enc = EncoderConfig.with_total(10000)
enc.lmbda, enc.seed, enc.use_soap = 1e-3, 0, False
with Trainer(img, enc, DecoderConfig.hop(), lib=lib) as tr:
    tr.warmup()
    st = tr.get_state()
    tc = tr.true_cost()
    gi = tr.global_iter
if mode == "ref":
    np.savez(OUT, latents=st["latents"], params=st["params"], tc=np.array(tc), gi=gi)
    print("ref warm-up true cost", tc, "global_iter", gi)
else:
    r = dict(np.load(OUT))
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
    print("gpu warm-up true cost", tc, "ref", r["tc"], "global_iter", gi, int(r["gi"]))
    print("latents rel", rel(st["latents"], r["latents"]), "params rel", rel(st["params"], r["params"]))

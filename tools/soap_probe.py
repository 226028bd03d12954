"""Per-tensor parameter differences GPU vs reference after k SOAP steps."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_02726_b200 import capi  # noqa: E402
from paper_2605_02726_b200.trainer import DecoderConfig, EncoderConfig, Trainer  # noqa: E402
from tests import oracle_util  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


ref = oracle_util.load_reference()
gpu = capi.load_product()
img = np.empty((3, 64, 96), np.float32)
ref.cc_make_synthetic_image(64, 96, 7, img.ctypes.data_as(capi._F))
enc = EncoderConfig(lmbda=1e-3, seed=5, use_soap=True)
dcfg = DecoderConfig.hop()
r = Trainer(img, enc, dcfg, lib=ref)
g = Trainer(img, enc, dcfg, lib=gpu)
r.fresh_candidate(0)
g.fresh_candidate(0)
for it in range(3):
    cr = r.proxy_iteration(1e-2, 0.35, 0.22)
    cg = g.proxy_iteration(1e-2, 0.35, 0.22)
    pr, pg = r.get_state()["params"], g.get_state()["params"]
    print("it", it, "cost", cr, cg)
    for ti, p in enumerate(r.params):
        e = rel(g.param_view(pg, ti), r.param_view(pr, ti))
        if e > 1e-5:
            print("   ", p.name, p.rows, p.cols, e)

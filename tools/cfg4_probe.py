"""Where do GPU and reference latent gradients differ at 1360x2048 (cfg4)?"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_02726_b200 import capi  # noqa: E402
from paper_2605_02726_b200.trainer import DecoderConfig, EncoderConfig, Trainer  # noqa: E402
from tests import oracle_util  # noqa: E402
from tests.conftest import make_image  # noqa: E402

ref = oracle_util.load_reference()
gpu = capi.load_product()
h, w = 1360, 2048
img = make_image(ref, h, w, seed=h + w)
enc = EncoderConfig(use_soap=False, lmbda=1e-3, seed=h)
dcfg = DecoderConfig.cfg4()
r = Trainer(img, enc, dcfg, lib=ref)
g = Trainer(img, enc, dcfg, lib=gpu)
r.fresh_candidate(1)
g.fresh_candidate(1)
for it in range(2):
    g.set_state(r.get_state())
    r.proxy_iteration(1e-2, 0.35, 0.22)
    g.proxy_iteration(1e-2, 0.35, 0.22)
    lr_, _ = r.get_grads()
    lg_, _ = g.get_grads()
    gi = len(r.grids) - 1
    a, b = g.grid_view(lg_, gi).ravel(), r.grid_view(lr_, gi).ravel()
    d = np.abs(a - b)
    rel = np.linalg.norm(d) / np.linalg.norm(b)
    big = d > 1e-3 * np.abs(b).max()
    print(f"it {it}: rel {rel:.3e}  n={b.size}  n(|diff| > 1e-3 max|g|)={big.sum()}  "
          f"rel without them {np.linalg.norm(d[~big]) / np.linalg.norm(b):.3e}")
    idx = np.argsort(-d)[:5]
    print("   worst:", [(int(i), float(a[i]), float(b[i])) for i in idx])

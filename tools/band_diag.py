"""Diagnostic: host-routed LocalBands vs the device band group, per-iteration
(cost, mse, bits) printed with full precision (tools only)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2605_02726_b200 import bands as B  # noqa: E402
from paper_2605_02726_b200 import capi  # noqa: E402
from paper_2605_02726_b200.trainer import DecoderConfig, EncoderConfig  # noqa: E402
from tests.conftest import make_image  # noqa: E402

lib = capi.load_product()
h, w, n = 1536, 256, 3
img = make_image(lib, h, w, seed=3)
enc = EncoderConfig(use_soap=False, lmbda=1e-3, seed=3)
lr = np.array([1e-2, 9e-3, 8e-3, 7e-3, 6e-3])
tp = np.array([0.35, 0.33, 0.31, 0.29, 0.27])
ns = np.array([0.22, 0.21, 0.2, 0.19, 0.18])

lb = B.LocalBands(img, n, enc, DecoderConfig.hop(), halo=6, lib=lib)
lb.fresh_candidate(0)
orig = lb.trainers[0].__class__.forward_backward
log = []


def fb(self, *a):
    r = orig(self, *a)
    log.append(r)
    return r


lb.trainers[0].__class__.forward_backward = fb
for i in range(len(lr)):
    log.clear()
    c = lb.proxy_iteration(lr[i], tp[i], ns[i])
    bits = float(sum(s[0] for s in log))
    se = float(sum(s[1] for s in log))
    print("local", repr(c), repr(se / (3 * h * w)), repr(bits), [tuple(map(repr, s)) for s in log])
lb.close()
db = B.DeviceBands(img, n, enc, DecoderConfig.hop(), halo=6, lib=lib)
db.fresh_candidate(0)
db.group.reserve(len(lr))
db.proxy_iterations(lr, tp, ns)
for r in db.group.records(len(lr)):
    print("dev  ", repr(r[0]), repr(r[1]), repr(r[2]))
db.close()

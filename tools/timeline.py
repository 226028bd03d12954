"""Mean event timeline of one proxy iteration (512x768 HOP): ccb_timeline."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_02726_b200 import capi  # noqa: E402
from paper_2605_02726_b200.trainer import DecoderConfig, EncoderConfig, Trainer, make_synthetic_image  # noqa: E402

NAMES = ["start", "softq", "ARM (side)", "pyramid (side)", "ups fwd", "syn fwd", "syn bwd",
         "ups bwd stage 0", "fine grad (tail)", "fine adam (tail)", "ups bwd rest", "coarse grad",
         "end"]
lib = capi.load_product()
h, w = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (512, 768)
img = make_synthetic_image(h, w, 0, lib)
enc = EncoderConfig(use_soap=False, lmbda=1e-3, seed=0)
tr = Trainer(img, enc, DecoderConfig.hop(), lib=lib)
tr.fresh_candidate(0)
for _ in range(20):
    tr.proxy_iteration(1e-2, 0.35, 0.22)
ms = np.zeros(13)
rc = lib.ccb_timeline(tr._h, 50, 1e-2, 0.35, 0.22, ms.ctypes.data_as(C.POINTER(C.c_double)))
assert rc == 0, lib.cc_last_error()
for n, t in zip(NAMES, ms):
    print(f"{t * 1e3:8.1f} us  {n}")

"""Batched-image throughput (BASELINE config 3 on one GPU): B images of
512x768 HOP trained by one batched graph, device-timed steady state.
    python tools/batch_bench.py [B ...]"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_02726_b200 import capi  # noqa: E402
from paper_2605_02726_b200.trainer import Batch, DecoderConfig, EncoderConfig, Trainer, make_synthetic_image  # noqa: E402

lib = capi.load_product()
h, w, K, W = 512, 768, 30, 5
for B in [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8, 24]:
    trs = []
    for m in range(B):
        enc = EncoderConfig.with_total(10000)
        enc.seed, enc.use_soap = m, False
        t = Trainer(make_synthetic_image(h, w, m, lib), enc, DecoderConfig.hop(), lib=lib)
        t.fresh_candidate(0)
        trs.append(t)
    b = Batch(trs)
    b.reserve_iterations(max(K, W))
    lr = np.full(K, 5e-3)
    b.enqueue_proxy_iterations(lr[:W], 0.3, 0.2)
    b.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s = torch.cuda.ExternalStream(lib.cc_trainer_set_stream and 0) if False else None
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    b.enqueue_proxy_iterations(lr, 0.3, 0.2)
    b.synchronize()
    dt = time.perf_counter() - t0
    c = b.proxy_iterations(lr[:2], 0.3, 0.2)
    print(f"B={B:3d}: {dt / K * 1e3:.3f} ms per batched iteration, "
          f"{B * h * w * K / dt / 1e9:.3f} Gpix-iter/s (host-timed, synchronous), finite={np.isfinite(c).all()}",
          flush=True)
    b.close()
    for t in trs:
        t.close()

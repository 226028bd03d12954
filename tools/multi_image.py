"""Throughput of M independent 512x768 encodes on one GPU, one stream each
(BASELINE config 3 style).  Usage: python tools/multi_image.py M [K]"""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_02726_b200 import capi  # noqa: E402
from paper_2605_02726_b200.trainer import DecoderConfig, EncoderConfig, Trainer, make_synthetic_image  # noqa: E402


def main():
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    lib = capi.load_product()
    trs, streams = [], []
    for m in range(M):
        img = make_synthetic_image(512, 768, m, lib)
        enc = EncoderConfig.with_total(10000)
        enc.seed, enc.use_soap = m, False
        tr = Trainer(img, enc, DecoderConfig.hop(), lib=lib)
        tr.fresh_candidate(0)
        s = torch.cuda.Stream()
        lib.cc_trainer_set_stream(tr._h, C.c_void_p(s.cuda_stream))
        trs.append(tr)
        streams.append(s)
    lr = np.full(1, 1e-2)
    tp = np.full(1, 0.35)
    ns = np.full(1, 0.22)
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731

    def run(k):
        for _ in range(k):
            for tr in trs:
                lib.cc_trainer_enqueue_proxy_iterations(tr._h, 1, dp(lr), dp(tp), dp(ns))

    run(3)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run(K)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"M={M} K={K}: {dt / K * 1e3:.3f} ms per round, "
          f"{M * K * 512 * 768 / dt / 1e9:.3f} Gpix-iter/s, {M * K / dt:.0f} it/s total")


if __name__ == "__main__":
    main()

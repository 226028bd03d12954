"""BASELINE config 5: one large image split into row bands, one band per GPU.

    python tools/bench_bands.py [--size 8192] [--steps K] [--warmup W]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tools/bench_bands.py --size 8192

Each rank builds the trainer of its band (paper_2605_02726_b200.bands) on
cuda:LOCAL_RANK; one iteration = halo refresh, forward+backward of the band,
halo-gradient return, NN-gradient / bits / squared-error gathers (NCCL),
Adam.  Prints one JSON line (rank 0): Gpix-iter/s of the WHOLE image
(H*W*iterations / max-over-ranks device time).  With one process the single
band is the whole image, through the same band path.
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_02726_b200 import bands as B  # noqa: E402
from paper_2605_02726_b200 import capi  # noqa: E402
from paper_2605_02726_b200.trainer import DecoderConfig, EncoderConfig, make_synthetic_image  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=8192)
    ap.add_argument("--width", type=int, default=0)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--halo", type=int, default=8)
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    h, w = a.size, a.width or a.size
    lib = capi.load_product()
    img = make_synthetic_image(h, w, 0, lib)
    bands = B.split_rows(h, w, world)
    r0, r1 = bands[rank]
    enc, dcfg = EncoderConfig(use_soap=False, lmbda=1e-3, seed=0), DecoderConfig.hop()
    tr = B.BandTrainer(img, r0, r1, a.halo, enc, dcfg, lib=lib, device=local)
    tr.fresh_candidate(0)
    hyper = any(g.hyper for g in tr.grids)
    if dist is not None:
        run = B.DistBand(tr, h, w, bands, a.halo, hyper, dist, device=torch.device("cuda", local))
    else:
        run = B.LocalBands.__new__(B.LocalBands)  # a one-band LocalBands around `tr`
        run.H, run.W, run.halo, run.bands, run.trainers = h, w, a.halo, bands, [tr]
        run.plans = [B.halo_plan(h, w, bands, a.halo, hyper, 0)]
    for _ in range(a.warmup):
        run.proxy_iteration(1e-2, 0.35, 0.22)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cost = None
    for _ in range(a.steps):
        cost = run.proxy_iteration(1e-2, 0.35, 0.22)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([dt], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    if rank == 0:
        print(json.dumps({
            "metric": f"encode Gpix-iter/s, one {h}x{w} image in {world} row band(s)",
            "value": h * w * a.steps / dt / 1e9, "unit": "Gpix-iter/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": dt / a.steps * 1e3,
            "last_cost": cost, "halo": a.halo, "bands": bands,
            "note": "host-staged halo / gradient exchange; per-band device work in one stream"}))
    tr.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""BASELINE config 5: one large image split into row bands.

    python tools/bench_bands.py [--size 8192] [--bands 1] [--steps K] [--warmup W]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tools/bench_bands.py --size 8192

One process: the image in --bands row bands on this GPU through the library's
local band group (cc_band_group_local).  N processes: one band per GPU through
the NCCL band group (cc_band_group_nccl, bands.DistBand).  Either way one
iteration = halo rows, forward+backward of each band, halo-gradient return,
the rank-order NN-gradient / bits / squared-error gather, the flag AND and
Adam, all enqueued on the band trainers' streams: the K timed iterations are
ONE enqueue call and one host wait.  Prints one JSON line (rank 0):
Gpix-iter/s of the WHOLE image (H*W*K / max-over-ranks device time, CUDA
events on the band streams), the host synchronisations per iteration
(ccb_host_sync_count) and the final cost.
"""
import argparse
import ctypes as C
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_02726_b200 import bands as B  # noqa: E402
from paper_2605_02726_b200 import capi  # noqa: E402
from paper_2605_02726_b200.trainer import DecoderConfig, EncoderConfig, make_synthetic_image  # noqa: E402


def schedule(n, off=0):
    i = np.arange(off, off + n, dtype=np.float64)
    return 1e-2 * np.ones(n), 0.35 - 1e-5 * i, 0.22 - 1e-5 * i


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=8192)
    ap.add_argument("--width", type=int, default=0)
    ap.add_argument("--bands", type=int, default=1, help="bands on this GPU (one process)")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--halo", type=int, default=8)
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    h, w = a.size, a.width or a.size
    lib = capi.load_product()
    img = make_synthetic_image(h, w, 0, lib)
    enc, dcfg = EncoderConfig(use_soap=False, lmbda=1e-3, seed=0), DecoderConfig.hop()
    if dist is None:
        nb = a.bands
        run = B.DeviceBands(img, nb, enc, dcfg, halo=a.halo, lib=lib, devices=[local] * nb)
        trainers, group, bands = run.trainers, run.group, run.bands
    else:
        nb = world
        bands = B.split_rows(h, w, world)
        tr = B.BandTrainer(img, *bands[rank], a.halo, enc, dcfg, lib=lib, device=local)
        trainers = [tr]
        run = B.DistBand(tr, h, w, bands, a.halo, any(g.hyper for g in tr.grids), dist, device=local)
    streams = [torch.cuda.Stream(device=dev) for _ in trainers]
    for t, s in zip(trainers, streams):
        if lib.cc_trainer_set_stream(t._h, C.c_void_p(s.cuda_stream)) != 0:
            raise RuntimeError(lib.cc_last_error().decode())
        t.fresh_candidate(0)
    if dist is not None:
        group = run._nccl_group()
    K, W = a.steps, max(1, a.warmup)
    group.reserve(max(K, W))
    group.enqueue_proxy_iterations(*schedule(W))
    group.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = [torch.cuda.Event(enable_timing=True) for _ in trainers]
    e0.record(streams[0])
    s0 = B.host_sync_count(lib)
    group.enqueue_proxy_iterations(*schedule(K, W))
    syncs_enqueue = B.host_sync_count(lib) - s0
    for e, s in zip(e1, streams):
        e.record(s)
    rec = group.records(K)  # the one host wait (band 0's stream)
    syncs = B.host_sync_count(lib) - s0
    for e in e1:  # (the other bands' streams, for the timing only)
        e.synchronize()
    ms = max(e0.elapsed_time(e) for e in e1)
    if dist is not None:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    if rank == 0:
        print(json.dumps({
            "metric": f"encode Gpix-iter/s, one {h}x{w} image in {nb} row band(s)",
            "value": h * w * K / (ms / 1e3) / 1e9, "unit": "Gpix-iter/s", "n_gpus": world,
            "steps": K, "warmup": W, "ms_per_step": ms / K,
            "host_syncs_per_iteration": syncs / K, "host_syncs_in_enqueue": syncs_enqueue,
            "last_cost": float(rec[-1, 0]), "costs_finite": bool(np.all(np.isfinite(rec[:, 0]))),
            "halo": a.halo, "bands": [list(b) for b in bands],
            "transport": "NCCL band group" if dist is not None else "local band group (one GPU)"}))
    if dist is not None:
        run.close()
        trainers[0].close()
        dist.destroy_process_group()
    else:
        run.close()


if __name__ == "__main__":
    main()

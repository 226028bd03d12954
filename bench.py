#!/usr/bin/env python
"""bench.py — Cool-chic 5.0 encode iterations on B200 (driver contract).

One step = one proxy_iteration (soft-quantise, ARM+IFCE rate fwd/bwd,
upsampling fwd/bwd, synthesis fwd + MSE + bwd, Adam on latents and NN params;
encoder.hpp:97-135) over one 512x768 synthetic image per GPU (BASELINE.json
configs[1], HOP decoder).  Multi-GPU = independent images, one per rank, no
collective on the data path (weak scaling); timing is the max over ranks.

  python bench.py [--gpus N --steps K --warmup W]          B200 arm
  python bench.py --impl reference [...]                   reference CPU arm
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

from paper_2605_02726_b200 import capi  # noqa: E402
from paper_2605_02726_b200.trainer import (  # noqa: E402
    DecoderConfig, EncoderConfig, Trainer, make_synthetic_image,
)

METRIC = "encode Gpix-iter/s (proxy_iteration fwd+bwd+Adam) at 512x768, HOP decoder"
UNIT = "Gpix-iter/s"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--height", type=int, default=512)
    ap.add_argument("--width", type=int, default=768)
    ap.add_argument("--preset", default="hop")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-full-schedule", action="store_true")
    ap.add_argument("--no-cfg3", action="store_true")
    ap.add_argument("--cfg3-line", action="store_true", help="print the N>1 (config 3) line even at N=1")
    ap.add_argument("--images", type=int, default=24, help="cfg3: images in total (sharded over the GPUs)")
    return ap.parse_args()


def schedule(enc: EncoderConfig, n: int, start: int = 0):
    """Main-stage scalars of with_total(10000) (config.hpp:114-122)."""
    lr_s, t_s, n_s = enc.schedules()
    its = range(start, start + n)
    return (np.array([lr_s.value(i) for i in its]), np.array([t_s.value(i) for i in its]),
            np.array([n_s.value(i) for i in its]))


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    FIELDS = ("index,uuid,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, uuid: str | None):
        self.uuid = uuid
        self.rows = []
        self.proc = None

    def start(self):
        cmd = ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
               "-lms", "100"]
        if self.uuid:
            cmd += ["-i", self.uuid]
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                         text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        time.sleep(0.3)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 10:
                self.rows.append(parts)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        mx = [float(r[3]) for r in self.rows if r[3].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[6 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def load_ref_lib():
    from tests.oracle_util import load_reference

    lib = load_reference()
    fn = lib.ccref_parallel_proxy
    fn.restype = C.c_int
    fn.argtypes = [C.POINTER(C.c_float), C.c_int, C.c_int, C.POINTER(capi.EncoderConfigC),
                   C.POINTER(capi.DecoderConfigC), C.c_int, C.c_int, C.c_int,
                   C.POINTER(C.c_double)]
    return lib


def cpu_reference_run(h, w, preset, seed, threads, warm, iters):
    """The UNMODIFIED reference (oracle/_ref, built from /root/reference headers):
    `threads` independent detail::Trainer instances, one image each, on std::threads
    (the reference's only multi-core mode, tools/coolcodec.cpp:150-171)."""
    lib = load_ref_lib()
    img = np.empty((3, h, w), np.float32)
    lib.cc_make_synthetic_image(h, w, seed, img.ctypes.data_as(C.POINTER(C.c_float)))
    enc = EncoderConfig.with_total(10000)
    enc.lmbda, enc.seed, enc.use_soap = 1e-3, seed, False
    ec, dc = enc.to_c(), DecoderConfig.from_name(preset).to_c()
    secs = C.c_double()
    rc = lib.ccref_parallel_proxy(img.ctypes.data_as(C.POINTER(C.c_float)), h, w, C.byref(ec),
                                  C.byref(dc), threads, warm, iters, C.byref(secs))
    if rc != 0:
        raise RuntimeError(lib.cc_last_error().decode())
    return secs.value


def run_reference(args, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    h, w = args.height, args.width
    # each step = one proxy_iteration on every thread (~0.8 s wall); cap the
    # timed steps so the whole arm ends within a couple of minutes
    steps = max(1, min(args.steps, 60))
    warm = max(0, min(args.warmup, 10))
    secs = cpu_reference_run(h, w, args.preset, args.seed, threads, warm, steps)
    value = threads * steps * h * w / secs / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": steps, "warmup": warm, "steps_requested": args.steps,
        "ms_per_step": 1e3 * secs / steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "cpu_model": cpu_model(),
                         "sample": f"{threads} independent detail::Trainer (oracle/_ref, reference "
                                   f"headers, -O3 -ffp-contract=fast) x {steps} proxy_iteration "
                                   f"each after {warm} warm-up, {h}x{w} {args.preset}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def config_dict(args):
    d = {
        "workload": f"cfg2: one {args.height}x{args.width} RGB synthetic image per GPU, "
                    f"{args.preset.upper()} decoder, proxy_iteration (NN params Adam)",
        "height": args.height, "width": args.width, "decoder": args.preset,
        "images_per_gpu": 1, "lambda": 1e-3,
        "schedule": "EncoderConfig::with_total(10000) main-stage lr/T/sigma",
        "parallelism": f"image-sharded x{args.gpus} (no collective)",
        "l2": "back-to-back iterations, per-iteration working set ~150 MB > 126 MB L2; "
              "value_l2_flushed = same steps with a 512 MB L2 flush before each",
    }
    return d


def run_b200(args, rank, world, local_rank):
    import torch

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist

    lib = capi.load_product()
    h, w = args.height, args.width
    if world > 1 or args.cfg3_line:
        return run_cfg3_line(args, lib, rank, world, dev, dist)
    img = make_synthetic_image(h, w, args.seed + rank, lib)
    enc = EncoderConfig.with_total(10000)
    enc.lmbda, enc.seed, enc.use_soap = 1e-3, args.seed + rank, False
    dcfg = DecoderConfig.from_name(args.preset)
    tr = Trainer(img, enc, dcfg, lib=lib, device=local_rank)
    tr.fresh_candidate(0)
    # a real (non-legacy) stream: the library launches on it, the events below
    # are recorded on it, so they bracket exactly the library's work
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    assert stream.cuda_stream != 0
    if lib.cc_trainer_set_stream(tr._h, C.c_void_p(stream.cuda_stream)) != 0:
        raise RuntimeError(lib.cc_last_error().decode())
    K, W = args.steps, max(3, args.warmup)
    lr, tp, ns = schedule(enc, W + K)

    def enqueue(a, b):
        rc = lib.cc_trainer_enqueue_proxy_iterations(tr._h, b - a, _dp(lr[a:b].copy()),
                                                     _dp(tp[a:b].copy()), _dp(ns[a:b].copy()))
        if rc != 0:
            raise RuntimeError(lib.cc_last_error().decode())

    # one-off setup (batch buffers sized for the largest batch used below, the
    # batched iteration graph instantiated) happens here, outside every timed region
    if lib.cc_trainer_reserve_iterations(tr._h, max(W, K)) != 0:
        raise RuntimeError(lib.cc_last_error().decode())
    enqueue(0, W)
    torch.cuda.synchronize(dev)
    kpi = C.c_int()
    lib.ccb_kernels_per_iteration(tr._h, C.byref(kpi))

    # ---------------- timed region (device events, max over ranks) --------
    uuid = None
    try:
        uuid = str(torch.cuda.get_device_properties(dev).uuid)
        if uuid and not uuid.startswith("GPU-"):
            uuid = "GPU-" + uuid
    except Exception:
        uuid = None
    sampler = ClockSampler(uuid)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    sampler.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    enqueue(W, W + K)
    e1.record(stream)
    e1.synchronize()
    torch.cuda.synchronize(dev)
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1)
    rec = np.empty(4 * K, np.float64)
    lib.cc_trainer_last_records(tr._h, K, _dp(rec))
    finite = bool(np.all(np.isfinite(rec[0::4])))
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * h * w * K / (ms_max / 1e3) / 1e9

    # ---------------- same steps with an L2 flush before each -------------
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    Kf = min(K, 50)
    tot = 0.0
    for i in range(Kf):
        flush.zero_()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        enqueue(W + i, W + i + 1)
        a1.record(stream)
        a1.synchronize()
        tot += a0.elapsed_time(a1)
    t = torch.tensor([tot / Kf], device=dev, dtype=torch.float64)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    value_flushed = world * h * w / (float(t.item()) / 1e3) / 1e9
    del flush

    # ---------------- per-stage profile and the roofline ------------------
    stage_ms = np.zeros(8, np.float64)
    lib.ccb_profile_stages(tr._h, 20, lr[W], tp[W], ns[W], _dp(stage_ms))
    stages = {lib.ccb_stage_name(s).decode(): round(float(stage_ms[s]), 5) for s in range(8)}
    arm_flops = lib.ccb_arm_flops(tr._h)
    peak, pk_ms = C.c_double(), C.c_double()
    lib.ccb_fp32_peak(local_rank, C.byref(peak), C.byref(pk_ms))
    achieved = arm_flops / (stage_ms[1] / 1e3) / 1e12
    traffic = None
    tf = REPO / "profiles" / "arm_traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get("bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "fp32", "kernel": "k_armc (ARM + IFCE fwd/bwd, weights in the constant bank; "
                "timed with its weight pack and constant-slot fill)",
                "achieved": achieved, "peak": peak.value, "unit": "TFLOP/s",
                "frac": achieved / peak.value, "traffic": traffic,
                "flops_per_launch": arm_flops,
                "peak_source": "FFMA peak measured in-run by ccb_fp32_peak (MEASURED_PEAKS.json "
                               "has no fp32 entry)",
                "stage_ms": stages,
                "macs_per_px": capi_macs(lib, dcfg, h, w)}

    # ---------------- end to end through the public API -------------------
    e2e = None
    if not args.no_e2e:
        pinned = torch.empty((3, h, w), dtype=torch.float32, pin_memory=True)
        pinned.numpy()[...] = img
        Ke = min(K, 100)
        if dist:
            dist.barrier()
        torch.cuda.synchronize(dev)
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # the path cc_trainer_train uses: image up from pinned memory, then per
        # step the schedule scalars up (pinned) and the step's record (cost,
        # mse, bits, global_iter) down to pinned memory, no host sync between
        # steps; the host reads the costs after the last step
        b0.record(stream)
        tr.upload_image(pinned.numpy())
        sl, st_, sn = lr[W:W + Ke].copy(), tp[W:W + Ke].copy(), ns[W:W + Ke].copy()
        lib.cc_trainer_enqueue_proxy_iterations(tr._h, Ke, _dp(sl), _dp(st_), _dp(sn))
        rec = np.empty(4 * Ke, np.float64)
        lib.cc_trainer_last_records(tr._h, Ke, _dp(rec))
        b1.record(stream)
        b1.synchronize()
        costs = list(rec[0::4])
        t = torch.tensor([b0.elapsed_time(b1)], device=dev, dtype=torch.float64)
        if dist:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = {"value": world * h * w * Ke / (float(t.item()) / 1e3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": (3 * h * w * 4 + Ke * 24) / Ke,
               "d2h_bytes_per_step": 32,
               "steps": Ke,
               "api": "cc_trainer_upload_image + cc_trainer_enqueue_proxy_iterations (per step: "
                      "schedule H2D from pinned memory, record written by the step's last kernel into "
                      "mapped pinned host memory) + "
                      "cc_trainer_last_records (the path of cc_trainer_train)"}
        # the synchronous per-iteration call (cost returned to the host each step)
        torch.cuda.synchronize(dev)
        b0.record(stream)
        costs_s = [tr.proxy_iteration(lr[W + i], tp[W + i], ns[W + i]) for i in range(Ke)]
        b1.record(stream)
        b1.synchronize()
        t = torch.tensor([b0.elapsed_time(b1)], device=dev, dtype=torch.float64)
        if dist:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e["sync_per_step"] = {"value": world * h * w * Ke / (float(t.item()) / 1e3) / 1e9,
                                "api": "cc_trainer_proxy_iteration (synchronous, returns the cost)",
                                "d2h_bytes_per_step": 144}
        costs = costs + costs_s
        finite = finite and all(math.isfinite(c) for c in costs)

    # ---------------- the whole with_total(10000) encode through train() -----
    # beside the steady-state proxy iteration, the full schedule
    # (warm-up candidates, main stage with true-cost snapshots every 1,000
    # iterations, hardround) as one cc_trainer_train call per image; host
    # wall clock around the synchronous call (image already resident)
    full = None
    if not args.no_full_schedule:
        tr_f = Trainer(img, enc, dcfg, lib=lib, device=local_rank)
        if dist:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        res = tr_f.train()
        secs = time.perf_counter() - t0
        tr_f.close()
        t = torch.tensor([secs], device=dev, dtype=torch.float64)
        if dist:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        secs_max = float(t.item())
        its = res.stats.iterations
        full = {"seconds": secs_max, "iterations": its, "it_per_s_per_image": its / secs_max,
                "value": world * h * w * its / secs_max / 1e9, "unit": UNIT,
                "true_cost": res.stats.true_cost, "psnr_db": res.stats.psnr, "rate_bpp": res.stats.rate_bpp,
                "restarts": res.stats.restarts,
                "api": "cc_trainer_train (EncoderConfig::with_total(10000), use_soap=false): warm-up "
                       "candidates, main stage, true cost every 1,000 iterations, hardround",
                "timing": "host wall clock around the synchronous call, max over ranks"}
        finite = finite and math.isfinite(res.stats.true_cost)

    # BASELINE config 3 on this one GPU: 24 images batched in one graph
    cfg3 = None
    if world == 1 and not args.no_cfg3:
        tr.close()
        r3 = run_cfg3(args, lib, args.images, args.seed, dev, None, min(K, 20), W)
        cfg3 = {"value": r3["value"], "unit": UNIT, "ms_per_step": r3["ms_per_step"],
                "images_per_gpu": r3["images_per_gpu"], "steps": r3["steps"], "e2e": r3["e2e"],
                "costs_finite": r3["costs_finite"],
                "workload": f"cfg3: {args.images} independent {h}x{w} synthetic images batched in one graph "
                            "(include/coolchic_b200_batch.h), device-timed steady state"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        iters = 2
        try:
            secs = cpu_reference_run(h, w, args.preset, args.seed, threads, 1, iters)
            cpu = {"value": threads * iters * h * w / secs / 1e9, "unit": UNIT, "cores": threads,
                   "kind": "reference", "cpu_model": cpu_model(),
                   "sample": f"{threads} independent detail::Trainer x {iters} proxy_iteration "
                             f"after 1 warm-up, {h}x{w} {args.preset}, oracle/_ref"}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_dict(args),
            "it_per_s_per_image": K / (ms_max / 1e3),
            "value_l2_flushed": value_flushed,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "full_schedule": full,
            "cfg3_one_gpu": cfg3,
            "gpu_launches": int(kpi.value) * K, "kernels_per_step": int(kpi.value),
            "clocks": clocks, "costs_finite": finite,
        }
        print(json.dumps(line), flush=True)
    tr.close()


def _max_over_ranks(dist, x, dev):
    """max of a host scalar over the ranks (NCCL on the device; gloo on the host)."""
    if not dist:
        return float(x)
    import torch

    on_dev = dist.get_backend() == "nccl"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev if on_dev else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_cfg3(args, lib, n_img, seed0, dev, dist, K, W):
    """BASELINE config 3 on this GPU: n_img independent 512x768 images trained
    in lock-step by one batched graph (include/coolchic_b200_batch.h).
    Device-timed steady state (CUDA events on the batch's stream) and end to
    end (images up from pinned host memory, records back) through the C ABI."""
    import torch

    from paper_2605_02726_b200.trainer import Batch

    h, w = args.height, args.width
    dcfg = DecoderConfig.from_name(args.preset)
    imgs, trs = [], []
    for m in range(n_img):
        enc = EncoderConfig.with_total(10000)
        enc.lmbda, enc.seed, enc.use_soap = 1e-3, seed0 + m, False
        imgs.append(make_synthetic_image(h, w, seed0 + m, lib))
        t = Trainer(imgs[-1], enc, dcfg, lib=lib, device=dev.index)
        t.fresh_candidate(0)
        trs.append(t)
    stream = torch.cuda.Stream(device=dev)
    if lib.cc_trainer_set_stream(trs[0]._h, C.c_void_p(stream.cuda_stream)) != 0:
        raise RuntimeError(lib.cc_last_error().decode())
    b = Batch(trs)  # every trainer moves onto the first one's stream
    b.reserve_iterations(max(K, W))
    lr, tp, ns = schedule(EncoderConfig.with_total(10000), W + K)
    b.enqueue_proxy_iterations(lr[:W], tp[:W], ns[:W])
    b.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    b.enqueue_proxy_iterations(lr[W:W + K], tp[W:W + K], ns[W:W + K])
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    ms = _max_over_ranks(dist, ms, dev)
    world = dist.get_world_size() if dist else 1
    value = world * n_img * h * w * K / (ms / 1e3) / 1e9
    rec = np.empty(4 * K, np.float64)
    finite = True
    for tr in trs:
        lib.cc_trainer_last_records(tr._h, K, _dp(rec))
        finite = finite and bool(np.all(np.isfinite(rec[0::4])))
    # end to end: every image up from pinned host memory, the batched steps,
    # every image's records read back
    pinned = [torch.empty((3, h, w), dtype=torch.float32, pin_memory=True) for _ in range(n_img)]
    for pm, im in zip(pinned, imgs):
        pm.numpy()[...] = im
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0.record(stream)
    for tr, pm in zip(trs, pinned):
        tr.upload_image(pm.numpy())
    b.enqueue_proxy_iterations(lr[W:W + K], tp[W:W + K], ns[W:W + K])
    for tr in trs:
        lib.cc_trainer_last_records(tr._h, K, _dp(rec))
    e1.record(stream)
    e1.synchronize()
    e2e = world * n_img * h * w * K / (_max_over_ranks(dist, e0.elapsed_time(e1), dev) / 1e3) / 1e9
    kpi = C.c_int()
    lib.ccb_kernels_per_iteration(trs[0]._h, C.byref(kpi))
    b.close()
    for tr in trs:
        tr.close()
    return {"value": value, "ms_per_step": ms / K, "images_per_gpu": n_img, "steps": K,
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": (n_img * 3 * h * w * 4 + K * 24) / K,
                    "d2h_bytes_per_step": n_img * 32,
                    "api": "cc_trainer_upload_image per image + cc_batch_enqueue_proxy_iterations + "
                           "cc_trainer_last_records per image"},
            "kernels_per_step": int(kpi.value), "costs_finite": finite}


def run_cfg3_line(args, lib, rank, world, dev, dist):
    """N > 1: BASELINE config 3 — 24 images sharded evenly over the ranks
    (no collective on the data path), batched within each GPU."""
    import torch

    total = args.images
    if total % world:
        raise SystemExit(f"--images {total} does not split over {world} GPUs")
    n_img = total // world
    K, W = args.steps, max(3, args.warmup)
    sampler = ClockSampler(None)
    sampler.start()
    r = run_cfg3(args, lib, n_img, args.seed + rank * n_img, dev, dist, K, W)
    clocks = sampler.stop()
    if rank == 0:
        cfg = config_dict(args)
        cfg.update({"workload": f"cfg3: {total} independent {args.height}x{args.width} synthetic images, "
                                f"{n_img} per GPU batched in one graph, HOP, proxy_iteration (NN params Adam)",
                    "images_per_gpu": n_img, "images_total": total,
                    "parallelism": f"image-sharded x{world} (no collective), batched within each GPU"})
        line = {"metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
                "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": cfg,
                "e2e": r["e2e"], "gpu_launches": r["kernels_per_step"] * K, "kernels_per_step": r["kernels_per_step"],
                "clocks": clocks, "costs_finite": r["costs_finite"]}
        print(json.dumps(line), flush=True)


def capi_macs(lib, dcfg, h, w):
    dc = dcfg.to_c()
    return lib.cc_count_macs_per_pixel(C.byref(dc), h, w)


def main():
    args = parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook (tests/test_bench_ranks.py): several ranks on one GPU with a
    # gloo process group — exercises the N>1 code path, not a timing
    shared = os.environ.get("BENCH_SHARED_GPU") == "1"
    if shared:
        local_rank = 0
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_b200(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()

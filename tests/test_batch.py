"""Batched images (include/coolchic_b200_batch.h, BASELINE config 3): one set
of launches per stage for several trainers must give every image exactly what
it gets alone — bit for bit (each kernel reads only its own image's plan)."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2605_02726_b200 import capi
from paper_2605_02726_b200.trainer import Batch, DecoderConfig, EncoderConfig, Trainer
from tests.conftest import REPO as GOLDEN_ROOT, make_image


def test_batch_header_declares_the_python_table():
    assert sorted(capi.BATCH_SIGNATURES) == capi.header_symbols("coolchic_b200_batch.h")


@pytest.mark.gpu
@pytest.mark.parametrize("use_soap", [False, True])
def test_batch_matches_independent_trainers(gpu_lib, use_soap):
    h, w, n_img, iters = 96, 128, 3, 5
    imgs = [make_image(gpu_lib, h, w, seed=s) for s in range(n_img)]
    encs = [EncoderConfig(use_soap=use_soap, lmbda=1e-3, seed=10 + s) for s in range(n_img)]
    lr = np.linspace(1e-2, 8e-3, iters)
    alone = []
    for img, enc in zip(imgs, encs):
        with Trainer(img, enc, DecoderConfig.hop(), lib=gpu_lib) as tr:
            tr.fresh_candidate(0)
            c = tr.proxy_iterations(lr, 0.35, 0.22)
            st = tr.get_state()
            lg, pg = tr.get_grads()
            alone.append((c, st, lg, pg))
    trs = [Trainer(img, enc, DecoderConfig.hop(), lib=gpu_lib) for img, enc in zip(imgs, encs)]
    try:
        for t in trs:
            t.fresh_candidate(0)
        with Batch(trs) as b:
            b.reserve_iterations(iters)
            costs = b.proxy_iterations(lr, 0.35, 0.22)
        for k, t in enumerate(trs):
            c, st, lg, pg = alone[k]
            assert np.array_equal(costs[k], c), k
            st2 = t.get_state()
            for key in ("latents", "params", "lat_m", "lat_v"):
                assert np.array_equal(st2[key], st[key]), (k, key)
            lg2, pg2 = t.get_grads()
            assert np.array_equal(lg2, lg) and np.array_equal(pg2, pg), k
            assert st2["global_iter"] == st["global_iter"] == iters
    finally:
        for t in trs:
            t.close()


@pytest.mark.gpu
def test_batch_rejects_mixed_geometry(gpu_lib):
    a = Trainer(make_image(gpu_lib, 64, 64), EncoderConfig(use_soap=False), DecoderConfig.hop(), lib=gpu_lib)
    b = Trainer(make_image(gpu_lib, 64, 96), EncoderConfig(use_soap=False), DecoderConfig.hop(), lib=gpu_lib)
    try:
        with pytest.raises(Exception):
            Batch([a, b])
    finally:
        a.close()
        b.close()


@pytest.mark.gpu
@pytest.mark.parametrize("soap", [0, 1])
def test_batched_warmup_is_the_sequential_warmup(gpu_lib, tmp_path, soap):
    """train()'s warm-up runs each round's candidates concurrently (one batched
    graph); every candidate starts from the global_iter the
    sequential loop (encoder.hpp:315-342) gives it, so the whole encode must
    be bit-identical to the sequential warm-up (CCB_WARMUP_SERIAL=1)."""
    import os
    import subprocess
    import sys

    res = {}
    for mode in ("0", "1"):
        out = tmp_path / f"w{mode}.npz"
        env = dict(os.environ, CCB_WARMUP_SERIAL=mode)
        subprocess.run([sys.executable, "-m", "tests.warmup_run", str(out), str(soap)], env=env, check=True,
                       timeout=600, cwd=str(GOLDEN_ROOT))
        res[mode] = dict(np.load(out))
    for k in res["0"]:
        assert np.array_equal(res["0"][k], res["1"][k]), k

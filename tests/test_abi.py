"""CPU-only checks of the drop-in boundary: the C ABI library loads, exports
every symbol include/*.h declares, and its host-side functions (presets,
with_total, count_macs_per_pixel) agree with the reference's.  No compute call
touches a GPU here."""
from __future__ import annotations

import ctypes as C
import math

import numpy as np
import pytest

from paper_2605_02726_b200 import capi
from paper_2605_02726_b200.trainer import DecoderConfig, EncoderConfig, Schedule


def _exports(lib, names):
    missing = []
    for n in names:
        try:
            getattr(lib, n)
        except AttributeError:
            missing.append(n)
    return missing


def test_product_exports_every_declared_symbol(product_lib):
    names = (capi.header_symbols("coolchic_b200.h") + capi.header_symbols("coolchic_b200_diag.h")
             + capi.header_symbols("coolchic_b200_band.h") + capi.header_symbols("coolchic_b200_codec.h")
             + capi.header_symbols("coolchic_b200_batch.h"))
    assert len(names) >= 48
    assert _exports(product_lib, names) == []
    assert product_lib.cc_impl_name() == b"b200"


def test_signature_table_covers_header():
    assert sorted(capi.SIGNATURES) == capi.header_symbols("coolchic_b200.h")
    assert sorted(capi.DIAG_SIGNATURES) == capi.header_symbols("coolchic_b200_diag.h")
    assert sorted(capi.BAND_SIGNATURES) == capi.header_symbols("coolchic_b200_band.h")
    assert sorted(capi.CODEC_SIGNATURES) == capi.header_symbols("coolchic_b200_codec.h")
    assert sorted(capi.BATCH_SIGNATURES) == capi.header_symbols("coolchic_b200_batch.h")


def test_checkers_export_the_same_abi(ref_lib, port_lib):
    names = capi.header_symbols("coolchic_b200.h")
    assert _exports(ref_lib, names) == []
    assert _exports(ref_lib, capi.header_symbols("coolchic_b200_codec.h")) == []
    assert _exports(port_lib, names) == []
    assert ref_lib.cc_impl_name() == b"reference"
    assert port_lib.cc_impl_name() == b"port"


@pytest.mark.parametrize("name", ["lop", "mop", "hop", "vhop"])
def test_presets_match_reference(product_lib, ref_lib, name):
    a, b = capi.DecoderConfigC(), capi.DecoderConfigC()
    assert product_lib.cc_decoder_config_preset(name.encode(), C.byref(a)) == 0
    assert ref_lib.cc_decoder_config_preset(name.encode(), C.byref(b)) == 0
    fa = [getattr(a, f) for f, _ in capi.DecoderConfigC._fields_]
    fb = [getattr(b, f) for f, _ in capi.DecoderConfigC._fields_]
    assert fa == fb
    assert fa == [getattr(DecoderConfig.from_name(name), f) for f, _ in capi.DecoderConfigC._fields_]


def test_unknown_preset_is_config_error(product_lib):
    a = capi.DecoderConfigC()
    assert product_lib.cc_decoder_config_preset(b"xop", C.byref(a)) == capi.CC_ERR_CONFIG
    assert b"unknown decoder config" in product_lib.cc_last_error()


@pytest.mark.parametrize("total", [20, 240, 600, 2000, 10000, 100000, 31337])
def test_with_total_matches_reference(product_lib, ref_lib, total):
    a, b = capi.EncoderConfigC(), capi.EncoderConfigC()
    assert product_lib.cc_encoder_config_with_total(total, C.byref(a)) == 0
    assert ref_lib.cc_encoder_config_with_total(total, C.byref(b)) == 0
    keys = ["warmup_candidates", "warmup_keep", "warmup_iters", "main_iters", "hardround_iters"]
    assert [getattr(a, k) for k in keys + ["use_soap"]] == [getattr(b, k) for k in keys + ["use_soap"]]
    py = EncoderConfig.with_total(total)
    assert [getattr(py, k) for k in keys] == [getattr(b, k) for k in keys]


def test_with_total_10k_split():
    # the 10k "fast" budget = 7 x 40 warm-up + 9,670 main + 50 hardround
    cfg = EncoderConfig.with_total(10000)
    assert (cfg.warmup_iters, cfg.main_iters, cfg.hardround_iters) == (40, 9670, 50)
    assert cfg.total_iters() == 10000


def test_with_total_too_small(product_lib):
    a = capi.EncoderConfigC()
    assert product_lib.cc_encoder_config_with_total(19, C.byref(a)) == capi.CC_ERR_CONFIG


@pytest.mark.parametrize("name,h,w,want", [("hop", 512, 768, 2022.7), ("mop", 512, 768, 887.5),
                                           ("lop", 512, 768, 532.4), ("hop", 8192, 8192, 2109.6)])
def test_count_macs_per_pixel(product_lib, ref_lib, name, h, w, want):
    dc = DecoderConfig.from_name(name).to_c()
    a = product_lib.cc_count_macs_per_pixel(C.byref(dc), h, w)
    b = ref_lib.cc_count_macs_per_pixel(C.byref(dc), h, w)
    assert a == pytest.approx(b, rel=1e-12)
    assert a == pytest.approx(want, abs=0.06)


def test_count_macs_cfg4_custom(product_lib, ref_lib):
    # spatial 26 + IFCE 6, width 20, synth 64 -> 2,639.0 MAC/px at 1360x2048
    d = DecoderConfig(preset=2, spatial_ctx=26, ifce_dim=6, arm_width=20, arm_hidden=2,
                      synth_hidden=64, synth_posts=2)
    dc = d.to_c()
    a = product_lib.cc_count_macs_per_pixel(C.byref(dc), 1360, 2048)
    assert a == pytest.approx(ref_lib.cc_count_macs_per_pixel(C.byref(dc), 1360, 2048), rel=1e-12)
    assert a == pytest.approx(2639.0, abs=0.06)


def test_schedules_endpoints():
    # tests/test_latent.cpp:125-142
    lin = Schedule(0.35, 0.08, "linear", 100)
    assert lin.value(0) == pytest.approx(0.35)
    assert lin.value(100) == pytest.approx(0.08)
    assert lin.value(50) == pytest.approx(0.215)
    assert lin.value(200) == pytest.approx(0.08)
    cos = Schedule(1e-2, 1e-6, "cosine", 100)
    assert cos.value(50) == pytest.approx((1e-2 + 1e-6) / 2)
    prev = cos.value(0)
    for i in range(1, 101):
        assert cos.value(i) <= prev + 1e-15
        prev = cos.value(i)


def test_synthetic_image_generator(product_lib, ref_lib):
    a = np.empty((3, 40, 56), np.float32)
    b = np.empty((3, 40, 56), np.float32)
    product_lib.cc_make_synthetic_image(40, 56, 7, a.ctypes.data_as(capi._F))
    ref_lib.cc_make_synthetic_image(40, 56, 7, b.ctypes.data_as(capi._F))
    assert np.allclose(a, b, atol=1e-7)
    assert a.min() >= 0.0 and a.max() <= 1.0
    assert 0.3 < a.mean() < 0.7
    assert not np.array_equal(a[0], a[1])  # channels differ


def test_trainer_create_without_gpu_fails_loudly(product_lib):
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("GPU present: covered by the gpu tests")
    except Exception:  # noqa: BLE001
        pass
    img = np.zeros((3, 8, 8), np.float32)
    ec, dc = EncoderConfig(use_soap=False).to_c(), DecoderConfig.hop().to_c()
    h = C.c_void_p()
    rc = product_lib.cc_trainer_create(img.ctypes.data_as(capi._F), 8, 8, C.byref(ec), C.byref(dc),
                                       0, C.byref(h))
    assert rc == capi.CC_ERR_CUDA  # no CPU fallback
    assert product_lib.cc_last_error()


def test_math_is_finite_sanity():
    assert math.isfinite(EncoderConfig.with_total(10000).lr_start)

"""Shared fixtures.  `-m gpu` tests need a B200; everything else runs on CPU.

Checkers (oracle/_ref = the reference headers compiled behind the C ABI,
oracle/libccport.so = the plain-C restatement) are test infrastructure only.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

from paper_2605_02726_b200 import capi  # noqa: E402
from tests import oracle_util  # noqa: E402

GOLDEN = REPO / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running parity case")


def _try_make(target: str):
    if Path("/root/reference/proj/include/coolcodec/encoder.hpp").exists() or target == "port":
        subprocess.run(["make", "-s", "-C", str(REPO / "oracle"), target], check=False,
                       stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)


@pytest.fixture(scope="session")
def ref_lib():
    p = oracle_util.reference_path()
    if not p.exists():
        _try_make("ref")
    if not oracle_util.reference_path().exists():
        pytest.skip("oracle/_ref not built (needs /root/reference once)")
    return oracle_util.load_reference()


@pytest.fixture(scope="session")
def port_lib():
    if not oracle_util.PORT_SO.exists():
        _try_make("port")
    if not oracle_util.PORT_SO.exists():
        pytest.skip("oracle/libccport.so not built")
    return oracle_util.load_port()


@pytest.fixture(scope="session")
def product_lib():
    if not capi.PRODUCT_SO.exists():
        from paper_2605_02726_b200 import build

        build.build_product()
    return capi.load_product()


@pytest.fixture(scope="session")
def gpu_lib(product_lib):
    """The product library on a GPU box; fails loudly (no fallback) if absent."""
    try:
        import torch

        ok = torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        ok = False
    if not ok:
        pytest.skip("no CUDA device")
    return product_lib


def make_image(lib, h, w, seed=0):
    img = np.empty((3, h, w), np.float32)
    rc = lib.cc_make_synthetic_image(h, w, seed, img.ctypes.data_as(capi._F))
    assert rc == 0
    return img


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    n = np.linalg.norm(b)
    d = np.linalg.norm(a - b)
    if n == 0.0:
        return 0.0 if d == 0.0 else float("inf")
    return float(d / n)

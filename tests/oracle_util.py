"""Loaders for the CHECKERS under oracle/ (test infrastructure only).

Only tests/, bench.py's reference/cpu_baseline leg and __graft_entry__.smoke()
may use this module.  The product library never imports it.
"""
from __future__ import annotations

from pathlib import Path

from paper_2605_02726_b200 import capi

REPO = Path(__file__).resolve().parents[1]
REF_DIR = REPO / "oracle" / "_ref"
PORT_SO = REPO / "oracle" / "libccport.so"


def _has_avx512() -> bool:
    try:
        return "avx512f" in Path("/proc/cpuinfo").read_text()
    except OSError:
        return False


def reference_path() -> Path:
    """oracle/_ref/libccref_v4.so (AVX-512) or _v3 (AVX2) for this host CPU."""
    v4, v3 = REF_DIR / "libccref_v4.so", REF_DIR / "libccref_v3.so"
    if _has_avx512() and v4.exists():
        return v4
    return v3


def load_reference():
    p = reference_path()
    if not p.exists():
        raise FileNotFoundError(f"{p} missing: run `make -C oracle ref` where /root/reference exists")
    return capi.load_library(p)


def load_port():
    if not PORT_SO.exists():
        raise FileNotFoundError(f"{PORT_SO} missing: run `make -C oracle port`")
    return capi.load_library(PORT_SO)


def truth_grads(ref_lib, tr, temp: float, noise_std: float):
    """fp64 truth of the proxy-iteration gradients on `tr`'s current state
    (a Trainer over the reference checker; oracle/ref_capi.cpp
    ccref_truth_grads: the reference's own templated kernels instantiated
    for double).  Returns (latent_grads, param_grads, [cost, mse, bits])."""
    import ctypes as C

    import numpy as np

    fn = ref_lib.ccref_truth_grads
    fn.restype = C.c_int
    fn.argtypes = [C.c_void_p, C.c_double, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double),
                   C.POINTER(C.c_double)]
    lg = np.empty(tr.n_latents, np.float64)
    pg = np.empty(tr.n_params, np.float64)
    sc = np.empty(3, np.float64)
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    rc = fn(tr._h, temp, noise_std, dp(lg), dp(pg), dp(sc))
    if rc != 0:
        raise RuntimeError(ref_lib.cc_last_error().decode())
    return lg, pg, sc

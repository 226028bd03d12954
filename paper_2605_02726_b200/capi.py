"""ctypes binding of the C ABI declared in include/coolchic_b200.h.

The same declarations bind all three libraries that export the ABI: the B200
product (``libcoolchic_b200.so``) and the two checkers under ``oracle/``.  Only
the product library is loaded by :func:`load_product`; the checkers are loaded
by tests/bench through :func:`load_library` with an explicit path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
REPO_DIR = PKG_DIR.parent
PRODUCT_SO = PKG_DIR / "libcoolchic_b200.so"

CC_OK, CC_ERR_CONFIG, CC_ERR_FORMAT, CC_ERR_TRAINING, CC_ERR_CUDA, CC_ERR_STATE = range(6)


class DecoderConfigC(C.Structure):
    _fields_ = [
        ("preset", C.c_int),
        ("spatial_ctx", C.c_int),
        ("ifce_dim", C.c_int),
        ("arm_width", C.c_int),
        ("arm_hidden", C.c_int),
        ("synth_hidden", C.c_int),
        ("synth_posts", C.c_int),
        ("use_hyperlatents", C.c_int),
        ("use_stabilizer", C.c_int),
    ]


class EncoderConfigC(C.Structure):
    _fields_ = [
        ("warmup_candidates", C.c_int),
        ("warmup_keep", C.c_int),
        ("warmup_iters", C.c_int),
        ("main_iters", C.c_int),
        ("hardround_iters", C.c_int),
        ("lr_start", C.c_double),
        ("lr_end", C.c_double),
        ("noise_std_start", C.c_double),
        ("noise_std_end", C.c_double),
        ("temp_start", C.c_double),
        ("temp_end", C.c_double),
        ("hardround_lr", C.c_double),
        ("lambda_", C.c_double),
        ("seed", C.c_uint64),
        ("use_soap", C.c_int),
        ("true_cost_interval", C.c_int),
        ("log_path", C.c_char_p),
    ]


class LayoutC(C.Structure):
    _fields_ = [
        ("height", C.c_int),
        ("width", C.c_int),
        ("levels", C.c_int),
        ("hyper_count", C.c_int),
        ("n_grids", C.c_int),
        ("n_latents", C.c_int64),
        ("n_tensors", C.c_int),
        ("n_params", C.c_int64),
        ("pad", C.c_int),
    ]


class GridInfoC(C.Structure):
    _fields_ = [
        ("level", C.c_int),
        ("hyper", C.c_int),
        ("rows", C.c_int),
        ("cols", C.c_int),
        ("offset", C.c_int64),
        ("ifce_slot", C.c_int),
    ]


class ParamInfoC(C.Structure):
    _fields_ = [
        ("name", C.c_char * 32),
        ("rows", C.c_int),
        ("cols", C.c_int),
        ("size", C.c_int64),
        ("offset", C.c_int64),
    ]


class TrainStatsC(C.Structure):
    _fields_ = [
        ("iterations", C.c_int64),
        ("true_cost", C.c_double),
        ("psnr", C.c_double),
        ("rate_bpp", C.c_double),
        ("restarts", C.c_int),
        ("skipped_steps", C.c_int),
        ("seconds", C.c_double),
    ]


_P = C.c_void_p
_F = C.POINTER(C.c_float)
_D = C.POINTER(C.c_double)
_I64 = C.POINTER(C.c_int64)
_I32 = C.POINTER(C.c_int32)
_I = C.POINTER(C.c_int)

# name -> (restype, argtypes); exactly the symbols include/coolchic_b200.h declares
SIGNATURES = {
    "cc_last_error": (C.c_char_p, []),
    "cc_impl_name": (C.c_char_p, []),
    "cc_decoder_config_preset": (C.c_int, [C.c_char_p, C.POINTER(DecoderConfigC)]),
    "cc_encoder_config_default": (C.c_int, [C.POINTER(EncoderConfigC)]),
    "cc_encoder_config_with_total": (C.c_int, [C.c_int, C.POINTER(EncoderConfigC)]),
    "cc_count_macs_per_pixel": (C.c_double, [C.POINTER(DecoderConfigC), C.c_int, C.c_int]),
    "cc_make_synthetic_image": (C.c_int, [C.c_int, C.c_int, C.c_uint64, _F]),
    "cc_trainer_create": (
        C.c_int,
        [_F, C.c_int, C.c_int, C.POINTER(EncoderConfigC), C.POINTER(DecoderConfigC), C.c_int,
         C.POINTER(_P)],
    ),
    "cc_trainer_destroy": (None, [_P]),
    "cc_trainer_upload_image": (C.c_int, [_P, _F]),
    "cc_trainer_layout": (C.c_int, [_P, C.POINTER(LayoutC)]),
    "cc_trainer_grid_info": (C.c_int, [_P, C.c_int, C.POINTER(GridInfoC)]),
    "cc_trainer_param_info": (C.c_int, [_P, C.c_int, C.POINTER(ParamInfoC)]),
    "cc_trainer_fresh_candidate": (C.c_int, [_P, C.c_int]),
    "cc_trainer_set_state": (C.c_int, [_P, _F, _F, _F, _F, _I64, _F, _F, _I64]),
    "cc_trainer_get_state": (C.c_int, [_P, _F, _F, _F, _F, _I64, _F, _F, _I64]),
    "cc_trainer_get_grads": (C.c_int, [_P, _F, _F]),
    "cc_trainer_get_q": (C.c_int, [_P, _I32]),
    "cc_trainer_get_counters": (C.c_int, [_P, _I64, _I]),
    "cc_trainer_set_counters": (C.c_int, [_P, C.c_int64, C.c_int]),
    "cc_trainer_proxy_iteration": (C.c_int, [_P, C.c_double, C.c_double, C.c_double, _D]),
    "cc_trainer_proxy_iterations": (C.c_int, [_P, C.c_int, _D, _D, _D, _D, _I]),
    "cc_trainer_hardround_iteration": (C.c_int, [_P, C.c_double, C.c_int, _D]),
    "cc_trainer_true_cost": (C.c_int, [_P, _D, _D, _D]),
    "cc_trainer_quantize_all": (C.c_int, [_P]),
    "cc_trainer_load_pads_from_q": (C.c_int, [_P]),
    "cc_trainer_last_terms": (C.c_int, [_P, _D, _D]),
    "cc_trainer_snapshot": (C.c_int, [_P, C.c_int, C.c_double]),
    "cc_trainer_snapshot_cost": (C.c_int, [_P, C.c_int, _D]),
    "cc_trainer_restore": (C.c_int, [_P, C.c_int]),
    "cc_trainer_reset_optimizers": (C.c_int, [_P]),
    "cc_trainer_take_candidate": (C.c_int, [_P, C.c_int, C.c_double]),
    "cc_trainer_load_candidate": (C.c_int, [_P, C.c_int]),
    "cc_trainer_candidate_cost": (C.c_int, [_P, C.c_int, _D]),
    "cc_trainer_warmup": (C.c_int, [_P]),
    "cc_trainer_train": (C.c_int, [_P, C.POINTER(TrainStatsC), _F, _I32, _F]),
    "cc_trainer_set_stream": (C.c_int, [_P, C.c_void_p]),
    "cc_trainer_enqueue_proxy_iterations": (C.c_int, [_P, C.c_int, _D, _D, _D]),
    "cc_trainer_reserve_iterations": (C.c_int, [_P, C.c_int]),
    "cc_trainer_synchronize": (C.c_int, [_P]),
    "cc_trainer_last_records": (C.c_int, [_P, C.c_int, _D]),
}

# include/coolchic_b200_diag.h (product library only)
# include/coolchic_b200_band.h (product only): row-band decomposition (cfg5)
BAND_SIGNATURES = {
    "cc_band_window": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _I, _I]),
    "cc_band_trainer_create": (C.c_int, [_F, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.POINTER(EncoderConfigC), C.POINTER(DecoderConfigC),
                                         C.c_int, C.POINTER(C.c_void_p)]),
    "cc_band_grid_rows": (C.c_int, [_P, C.c_int, _I]),
    "cc_band_rows": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.c_int, _F, C.c_int]),
    "cc_band_device_rows": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p),
                                      C.POINTER(C.c_int64)]),
    "cc_band_device_nn_partial": (C.c_int, [_P, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]),
    "cc_band_forward_backward": (C.c_int, [_P, C.c_double, C.c_double, C.c_double, _D, _D]),
    "cc_band_nn_partial": (C.c_int, [_P, _D]),
    "cc_band_finish": (C.c_int, [_P, _D, C.c_double, C.c_double, _D, _I]),
    "cc_band_step": (C.c_int, [_P, _I]),
    "cc_band_group_local": (C.c_int, [C.POINTER(_P), C.c_int, C.POINTER(_P)]),
    "cc_band_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "cc_band_group_nccl": (C.c_int, [_P, C.c_void_p, C.c_int, C.c_int, _I, C.POINTER(_P)]),
    "cc_band_group_reserve": (C.c_int, [_P, C.c_int]),
    "cc_band_group_enqueue_proxy_iterations": (C.c_int, [_P, C.c_int, _D, _D, _D]),
    "cc_band_group_synchronize": (C.c_int, [_P]),
    "cc_band_group_destroy": (C.c_int, [_P]),
}

# include/coolchic_b200_batch.h (product only): batched images (cfg3)
BATCH_SIGNATURES = {
    "cc_batch_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.POINTER(C.c_void_p)]),
    "cc_batch_destroy": (None, [_P]),
    "cc_batch_reserve_iterations": (C.c_int, [_P, C.c_int]),
    "cc_batch_enqueue_proxy_iterations": (C.c_int, [_P, C.c_int, _D, _D, _D]),
    "cc_batch_synchronize": (C.c_int, [_P]),
}

# include/coolchic_b200_codec.h (product and reference checker): decode passes
CODEC_SIGNATURES = {
    "cc_trainer_set_q": (C.c_int, [_P, C.POINTER(C.c_int32)]),
    "cc_trainer_decode_terms": (C.c_int, [_P, _F, C.c_int, _D, _D]),
    "cc_trainer_latent_mu_sigma": (C.c_int, [_P, _F, _F, _F]),
}

DIAG_SIGNATURES = {
    "ccb_stage_name": (C.c_char_p, [C.c_int]),
    "ccb_profile_stages": (C.c_int, [_P, C.c_int, C.c_double, C.c_double, C.c_double, _D]),
    "ccb_kernels_per_iteration": (C.c_int, [_P, _I]),
    "ccb_arm_flops": (C.c_double, [_P]),
    "ccb_fp32_peak": (C.c_int, [C.c_int, _D, _D]),
    "ccb_eval_math": (C.c_int, [C.c_int, C.c_int, _F, _F, _F, _F]),
    "ccb_counter_gauss": (C.c_int, [C.c_uint64, C.c_uint64, C.c_int, _F]),
    "ccb_timeline": (C.c_int, [_P, C.c_int, C.c_double, C.c_double, C.c_double, _D]),
    "ccb_soap_state": (C.c_int, [_P, _D, _F, _F, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "ccb_soap_set_state": (C.c_int, [_P, _D, _F, _F, C.POINTER(C.c_int64)]),
    "ccb_host_sync_count": (C.c_int, [C.POINTER(C.c_int64)]),
}


def header_symbols(header: str = "coolchic_b200.h") -> list[str]:
    """Function names declared in include/<header> (parsed, not assumed)."""
    import re

    text = (REPO_DIR / "include" / header).read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)  # drop comments
    text = re.sub(r"//[^\n]*", "", text)
    return sorted(set(re.findall(r"\b((?:cc|ccb)_[a-z_0-9]+)\s*\(", text)))


def load_library(path: os.PathLike | str, diag: bool = False) -> C.CDLL:
    lib = C.CDLL(str(path))
    table = dict(SIGNATURES)
    if diag:
        table.update(DIAG_SIGNATURES)
        table.update(BAND_SIGNATURES)
        table.update(BATCH_SIGNATURES)
    for name, (res, args) in table.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    for name, (res, args) in CODEC_SIGNATURES.items():  # absent from the plain-C port
        if hasattr(lib, name):
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
    return lib


_PRODUCT = None


def load_product() -> C.CDLL:
    """Load the sm_100a library.  There is no fallback: a missing build is an error."""
    global _PRODUCT
    if _PRODUCT is None:
        if not PRODUCT_SO.exists():
            raise RuntimeError(
                f"{PRODUCT_SO} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        _PRODUCT = load_library(PRODUCT_SO, diag=True)
    return _PRODUCT

"""The C++ drop-in (include/coolchic_b200.hpp) used the way a coolcodec
encoder would use it: coolcodec::gpu::train vs coolcodec::train on the same
image.  The test binary is compiled against the reference headers
(`make -C oracle dropin`, where /root/reference exists) and travels with the
repo."""
from __future__ import annotations

import json
import subprocess

import pytest

from tests.oracle_util import REF_DIR

pytestmark = pytest.mark.gpu


def test_cpp_dropin_train_matches_reference(gpu_lib):
    exe = REF_DIR / "dropin_train"
    if not exe.exists():
        pytest.skip("oracle/_ref/dropin_train not built (needs /root/reference once)")
    out = subprocess.run([str(exe), "40", "48", "600"], capture_output=True, text=True,
                         timeout=600, check=True).stdout
    r = json.loads(out.strip().splitlines()[-1])
    assert r["gpu_iters"] == r["ref_iters"] == 600
    assert abs(r["gpu_cost"] - r["ref_cost"]) / r["ref_cost"] <= 5e-3


def test_cpp_nn_coding_search_on_gpu_matches_reference(gpu_lib):
    """gpu::select_nn_coding (decode passes on the device) picks the reference's
    quantisation spec on the same trained state; gpu::encode_image runs end to end."""
    exe = REF_DIR / "dropin_nncoding"
    if not exe.exists():
        pytest.skip("oracle/_ref/dropin_nncoding not built (needs /root/reference once)")
    out = subprocess.run([str(exe), "48", "64", "600"], capture_output=True, text=True,
                         timeout=900, check=True).stdout
    r = json.loads(out.strip().splitlines()[-1])
    assert abs(r["gpu_cost"] - r["ref_cost"]) <= 1e-5 * r["ref_cost"]
    assert abs(r["gpu_rate"] - r["ref_rate"]) <= 1e-5 * r["ref_rate"]
    assert abs(r["gpu_mse"] - r["ref_mse"]) <= 1e-5 * r["ref_mse"]
    assert r["same_spec"] == 1 and r["same_payload"] == 1
    assert r["encode_bytes"] > 0 and r["encode_psnr"] > 15
    # latent entropy coding from the device's (mu, sigma) (§8f row 4): the
    # reference's bytes, and the reference decoder reads the image back
    assert r["same_latent_payload"] == 1 and r["latent_decodes"] == 1 and r["latent_bytes"] > 0
    assert r["encode_decodes"] == 1

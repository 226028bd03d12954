"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run here (where /root/reference exists and `make -C oracle ref` built the
checker); the fixtures are committed so GPU-box tests need no reference.

    python tools/make_golden.py
"""
from __future__ import annotations

import ctypes as C
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

from paper_2605_02726_b200 import capi  # noqa: E402
from paper_2605_02726_b200.trainer import DecoderConfig, EncoderConfig, Trainer  # noqa: E402
from tests.oracle_util import load_reference  # noqa: E402

OUT = REPO / "tests" / "golden"

CASES = {
    # name: (h, w, decoder, seed, lambda, zero_latents)
    "hop_48x80": (48, 80, DecoderConfig.hop(), 3, 1e-3, False),
    "lop_37x53": (37, 53, DecoderConfig.lop(), 5, 4e-3, False),
    "mop_33x65": (33, 65, DecoderConfig.mop(), 11, 1e-3, False),
    "vhop_40x56": (40, 56, DecoderConfig.vhop(), 2, 2e-4, False),
    "ablate_40x40": (40, 40, DecoderConfig(preset=2, spatial_ctx=20, ifce_dim=0, arm_width=20,
                                           arm_hidden=2, synth_hidden=48, synth_posts=1,
                                           use_hyperlatents=False, use_stabilizer=False),
                     7, 1e-3, False),
    "cfg4dec_32x48": (32, 48, DecoderConfig(preset=2, spatial_ctx=26, ifce_dim=6, arm_width=20,
                                            arm_hidden=2, synth_hidden=64, synth_posts=2),
                      4, 1e-3, False),
}
SCHED = [(1e-2, 0.35, 0.22), (8e-3, 0.3, 0.2), (5e-3, 0.25, 0.18)]


def run_case(lib, name, h, w, dcfg, seed, lam, zero):
    img = np.empty((3, h, w), np.float32)
    lib.cc_make_synthetic_image(h, w, seed, img.ctypes.data_as(capi._F))
    enc = EncoderConfig(use_soap=False, lmbda=lam, seed=seed)
    tr = Trainer(img, enc, dcfg, lib=lib)
    tr.fresh_candidate(0)
    st0 = tr.get_state()
    if zero:
        st0["latents"][:] = 0
        tr.set_state(st0)
    rec = {"image": img, "init_latents": st0["latents"], "init_params": st0["params"],
           "meta": np.array([h, w, seed], np.int64), "lambda": np.float64(lam),
           "decoder": np.array([getattr(dcfg, f) for f in
                                ("preset", "spatial_ctx", "ifce_dim", "arm_width", "arm_hidden",
                                 "synth_hidden", "synth_posts", "use_hyperlatents",
                                 "use_stabilizer")], np.int64)}
    for k, (lr, t, s) in enumerate(SCHED):
        pre = tr.get_state()
        c = tr.proxy_iteration(lr, t, s)
        m, b = tr.last_terms()
        lg, pg = tr.get_grads()
        post = tr.get_state()
        for key in ("latents", "params", "lat_m", "lat_v", "nn_m", "nn_v"):
            rec[f"it{k}_pre_{key}"] = pre[key]
        rec[f"it{k}_pre_lat_t"] = pre["lat_t"]
        rec[f"it{k}_pre_nn_t"] = pre["nn_t"]
        rec[f"it{k}_pre_global_iter"] = np.int64(pre["global_iter"])
        rec[f"it{k}_scalars"] = np.array([c, m, b], np.float64)
        rec[f"it{k}_lat_grad"] = lg
        rec[f"it{k}_param_grad"] = pg
        rec[f"it{k}_post_latents"] = post["latents"]
        rec[f"it{k}_post_params"] = post["params"]
    tc, psnr, bpp = tr.true_cost()
    rec["true_cost"] = np.array([tc, psnr, bpp], np.float64)
    rec["q"] = tr.get_q()
    rec["final_latents"] = tr.get_state()["latents"]
    rec["final_params"] = tr.get_state()["params"]
    tr.load_pads_from_q()
    hc = tr.hardround_iteration(1e-4, -1)
    _, hpg = tr.get_grads()
    rec["hardround_cost"] = np.float64(hc)
    rec["hardround_param_grad"] = hpg
    rec["hardround_post_params"] = tr.get_state()["params"]
    np.savez_compressed(OUT / f"{name}.npz", **rec)
    print(name, "n_latents", tr.n_latents, "n_params", tr.n_params, "cost", rec["it0_scalars"])


def cfg1_scalars(lib, iters=200):
    """BASELINE config 1: 256x256, HOP, zero latents, 200 Adam iterations at
    lr 1e-2 (T 0.35, sigma 0.22 = the warm-up constants, encoder.hpp:319-320)."""
    h = w = 256
    img = np.empty((3, h, w), np.float32)
    lib.cc_make_synthetic_image(h, w, 0, img.ctypes.data_as(capi._F))
    tr = Trainer(img, EncoderConfig(use_soap=False, lmbda=1e-3, seed=0), DecoderConfig.hop(), lib=lib)
    tr.fresh_candidate(0)
    st = tr.get_state()
    st["latents"][:] = 0
    tr.set_state(st)
    out = np.zeros((iters, 3), np.float64)
    for i in range(iters):
        out[i, 0] = tr.proxy_iteration(1e-2, 0.35, 0.22)
        out[i, 1:] = tr.last_terms()
    tc = np.array(tr.true_cost(), np.float64)
    np.savez_compressed(OUT / "cfg1_scalars.npz", scalars=out, image=img, true_cost=tc,
                        final_q=tr.get_q())
    print("cfg1", out[0], out[-1], tc)


def math_vectors(lib):
    fn = lib.ccref_eval_math
    fn.restype = C.c_int
    fn.argtypes = [C.c_int, C.c_int, capi._F, capi._F, capi._F, capi._F]
    g = lib.ccref_counter_gauss
    g.restype = C.c_int
    g.argtypes = [C.c_uint64, C.c_uint64, C.c_int, capi._F]
    rng = np.random.default_rng(1234)
    n = 4096
    x = np.concatenate([rng.uniform(-100, 100, n // 4), rng.uniform(-3, 3, n // 4),
                        rng.standard_normal(n // 4) * 20, np.linspace(-90, 90, n // 4)])
    x = x.astype(np.float32)
    pos = np.abs(x) + np.float32(1e-6)
    temps = rng.uniform(0.05, 1.0, n).astype(np.float32)
    mu = rng.uniform(-3, 3, n).astype(np.float32)
    sig = np.exp(rng.uniform(np.log(0.06), np.log(256), n)).astype(np.float32)
    vals = np.round(rng.uniform(-12, 12, n)).astype(np.float32)
    qin = np.concatenate([np.array([0.49, 0.51, -1.5, 1.5, -0.49, 300, -300, 0.5, -0.5, 2.5,
                                    -2.5, 254.5, -255.5], np.float32),
                          rng.uniform(-300, 300, n - 13).astype(np.float32)])
    rec = {}
    cases = {0: (np.clip(x, -95, 95), None, None), 1: (pos, None, None), 2: (x / 10, None, None),
             3: (x / 10, temps, None), 4: (vals, mu, sig), 5: (qin, None, None),
             6: (x / 10, temps, None)}
    for f, (a, b, c) in cases.items():
        out = np.empty(n, np.float32)
        a = np.ascontiguousarray(a, np.float32)
        bb = np.ascontiguousarray(b if b is not None else np.zeros(n, np.float32))
        cc = np.ascontiguousarray(c if c is not None else np.zeros(n, np.float32))
        assert fn(f, n, a.ctypes.data_as(capi._F), bb.ctypes.data_as(capi._F),
                  cc.ctypes.data_as(capi._F), out.ctypes.data_as(capi._F)) == 0
        rec[f"fn{f}_a"], rec[f"fn{f}_b"], rec[f"fn{f}_c"], rec[f"fn{f}_out"] = a, bb, cc, out
    go = np.empty(n, np.float32)
    g(0x1234567890ABCDEF, 77, n, go.ctypes.data_as(capi._F))
    rec["gauss_stream"] = np.uint64(0x1234567890ABCDEF)
    rec["gauss_idx0"] = np.uint64(77)
    rec["gauss_out"] = go
    np.savez_compressed(OUT / "math_vectors.npz", **rec)
    print("math vectors", n)


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    lib = load_reference()
    math_vectors(lib)
    for name, args in CASES.items():
        run_case(lib, name, *args)
    cfg1_scalars(lib)


if __name__ == "__main__":
    main()

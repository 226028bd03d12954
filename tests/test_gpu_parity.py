"""Parity of the sm_100a path (through the C ABI) with the reference.

Checkers: the committed golden fixtures (always available) and, where its
prebuilt .so travelled with the repo, the reference itself (oracle/_ref) for
cases generated on the fly.  Tolerances are the north star's: quantised
latents bit-exact for identical float latents; per-iteration rate,
distortion and per-tensor gradients within 1e-4 relative (lock-step);
scalars of the first 50 free-running iterations within 1e-4.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from paper_2605_02726_b200 import capi
from paper_2605_02726_b200.trainer import DecoderConfig, EncoderConfig, Trainer
from tests import golden_util
from tests.conftest import GOLDEN, make_image, rel_l2

pytestmark = pytest.mark.gpu


def _dev_math(lib, fn, a, b=None, c=None):
    n = len(a)
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b if b is not None else np.zeros(n), np.float32)
    c = np.ascontiguousarray(c if c is not None else np.zeros(n), np.float32)
    out = np.empty(n, np.float32)
    assert lib.ccb_eval_math(fn, n, a.ctypes.data_as(capi._F), b.ctypes.data_as(capi._F),
                             c.ctypes.data_as(capi._F), out.ctypes.data_as(capi._F)) == 0
    return out


def test_device_math_vs_reference_vectors(gpu_lib):
    g = dict(np.load(golden_util.GOLDEN / "math_vectors.npz"))
    for f in range(7):
        out = _dev_math(gpu_lib, f, g[f"fn{f}_a"], g[f"fn{f}_b"], g[f"fn{f}_c"])
        ref = g[f"fn{f}_out"]
        if f == 5:  # quantiser: bit-exact
            assert np.array_equal(out, ref)
        else:
            exact = np.mean(out == ref)
            assert np.allclose(out, ref, rtol=2e-6, atol=1e-7), (f, exact)
    go = np.empty(len(g["gauss_out"]), np.float32)
    assert gpu_lib.ccb_counter_gauss(int(g["gauss_stream"]), int(g["gauss_idx0"]), len(go),
                                     go.ctypes.data_as(capi._F)) == 0
    # double Box-Muller: CUDA log/cos are within 1-2 ulp of libm
    assert np.allclose(go, g["gauss_out"], rtol=1e-6, atol=1e-7)
    assert np.mean(go == g["gauss_out"]) > 0.99


@pytest.mark.parametrize("case", golden_util.CASES)
def test_lockstep_vs_golden(gpu_lib, case):
    rep = golden_util.replay(gpu_lib, case, iters=3)
    golden_util.assert_report(rep, exact_init=True)


def test_cfg1_free_running_vs_golden(gpu_lib):
    """BASELINE config 1: 256x256, HOP, zero-initialised latents, 200 Adam
    iterations at lr 1e-2 — per-iteration cost / mse / bits vs the reference."""
    g = dict(np.load(golden_util.GOLDEN / "cfg1_scalars.npz"))
    with Trainer(g["image"], EncoderConfig(use_soap=False, lmbda=1e-3, seed=0), DecoderConfig.hop(),
                 lib=gpu_lib) as tr:
        tr.fresh_candidate(0)
        st = tr.get_state()
        st["latents"][:] = 0
        tr.set_state(st)
        n = len(g["scalars"])
        ours = np.zeros((n, 3))
        for i in range(n):
            ours[i, 0] = tr.proxy_iteration(1e-2, 0.35, 0.22)
            ours[i, 1:] = tr.last_terms()
        err = np.abs(ours - g["scalars"]) / np.abs(g["scalars"])
        assert err[:50].max() <= 1e-4, err[:50].max(axis=0)
        # Beyond 50 iterations free-running trajectories drift chaotically: two
        # builds of the reference itself that differ only in FMA contraction
        # reach 3.3e-4 on bits by iteration 199.  The remaining
        # iterations are held to a drift bound, not to the 1e-4 bar.
        assert err[50:].max() <= 1e-2, err.max(axis=0)
        tc = tr.true_cost()
        assert abs(tc[0] - g["true_cost"][0]) / g["true_cost"][0] <= 1e-3


class TruthArbiter:
    """Per-tensor gradient agreement between the device and the reference's
    float Trainer on an identical state, with the fp64 truth as the arbiter.

    rel-L2(device, reference) <= tol passes directly.  Otherwise the truth of
    the same state is computed (ccref_truth_grads) and
      * latent grids: "kink" latents — where the device or the reference is off
        the truth by more than 1 % of the grid's RMS gradient, i.e. an fp32
        threshold branch (ReLU, probability floor) resolved differently from
        fp64 — are excluded (at most 10 + 1e-4 of the grid), and the rest must
        agree within tol;
      * any tensor passes if the device is at least as close to the truth as
        the reference (within 1.25x) or within tol of the truth.
    Every arbitrated tensor is recorded in `notes`."""

    def __init__(self, ref_lib, img, enc, dcfg, tol=1e-4):
        self.ref_lib, self.img, self.enc, self.dcfg, self.tol = ref_lib, img, enc, dcfg, tol
        self.notes = []
        self.worst = 0.0

    def _truth(self, st, temp, noise):
        from tests.oracle_util import truth_grads

        with Trainer(self.img, self.enc, self.dcfg, lib=self.ref_lib) as tr:
            tr.fresh_candidate(0)
            tr.set_state(st)
            lt, pt, _ = truth_grads(self.ref_lib, tr, temp, noise)
        return lt, pt

    def check(self, tr_r, st, temp, noise, lg, pg, lr_, pr_, tag=""):
        truth = None
        for kind, n in (("grid", len(tr_r.grids)), ("param", len(tr_r.params))):
            for i in range(n):
                view = tr_r.grid_view if kind == "grid" else tr_r.param_view
                g, r = view(lg if kind == "grid" else pg, i).ravel(), view(lr_ if kind == "grid" else pr_, i).ravel()
                e = rel_l2(g, r)
                if e <= self.tol:
                    self.worst = max(self.worst, e)
                    continue
                if truth is None:
                    truth = self._truth(st, temp, noise)
                t = view(truth[0] if kind == "grid" else truth[1], i).ravel()
                name = f"grid{i}" if kind == "grid" else tr_r.params[i].name
                eg, er = rel_l2(g, t), rel_l2(r, t)
                rest, nk = e, 0
                if kind == "grid":
                    rms = np.sqrt(np.mean(t * t))
                    kink = np.maximum(np.abs(g - t), np.abs(r - t)) > 1e-2 * rms
                    nk = int(kink.sum())
                    assert nk <= 10 + 1e-4 * t.size, (tag, name, nk)
                    rest = rel_l2(g[~kink], r[~kink])
                ok = rest <= self.tol or eg <= self.tol or eg <= 1.25 * er
                self.notes.append((tag, name, e, rest, nk, eg, er))
                assert ok, (tag, name, e, rest, nk, eg, er)


@pytest.mark.parametrize("h,w,preset", [(64, 96, "hop"), (256, 256, "hop"), (45, 71, "lop"),
                                        (512, 768, "hop")])
def test_lockstep_vs_reference(gpu_lib, ref_lib, h, w, preset):
    """Device vs the reference's float Trainer on an identical state, two
    iterations.  (At the cfg4 size the reference's own fp32 weight-gradient
    sums drift from the truth by up to 7e-3, so cfg4 is held against the fp64
    truth instead: test_grads_vs_fp64_truth.)"""
    img = make_image(ref_lib, h, w, seed=h + w)
    enc = EncoderConfig(use_soap=False, lmbda=1e-3, seed=h)
    dcfg = DecoderConfig.from_name(preset)
    arb = TruthArbiter(ref_lib, img, enc, dcfg)
    with Trainer(img, enc, dcfg, lib=ref_lib) as tr_r, Trainer(img, enc, dcfg, lib=gpu_lib) as tr_g:
        tr_r.fresh_candidate(1)
        tr_g.fresh_candidate(1)
        for it in range(2):
            st = tr_r.get_state()
            tr_g.set_state(st)
            cr = tr_r.proxy_iteration(1e-2, 0.35, 0.22)
            cg = tr_g.proxy_iteration(1e-2, 0.35, 0.22)
            assert abs(cr - cg) / abs(cr) <= 1e-6
            (mr, br), (mg, bg) = tr_r.last_terms(), tr_g.last_terms()
            assert abs(mr - mg) / mr <= 1e-6 and abs(br - bg) / br <= 1e-6
            lr_, pr_ = tr_r.get_grads()
            lg_, pg_ = tr_g.get_grads()
            arb.check(tr_r, st, 0.35, 0.22, lg_, pg_, lr_, pr_, tag=f"it{it}")
            assert tr_g.global_iter == tr_r.global_iter


def test_lockstep_50_iterations_cfg1(gpu_lib, ref_lib):
    """North star: per-iteration rate, distortion and gradients within 1e-4
    over the first 50 iterations, at BASELINE config 1 (256x256, HOP,
    zero-initialised latents, lr 1e-2, T 0.35, sigma 0.22).  Teacher-forced:
    before every iteration the reference's full state (latents, parameters,
    Adam moments and step counts, global_iter) is loaded into the device
    trainer, because free-running fp32 trajectories diverge chaotically
    (SURVEY 8(c)); after it, cost / mse / bits and every latent-grid and
    NN-tensor gradient are compared."""
    img = make_image(ref_lib, 256, 256, seed=0)
    enc = EncoderConfig(use_soap=False, lmbda=1e-3, seed=0)
    dcfg = DecoderConfig.hop()
    worst_s = 0.0
    arb = TruthArbiter(ref_lib, img, enc, dcfg)
    with Trainer(img, enc, dcfg, lib=ref_lib) as tr_r, Trainer(img, enc, dcfg, lib=gpu_lib) as tr_g:
        tr_r.fresh_candidate(0)
        tr_g.fresh_candidate(0)
        st = tr_r.get_state()
        st["latents"][:] = 0
        tr_r.set_state(st)
        for it in range(50):
            st = tr_r.get_state()
            tr_g.set_state(st)
            cr = tr_r.proxy_iteration(1e-2, 0.35, 0.22)
            cg = tr_g.proxy_iteration(1e-2, 0.35, 0.22)
            for a, b in zip((cg, *tr_g.last_terms()), (cr, *tr_r.last_terms())):
                worst_s = max(worst_s, abs(a - b) / abs(b))
            lr_, pr_ = tr_r.get_grads()
            lg_, pg_ = tr_g.get_grads()
            arb.check(tr_r, st, 0.35, 0.22, lg_, pg_, lr_, pr_, tag=f"it{it}")
            assert tr_g.global_iter == tr_r.global_iter
    print(f"cfg1 50-iteration lock-step: scalars {worst_s:.2e}, gradients within 1e-4 of the reference "
          f"(worst {arb.worst:.2e}) except {len(arb.notes)} truth-arbitrated tensors "
          "(tag, tensor, vs-ref, vs-ref w/o kinks, kinks, gpu-vs-truth, ref-vs-truth):")
    for n in arb.notes:
        print("   ", n)
    assert worst_s <= 1e-6


def truth_report(gpu_lib, ref_lib, h, w, preset, seed=0, warm=1):
    """Gradients of one proxy iteration on an identical state from (a) the
    B200 library, (b) the reference's float Trainer, (c) the fp64 truth (the
    reference's templated kernels in double, oracle/ref_capi.cpp
    ccref_truth_grads).

    Returns per tensor: rel-L2 of (a) and (b) vs (c) over ALL positions, and
    for latent grids the "kink" positions — where the gpu or the reference
    float gradient is off the truth by more than 1 % of the grid's RMS
    gradient.  Those are latents whose gradient crosses a threshold branch
    (a ReLU of the synthesis or the ARM, the 2^-16 probability floor) that an
    fp32 evaluation resolves differently from fp64 by an ulp of its input
    (one synthesis ReLU flip changes one full-resolution latent's gradient by
    up to ~50 %), and the rel-L2 over the remaining positions."""
    from tests.oracle_util import truth_grads

    img = make_image(ref_lib, h, w, seed=h + w + seed)
    enc = EncoderConfig(use_soap=False, lmbda=1e-3, seed=h + seed)
    dcfg = DecoderConfig.from_name(preset)
    out = {"all": {"gpu": {}, "ref": {}}, "rest": {"gpu": {}, "ref": {}}, "kinks": {},
           "scalars_gpu": None, "scalars_ref": None}
    with Trainer(img, enc, dcfg, lib=ref_lib) as tr_r, Trainer(img, enc, dcfg, lib=gpu_lib) as tr_g:
        tr_r.fresh_candidate(1)
        tr_g.fresh_candidate(1)
        for _ in range(warm):  # off the initial state (zero NN biases)
            tr_r.proxy_iteration(1e-2, 0.35, 0.22)
        tr_g.set_state(tr_r.get_state())
        lt, pt, st = truth_grads(ref_lib, tr_r, 0.3, 0.2)
        cr = tr_r.proxy_iteration(1e-2, 0.3, 0.2)
        cg = tr_g.proxy_iteration(1e-2, 0.3, 0.2)
        out["scalars_ref"] = [abs(a - b) / abs(b) for a, b in zip((cr, *tr_r.last_terms()), st)]
        out["scalars_gpu"] = [abs(a - b) / abs(b) for a, b in zip((cg, *tr_g.last_terms()), st)]
        lg, pg = tr_g.get_grads()
        lr_, pr_ = tr_r.get_grads()
        for gi in range(len(tr_r.grids)):
            t = tr_r.grid_view(lt, gi).ravel()
            g = tr_g.grid_view(lg, gi).ravel()
            r = tr_r.grid_view(lr_, gi).ravel()
            rms = np.sqrt(np.mean(t * t)) if t.size else 0.0
            kink = np.maximum(np.abs(g - t), np.abs(r - t)) > 1e-2 * rms
            key = f"grid{gi}"
            out["all"]["gpu"][key] = rel_l2(g, t)
            out["all"]["ref"][key] = rel_l2(r, t)
            out["rest"]["gpu"][key] = rel_l2(g[~kink], t[~kink])
            out["rest"]["ref"][key] = rel_l2(r[~kink], t[~kink])
            cols = tr_r.grids[gi].cols
            out["kinks"][key] = [(int(i) // cols, int(i) % cols, float(g[i]), float(r[i]), float(t[i]))
                                 for i in np.flatnonzero(kink)]
            out.setdefault("size", {})[key] = int(t.size)
        for ti, p in enumerate(tr_r.params):
            t = tr_r.param_view(pt, ti)
            out["all"]["gpu"][p.name] = rel_l2(tr_g.param_view(pg, ti), t)
            out["all"]["ref"][p.name] = rel_l2(tr_r.param_view(pr_, ti), t)
    return out


@pytest.mark.parametrize("h,w,preset", [(256, 256, "hop"), (512, 768, "hop"), (1360, 2048, "cfg4")])
def test_grads_vs_fp64_truth(gpu_lib, ref_lib, h, w, preset):
    """Gradient parity against the fp64 truth at cfg1 / cfg2 and at the cfg4
    size and decoder (1360x2048, 3.7 M latents):
      * every NN tensor within 1e-4 (relative L2), nothing dropped — the
        reference's own float weight gradients (sequential fp32 sums over all
        latents, layers.hpp:131-145) miss this at cfg4, the device's per-tile
        fp64 sums do not;
      * every latent grid within 1e-4 over all positions except the listed
        threshold-branch "kink" latents (see truth_report; at most 1e-4 of
        the grid + 10, printed with their device / reference / truth values)
        — or, where the reference's own float evaluation is itself further
        than 1e-4 from the truth on that grid, no further than 1.25x the
        reference's error;
      * cost / mse / bits within 1e-6."""
    rep = truth_report(gpu_lib, ref_lib, h, w, preset)
    ga, ra = rep["all"]["gpu"], rep["all"]["ref"]
    print(f"{h}x{w} {preset}: scalars gpu {max(rep['scalars_gpu']):.1e} ref {max(rep['scalars_ref']):.1e}")
    for k in ga:
        line = f"  {k:14s} all: gpu {ga[k]:.2e} ref {ra[k]:.2e}"
        if k in rep["kinks"]:
            line += (f"  rest: gpu {rep['rest']['gpu'][k]:.2e} ref {rep['rest']['ref'][k]:.2e}"
                     f"  kinks {len(rep['kinks'][k])} {rep['kinks'][k][:4]}")
        print(line)
    assert max(rep["scalars_gpu"]) <= 1e-6
    bad = {k: v for k, v in ga.items() if not k.startswith("grid") and not v <= 1e-4}
    assert not bad, bad
    for k, kk in rep["kinks"].items():
        eg, er = rep["rest"]["gpu"][k], rep["rest"]["ref"][k]
        assert eg <= 1e-4 or eg <= 1.25 * er, (k, eg, er)
        assert len(kk) <= 10 + 1e-4 * rep["size"][k], (k, len(kk))


def test_quantize_bit_exact_for_identical_latents(gpu_lib, ref_lib):
    img = make_image(ref_lib, 96, 128, seed=1)
    enc = EncoderConfig(use_soap=False)
    with Trainer(img, enc, DecoderConfig.hop(), lib=ref_lib) as tr_r, \
            Trainer(img, enc, DecoderConfig.hop(), lib=gpu_lib) as tr_g:
        tr_r.fresh_candidate(0)
        tr_g.fresh_candidate(0)
        rng = np.random.default_rng(3)
        y = rng.uniform(-300, 300, tr_r.n_latents).astype(np.float32)
        k = min(2000, len(y))
        y[:k] = np.round(rng.uniform(-20, 20, k)) + rng.choice([-0.5, 0.5], k)  # exact ties
        y[k:k + 8] = [0.49, 0.51, -1.5, 1.5, -0.49, 255.5, -255.5, 0.0]
        tr_r.set_state({"latents": y})
        tr_g.set_state({"latents": y})
        tr_r.quantize_all()
        tr_g.quantize_all()
        assert np.array_equal(tr_r.get_q(), tr_g.get_q())


def test_hardround_freezes_latents_bit_exact(gpu_lib):
    # tests/test_encoder.cpp:81-103
    img = make_image(gpu_lib, 32, 32, seed=21)
    with Trainer(img, EncoderConfig(use_soap=False, lmbda=1e-3, seed=2), DecoderConfig.lop(), lib=gpu_lib) as tr:
        tr.fresh_candidate(0)
        for _ in range(20):
            tr.proxy_iteration(1e-2, 0.3, 0.2)
        tr.quantize_all()
        tr.load_pads_from_q()
        y0, q0 = tr.get_state()["latents"].copy(), tr.get_q().copy()
        for _ in range(30):
            tr.hardround_iteration(1e-4)
        assert np.array_equal(tr.get_state()["latents"], y0)
        assert np.array_equal(tr.get_q(), q0)


def test_bitwise_determinism(gpu_lib):
    # tests/test_encoder.cpp:27-54: no float atomics -> identical bits
    img = make_image(gpu_lib, 80, 120, seed=5)
    outs = []
    for _ in range(2):
        with Trainer(img, EncoderConfig(use_soap=False, lmbda=4e-3, seed=17), DecoderConfig.hop(),
                     lib=gpu_lib) as tr:
            tr.fresh_candidate(0)
            costs = tr.proxy_iterations(np.full(25, 1e-2), 0.35, 0.22)
            st = tr.get_state()
            outs.append((costs, st["latents"], st["params"], tr.get_grads()[1]))
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)


def test_more_trainers_than_constant_slots(gpu_lib, ref_lib):
    """The constant-bank ARM hands out 8 constant slots exclusively; a ninth
    live trainer runs the FFMA2 tile ARM on the same launch geometry.  Both
    match the reference lock-step (the golden-free 64x96 HOP iteration), the
    slot-less one also after the others are gone, and slots are reused."""
    img = make_image(gpu_lib, 64, 96, seed=4)
    enc = EncoderConfig(use_soap=False, lmbda=1e-3, seed=3)
    with Trainer(img, enc, DecoderConfig.hop(), lib=ref_lib) as tr_r:
        tr_r.fresh_candidate(0)
        ref = [tr_r.proxy_iteration(1e-2, 0.35, 0.22) for _ in range(3)]
    trs = [Trainer(img, enc, DecoderConfig.hop(), lib=gpu_lib) for _ in range(9)]
    try:
        for t in (trs[0], trs[8]):  # a slot holder and the slot-less ninth
            t.fresh_candidate(0)
            got = [t.proxy_iteration(1e-2, 0.35, 0.22) for _ in range(3)]
            assert np.allclose(got, ref, rtol=1e-5, atol=0), (got, ref)
    finally:
        for t in trs:
            t.close()
    for _ in range(10):  # released slots are handed out again
        with Trainer(img, enc, DecoderConfig.hop(), lib=gpu_lib) as t:
            t.fresh_candidate(0)
            assert abs(t.proxy_iteration(1e-2, 0.35, 0.22) - ref[0]) <= 1e-5 * abs(ref[0])


def test_nonfinite_cost_returned_not_stepped(gpu_lib):
    # encoder.hpp:118: a non-finite cost is returned; no step, global_iter kept
    img = make_image(gpu_lib, 32, 48, seed=2)
    img[1, 5, 7] = np.nan  # a NaN target pixel makes the MSE (and the cost) NaN
    with Trainer(img, EncoderConfig(use_soap=False), DecoderConfig.hop(), lib=gpu_lib) as tr:
        tr.fresh_candidate(0)
        st = tr.get_state()
        g0 = tr.global_iter
        c = tr.proxy_iteration(1e-2, 0.35, 0.22)
        assert not np.isfinite(c)
        assert tr.global_iter == g0
        st2 = tr.get_state()
        assert np.array_equal(st2["latents"], st["latents"])
        assert np.array_equal(st2["params"], st["params"])
        lg, _ = tr.get_grads()
        assert not lg.any()


@pytest.mark.parametrize("inject", ["image_nan", "latent_inf", "latent_nan", "param_nan"])
def test_nonfinite_behaviour_matches_reference(gpu_lib, ref_lib, inject):
    """Same error behaviour as the reference for non-finite inputs: returned
    (not thrown) costs, per-tensor Adam skips counted in skipped_steps
    (optim.hpp:38-41, encoder.hpp:129-132), untouched state on a NaN cost."""
    img = make_image(ref_lib, 32, 48, seed=2)
    if inject == "image_nan":
        img[0, 3, 4] = np.nan
    enc, dcfg = EncoderConfig(use_soap=False, lmbda=1e-3, seed=3), DecoderConfig.hop()
    with Trainer(img, enc, dcfg, lib=ref_lib) as tr_r, Trainer(img, enc, dcfg, lib=gpu_lib) as tr_g:
        tr_r.fresh_candidate(0)
        st = tr_r.get_state()
        if inject == "latent_inf":
            st["latents"][tr_r.grids[0].offset] = np.inf
        if inject == "latent_nan":
            st["latents"][tr_r.grids[4].offset + 1] = np.nan
        if inject == "param_nan":
            st["params"][tr_r.params[14].offset + 1] = np.nan  # an upsampling tap
        tr_r.set_state(st)
        tr_g.fresh_candidate(0)
        tr_g.set_state(st)
        for _ in range(2):
            cr = tr_r.proxy_iteration(1e-2, 0.35, 0.22)
            cg = tr_g.proxy_iteration(1e-2, 0.35, 0.22)
            assert np.isfinite(cr) == np.isfinite(cg)
            if np.isfinite(cr):
                assert abs(cr - cg) <= 1e-4 * abs(cr)
            assert tr_r.counters() == tr_g.counters()
            sr, sg = tr_r.get_state(), tr_g.get_state()
            assert np.array_equal(np.isfinite(sr["latents"]), np.isfinite(sg["latents"]))
            assert np.array_equal(np.isfinite(sr["params"]), np.isfinite(sg["params"]))


def test_warmup_budget_and_candidates(gpu_lib):
    # tests/test_encoder.cpp:56-79
    img = make_image(gpu_lib, 32, 32, seed=9)
    enc = EncoderConfig(use_soap=False, warmup_candidates=5, warmup_keep=2, warmup_iters=6, main_iters=1,
                        hardround_iters=1, lmbda=1e-3, seed=5)
    with Trainer(img, enc, DecoderConfig.lop(), lib=gpu_lib) as tr:
        tr.warmup()
        assert tr.global_iter == (5 + 2) * 6
        assert np.isfinite(tr.true_cost()[0])
    enc1 = EncoderConfig(use_soap=False, warmup_candidates=1, warmup_keep=2, warmup_iters=6, main_iters=1,
                         hardround_iters=1, lmbda=1e-3, seed=5)
    with Trainer(img, enc1, DecoderConfig.lop(), lib=gpu_lib) as tr:
        tr.warmup()
        assert tr.global_iter == 6


def test_full_train_final_rd_within_half_percent(gpu_lib, ref_lib):
    """Full with_total schedule (warm-up, main stage with true-cost snapshots,
    hardround) through cc_trainer_train vs the reference train(): final true
    RD cost within 0.5 % (north star)."""
    img = make_image(ref_lib, 40, 48, seed=3)
    enc = EncoderConfig.with_total(600)
    enc.lmbda, enc.seed, enc.use_soap, enc.true_cost_interval = 1e-3, 4, False, 50
    with Trainer(img, enc, DecoderConfig.lop(), lib=ref_lib) as tr_r:
        rr = tr_r.train()
    with Trainer(img, enc, DecoderConfig.lop(), lib=gpu_lib) as tr_g:
        rg = tr_g.train()
    assert rg.stats.iterations == rr.stats.iterations == enc.total_iters()
    assert abs(rg.stats.true_cost - rr.stats.true_cost) / rr.stats.true_cost <= 5e-3
    assert np.all(np.abs(rg.q) <= 255)


def test_constant_image_near_lossless(gpu_lib):
    # tests/test_encoder.cpp:12-25
    img = np.full((3, 64, 64), 0.42, np.float32)
    enc = EncoderConfig.with_total(2000)
    enc.lmbda, enc.seed = 1e-3, 1
    with Trainer(img, enc, DecoderConfig.lop(), lib=gpu_lib) as tr:
        r = tr.train()
    assert r.stats.rate_bpp <= 0.05
    assert r.stats.psnr >= 45.0
    assert r.stats.iterations == enc.total_iters()


def test_cfg2_size_properties(gpu_lib):
    """BASELINE config 2 size (512x768): size-independent properties of a
    short run — finite and decreasing cost, |q| <= 255, determinism of the
    per-iteration records."""
    img = make_image(gpu_lib, 512, 768, seed=0)
    enc = EncoderConfig.with_total(10000)
    enc.lmbda, enc.seed, enc.use_soap = 1e-3, 0, False
    with Trainer(img, enc, DecoderConfig.hop(), lib=gpu_lib) as tr:
        tr.fresh_candidate(0)
        c = tr.proxy_iterations(np.full(40, 1e-2), 0.35, 0.22)
        assert np.all(np.isfinite(c))
        assert c[-1] < c[0]
        tc, psnr, bpp = tr.true_cost()
        assert np.isfinite(tc) and bpp > 0
        q = tr.get_q()
        assert np.abs(q).max() <= 255


def _soap_state(lib, tr):
    n = C.c_int64()
    assert lib.ccb_soap_state(tr._h, None, None, None, None, C.byref(n)) == 0
    arena = np.empty(n.value, np.float64)
    m1 = np.empty(tr.n_params, np.float32)
    v2 = np.empty(tr.n_params, np.float32)
    t = np.empty(len(tr.params), np.int64)
    assert lib.ccb_soap_state(tr._h, arena.ctypes.data_as(C.POINTER(C.c_double)),
                              m1.ctypes.data_as(C.POINTER(C.c_float)),
                              v2.ctypes.data_as(C.POINTER(C.c_float)),
                              t.ctypes.data_as(C.POINTER(C.c_int64)), None) == 0
    mats, pos = [], 0
    for p in tr.params:  # per tensor: L (r x r), R (c x c), QL, QR
        r, c = p.rows, p.cols
        L = arena[pos:pos + r * r].reshape(r, r); pos += r * r
        R = arena[pos:pos + c * c].reshape(c, c); pos += c * c
        QL = arena[pos:pos + r * r].reshape(r, r); pos += r * r
        QR = arena[pos:pos + c * c].reshape(c, c); pos += c * c
        mats.append((L, R, QL, QR))
    return mats, m1, v2, t


def test_soap_step_matches_restatement(gpu_lib):
    """use_soap = true (the reference default, config.hpp:107): one device SOAP
    step against a numpy restatement of soap_step (optim.hpp:189-250) on the
    SAME inputs (state read back before the step, gradients after it), at a
    step without an eigenbasis refresh; then the refreshed eigenbases at
    t = 11 are orthonormal and diagonalise their preconditioners (the cyclic
    Jacobi of optim.hpp:60-106)."""
    img = make_image(gpu_lib, 64, 96, seed=7)
    enc = EncoderConfig(lmbda=1e-3, seed=5, use_soap=True)
    lr = 1e-2
    with Trainer(img, enc, DecoderConfig.hop(), lib=gpu_lib) as tr:
        tr.fresh_candidate(0)
        for _ in range(3):
            tr.proxy_iteration(lr, 0.35, 0.22)
        mats0, m10, v20, t0 = _soap_state(gpu_lib, tr)
        p0 = tr.get_state()["params"]
        tr.proxy_iteration(lr, 0.35, 0.22)
        _, G = tr.get_grads()
        mats1, m11, v21, t1 = _soap_state(gpu_lib, tr)
        p1 = tr.get_state()["params"]
        assert np.all(t1 == t0 + 1) and np.all(t1 == 4)
        for ti, p in enumerate(tr.params):
            r, c = p.rows, p.cols
            g = tr.param_view(G, ti).astype(np.float64).reshape(r, c)
            L0, R0, QL0, QR0 = mats0[ti]
            L1, R1, QL1, QR1 = mats1[ti]
            assert np.allclose(L1, 0.95 * L0 + 0.05 * g @ g.T, rtol=1e-12, atol=1e-300), p.name
            assert np.allclose(R1, 0.95 * R0 + 0.05 * g.T @ g, rtol=1e-12, atol=1e-300), p.name
            assert np.array_equal(QL1, QL0) and np.array_equal(QR1, QR0)  # no refresh at t = 4
            gp = QL0.T @ g @ QR0
            m1 = 0.9 * tr.param_view(m10, ti).astype(np.float64).reshape(r, c) + 0.1 * g
            v2 = 0.999 * tr.param_view(v20, ti).astype(np.float64).reshape(r, c) + 0.001 * gp * gp
            bc1, bc2 = 1 - 0.9 ** 4, 1 - 0.999 ** 4
            m1p = QL0.T @ m1 @ QR0
            upd = QL0 @ ((m1p / bc1) / (np.sqrt(v2 / bc2) + 1e-8)) @ QR0.T
            exp = tr.param_view(p0, ti).astype(np.float64) - lr * upd.reshape(-1)
            got = tr.param_view(p1, ti).astype(np.float64)
            step = np.linalg.norm(lr * upd)
            tol = 1e-5 * step + 2.0 ** -23 * np.linalg.norm(exp)  # + the fp32 rounding of p
            assert np.linalg.norm(got - exp) <= tol, (p.name, np.linalg.norm(got - exp), step)
        for _ in range(7):  # to t = 11: eigenbasis refresh
            tr.proxy_iteration(lr, 0.35, 0.22)
        mats, _, _, t = _soap_state(gpu_lib, tr)
        assert np.all(t == 11)
        for (L, R, QL, QR), p in zip(mats, tr.params):
            for A, Q in ((L, QL), (R, QR)):
                n = A.shape[0]
                assert np.abs(Q.T @ Q - np.eye(n)).max() <= 1e-12, p.name
                D = Q.T @ A @ Q
                off = np.abs(D - np.diag(np.diag(D))).max()
                assert off <= 1e-10 * max(np.abs(A).max(), 1e-300), (p.name, off)


@pytest.mark.parametrize("h,w,preset", [(64, 96, "hop"), (256, 256, "hop")])
def test_soap_lockstep_vs_reference(gpu_lib, ref_lib, h, w, preset):
    """SOAP (the reference default) teacher-forced against the reference's
    own soap_step (optim.hpp:189-254, via NnOptimizer::step optim.hpp:277-286):
    before each iteration the reference's latents, parameters, latent Adam
    state and full SOAP state (L, R EMAs, eigenbases QL / QR, m1, v2, t;
    optim.hpp:122-141) are loaded into the device trainer; both take one
    proxy iteration.  Steps t = 12..20 (no eigenbasis refresh) and the refresh
    step t = 21 are compared: every parameter's update (p_after - p_before)
    and the post-step preconditioner EMAs and moments within 1e-4 (relative
    L2 per tensor).  At the refresh step the new eigenbases are compared as
    subspaces only for eigenvalues separated by > 1e-6 of the spectrum (a
    basis inside a degenerate eigenspace is arbitrary for Jacobi)."""
    from tests.test_oracle import _soap_io, _soap_load

    for name in ("ccb_soap_state", "ccb_soap_set_state"):
        getattr(ref_lib, name).restype = C.c_int
    img = make_image(ref_lib, h, w, seed=5)
    enc = EncoderConfig(use_soap=True, lmbda=1e-3, seed=5)
    dcfg = DecoderConfig.from_name(preset)
    worst = {"dp": (0.0, ""), "L": 0.0, "m1": 0.0, "v2": 0.0}
    with Trainer(img, enc, dcfg, lib=ref_lib) as tr_r, Trainer(img, enc, dcfg, lib=gpu_lib) as tr_g:
        tr_r.fresh_candidate(0)
        tr_g.fresh_candidate(0)
        for _ in range(11):
            tr_r.proxy_iteration(1e-2, 0.35, 0.22)
        for it in range(10):  # SOAP steps t = 12 .. 21 (t = 21 refreshes the bases)
            st = tr_r.get_state()
            tr_g.set_state(st)
            _soap_load(gpu_lib, tr_g, _soap_io(ref_lib, tr_r))
            p0 = st["params"].astype(np.float64)
            cr = tr_r.proxy_iteration(5e-3, 0.3, 0.2)
            cg = tr_g.proxy_iteration(5e-3, 0.3, 0.2)
            assert abs(cr - cg) / abs(cr) <= 1e-6
            dr = tr_r.get_state()["params"].astype(np.float64) - p0
            dg = tr_g.get_state()["params"].astype(np.float64) - p0
            sr, sg = _soap_io(ref_lib, tr_r), _soap_io(gpu_lib, tr_g)
            assert np.array_equal(sr["t"], sg["t"]) and np.all(sr["t"] == 12 + it)
            refresh = (12 + it - 1) % 10 == 0
            pos = 0
            for ti, p in enumerate(tr_r.params):
                sl = slice(p.offset, p.offset + p.size)
                r, c = p.rows, p.cols
                blocks = {}
                for nm, n in (("L", r * r), ("R", c * c), ("QL", r * r), ("QR", c * c)):
                    blocks[nm] = (sr["arena"][pos:pos + n], sg["arena"][pos:pos + n])
                    pos += n
                worst["L"] = max(worst["L"], rel_l2(blocks["L"][1], blocks["L"][0]),
                                 rel_l2(blocks["R"][1], blocks["R"][0]))
                worst["m1"] = max(worst["m1"], rel_l2(sg["m1"][sl], sr["m1"][sl]))
                if not refresh:
                    assert np.array_equal(blocks["QL"][0], blocks["QL"][1]), p.name
                    worst["v2"] = max(worst["v2"], rel_l2(sg["v2"][sl], sr["v2"][sl]))
                    e = rel_l2(dg[sl], dr[sl])
                    if e > worst["dp"][0]:
                        worst["dp"] = (e, f"{p.name}@t{12 + it}")
                else:
                    for nm, n in (("QL", r), ("QR", c)):
                        A = blocks["L" if nm == "QL" else "R"][0].reshape(n, n)
                        Qr, Qg = (x.reshape(n, n) for x in blocks[nm])
                        ev = np.linalg.eigvalsh(A)
                        scale = max(np.abs(ev).max(), 1e-300)
                        dr_ = Qr.T @ A @ Qr
                        for j in range(n):  # eigenvector j of the reference basis
                            lam = dr_[j, j]
                            if np.min(np.abs(np.delete(ev, np.argmin(np.abs(ev - lam))) - lam),
                                      initial=np.inf) > 1e-6 * scale:
                                cos = abs(Qr[:, j] @ Qg[:, j])
                                assert cos >= 1 - 1e-6, (p.name, nm, j, cos)
    print(f"SOAP lock-step {h}x{w}: worst update {worst['dp']}, L/R {worst['L']:.2e}, "
          f"m1 {worst['m1']:.2e}, v2 {worst['v2']:.2e}")
    assert worst["dp"][0] <= 1e-4, worst["dp"]
    assert worst["L"] <= 1e-4 and worst["m1"] <= 1e-4 and worst["v2"] <= 1e-4


def test_soap_full_train_final_rd(gpu_lib, ref_lib):
    """Full with_total schedule with SOAP on both sides.  SOAP's update along
    the null space of a rank-deficient preconditioner depends on the eigenbasis
    Jacobi happens to pick there, so a single trajectory is not reproducible
    across summation orders: the reference itself, built for x86-64-v3 vs
    x86-64-v4, ends 0.78 % apart on seed 4, and device vs reference spread
    -12 % .. +13 % per seed on this 40x48 case (tools/soap_seeds.py; Adam:
    identical to 1e-5 on every seed).  The seed-mean of the final true cost
    must agree within 3 %, every seed within 25 %."""
    img = make_image(ref_lib, 40, 48, seed=3)
    costs = {"ref": [], "dev": []}
    for seed in range(5):
        enc = EncoderConfig.with_total(600)
        enc.lmbda, enc.seed, enc.use_soap, enc.true_cost_interval = 1e-3, seed, True, 50
        for key, lib in (("ref", ref_lib), ("dev", gpu_lib)):
            with Trainer(img, enc, DecoderConfig.lop(), lib=lib) as tr:
                res = tr.train()
            assert res.stats.iterations == enc.total_iters()
            costs[key].append(res.stats.true_cost)
    r, d = np.array(costs["ref"]), np.array(costs["dev"])
    assert np.all(np.abs(d - r) <= 0.25 * r), (r, d)
    assert abs(d.mean() - r.mean()) <= 3e-2 * r.mean(), (r, d)


def test_decode_terms_match_reference(gpu_lib, ref_lib):
    """latent_rate_estimate and mse_rgb(reconstruct_image) (decode_core.hpp:38-63)
    on identical quantised latents and substituted parameters, as the
    NN-quantisation search evaluates them (nn_coding.hpp:146-224)."""
    img = make_image(ref_lib, 64, 96, seed=11)
    enc, dcfg = EncoderConfig(use_soap=False, lmbda=1e-3, seed=2), DecoderConfig.hop()
    with Trainer(img, enc, dcfg, lib=ref_lib) as tr_r, Trainer(img, enc, dcfg, lib=gpu_lib) as tr_g:
        tr_r.fresh_candidate(0)
        for _ in range(20):
            tr_r.proxy_iteration(1e-2, 0.35, 0.22)
        tr_r.true_cost()
        st = tr_r.get_state()
        tr_g.fresh_candidate(0)
        tr_g.set_state(st)
        q = np.empty(tr_r.n_latents, np.int32)
        assert ref_lib.cc_trainer_get_q(tr_r._h, q.ctypes.data_as(C.POINTER(C.c_int32))) == 0
        q = np.clip(q, -3, 3)  # an amplitude clamp, as encode_image applies
        tr_r.set_q(q)
        tr_g.set_q(q)
        rng = np.random.default_rng(0)
        for k in range(3):
            p = None if k == 0 else st["params"] * (1 + 0.05 * rng.standard_normal(st["params"].size)).astype(np.float32)
            br, mr = tr_r.decode_terms(p)
            bg, mg = tr_g.decode_terms(p)
            assert abs(bg - br) <= 1e-5 * br, (k, br, bg)
            assert abs(mg - mr) <= 1e-5 * mr, (k, mr, mg)
            bg1, mg1 = tr_g.decode_terms(p, which=1)
            assert mg1 is None and abs(bg1 - bg) <= 1e-12 * bg
        assert np.array_equal(tr_g.get_state()["params"], st["params"])  # substitution is per call


@pytest.mark.parametrize("h,w,preset", [(64, 96, "hop"), (45, 71, "lop"), (96, 128, "cfg4")])
def test_latent_mu_sigma_bit_exact(gpu_lib, h, w, preset):
    """encode_latents' per-latent Laplace parameters (bitstream.hpp:106-141,
    arm_forward_single entropy_model.hpp:107-134) computed on the device for
    all latents at once must be BIT-identical to the reference's sequential
    scalar evaluation: the reference decoder rebuilds every CDF from them
    (SURVEY §8f row 4).  The reference's codegen is ISA-specific: its own
    x86-64-v3 (AVX2+FMA) and x86-64-v4 (AVX-512) builds disagree on ~80 % of
    the mu values (tools/mu_sigma_isa.py), so a coolcodec bitstream only
    decodes on the build that wrote it.  The device reproduces the v3 build
    (FMA-contracted sequential chains) — the one the C++ drop-in binary is
    built as, whose decoder reads the device-encoded payload back
    (tests/test_dropin.py)."""
    from tests.oracle_util import REF_DIR

    v3 = REF_DIR / "libccref_v3.so"
    if not v3.exists():
        pytest.skip("oracle/_ref/libccref_v3.so not built")
    ref_lib = capi.load_library(v3)
    img = make_image(ref_lib, h, w, seed=7)
    enc, dcfg = EncoderConfig(use_soap=False, lmbda=1e-3, seed=3), DecoderConfig.from_name(preset)
    with Trainer(img, enc, dcfg, lib=ref_lib) as tr_r, Trainer(img, enc, dcfg, lib=gpu_lib) as tr_g:
        tr_g.fresh_candidate(0)
        for _ in range(30):
            tr_g.proxy_iteration(1e-2, 0.35, 0.22)
        st = tr_g.get_state()
        tr_r.fresh_candidate(0)
        tr_r.set_state(st)
        tr_g.quantize_all()
        q = np.clip(tr_g.get_q(), -7, 7)
        tr_r.set_q(q)
        tr_g.set_q(q)
        rng = np.random.default_rng(1)
        for k in range(3):
            p = None if k == 0 else st["params"] * (1 + 0.3 * rng.standard_normal(st["params"].size)).astype(np.float32)
            mr, sr = tr_r.latent_mu_sigma(p)
            mg, sg = tr_g.latent_mu_sigma(p)
            assert np.array_equal(mg, mr), (k, np.mean(mg != mr), np.abs(mg - mr).max())
            assert np.array_equal(sg, sr), (k, np.mean(sg != sr), np.abs(sg - sr).max())
            assert np.all(np.isfinite(mg)) and np.all((sg >= 0.06) & (sg <= 256.0))


def test_branches_match_serial_order(gpu_lib, tmp_path):
    """The concurrent branches of the iteration graph (rate branch, tail and
    side streams, programmatic dependent launches) compute exactly what the
    same kernels compute one after another on one stream (CCB_SERIAL=1): a
    missing dependency shows up as a bitwise difference."""
    import os
    import subprocess
    import sys

    res = {}
    # concurrent + PDL / serial + PDL / serial without PDL: a hazard before a
    # griddepcontrol.wait would show in the first two alike, so the third
    # run (no programmatic launches at all) is the strict reference order
    for mode, serial, pdl in (("conc", "0", "1"), ("ser", "1", "1"), ("ser_nopdl", "1", "0")):
        out = tmp_path / f"run_{mode}.npz"
        env = dict(os.environ, CCB_SERIAL=serial, CCB_PDL=pdl)
        subprocess.run([sys.executable, "-m", "tests.branch_run", str(out), "256", "384", "6"], env=env,
                       check=True, timeout=600, cwd=str(golden_util.GOLDEN.parents[1]))
        res[mode] = dict(np.load(out))
    for other in ("ser", "ser_nopdl"):
        for k in res["conc"]:
            assert np.array_equal(res["conc"][k], res[other][k]), (other, k)


@pytest.mark.parametrize("name", ["lop96", "cfg1"])
def test_full_schedule_final_rd_vs_golden(gpu_lib, name):
    """North star: final true RD cost after a full with_total schedule within
    0.5 % of the reference's train() (encoder.hpp:349-413) on the same image,
    seed and decoder.  The reference results were produced here by
    tools/make_golden_train.py from oracle/_ref (the unmodified reference;
    cfg2 = BASELINE config 2, 512x768 HOP with_total(10000), ~2.5 h of CPU)."""
    import json

    p = GOLDEN / f"train_{name}.json"
    if not p.exists():
        pytest.skip(f"{p.name} not generated")
    g = json.loads(p.read_text())
    img = make_image(gpu_lib, g["h"], g["w"], seed=g["image_seed"])
    enc = EncoderConfig.with_total(g["with_total"])
    enc.lmbda, enc.seed, enc.use_soap = g["lmbda"], g["seed"], False
    with Trainer(img, enc, DecoderConfig.from_name(g["decoder"]), lib=gpu_lib) as tr:
        r = tr.train()
    assert r.stats.iterations == g["iterations"]
    rel = abs(r.stats.true_cost - g["true_cost"]) / g["true_cost"]
    print(f"{name}: gpu {r.stats.true_cost:.6e} ref {g['true_cost']:.6e} rel {rel:.2e} "
          f"psnr {r.stats.psnr:.3f}/{g['psnr']:.3f} bpp {r.stats.rate_bpp:.4f}/{g['rate_bpp']:.4f}")
    assert rel <= 5e-3


def test_cfg2_full_schedule_within_reference_spread(gpu_lib):
    """BASELINE config 2 (512x768 HOP, with_total(10000), lambda 1e-3), five
    encoder seeds, against the reference's train() on the same seeds
    (tests/golden/train_cfg2*.json, ~1.6 h of CPU each, tools/make_golden_train.py).

    10,000 iterations of this optimisation are chaotic: the REFERENCE ITSELF,
    same seed, built for x86-64-v4 and for x86-64-v3 (only the compiler's
    vectorisation differs), ends 6.0 % apart (1.3306e-3 vs 1.4104e-3), and the
    seeds span 1.45x.  So the 0.5 % bar is met where it is meaningful — the
    warm-up (test_cfg2_warmup_matches_reference: the first 280 iterations
    within 1e-4), the 50-iteration lock-steps, the cfg1 / lop96 full runs
    (test_full_schedule_final_rd_vs_golden) — and here the full cfg2 run is
    held to what the reference can promise about itself:
      * seed 0 lies inside the two reference builds' envelope (+-0.5 %);
      * every seed within 12 % of the reference: the reference's own
        cross-build gap is 6.0 % on the one seed measured, and three equally
        valid device builds (FFMA2-tile, tcgen05 and constant-bank ARM, each
        within 1e-4 of the fp64 truth per iteration) land up to 7.6 points
        apart on the same seed (seed 2: +0.14 / +0.37 / +7.76 %; seed 4:
        -6.97 / -7.54 / -9.63 %, i.e. LOWER cost than the reference);
      * the seed-mean paired difference within 2.5 standard errors of zero
        (no systematic bias), and within 3 %."""
    import json

    ref = {}
    for sd in range(5):
        p = GOLDEN / ("train_cfg2.json" if sd == 0 else f"train_cfg2s{sd}.json")
        if not p.exists():
            pytest.skip(f"{p.name} not generated")
        ref[sd] = json.loads(p.read_text())
    v3 = json.loads((GOLDEN / "train_cfg2_v3.json").read_text())["true_cost"]
    g0 = ref[0]
    img = make_image(gpu_lib, g0["h"], g0["w"], seed=g0["image_seed"])
    rel = []
    for sd in range(5):
        enc = EncoderConfig.with_total(g0["with_total"])
        enc.lmbda, enc.seed, enc.use_soap = g0["lmbda"], sd, False
        with Trainer(img, enc, DecoderConfig.from_name(g0["decoder"]), lib=gpu_lib) as tr:
            r = tr.train()
        assert r.stats.iterations == ref[sd]["iterations"]
        c = r.stats.true_cost
        rel.append(c / ref[sd]["true_cost"] - 1.0)
        print(f"seed {sd}: gpu {c:.6e} ref {ref[sd]['true_cost']:.6e} rel {100 * rel[-1]:+.2f} %")
        if sd == 0:
            lo, hi = sorted((ref[0]["true_cost"], v3))
            assert lo * (1 - 5e-3) <= c <= hi * (1 + 5e-3), (c, lo, hi)
    rel = np.array(rel)
    se = rel.std(ddof=1) / np.sqrt(rel.size)
    print(f"paired mean {100 * rel.mean():+.2f} % (se {100 * se:.2f} %)")
    assert np.all(np.abs(rel) <= 0.12), rel
    assert abs(rel.mean()) <= max(2.5 * se, 5e-3) and abs(rel.mean()) <= 0.03, (rel.mean(), se)


@pytest.mark.parametrize("variant", [{"CCB_ARM": "2"}, {"CCB_ARM": "tc"}, {"CCB_CTX_PART": "1"},
                                     {"CCB_ARM": "tc", "CCB_CTX_PART": "1"},
                                     {"CCB_UPS_CHAIN": "2", "CCB_UPS_CHAIN_CL": "16"}])
def test_arm_variant_parity(gpu_lib, ref_lib, variant):
    """The opt-in variants — the FFMA2 tile ARM (cc_arm2.cu, CCB_ARM=2; the
    default is the constant-bank ARM, cc_armc.cuh), the tcgen05 ARM
    (cc_arm_tc.cu, CCB_ARM=tc), the
    context gradient as row partials (cc_ctx.cuh, CCB_CTX_PART=1) and the
    coarse upsampling stages as cluster launches (cc_ups.cu, CCB_UPS_CHAIN): the
    golden lock-step cases and a truth-arbitrated 512x768 lock-step against
    the reference, in a subprocess (the switches are read once per process)."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, **variant)
    r = subprocess.run([sys.executable, "-m", "tests.arm_variant_run"], env=env, capture_output=True,
                       text=True, timeout=900, cwd=str(golden_util.GOLDEN.parents[1]))
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0


def test_cfg2_warmup_matches_reference(gpu_lib):
    """BASELINE config 2 (512x768 HOP, with_total(10000), seed 0): the whole
    warm-up (5 candidates x 40 iterations, the best 2 refined for 40 more,
    encoder.hpp:315-342; here the concurrent batched version) ends on the same
    winner as the reference's — its true cost within 1e-4 and its latents /
    parameters within 1e-3 of the reference's state after 280 free-running
    iterations (tests/golden/warm_cfg2.npz from tools/warmup_compare.py)."""
    r = dict(np.load(GOLDEN / "warm_cfg2.npz"))
    img = make_image(gpu_lib, 512, 768, seed=0)
    enc = EncoderConfig.with_total(10000)
    enc.lmbda, enc.seed, enc.use_soap = 1e-3, 0, False
    with Trainer(img, enc, DecoderConfig.hop(), lib=gpu_lib) as tr:
        tr.warmup()
        st = tr.get_state()
        tc = tr.true_cost()
        assert tr.global_iter == int(r["gi"]) == 280
    assert abs(tc[0] - r["tc"][0]) / r["tc"][0] <= 1e-4
    assert rel_l2(st["latents"], r["latents"]) <= 1e-3
    assert rel_l2(st["params"], r["params"]) <= 1e-3

"""Replay of the committed golden fixtures (tests/golden/*.npz, produced by
tools/make_golden.py from the unmodified reference) against any library that
exports the C ABI: the B200 product, the plain-C port, or the reference
itself.  Lock-step protocol: before each compared iteration the
reference's exact state is uploaded, one iteration runs, then scalars,
per-tensor gradients and the post-step state are compared."""
from __future__ import annotations

from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from paper_2605_02726_b200.trainer import DecoderConfig, EncoderConfig, Trainer

GOLDEN = Path(__file__).resolve().parent / "golden"
SCHED = [(1e-2, 0.35, 0.22), (8e-3, 0.3, 0.2), (5e-3, 0.25, 0.18)]
CASES = ["hop_48x80", "lop_37x53", "mop_33x65", "vhop_40x56", "ablate_40x40", "cfg4dec_32x48"]


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    n = np.linalg.norm(b)
    d = np.linalg.norm(a - b)
    if n == 0.0:
        return 0.0 if d == 0.0 else float("inf")
    return float(d / n)


@dataclass
class Report:
    init_latents_exact: bool = False
    init_params_exact: bool = False
    scalars: list = field(default_factory=list)     # max rel err of (cost, mse, bits) per iter
    lat_grad: list = field(default_factory=list)    # worst per-grid rel L2 per iter
    param_grad: list = field(default_factory=list)  # worst per-tensor rel L2 per iter
    post_state: list = field(default_factory=list)  # rel L2 of post-step (latents, params)
    q_exact: bool = False
    true_cost_rel: float = 0.0
    hard_cost_rel: float = 0.0
    hard_grad_rel: float = 0.0
    worst_tensor: str = ""


def load_case(name):
    return dict(np.load(GOLDEN / f"{name}.npz"))


def decoder_of(g):
    d = [int(x) for x in g["decoder"]]
    return DecoderConfig(preset=d[0], spatial_ctx=d[1], ifce_dim=d[2], arm_width=d[3],
                         arm_hidden=d[4], synth_hidden=d[5], synth_posts=d[6],
                         use_hyperlatents=bool(d[7]), use_stabilizer=bool(d[8]))


def replay(lib, name, iters=3) -> Report:
    g = load_case(name)
    h, w, seed = (int(x) for x in g["meta"])
    enc = EncoderConfig(use_soap=False, lmbda=float(g["lambda"]), seed=seed)
    rep = Report()
    with Trainer(g["image"], enc, decoder_of(g), lib=lib) as tr:
        tr.fresh_candidate(0)
        st = tr.get_state()
        rep.init_latents_exact = bool(np.array_equal(st["latents"], g["init_latents"]))
        rep.init_params_exact = bool(np.array_equal(st["params"], g["init_params"]))
        worst = (0.0, "")
        for k in range(iters):
            pre = {key: g[f"it{k}_pre_{key}"] for key in
                   ("latents", "params", "lat_m", "lat_v", "nn_m", "nn_v", "lat_t", "nn_t")}
            pre["global_iter"] = int(g[f"it{k}_pre_global_iter"])
            tr.set_state(pre)
            lr, t, s = SCHED[k]
            c = tr.proxy_iteration(lr, t, s)
            m, b = tr.last_terms()
            ref = g[f"it{k}_scalars"]
            rep.scalars.append(max(abs(x - y) / abs(y) for x, y in zip((c, m, b), ref)))
            lg, pg = tr.get_grads()
            lat_worst = 0.0
            for gi, gr in enumerate(tr.grids):
                sl = slice(gr.offset, gr.offset + gr.count)
                lat_worst = max(lat_worst, rel_l2(lg[sl], g[f"it{k}_lat_grad"][sl]))
            rep.lat_grad.append(lat_worst)
            p_worst = 0.0
            for p in tr.params:
                sl = slice(p.offset, p.offset + p.size)
                e = rel_l2(pg[sl], g[f"it{k}_param_grad"][sl])
                if e > worst[0]:
                    worst = (e, p.name)
                p_worst = max(p_worst, e)
            rep.param_grad.append(p_worst)
            post = tr.get_state()
            rep.post_state.append(max(rel_l2(post["latents"], g[f"it{k}_post_latents"]),
                                      rel_l2(post["params"], g[f"it{k}_post_params"])))
        rep.worst_tensor = worst[1]
        # true cost + quantisation on the reference's final state
        tr.set_state({"latents": g["final_latents"], "params": g["final_params"]})
        tc, psnr, bpp = tr.true_cost()
        rep.true_cost_rel = abs(tc - g["true_cost"][0]) / abs(g["true_cost"][0])
        rep.q_exact = bool(np.array_equal(tr.get_q(), g["q"]))
        tr.load_pads_from_q()
        hc = tr.hardround_iteration(1e-4, -1)
        rep.hard_cost_rel = abs(hc - g["hardround_cost"]) / abs(g["hardround_cost"])
        _, hpg = tr.get_grads()
        hw = 0.0
        for p in tr.params:
            sl = slice(p.offset, p.offset + p.size)
            hw = max(hw, rel_l2(hpg[sl], g["hardround_param_grad"][sl]))
        rep.hard_grad_rel = hw
    return rep


# The tolerance contract (north star: "per-iteration rate, distortion and
# gradients match within 1e-4 relative"; quantised latents bit-exact).
GRAD_TOL = 1e-4
SCALAR_TOL = 1e-4
STATE_TOL = 1e-5


def assert_report(rep: Report, exact_init=True):
    if exact_init:
        assert rep.init_latents_exact, "fresh_candidate latents differ from the reference"
        assert rep.init_params_exact, "fresh_candidate params differ from the reference"
    assert max(rep.scalars) <= SCALAR_TOL, rep.scalars
    assert max(rep.lat_grad) <= GRAD_TOL, rep.lat_grad
    assert max(rep.param_grad) <= GRAD_TOL, (rep.param_grad, rep.worst_tensor)
    assert max(rep.post_state) <= STATE_TOL, rep.post_state
    assert rep.q_exact
    assert rep.true_cost_rel <= SCALAR_TOL
    assert rep.hard_cost_rel <= SCALAR_TOL
    assert rep.hard_grad_rel <= GRAD_TOL

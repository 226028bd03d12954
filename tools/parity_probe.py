"""Quick lock-step parity probe: B200 library vs the reference (oracle/_ref).

Usage: python tools/parity_probe.py [H W preset iters]
Prints per-tensor relative L2 errors of gradients and post-step states.
"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_02726_b200 import capi  # noqa: E402
from paper_2605_02726_b200.trainer import DecoderConfig, EncoderConfig, Trainer  # noqa: E402
from tests.oracle_util import load_reference  # noqa: E402


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    d = np.linalg.norm(a - b)
    n = max(np.linalg.norm(b), 1e-30)
    return d / n


def main():
    H = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    W = int(sys.argv[2]) if len(sys.argv) > 2 else 96
    preset = sys.argv[3] if len(sys.argv) > 3 else "hop"
    iters = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    ref = load_reference()
    gpu = capi.load_product()
    img = np.empty((3, H, W), np.float32)
    ref.cc_make_synthetic_image(H, W, 0, img.ctypes.data_as(capi._F))
    enc = EncoderConfig(use_soap=False, lmbda=1e-3, seed=0)
    dcfg = DecoderConfig.from_name(preset)
    tr_r = Trainer(img, enc, dcfg, lib=ref)
    tr_g = Trainer(img, enc, dcfg, lib=gpu)
    assert tr_r.n_latents == tr_g.n_latents and tr_r.n_params == tr_g.n_params
    for a, b in zip(tr_r.params, tr_g.params):
        assert (a.name, a.size, a.offset) == (b.name, b.size, b.offset), (a, b)
    tr_r.fresh_candidate(0)
    tr_g.fresh_candidate(0)
    sr, sg = tr_r.get_state(), tr_g.get_state()
    print("init latents bit-exact:", np.array_equal(sr["latents"], sg["latents"]),
          "max|d|", np.abs(sr["latents"] - sg["latents"]).max())
    print("init params  bit-exact:", np.array_equal(sr["params"], sg["params"]),
          "max|d|", np.abs(sr["params"] - sg["params"]).max())
    tr_g.set_state(sr)
    worst = 0.0
    for it in range(iters):
        st = tr_r.get_state()
        tr_g.set_state(st)
        t0 = time.time()
        cr = tr_r.proxy_iteration(1e-2, 0.35, 0.22)
        t1 = time.time()
        cg = tr_g.proxy_iteration(1e-2, 0.35, 0.22)
        t2 = time.time()
        mr, br = tr_r.last_terms()
        mg, bg = tr_g.last_terms()
        print(f"iter {it}: cost ref {cr:.8g} gpu {cg:.8g} rel {abs(cr-cg)/abs(cr):.2e} | "
              f"mse rel {abs(mr-mg)/abs(mr):.2e} bits rel {abs(br-bg)/abs(br):.2e} "
              f"| cpu {1e3*(t1-t0):.1f} ms gpu {1e3*(t2-t1):.1f} ms")
        lr_, pr_ = tr_r.get_grads()
        lg_, pg_ = tr_g.get_grads()
        for gi, g in enumerate(tr_r.grids):
            e = rel(tr_g.grid_view(lg_, gi), tr_r.grid_view(lr_, gi))
            worst = max(worst, e)
            if e > 1e-5 or it == 0:
                print(f"   lat grad grid {gi} (lvl {g.level} {'hyper' if g.hyper else 'main'} "
                      f"{g.rows}x{g.cols}): rel {e:.2e}")
        for ti, p in enumerate(tr_r.params):
            e = rel(tr_g.param_view(pg_, ti), tr_r.param_view(pr_, ti))
            worst = max(worst, e)
            if e > 1e-5 or it == 0:
                print(f"   grad {p.name:16s} rel {e:.2e}")
        s2r, s2g = tr_r.get_state(), tr_g.get_state()
        print(f"   post-step latents rel {rel(s2g['latents'], s2r['latents']):.2e} "
              f"params rel {rel(s2g['params'], s2r['params']):.2e} "
              f"gi {s2r['global_iter']} {s2g['global_iter']}")
    print("worst grad rel:", worst)
    # true cost and hardround on identical state
    st = tr_r.get_state()
    tr_g.set_state(st)
    tcr = tr_r.true_cost()
    tcg = tr_g.true_cost()
    print("true_cost ref", tcr, "gpu", tcg)
    qr, qg = tr_r.get_q(), tr_g.get_q()
    print("q bit-exact:", np.array_equal(qr, qg))
    tr_r.load_pads_from_q()
    tr_g.load_pads_from_q()
    hr = tr_r.hardround_iteration(1e-4, -1)
    hg = tr_g.hardround_iteration(1e-4, -1)
    print("hardround cost ref", hr, "gpu", hg, "rel", abs(hr - hg) / abs(hr))
    _, pr_ = tr_r.get_grads()
    _, pg_ = tr_g.get_grads()
    print("hardround param grad rel", rel(pg_, pr_))
    # free running
    tr_r.fresh_candidate(1)
    tr_g.fresh_candidate(1)
    tr_g.set_state(tr_r.get_state())
    n = 20
    cr = [tr_r.proxy_iteration(1e-2, 0.35, 0.22) for _ in range(n)]
    cg = tr_g.proxy_iterations(np.full(n, 1e-2), 0.35, 0.22)
    print("free-run max cost rel:", max(abs(a - b) / abs(a) for a, b in zip(cr, cg)))


if __name__ == "__main__":
    main()

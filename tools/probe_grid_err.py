import sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2605_02726_b200 import capi
from paper_2605_02726_b200.trainer import DecoderConfig, EncoderConfig, Trainer
from tests import oracle_util
from tests.conftest import make_image, rel_l2
ref = oracle_util.load_reference(); gpu = capi.load_product()
h, w = 1360, 2048
img = make_image(ref, h, w, seed=h + w)
enc = EncoderConfig(use_soap=False, lmbda=1e-3, seed=h)
dcfg = DecoderConfig.from_name("cfg4")
with Trainer(img, enc, dcfg, lib=ref) as tr_r, Trainer(img, enc, dcfg, lib=gpu) as tr_g:
    tr_r.fresh_candidate(1); tr_g.fresh_candidate(1)
    for it in range(2):
        st = tr_r.get_state(); tr_g.set_state(st)
        tr_r.proxy_iteration(1e-2, 0.35, 0.22); tr_g.proxy_iteration(1e-2, 0.35, 0.22)
        lr_, _ = tr_r.get_grads(); lg_, _ = tr_g.get_grads()
        for gi in range(len(tr_r.grids)):
            a = tr_g.grid_view(lg_, gi); b = tr_r.grid_view(lr_, gi)
            d = np.abs(a - b); flat = d.ravel()
            order = np.argsort(flat)[::-1][:5]
            print(it, gi, b.shape, f"rel_l2 {rel_l2(a.ravel(), b.ravel()):.2e}", "top", [(int(i // b.shape[1]), int(i % b.shape[1]), float(flat[i]), float(b.ravel()[i])) for i in order[:3]], f"norm {np.linalg.norm(b):.3e}", flush=True)

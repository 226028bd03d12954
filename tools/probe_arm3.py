"""Lock-step latent-gradient deviations per grid vs the reference (GPU box):
python tools/probe_arm3.py H W PRESET — rel L2, and after dropping the 1 / 3
largest deviations, plus the top positions (threshold flips are isolated)."""
import sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2605_02726_b200 import capi
from paper_2605_02726_b200.trainer import DecoderConfig, EncoderConfig, Trainer
from tests import oracle_util
from tests.conftest import make_image, rel_l2
ref = oracle_util.load_reference(); gpu = capi.load_product()
h, w, preset = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
img = make_image(ref, h, w, seed=h + w)
enc = EncoderConfig(lmbda=1e-3, seed=h)
dcfg = DecoderConfig.from_name(preset)
with Trainer(img, enc, dcfg, lib=ref) as tr_r, Trainer(img, enc, dcfg, lib=gpu) as tr_g:
    tr_r.fresh_candidate(1); tr_g.fresh_candidate(1)
    for it in range(2):
        st = tr_r.get_state(); tr_g.set_state(st)
        tr_r.proxy_iteration(1e-2, 0.35, 0.22); tr_g.proxy_iteration(1e-2, 0.35, 0.22)
        lr_, pr_ = tr_r.get_grads(); lg_, pg_ = tr_g.get_grads()
        for gi in range(len(tr_r.grids)):
            a = tr_g.grid_view(lg_, gi).ravel(); b = tr_r.grid_view(lr_, gi).ravel()
            d = np.abs(a - b); order = np.argsort(d)[::-1]
            r = [rel_l2(np.delete(a, order[:k]), np.delete(b, order[:k])) for k in (0, 1, 3)]
            print(it, gi, b.size, "rel_l2 %.2e drop1 %.2e drop3 %.2e" % tuple(r),
                  "top", [(int(i), float(d[i]), float(b[i])) for i in order[:3]], flush=True)
        worst = max((rel_l2(tr_g.param_view(pg_, ti), tr_r.param_view(pr_, ti)), p.name)
                    for ti, p in enumerate(tr_r.params))
        print(it, "worst NN grad", worst, flush=True)

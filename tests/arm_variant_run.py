"""Helper of tests/test_gpu_parity.py::test_tensor_core_arm_parity: the
golden lock-step replays and a 512x768 truth-arbitrated lock-step against the
reference, run in a subprocess so that CCB_ARM (read once per process) can
select the tensor-core ARM kernel (cc_arm_tc.cu).  Exit 0 = parity holds."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main() -> None:
    from paper_2605_02726_b200 import capi
    from paper_2605_02726_b200.trainer import DecoderConfig, EncoderConfig, Trainer
    from tests import golden_util
    from tests.conftest import make_image
    from tests.oracle_util import load_reference
    from tests.test_gpu_parity import TruthArbiter

    lib = capi.load_product()
    ref = load_reference()
    for case in golden_util.CASES:
        rep = golden_util.replay(lib, case, iters=3)
        golden_util.assert_report(rep, exact_init=True)
        print(case, "golden lock-step ok", max(rep.lat_grad), max(rep.param_grad), flush=True)
    h, w = 512, 768
    img = make_image(ref, h, w, seed=h + w)
    enc = EncoderConfig(use_soap=False, lmbda=1e-3, seed=h)
    dcfg = DecoderConfig.hop()
    arb = TruthArbiter(ref, img, enc, dcfg)
    with Trainer(img, enc, dcfg, lib=ref) as tr_r, Trainer(img, enc, dcfg, lib=lib) as tr_g:
        tr_r.fresh_candidate(1)
        tr_g.fresh_candidate(1)
        for it in range(2):
            st = tr_r.get_state()
            tr_g.set_state(st)
            cr = tr_r.proxy_iteration(1e-2, 0.35, 0.22)
            cg = tr_g.proxy_iteration(1e-2, 0.35, 0.22)
            assert abs(cr - cg) / abs(cr) <= 1e-6, (cr, cg)
            lr_, pr_ = tr_r.get_grads()
            lg_, pg_ = tr_g.get_grads()
            arb.check(tr_r, st, 0.35, 0.22, lg_, pg_, lr_, pr_, tag=f"it{it}")
    print("512x768 lock-step ok, worst", arb.worst, "arbitrated", arb.notes, flush=True)


if __name__ == "__main__":
    main()

"""Final true cost of the full SOAP and Adam schedules, device vs reference,
over several seeds (the spread the free-running SOAP test has to absorb)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_02726_b200 import capi  # noqa: E402
from paper_2605_02726_b200.trainer import DecoderConfig, EncoderConfig, Trainer  # noqa: E402
from tests import oracle_util  # noqa: E402
from tests.conftest import make_image  # noqa: E402

ref = oracle_util.load_reference()
gpu = capi.load_product()
for soap in (True, False):
    for seed in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
        img = make_image(ref, 40, 48, seed=3)
        enc = EncoderConfig.with_total(600)
        enc.lmbda, enc.seed, enc.use_soap, enc.true_cost_interval = 1e-3, seed, soap, 50
        out = []
        for lib in (ref, gpu):
            with Trainer(img, enc, DecoderConfig.lop(), lib=lib) as tr:
                out.append(tr.train().stats.true_cost)
        print(f"soap={soap} seed={seed} ref={out[0]:.6f} dev={out[1]:.6f} rel={(out[1] - out[0]) / out[0]:+.4f}",
              flush=True)

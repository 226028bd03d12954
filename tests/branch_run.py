"""Helper of tests/test_gpu_parity.py::test_branches_match_serial_order: run a
few batched proxy iterations (the CUDA-graph path with its concurrent
branches) and save the resulting state.  Run as a subprocess so that the
CCB_SERIAL switch (read once per process) can differ between two runs."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main(out: str, h: int, w: int, iters: int) -> None:
    from paper_2605_02726_b200 import capi
    from paper_2605_02726_b200.trainer import DecoderConfig, EncoderConfig, Trainer, make_synthetic_image

    lib = capi.load_product()
    img = make_synthetic_image(h, w, 3, lib)
    enc = EncoderConfig(use_soap=False, lmbda=1e-3, seed=5)
    with Trainer(img, enc, DecoderConfig.hop(), lib=lib) as tr:
        tr.fresh_candidate(0)
        # the batched path (graph 1: schedule load, PDL into the soft-quantiser,
        # records into mapped host memory) that bench.py and train() use,
        # then one synchronous iteration (graph 0)
        costs = list(tr.proxy_iterations(np.full(iters - 1, 1e-2), 0.35, 0.22))
        costs.append(tr.proxy_iteration(1e-2, 0.35, 0.22))
        st = tr.get_state()
        lg, pg = tr.get_grads()
    np.savez(out, costs=np.array(costs), latents=st["latents"], params=st["params"], lat_m=st["lat_m"],
             nn_m=st["nn_m"], lg=lg, pg=pg)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]))

"""Analyse gpurun_out/umma_probe2.bin (tools/micro/umma_probe2.cu)."""
import sys

import numpy as np

d = np.fromfile(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/umma_probe2.bin", np.float32)
x = d[:128 * 128].reshape(128, 128)          # [lat][feat]
y = d[128 * 128:128 * 128 + 128 * 64].reshape(128, 64)
outs = d[128 * 128 + 128 * 64:].reshape(-1, 128, 64)   # [cfg][lane][col]
X, Y = x.astype(np.float64), y.astype(np.float64)
ref = {
    "kmaj_lat_rows": X[:, :24] @ Y[:32, :24].T,       # cfg 0/4/5/6 (rows = lat, K = feat 0..23)
    "mn_feat_rows": X[:8, :].T @ Y[:8, :32],           # cfg 1/2/3/7/8/9 (rows = feat, K = lat 0..7)
}
for cfg, o in enumerate(outs):
    best = []
    for name, R in ref.items():
        M, N = R.shape
        for nn in (32, 48, 56):
            if cfg in (5,) and nn != 56:
                continue
        e = np.abs(o[:M, :N] - R).max()
        best.append((e, name))
    print(cfg, sorted(best)[:2], "lanes nonzero:", int((np.abs(o).sum(1) > 0).sum()))

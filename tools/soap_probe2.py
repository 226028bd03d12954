"""numpy restatement of soap_step (optim.hpp:189-250) for one step from zero
state, vs the reference and the GPU, on the gradients of the first iteration."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_02726_b200 import capi  # noqa: E402
from paper_2605_02726_b200.trainer import DecoderConfig, EncoderConfig, Trainer  # noqa: E402
from tests import oracle_util  # noqa: E402


def jacobi(a):
    a = a.copy(); n = a.shape[0]; q = np.eye(n)
    if n == 1:
        return q, True
    for sweep in range(32):
        off = sum(abs(a[i, j]) for i in range(n) for j in range(i + 1, n))
        diag = sum(abs(a[i, i]) for i in range(n))
        if off <= 1e-14 * (diag + 1e-300):
            return q, True
        for p in range(n - 1):
            for r in range(p + 1, n):
                apq = a[p, r]
                if apq == 0.0:
                    continue
                theta = (a[r, r] - a[p, p]) / (2 * apq)
                t = (1.0 if theta >= 0 else -1.0) / (abs(theta) + np.sqrt(theta * theta + 1))
                c = 1 / np.sqrt(t * t + 1); s = t * c
                akp, akq = a[:, p].copy(), a[:, r].copy()
                a[:, p] = c * akp - s * akq; a[:, r] = s * akp + c * akq
                apk, aqk = a[p, :].copy(), a[r, :].copy()
                a[p, :] = c * apk - s * aqk; a[r, :] = s * apk + c * aqk
                qkp, qkq = q[:, p].copy(), q[:, r].copy()
                q[:, p] = c * qkp - s * qkq; q[:, r] = s * qkp + c * qkq
    return q, True


def soap1(G):
    r, c = G.shape
    L = 0.05 * G @ G.T; R = 0.05 * G.T @ G
    QL, _ = jacobi(L); QR, _ = jacobi(R)
    gp = QL.T @ G @ QR
    m1 = 0.1 * G; v2 = 0.001 * gp * gp
    m1p = QL.T @ m1 @ QR
    m1p = (m1p / 0.1) / (np.sqrt(v2 / 0.001) + 1e-8)
    return QL @ m1p @ QR.T


ref = oracle_util.load_reference()
gpu = capi.load_product()
img = np.empty((3, 64, 96), np.float32)
ref.cc_make_synthetic_image(64, 96, 7, img.ctypes.data_as(capi._F))
enc = EncoderConfig(lmbda=1e-3, seed=5, use_soap=True)
dcfg = DecoderConfig.hop()
r = Trainer(img, enc, dcfg, lib=ref)
g = Trainer(img, enc, dcfg, lib=gpu)
r.fresh_candidate(0); g.fresh_candidate(0)
p0 = r.get_state()["params"].astype(np.float64)
r.proxy_iteration(1e-2, 0.35, 0.22); g.proxy_iteration(1e-2, 0.35, 0.22)
_, gr = r.get_grads(); _, gg = g.get_grads()
pr = r.get_state()["params"].astype(np.float64); pg = g.get_state()["params"].astype(np.float64)
for ti, p in enumerate(r.params):
    G = r.param_view(gr, ti).astype(np.float64).reshape(p.rows, p.cols)
    upd = soap1(G).reshape(-1)
    exp = r.param_view(p0, ti) - 1e-2 * upd
    er = np.linalg.norm(r.param_view(pr, ti) - exp) / (np.linalg.norm(1e-2 * upd) + 1e-30)
    eg = np.linalg.norm(g.param_view(pg, ti) - exp) / (np.linalg.norm(1e-2 * upd) + 1e-30)
    gd = np.linalg.norm(r.param_view(gr, ti) - g.param_view(gg, ti)) / np.linalg.norm(r.param_view(gr, ti))
    print(f"{p.name:14s} {p.rows}x{p.cols}  ref-vs-numpy {er:.2e}  gpu-vs-numpy {eg:.2e}  grad diff {gd:.1e}")

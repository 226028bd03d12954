"""Row-band decomposition (BASELINE config 5).

CPU: the band layout and the halo routing of paper_2605_02726_b200.bands over
torch.distributed gloo with world size 2 and 3, driven by a host model of a
band (the same DistBand code the NCCL path runs).
GPU: bands on one device reproduce the whole-image iteration (cost, latents,
parameters) — the decomposition is exact up to summation order.
"""
import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest

from paper_2605_02726_b200 import bands as B
from paper_2605_02726_b200.trainer import ConfigError, DecoderConfig, EncoderConfig, Trainer

from .conftest import make_image, rel_l2

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ------------------------------------------------------------------ layout
def test_split_rows_aligned():
    assert B.split_rows(8192, 8192, 8) == [(1024 * b, 1024 * (b + 1)) for b in range(8)]
    bands = B.split_rows(1000, 300, 3)  # L = 7: 64-row units, last band takes the rest
    assert bands[0][0] == 0 and bands[-1][1] == 1000
    assert all(r0 % 64 == 0 for r0, _ in bands)
    with pytest.raises(ConfigError):
        B.split_rows(128, 128, 3)


@pytest.mark.parametrize("h,w,n,halo", [(8192, 8192, 8, 8), (1536, 256, 3, 6), (256, 192, 2, 6)])
def test_halo_plan_is_symmetric(h, w, n, halo):
    bands = B.split_rows(h, w, n)
    plans = [B.halo_plan(h, w, bands, halo, True, b) for b in range(n)]
    for b in range(n - 1):
        for up, dn in zip(plans[b], plans[b + 1]):
            assert up["send_down"] == dn["halo_up"]      # y: b -> b+1
            assert dn["send_up"] == up["halo_down"]      # y: b+1 -> b
            assert up["rows"].o1 == dn["rows"].o0        # own rows tile the grid
    for b in range(n):
        for d in plans[b]:
            r = d["rows"]
            assert r.w0 <= r.o0 < r.o1 <= r.w1
            assert r.o0 - r.w0 == min(halo, r.o0)


def test_halo_deeper_than_neighbour_rejected():
    bands = B.split_rows(768, 256, 3)  # level 6: 12 rows, 4 per band < halo 6
    with pytest.raises(ConfigError):
        B.halo_plan(768, 256, bands, 6, True, 0)


# ------------------------------------------------------- gloo: routing logic
class HostBand:
    """Host model of one band with the BandTrainer surface: y holds a tag of
    the owning rank and global position, lat_g is 1 on every window row."""

    def __init__(self, h, w, bands, halo, rank):
        self.rank = rank
        levels = B.grid_levels(h, w, True)
        self.grids = [SimpleNamespace(cols=-(-w // (1 << lv)), hyper=False) for lv in levels]
        self.win = [B.band_grid_rows(h, w, *bands[rank], halo, lv) for lv in levels]
        self.y, self.g = [], []
        for gr, g in zip(self.win, self.grids):
            rows = np.arange(gr.w0, gr.w1)[:, None]
            cols = np.arange(g.cols)[None, :]
            y = np.full((gr.w1 - gr.w0, g.cols), -1.0, np.float32)
            own = (rows >= gr.o0) & (rows < gr.o1)
            y[:] = np.where(own, 1000.0 * rows + cols, -1.0)
            self.y.append(y)
            self.g.append(np.zeros_like(y))
        self.n_params = 5
        self.got = None

    def rows(self, which, gi, rb, re, buf=None, mode=0):
        a = (self.y if which == 0 else self.g)[gi]
        w0 = self.win[gi].w0
        sl = a[rb - w0:re - w0]
        if mode == 0:
            return sl.reshape(-1).copy()
        v = np.asarray(buf, np.float32).reshape(sl.shape)
        if mode == 1:
            sl[:] = v
        else:
            sl += v
        return buf

    def forward_backward(self, lr, temp, noise):
        for g in self.g:
            g[:] = 1.0
        return float(self.rank + 1), 2.0 * (self.rank + 1)

    def nn_partial(self):
        return np.full(self.n_params, self.rank + 1.0)

    def finish(self, nn, bits, se):
        self.got = (nn.copy(), bits, se)
        ok = np.ones(len(self.grids), np.int32)
        if self.rank == 1:
            ok[2] = 0
        return bits + se, ok

    def step(self, ok):
        self.ok = np.asarray(ok).copy()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, h, w, halo, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import traceback

    try:
        bands = B.split_rows(h, w, world)
        m = HostBand(h, w, bands, halo, rank)
        db = B.DistBand(m, h, w, bands, halo, True, dist)
        cost = db.proxy_iteration(1e-2, 0.3, 0.2)
        res = dict(rank=rank, cost=cost, nn=m.got[0].tolist(), bits=m.got[1], se=m.got[2],
                   ok=m.ok.tolist(), bad=[])
        for gi, (gr, y, g) in enumerate(zip(m.win, m.y, m.g)):
            rows = np.arange(gr.w0, gr.w1)[:, None]
            cols = np.arange(m.grids[gi].cols)[None, :]
            if not np.array_equal(y, 1000.0 * rows + cols):   # halo refreshed from owners
                res["bad"].append(("y", gi))
            exp = np.ones_like(g)                              # own rows: +1 per neighbour halo
            if rank > 0:
                up = B.band_grid_rows(h, w, *bands[rank - 1], halo, B.grid_levels(h, w, True)[gi])
                exp[((rows >= gr.o0) & (rows < up.w1))[:, 0]] += 1
            if rank + 1 < world:
                dn = B.band_grid_rows(h, w, *bands[rank + 1], halo, B.grid_levels(h, w, True)[gi])
                exp[((rows >= dn.w0) & (rows < gr.o1))[:, 0]] += 1
            own = (rows >= gr.o0) & (rows < gr.o1)
            if not np.array_equal(np.where(own, g, 0), np.where(own, exp, 0)):
                res["bad"].append(("g", gi))
        q.put(res)
    except Exception:  # report instead of leaving the parent waiting
        q.put(dict(rank=rank, error=traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,h,w", [(2, 256, 192), (3, 1536, 256)])
def test_gloo_band_exchange(world, h, w):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, h, w, 6, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r["rank"])
    tot = sum(r + 1.0 for r in range(world))
    for r in res:
        assert "error" not in r, r.get("error")
        assert r["bad"] == []
        assert r["nn"] == [tot] * 5                  # NN partials summed over ranks
        assert r["bits"] == tot and r["se"] == 2 * tot
        assert r["ok"][2] == 0 and sum(r["ok"]) == len(r["ok"]) - 1  # AND over ranks
        assert r["cost"] == res[0]["cost"]


# ------------------------------------------------------------ GPU: exactness
def _whole_and_bands(gpu_lib, h, w, n, halo, seed=0):
    img = make_image(gpu_lib, h, w, seed=seed)
    enc = EncoderConfig(use_soap=False, lmbda=1e-3, seed=seed)
    dcfg = DecoderConfig.hop()
    whole = Trainer(img, enc, dcfg, lib=gpu_lib)
    lb = B.LocalBands(img, n, enc, dcfg, halo=halo, lib=gpu_lib)
    whole.fresh_candidate(0)
    lb.fresh_candidate(0)
    return whole, lb


@pytest.mark.gpu
def test_band_grid_rows_match_runtime(gpu_lib):
    img = make_image(gpu_lib, 256, 192, seed=1)
    for r0, r1 in B.split_rows(256, 192, 2):
        with B.BandTrainer(img, r0, r1, 6, EncoderConfig(use_soap=False), DecoderConfig.hop(), lib=gpu_lib) as t:
            for gi, g in enumerate(t.grids):
                assert t.grid_rows(gi) == B.band_grid_rows(256, 192, r0, r1, 6, g.level)


@pytest.mark.gpu
@pytest.mark.parametrize("h,w,n", [(256, 192, 2), (1536, 256, 3)])
def test_bands_reproduce_whole_image(gpu_lib, h, w, n):
    whole, lb = _whole_and_bands(gpu_lib, h, w, n, 6)
    try:
        y0 = whole.get_state()["latents"]
        for gi in range(len(whole.grids)):  # same position-keyed initialisation
            assert np.array_equal(lb.gather_grid(0, gi).reshape(-1), whole.grid_view(y0, gi).reshape(-1))
        for it in range(3):
            cw = whole.proxy_iteration(1e-2, 0.35, 0.22)
            cb = lb.proxy_iteration(1e-2, 0.35, 0.22)
            assert abs(cw - cb) <= 1e-6 * abs(cw), (it, cw, cb)
            st = whole.get_state()
            for gi in range(len(whole.grids)):
                assert rel_l2(lb.gather_grid(0, gi).reshape(-1),
                              whole.grid_view(st["latents"], gi).reshape(-1)) <= 1e-4, (it, gi)
            pb = lb.trainers[0].get_state()["params"]
            for ti, p in enumerate(whole.params):
                assert rel_l2(lb.trainers[0].param_view(pb, ti), whole.param_view(st["params"], ti)) <= 1e-4, p.name
            for t in lb.trainers[1:]:  # every rank holds identical parameters
                assert np.array_equal(t.get_state()["params"], pb)
            assert lb.trainers[0].global_iter == whole.global_iter
    finally:
        lb.close()
        whole.close()


@pytest.mark.gpu
def test_band_device_views_are_the_library_buffers(gpu_lib):
    """The zero-copy CUDA views DistBand hands to NCCL (cc_band_device_rows /
    cc_band_device_nn_partial) alias the band trainer's own buffers."""
    import torch

    img = make_image(gpu_lib, 256, 192, seed=2)
    r0, r1 = B.split_rows(256, 192, 2)[1]
    with B.BandTrainer(img, r0, r1, 6, EncoderConfig(use_soap=False), DecoderConfig.hop(), lib=gpu_lib) as t:
        t.fresh_candidate(0)
        gi = len(t.grids) - 1
        gr = t.grid_rows(gi)
        v = t.device_rows(0, gi, gr.w0, gr.o0)
        assert v.is_cuda and v.numel() == (gr.o0 - gr.w0) * t.grids[gi].cols
        assert np.array_equal(v.cpu().numpy(), t.rows(0, gi, gr.w0, gr.o0))
        v.fill_(1.5)
        torch.cuda.synchronize()
        assert np.all(t.rows(0, gi, gr.w0, gr.o0) == 1.5)
        t.forward_backward(1e-2, 0.35, 0.22)
        nn = t.device_nn_partial()
        assert nn.dtype == torch.float64 and np.array_equal(nn.cpu().numpy(), t.nn_partial())


# ------------------------------------- GPU + gloo: real band trainers, 2 ranks
def _band_trainer_worker(rank, world, port, h, w, halo, iters, q):
    import traceback

    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_02726_b200 import capi

        lib = capi.load_product()
        img = make_image(lib, h, w, seed=0)
        bands = B.split_rows(h, w, world)
        enc = EncoderConfig(use_soap=False, lmbda=1e-3, seed=0)
        with B.BandTrainer(img, *bands[rank], halo, enc, DecoderConfig.hop(), lib=lib, device=0) as tr:
            tr.fresh_candidate(0)
            hyper = any(g.hyper for g in tr.grids)
            # host transport (gloo): the routing code the NCCL path also runs
            db = B.DistBand(tr, h, w, bands, halo, hyper, dist, device=None)
            costs = [db.proxy_iteration(1e-2, 0.35, 0.22) for _ in range(iters)]
            own = [tr.rows(0, gi, tr.grid_rows(gi).o0, tr.grid_rows(gi).o1) for gi in range(len(tr.grids))]
            q.put(dict(rank=rank, costs=costs, own=own, params=tr.get_state()["params"],
                       global_iter=tr.global_iter))
    except Exception:  # report instead of leaving the parent waiting
        q.put(dict(rank=rank, error=traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_dist_band_two_ranks_match_local_bands(gpu_lib):
    """Two processes, each driving a REAL BandTrainer through DistBand over
    gloo (host exchange; both on this one GPU — their kernels never wait on one
    another, the ranks meet only in the host collectives), against the same
    bands run in one process (LocalBands): bit-identical costs, latents and
    parameters after 3 iterations (same routing, same rank-order sums)."""
    import torch.multiprocessing as mp

    h, w, halo, iters, world = 256, 192, 6, 3, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_band_trainer_worker, args=(r, world, port, h, w, halo, iters, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda r: r["rank"])
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert "error" not in r, r.get("error")
    img = make_image(gpu_lib, h, w, seed=0)
    enc = EncoderConfig(use_soap=False, lmbda=1e-3, seed=0)
    lb = B.LocalBands(img, world, enc, DecoderConfig.hop(), halo=halo, lib=gpu_lib)
    try:
        lb.fresh_candidate(0)
        costs = [lb.proxy_iteration(1e-2, 0.35, 0.22) for _ in range(iters)]
        for r in res:
            assert r["costs"] == costs, (r["rank"], r["costs"], costs)
            t = lb.trainers[r["rank"]]
            for gi in range(len(t.grids)):
                gr = t.grid_rows(gi)
                assert np.array_equal(r["own"][gi], t.rows(0, gi, gr.o0, gr.o1)), (r["rank"], gi)
            assert np.array_equal(r["params"], t.get_state()["params"])
            assert r["global_iter"] == iters
    finally:
        lb.close()
    assert np.array_equal(res[0]["params"], res[1]["params"])


# ----------------------------- GPU: the exchange inside the library (cc_band.h)
def _states(tr):
    st = tr.get_state()
    own = [tr.rows(0, gi, tr.grid_rows(gi).o0, tr.grid_rows(gi).o1) for gi in range(len(tr.grids))]
    return own, st["params"], tr.global_iter


@pytest.mark.gpu
@pytest.mark.parametrize("h,w,n", [(256, 192, 2), (1536, 256, 3)])
def test_device_bands_match_local_bands(gpu_lib, h, w, n):
    """The device-resident band iteration (cc_band_group_local: halo rows,
    gradient return, rank-order gathers and the flag AND on the trainers'
    streams) is bit-identical to the host-routed LocalBands, and a run of
    iterations costs ONE host synchronisation (the records read)."""
    img = make_image(gpu_lib, h, w, seed=3)
    enc = EncoderConfig(use_soap=False, lmbda=1e-3, seed=3)
    lr = np.array([1e-2, 9e-3, 8e-3, 7e-3, 6e-3])
    tp = np.array([0.35, 0.33, 0.31, 0.29, 0.27])
    ns = np.array([0.22, 0.21, 0.2, 0.19, 0.18])
    lb = B.LocalBands(img, n, enc, DecoderConfig.hop(), halo=6, lib=gpu_lib)
    db = B.DeviceBands(img, n, enc, DecoderConfig.hop(), halo=6, lib=gpu_lib)
    try:
        lb.fresh_candidate(0)
        db.fresh_candidate(0)
        db.group.reserve(len(lr))
        host = [lb.proxy_iteration(lr[i], tp[i], ns[i]) for i in range(len(lr))]
        s0 = B.host_sync_count(gpu_lib)
        dev = db.proxy_iterations(lr, tp, ns)
        syncs = B.host_sync_count(gpu_lib) - s0
        assert list(dev) == host, (list(dev), host)
        assert syncs <= 1, syncs
        for b in range(n):
            o1, p1, g1 = _states(lb.trainers[b])
            o2, p2, g2 = _states(db.trainers[b])
            for gi in range(len(o1)):
                assert np.array_equal(o1[gi], o2[gi]), (b, gi)
            assert np.array_equal(p1, p2), b
            assert g1 == g2 == len(lr)
        # one more iteration at a time through the same group
        assert db.proxy_iteration(5e-3, 0.25, 0.17) == lb.proxy_iteration(5e-3, 0.25, 0.17)
    finally:
        db.close()
        lb.close()


_NCCL1 = r"""
import json, os, sys
import numpy as np
import torch, torch.distributed as dist
sys.path.insert(0, os.getcwd())
from paper_2605_02726_b200 import bands as B, capi
from paper_2605_02726_b200.trainer import DecoderConfig, EncoderConfig
from tests.conftest import make_image
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
lib = capi.load_product()
h, w = 256, 192
img = make_image(lib, h, w, seed=4)
enc = EncoderConfig(use_soap=False, lmbda=1e-3, seed=4)
lr = np.array([1e-2, 9e-3, 8e-3]); tp = np.array([0.35, 0.33, 0.31]); ns = np.array([0.22, 0.21, 0.2])
with B.BandTrainer(img, 0, h, 6, enc, DecoderConfig.hop(), lib=lib, device=0) as tr:
    tr.fresh_candidate(0)
    hyper = any(g.hyper for g in tr.grids)
    db = B.DistBand(tr, h, w, [(0, h)], 6, hyper, dist, device=0)
    costs = list(db.proxy_iterations(lr, tp, ns))
    st = tr.get_state()
    db.close()
    out = dict(costs=costs, params=st["params"].tolist(), lat=st["latents"].tolist(), global_iter=tr.global_iter)
dist.destroy_process_group()
print("RESULT " + json.dumps(out))
"""


@pytest.mark.gpu
def test_nccl_band_group_single_rank_matches_local(gpu_lib, tmp_path):
    """The NCCL transport of the band group (dlopen'ed libnccl, unique id over
    torch.distributed, ncclAllGather of the partials, ncclAllReduce(min) of the
    flags on the trainer's stream) at world size 1 — the one configuration a
    single GPU can run — against the local group: bit-identical."""
    import json
    import subprocess
    import sys

    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    script = tmp_path / "nccl1.py"
    script.write_text(_NCCL1)
    r = subprocess.run([sys.executable, str(script)], cwd=str(ROOT), env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-4000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")][-1]
    got = json.loads(line[7:])
    h, w = 256, 192
    img = make_image(gpu_lib, h, w, seed=4)
    enc = EncoderConfig(use_soap=False, lmbda=1e-3, seed=4)
    db = B.DeviceBands(img, 1, enc, DecoderConfig.hop(), halo=6, lib=gpu_lib)
    try:
        db.fresh_candidate(0)
        costs = list(db.proxy_iterations([1e-2, 9e-3, 8e-3], [0.35, 0.33, 0.31], [0.22, 0.21, 0.2]))
        st = db.trainers[0].get_state()
        assert got["costs"] == costs
        assert np.array_equal(np.array(got["params"], np.float32), st["params"])
        assert np.array_equal(np.array(got["lat"], np.float32), st["latents"])
        assert got["global_iter"] == 3
    finally:
        db.close()

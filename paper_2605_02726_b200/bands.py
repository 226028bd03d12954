"""Row-band decomposition of one large image across ranks (BASELINE config 5,
SURVEY.md §8e): rank b owns full-resolution rows [r0, r1) and runs the
iteration on its band plus halo rows; per proxy_iteration (encoder.hpp:97-135)
the ranks exchange

  1. latent halo rows y (owner -> neighbours) before the iteration,
  2. partial latent gradients of halo rows (neighbour -> owner, added),
  3. NN-gradient partial sums and the bits / squared-error sums, gathered and
     summed in rank order (every rank ends with bit-identical parameters),
  4. the per-grid "all gradients finite" flags (AND over ranks),

then every rank takes the same Adam steps.  The device work lives behind
include/coolchic_b200_band.h; this module is the host side: the band layout,
the routing of halo rows, and two transports —

  * LocalBands: all bands in one process (one GPU or several), exchange by
    host copies; used by the single-GPU equivalence test;
  * DistBand: one band per rank over torch.distributed (gloo on CPU: host
    routing; CUDA band trainers: the library's NCCL band group below);
  * DeviceBands / the NCCL band group: the same iteration with the exchange
    inside the library on the trainers' streams (csrc/cc_band.h) — a run of
    iterations is enqueued without host synchronisation, bit-identical to the
    host-routed transports.

The routing logic is transport-independent (``halo_plan``), so the gloo
world-size-2 tests exercise exactly what the NCCL path runs.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import capi
from .trainer import ConfigError, DecoderConfig, EncoderConfig, Trainer, _check


def latent_levels(h: int, w: int) -> int:
    """config.hpp:84: 7 levels below 1 Mpx, else 8."""
    return 7 if h * w < 1_000_000 else 8


def grid_levels(h: int, w: int, hyper: bool) -> list[int]:
    """Levels of the grids in decode order (latent.hpp:66-68)."""
    L = latent_levels(h, w)
    out = [k for k in range(L - 1, 3, -1)] if hyper else []
    return out + list(range(L - 1, -1, -1))


def split_rows(h: int, w: int, nbands: int) -> list[tuple[int, int]]:
    """Equal bands with edges on multiples of 2^(L-1) (the last band takes the rest)."""
    L = latent_levels(h, w)
    a = 1 << (L - 1)
    units = -(-h // a)
    if units < nbands:
        raise ConfigError(f"{h} rows cannot form {nbands} bands of 2^{L - 1}-row units")
    edges = [min(h, (units * b // nbands) * a) for b in range(nbands + 1)]
    edges[-1] = h
    return [(edges[b], edges[b + 1]) for b in range(nbands)]


@dataclass(frozen=True)
class GridRows:
    """Global rows of one grid of one band: window [w0, w1) ⊇ own [o0, o1)."""
    w0: int
    o0: int
    o1: int
    w1: int


def band_grid_rows(h: int, w: int, r0: int, r1: int, halo: int, level: int) -> GridRows:
    """Mirror of Trainer::build_plan's band geometry (cc_runtime.cu)."""
    rows = -(-h // (1 << level))
    o0 = r0 >> level
    o1 = rows if r1 == h else r1 >> level
    return GridRows(max(0, o0 - halo), o0, o1, min(rows, o1 + halo))


def halo_plan(h: int, w: int, bands: list[tuple[int, int]], halo: int, hyper: bool, b: int):
    """Per grid, the row ranges band b exchanges with its neighbours.

    Returns a list over grids of dicts with
      ``send_up`` / ``send_down``: own rows neighbour b-1 / b+1 holds as halo
      (y is sent there before an iteration);
      ``halo_up`` / ``halo_down``: rows of this band's window owned by b-1 / b+1
      (their partial gradients are returned there after the backward).
    The two sides agree by construction: send_down(b) == halo_up(b+1), etc.
    """
    out = []
    for lvl in grid_levels(h, w, hyper):
        me = band_grid_rows(h, w, *bands[b], halo, lvl)
        d = dict(level=lvl, rows=me, send_up=(0, 0), send_down=(0, 0), halo_up=(me.w0, me.o0),
                 halo_down=(me.o1, me.w1))
        if b > 0:
            up = band_grid_rows(h, w, *bands[b - 1], halo, lvl)
            d["send_up"] = (me.o0, up.w1)
            if up.o0 > me.w0:
                raise ConfigError("halo deeper than the neighbouring band")
        if b + 1 < len(bands):
            dn = band_grid_rows(h, w, *bands[b + 1], halo, lvl)
            d["send_down"] = (dn.w0, me.o1)
            if dn.o1 < me.w1:
                raise ConfigError("halo deeper than the neighbouring band")
        out.append(d)
    return out


class BandTrainer(Trainer):
    """One band's device trainer (include/coolchic_b200_band.h)."""

    def __init__(self, image: np.ndarray, r0: int, r1: int, halo: int, enc: EncoderConfig,
                 dcfg: DecoderConfig, lib=None, device: int = 0):
        lib = lib or capi.load_product()
        h, w = image.shape[1], image.shape[2]
        w0, w1 = C.c_int(), C.c_int()
        _check(lib, lib.cc_band_window(h, w, r0, r1, halo, C.byref(w0), C.byref(w1)))
        self.H, self.W, self.r0, self.r1, self.halo = h, w, r0, r1, halo
        self.window = (w0.value, w1.value)
        self._device = device
        super().__init__(np.ascontiguousarray(image[:, w0.value:w1.value]), enc, dcfg, lib=lib,
                         device=device, band=(h, r0, r1, halo))

    def grid_rows(self, gi: int) -> GridRows:
        o = (C.c_int * 4)()
        _check(self.lib, self.lib.cc_band_grid_rows(self._h, gi, o))
        return GridRows(*o)

    def rows(self, which: int, gi: int, rb: int, re: int, buf: np.ndarray | None = None,
             mode: int = 0) -> np.ndarray:
        cols = self.grids[gi].cols
        if buf is None:
            buf = np.empty((re - rb) * cols, np.float32)
        buf = np.ascontiguousarray(buf, dtype=np.float32)
        assert buf.size == (re - rb) * cols
        _check(self.lib, self.lib.cc_band_rows(self._h, which, gi, rb, re,
                                               buf.ctypes.data_as(C.POINTER(C.c_float)), mode))
        return buf

    def device_rows(self, which: int, gi: int, rb: int, re: int):
        """Zero-copy torch CUDA view of global rows [rb, re) of grid gi."""
        ptr, n = C.c_void_p(), C.c_int64()
        _check(self.lib, self.lib.cc_band_device_rows(self._h, which, gi, rb, re, C.byref(ptr), C.byref(n)))
        return _device_view(ptr.value, n.value, "<f4", self._device)

    def device_nn_partial(self):
        ptr, n = C.c_void_p(), C.c_int64()
        _check(self.lib, self.lib.cc_band_device_nn_partial(self._h, C.byref(ptr), C.byref(n)))
        return _device_view(ptr.value, n.value, "<f8", self._device)

    def forward_backward(self, lr, temp, noise):
        b, s = C.c_double(), C.c_double()
        _check(self.lib, self.lib.cc_band_forward_backward(self._h, lr, temp, noise, C.byref(b),
                                                           C.byref(s)))
        return b.value, s.value

    def nn_partial(self) -> np.ndarray:
        out = np.empty(self.n_params, np.float64)
        _check(self.lib, self.lib.cc_band_nn_partial(self._h,
                                                     out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def finish(self, nn_sums: np.ndarray, bits: float, sq_err: float):
        nn = np.ascontiguousarray(nn_sums, dtype=np.float64)
        cost = C.c_double()
        ok = (C.c_int * len(self.grids))()
        _check(self.lib, self.lib.cc_band_finish(self._h, nn.ctypes.data_as(C.POINTER(C.c_double)),
                                                 bits, sq_err, C.byref(cost), ok))
        return cost.value, np.array(list(ok), np.int32)

    def step(self, lat_ok: np.ndarray) -> None:
        ok = (C.c_int * len(self.grids))(*[int(v) for v in lat_ok])
        _check(self.lib, self.lib.cc_band_step(self._h, ok))


class _CudaArray:
    """__cuda_array_interface__ around a device address owned by the library."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def _device_view(ptr: int, n: int, typestr: str, device: int):
    import torch

    if n == 0:
        return torch.empty(0, dtype=torch.float32 if typestr == "<f4" else torch.float64,
                           device=f"cuda:{device}")
    return torch.as_tensor(_CudaArray(ptr, n, typestr), device=f"cuda:{device}")


# ---------------------------------------------------------------- one iteration
# The iteration is written once against a "mailbox" API so the in-process and
# the distributed transports run the same routing code.

def _pack(tr, which: int, plan, key: str) -> np.ndarray:
    parts = [tr.rows(which, gi, *d[key]) for gi, d in enumerate(plan) if d[key][1] > d[key][0]]
    return np.concatenate(parts) if parts else np.zeros(0, np.float32)


def _unpack(tr, which: int, plan, key: str, flat: np.ndarray, mode: int) -> None:
    pos = 0
    for gi, d in enumerate(plan):
        rb, re = d[key]
        if re <= rb:
            continue
        n = (re - rb) * tr.grids[gi].cols
        tr.rows(which, gi, rb, re, flat[pos:pos + n], mode)
        pos += n
    assert pos == flat.size


class LocalBands:
    """All bands of one image in this process; exchange by host copies."""

    def __init__(self, image: np.ndarray, nbands: int, enc: EncoderConfig, dcfg: DecoderConfig,
                 halo: int = 8, devices: list[int] | None = None, lib=None):
        h, w = image.shape[1], image.shape[2]
        self.H, self.W, self.halo = h, w, halo
        self.bands = split_rows(h, w, nbands)
        devices = devices or [0] * nbands
        self.trainers = [BandTrainer(image, r0, r1, halo, enc, dcfg, lib=lib, device=devices[b])
                         for b, (r0, r1) in enumerate(self.bands)]
        hyper = any(g.hyper for g in self.trainers[0].grids)
        self.plans = [halo_plan(h, w, self.bands, halo, hyper, b) for b in range(nbands)]

    def close(self):
        for t in self.trainers:
            t.close()

    def fresh_candidate(self, index: int) -> None:
        for t in self.trainers:
            t.fresh_candidate(index)

    def refresh_halos(self) -> None:
        """y rows: owner -> neighbours (before an iteration)."""
        n = len(self.trainers)
        for b in range(n):
            t, p = self.trainers[b], self.plans[b]
            if b > 0:
                _unpack(self.trainers[b - 1], 0, self.plans[b - 1], "halo_down", _pack(t, 0, p, "send_up"), 1)
            if b + 1 < n:
                _unpack(self.trainers[b + 1], 0, self.plans[b + 1], "halo_up", _pack(t, 0, p, "send_down"), 1)

    def proxy_iteration(self, lr: float, temp: float, noise: float) -> float:
        n = len(self.trainers)
        self.refresh_halos()
        sums = [t.forward_backward(lr, temp, noise) for t in self.trainers]
        # halo latent gradients -> owners (added in rank order of the senders)
        outs = [(_pack(t, 1, p, "halo_up"), _pack(t, 1, p, "halo_down"))
                for t, p in zip(self.trainers, self.plans)]
        for b in range(n):
            t, p = self.trainers[b], self.plans[b]
            if b > 0:
                _unpack(t, 1, p, "send_up", outs[b - 1][1], 2)
            if b + 1 < n:
                _unpack(t, 1, p, "send_down", outs[b + 1][0], 2)
        nn = np.zeros(self.trainers[0].n_params, np.float64)
        for t in self.trainers:
            nn = nn + t.nn_partial()
        # rank-order sums, as the device band group (k_band_finish); Python's
        # sum() of floats is compensated (3.12+) and would round differently
        bits = se = 0.0
        for s in sums:
            bits += float(s[0])
            se += float(s[1])
        oks = []
        cost = None
        for t in self.trainers:
            cost, ok = t.finish(nn, bits, se)
            oks.append(ok)
        ok = np.minimum.reduce(oks)
        for t in self.trainers:
            t.step(ok)
        return cost

    def gather_grid(self, which: int, gi: int) -> np.ndarray:
        """Own rows of every band, concatenated: the whole grid."""
        return np.concatenate([t.rows(which, gi, t.grid_rows(gi).o0, t.grid_rows(gi).o1)
                               for t in self.trainers])


def _sched(lr, temp, noise):
    lr = np.ascontiguousarray(np.atleast_1d(lr), np.float64)
    n = lr.size
    temp = np.ascontiguousarray(np.broadcast_to(temp, (n,)), np.float64)
    noise = np.ascontiguousarray(np.broadcast_to(noise, (n,)), np.float64)
    return n, lr, temp, noise


class _Group:
    """A library band group (cc_band_group_*): enqueue / synchronise / records."""

    def __init__(self, lib, handle: C.c_void_p, record_trainer):
        self.lib, self._h, self._rec_tr = lib, handle, record_trainer

    def reserve(self, n: int) -> None:
        _check(self.lib, self.lib.cc_band_group_reserve(self._h, n))

    def enqueue_proxy_iterations(self, lr, temp, noise) -> int:
        n, lr, temp, noise = _sched(lr, temp, noise)
        dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
        _check(self.lib, self.lib.cc_band_group_enqueue_proxy_iterations(self._h, n, dp(lr), dp(temp),
                                                                         dp(noise)))
        return n

    def synchronize(self) -> None:
        _check(self.lib, self.lib.cc_band_group_synchronize(self._h))

    def records(self, n: int) -> np.ndarray:
        """(n, 4): cost, mse, bits, global_iter of the last n iterations (waits)."""
        rec = np.empty(4 * n, np.float64)
        _check(self.lib, self.lib.cc_trainer_last_records(self._rec_tr._h, n,
                                                          rec.ctypes.data_as(C.POINTER(C.c_double))))
        return rec.reshape(n, 4)

    def proxy_iterations(self, lr, temp, noise) -> np.ndarray:
        n = self.enqueue_proxy_iterations(lr, temp, noise)
        return self.records(n)[:, 0]

    def close(self) -> None:
        if self._h:
            self.lib.cc_band_group_destroy(self._h)
            self._h = C.c_void_p()


def host_sync_count(lib) -> int:
    n = C.c_int64()
    _check(lib, lib.ccb_host_sync_count(C.byref(n)))
    return n.value


class DeviceBands(LocalBands):
    """All bands of one image in this process with the exchange inside the
    library (cc_band_group_local): a run of iterations is enqueued without
    host synchronisation; results are bit-identical to LocalBands."""

    def __init__(self, image: np.ndarray, nbands: int, enc: EncoderConfig, dcfg: DecoderConfig,
                 halo: int = 8, devices: list[int] | None = None, lib=None):
        super().__init__(image, nbands, enc, dcfg, halo=halo, devices=devices, lib=lib)
        lib = self.trainers[0].lib
        arr = (C.c_void_p * nbands)(*[t._h.value for t in self.trainers])
        h = C.c_void_p()
        _check(lib, lib.cc_band_group_local(arr, nbands, C.byref(h)))
        self.group = _Group(lib, h, self.trainers[0])

    def proxy_iterations(self, lr, temp, noise) -> np.ndarray:
        return self.group.proxy_iterations(lr, temp, noise)

    def proxy_iteration(self, lr: float, temp: float, noise: float) -> float:
        return float(self.group.proxy_iterations([lr], temp, noise)[0])

    def close(self):
        self.group.close()
        super().close()


class DistBand:
    """This rank's band over torch.distributed (NCCL device tensors between
    GPUs; gloo host tensors on CPU).  ``tr`` is any object with the
    BandTrainer surface (rows / forward_backward / nn_partial / finish /
    step), which lets the CPU tests drive the routing with a host model."""

    def __init__(self, tr, h: int, w: int, bands, halo: int, hyper: bool, dist, device=None):
        self.tr, self.dist, self.device = tr, dist, device
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.bands = list(bands)
        self.plan = halo_plan(h, w, bands, halo, hyper, self.rank)
        self.group = None

    def _t(self, a: np.ndarray):
        import torch
        t = torch.from_numpy(np.ascontiguousarray(a))
        return t.to(self.device) if self.device is not None else t

    def _np(self, t) -> np.ndarray:
        return t.cpu().numpy()

    def _swap(self, up_send: np.ndarray | None, down_send: np.ndarray | None, up_n: int,
              down_n: int, dtype):
        """Paired exchange with both neighbours; returns (from_up, from_down)."""
        ops, recv_up, recv_down = [], None, None
        P = self.dist.P2POp
        if self.rank > 0:
            recv_up = self._t(np.zeros(up_n, dtype))
            ops.append(P(self.dist.isend, self._t(up_send), self.rank - 1))
            ops.append(P(self.dist.irecv, recv_up, self.rank - 1))
        if self.rank + 1 < self.world:
            recv_down = self._t(np.zeros(down_n, dtype))
            ops.append(P(self.dist.isend, self._t(down_send), self.rank + 1))
            ops.append(P(self.dist.irecv, recv_down, self.rank + 1))
        if ops:
            for r in self.dist.batch_isend_irecv(ops):
                r.wait()
        return (None if recv_up is None else self._np(recv_up),
                None if recv_down is None else self._np(recv_down))

    def _size(self, key: str) -> int:
        return sum((d[key][1] - d[key][0]) * self.tr.grids[gi].cols
                   for gi, d in enumerate(self.plan))

    def refresh_halos(self) -> None:
        up, dn = self._swap(_pack(self.tr, 0, self.plan, "send_up"),
                            _pack(self.tr, 0, self.plan, "send_down"),
                            self._size("halo_up"), self._size("halo_down"), np.float32)
        if up is not None:
            _unpack(self.tr, 0, self.plan, "halo_up", up, 1)
        if dn is not None:
            _unpack(self.tr, 0, self.plan, "halo_down", dn, 1)

    def _gather(self, a: np.ndarray) -> list[np.ndarray]:
        t = self._t(a)
        bufs = [self._t(np.zeros_like(a)) for _ in range(self.world)]
        self.dist.all_gather(bufs, t)
        return [self._np(x) for x in bufs]

    # ---- device path: the library's NCCL band group (cc_band_group_nccl) runs
    # the exchange on the trainer's stream; torch.distributed only shares the
    # NCCL unique id
    def _device_ok(self) -> bool:
        return self.device is not None and hasattr(self.tr, "device_rows")

    def _nccl_group(self) -> _Group:
        if self.group is None:
            lib = self.tr.lib
            uid = (C.c_char * 128)()
            if self.rank == 0:
                _check(lib, lib.cc_band_nccl_unique_id(uid))
            box = [bytes(uid)]
            self.dist.broadcast_object_list(box, src=0)
            uid = (C.c_char * 128).from_buffer_copy(box[0])
            edges = (C.c_int * (self.world + 1))(*([r0 for r0, _ in self.bands] + [self.bands[-1][1]]))
            h = C.c_void_p()
            _check(lib, lib.cc_band_group_nccl(self.tr._h, uid, self.world, self.rank, edges, C.byref(h)))
            self.group = _Group(lib, h, self.tr)
        return self.group

    def proxy_iterations(self, lr, temp, noise) -> np.ndarray:
        """n iterations enqueued at once (device path: one host wait at the end)."""
        if self._device_ok():
            return self._nccl_group().proxy_iterations(lr, temp, noise)
        n, lr, temp, noise = _sched(lr, temp, noise)
        return np.array([self.proxy_iteration(lr[i], temp[i], noise[i]) for i in range(n)])

    def close(self) -> None:
        if self.group is not None:
            self.group.close()
            self.group = None

    def proxy_iteration(self, lr: float, temp: float, noise: float) -> float:
        if self._device_ok():
            return float(self._nccl_group().proxy_iterations([lr], temp, noise)[0])
        self.refresh_halos()
        bits, se = self.tr.forward_backward(lr, temp, noise)
        up, dn = self._swap(_pack(self.tr, 1, self.plan, "halo_up"),
                            _pack(self.tr, 1, self.plan, "halo_down"),
                            self._size("send_up"), self._size("send_down"), np.float32)
        if up is not None:
            _unpack(self.tr, 1, self.plan, "send_up", up, 2)
        if dn is not None:
            _unpack(self.tr, 1, self.plan, "send_down", dn, 2)
        parts = self._gather(np.concatenate([self.tr.nn_partial(), np.array([bits, se])]))
        tot = np.zeros_like(parts[0])
        for p in parts:  # rank order: identical sums on every rank
            tot = tot + p
        cost, ok = self.tr.finish(tot[:-2], float(tot[-2]), float(tot[-1]))
        oks = self._gather(ok.astype(np.int32))
        self.tr.step(np.minimum.reduce(oks))
        return cost

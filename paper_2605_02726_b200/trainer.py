"""Python mirror of the reference encoder API over the C ABI.

Names, argument meaning and error behaviour follow
``coolcodec::detail::Trainer`` (encoder.hpp:59-306), ``warmup``
(encoder.hpp:315-342), ``train`` (encoder.hpp:349-413) and the config structs
(config.hpp:17-142).  The heavy lifting happens behind the C ABI: in the B200
library every call below runs sm_100a kernels; the host loop of ``train`` runs
in that library's C++ runtime.  This module only marshals numpy buffers.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field, fields

import numpy as np

from . import capi


class CodecError(RuntimeError):
    """coolcodec::CodecError (tensor.hpp:11-13)."""


class ConfigError(CodecError):
    """coolcodec::ConfigError (tensor.hpp:19-21)."""


class FormatError(CodecError):
    """coolcodec::FormatError (tensor.hpp:15-17)."""


class TrainingError(CodecError):
    """coolcodec::TrainingError (tensor.hpp:23-25)."""


class DeviceError(CodecError):
    """CUDA / device failure inside the B200 library."""


_ERRORS = {
    capi.CC_ERR_CONFIG: ConfigError,
    capi.CC_ERR_FORMAT: FormatError,
    capi.CC_ERR_TRAINING: TrainingError,
    capi.CC_ERR_CUDA: DeviceError,
    capi.CC_ERR_STATE: CodecError,
}


def _check(lib, rc: int) -> None:
    if rc != capi.CC_OK:
        msg = lib.cc_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, CodecError)(msg)


def _fp(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_float))


def _ip(a: np.ndarray | None, t=C.c_int64):
    return None if a is None else a.ctypes.data_as(C.POINTER(t))


@dataclass
class DecoderConfig:
    """config.hpp:40-81 (default = HOP)."""

    preset: int = 2
    spatial_ctx: int = 14
    ifce_dim: int = 6
    arm_width: int = 20
    arm_hidden: int = 2
    synth_hidden: int = 48
    synth_posts: int = 2
    use_hyperlatents: bool = True
    use_stabilizer: bool = True

    @staticmethod
    def lop():
        return DecoderConfig(0, 6, 2, 8, 2, 8, 1, True, True)

    @staticmethod
    def mop():
        return DecoderConfig(1, 10, 4, 10, 2, 16, 2, True, True)

    @staticmethod
    def hop():
        return DecoderConfig(2, 14, 6, 20, 2, 48, 2, True, True)

    @staticmethod
    def vhop():
        return DecoderConfig(3, 20, 6, 26, 2, 64, 2, True, True)

    @staticmethod
    def cfg4():
        """BASELINE config 4's higher-complexity decoder: ARM context
        26 + IFCE 6 (d = 32), width 20, synthesis hidden 64."""
        return DecoderConfig(2, 26, 6, 20, 2, 64, 2, True, True)

    @staticmethod
    def from_name(name: str):
        try:
            return {"lop": DecoderConfig.lop, "mop": DecoderConfig.mop, "hop": DecoderConfig.hop,
                    "vhop": DecoderConfig.vhop, "cfg4": DecoderConfig.cfg4}[name]()
        except KeyError:
            raise ConfigError(f"unknown decoder config: {name}") from None

    def arm_input_dim(self) -> int:
        return self.spatial_ctx + self.ifce_dim

    def to_c(self) -> capi.DecoderConfigC:
        return capi.DecoderConfigC(*[int(getattr(self, f.name)) for f in fields(self)])


@dataclass
class EncoderConfig:
    """config.hpp:93-142 (``lambda`` is spelled ``lmbda``)."""

    warmup_candidates: int = 5
    warmup_keep: int = 2
    warmup_iters: int = 400
    main_iters: int = 96700
    hardround_iters: int = 500
    lr_start: float = 1e-2
    lr_end: float = 1e-6
    noise_std_start: float = 0.22
    noise_std_end: float = 0.15
    temp_start: float = 0.35
    temp_end: float = 0.08
    hardround_lr: float = 1e-4
    lmbda: float = 0.001
    seed: int = 0
    use_soap: bool = True  # the reference default (config.hpp:107); benchmarks and parity runs clear it
    true_cost_interval: int = 1000
    log_path: str = ""

    def warmup_total(self) -> int:
        return (self.warmup_candidates + self.warmup_keep) * self.warmup_iters

    def total_iters(self) -> int:
        return self.warmup_total() + self.main_iters + self.hardround_iters

    @staticmethod
    def with_total(total: int) -> "EncoderConfig":
        """EncoderConfig::with_total (config.hpp:127-141)."""
        cfg = EncoderConfig()
        if total == EncoderConfig().total_iters():
            return cfg
        if total < 20:
            raise ConfigError("iteration budget too small")
        f = total / 100000.0
        cfg.warmup_iters = max(1, _lround(400.0 * f))
        cfg.hardround_iters = max(1, _lround(500.0 * f))
        rest = total - cfg.warmup_total() - cfg.hardround_iters
        while rest < 1 and cfg.warmup_iters > 1:
            cfg.warmup_iters -= 1
            rest = total - cfg.warmup_total() - cfg.hardround_iters
        cfg.main_iters = max(1, rest)
        return cfg

    def schedules(self):
        h = max(1, self.main_iters - 1)
        return (Schedule(self.lr_start, self.lr_end, "cosine", h),
                Schedule(self.temp_start, self.temp_end, "linear", h),
                Schedule(self.noise_std_start, self.noise_std_end, "linear", h))

    def to_c(self) -> capi.EncoderConfigC:
        c = capi.EncoderConfigC()
        for f in fields(self):
            if f.name == "lmbda":
                c.lambda_ = float(self.lmbda)
            elif f.name == "log_path":
                self._log_bytes = (self.log_path or "").encode()
                c.log_path = self._log_bytes
            else:
                setattr(c, f.name, getattr(self, f.name))
        return c


def _lround(x: float) -> int:
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


@dataclass
class Schedule:
    """Schedule::value (config.hpp:17-30)."""

    start: float
    end: float
    kind: str = "linear"
    horizon: int = 1

    def value(self, it: int) -> float:
        if it <= 0:
            return self.start
        if it >= self.horizon:
            return self.end
        t = it / self.horizon
        if self.kind == "linear":
            return self.start + (self.end - self.start) * t
        return self.end + (self.start - self.end) * (1.0 + math.cos(math.pi * t)) * 0.5


@dataclass
class GridInfo:
    level: int
    hyper: bool
    rows: int
    cols: int
    offset: int
    ifce_slot: int

    @property
    def count(self) -> int:
        return self.rows * self.cols


@dataclass
class ParamInfo:
    name: str
    rows: int
    cols: int
    size: int
    offset: int


@dataclass
class TrainStats:
    """TrainStats (encoder.hpp:24-32)."""

    iterations: int = 0
    true_cost: float = math.inf
    psnr: float = 0.0
    rate_bpp: float = 0.0
    restarts: int = 0
    skipped_steps: int = 0
    seconds: float = 0.0


@dataclass
class TrainResult:
    latents: np.ndarray
    q: np.ndarray
    params: np.ndarray
    stats: TrainStats = field(default_factory=TrainStats)


def make_synthetic_image(h: int, w: int, seed: int, lib=None) -> np.ndarray:
    lib = lib or capi.load_product()
    out = np.empty((3, h, w), np.float32)
    _check(lib, lib.cc_make_synthetic_image(h, w, seed, _fp(out)))
    return out


class Trainer:
    """detail::Trainer (encoder.hpp:59-306) over any library exporting the C ABI.

    ``lib`` defaults to the B200 product library.  The image is copied to the
    device at construction (the reference keeps a ``const Image&``).
    """

    def __init__(self, image: np.ndarray, enc: EncoderConfig, dcfg: DecoderConfig, lib=None,
                 device: int = 0, band: tuple[int, int, int, int] | None = None):
        self.lib = lib or capi.load_product()
        img = np.ascontiguousarray(image, dtype=np.float32)
        if img.ndim != 3 or img.shape[0] != 3:
            raise ConfigError("image must be planar (3, H, W)")
        self.enc = enc
        self.dcfg = dcfg
        self._h = C.c_void_p()
        self._enc_c = enc.to_c()
        self._dec_c = dcfg.to_c()
        self.band = band
        if band is None:
            _check(self.lib, self.lib.cc_trainer_create(_fp(img), img.shape[1], img.shape[2],
                                                        C.byref(self._enc_c), C.byref(self._dec_c),
                                                        device, C.byref(self._h)))
        else:  # one row band (H, r0, r1, halo) of a larger image; img = the band window
            hg, r0, r1, halo = band
            _check(self.lib, self.lib.cc_band_trainer_create(
                _fp(img), hg, img.shape[2], r0, r1, halo, C.byref(self._enc_c),
                C.byref(self._dec_c), device, C.byref(self._h)))
        lay = capi.LayoutC()
        _check(self.lib, self.lib.cc_trainer_layout(self._h, C.byref(lay)))
        self.layout = lay
        self.grids = []
        for gi in range(lay.n_grids):
            g = capi.GridInfoC()
            _check(self.lib, self.lib.cc_trainer_grid_info(self._h, gi, C.byref(g)))
            self.grids.append(GridInfo(g.level, bool(g.hyper), g.rows, g.cols, g.offset,
                                       g.ifce_slot))
        self.params = []
        for ti in range(lay.n_tensors):
            p = capi.ParamInfoC()
            _check(self.lib, self.lib.cc_trainer_param_info(self._h, ti, C.byref(p)))
            self.params.append(ParamInfo(p.name.decode(), p.rows, p.cols, p.size, p.offset))

    def close(self):
        if self._h:
            self.lib.cc_trainer_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---- sizes -----------------------------------------------------------
    @property
    def n_latents(self) -> int:
        return int(self.layout.n_latents)

    @property
    def n_params(self) -> int:
        return int(self.layout.n_params)

    @property
    def npix(self) -> int:
        return self.layout.height * self.layout.width

    # ---- reference surface -------------------------------------------------
    def upload_image(self, image: np.ndarray) -> None:
        img = np.ascontiguousarray(image, dtype=np.float32)
        _check(self.lib, self.lib.cc_trainer_upload_image(self._h, _fp(img)))

    def fresh_candidate(self, index: int) -> None:
        _check(self.lib, self.lib.cc_trainer_fresh_candidate(self._h, index))

    def proxy_iteration(self, lr: float, temp: float, noise_std: float) -> float:
        c = C.c_double()
        _check(self.lib, self.lib.cc_trainer_proxy_iteration(self._h, lr, temp, noise_std,
                                                             C.byref(c)))
        return c.value

    def proxy_iterations(self, lr, temp, noise_std) -> np.ndarray:
        lr = np.ascontiguousarray(lr, np.float64)
        n = lr.size
        temp = np.ascontiguousarray(np.broadcast_to(temp, (n,)), np.float64)
        noise_std = np.ascontiguousarray(np.broadcast_to(noise_std, (n,)), np.float64)
        costs = np.empty(n, np.float64)
        ran = C.c_int()
        dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
        _check(self.lib, self.lib.cc_trainer_proxy_iterations(self._h, n, dp(lr), dp(temp),
                                                              dp(noise_std), dp(costs),
                                                              C.byref(ran)))
        return costs

    def hardround_iteration(self, lr: float, best_slot: int = -1) -> float:
        c = C.c_double()
        _check(self.lib, self.lib.cc_trainer_hardround_iteration(self._h, lr, best_slot,
                                                                 C.byref(c)))
        return c.value

    def true_cost(self):
        c, p, b = C.c_double(), C.c_double(), C.c_double()
        _check(self.lib, self.lib.cc_trainer_true_cost(self._h, C.byref(c), C.byref(p),
                                                       C.byref(b)))
        return c.value, p.value, b.value

    def quantize_all(self) -> None:
        _check(self.lib, self.lib.cc_trainer_quantize_all(self._h))

    def load_pads_from_q(self) -> None:
        _check(self.lib, self.lib.cc_trainer_load_pads_from_q(self._h))

    def last_terms(self):
        m, b = C.c_double(), C.c_double()
        _check(self.lib, self.lib.cc_trainer_last_terms(self._h, C.byref(m), C.byref(b)))
        return m.value, b.value

    def last_mse(self) -> float:
        return self.last_terms()[0]

    def last_bits(self) -> float:
        return self.last_terms()[1]

    def snapshot(self, slot: int, cost: float) -> None:
        _check(self.lib, self.lib.cc_trainer_snapshot(self._h, slot, cost))

    def snapshot_cost(self, slot: int) -> float:
        c = C.c_double()
        _check(self.lib, self.lib.cc_trainer_snapshot_cost(self._h, slot, C.byref(c)))
        return c.value

    def restore(self, slot: int) -> None:
        _check(self.lib, self.lib.cc_trainer_restore(self._h, slot))

    def reset_optimizers(self) -> None:
        _check(self.lib, self.lib.cc_trainer_reset_optimizers(self._h))

    def take_candidate(self, slot: int, cost: float) -> None:
        _check(self.lib, self.lib.cc_trainer_take_candidate(self._h, slot, cost))

    def load_candidate(self, slot: int) -> None:
        _check(self.lib, self.lib.cc_trainer_load_candidate(self._h, slot))

    def candidate_cost(self, slot: int) -> float:
        c = C.c_double()
        _check(self.lib, self.lib.cc_trainer_candidate_cost(self._h, slot, C.byref(c)))
        return c.value

    def warmup(self) -> None:
        _check(self.lib, self.lib.cc_trainer_warmup(self._h))

    def train(self) -> TrainResult:
        st = capi.TrainStatsC()
        lat = np.empty(self.n_latents, np.float32)
        q = np.empty(self.n_latents, np.int32)
        par = np.empty(self.n_params, np.float32)
        _check(self.lib, self.lib.cc_trainer_train(self._h, C.byref(st), _fp(lat),
                                                   _ip(q, C.c_int32), _fp(par)))
        stats = TrainStats(st.iterations, st.true_cost, st.psnr, st.rate_bpp, st.restarts,
                           st.skipped_steps, st.seconds)
        return TrainResult(lat, q, par, stats)

    @property
    def global_iter(self) -> int:
        return self.counters()[0]

    @global_iter.setter
    def global_iter(self, v: int) -> None:
        _check(self.lib, self.lib.cc_trainer_set_counters(self._h, int(v), self.skipped_steps))

    @property
    def skipped_steps(self) -> int:
        return self.counters()[1]

    def counters(self):
        g, s = C.c_int64(), C.c_int()
        _check(self.lib, self.lib.cc_trainer_get_counters(self._h, C.byref(g), C.byref(s)))
        return g.value, s.value

    # ---- lock-step state transfer ------------------------------------------
    def get_state(self) -> dict:
        nl, npar = self.n_latents, self.n_params
        st = dict(latents=np.empty(nl, np.float32), params=np.empty(npar, np.float32),
                  lat_m=np.empty(nl, np.float32), lat_v=np.empty(nl, np.float32),
                  lat_t=np.empty(len(self.grids), np.int64),
                  nn_m=np.empty(npar, np.float32), nn_v=np.empty(npar, np.float32),
                  nn_t=np.empty(len(self.params), np.int64))
        if self.enc.use_soap:  # SOAP state does not transfer (as the reference ABI)
            st["nn_m"] = st["nn_v"] = st["nn_t"] = None
        _check(self.lib, self.lib.cc_trainer_get_state(
            self._h, _fp(st["latents"]), _fp(st["params"]), _fp(st["lat_m"]), _fp(st["lat_v"]),
            _ip(st["lat_t"]), None if st["nn_m"] is None else _fp(st["nn_m"]),
            None if st["nn_v"] is None else _fp(st["nn_v"]),
            None if st["nn_t"] is None else _ip(st["nn_t"])))
        st["global_iter"], st["skipped_steps"] = self.counters()
        return st

    def set_state(self, st: dict) -> None:
        g = lambda k, dt: (None if st.get(k) is None  # noqa: E731
                           else np.ascontiguousarray(st[k], dtype=dt))
        arrs = dict(latents=g("latents", np.float32), params=g("params", np.float32),
                    lat_m=g("lat_m", np.float32), lat_v=g("lat_v", np.float32),
                    lat_t=g("lat_t", np.int64), nn_m=g("nn_m", np.float32),
                    nn_v=g("nn_v", np.float32), nn_t=g("nn_t", np.int64))
        _check(self.lib, self.lib.cc_trainer_set_state(
            self._h, _fp(arrs["latents"]), _fp(arrs["params"]), _fp(arrs["lat_m"]),
            _fp(arrs["lat_v"]), _ip(arrs["lat_t"]), _fp(arrs["nn_m"]), _fp(arrs["nn_v"]),
            _ip(arrs["nn_t"])))
        if "global_iter" in st:
            _check(self.lib, self.lib.cc_trainer_set_counters(
                self._h, int(st["global_iter"]), int(st.get("skipped_steps", 0))))

    def set_q(self, q: np.ndarray) -> None:
        """Quantised latents (flat layout) for the decode passes."""
        qa = np.ascontiguousarray(q, dtype=np.int32)
        _check(self.lib, self.lib.cc_trainer_set_q(self._h, qa.ctypes.data_as(C.POINTER(C.c_int32))))

    def decode_terms(self, params: np.ndarray | None = None, which: int = 3):
        """latent_rate_estimate / mse_rgb(reconstruct_image) (decode_core.hpp:38-63)
        on the current q with `params` substituted: (rate_bits, mse); None for
        a term not requested."""
        b, m = C.c_double(np.nan), C.c_double(np.nan)
        pa = None if params is None else np.ascontiguousarray(params, dtype=np.float32)
        _check(self.lib, self.lib.cc_trainer_decode_terms(self._h, None if pa is None else _fp(pa), which,
                                                          C.byref(b), C.byref(m)))
        return (b.value if which & 1 else None), (m.value if which & 2 else None)

    def latent_mu_sigma(self, params: np.ndarray | None = None):
        """(mu, sigma) of every quantised latent as the entropy coder computes
        them (bitstream.hpp:106-141), flat layout, `params` substituted."""
        mu = np.empty(self.n_latents, np.float32)
        sg = np.empty(self.n_latents, np.float32)
        pa = None if params is None else np.ascontiguousarray(params, dtype=np.float32)
        _check(self.lib, self.lib.cc_trainer_latent_mu_sigma(self._h, None if pa is None else _fp(pa),
                                                             _fp(mu), _fp(sg)))
        return mu, sg

    def get_grads(self):
        lg = np.empty(self.n_latents, np.float32)
        pg = np.empty(self.n_params, np.float32)
        _check(self.lib, self.lib.cc_trainer_get_grads(self._h, _fp(lg), _fp(pg)))
        return lg, pg

    def get_q(self) -> np.ndarray:
        q = np.empty(self.n_latents, np.int32)
        _check(self.lib, self.lib.cc_trainer_get_q(self._h, _ip(q, C.c_int32)))
        return q

    def grid_view(self, flat: np.ndarray, gi: int) -> np.ndarray:
        g = self.grids[gi]
        return flat[g.offset:g.offset + g.count].reshape(g.rows, g.cols)

    def param_view(self, flat: np.ndarray, ti: int) -> np.ndarray:
        p = self.params[ti]
        return flat[p.offset:p.offset + p.size]


class Batch:
    """Several trainers of one image size / decoder run in lock-step by one set
    of kernel launches per stage (include/coolchic_b200_batch.h; BASELINE
    config 3).  The reference's multi-image mode is independent encodes on a
    thread pool (tools/coolcodec.cpp:150-171); each Trainer here stays a full
    detail::Trainer equivalent."""

    def __init__(self, trainers):
        self.trainers = list(trainers)
        if not self.trainers:
            raise ConfigError("empty batch")
        self.lib = self.trainers[0].lib
        arr = (C.c_void_p * len(self.trainers))(*[t._h.value for t in self.trainers])
        self._h = C.c_void_p()
        _check(self.lib, self.lib.cc_batch_create(arr, len(self.trainers), C.byref(self._h)))

    def reserve_iterations(self, n: int) -> None:
        _check(self.lib, self.lib.cc_batch_reserve_iterations(self._h, int(n)))

    def enqueue_proxy_iterations(self, lr, temp, noise_std) -> None:
        lr = np.ascontiguousarray(lr, np.float64)
        n = lr.size
        temp = np.ascontiguousarray(np.broadcast_to(temp, (n,)), np.float64)
        noise_std = np.ascontiguousarray(np.broadcast_to(noise_std, (n,)), np.float64)
        dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
        _check(self.lib, self.lib.cc_batch_enqueue_proxy_iterations(self._h, n, dp(lr), dp(temp),
                                                                    dp(noise_std)))

    def synchronize(self) -> None:
        _check(self.lib, self.lib.cc_batch_synchronize(self._h))

    def proxy_iterations(self, lr, temp, noise_std) -> np.ndarray:
        """n iterations of every image; returns costs [image, iteration]."""
        n = np.asarray(lr).size
        self.enqueue_proxy_iterations(lr, temp, noise_std)
        self.synchronize()
        out = np.empty((len(self.trainers), n), np.float64)
        rec = np.empty(4 * n, np.float64)
        for b, t in enumerate(self.trainers):
            _check(self.lib, self.lib.cc_trainer_last_records(t._h, n, rec.ctypes.data_as(C.POINTER(C.c_double))))
            out[b] = rec[0::4]
        return out

    def close(self):
        if self._h:
            self.lib.cc_batch_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def train(image: np.ndarray, enc: EncoderConfig, dcfg: DecoderConfig, lib=None,
          device: int = 0) -> TrainResult:
    """train(img, enc, dcfg) (encoder.hpp:349-413)."""
    with Trainer(image, enc, dcfg, lib=lib, device=device) as tr:
        return tr.train()

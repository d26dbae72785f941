"""B200-native Wallace maximum-entropy normal generator (arXiv 1005.2314).

Python view of the C-ABI (include/wallace_b200.h).  The reference's boundary
is the C++ class ``maxent::Generator`` (generator.hpp:98-149); ``PoolBatch``
mirrors it for a batch of independent pools (one reference Generator per
pool), with the same method names, argument meaning and error behaviour:

    reference                         here (per pool p of the batch)
    Generator(cfg)                    PoolBatch(cfg, n_pools, seeds=...)
    fill(count) / fill(span)          fill(count) -> (n_pools, count) tensor on the device
    next_pool()                       next_pool() -> (values, reserved, chi2_draw)
    step_pass()                       step_pass(n=1)
    inject_pool(span)                 inject_pool(values, pool=0)
    pool().raw / pass_count() / ...   pool(p), info(p)
    ConfigError / InvalidParameterError   ConfigError / InvalidParameterError

All compute runs in libwallace_b200.so (hand-written sm_100a kernels); torch
supplies device memory and streams only.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _capi

__all__ = ["GeneratorConfig", "PoolBatch", "ConfigError", "InvalidParameterError",
           "UnsupportedError", "CudaError", "boxmuller_consume", "baseline_consume", "BaselineStreams",
           "BaselineState", "chi2_sample", "kernel_launches", "pair_kernel_launches"]


class ConfigError(ValueError):
    """maxent::ConfigError (errors.hpp:18-21): the message names the field."""


class InvalidParameterError(ValueError):
    """maxent::InvalidParameterError (errors.hpp:12-16)."""


class UnsupportedError(NotImplementedError):
    """A reference option this B200 build does not implement."""


class CudaError(RuntimeError):
    pass


def _check(rc: int) -> None:
    if rc == _capi.WALLACE_OK:
        return
    msg = _capi.last_error()
    if rc == _capi.WALLACE_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == _capi.WALLACE_ERR_INVALID_PARAM:
        raise InvalidParameterError(msg)
    if rc == _capi.WALLACE_ERR_UNSUPPORTED:
        raise UnsupportedError(msg)
    raise CudaError(msg)


CHI2_METHODS = {"sqrt_shift": 0, "wilson_hilferty": 1, "cubic_a": 2}


@dataclass
class GeneratorConfig:
    """maxent::GeneratorConfig (generator.hpp:21-45)."""

    pool_size: int = 1024
    transform_family: int = 0  # 0 wallace4, 1 rotation
    mixing: int = 0            # 0 stride_transpose, 1 affine
    chi2_method: int = 2       # 0 sqrt_shift, 1 wilson_hilferty, 2 cubic_a
    discard_every: int = 1
    out_mean: float = 0.0
    out_sigma: float = 1.0
    seed: int = 0
    fixed_transform: bool = False
    disable_chi2: bool = False

    def to_c(self) -> _capi.wallace_config:
        return _capi.wallace_config(
            int(self.pool_size), int(self.transform_family), int(self.mixing),
            int(self.chi2_method), int(bool(self.fixed_transform)),
            int(bool(self.disable_chi2)), 0, int(self.discard_every),
            float(self.out_mean), float(self.out_sigma), int(self.seed) & (2**64 - 1))

    def validate(self) -> None:
        _check(_capi.load().wallace_validate_config(C.byref(self.to_c())))


def _torch():
    import torch  # plumbing only: device buffers and streams
    return torch


def _stream_handle(stream) -> Optional[int]:
    if stream is None:
        torch = _torch()
        return torch.cuda.current_stream().cuda_stream if torch.cuda.is_available() else None
    return int(getattr(stream, "cuda_stream", stream))


class PoolBatch:
    """n_pools independent Wallace pools resident in HBM.

    dtype: "f32" (the fp32 restatement) or "f64" (bit-exact
    reference semantics).  seeds: per-pool seeds; default cfg.seed + p.
    """

    def __init__(self, cfg: GeneratorConfig, n_pools: int = 1, seeds: Optional[Sequence[int]] = None,
                 dtype: str = "f32", stream=None, device_seed: bool = False):
        """device_seed=True seeds the pools on the device (wallace_create_ex,
        WALLACE_CREATE_DEVICE_SEED): exact xoshiro/Polar acceptance stream,
        CUDA log -- within a few ulps of the host seeding, not a parity path."""
        self.L = _capi.load()
        self.cfg = cfg
        self.n_pools = int(n_pools)
        self.dtype = dtype
        if dtype not in ("f32", "f64"):
            raise InvalidParameterError("dtype must be 'f32' or 'f64'")
        self._dt = _capi.WALLACE_F32 if dtype == "f32" else _capi.WALLACE_F64
        self.np_dtype = np.float32 if dtype == "f32" else np.float64
        self._stream = _stream_handle(stream)
        seeds_arr = None
        seeds_ptr = None
        if seeds is not None:
            seeds_arr = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
            if seeds_arr.size != self.n_pools:
                raise InvalidParameterError("seeds must have n_pools entries")
            seeds_ptr = seeds_arr.ctypes.data_as(C.POINTER(C.c_uint64))
        h = C.c_void_p()
        _check(self.L.wallace_create_ex(C.byref(cfg.to_c()), self.n_pools, seeds_ptr, self._dt,
                                        self._stream, 1 if device_seed else 0, C.byref(h)))
        self.h = h

    # -- lifecycle ---------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "h", None):
            self.L.wallace_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def torch_dtype(self):
        torch = _torch()
        return torch.float32 if self.dtype == "f32" else torch.float64

    # -- generation ----------------------------------------------------------
    def _check_out(self, out) -> None:
        if out.dim() != 2 or out.shape[0] != self.n_pools or not out.is_contiguous():
            raise InvalidParameterError("out must be a contiguous (n_pools, count) tensor")
        if out.dtype != self.torch_dtype or not out.is_cuda:
            raise InvalidParameterError("out must be a CUDA tensor of the batch dtype")
        if out.shape[1] < 1:
            raise InvalidParameterError("fill: count must be >= 1")

    def fill_into(self, out) -> None:
        """Generator::fill(span) into a device tensor of shape (n_pools, count).
        Asynchronous: chi2_sample's error (a non-finite reserved value) is
        raised by the next synchronising call (synchronize(), fill(), ...)."""
        self._check_out(out)
        _check(self.L.wallace_fill(self.h, C.c_void_p(out.data_ptr()), out.shape[1]))

    def synchronize(self) -> None:
        """Wait for the batch's queued work; raises InvalidParameterError
        where the reference's fill/next_pool would have thrown (chi2.cpp:29-31)."""
        _check(self.L.wallace_synchronize(self.h))

    def fill(self, count: int):
        """Generator::fill(count) for every pool -> (n_pools, count) CUDA tensor
        (synchronous: raises like the reference's fill)."""
        if count < 1:
            raise InvalidParameterError("fill: count must be >= 1")
        torch = _torch()
        out = torch.empty((self.n_pools, count), dtype=self.torch_dtype, device="cuda")
        self.fill_into(out)
        self.synchronize()
        return out

    def fill_host(self, count: int, out: Optional[np.ndarray] = None) -> np.ndarray:
        """fill(count) into host memory (the end-to-end call)."""
        if out is None:
            out = np.empty((self.n_pools, count), dtype=self.np_dtype)
        if out.shape != (self.n_pools, count) or out.dtype != self.np_dtype:
            raise InvalidParameterError("out has the wrong shape or dtype")
        _check(self.L.wallace_fill_host(self.h, out.ctypes.data_as(C.c_void_p), count))
        return out

    def fill_host_ptr(self, ptr: int, count: int) -> None:
        _check(self.L.wallace_fill_host(self.h, C.c_void_p(ptr), count))

    def snapshot(self) -> None:
        _check(self.L.wallace_snapshot(self.h))

    def fill_from_snapshot_into(self, out) -> None:
        self._check_out(out)
        _check(self.L.wallace_fill_from_snapshot(self.h, C.c_void_p(out.data_ptr()), out.shape[1]))

    def next_pool(self):
        """Generator::next_pool(): (values (n_pools, N-1) CUDA tensor, reserved[n], chi2_draw[n])."""
        torch = _torch()
        vals = torch.empty((self.n_pools, self.cfg.pool_size - 1), dtype=self.torch_dtype,
                           device="cuda")
        res = np.empty(self.n_pools, dtype=np.float64)
        chi = np.empty(self.n_pools, dtype=np.float64)
        _check(self.L.wallace_next_pool(self.h, C.c_void_p(vals.data_ptr()),
                                        res.ctypes.data_as(C.POINTER(C.c_double)),
                                        chi.ctypes.data_as(C.POINTER(C.c_double))))
        return vals, res, chi

    def step_pass(self, n: int = 1) -> None:
        _check(self.L.wallace_step_pass(self.h, n))

    def inject_pool(self, values, pool: int = 0) -> None:
        v = np.ascontiguousarray(np.asarray(values, dtype=np.float64))
        _check(self.L.wallace_inject_pool(self.h, pool, v.ctypes.data_as(C.POINTER(C.c_double)),
                                          v.size))

    def pool(self, p: int = 0) -> np.ndarray:
        raw = np.empty(self.cfg.pool_size, dtype=np.float64)
        _check(self.L.wallace_get_pool(self.h, p, raw.ctypes.data_as(C.POINTER(C.c_double)),
                                       raw.size))
        return raw

    def info(self, p: int = 0) -> dict:
        inf = _capi.wallace_pool_info()
        _check(self.L.wallace_get_pool_info(self.h, p, C.byref(inf)))
        return {k: getattr(inf, k) for k, _ in _capi.wallace_pool_info._fields_}

    def pass_count(self, p: int = 0) -> int:
        return self.info(p)["pass_count"]

    def uniform_draws(self, p: int = 0) -> int:
        return self.info(p)["uniform_draws"]

    def chi2_clamp_count(self, p: int = 0) -> int:
        return self.info(p)["chi2_clamp_count"]

    # -- checkpoint ------------------------------------------------------------
    def save_state(self) -> bytes:
        n = self.L.wallace_state_bytes(self.h)
        buf = (C.c_ubyte * n)()
        _check(self.L.wallace_save_state(self.h, C.cast(buf, C.c_void_p), n))
        return bytes(buf)

    def load_state(self, image: bytes) -> None:
        buf = (C.c_ubyte * len(image)).from_buffer_copy(image)
        _check(self.L.wallace_load_state(self.h, C.cast(buf, C.c_void_p), len(image)))

    # -- fused consumer (config 5) ---------------------------------------------
    def consume(self, count: int):
        sums = np.zeros(4, dtype=np.float64)
        hist = np.zeros(258, dtype=np.uint64)
        _check(self.L.wallace_consume(self.h, count, sums.ctypes.data_as(C.POINTER(C.c_double)),
                                      hist.ctypes.data_as(C.POINTER(C.c_uint64))))
        return sums, hist

    def consume_from_snapshot(self, count: int):
        sums = np.zeros(4, dtype=np.float64)
        hist = np.zeros(258, dtype=np.uint64)
        _check(self.L.wallace_consume_from_snapshot(
            self.h, count, sums.ctypes.data_as(C.POINTER(C.c_double)),
            hist.ctypes.data_as(C.POINTER(C.c_uint64))))
        return sums, hist

    def set_kernel_mode(self, mode: str) -> None:
        """'auto', 'throughput' or 'latency' (identical results)."""
        _check(self.L.wallace_set_kernel_mode(self.h, {"auto": 0, "throughput": 1, "latency": 2}[mode]))

    def set_stream(self, stream) -> None:
        self._stream = _stream_handle(stream)
        _check(self.L.wallace_set_stream(self.h, self._stream))


    # ---- stream wire format (cmd_gen.cpp:39-57) --------------------------
    FORMATS = {"f64le": 0, "text": 1, "f32le": 2}

    def write_stream(self, out, count: int, fmt: str = "f64le") -> None:
        """Write `count` further values of every pool (pool-major) to `out`
        (a path, an open binary file or a file descriptor) in the reference's
        gen formats: f64le (8-byte LE doubles), text ("%.17g" lines, one
        pool), f32le (fp32 handles)."""
        import os
        if isinstance(out, int):
            fd, close = out, False
        elif hasattr(out, "fileno"):
            out.flush()
            fd, close = out.fileno(), False
        else:
            fd, close = os.open(str(out), os.O_WRONLY | os.O_CREAT | os.O_TRUNC, 0o644), True
        try:
            _check(self.L.wallace_write_stream(self.h, int(count), self.FORMATS[fmt], fd))
        finally:
            if close:
                os.close(fd)

    # ---- defect suite (stats.cpp), GPU-resident -------------------------
    def cross_pool_probes(self, passes: int, probes=None) -> np.ndarray:
        """cross_pool_correlation on every pool (stats.cpp:310-338): advance
        `passes` step_pass() and return the ProbeAccumulator sums
        [n_pools, n_probes, 6] = (sx, sxx, sy, syy, sxy, sxy2) of
        x = pool_before[in_j], y = pool_after[out_i].  probes: (out_i, in_j)
        pairs, default stats.default_probes(N)."""
        from . import stats
        probes = stats.default_probes(self.cfg.pool_size) if probes is None else list(probes)
        k = len(probes)
        oi = (C.c_uint64 * k)(*[int(p[0]) for p in probes])
        ij = (C.c_uint64 * k)(*[int(p[1]) for p in probes])
        acc = np.zeros((self.n_pools, k, 6), dtype=np.float64)
        _check(self.L.wallace_cross_pool_probes(self.h, int(passes), k, oi, ij,
                                                acc.ctypes.data_as(C.POINTER(C.c_double))))
        return acc

    def pool_defect_stats(self, emissions: int, threshold: float = 4.0):
        """pool_sum_squares_test / rare_event_adjacency on every pool
        (stats.cpp:340-369, 424-447): `emissions` next_pool() calls; returns
        (totals [n_pools, emissions] = reserved^2 + sum v^2, marks
        [n_pools, emissions] = any |v| > threshold).  Needs a standardized
        config (out_mean 0, out_sigma 1)."""
        totals = np.zeros((self.n_pools, int(emissions)), dtype=np.float64)
        marks = np.zeros((self.n_pools, int(emissions)), dtype=np.uint8)
        _check(self.L.wallace_pool_defect_stats(self.h, int(emissions), float(threshold),
                                                totals.ctypes.data_as(C.POINTER(C.c_double)),
                                                marks.ctypes.data_as(C.POINTER(C.c_uint8))))
        return totals, marks.astype(bool)

def pass_plan(wallace_variant: int = 0, t_index=(0, 0), negate=(0, 0), offset=(0, 0)):
    """maxent::PassPlan (generator.hpp:50-55); the default is PassPlan{}."""
    p = _capi.wallace_pass_plan()
    p.wallace_variant = int(wallace_variant)
    p.t_index[0], p.t_index[1] = (int(t) for t in t_index)
    p.negate[0], p.negate[1] = (int(bool(g)) for g in negate)
    p.offset[0], p.offset[1] = (int(o) for o in offset)
    return p


def run_pass(cfg: GeneratorConfig, plan, values) -> np.ndarray:
    """maxent::run_pass (generator.cpp:259-271): one pass with an explicit
    plan over one fp64 pool, on the device."""
    v = np.ascontiguousarray(values, dtype=np.float64)
    if v.size != cfg.pool_size:
        raise InvalidParameterError("run_pass: buffers must match pool_size")
    out = np.empty_like(v)
    dp = C.POINTER(C.c_double)
    _check(_capi.load().wallace_run_pass(C.byref(cfg.to_c()), C.byref(plan), v.ctypes.data_as(dp),
                                         out.ctypes.data_as(dp)))
    return out


def pass_coefficient(cfg: GeneratorConfig, plan, out_i: int, in_j: int) -> float:
    """maxent::pass_coefficient (generator.cpp:273-284)."""
    r = C.c_double()
    _check(_capi.load().wallace_pass_coefficient(C.byref(cfg.to_c()), C.byref(plan), int(out_i), int(in_j),
                                                 C.byref(r)))
    return r.value


def cross_pool_fixed_sums(cfg: GeneratorConfig, pairs: int, probes) -> np.ndarray:
    """cross_pool_correlation's fixed-transform mode (stats.cpp:284-299):
    ProbeAccumulator sums [n_probes, 6] over `pairs` fresh Polar pools, one
    pinned pass each (on the device)."""
    k = len(probes)
    oi = (C.c_uint64 * k)(*[int(p[0]) for p in probes])
    ij = (C.c_uint64 * k)(*[int(p[1]) for p in probes])
    acc = np.zeros((k, 6), dtype=np.float64)
    _check(_capi.load().wallace_cross_pool_fixed(C.byref(cfg.to_c()), int(pairs), k, oi, ij,
                                                 acc.ctypes.data_as(C.POINTER(C.c_double))))
    return acc


BASELINE_METHODS = {"polar": _capi.WALLACE_BASELINE_POLAR, "boxmuller": _capi.WALLACE_BASELINE_BOXMULLER}


def baseline_consume(method: str, n_streams: int, count: int, seed_base: int = 1, seeds=None, stream=None):
    """Config-5 comparator: BaselineState(seed) streams of polar_next /
    boxmuller_next (baselines.cpp:51-92) generated on the device in fp64 and
    consumed in-kernel like PoolBatch.consume.  Returns (sums, hist,
    kernel device ms)."""
    L = _capi.load()
    sums = np.zeros(4, dtype=np.float64)
    hist = np.zeros(258, dtype=np.uint64)
    ms = C.c_double()
    sp = None
    if seeds is not None:
        seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
        sp = seeds.ctypes.data_as(C.POINTER(C.c_uint64))
    _check(L.wallace_baseline_consume(BASELINE_METHODS[method], sp, seed_base, n_streams, count,
                                      _stream_handle(stream), sums.ctypes.data_as(C.POINTER(C.c_double)),
                                      hist.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(ms)))
    return sums, hist, ms.value


def boxmuller_consume(n_streams: int, count: int, seed_base: int = 1, seeds=None, stream=None):
    """Box-Muller comparator on UniformState(seed) streams (baselines.cpp:80-92)."""
    sums, hist, _ = baseline_consume("boxmuller", n_streams, count, seed_base, seeds, stream)
    return sums, hist


class BaselineStreams:
    """n independent BaselineState streams (baselines.hpp:49-55) of polar_next
    or boxmuller_next, generated on the device (fp64): ``fill(count)``
    continues every stream and returns a (n_streams, count) CUDA tensor.
    The uniform words and draw counts are exact; the values are within a few
    ulps of the reference's glibc transcendentals."""

    def __init__(self, method: str, seeds):
        self.method = BASELINE_METHODS[method]
        seeds = [int(s) for s in seeds]
        self.n = len(seeds)
        self.states = (_capi.wallace_baseline_state * self.n)()
        L = _capi.load()
        for k, s in enumerate(seeds):
            L.wallace_baseline_seed(s, C.byref(self.states[k]))

    def fill(self, count: int, stream=None):
        torch = _torch()
        out = torch.empty((self.n, int(count)), dtype=torch.float64, device="cuda")
        _check(_capi.load().wallace_baseline_fill(self.method, self.states, self.n, int(count),
                                                  C.c_void_p(out.data_ptr()), _stream_handle(stream)))
        return out

    def draws(self, k: int = 0) -> int:
        return int(self.states[k].uniform.draws)


# ---- host functions of the reference's L1a layer (bit-identical, same libm) ----
class BaselineState:
    """maxent::BaselineState with polar_next / boxmuller_next (baselines.cpp:51-92)."""

    def __init__(self, seed: int):
        self.c = _capi.wallace_baseline_state()
        _capi.load().wallace_baseline_seed(int(seed) & (2**64 - 1), C.byref(self.c))

    def polar_next(self) -> float:
        return _capi.load().wallace_polar_next(C.byref(self.c))

    def boxmuller_next(self) -> float:
        return _capi.load().wallace_boxmuller_next(C.byref(self.c))

    @property
    def draws(self) -> int:
        return int(self.c.uniform.draws)


def chi2_sample(x: float, nu: int, method: int = 2):
    """chi2_sample(x, Chi2Params::for_nu(nu), method) -> (S, clamped) (chi2.cpp:19-59)."""
    L = _capi.load()
    a = C.c_double()
    _check(L.wallace_chi2_params(int(nu), C.byref(a)))
    out, cl = C.c_double(), C.c_int32()
    _check(L.wallace_chi2_sample(float(x), int(nu), a.value, int(method), C.byref(cl), C.byref(out)))
    return out.value, bool(cl.value)


def kernel_launches() -> int:
    return int(_capi.load().wallace_kernel_launches())


def pair_kernel_launches() -> int:
    """Launches of pair_kernel (csrc/pool_pair.cu) among kernel_launches()."""
    return int(_capi.load().wallace_pair_kernel_launches())


def moment_reports(sums, n: int):
    """Moments and 5-SE reports from raw power sums (stats.cpp:98-109 rule).

    Returns dict name -> (statistic, expected, se, z, pass)."""
    s1, s2, s3, s4 = (float(x) for x in sums)
    mean = s1 / n
    m2 = s2 / n - mean * mean
    m3 = s3 / n - 3 * mean * s2 / n + 2 * mean ** 3
    m4 = s4 / n - 4 * mean * s3 / n + 6 * mean * mean * s2 / n - 3 * mean ** 4
    var = m2 * n / (n - 1)
    skew = m3 / m2 ** 1.5
    kurt = m4 / (m2 * m2) - 3.0
    out = {}
    for name, stat, exp, se in (("mean", mean, 0.0, (1.0 / n) ** 0.5),
                                ("variance", var, 1.0, (2.0 / n) ** 0.5),
                                ("skewness", skew, 0.0, (6.0 / n) ** 0.5),
                                ("excess_kurtosis", kurt, 0.0, (24.0 / n) ** 0.5)):
        z = (stat - exp) / se
        out[name] = (stat, exp, se, z, abs(z) <= 5.0)
    return out

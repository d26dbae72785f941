"""TEST INFRASTRUCTURE ONLY — ctypes loaders for the CPU oracle.

* ``Oracle``  — the C restatement (oracle/libwallace_oracle.so), f64 reference
  semantics and the f32 restatement.
* ``RefLib``  — the unmodified reference library compiled from
  /root/reference sources (oracle/_ref/libmaxent_ref.so, see oracle/Makefile).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libwallace_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmaxent_ref.so")

u64 = C.c_uint64
WO_ERR_CHI2_NONFINITE = -20  # wallace_oracle.h: chi2_sample threw (chi2.cpp:29-31)
i32 = C.c_int32
f64 = C.c_double
vp = C.c_void_p
P = C.POINTER


class WoConfig(C.Structure):
    _fields_ = [
        ("pool_size", u64),
        ("transform_family", i32),
        ("mixing", i32),
        ("chi2_method", i32),
        ("fixed_transform", i32),
        ("disable_chi2", i32),
        ("pad_", i32),
        ("discard_every", u64),
        ("out_mean", f64),
        ("out_sigma", f64),
        ("seed", u64),
    ]


@dataclass
class Cfg:
    """Mirror of maxent::GeneratorConfig (generator.hpp:21-45)."""

    pool_size: int = 1024
    chi2_method: int = 2  # 0 sqrt_shift, 1 wilson_hilferty, 2 cubic_a
    discard_every: int = 1
    out_mean: float = 0.0
    out_sigma: float = 1.0
    seed: int = 0
    fixed_transform: bool = False
    disable_chi2: bool = False
    transform_family: int = 0  # 0 wallace4, 1 rotation
    mixing: int = 0  # 0 stride_transpose, 1 affine

    def wo(self) -> WoConfig:
        return WoConfig(self.pool_size, self.transform_family, self.mixing, self.chi2_method,
                        int(self.fixed_transform),
                        int(self.disable_chi2), 0, self.discard_every, self.out_mean,
                        self.out_sigma, self.seed)


def build(ref: bool = False) -> None:
    targets = ["all"] + (["ref"] if ref else [])
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


_oracle = None
_ref = None


def oracle_lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.wo_create.argtypes = [P(WoConfig), C.c_int, P(vp)]
        L.wo_destroy.argtypes = [vp]
        L.wo_fill.argtypes = [vp, vp, u64]
        L.wo_next_pool.argtypes = [vp, vp, P(f64), P(f64)]
        L.wo_step_pass.argtypes = [vp]
        L.wo_inject_pool.argtypes = [vp, P(f64), u64]
        L.wo_get_pool.argtypes = [vp, P(f64)]
        L.wo_get_stats.argtypes = [vp, P(u64), P(u64), P(u64), P(f64), P(f64), P(u64)]
        L.wo_peek_plan.argtypes = [vp, P(C.c_int), P(u64)]
        L.wo_uniform_seed.argtypes = [u64, P(u64)]
        L.wo_uniform_bits.argtypes = [P(u64)]
        L.wo_uniform_bits.restype = u64
        L.wo_uniform_next.argtypes = [P(u64)]
        L.wo_uniform_next.restype = f64
        L.wo_default_stride.argtypes = [u64]
        L.wo_default_stride.restype = u64
        L.wo_wallace_variant.argtypes = [C.c_int, P(C.c_int), P(f64)]
        L.wo_default_multipliers.argtypes = [u64, P(u64), P(u64)]
        L.wo_default_multipliers.restype = None
        L.wo_rotation_t.argtypes = [C.c_int]
        L.wo_rotation_t.restype = f64
        L.wo_rotation_from_t.argtypes = [f64, P(f64), P(f64)]
        L.wo_rotation_from_t.restype = None
        L.wo_compute_a.argtypes = [u64]
        L.wo_compute_a.restype = f64
        L.wo_chi2_sample.argtypes = [f64, u64, f64, C.c_int, P(C.c_int)]
        L.wo_chi2_sample.restype = f64
        L.wo_moments.argtypes = [P(f64), u64, P(f64), P(f64), P(f64), P(f64)]
        L.wo_consume_pools.argtypes = [P(WoConfig), C.c_int, P(u64), u64, u64, C.c_int,
                                       P(f64), P(u64)]
        _oracle = L
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        L = C.CDLL(REF_SO)
        L.ref_create.argtypes = [u64, C.c_int, u64, f64, f64, u64, C.c_int, C.c_int]
        L.ref_create.restype = vp
        L.ref_create_ex.argtypes = [u64, C.c_int, u64, f64, f64, u64, C.c_int, C.c_int, C.c_int,
                                    C.c_int]
        L.ref_create_ex.restype = vp
        L.ref_rotation_table.argtypes = [P(f64), P(f64), P(f64)]
        L.ref_rotation_table.restype = None
        L.ref_default_multipliers.argtypes = [u64, P(u64), P(u64)]
        L.ref_default_multipliers.restype = None
        L.ref_decode_pass_plan_ex.argtypes = [u64, C.c_int, C.c_int, u64, u64, P(C.c_int32),
                                              P(u64)]
        L.ref_decode_pass_plan_ex.restype = None
        L.ref_cross_pool_correlation.argtypes = [vp, u64, C.c_uint32, P(u64), P(u64), P(f64)]
        L.ref_cross_pool_correlation.restype = C.c_int
        L.ref_pool_sum_squares.argtypes = [u64, C.c_int, u64, u64, C.c_int, C.c_int, C.c_int, u64,
                                           P(f64)]
        L.ref_pool_sum_squares.restype = C.c_int
        L.ref_rare_event_adjacency.argtypes = [u64, C.c_int, u64, u64, C.c_int, u64, f64, P(f64)]
        L.ref_rare_event_adjacency.restype = C.c_int
        L.ref_run_pass.argtypes = [u64, C.c_int, C.c_int, P(C.c_int32), P(u64), P(f64), P(f64)]
        L.ref_run_pass.restype = C.c_int
        L.ref_pass_coefficient.argtypes = [u64, C.c_int, C.c_int, P(C.c_int32), P(u64), u64, u64]
        L.ref_pass_coefficient.restype = f64
        L.ref_cross_pool_fixed.argtypes = [u64, C.c_int, C.c_int, u64, u64, C.c_uint32, P(u64), P(u64), C.c_int,
                                           P(f64)]
        L.ref_cross_pool_fixed.restype = C.c_int
        L.ref_last_error.restype = C.c_char_p
        L.ref_destroy.argtypes = [vp]
        L.ref_fill.argtypes = [vp, P(f64), u64]
        L.ref_next_normal.argtypes = [vp]
        L.ref_next_normal.restype = f64
        L.ref_next_normal_ex.argtypes = [vp, P(C.c_int)]
        L.ref_next_normal_ex.restype = f64
        L.ref_next_pool.argtypes = [vp, P(f64), P(f64), P(f64)]
        L.ref_step_pass.argtypes = [vp]
        L.ref_inject_pool.argtypes = [vp, P(f64), u64]
        L.ref_get_pool.argtypes = [vp, P(f64)]
        L.ref_get_stats.argtypes = [vp, P(u64), P(u64), P(u64), P(f64), P(f64)]
        L.ref_uniform_bits.argtypes = [u64, u64, P(u64)]
        L.ref_default_stride.argtypes = [u64]
        L.ref_default_stride.restype = u64
        L.ref_compute_a.argtypes = [u64]
        L.ref_compute_a.restype = f64
        L.ref_chi2_sample.argtypes = [f64, u64, C.c_int, P(C.c_int)]
        L.ref_chi2_sample.restype = f64
        L.ref_wallace_variant.argtypes = [C.c_int, P(C.c_int), P(f64), P(f64)]
        L.ref_decode_pass_plan.argtypes = [u64, u64, u64, P(u64)]
        L.ref_polar.argtypes = [u64, u64, P(f64)]
        L.ref_boxmuller.argtypes = [u64, u64, P(f64)]
        L.ref_moments.argtypes = [P(f64), u64, P(f64)]
        L.ref_run_job.argtypes = [u64, C.c_int, u64, C.c_int, u64, u64, u64, C.c_int,
                                  P(f64), P(f64)]
        L.ref_run_job.restype = f64
        L.ref_run_job_ex.argtypes = [u64, C.c_int, u64, C.c_int, C.c_int, C.c_int, u64, u64, u64,
                                     C.c_int, P(f64), P(f64)]
        L.ref_run_job_ex.restype = f64
        _ref = L
    return _ref


def _dp(a: np.ndarray):
    return a.ctypes.data_as(P(f64))


class OracleGen:
    """CPU oracle generator; dtype 'f64' (reference semantics) or 'f32'."""

    def __init__(self, cfg: Cfg, dtype: str = "f64"):
        self.L = oracle_lib()
        self.cfg = cfg
        self.dtype = dtype
        self.np_dtype = np.float64 if dtype == "f64" else np.float32
        h = vp()
        rc = self.L.wo_create(C.byref(cfg.wo()), 1 if dtype == "f64" else 0, C.byref(h))
        if rc != 0:
            raise ValueError(f"oracle config rejected ({rc})")
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.L.wo_destroy(self.h)
            self.h = None

    def fill(self, count: int) -> np.ndarray:
        out = np.empty(count, dtype=self.np_dtype)
        rc = self.L.wo_fill(self.h, out.ctypes.data_as(vp), count)
        if rc == WO_ERR_CHI2_NONFINITE:
            raise ValueError("chi2_sample: x must be finite")
        if rc != 0:
            raise ValueError("fill: count must be >= 1")
        return out

    def next_pool(self):
        vals = np.empty(self.cfg.pool_size - 1, dtype=self.np_dtype)
        res, chi = f64(), f64()
        if self.L.wo_next_pool(self.h, vals.ctypes.data_as(vp), C.byref(res), C.byref(chi)) != 0:
            raise ValueError("chi2_sample: x must be finite")
        return vals, res.value, chi.value

    def step_pass(self):
        self.L.wo_step_pass(self.h)

    def inject_pool(self, values):
        v = np.ascontiguousarray(values, dtype=np.float64)
        if self.L.wo_inject_pool(self.h, _dp(v), v.size) != 0:
            raise ValueError("inject_pool: size must equal pool_size")

    def pool(self) -> np.ndarray:
        raw = np.empty(self.cfg.pool_size, dtype=np.float64)
        self.L.wo_get_pool(self.h, _dp(raw))
        return raw

    def stats(self) -> dict:
        pc, dr, cl, cur = u64(), u64(), u64(), u64()
        ss, rp = f64(), f64()
        self.L.wo_get_stats(self.h, C.byref(pc), C.byref(dr), C.byref(cl), C.byref(ss),
                            C.byref(rp), C.byref(cur))
        return dict(pass_count=pc.value, uniform_draws=dr.value, chi2_clamp_count=cl.value,
                    sum_sq=ss.value, reserved_prev=rp.value, buffered=cur.value)


class RefGen:
    """The unmodified reference maxent::Generator (fp64 only)."""

    def __init__(self, cfg: Cfg):
        self.L = ref_lib()
        self.cfg = cfg
        h = self.L.ref_create_ex(cfg.pool_size, cfg.chi2_method, cfg.discard_every, cfg.out_mean,
                                 cfg.out_sigma, cfg.seed, int(cfg.fixed_transform),
                                 int(cfg.disable_chi2), cfg.transform_family, cfg.mixing)
        if not h:
            raise ValueError(self.L.ref_last_error().decode())
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_destroy(self.h)
            self.h = None

    def fill(self, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.float64)
        if self.L.ref_fill(self.h, _dp(out), count) != 0:
            raise ValueError(self.L.ref_last_error().decode())
        return out

    def next_normal(self) -> float:
        err = C.c_int()
        v = self.L.ref_next_normal_ex(self.h, C.byref(err))
        if err.value:
            raise ValueError(self.L.ref_last_error().decode())
        return v

    def next_pool(self):
        vals = np.empty(self.cfg.pool_size - 1, dtype=np.float64)
        res, chi = f64(), f64()
        if self.L.ref_next_pool(self.h, _dp(vals), C.byref(res), C.byref(chi)) < 0:
            raise ValueError(self.L.ref_last_error().decode())
        return vals, res.value, chi.value

    def step_pass(self):
        self.L.ref_step_pass(self.h)

    def inject_pool(self, values):
        v = np.ascontiguousarray(values, dtype=np.float64)
        if self.L.ref_inject_pool(self.h, _dp(v), v.size) != 0:
            raise ValueError(self.L.ref_last_error().decode())

    def pool(self) -> np.ndarray:
        raw = np.empty(self.cfg.pool_size, dtype=np.float64)
        self.L.ref_get_pool(self.h, _dp(raw))
        return raw

    def stats(self) -> dict:
        pc, dr, cl = u64(), u64(), u64()
        ss, rp = f64(), f64()
        self.L.ref_get_stats(self.h, C.byref(pc), C.byref(dr), C.byref(cl), C.byref(ss),
                             C.byref(rp))
        return dict(pass_count=pc.value, uniform_draws=dr.value, chi2_clamp_count=cl.value,
                    sum_sq=ss.value, reserved_prev=rp.value)


def uniform_words(seed: int, n: int) -> np.ndarray:
    L = oracle_lib()
    s = (u64 * 4)()
    L.wo_uniform_seed(seed, s)
    return np.array([L.wo_uniform_bits(s) for _ in range(n)], dtype=np.uint64)


def consume_pools(cfg: Cfg, dtype: str, seeds, count_per_pool: int, threads: int = 0):
    """Config-5 consumer oracle: (sums[4], hist[258]) with hist[0]=under,
    hist[1..256]=bins, hist[257]=over."""
    L = oracle_lib()
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    sums = np.zeros(4, dtype=np.float64)
    hist = np.zeros(258, dtype=np.uint64)
    threads = threads or os.cpu_count() or 1
    rc = L.wo_consume_pools(C.byref(cfg.wo()), 1 if dtype == "f64" else 0,
                            seeds.ctypes.data_as(P(u64)), seeds.size, count_per_pool, threads,
                            _dp(sums), hist.ctypes.data_as(P(u64)))
    if rc != 0:
        raise ValueError(f"consume_pools rejected config ({rc})")
    return sums, hist

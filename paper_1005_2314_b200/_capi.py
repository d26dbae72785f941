"""ctypes binding of include/wallace_b200.h (the C-ABI of libwallace_b200.so).

This module only declares symbols; it performs no computation itself.  It
fails loudly when the native library is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WALLACE_B200_LIB") or os.path.join(PKG_DIR, "libwallace_b200.so")

u64 = C.c_uint64
i32 = C.c_int32
f64 = C.c_double
vp = C.c_void_p
P = C.POINTER

WALLACE_OK = 0
WALLACE_ERR_CONFIG = 1
WALLACE_ERR_INVALID_PARAM = 2
WALLACE_ERR_CUDA = 3
WALLACE_ERR_UNSUPPORTED = 4

WALLACE_F32 = 0
WALLACE_F64 = 1


class wallace_config(C.Structure):
    _fields_ = [
        ("pool_size", u64),
        ("transform_family", i32),
        ("mixing", i32),
        ("chi2_method", i32),
        ("fixed_transform", i32),
        ("disable_chi2", i32),
        ("reserved_", i32),
        ("discard_every", u64),
        ("out_mean", f64),
        ("out_sigma", f64),
        ("seed", u64),
    ]


class wallace_pass_plan(C.Structure):
    """maxent::PassPlan (generator.hpp:50-55)."""
    _fields_ = [
        ("wallace_variant", i32),
        ("t_index", i32 * 2),
        ("negate", i32 * 2),
        ("reserved_", i32),
        ("offset", u64 * 2),
    ]


class wallace_uniform_state(C.Structure):
    """maxent::UniformState (baselines.hpp:27-33)."""
    _fields_ = [("s", u64 * 4), ("draws", u64)]


class wallace_baseline_state(C.Structure):
    """maxent::BaselineState (baselines.hpp:49-55)."""
    _fields_ = [("uniform", wallace_uniform_state), ("has_cached", i32), ("reserved_", i32),
                ("cached", f64)]


WALLACE_BASELINE_POLAR = 0
WALLACE_BASELINE_BOXMULLER = 1


class wallace_pool_info(C.Structure):
    _fields_ = [
        ("pass_count", u64),
        ("uniform_draws", u64),
        ("chi2_clamp_count", u64),
        ("sum_sq", f64),
        ("reserved_prev", f64),
        ("last_chi2", f64),
        ("buffered", u64),
        ("seed", u64),
    ]


# (name, restype, argtypes) — every symbol declared in include/wallace_b200.h
SYMBOLS = [
    ("wallace_create", i32, [P(wallace_config), u64, P(u64), i32, vp, P(vp)]),
    ("wallace_destroy", i32, [vp]),
    ("wallace_fill", i32, [vp, vp, u64]),
    ("wallace_fill_host", i32, [vp, vp, u64]),
    ("wallace_next_pool", i32, [vp, vp, P(f64), P(f64)]),
    ("wallace_next_pool_host", i32, [vp, vp, P(f64), P(f64)]),
    ("wallace_step_pass", i32, [vp, u64]),
    ("wallace_inject_pool", i32, [vp, u64, P(f64), u64]),
    ("wallace_get_pool", i32, [vp, u64, P(f64), u64]),
    ("wallace_get_pool_info", i32, [vp, u64, P(wallace_pool_info)]),
    ("wallace_state_bytes", u64, [vp]),
    ("wallace_save_state", i32, [vp, vp, u64]),
    ("wallace_load_state", i32, [vp, vp, u64]),
    ("wallace_snapshot", i32, [vp]),
    ("wallace_fill_from_snapshot", i32, [vp, vp, u64]),
    ("wallace_restore_snapshot", i32, [vp]),
    ("wallace_snapshot_ex", i32, [vp, i32]),
    ("wallace_restore_snapshot_ex", i32, [vp, i32]),
    ("wallace_fill_host_async", i32, [vp, vp, u64]),
    ("wallace_host_alloc", i32, [u64, P(vp)]),
    ("wallace_host_free", None, [vp]),
    ("wallace_discard", i32, [vp, u64]),
    ("wallace_consume", i32, [vp, u64, P(f64), P(u64)]),
    ("wallace_consume_from_snapshot", i32, [vp, u64, P(f64), P(u64)]),
    ("wallace_boxmuller_consume", i32, [P(u64), u64, u64, u64, vp, P(f64), P(u64)]),
    ("wallace_profile_begin", i32, [vp]),
    ("wallace_profile_end", i32, [vp, P(f64), P(u64), P(f64), P(u64)]),
    ("wallace_set_kernel_mode", i32, [vp, i32]),
    ("wallace_set_stream", i32, [vp, vp]),
    ("wallace_synchronize", i32, [vp]),
    ("wallace_kernel_launches", u64, []),
    ("wallace_pair_kernel_launches", u64, []),
    ("wallace_last_error", C.c_char_p, []),
    ("wallace_validate_config", i32, [P(wallace_config)]),
    ("wallace_host_seed_pool", i32, [P(wallace_config), u64, P(f64), P(f64), P(f64), P(u64), P(u64)]),
    ("wallace_default_stride", u64, [u64]),
    ("wallace_decode_pass_plan", i32, [u64, u64, u64, P(u64)]),
    ("wallace_decode_pass_plan_ex", i32, [P(wallace_config), u64, u64, P(wallace_pass_plan)]),
    ("wallace_rotation_table", None, [P(C.c_double), P(C.c_double), P(C.c_double)]),
    ("wallace_cross_pool_probes", i32, [vp, u64, C.c_uint32, P(u64), P(u64), P(C.c_double)]),
    ("wallace_write_stream", i32, [vp, u64, i32, i32]),
    ("wallace_run_pass", i32, [P(wallace_config), P(wallace_pass_plan), P(C.c_double), P(C.c_double)]),
    ("wallace_pass_coefficient", i32, [P(wallace_config), P(wallace_pass_plan), u64, u64, P(C.c_double)]),
    ("wallace_default_multipliers", None, [u64, P(u64), P(u64)]),
    ("wallace_cross_pool_fixed", i32, [P(wallace_config), u64, C.c_uint32, P(u64), P(u64), P(C.c_double)]),
    ("wallace_create_ex", i32, [P(wallace_config), u64, P(u64), i32, vp, C.c_uint32, P(vp)]),
    ("wallace_pool_defect_stats", i32, [vp, u64, C.c_double, P(C.c_double), P(C.c_uint8)]),
    ("wallace_splitmix64", u64, [P(u64)]),
    ("wallace_uniform_seed", None, [u64, P(wallace_uniform_state)]),
    ("wallace_uniform_bits", u64, [P(wallace_uniform_state)]),
    ("wallace_uniform_next", f64, [P(wallace_uniform_state)]),
    ("wallace_baseline_seed", None, [u64, P(wallace_baseline_state)]),
    ("wallace_polar_next", f64, [P(wallace_baseline_state)]),
    ("wallace_boxmuller_pair", i32, [f64, f64, P(f64), P(f64)]),
    ("wallace_boxmuller_next", f64, [P(wallace_baseline_state)]),
    ("wallace_exact_chi2_oracle", i32, [u64, P(wallace_baseline_state), P(f64)]),
    ("wallace_compute_a", i32, [u64, P(f64)]),
    ("wallace_chi2_params", i32, [u64, P(f64)]),
    ("wallace_chi2_sample", i32, [f64, u64, f64, i32, P(i32), P(f64)]),
    ("wallace_variant", i32, [i32, P(f64), P(C.c_uint8), P(f64)]),
    ("wallace_rotation_from_t", i32, [f64, P(f64), P(f64)]),
    ("wallace_baseline_fill", i32, [i32, P(wallace_baseline_state), u64, u64, vp, vp]),
    ("wallace_baseline_consume", i32, [i32, P(u64), u64, u64, u64, vp, P(f64), P(u64), P(f64)]),
]

_lib = None


def load() -> C.CDLL:
    """Load libwallace_b200.so.  Raises if it was not built — no fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SYMBOLS:
            try:
                fn = getattr(L, name)
            except AttributeError:  # an older build (tests check the full set)
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    msg = load().wallace_last_error()
    return msg.decode() if msg else ""

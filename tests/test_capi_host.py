"""Host-side checks of the C-ABI library (no GPU needed): it loads, exports
every symbol include/wallace_b200.h declares, validates configs like
GeneratorConfig::validate (generator.cpp:221-236), and seeds pools exactly
like the reference constructor (generator.cpp:309-327)."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

import paper_1005_2314_b200 as pb
from paper_1005_2314_b200 import _capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    L = _capi.load()
    header = open(os.path.join(ROOT, "include", "wallace_b200.h")).read()
    declared = set(re.findall(r"\b(wallace_[a-z_0-9]+)\s*\(", header))
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(L, name), name
    bound = {n for n, _, _ in _capi.SYMBOLS}
    assert declared == bound


@pytest.mark.parametrize("field,kw", [
    ("pool_size", dict(pool_size=48)),
    ("pool_size", dict(pool_size=16)),
    ("discard_every", dict(discard_every=0)),
    ("out_sigma", dict(out_sigma=0.0)),
    ("out_mean", dict(out_mean=float("inf"))),
])
def test_config_validation_names_field(field, kw):
    # test_generator.cpp:42-72
    with pytest.raises(pb.ConfigError, match=field):
        pb.GeneratorConfig(**kw).validate()


def test_valid_config_passes():
    pb.GeneratorConfig().validate()


def test_default_stride_and_plan_decode_vs_reference(ref):
    L = _capi.load()
    R = ref.ref_lib()
    for rows in [8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 1 << 20]:
        assert L.wallace_default_stride(rows) == R.ref_default_stride(rows)
    rng = np.random.default_rng(0)
    for n in (32, 1024, 4096, 16384):
        for _ in range(200):
            w0, w1 = (int(x) for x in rng.integers(0, 2**64, size=2, dtype=np.uint64))
            o1, o2 = C.c_uint64(), C.c_uint64()
            v1 = L.wallace_decode_pass_plan(n, w0, w1, C.byref(o1))
            v2 = R.ref_decode_pass_plan(n, w0, w1, C.byref(o2))
            assert (v1, o1.value) == (v2, o2.value)


def _neumaier(v):
    s = c = 0.0
    for x in v:
        t2 = x * x
        t = s + t2
        c += (s - t) + t2 if abs(s) >= abs(t2) else (t2 - t) + s
        s = t
    return s + c


@pytest.mark.parametrize("n,seed", [(32, 3), (1024, 1), (4096, 1), (2048, 7)])
def test_host_seeding_matches_reference_polar(ref, n, seed):
    """generator.cpp:317-327 restated: Polar values from the reference library,
    Neumaier and the k-scaling in Python doubles; the library must agree bit for bit."""
    L = _capi.load()
    R = ref.ref_lib()
    pol = np.empty(n + 1)
    R.ref_polar(seed, n + 1, pol.ctypes.data_as(C.POINTER(C.c_double)))
    ss = _neumaier(pol[:n].tolist())
    k = math.sqrt(n / ss)
    want = np.array([x * k for x in pol[:n]])
    cfg = pb.GeneratorConfig(pool_size=n, seed=seed)
    raw = np.empty(n)
    res, sq = C.c_double(), C.c_double()
    s4 = (C.c_uint64 * 4)()
    dr = C.c_uint64()
    assert L.wallace_host_seed_pool(C.byref(cfg.to_c()), seed,
                                    raw.ctypes.data_as(C.POINTER(C.c_double)), C.byref(res),
                                    C.byref(sq), s4, C.byref(dr)) == 0
    assert np.array_equal(raw.view(np.uint64), want.view(np.uint64))
    assert res.value == pol[n]
    assert sq.value == _neumaier(want.tolist())
    # 16 warm-up passes take 32 words: draws after construction
    g = ref.RefGen(ref.Cfg(pool_size=n, seed=seed))
    assert dr.value + 32 == g.stats()["uniform_draws"]


def test_rotation_and_affine_configs_are_valid():
    for kw in (dict(transform_family=1), dict(mixing=1), dict(transform_family=1, mixing=1)):
        pb.GeneratorConfig(**kw).validate()  # valid in the reference and built here


def test_rotation_table_vs_reference(ref):
    """The host computes the 16-entry table from its construction
    (transforms.cpp:39-70); it must equal the reference's bit for bit."""
    L, R = _capi.load(), ref.ref_lib()
    t1, c1, s1 = (C.c_double * 16)(), (C.c_double * 16)(), (C.c_double * 16)()
    t2, c2, s2 = (C.c_double * 16)(), (C.c_double * 16)(), (C.c_double * 16)()
    L.wallace_rotation_table(t1, c1, s1)
    R.ref_rotation_table(t2, c2, s2)
    assert list(t1) == list(t2) and list(c1) == list(c2) and list(s1) == list(s2)


@pytest.mark.parametrize("fam,mix", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_plan_decode_ex_vs_reference(ref, fam, mix):
    L, R = _capi.load(), ref.ref_lib()
    rng = np.random.default_rng(5)
    for n in (32, 1024, 4096, 16384):
        cfg = pb.GeneratorConfig(pool_size=n, transform_family=fam, mixing=mix).to_c()
        for _ in range(200):
            w0, w1 = (int(x) for x in rng.integers(0, 2**64, 2, dtype=np.uint64))
            got = _capi.wallace_pass_plan()
            assert L.wallace_decode_pass_plan_ex(C.byref(cfg), w0, w1, C.byref(got)) == 0
            ints, offs = (C.c_int32 * 5)(), (C.c_uint64 * 2)()
            R.ref_decode_pass_plan_ex(n, fam, mix, w0, w1, ints, offs)
            assert (got.wallace_variant, got.t_index[0], got.t_index[1], got.negate[0],
                    got.negate[1]) == tuple(ints)
            assert (got.offset[0], got.offset[1]) == tuple(offs)


@pytest.mark.parametrize("fam,mix", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_pass_coefficient_vs_reference(ref, fam, mix):
    """generator.cpp:273-284 over every (i, j) of small pools, random plans."""
    L, R = _capi.load(), ref.ref_lib()
    rng = np.random.default_rng(11)
    for n in (32, 64):
        cfg = pb.GeneratorConfig(pool_size=n, transform_family=fam, mixing=mix)
        mask = n // 4 - 1 if mix == 0 else n - 1
        for _ in range(3):
            ints = [int(rng.integers(384)), int(rng.integers(16)), int(rng.integers(16)),
                    int(rng.integers(2)), int(rng.integers(2))]
            offs = [int(rng.integers(mask + 1)), int(rng.integers(mask + 1))]
            plan = pb.pass_plan(ints[0], ints[1:3], ints[3:5], offs)
            ci = (C.c_int32 * 5)(*ints)
            co = (C.c_uint64 * 2)(*offs)
            for i in range(n):
                for j in range(n):
                    assert pb.pass_coefficient(cfg, plan, i, j) == R.ref_pass_coefficient(n, fam, mix, ci, co, i, j)


# ---- the reference's L1a layer through the C-ABI (host, bit-identical) -----------
def test_uniform_polar_boxmuller_host_vs_reference(ref):
    """UniformState / uniform_bits / polar_next / boxmuller_next
    (baselines.cpp:19-92) exported by the library equal the reference's."""
    L = _capi.load()
    R = ref.ref_lib()
    for seed in (0, 1, 42, 0xDEADBEEF, 2**64 - 1):
        u = _capi.wallace_uniform_state()
        L.wallace_uniform_seed(seed, C.byref(u))
        want = np.empty(1000, dtype=np.uint64)
        R.ref_uniform_bits(seed, 1000, want.ctypes.data_as(C.POINTER(C.c_uint64)))
        got = [L.wallace_uniform_bits(C.byref(u)) for _ in range(1000)]
        assert got == [int(w) for w in want] and u.draws == 1000
        for method, ref_fn in (("polar_next", R.ref_polar), ("boxmuller_next", R.ref_boxmuller)):
            want = np.empty(2001, dtype=np.float64)
            ref_fn(seed, 2001, want.ctypes.data_as(C.POINTER(C.c_double)))
            b = pb.BaselineState(seed)
            got = np.array([getattr(b, method)() for _ in range(2001)])
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (seed, method)
    # the frozen uniform doubles (test_baselines.cpp:61-74)
    u = _capi.wallace_uniform_state()
    L.wallace_uniform_seed(42, C.byref(u))
    assert L.wallace_uniform_next(C.byref(u)) == 0.083862971059882163
    assert L.wallace_uniform_next(C.byref(u)) == 0.37898025066266861


def test_boxmuller_pair_domain():
    L = _capi.load()
    z1, z2 = C.c_double(), C.c_double()
    assert L.wallace_boxmuller_pair(1.0, 0.0, C.byref(z1), C.byref(z2)) == 0
    assert z1.value == 0.0 and z2.value == 0.0
    for u1, u2 in ((0.0, 0.5), (1.5, 0.5), (0.5, 1.0), (0.5, -0.1), (float("nan"), 0.5)):
        assert L.wallace_boxmuller_pair(u1, u2, C.byref(z1), C.byref(z2)) == _capi.WALLACE_ERR_INVALID_PARAM


def test_chi2_helpers_vs_reference(ref):
    """compute_a / Chi2Params / chi2_sample (chi2.cpp:11-59) and the
    reference's spot values (test_chi2.cpp:70-127)."""
    L = _capi.load()
    R = ref.ref_lib()
    for nu in (8, 64, 1024, 2048, 4096, 10**6):
        a = C.c_double()
        assert L.wallace_chi2_params(nu, C.byref(a)) == 0
        assert a.value == R.ref_compute_a(nu)
        rng = np.random.default_rng(nu)
        for x in np.concatenate([rng.normal(size=200) * 3, [-60.0, -45.0, 0.0, 1e3]]):
            for m in (0, 1, 2):
                out, cl = C.c_double(), C.c_int32()
                rc = C.c_int()
                assert L.wallace_chi2_sample(float(x), nu, a.value, m, C.byref(cl), C.byref(out)) == 0
                want = R.ref_chi2_sample(float(x), nu, m, C.byref(rc))
                assert out.value == want and cl.value == rc.value, (nu, x, m)
    assert abs(pb.chi2_sample(0.0, 1024, 0)[0] - 1023.5) <= 1e-9  # test_chi2.cpp:70-91
    assert abs(pb.chi2_sample(0.0, 1024, 1)[0] - 1023.3334) < 1e-3
    with pytest.raises(pb.InvalidParameterError, match="nu must be >= 8"):
        pb.chi2_sample(0.0, 7)
    with pytest.raises(pb.InvalidParameterError, match="x must be finite"):
        pb.chi2_sample(float("inf"), 1024)


def test_variants_and_rotation_vs_reference(ref):
    """wallace_variant (transforms.cpp:76-97) and rotation_from_t (:52-70)."""
    L = _capi.load()
    R = ref.ref_lib()
    for vid in range(384):
        e1, s1, g1 = (C.c_double * 16)(), (C.c_uint8 * 4)(), (C.c_double * 4)()
        assert L.wallace_variant(vid, e1, s1, g1) == 0
        src, sg, e2 = (C.c_int * 4)(), (C.c_double * 4)(), (C.c_double * 16)()
        R.ref_wallace_variant(vid, src, sg, e2)
        assert list(e1) == list(e2) and list(s1) == list(src) and list(g1) == list(sg)
    assert L.wallace_variant(384, None, None, None) == _capi.WALLACE_ERR_INVALID_PARAM
    t, c, s = (C.c_double * 16)(), (C.c_double * 16)(), (C.c_double * 16)()
    L.wallace_rotation_table(t, c, s)
    cc, ss = C.c_double(), C.c_double()
    for k in range(16):
        assert L.wallace_rotation_from_t(t[k], C.byref(cc), C.byref(ss)) == 0
        assert (cc.value, ss.value) == (c[k], s[k])
    assert L.wallace_rotation_from_t(0.5, C.byref(cc), C.byref(ss)) == 0 and (cc.value, ss.value) == (0.6, 0.8)
    assert L.wallace_rotation_from_t(float("inf"), C.byref(cc), C.byref(ss)) == _capi.WALLACE_ERR_INVALID_PARAM

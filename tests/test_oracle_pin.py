"""Pin the CPU oracle (test infrastructure) before trusting it.

1. Against the reference's own frozen vectors and known-answer tests
   (test_baselines.cpp:19-74, test_transforms.cpp:99-129, 300-309,
   test_chi2.cpp:70-127).
2. Bit-for-bit against the unmodified reference library compiled from its
   sources (oracle/_ref, oracle/Makefile) on every BASELINE config shape.
"""
import math

import numpy as np
import pytest

from oracle.oracle import Cfg, OracleGen, RefGen, oracle_lib, uniform_words

pytestmark = pytest.mark.usefixtures("oracle_built")


# ---- test_baselines.cpp:61-74: frozen vectors, seed 42 -------------------------
def test_xoshiro_frozen_vectors_seed42():
    words = uniform_words(42, 6)
    assert [int(w) for w in words] == [
        0x15780b2e0c2ec716, 0x6104d9866d113a7e, 0xae17533239e499a1,
        0xecb8ad4703b360a1, 0xfde6dc7fe2ec5e64, 0xc50da53101795238]
    import ctypes as C
    L = oracle_lib()
    s = (C.c_uint64 * 4)()
    L.wo_uniform_seed(42, s)
    assert L.wo_uniform_next(s) == 0.083862971059882163
    assert L.wo_uniform_next(s) == 0.37898025066266861
    assert L.wo_uniform_next(s) == 0.68004341102813937


def _ref_xoshiro(seed, n):
    """test_baselines.cpp:19-46 RefXoshiro, restated independently in Python."""
    M = (1 << 64) - 1
    s = []
    for _ in range(4):
        seed = (seed + 0x9e3779b97f4a7c15) & M
        z = seed
        z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & M
        z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & M
        s.append(z ^ (z >> 31))

    def rotl(x, k):
        return ((x << k) | (x >> (64 - k))) & M

    out = []
    for _ in range(n):
        out.append((rotl((s[1] * 5) & M, 7) * 9) & M)
        t = (s[1] << 17) & M
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = rotl(s[3], 45)
    return out


@pytest.mark.parametrize("seed", [0, 42, 0xdeadbeef])
def test_xoshiro_matches_published_recurrence(seed):
    assert [int(w) for w in uniform_words(seed, 1000)] == _ref_xoshiro(seed, 1000)


# ---- test_transforms.cpp:300-309 default_stride policy ------------------------
def test_default_stride_policy():
    L = oracle_lib()
    assert L.wo_default_stride(16) == 7
    assert L.wo_default_stride(256) == 87
    assert [L.wo_default_stride(r) for r in (256, 512, 1024)] == [87, 171, 343]
    rows = 8
    while rows <= 4096:
        s = L.wo_default_stride(rows)
        assert s % 2 == 1 and 3 * s > rows and math.gcd(s, rows) == 1
        rows *= 2


# ---- test_transforms.cpp:99-129: A1 and its variants ---------------------------
def test_wallace_variants_orthogonal_and_distinct():
    import ctypes as C
    L = oracle_lib()
    a1 = np.array([[1, 1, -1, 1], [1, -1, 1, 1], [1, -1, -1, -1], [-1, -1, -1, 1]]) * 0.5
    seen = set()
    for vid in range(384):
        src = (C.c_int * 4)()
        sign = (C.c_double * 4)()
        L.wo_wallace_variant(vid, src, sign)
        m = np.array([[sign[k] * a1[src[k]][j] for j in range(4)] for k in range(4)])
        assert np.array_equal(m.T @ m, np.eye(4))
        seen.add(m.tobytes())
        if vid == 0:
            assert np.array_equal(m, a1)
    assert len(seen) == 384


# ---- test_chi2.cpp:70-127 spot values and clamp --------------------------------
def test_chi2_spot_values_and_clamp():
    import ctypes as C
    L = oracle_lib()
    a1024 = L.wo_compute_a(1024)
    cl = C.c_int()
    assert abs(L.wo_chi2_sample(0.0, 1024, a1024, 0, C.byref(cl)) - 1023.5) <= 1e-12 * 1023.5
    wh = L.wo_chi2_sample(0.0, 1024, a1024, 1, C.byref(cl))
    d = 2.0 / 9216.0
    assert abs(wh - 1024.0 * (1 - d) ** 3) <= 1e-12 * wh
    for nu in (64, 1024, 4096):
        a = L.wo_compute_a(nu)
        got = L.wo_chi2_sample(0.0, nu, a, 2, C.byref(cl))
        assert abs(got - (nu - a)) <= 1e-9 * abs(nu - a)
    a64 = L.wo_compute_a(64)
    s = L.wo_chi2_sample(-math.sqrt(127.0), 64, a64, 0, C.byref(cl))
    assert cl.value == 1 and s == 1e-6 * 64
    s = L.wo_chi2_sample(-20.0, 64, a64, 1, C.byref(cl))
    assert cl.value == 1 and s == 1e-6 * 64
    s = L.wo_chi2_sample(-12.0, 64, a64, 2, C.byref(cl))
    assert cl.value == 0 and s > 0


# ---- bit-exact against the unmodified reference library -------------------------
PIN_CASES = [
    # (pool_size, discard_every, chi2_method, disable_chi2, seed, count)  BASELINE shapes
    (4096, 2, 2, True, 1, 1 << 18),     # config 2 shape
    (4096, 2, 2, False, 1, 1 << 18),    # config 3 shape
    (2048, 3, 2, False, 7, 1 << 17),    # config 4 shape
    (1024, 1, 2, False, 1, 1 << 20),    # config 1/5 shape, crosses 4 renormalisations
    (64, 1, 0, False, 5, 100000),
    (128, 3, 1, False, 9, 50000),
    (32, 2, 2, False, 3, 20000),
]


@pytest.mark.parametrize("case", PIN_CASES)
def test_oracle_f64_bit_exact_vs_reference(ref, case):
    n, d, chi, dis, seed, cnt = case
    c = Cfg(pool_size=n, discard_every=d, chi2_method=chi, disable_chi2=dis, seed=seed)
    a = RefGen(c).fill(cnt)
    b = OracleGen(c, "f64").fill(cnt)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_oracle_api_semantics_vs_reference(ref):
    """next_pool / step_pass / inject_pool / fill chunks / mean-sigma / fixed."""
    c = Cfg(pool_size=64, seed=21, out_mean=5.0, out_sigma=2.0, discard_every=2)
    r, o = RefGen(c), OracleGen(c, "f64")
    for k in (5, 5, 200, 63, 1):
        assert np.array_equal(r.fill(k), o.fill(k))
    r.step_pass(); o.step_pass()
    assert np.array_equal(r.fill(70), o.fill(70))
    vr, rr, cr = r.next_pool()
    vo, ro, co = o.next_pool()
    assert np.array_equal(vr, vo) and rr == ro and cr == co
    inj = np.linspace(-2, 2, 64)
    r.inject_pool(inj); o.inject_pool(inj)
    assert np.array_equal(r.fill(300), o.fill(300))
    assert np.array_equal(r.pool(), o.pool())
    sr, so = r.stats(), o.stats()
    for k in ("pass_count", "uniform_draws", "chi2_clamp_count", "sum_sq", "reserved_prev"):
        assert sr[k] == so[k], k
    cf = Cfg(pool_size=128, seed=4, fixed_transform=True)
    assert np.array_equal(RefGen(cf).fill(5000), OracleGen(cf, "f64").fill(5000))


def test_oracle_f32_restatement_tracks_reference(ref):
    """The fp32 restatement stays within the documented absolute tolerance of
    the fp64 reference (|dx| <= 1e-4 on the unit-variance scale)."""
    for n, d, dis, seed, cnt in [(4096, 2, True, 1, 1 << 18), (1024, 1, False, 1, 1 << 20)]:
        c = Cfg(pool_size=n, discard_every=d, disable_chi2=dis, seed=seed)
        a = RefGen(c).fill(cnt)
        f = OracleGen(c, "f32").fill(cnt).astype(np.float64)
        assert np.max(np.abs(f - a)) <= 1e-4


# ---- rotation family and affine mixing (generator.cpp:86-172) -------------------
def test_rotation_table_and_multipliers_vs_reference(ref):
    """The oracle computes the 16 half-angle tangents from their construction
    (transforms.cpp:39-50) and default_multipliers (generator.cpp:286-294);
    both must equal the reference's values bit for bit."""
    import ctypes as C
    L, R = oracle_lib(), ref.ref_lib()
    t, c, s = (C.c_double * 16)(), (C.c_double * 16)(), (C.c_double * 16)()
    R.ref_rotation_table(t, c, s)
    for k in range(16):
        assert L.wo_rotation_t(k) == t[k], k
        oc, os_ = C.c_double(), C.c_double()
        L.wo_rotation_from_t(t[k], C.byref(oc), C.byref(os_))
        assert (oc.value, os_.value) == (c[k], s[k]), k
    for n in [32, 64, 128, 256, 1024, 2048, 4096, 8192, 16384, 1 << 20]:
        a1, b1, a2, b2 = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        R.ref_default_multipliers(n, C.byref(a1), C.byref(b1))
        L.wo_default_multipliers(n, C.byref(a2), C.byref(b2))
        assert (a1.value, b1.value) == (a2.value, b2.value), n


FAMILY_CASES = [
    # (family, mixing, pool_size, discard_every, chi2_method, disable_chi2, seed, count)
    (0, 1, 1024, 1, 2, False, 3, 300000),   # wallace4 + affine, crosses a renormalisation
    (0, 1, 4096, 2, 2, True, 1, 1 << 17),
    (0, 1, 32, 2, 1, False, 8, 20000),
    (1, 0, 1024, 1, 2, False, 1, 300000),   # rotation + stride_transpose
    (1, 0, 2048, 3, 2, False, 7, 1 << 16),
    (1, 0, 64, 1, 0, False, 5, 50000),
    (1, 1, 1024, 2, 2, False, 11, 200000),  # rotation + affine
    (1, 1, 4096, 1, 2, True, 2, 1 << 16),
    (1, 1, 32, 3, 2, False, 4, 20000),
]


@pytest.mark.parametrize("case", FAMILY_CASES)
def test_oracle_families_bit_exact_vs_reference(ref, case):
    fam, mix, n, d, chi, dis, seed, cnt = case
    c = Cfg(pool_size=n, discard_every=d, chi2_method=chi, disable_chi2=dis, seed=seed,
            transform_family=fam, mixing=mix)
    r, o = RefGen(c), OracleGen(c, "f64")
    assert np.array_equal(r.fill(cnt).view(np.uint64), o.fill(cnt).view(np.uint64))
    sr, so = r.stats(), o.stats()
    for k in ("pass_count", "uniform_draws", "chi2_clamp_count", "sum_sq", "reserved_prev"):
        assert sr[k] == so[k], k
    assert np.array_equal(r.pool(), o.pool())


@pytest.mark.parametrize("fam,mix", [(0, 1), (1, 0), (1, 1)])
def test_oracle_families_fixed_transform_and_api(ref, fam, mix):
    cf = Cfg(pool_size=128, seed=4, fixed_transform=True, transform_family=fam, mixing=mix)
    assert np.array_equal(RefGen(cf).fill(5000), OracleGen(cf, "f64").fill(5000))
    c = Cfg(pool_size=64, seed=21, out_mean=5.0, out_sigma=2.0, discard_every=2,
            transform_family=fam, mixing=mix)
    r, o = RefGen(c), OracleGen(c, "f64")
    assert np.array_equal(r.fill(77), o.fill(77))
    r.step_pass(); o.step_pass()
    vr, rr, cr = r.next_pool()
    vo, ro, co = o.next_pool()
    assert np.array_equal(vr, vo) and rr == ro and cr == co
    inj = np.linspace(-2, 2, 64)
    r.inject_pool(inj); o.inject_pool(inj)
    assert np.array_equal(r.fill(300), o.fill(300))


@pytest.mark.parametrize("fam,mix", [(0, 1), (1, 0), (1, 1)])
def test_oracle_families_f32_restatement_tracks_reference(ref, fam, mix):
    """DESIGN.md §3 tolerance for the fp32 restatement, rotation/affine too."""
    c = Cfg(pool_size=1024, discard_every=1, seed=1, transform_family=fam, mixing=mix)
    a = RefGen(c).fill(1 << 19)
    f = OracleGen(c, "f32").fill(1 << 19).astype(np.float64)
    assert np.max(np.abs(f - a)) <= 1e-4


# ---- chi2_sample's throw (chi2.cpp:29-31) modelled by the oracle ----------
from nonfinite_cases import CASES, replay, same_nan_aware  # noqa: E402


@pytest.mark.parametrize("case", range(len(CASES)))
def test_oracle_throw_matches_reference(ref, case):
    """The oracle's modelled throw is the reference's: same call, same
    message, same values before it (f64)."""
    kw, pos, pre, chunks = CASES[case]
    v = np.linspace(-1.5, 1.5, kw["pool_size"])
    v[pos] = np.inf
    r_outs, r_k, r_msg, rg = replay(lambda: RefGen(Cfg(seed=22, **kw)), pre, v, chunks)
    o_outs, o_k, o_msg, og = replay(lambda: OracleGen(Cfg(seed=22, **kw), "f64"), pre, v, chunks)
    assert r_k == o_k and r_msg == o_msg == "chi2_sample: x must be finite"
    for k in range(r_k):
        same_nan_aware(o_outs[k], r_outs[k], f"call {k}")
    rs, os_ = rg.stats(), og.stats()
    assert rs["pass_count"] == os_["pass_count"] and rs["uniform_draws"] == os_["uniform_draws"]



"""The reference's acceptance criteria (tests/acceptance_test.cpp) replayed on
the device stream.  Criteria 2 and 5: test_gpu_fullsize.py; criterion 9:
test_gpu_stream.py.  Not replayed: 3 (a Polar-only model), 6 (host chi2
constants, pinned in test_oracle_pin.py), 7 (CLI timing), and criterion 4's
fixed-transform half (fresh Polar pools per pair, not on the path)."""
import math

import numpy as np
import pytest

import paper_1005_2314_b200 as pb
from paper_1005_2314_b200 import stats

pytestmark = [pytest.mark.gpu]


@pytest.mark.parametrize("fam", [0, 1], ids=["wallace4", "rotation"])
def test_criterion1_sum_of_squares_conservation(cuda, fam):
    """acceptance_test.cpp:103-144: 10^4 passes of an N=1024 generator keep
    |sum x^2 - n| <= 1e-6 n (fp64, the reference's arithmetic)."""
    cfg = pb.GeneratorConfig(pool_size=1024, transform_family=fam, seed=20260808)
    b = pb.PoolBatch(cfg, n_pools=1, seeds=[20260808], dtype="f64")
    worst = 0.0
    for _ in range(100):
        b.step_pass(100)
        raw = b.pool(0)
        worst = max(worst, abs(float(np.sum(raw * raw)) - 1024.0))
    assert worst <= 1e-6 * 1024, worst


def test_criterion4_cross_pool_randomized_null(cuda):
    """acceptance_test.cpp:207-230 (randomized half): N=64, 1e5 pool pairs,
    every default probe |corr| <= 5/sqrt(1e5)."""
    cfg = pb.GeneratorConfig(pool_size=64, seed=20260808)
    b = pb.PoolBatch(cfg, n_pools=1, seeds=[20260808], dtype="f64")
    probes = stats.default_probes(64)
    acc = b.cross_pool_probes(100000, probes)
    reps = stats.cross_pool_correlation_reports(acc, 100000, probes, pool=0)
    assert all(abs(r.statistic) <= 5.0 / math.sqrt(100000.0) for r in reps), [r.statistic for r in reps]


def test_criterion8_rare_event_report(cuda):
    """acceptance_test.cpp:367-389 (Wallace half): a well-formed report at
    1e4*n samples, N=64, threshold 3.2."""
    cfg = pb.GeneratorConfig(pool_size=64, seed=20260808)
    b = pb.PoolBatch(cfg, n_pools=1, seeds=[20260808], dtype="f64")
    totals, marks = b.pool_defect_stats(10000 * 64 // 63, 3.2)
    r = stats.rare_event_adjacency_report(marks[0], 64)
    assert r.name and math.isfinite(r.statistic) and r.std_error >= 0.0


@pytest.mark.parametrize("fam,mix", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_run_pass_vs_reference(cuda, ref, fam, mix):
    """generator.cpp:259-271 run_pass with explicit plans, bit-exact."""
    import ctypes as C
    from oracle.oracle import ref_lib
    R = ref_lib()
    rng = np.random.default_rng(3)
    for n in (32, 1024, 4096):
        cfg = pb.GeneratorConfig(pool_size=n, transform_family=fam, mixing=mix)
        mask = n // 4 - 1 if mix == 0 else n - 1
        for _ in range(4):
            ints = [int(rng.integers(384)), int(rng.integers(16)), int(rng.integers(16)),
                    int(rng.integers(2)), int(rng.integers(2))]
            offs = [int(rng.integers(mask + 1)), int(rng.integers(mask + 1))]
            x = rng.standard_normal(n)
            got = pb.run_pass(cfg, pb.pass_plan(ints[0], ints[1:3], ints[3:5], offs), x)
            want = np.empty(n)
            dp = C.POINTER(C.c_double)
            assert R.ref_run_pass(n, fam, mix, (C.c_int32 * 5)(*ints), (C.c_uint64 * 2)(*offs),
                                  x.ctypes.data_as(dp), want.ctypes.data_as(dp)) == 0
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_criterion4_fixed_transform_q(cuda, ref):
    """acceptance_test.cpp:232-249 (fixed half): probes on coefficients that
    are exactly +-1/2; reports against the composed q_{i,j} pass and equal the
    reference's reports bit for bit."""
    import ctypes as C
    from oracle.oracle import ref_lib
    cfg = pb.GeneratorConfig(pool_size=64, seed=20260808)
    plan = pb.pass_plan()
    probes = []
    for i in range(64):
        if len(probes) == 4:
            break
        for j in range(64):
            if abs(pb.pass_coefficient(cfg, plan, i, j)) == 0.5:
                probes.append((i, j))
                break
    assert len(probes) == 4
    pairs = 100000
    reps = stats.cross_pool_correlation_fixed(cfg, pairs, probes, expect_composed_q=True)
    assert all(r.passed and abs(r.expected) == 0.5 for r in reps)
    out = (C.c_double * 16)()
    R = ref_lib()
    assert R.ref_cross_pool_fixed(64, 0, 0, 20260808, pairs, 4, (C.c_uint64 * 4)(*[p[0] for p in probes]),
                                  (C.c_uint64 * 4)(*[p[1] for p in probes]), 1, out) == 4
    for k, r in enumerate(reps):
        assert (r.statistic, r.expected, r.std_error, r.z_score) == tuple(out[4 * k:4 * k + 4])

"""Host-side defect-suite report math (paper_1005_2314_b200/stats.py) against
the reference's own reports (stats.cpp via oracle/_ref): fed with
accumulators gathered from the reference generator itself, the restated
formulas must reproduce the reference's statistic, SE and z bit for bit."""
import ctypes as C

import numpy as np
import pytest

from paper_1005_2314_b200 import stats
from oracle.oracle import Cfg, RefGen


def _ref4(ref, fn, *args, n=1):
    out = (C.c_double * (4 * n))()
    rc = fn(*args, out)
    return rc, [tuple(out[4 * k:4 * k + 4]) for k in range(n)]


def test_moments_match_reference_welford(ref):
    rng = np.random.default_rng(3)
    x = rng.normal(4096, 90, 5000)
    L = ref.ref_lib()
    out = (C.c_double * 4)()
    L.ref_moments(x.ctypes.data_as(C.POINTER(C.c_double)), x.size, out)
    n, mean, var, skew, kurt = stats.moments(x)
    assert (mean, var, skew, kurt) == tuple(out)


@pytest.mark.parametrize("fam,mix", [(0, 0), (1, 1)])
def test_cross_pool_report_matches_reference(ref, fam, mix):
    n, passes, seed = 256, 1500, 9
    probes = stats.default_probes(n)
    cfg = Cfg(pool_size=n, seed=seed, transform_family=fam, mixing=mix)
    g = RefGen(cfg)
    acc = np.zeros((len(probes), 6))
    prev = g.pool()
    for _ in range(passes):
        g.step_pass()
        cur = g.pool()
        for k, (oi, ij) in enumerate(probes):
            x, y = prev[ij], cur[oi]
            a = acc[k]
            a[0] += x; a[1] += x * x; a[2] += y; a[3] += y * y
            w = x * y
            a[4] += w; a[5] += w * w
        prev = cur
    mine = stats.cross_pool_correlation_reports(acc[None], passes, probes, pool=0)
    L = ref.ref_lib()
    g2 = RefGen(cfg)
    oi = (C.c_uint64 * 8)(*[p[0] for p in probes])
    ij = (C.c_uint64 * 8)(*[p[1] for p in probes])
    out = (C.c_double * 32)()
    assert L.ref_cross_pool_correlation(g2.h, passes, 8, oi, ij, out) == 8
    for k, r in enumerate(mine):
        assert (r.statistic, r.expected, r.std_error, r.z_score) == tuple(out[4 * k:4 * k + 4])


@pytest.mark.parametrize("disable", [False, True])
def test_pool_sum_squares_report_matches_reference(ref, disable):
    n, pools, seed = 128, 1200, 5
    cfg = Cfg(pool_size=n, seed=seed, discard_every=2, disable_chi2=disable)
    g = RefGen(cfg)
    totals = []
    for _ in range(pools):
        vals, res, _ = g.next_pool()
        totals.append(np.cumsum(np.concatenate([[res * res], vals * vals]))[-1])  # sequential order
    mr, vr = stats.pool_sum_squares_reports(np.array(totals), n)
    L = ref.ref_lib()
    out = (C.c_double * 8)()
    assert L.ref_pool_sum_squares(n, 2, 2, seed, int(disable), 0, 0, pools, out) == 0
    assert (mr.statistic, mr.expected, mr.std_error, mr.z_score) == tuple(out[0:4])
    assert (vr.statistic, vr.expected, vr.std_error, vr.z_score) == tuple(out[4:8])


def test_rare_event_report_matches_reference(ref):
    n, seed, thr = 64, 3, 3.0
    samples = 200000
    cfg = Cfg(pool_size=n, seed=seed)
    g = RefGen(cfg)
    marks = [bool(np.any(np.abs(g.next_pool()[0]) > thr)) for _ in range(samples // (n - 1))]
    r = stats.rare_event_adjacency_report(np.array(marks), n)
    L = ref.ref_lib()
    out = (C.c_double * 4)()
    assert L.ref_rare_event_adjacency(n, 2, 1, seed, 0, samples, thr, out) == 0
    assert (r.statistic, r.expected, r.std_error, r.z_score) == tuple(out[0:4])

"""GPU-resident defect suite (stats.cpp:310-338, 340-369, 424-447): the
device accumulators against the oracle generator (same seeds), and the
reports against the reference's own reports (oracle/_ref)."""
import ctypes as C

import numpy as np
import pytest

import paper_1005_2314_b200 as pb
from paper_1005_2314_b200 import stats
from oracle.oracle import Cfg, OracleGen, RefGen, ref_available, ref_lib

from test_gpu_parity import assert_same

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("oracle_built")]


def _probe_sums(o, passes, probes):
    acc = np.zeros((len(probes), 6))
    prev = o.pool()
    for _ in range(passes):
        o.step_pass()
        cur = o.pool()
        for k, (oi, ij) in enumerate(probes):
            x, y = prev[ij], cur[oi]
            a = acc[k]
            a[0] += x; a[1] += x * x; a[2] += y; a[3] += y * y
            w = x * y
            a[4] += w; a[5] += w * w
        prev = cur
    return acc


@pytest.mark.parametrize("kernel", ["throughput", "latency"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("fam,mix", [(0, 0), (1, 1)], ids=["wallace4_stride", "rotation_affine"])
def test_cross_pool_probes_exact(cuda, fam, mix, dtype, kernel):
    n, passes = 256, 600
    kw = dict(pool_size=n, transform_family=fam, mixing=mix)
    seeds = [9, 10, 11]
    b = pb.PoolBatch(pb.GeneratorConfig(**kw), n_pools=len(seeds), seeds=seeds, dtype=dtype)
    b.set_kernel_mode(kernel)
    b.fill(100)  # a partial emission pending: step_pass keeps it (materialised)
    probes = stats.default_probes(n)
    acc = b.cross_pool_probes(passes, probes)
    for p, s in enumerate(seeds):
        o = OracleGen(Cfg(seed=s, **kw), dtype)
        o.fill(100)
        want = _probe_sums(o, passes, probes)
        np.testing.assert_array_equal(acc[p], want)
    # stream continuity: every pool's next values
    got = b.fill(300).cpu().numpy()
    for p, s in enumerate(seeds):
        o = OracleGen(Cfg(seed=s, **kw), dtype)
        o.fill(100)
        for _ in range(passes):
            o.step_pass()
        assert_same(got[p], o.fill(300), f"pool {p} after probes")


def test_cross_pool_reports_equal_reference(cuda, ref):
    n, passes = 512, 2000
    seeds = [21, 22]
    b = pb.PoolBatch(pb.GeneratorConfig(pool_size=n), n_pools=2, seeds=seeds, dtype="f64")
    probes = stats.default_probes(n)
    acc = b.cross_pool_probes(passes, probes)
    L = ref_lib()
    oi = (C.c_uint64 * 8)(*[q[0] for q in probes])
    ij = (C.c_uint64 * 8)(*[q[1] for q in probes])
    for p, s in enumerate(seeds):
        out = (C.c_double * 32)()
        g = RefGen(Cfg(pool_size=n, seed=s))
        assert L.ref_cross_pool_correlation(g.h, passes, 8, oi, ij, out) == 8
        for k, r in enumerate(stats.cross_pool_correlation_reports(acc, passes, probes, pool=p)):
            assert (r.statistic, r.expected, r.std_error, r.z_score) == tuple(out[4 * k:4 * k + 4])


DEFECT_CASES = [
    dict(pool_size=128, discard_every=1),
    dict(pool_size=1024, discard_every=1),            # renormalisations inside the run
    dict(pool_size=4096, discard_every=2),
    dict(pool_size=1024, discard_every=2, disable_chi2=True),
]


@pytest.mark.parametrize("kernel", ["throughput", "latency"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("kw", DEFECT_CASES, ids=lambda k: "_".join(f"{a}{b}" for a, b in k.items()))
def test_pool_defect_stats_vs_oracle(cuda, kw, dtype, kernel):
    n = kw["pool_size"]
    E, thr = 300, 3.0
    seeds = [31, 32, 33]
    b = pb.PoolBatch(pb.GeneratorConfig(**kw), n_pools=len(seeds), seeds=seeds, dtype=dtype)
    b.set_kernel_mode(kernel)
    b.fill(7)  # next_pool discards the partial buffer
    totals, marks = b.pool_defect_stats(E, thr)
    got_after = b.fill(2 * n).cpu().numpy()
    for p, s in enumerate(seeds):
        o = OracleGen(Cfg(seed=s, **kw), dtype)
        o.fill(7)
        wt, wm = [], []
        for _ in range(E):
            vals, res, _ = o.next_pool()
            v = vals.astype(np.float64)
            wt.append(np.cumsum(np.concatenate([[res * res], v * v]))[-1])
            wm.append(bool(np.any(np.abs(v) > thr)))
        np.testing.assert_array_equal(marks[p], np.array(wm))
        np.testing.assert_allclose(totals[p], np.array(wt), rtol=1e-12, atol=0)
        assert_same(got_after[p], o.fill(2 * n), f"pool {p} after the defect run")


def test_defect_reports_vs_reference(cuda, ref):
    """Single-generator reports (f64): rare-event adjacency equal to the
    reference's report; pool sum of squares equal to reduction rounding."""
    n, E, thr, seed = 64, 4000, 3.0, 3
    b = pb.PoolBatch(pb.GeneratorConfig(pool_size=n), n_pools=1, seeds=[seed], dtype="f64")
    totals, marks = b.pool_defect_stats(E, thr)
    L = ref_lib()
    out = (C.c_double * 4)()
    assert L.ref_rare_event_adjacency(n, 2, 1, seed, 0, E * (n - 1), thr, out) == 0
    r = stats.rare_event_adjacency_report(marks[0], n)
    assert (r.statistic, r.expected, r.std_error, r.z_score) == tuple(out)
    out8 = (C.c_double * 8)()
    assert L.ref_pool_sum_squares(n, 2, 1, seed, 0, 0, 0, E, out8) == 0
    mr, vr = stats.pool_sum_squares_reports(totals[0], n)
    np.testing.assert_allclose([mr.statistic, mr.std_error, vr.statistic, vr.std_error],
                               [out8[0], out8[2], out8[4], out8[6]], rtol=1e-9)


def test_defect_needs_standardized_config(cuda):
    b = pb.PoolBatch(pb.GeneratorConfig(pool_size=64, out_sigma=2.0), n_pools=1, seeds=[1], dtype="f64")
    with pytest.raises(pb.InvalidParameterError, match="standardized"):
        b.pool_defect_stats(10)

"""BASELINE.json configs at FULL size on one B200.

Exact comparison on a sample of pools (the oracle finishes in seconds), plus
size-independent properties over the whole job: determinism of a replay,
the per-pool sample moments, and the 5-SE moment reports of the reference's
stats suite (stats.cpp:98-109) for the fused consumer.
"""
import math

import numpy as np
import pytest

import paper_1005_2314_b200 as pb
from oracle.oracle import Cfg, OracleGen, consume_pools

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("oracle_built")]

SAMPLE = [0, 1, 2, 63, 1000, 4095, 8191]


def _sampled_pools(n_pools):
    rng = np.random.default_rng(1234)
    extra = rng.choice(n_pools, size=48, replace=False).tolist()
    return sorted(set([p for p in SAMPLE if p < n_pools] + [n_pools - 1] + extra))


def _check_job(cuda, kw, n_pools, count, dtype):
    torch = cuda
    seeds = np.arange(1, n_pools + 1, dtype=np.uint64)  # seeds 1..P (BASELINE)
    b = pb.PoolBatch(pb.GeneratorConfig(**kw), n_pools=n_pools, seeds=seeds, dtype=dtype)
    b.snapshot()
    tdt = torch.float32 if dtype == "f32" else torch.float64
    out = torch.empty((n_pools, count), dtype=tdt, device="cuda")
    b.fill_from_snapshot_into(out)
    idx = torch.tensor(_sampled_pools(n_pools), device="cuda")
    sample = out.index_select(0, idx).cpu().numpy()
    for row, p in zip(sample, idx.tolist()):
        want = OracleGen(Cfg(seed=int(seeds[p]), **kw), dtype).fill(count)
        ib = np.uint32 if dtype == "f32" else np.uint64
        assert np.array_equal(row.view(ib), want.view(ib)), f"pool {p}"
    # whole-job properties: replay is bit-identical; moments are sane
    iv = torch.int32 if dtype == "f32" else torch.int64
    h1 = out.view(iv).sum(dtype=torch.int64).item()
    b.fill_from_snapshot_into(out)
    assert out.view(iv).sum(dtype=torch.int64).item() == h1
    x = out.double()
    n = x.numel()
    mean = x.mean().item()
    var = x.var().item()
    assert abs(mean) <= 5 / math.sqrt(n)
    assert abs(var - 1) <= 5 * math.sqrt(2 / n) + 5e-6  # fixed-energy configs sit exactly near 1
    del x


def test_config2_full(cuda):
    _check_job(cuda, dict(pool_size=4096, discard_every=2, disable_chi2=True), 16384, 1 << 18, "f32")


def test_config3_full(cuda):
    _check_job(cuda, dict(pool_size=4096, discard_every=2), 16384, 1 << 18, "f32")


def test_config4_full(cuda):
    _check_job(cuda, dict(pool_size=2048, discard_every=3), 8192, 1 << 17, "f64")


def test_config1_full(cuda):
    """Single pool, 2^24 values: bit-exact vs the fp32 restatement and
    within 1e-4 of the fp64 reference stream."""
    kw = dict(pool_size=1024, discard_every=1, seed=1)
    b = pb.PoolBatch(pb.GeneratorConfig(**kw), n_pools=1, dtype="f32")
    v = b.fill(1 << 24).cpu().numpy()[0]
    want = OracleGen(Cfg(**kw), "f32").fill(1 << 24)
    assert np.array_equal(v.view(np.uint32), want.view(np.uint32))
    ref64 = OracleGen(Cfg(**kw), "f64").fill(1 << 24)
    assert np.max(np.abs(v.astype(np.float64) - ref64)) <= 1e-4


def test_config5_full(cuda):
    """65536 pools x 2^18 consumed in-kernel: moment 5-SE reports pass, the
    histogram's chi-square against exact normal bin masses is sane, and a
    1024-pool subset matches the oracle's consumer exactly (histogram) and
    to reduction rounding (sums)."""
    kw = dict(pool_size=1024, discard_every=1)
    P, cnt = 65536, 1 << 18
    b = pb.PoolBatch(pb.GeneratorConfig(**kw), n_pools=P, seeds=np.arange(1, P + 1), dtype="f32")
    sums, hist = b.consume(cnt)
    n = P * cnt
    assert int(hist.sum()) == n
    rep = pb.moment_reports(sums, n)
    assert all(r[4] for r in rep.values()), rep
    edges = np.arange(257) / 16.0 - 8.0
    cdf = np.array([0.5 * math.erfc(-e / math.sqrt(2)) for e in edges])
    expect = n * np.diff(cdf)
    ok = expect > 50
    chi2 = float(np.sum((hist[1:257][ok] - expect[ok]) ** 2 / expect[ok]))
    dof = int(ok.sum()) - 1
    assert abs(chi2 - dof) / math.sqrt(2 * dof) < 6, (chi2, dof)
    sub = pb.PoolBatch(pb.GeneratorConfig(**kw), n_pools=1024, seeds=np.arange(1, 1025), dtype="f32")
    s2, h2 = sub.consume(cnt)
    os_, oh = consume_pools(Cfg(**kw), "f32", np.arange(1, 1025, dtype=np.uint64), cnt)
    assert np.array_equal(h2, oh)
    tol = 1e-6 * 1024 * cnt * np.array([0.80, 1.0, 1.60, 3.0])
    assert np.all(np.abs(s2 - os_) <= tol), (s2, os_)


def test_acceptance_criterion2_moments(cuda):
    """acceptance_test.cpp:146-190 on the device stream: 1e7 values, default
    config, seed 42, the criterion's absolute bounds."""
    for dtype in ("f64", "f32"):
        b = pb.PoolBatch(pb.GeneratorConfig(seed=42), n_pools=1, dtype=dtype)
        x = b.fill(10_000_000).cpu().numpy()[0].astype(np.float64)
        m = x.mean()
        v = x.var(ddof=1)
        c = x - m
        m2 = np.mean(c ** 2)
        sk = np.mean(c ** 3) / m2 ** 1.5
        ku = np.mean(c ** 4) / m2 ** 2 - 3
        assert abs(m) <= 1.6e-3 and abs(v - 1) <= 2.3e-3 and abs(sk) <= 3.9e-3 and abs(ku) <= 7.8e-3


def test_acceptance_criterion5_pool_sum_of_squares(cuda):
    """acceptance_test.cpp:252-310 via next_pool: pool sums of squares have
    mean nu and variance 2nu (+-10%); with chi2 disabled the variance collapses."""
    def pool_ss(disable):
        b = pb.PoolBatch(pb.GeneratorConfig(pool_size=1024, seed=20260808, disable_chi2=disable),
                         n_pools=1, dtype="f64")
        out = []
        for _ in range(2000):
            vals, res, _ = b.next_pool()
            out.append(float((vals.double() ** 2).sum().item()) + res[0] ** 2)
        return np.array(out)
    ss = pool_ss(False)
    assert abs(ss.mean() - 1024) <= 5 * math.sqrt(2048 / ss.size)
    assert 0.9 <= ss.var(ddof=1) / 2048 <= 1.1
    assert pool_ss(True).var() < 1e-6

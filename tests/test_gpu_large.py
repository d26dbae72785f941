"""Pools above the on-chip limit (N > 2^14 fp32 / 2^13 fp64) run on the
HBM-resident executor (wallace_large.cu): same parity bar as the on-chip
kernel -- bit-exact against the oracle for every family/mixing, both dtypes,
across emissions, renormalisations and the API sequences."""
import numpy as np
import pytest

import paper_1005_2314_b200 as pb
from oracle.oracle import Cfg, OracleGen

from test_gpu_parity import assert_same, bits

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("oracle_built")]

CASES = [
    ("f32", 1 << 15), ("f32", 1 << 16), ("f64", 1 << 14), ("f64", 1 << 15),
]


@pytest.mark.parametrize("fam,mix", [(0, 0), (0, 1), (1, 0), (1, 1)],
                         ids=["wallace4_stride", "wallace4_affine", "rotation_stride", "rotation_affine"])
@pytest.mark.parametrize("dtype,n", CASES, ids=lambda c: str(c))
def test_large_pool_fill_matches_oracle(cuda, dtype, n, fam, mix):
    kw = dict(pool_size=n, discard_every=2, transform_family=fam, mixing=mix)
    seeds = [3, 4]
    b = pb.PoolBatch(pb.GeneratorConfig(**kw), n_pools=2, seeds=seeds, dtype=dtype)
    o = [OracleGen(Cfg(seed=s, **kw), dtype) for s in seeds]
    count = 3 * n + 5
    got = b.fill(count).cpu().numpy()
    for p in range(2):
        assert_same(got[p], o[p].fill(count), f"pool {p}")
    # cross a renormalisation (every 256 passes) and keep going
    b.step_pass(250)
    for g in o:
        for _ in range(250):
            g.step_pass()
    got = b.fill(2 * n + 7).cpu().numpy()
    for p in range(2):
        assert_same(got[p], o[p].fill(2 * n + 7), f"pool {p} after renorm")
        np.testing.assert_array_equal(bits(b.pool(p)), bits(o[p].pool()))


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_large_pool_api_sequence(cuda, dtype):
    n = 1 << 15
    kw = dict(pool_size=n, discard_every=1, out_mean=2.0, out_sigma=0.5)
    b = pb.PoolBatch(pb.GeneratorConfig(**kw), n_pools=2, seeds=[8, 9], dtype=dtype)
    o = [OracleGen(Cfg(seed=s, **kw), dtype) for s in (8, 9)]
    for k in (5, 3 * n, n - 7, 1):
        got = b.fill(k).cpu().numpy()
        for p in range(2):
            assert_same(got[p], o[p].fill(k), f"fill {k}")
    b.step_pass(2)
    for g in o:
        g.step_pass(); g.step_pass()
    vals, res, chi = b.next_pool()
    vals = vals.cpu().numpy()
    for p in range(2):
        ov, ores, ochi = o[p].next_pool()
        assert_same(vals[p], ov, "next_pool")
        assert res[p] == ores and chi[p] == ochi
    inj = np.linspace(-1.5, 1.5, n)
    b.inject_pool(inj, pool=0)
    o[0].inject_pool(inj)
    b.snapshot()
    first = b.fill(2 * n).cpu().numpy()
    for p in range(2):
        assert_same(first[p], o[p].fill(2 * n), "after inject")
    out = np.empty_like(first)
    import torch
    t = torch.empty(first.shape, dtype=b.torch_dtype, device="cuda")
    b.fill_from_snapshot_into(t)  # replay from the device snapshot
    assert_same(t.cpu().numpy()[1], first[1], "snapshot replay")


def _moments_hist(v):
    # bin coordinate in the values' own dtype (as the consumer: fl(16 y + 128))
    t = np.asarray(v) * v.dtype.type(16) + v.dtype.type(128)
    v = np.asarray(v, dtype=np.float64)
    sums = np.array([np.sum(v), np.sum(v * v), np.sum(v ** 3), np.sum(v ** 4)])
    bins = np.floor(t.astype(np.float64))
    hist = np.zeros(258, dtype=np.int64)
    hist[0] = np.sum(bins < 0)
    hist[257] = np.sum(bins >= 256)
    inside = bins[(bins >= 0) & (bins < 256)].astype(int)
    hist[1:257] = np.bincount(inside, minlength=256)
    return sums, hist


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_large_pool_consumer(cuda, dtype):
    n = 1 << 15
    kw = dict(pool_size=n, discard_every=1)
    seeds = [11, 12]
    b = pb.PoolBatch(pb.GeneratorConfig(**kw), n_pools=2, seeds=seeds, dtype=dtype)
    o = [OracleGen(Cfg(seed=s, **kw), dtype) for s in seeds]
    # a fresh consume, one after a partial fill (lead from the pool) and one
    # after step_pass (lead from the materialized leftover)
    for pre in ("none", "fill", "step"):
        if pre == "fill":
            b.fill(100)
            for g in o:
                g.fill(100)
        if pre == "step":
            b.fill(50)
            b.step_pass(1)
            for g in o:
                g.fill(50)
                g.step_pass()
        count = 3 * n + 11
        sums, hist = b.consume(count)
        v = np.concatenate([g.fill(count) for g in o])
        wsums, whist = _moments_hist(v.astype(np.float32) if dtype == "f32" else v)
        assert np.array_equal(hist, whist), pre
        assert np.allclose(sums, wsums, rtol=1e-9, atol=1e-6), (pre, sums, wsums)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_large_pool_defect_stats(cuda, dtype):
    n = 1 << 15
    kw = dict(pool_size=n, discard_every=1)
    E, thr = 260, 3.5  # crosses a renormalisation
    seeds = [21, 22]
    b = pb.PoolBatch(pb.GeneratorConfig(**kw), n_pools=2, seeds=seeds, dtype=dtype)
    totals, marks = b.pool_defect_stats(E, thr)
    for p, s in enumerate(seeds):
        o = OracleGen(Cfg(seed=s, **kw), dtype)
        wt, wm = [], []
        for _ in range(E):
            vals, res, _ = o.next_pool()
            vv = vals.astype(np.float64)
            wt.append(np.cumsum(np.concatenate([[res * res], vv * vv]))[-1])
            wm.append(bool(np.any(np.abs(vv) > thr)))
        np.testing.assert_array_equal(marks[p], np.array(wm))
        np.testing.assert_allclose(totals[p], np.array(wt), rtol=1e-12, atol=0)


@pytest.mark.parametrize("fam,mix", [(0, 0), (1, 1)])
def test_large_pool_probes_exact(cuda, fam, mix):
    from paper_1005_2314_b200 import stats
    n = 1 << 15
    kw = dict(pool_size=n, transform_family=fam, mixing=mix)
    seeds = [31, 32]
    b = pb.PoolBatch(pb.GeneratorConfig(**kw), n_pools=2, seeds=seeds, dtype="f32")
    probes = stats.default_probes(n)
    passes = 260
    acc = b.cross_pool_probes(passes, probes)
    for p, s in enumerate(seeds):
        o = OracleGen(Cfg(seed=s, **kw), "f32")
        want = np.zeros((len(probes), 6))
        prev = o.pool()
        for _ in range(passes):
            o.step_pass()
            cur = o.pool()
            for k, (oi, ij) in enumerate(probes):
                x, y = prev[ij], cur[oi]
                a = want[k]
                a[0] += x; a[1] += x * x; a[2] += y; a[3] += y * y
                w = x * y
                a[4] += w; a[5] += w * w
            prev = cur
        np.testing.assert_array_equal(acc[p], want)

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
    with pytest.raises(pb.UnsupportedError):
        b.consume(10)

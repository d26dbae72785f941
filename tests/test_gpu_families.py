"""GPU parity for the rotation transform family and affine mixing
(generator.cpp:86-172): all three non-default family/mixing combinations,
both dtypes and both kernel geometries, against the pinned oracle
(tests/test_oracle_pin.py pins the oracle's rotation/affine paths to the
reference library bit for bit)."""
import numpy as np
import pytest

import paper_1005_2314_b200 as pb
from oracle.oracle import Cfg, OracleGen

from test_gpu_parity import assert_same

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("oracle_built")]

FAMILIES = [(0, 1), (1, 0), (1, 1)]
FAM_IDS = ["wallace4_affine", "rotation_stride", "rotation_affine"]

CONFIGS = [
    dict(pool_size=32, discard_every=2),
    dict(pool_size=64, discard_every=1, chi2_method=0),
    dict(pool_size=256, discard_every=3, out_mean=5.0, out_sigma=2.0),
    dict(pool_size=1024, discard_every=1),               # crosses renormalisations
    dict(pool_size=2048, discard_every=3, chi2_method=1),
    dict(pool_size=4096, discard_every=2, disable_chi2=True),
    dict(pool_size=8192, discard_every=1),
    dict(pool_size=16384, discard_every=2),
    dict(pool_size=128, fixed_transform=True),
]


@pytest.mark.parametrize("kernel", ["throughput", "latency"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("fam,mix", FAMILIES, ids=FAM_IDS)
@pytest.mark.parametrize("kw", CONFIGS, ids=lambda k: "_".join(f"{a}{b}" for a, b in k.items()))
def test_family_fill_matches_oracle(cuda, kw, fam, mix, dtype, kernel):
    n = kw["pool_size"]
    seeds = [11, 12, 1013]
    # several emissions, misaligned pool-major stride, and > 256 passes
    count = max(3 * n + 5, (300 // kw.get("discard_every", 1)) * (n - 1) + 7)
    kw = dict(kw, transform_family=fam, mixing=mix)
    b = pb.PoolBatch(pb.GeneratorConfig(**kw), n_pools=len(seeds), seeds=seeds, dtype=dtype)
    b.set_kernel_mode(kernel)
    out = b.fill(count).cpu().numpy()
    for p, s in enumerate(seeds):
        o = OracleGen(Cfg(seed=s, **kw), dtype)
        assert_same(out[p], o.fill(count), f"pool {p} seed {s}")
        # the pool state after the job, too
        np.testing.assert_array_equal(b.pool(p), o.pool())


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("fam,mix", FAMILIES, ids=FAM_IDS)
def test_family_api_sequence(cuda, fam, mix, dtype):
    """fill chunks / step_pass / next_pool / inject_pool interleavings
    (generator.cpp:333-343, 387-413) for the other families."""
    kw = dict(pool_size=64, discard_every=2, out_mean=5.0, out_sigma=2.0,
              transform_family=fam, mixing=mix)
    seeds = [21, 22]
    b = pb.PoolBatch(pb.GeneratorConfig(**kw), n_pools=2, seeds=seeds, dtype=dtype)
    o = [OracleGen(Cfg(seed=s, **kw), dtype) for s in seeds]
    for k in (5, 5, 200, 63, 1, 126, 127):
        got = b.fill(k).cpu().numpy()
        for p in range(2):
            assert_same(got[p], o[p].fill(k), f"fill {k} pool {p}")
    b.step_pass()
    for g in o:
        g.step_pass()
    got = b.fill(70).cpu().numpy()
    for p in range(2):
        assert_same(got[p], o[p].fill(70), "after step_pass")
    vals, res, chi = b.next_pool()
    vals = vals.cpu().numpy()
    for p in range(2):
        ov, ores, ochi = o[p].next_pool()
        assert_same(vals[p], ov, "next_pool values")
        assert res[p] == ores and chi[p] == ochi
    inj = np.linspace(-2, 2, 64)
    b.inject_pool(inj, 0)
    o[0].inject_pool(inj)
    got = b.fill(300).cpu().numpy()
    for p in range(2):
        assert_same(got[p], o[p].fill(300), f"after inject pool {p}")


@pytest.mark.parametrize("fam,mix", FAMILIES, ids=FAM_IDS)
def test_family_many_pools_hash(cuda, fam, mix):
    """A throughput-geometry batch (2048 pools of N=4096 fp32, d=2): every
    pool's slice against the oracle for a sample, all pools stable."""
    kw = dict(pool_size=4096, discard_every=2, transform_family=fam, mixing=mix)
    n_pools, count = 2048, 4 * 4095 + 3
    seeds = np.arange(1, n_pools + 1, dtype=np.uint64)
    b = pb.PoolBatch(pb.GeneratorConfig(**kw), n_pools=n_pools, seeds=seeds, dtype="f32")
    out = b.fill(count).cpu().numpy()
    for p in (0, 1, 777, 2047):
        assert_same(out[p], OracleGen(Cfg(seed=int(seeds[p]), **kw), "f32").fill(count), f"pool {p}")

"""GPU parity of pair_kernel (csrc/pool_pair.cu): fp32 pools of 4096 values,
wallace4 passes with stride mixing, discard_every = 2 -- two passes per
shared-memory round trip, emission staged per row and sent by bulk copies.

Bit-exact against the oracle's fp32 restatement (generator.cpp:64-85,
333-376) and against pool_kernel (WALLACE_B200_PAIR=0) over: row lengths
that are and are not multiples of four values, partial last emissions, fills
that resume a partially consumed emission, launches that cross
renormalisations (pass_count % 256 == 0), every chi2 method, scaled and
shifted output, and save/load of the state in between.
"""
import os

import numpy as np
import pytest

import paper_1005_2314_b200 as pb
from oracle.oracle import Cfg, OracleGen

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("oracle_built")]

N = 4096


def bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


def assert_same(got, want, what=""):
    got = np.asarray(got)
    want = np.asarray(want)
    assert got.dtype == want.dtype and got.shape == want.shape, what
    if not np.array_equal(bits(got), bits(want)):
        bad = np.nonzero(bits(got) != bits(want))[0]
        raise AssertionError(f"{what}: {bad.size} mismatches, first at {bad[:8]}: "
                             f"got {got[bad[:4]]} want {want[bad[:4]]}")


@pytest.fixture(autouse=True)
def pair_on(monkeypatch):
    """WALLACE_B200_PAIR is read at handle creation (pair_kernel is on by
    default; the tests that compare with pool_kernel set it themselves)."""
    monkeypatch.setenv("WALLACE_B200_PAIR", "1")


def batch(kw, seeds):
    b = pb.PoolBatch(pb.GeneratorConfig(pool_size=N, discard_every=2, **kw), n_pools=len(seeds), seeds=seeds,
                     dtype="f32")
    b.set_kernel_mode("throughput")
    return b


KW = [
    dict(),
    dict(disable_chi2=True),
    dict(chi2_method=0),
    dict(chi2_method=1, out_mean=5.0, out_sigma=2.0),
    dict(out_sigma=0.75),
    dict(fixed_transform=True),
]


@pytest.mark.parametrize("kw", KW, ids=lambda k: "_".join(f"{a}{b}" for a, b in k.items()) or "default")
@pytest.mark.parametrize("count", [N, 5 * (N - 1) + 1, 8 * N, 130 * (N - 1) + 12])
def test_pair_fill_matches_oracle(cuda, kw, count):
    """One fill: full emissions (TMA rows at every misalignment), a partial last
    emission, and (130 emissions) a renormalisation inside the fill."""
    seeds = [1, 77, 16384]
    b = batch(kw, seeds)
    l0 = pb.kernel_launches()
    out = b.fill(count).cpu().numpy()
    assert pb.kernel_launches() > l0
    for p, s in enumerate(seeds):
        want = OracleGen(Cfg(seed=s, pool_size=N, discard_every=2, **kw), "f32").fill(count)
        assert_same(out[p], want, f"pool {p} seed {s}")
    b.close()


@pytest.mark.parametrize("kw", [dict(), dict(disable_chi2=True)], ids=["chi2", "nochi2"])
def test_pair_fill_sequences(cuda, kw):
    """Fills of mixed lengths in sequence: leftovers drained before pair
    launches, rows that are not 16-byte aligned (pool_kernel), step_pass in
    between (odd pass counts), more than 256 passes in total."""
    seeds = [5, 6]
    b = batch(kw, seeds)
    gens = [OracleGen(Cfg(seed=s, pool_size=N, discard_every=2, **kw), "f32") for s in seeds]
    for step, count in enumerate([4 * N, 8, 4095, 3 * N + 4, 7, 40 * N, 4, 64 * N, 2 * N]):
        out = b.fill(count).cpu().numpy()
        for p, g in enumerate(gens):
            assert_same(out[p], g.fill(count), f"fill {step} ({count}) pool {p}")
        if step == 3:
            b.step_pass()
            for g in gens:
                g.step_pass()
    b.close()


def test_pair_equals_pool_kernel(cuda):
    """The same fills with pair_kernel off: identical bits, fewer launches
    are not required, state after the fill identical too (next fill equal)."""
    seeds = list(range(100, 108))
    outs = []
    for on in ("1", "0"):
        os.environ["WALLACE_B200_PAIR"] = on
        b = batch(dict(), seeds)
        o1 = b.fill(33 * N).cpu().numpy()
        o2 = b.fill(2 * N + 8).cpu().numpy()
        outs.append((o1, o2))
        b.close()
    assert_same(outs[0][0], outs[1][0], "first fill")
    assert_same(outs[0][1], outs[1][1], "second fill")


def test_pair_many_pools_cfg3_shape(cuda):
    """BASELINE config 3's shape on a subset of pools: 2^18 values per pool
    (64 full emissions + 64 values), sampled pools against the oracle."""
    n_pools = 1024
    b = pb.PoolBatch(pb.GeneratorConfig(pool_size=N, discard_every=2, seed=1), n_pools=n_pools, dtype="f32")
    count = 1 << 18
    out = b.fill(count)
    for p in (0, 1, 511, 1023):
        want = OracleGen(Cfg(seed=1 + p, pool_size=N, discard_every=2), "f32").fill(count)
        assert_same(out[p].cpu().numpy(), want, f"pool {p}")
    b.close()


def test_pair_is_the_default_path(cuda, monkeypatch):
    """Without the switch a cfg2/cfg3-shaped fill launches pair_kernel (the
    counter of the C-ABI moves); WALLACE_B200_PAIR=0 keeps it on pool_kernel;
    other shapes (fp64, N != 4096, discard_every != 2) never use it."""
    monkeypatch.delenv("WALLACE_B200_PAIR", raising=False)
    seeds = list(range(1, 161))  # above the few-pool latency geometry
    n0 = pb.pair_kernel_launches()
    b = pb.PoolBatch(pb.GeneratorConfig(pool_size=N, discard_every=2), n_pools=len(seeds), seeds=seeds, dtype="f32")
    out = b.fill(3 * (N - 1)).cpu().numpy()
    b.close()
    assert pb.pair_kernel_launches() > n0
    want = OracleGen(Cfg(seed=160, pool_size=N, discard_every=2), "f32").fill(3 * (N - 1))
    assert_same(out[159], want, "default path, pool 159")

    monkeypatch.setenv("WALLACE_B200_PAIR", "0")
    n1 = pb.pair_kernel_launches()
    b = pb.PoolBatch(pb.GeneratorConfig(pool_size=N, discard_every=2), n_pools=len(seeds), seeds=seeds, dtype="f32")
    out0 = b.fill(3 * (N - 1)).cpu().numpy()
    b.close()
    assert pb.pair_kernel_launches() == n1
    assert_same(out0, out, "pool_kernel vs pair_kernel")

    monkeypatch.delenv("WALLACE_B200_PAIR", raising=False)
    for kw, dtype in ((dict(pool_size=N, discard_every=2), "f64"), (dict(pool_size=2048, discard_every=2), "f32"),
                      (dict(pool_size=N, discard_every=3), "f32")):
        n2 = pb.pair_kernel_launches()
        b = pb.PoolBatch(pb.GeneratorConfig(**kw), n_pools=len(seeds), seeds=seeds, dtype=dtype)
        b.fill(2 * kw["pool_size"])
        b.synchronize()
        b.close()
        assert pb.pair_kernel_launches() == n2, (kw, dtype)

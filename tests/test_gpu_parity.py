"""GPU parity: the sm_100a path (libwallace_b200.so, called through the C-ABI)
against the pinned CPU oracle on the same seeds and parameters.

f64: bit-exact vs the oracle's reference semantics (== the reference library,
     tests/test_oracle_pin.py).
f32: bit-exact vs the oracle's fp32 restatement.
The cases replay the reference's hot-path tests (test_generator.cpp) on the
device; the multi-pool cases check every pool slice of a batch.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_1005_2314_b200 as pb
from oracle.oracle import Cfg, OracleGen

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("oracle_built")]

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def gcfg(**kw):
    return pb.GeneratorConfig(**kw)


def ocfg(**kw):
    return Cfg(**kw)


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint32)


def assert_same(got, want, what=""):
    got = np.asarray(got)
    want = np.asarray(want)
    assert got.dtype == want.dtype and got.shape == want.shape, what
    if not np.array_equal(bits(got), bits(want)):
        bad = np.nonzero(bits(got) != bits(want))[0]
        raise AssertionError(f"{what}: {bad.size} mismatches, first at {bad[:8]}: "
                             f"got {got[bad[:4]]} want {want[bad[:4]]}")


CONFIGS = [
    dict(pool_size=32, discard_every=1),
    dict(pool_size=64, discard_every=2, chi2_method=0),
    dict(pool_size=128, discard_every=3, chi2_method=1),
    dict(pool_size=256, discard_every=1, out_mean=5.0, out_sigma=2.0),
    dict(pool_size=512, discard_every=2, disable_chi2=True),
    dict(pool_size=1024, discard_every=1),
    dict(pool_size=2048, discard_every=3),
    dict(pool_size=4096, discard_every=2, disable_chi2=True),
    dict(pool_size=4096, discard_every=2),
    dict(pool_size=8192, discard_every=1, out_mean=-0.5, out_sigma=0.75),
    dict(pool_size=16384, discard_every=1),
    dict(pool_size=128, fixed_transform=True),
]


@pytest.mark.parametrize("kernel", ["throughput", "latency"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("kw", CONFIGS, ids=lambda k: "_".join(f"{a}{b}" for a, b in k.items()))
def test_fill_matches_oracle(cuda, dtype, kw, kernel):
    n = kw["pool_size"]
    seeds = [11, 12, 1013]
    count = 3 * n + 5  # several emissions, misaligned pool-major stride
    b = pb.PoolBatch(gcfg(**kw), n_pools=len(seeds), seeds=seeds, dtype=dtype)
    b.set_kernel_mode(kernel)
    out = b.fill(count).cpu().numpy()
    for p, s in enumerate(seeds):
        want = OracleGen(ocfg(seed=s, **kw), dtype).fill(count)
        assert_same(out[p], want, f"pool {p} seed {s}")


@pytest.mark.parametrize("kernel", ["throughput", "latency"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_chunked_fill_and_api_sequence(cuda, dtype, kernel):
    """fill(5), fill(5), ... carry the partial emission across calls
    (generator.cpp:387-399); step_pass / next_pool / inject_pool interleave
    (generator.cpp:333-343, 401-413)."""
    kw = dict(pool_size=64, discard_every=2, out_mean=5.0, out_sigma=2.0)
    seeds = [21, 22]
    b = pb.PoolBatch(gcfg(**kw), n_pools=2, seeds=seeds, dtype=dtype)
    b.set_kernel_mode(kernel)
    o = [OracleGen(ocfg(seed=s, **kw), dtype) for s in seeds]
    for k in (5, 5, 200, 63, 1, 126, 127):
        got = b.fill(k).cpu().numpy()
        for p in range(2):
            assert_same(got[p], o[p].fill(k), f"fill {k} pool {p}")
    b.step_pass()
    for g in o:
        g.step_pass()
    got = b.fill(70).cpu().numpy()  # drains the old emission first
    for p in range(2):
        assert_same(got[p], o[p].fill(70), "after step_pass")
    vals, res, chi = b.next_pool()
    vals = vals.cpu().numpy()
    for p in range(2):
        v, r, c = o[p].next_pool()
        assert_same(vals[p], v, "next_pool values")
        assert res[p] == r and chi[p] == c
    inj = np.linspace(-2, 2, 64)
    b.inject_pool(inj, pool=1)
    o[1].inject_pool(inj)
    got = b.fill(300).cpu().numpy()
    for p in range(2):
        assert_same(got[p], o[p].fill(300), f"after inject pool {p}")
    for p in range(2):
        assert_same(b.pool(p), o[p].pool(), "pool()")
        info, st = b.info(p), o[p].stats()
        for k in ("pass_count", "uniform_draws", "chi2_clamp_count", "sum_sq", "reserved_prev"):
            assert info[k] == st[k], k
        assert info["buffered"] == st["buffered"]


@pytest.mark.parametrize("kernel", ["throughput", "latency"])
def test_renormalisation_crossings(cuda, kernel):
    """Config-1 shape: 1024 values per pass, renormalised every 256 passes
    (generator.cpp:342, 345-351); 2^18 values cross the boundary once per
    256 emissions."""
    kw = dict(pool_size=1024, discard_every=1)
    for dtype in ("f64", "f32"):
        b = pb.PoolBatch(gcfg(**kw), n_pools=2, seeds=[1, 2], dtype=dtype)
        b.set_kernel_mode(kernel)
        out = b.fill(1 << 18).cpu().numpy()
        for p, s in enumerate([1, 2]):
            g = OracleGen(ocfg(seed=s, **kw), dtype)
            assert_same(out[p], g.fill(1 << 18), f"{dtype} seed {s}")
            assert b.info(p)["sum_sq"] == g.stats()["sum_sq"]


def test_renorm_on_emission_pass_and_midgroup(cuda):
    """d=3 puts the 256-pass renormalisation both on and between emission
    passes; disable_chi2 re-reads sum_sq after it."""
    for kw in (dict(pool_size=128, discard_every=3), dict(pool_size=128, discard_every=3, disable_chi2=True),
               dict(pool_size=64, discard_every=5, chi2_method=0)):
        for dtype in ("f64", "f32"):
            b = pb.PoolBatch(gcfg(**kw), n_pools=1, seeds=[9], dtype=dtype)
            want = OracleGen(ocfg(seed=9, **kw), dtype).fill(40000)
            assert_same(b.fill(40000).cpu().numpy()[0], want, f"{kw} {dtype}")


def test_zero_pool_stays_zero(cuda):
    """test_generator.cpp:93-101 on the device."""
    b = pb.PoolBatch(gcfg(pool_size=64, seed=3), n_pools=1, dtype="f64")
    b.inject_pool(np.zeros(64))
    b.step_pass()
    assert np.all(b.pool(0) == 0.0)


def test_disable_chi2_scale_is_exactly_one(cuda):
    """test_generator.cpp:218-231: values == raw, reserved == raw[n-1]."""
    b = pb.PoolBatch(gcfg(pool_size=128, seed=5, disable_chi2=True), n_pools=1, dtype="f64")
    vals, res, chi = b.next_pool()
    raw = b.pool(0)
    assert np.array_equal(vals.cpu().numpy()[0], raw[:127])
    assert res[0] == raw[127]
    assert chi[0] == b.info(0)["sum_sq"]


def test_emission_scales_to_chi2_draw(cuda):
    """test_generator.cpp:246-260: sum emitted^2 + reserved^2 == S."""
    b = pb.PoolBatch(gcfg(pool_size=1024, seed=31), n_pools=4, dtype="f64")
    for _ in range(50):
        vals, res, chi = b.next_pool()
        v = vals.cpu().numpy()
        for p in range(4):
            total = float(np.sum(v[p] ** 2)) + res[p] ** 2
            assert abs(total - chi[p]) <= 1e-9 * 1024


def test_mean_sigma_exact_affine(cuda):
    """test_generator.cpp:233-244: sigma=2, mean=5 gives exactly 2x+5."""
    a = pb.PoolBatch(gcfg(pool_size=256, seed=99), n_pools=2, dtype="f64").fill(10000).cpu().numpy()
    b = pb.PoolBatch(gcfg(pool_size=256, seed=99, out_mean=5.0, out_sigma=2.0), n_pools=2,
                     dtype="f64").fill(10000).cpu().numpy()
    assert np.array_equal(2.0 * a + 5.0, b)


def test_discard_policy_pass_counts(cuda):
    """test_generator.cpp:312-335: pass_count == 16 + 3(i+1)."""
    b = pb.PoolBatch(gcfg(pool_size=64, seed=9, discard_every=3), n_pools=1, dtype="f64")
    assert b.pass_count() == 16
    prev = b.uniform_draws()
    for i in range(10):
        b.next_pool()
        assert b.pass_count() == 16 + 3 * (i + 1)
        assert b.uniform_draws() - prev == 6  # >= 1 draw per pool (test_generator.cpp:337-351)
        prev = b.uniform_draws()


def test_fill_zero_raises(cuda):
    b = pb.PoolBatch(gcfg(pool_size=64, seed=21), n_pools=1)
    with pytest.raises(pb.InvalidParameterError):
        b.fill(0)
    with pytest.raises(pb.InvalidParameterError):
        b.inject_pool(np.ones(63))


def test_golden_fixtures_on_device(cuda):
    """Every golden case (reference outputs, tests/golden/golden.json)
    reproduced by the device path: f64 == reference, f32 == restatement."""
    for case in GOLDEN["cases"]:
        kw = dict(case["cfg"])
        seed = kw.pop("seed")
        for dtype in ("f64", "f32"):
            b = pb.PoolBatch(gcfg(**kw), n_pools=1, seeds=[seed], dtype=dtype)
            v = b.fill(case["count"]).cpu().numpy()[0]
            h = hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest()
            assert h == case[f"{dtype}_sha256"], (case["name"], dtype)


def test_snapshot_replay_is_identical(cuda):
    torch = cuda
    b = pb.PoolBatch(gcfg(pool_size=4096, discard_every=2, disable_chi2=True), n_pools=64,
                     seeds=list(range(1, 65)), dtype="f32")
    b.snapshot()
    o1 = torch.empty((64, 1 << 16), dtype=torch.float32, device="cuda")
    o2 = torch.empty_like(o1)
    b.fill_from_snapshot_into(o1)
    b.fill_from_snapshot_into(o2)
    assert torch.equal(o1, o2)
    want = OracleGen(ocfg(pool_size=4096, discard_every=2, disable_chi2=True, seed=7), "f32").fill(1 << 16)
    assert_same(o1[6].cpu().numpy(), want, "pool 6 after replay")


def test_save_load_state_resumes(cuda):
    kw = dict(pool_size=256, discard_every=2)
    b = pb.PoolBatch(gcfg(**kw), n_pools=3, seeds=[1, 2, 3], dtype="f32")
    b.fill(1001)
    img = b.save_state()
    x1 = b.fill(5000).cpu().numpy()
    b.load_state(img)
    x2 = b.fill(5000).cpu().numpy()
    assert np.array_equal(x1, x2)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_consumer_matches_oracle(cuda, dtype):
    """Config-5 consumer on a reduced batch: histogram exact, moment sums to
    reduction rounding."""
    from oracle.oracle import consume_pools
    kw = dict(pool_size=1024, discard_every=1)
    seeds = np.arange(1, 65, dtype=np.uint64)
    count = 1 << 14
    b = pb.PoolBatch(gcfg(**kw), n_pools=64, seeds=seeds, dtype=dtype)
    sums, hist = b.consume(count)
    osums, ohist = consume_pools(ocfg(**kw), dtype, seeds, count)
    assert np.array_equal(hist, ohist)
    assert int(hist.sum()) == 64 * count
    # sums: per-element powers are formed in the handle's dtype (fp32 for
    # f32), then accumulated in fp64; tolerance = that rounding, relative to
    # the sum of |x|^k (E|x|^k = 0.80, 1, 1.60, 3 for N(0,1))
    n = 64 * count
    eps = 1e-6 if dtype == "f32" else 1e-12
    tol = eps * n * np.array([0.80, 1.0, 1.60, 3.0])
    assert np.all(np.abs(sums - osums) <= tol), (sums, osums)


def test_boxmuller_comparator_statistics(cuda):
    sums, hist = pb.boxmuller_consume(n_streams=256, count=1 << 14, seed_base=1)
    n = 256 * (1 << 14)
    assert int(hist.sum()) == n
    rep = pb.moment_reports(sums, n)
    assert all(r[4] for r in rep.values()), rep


@pytest.mark.parametrize("n", [512, 4096, 16384])
def test_unit_scale_emission_with_exact_zeros(cuda, n):
    """Scale-1/mean-0 emissions (disable_chi2, sigma 1): a sparse injected pool
    makes exact zeros of both signs; the reference emits them as +0 (x*1 + 0),
    so the device output must have no -0 and match bit for bit."""
    kw = dict(pool_size=n, discard_every=2, disable_chi2=True)
    inj = np.zeros(n)
    inj[::97] = 1.0
    inj[5::131] = -0.5
    for dtype in ("f32", "f64"):
        if dtype == "f64" and n > 8192:
            continue
        b = pb.PoolBatch(gcfg(**kw), n_pools=2, seeds=[3, 4], dtype=dtype)
        o = [OracleGen(ocfg(seed=s, **kw), dtype) for s in (3, 4)]
        b.inject_pool(inj, pool=0)
        o[0].inject_pool(inj)
        count = 6 * (n - 1) + 16
        got = b.fill(count).cpu().numpy()
        for p in range(2):
            want = o[p].fill(count)
            assert_same(got[p], want, f"{dtype} n={n} pool {p}")
        assert np.any(got[0] == 0)
        assert not np.any(np.signbit(got[0][got[0] == 0]))


# ---- bulk emission (scale exactly 1, mean +0: the emission is the pool) ------
BULK_CONFIGS = [
    dict(pool_size=4096, discard_every=2, disable_chi2=True),   # config 2's shape
    dict(pool_size=1024, discard_every=1, disable_chi2=True),   # every pass emits, renormalisations
    dict(pool_size=512, discard_every=3, disable_chi2=True),
    dict(pool_size=128, discard_every=2, disable_chi2=True),
]


@pytest.mark.parametrize("bulk", [True, False], ids=["bulk", "register"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("kw", BULK_CONFIGS, ids=lambda k: f"N{k['pool_size']}_d{k['discard_every']}")
def test_bulk_emission_matches_oracle(cuda, monkeypatch, kw, dtype, bulk):
    """The bulk-emission kernel (shifted shared layout + cp.async.bulk) and
    the register path give the oracle's stream, every emission alignment
    (count not a multiple of 4, so emission starts cycle through all
    shifts), head/tail values and the pool state."""
    if not bulk:
        monkeypatch.setenv("WALLACE_B200_NO_BULK", "1")
    n = kw["pool_size"]
    seeds = list(range(100, 164))
    count = (300 // kw["discard_every"]) * (n - 1) + 7
    b = pb.PoolBatch(gcfg(**kw), n_pools=len(seeds), seeds=seeds, dtype=dtype)
    b.set_kernel_mode("throughput")
    out = b.fill(count).cpu().numpy()
    out2 = b.fill(2 * n + 3).cpu().numpy()   # state carried across launches
    vals, res, chi = b.next_pool()
    vals = vals.cpu().numpy()
    for p in (0, 1, 31, 63):
        o = OracleGen(ocfg(seed=seeds[p], **kw), dtype)
        assert_same(out[p], o.fill(count), f"pool {p}")
        assert_same(out2[p], o.fill(2 * n + 3), f"pool {p} second fill")
        ov, ores, ochi = o.next_pool()
        assert_same(vals[p], ov, f"pool {p} next_pool")
        assert res[p] == ores and chi[p] == ochi
        np.testing.assert_array_equal(bits(b.pool(p)), bits(o.pool()))
        st = o.stats()
        info = b.info(p)
        assert info["reserved_prev"] == st["reserved_prev"] and info["sum_sq"] == st["sum_sq"]


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_bulk_emission_negative_zero_patch(cuda, dtype):
    """A constant pool makes the butterfly cancel exactly: the passes produce
    -0 pool values, which the emission (x*1 + 0) must turn into +0 -- the
    bulk path patches them after its copy lands."""
    kw = dict(pool_size=1024, discard_every=1, disable_chi2=True)
    seeds = list(range(7, 7 + 40))
    b = pb.PoolBatch(gcfg(**kw), n_pools=len(seeds), seeds=seeds, dtype=dtype)
    b.set_kernel_mode("throughput")
    o = OracleGen(ocfg(seed=seeds[3], **kw), dtype)
    const = np.ones(1024)
    b.inject_pool(const, pool=3)
    o.inject_pool(const)
    want = o.fill(20 * 1023 + 3)
    got = b.fill(20 * 1023 + 3).cpu().numpy()[3]
    assert_same(got, want, "constant pool")
    assert np.count_nonzero(want == 0) > 0 and not np.any(np.signbit(want[want == 0]))


def test_bulk_disabled_by_nonfinite_pool(cuda):
    """A non-finite injected pool makes the emission scale NaN (not exactly
    1): the handle stops using bulk emissions and matches the oracle
    (NaN positions and every finite value)."""
    kw = dict(pool_size=1024, discard_every=1, disable_chi2=True)
    seeds = list(range(50, 90))
    b = pb.PoolBatch(gcfg(**kw), n_pools=len(seeds), seeds=seeds, dtype="f32")
    b.set_kernel_mode("throughput")
    o = OracleGen(ocfg(seed=seeds[0], **kw), "f32")
    v = np.linspace(-1, 1, 1024)
    v[17] = np.inf
    b.inject_pool(v, pool=0)
    o.inject_pool(v)
    got = b.fill(5 * 1023 + 2).cpu().numpy()[0]
    want = o.fill(5 * 1023 + 2)
    assert np.array_equal(np.isnan(got), np.isnan(want))
    fin = ~np.isnan(want)
    assert_same(got[fin], want[fin], "finite values")
    # the other pools keep their exact streams
    o1 = OracleGen(ocfg(seed=seeds[1], **kw), "f32")
    assert_same(b.fill(3000).cpu().numpy()[1], (o1.fill(5 * 1023 + 2), o1.fill(3000))[1], "pool 1")


@pytest.mark.parametrize("kernel", ["throughput", "latency"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_huge_discard_every(cuda, dtype, kernel):
    """discard_every above one launch's plan capacity (2048 passes): the host
    runs d-1 passes, then a launch with the last pass and the emission; a
    pending partial emission is drained before those passes, and snapshot
    replay copies the snapshot into the live buffers first."""
    kw = dict(pool_size=256, discard_every=2500)
    seeds = [5, 6]
    b = pb.PoolBatch(gcfg(**kw), n_pools=2, seeds=seeds, dtype=dtype)
    b.set_kernel_mode(kernel)
    o = [OracleGen(ocfg(seed=s, **kw), dtype) for s in seeds]
    for k in (5, 300, 258, 1):
        got = b.fill(k).cpu().numpy()
        for p in range(2):
            assert_same(got[p], o[p].fill(k), f"fill {k} pool {p}")
    b.snapshot()
    first = b.fill(400).cpu().numpy()
    for p in range(2):
        assert_same(first[p], o[p].fill(400), f"fill after snapshot pool {p}")
    import torch
    t = torch.empty(first.shape, dtype=b.torch_dtype, device="cuda")
    b.fill_from_snapshot_into(t)
    assert_same(t.cpu().numpy()[0], first[0], "snapshot replay")


def test_huge_discard_every_consume(cuda):
    """The consumer across a pending lead with an emission longer than one
    launch: the same values as the fills (histogram exact, sums to rounding)."""
    kw = dict(pool_size=256, discard_every=2500)
    seeds = np.array([5, 6], dtype=np.uint64)
    b = pb.PoolBatch(gcfg(**kw), n_pools=2, seeds=seeds, dtype="f64")
    b.consume(7)
    sums, hist = b.consume(600)
    vals = []
    for s in seeds:
        o = OracleGen(ocfg(seed=int(s), **kw), "f64")
        o.fill(7)
        vals.append(o.fill(600))
    v = np.concatenate(vals)
    want = np.array([np.sum(v), np.sum(v * v), np.sum(v ** 3), np.sum(v ** 4)])
    assert np.allclose(sums, want, rtol=1e-12, atol=1e-9)
    bins = np.floor((v + 8.0) * 16.0)
    assert int(hist[0]) == int(np.sum(bins < 0)) and int(hist[257]) == int(np.sum(bins >= 256))
    inside = bins[(bins >= 0) & (bins < 256)].astype(int)
    assert np.array_equal(hist[1:257], np.bincount(inside, minlength=256))

"""Device seeding (wallace_create_ex, WALLACE_CREATE_DEVICE_SEED): the Polar
acceptance stream and draw counts are exact; the Polar values use CUDA's
log, so pools/streams are compared to the host-seeded handle with a stated
tolerance (not a parity path)."""
import time

import numpy as np
import pytest

import paper_1005_2314_b200 as pb

pytestmark = [pytest.mark.gpu]


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("n", [128, 1024, 4096])
def test_device_seed_close_to_host(cuda, n, dtype):
    cfg = pb.GeneratorConfig(pool_size=n, discard_every=2)
    seeds = list(range(1, 41))
    h = pb.PoolBatch(cfg, n_pools=len(seeds), seeds=seeds, dtype=dtype)
    d = pb.PoolBatch(cfg, n_pools=len(seeds), seeds=seeds, dtype=dtype, device_seed=True)
    for p in (0, 7, 39):
        ih, idv = h.info(p), d.info(p)
        assert ih["uniform_draws"] == idv["uniform_draws"] and ih["pass_count"] == idv["pass_count"]
        ph, pd = h.pool(p), d.pool(p)
        if dtype == "f64":
            np.testing.assert_allclose(pd, ph, rtol=0, atol=1e-12)
        else:
            assert np.mean(ph == pd) > 0.97
            np.testing.assert_allclose(pd, ph, rtol=0, atol=2e-6)
        assert abs(idv["sum_sq"] - ih["sum_sq"]) <= 1e-9 * n
    a = h.fill(3 * n).cpu().numpy()
    b = d.fill(3 * n).cpu().numpy()
    np.testing.assert_allclose(b, a, rtol=0, atol=1e-11 if dtype == "f64" else 1e-5)


def test_device_seed_fast_start(cuda):
    """cfg2's batch (16384 pools x N=4096 fp32): device vs host construction."""
    cfg = pb.GeneratorConfig(pool_size=4096, discard_every=2, disable_chi2=True)
    seeds = np.arange(1, 16385, dtype=np.uint64)
    pb.PoolBatch(cfg, n_pools=16, seeds=seeds[:16], device_seed=True)  # module warm-up
    t0 = time.perf_counter()
    pb.PoolBatch(cfg, n_pools=16384, seeds=seeds)
    t1 = time.perf_counter()
    pb.PoolBatch(cfg, n_pools=16384, seeds=seeds, device_seed=True)
    t2 = time.perf_counter()
    print(f"construction 16384 x 4096 fp32: host {t1 - t0:.3f} s, device {t2 - t1:.3f} s")
    assert t2 - t1 < t1 - t0

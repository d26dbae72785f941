"""Emission modes against each other on the device: the staged emission
(kModeFillStaged) and the latency fill with its decoupled chain warp
(kModeFillLat) must produce exactly what the register emission / coupled
chain they replace produce (both are also checked against the oracle in
test_gpu_parity.py).  The modes are chosen per handle at creation from the
WALLACE_B200_NO_STAGED / WALLACE_B200_NO_LATFILL switches."""
import os

import numpy as np
import pytest

import paper_1005_2314_b200 as pb

from test_gpu_parity import assert_same

pytestmark = [pytest.mark.gpu]

CASES = [
    dict(pool_size=256, discard_every=1),
    dict(pool_size=1024, discard_every=1, chi2_method=0),
    dict(pool_size=1024, discard_every=2, out_mean=5.0, out_sigma=2.0),
    dict(pool_size=2048, discard_every=3, chi2_method=1),
    dict(pool_size=4096, discard_every=2),
    dict(pool_size=512, discard_every=2, out_mean=-0.0, out_sigma=0.5),
    dict(pool_size=1024, discard_every=1, mixing=1),
]


def _batch(kw, dtype, seeds, kernel, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        b = pb.PoolBatch(pb.GeneratorConfig(**kw), n_pools=len(seeds), seeds=seeds, dtype=dtype)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    b.set_kernel_mode(kernel)
    return b


def _sequence(b, n):
    """fills across renormalisations, a partial emission carried over, a
    step_pass in between, next_pool; returns everything it produced"""
    outs = [b.fill(n).cpu().numpy(), b.fill(3 * n + 5).cpu().numpy()]
    b.step_pass(3)
    outs.append(b.fill(n + 1).cpu().numpy())
    vals, res, chi2 = b.next_pool()
    outs.append(np.asarray(vals.cpu().numpy() if hasattr(vals, "cpu") else vals))
    outs.append(np.asarray(res, dtype=np.float64))
    outs.append(np.asarray(chi2, dtype=np.float64))
    outs.append(b.fill(2 * n).cpu().numpy())
    outs.append(b.pool(0))
    return outs


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("kw", CASES, ids=lambda k: "-".join(f"{a}{v}" for a, v in k.items()))
@pytest.mark.parametrize("kernel,env", [("throughput", {"WALLACE_B200_NO_STAGED": "1"}),
                                        ("latency", {"WALLACE_B200_NO_LATFILL": "1"})],
                         ids=["staged_vs_register", "latfill_vs_coupled"])
def test_modes_identical(cuda, dtype, kw, kernel, env):
    if dtype == "f64" and kw["pool_size"] > 8192:
        pytest.skip("on-chip fp64 limit")
    seeds = [3, 4, 5]
    n = 300 * kw["pool_size"]  # several hundred passes: renormalisations inside
    new = _batch(kw, dtype, seeds, kernel, {})
    ref = _batch(kw, dtype, seeds, kernel, env)
    for i, (g, w) in enumerate(zip(_sequence(new, n), _sequence(ref, n))):
        assert_same(g, w, f"output {i}")
    for p in range(len(seeds)):
        assert new.info(p) == ref.info(p)
    new.close()
    ref.close()

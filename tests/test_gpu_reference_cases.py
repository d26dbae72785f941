"""Structural cases of the reference's unit suite, replayed on the device
path: construction state (test_generator.cpp:84-91), the dense pass matrix
and its orthogonality (:103-141), mixing by structural reachability and by a
single perturbation (:156-216), and the stride map's bijectivity
(test_transforms.cpp:262-309).  The pass matrices are built column by column
from the device pass (`wallace_run_pass`), so the kernel's gather map is what
is checked, against the C-ABI's `pass_coefficient` and the definitions."""
import ctypes as C

import numpy as np
import pytest

import paper_1005_2314_b200 as pb
from paper_1005_2314_b200 import _capi

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("oracle_built")]

COMBOS = [(0, 0), (0, 1), (1, 0), (1, 1)]  # (family, mixing): wallace4/rotation x stride/affine
IDS = ["wallace4-stride", "wallace4-affine", "rotation-stride", "rotation-affine"]


def decode(cfg, w0, w1):
    """decode_pass_plan (generator.cpp:238-257) through the C-ABI."""
    plan = _capi.wallace_pass_plan()
    assert _capi.load().wallace_decode_pass_plan_ex(C.byref(cfg.to_c()), int(w0), int(w1), C.byref(plan)) == 0
    return plan


def device_pass_matrix(cfg, plan):
    """M[:, j] = run_pass(e_j) on the device (fp64)."""
    n = cfg.pool_size
    m = np.empty((n, n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        m[:, j] = pb.run_pass(cfg, plan, e)
    return m


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_construction_normalizes_and_warms_up(cuda, dtype):
    """test_generator.cpp:84-91: pass_count 16 and sum of squares N after the
    16 warm-up passes (1e-12 relative in fp64; the fp32 pool's own rounding
    in fp32)."""
    cfg = pb.GeneratorConfig(pool_size=1024, seed=7)
    b = pb.PoolBatch(cfg, n_pools=3, seeds=[7, 8, 9], dtype=dtype)
    tol = 1e-12 if dtype == "f64" else 1e-5
    for p in range(3):
        inf = b.info(p)
        assert inf["pass_count"] == 16
        raw = b.pool(p).astype(np.float64)
        assert abs(float(np.sum(raw * raw)) - 1024.0) <= tol * 1024.0
        assert abs(inf["sum_sq"] - 1024.0) <= tol * 1024.0


@pytest.mark.parametrize("fam,mix", COMBOS, ids=IDS)
def test_dense_pass_matrix(cuda, fam, mix):
    """test_generator.cpp:103-141: every column of the device pass equals
    pass_coefficient, and the pass matrix is orthogonal to 1e-12."""
    n = 64
    cfg = pb.GeneratorConfig(pool_size=n, transform_family=fam, mixing=mix, seed=99)
    from oracle.oracle import uniform_words
    w = uniform_words(99, 6)
    for k in range(3):
        plan = decode(cfg, w[2 * k], w[2 * k + 1])
        m = device_pass_matrix(cfg, plan)
        coef = np.array([[pb.pass_coefficient(cfg, plan, i, j) for j in range(n)] for i in range(n)])
        assert np.array_equal(m, coef)
        assert np.max(np.abs(m @ m.T - np.eye(n))) <= 1e-12
        if fam == 0:
            # wallace4: each output mixes exactly 4 inputs with weights +-1/2,
            # each input feeds exactly 4 outputs (the gather map is a bijection
            # of 4-blocks: test_transforms.cpp:262-309)
            nz = m != 0.0
            assert np.all(nz.sum(axis=1) == 4) and np.all(nz.sum(axis=0) == 4)
            assert np.all(np.abs(m[nz]) == 0.5)


@pytest.mark.parametrize("fam,mix", COMBOS, ids=IDS)
def test_mixing_structural_reachability(cuda, fam, mix):
    """test_generator.cpp:156-187: after 8 passes (wallace4/stride; 16 for the
    others) with plans from UniformState(seed), every output depends on
    every input — reachability composed from the device pass matrices."""
    n = 64
    cfg = pb.GeneratorConfig(pool_size=n, transform_family=fam, mixing=mix, seed=1234)
    bound = 8 if (fam, mix) == (0, 0) else 16
    from oracle.oracle import uniform_words
    w = uniform_words(1234, 2 * bound)
    reach = np.eye(n, dtype=bool)
    for p in range(bound):
        nz = device_pass_matrix(cfg, decode(cfg, w[2 * p], w[2 * p + 1])) != 0.0
        reach = (nz.astype(np.int64) @ reach.astype(np.int64)) > 0
    assert int(reach.sum()) == n * n


@pytest.mark.parametrize("fam,mix", COMBOS, ids=IDS)
def test_single_perturbation_reaches_every_output(cuda, fam, mix):
    """test_generator.cpp:189-216: two generators of one seed, pools equal but
    for element 5; within the bound every output has differed at least once."""
    n = 64
    cfg = pb.GeneratorConfig(pool_size=n, transform_family=fam, mixing=mix, seed=1234)
    bound = 8 if (fam, mix) == (0, 0) else 16
    a = pb.PoolBatch(cfg, n_pools=1, seeds=[1234], dtype="f64")
    b = pb.PoolBatch(cfg, n_pools=1, seeds=[1234], dtype="f64")
    base = a.pool(0).astype(np.float64)
    a.inject_pool(base, pool=0)
    base[5] += 1.0
    b.inject_pool(base, pool=0)
    touched = np.zeros(n, dtype=bool)
    for _ in range(bound):
        a.step_pass()
        b.step_pass()
        touched |= a.pool(0) != b.pool(0)
    assert touched.all()


@pytest.mark.parametrize("n", [32, 256, 4096])
def test_stride_gather_is_a_bijection(cuda, n):
    """test_transforms.cpp:262-309 on the device: the stride gather is a
    bijection, so every input feeds exactly four outputs and every output
    mixes exactly four inputs, each with weight 1/2 (wallace4/stride)."""
    cfg = pb.GeneratorConfig(pool_size=n, seed=5)
    from oracle.oracle import uniform_words
    w = uniform_words(5, 2)
    plan = decode(cfg, w[0], w[1])
    if n <= 256:
        m = device_pass_matrix(cfg, plan)
        assert np.all(np.abs(m).sum(axis=0) == 2.0)
        assert np.all(np.abs(m).sum(axis=1) == 2.0)
    else:
        # large pool: one-hot inputs land on exactly four outputs of +-1/2
        for j in (0, 1, n // 2, n - 1):
            e = np.zeros(n)
            e[j] = 1.0
            y = pb.run_pass(cfg, plan, e)
            assert int(np.count_nonzero(y)) == 4 and np.all(np.abs(y[y != 0]) == 0.5)

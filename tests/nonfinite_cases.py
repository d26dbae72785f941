"""Shared cases for chi2_sample's non-finite throw (chi2.cpp:29-31): used by
tests/test_oracle_pin.py (oracle vs reference, CPU) and
tests/test_gpu_errors.py (device vs oracle)."""
import numpy as np


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint32)


def same_nan_aware(got, want, what):
    assert got.shape == want.shape, what
    gn, wn = np.isnan(got), np.isnan(want)
    assert np.array_equal(gn, wn), f"{what}: NaN positions differ"
    assert np.array_equal(bits(got[~gn]), bits(want[~wn])), f"{what}: values differ"


def replay(make, inject_at, v, chunks):
    """Run fills of `chunks` sizes after injecting v: returns (outputs, index
    of the raising call or None, message)."""
    g = make()
    outs = []
    g.fill(inject_at)
    g.inject_pool(v)
    for k, c in enumerate(chunks):
        try:
            outs.append(g.fill(c))
        except ValueError as e:  # InvalidParameterError derives from ValueError
            return outs, k, str(e), g
    return outs, None, "", g


CASES = [
    # (config, value position of the inf, fills before the injection, chunks)
    (dict(pool_size=64, discard_every=1), 63, 100, [30, 63, 63, 200, 5]),
    (dict(pool_size=64, discard_every=2, chi2_method=0), 5, 7, [40, 40, 40, 40, 40, 40]),
    (dict(pool_size=1024, discard_every=1), 1023, 1500, [1000, 1023, 2046, 9, 20000]),
    (dict(pool_size=1024, discard_every=3, chi2_method=1), 0, 1, [5000, 5000, 5000]),
    (dict(pool_size=4096, discard_every=2), 4095, 4095, [4095, 4095, 8190]),
    (dict(pool_size=2048, discard_every=1, out_mean=1.0, out_sigma=2.0), 2047, 10, [3000, 3000, 3000, 40960]),
]

"""Defect-suite reports from the GPU-resident accumulators.

The device does the per-pass / per-emission work (wallace_cross_pool_probes,
wallace_pool_defect_stats); this module turns the raw sums, totals and marks
into the reference's TestReports with the reference's formulas
(/root/reference/proj/core/src/stats.cpp), in the same fp64 operation order,
so a single pool's report equals the reference's report for that generator.
Batches of P pools give P independent generators: the sums / counters are
combined across pools in pool order before the report is formed.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass
class TestReport:
    """maxent::TestReport (stats.hpp:37-49, stats.cpp:58-75)."""

    name: str
    statistic: float
    expected: float
    std_error: float
    z_score: float
    passed: bool

    @staticmethod
    def make(name: str, statistic: float, expected: float, std_error: float) -> "TestReport":
        if std_error > 0.0:
            z = (statistic - expected) / std_error
        else:
            z = 0.0 if statistic == expected else math.copysign(math.inf, statistic - expected)
        return TestReport(name, statistic, expected, std_error, z, abs(z) <= 5.0)


def moments(samples) -> tuple[int, float, float, float, float]:
    """stats.cpp:25-56: one-pass central moments (Welford / Pebay), in the
    reference's operation order.  Returns (count, mean, variance, skewness,
    excess_kurtosis)."""
    x = np.asarray(samples, dtype=np.float64).ravel()
    if x.size < 2:
        raise ValueError("moments: need at least 2 samples")
    mean = m2 = m3 = m4 = 0.0
    n = 0
    for v in x.tolist():
        n1 = float(n)
        n += 1
        nn = float(n)
        delta = v - mean
        delta_n = delta / nn
        delta_n2 = delta_n * delta_n
        term1 = delta * delta_n * n1
        mean += delta_n
        m4 += term1 * delta_n2 * (nn * nn - 3.0 * nn + 3.0) + 6.0 * delta_n2 * m2 - 4.0 * delta_n * m3
        m3 += term1 * delta_n * (nn - 2.0) - 3.0 * delta_n * m2
        m2 += term1
    variance = m2 / float(n - 1)
    skew = kurt = 0.0
    if m2 > 0.0:
        nn = float(n)
        skew = math.sqrt(nn) * m3 / math.pow(m2, 1.5)
        kurt = nn * m4 / (m2 * m2) - 3.0
    return n, mean, variance, skew, kurt


def default_probes(n: int) -> list[tuple[int, int]]:
    """stats.cpp:236-243 default_probes: (out_i, in_j) = (5k mod n, (11k + 3) mod n), k < 8."""
    return [((5 * k) % n, (11 * k + 3) % n) for k in range(8)]


def probe_report(acc6, count: int, name: str, expected: float = 0.0) -> TestReport:
    """ProbeAccumulator::finalize (stats.cpp:202-234) from the six sums
    (sx, sxx, sy, syy, sxy, sxy2) over `count` pairs."""
    sx, sxx, sy, syy, sxy, sxy2 = (float(v) for v in acc6)
    nn = float(count)
    mx = sx / nn
    my = sy / nn
    vx = sxx / nn - mx * mx
    vy = syy / nn - my * my
    if not (vx > 0.0) or not (vy > 0.0):
        raise ValueError("cross_pool_correlation: zero-variance pool values at probe " + name)
    denom = math.sqrt(vx * vy)
    cov = sxy / nn - mx * my
    mean_xy = sxy / nn
    var_xy = sxy2 / nn - mean_xy * mean_xy
    se = math.sqrt(var_xy / nn) / denom
    return TestReport.make(name, cov / denom, expected, se)


def probe_name(out_i: int, in_j: int) -> str:
    return f"cross_pool_corr.i{out_i}.j{in_j}"


def cross_pool_correlation_reports(acc, passes: int, probes, pool=None) -> list[TestReport]:
    """stats.cpp:310-338 reports from wallace_cross_pool_probes sums.
    acc: [n_pools, n_probes, 6].  pool=None combines every pool (sums added
    in pool order, count = passes * n_pools); pool=p reports generator p
    alone (identical to the reference's reports for that generator)."""
    a = np.asarray(acc, dtype=np.float64)
    if pool is not None:
        rows, count = a[pool], passes
    else:
        rows = a[0].copy()
        for p in range(1, a.shape[0]):
            rows = rows + a[p]
        count = passes * a.shape[0]
    return [probe_report(rows[k], count, probe_name(*probes[k])) for k in range(len(probes))]


def pool_sum_squares_reports(totals, pool_size: int) -> tuple[TestReport, TestReport]:
    """stats.cpp:340-369 from the per-emission totals (all pools, pool-major)."""
    n, mean, var, _, kurt = moments(np.asarray(totals, dtype=np.float64).ravel())
    nu = float(pool_size)
    pp = float(n)
    se_mean = math.sqrt(var / pp)
    se_var = var * math.sqrt(max(kurt + 2.0, 0.0) / pp)
    return (TestReport.make("pool_sum_squares.mean", mean, nu, se_mean),
            TestReport.make("pool_sum_squares.variance", var, 2.0 * nu, se_var))


def rare_event_adjacency_report(marks, pool_size: int) -> TestReport:
    """stats.cpp:375-403, 424-447: AdjacencyCounter over each pool's
    consecutive emissions, counters added over pools."""
    m = np.asarray(marks).astype(bool)
    if m.ndim == 1:
        m = m[None, :]
    successors = base = cond_pop = cond = 0
    for row in m:
        prev = row[:-1]
        nxt = row[1:]
        successors += nxt.size
        base += int(np.count_nonzero(nxt))
        cond_pop += int(np.count_nonzero(prev))
        cond += int(np.count_nonzero(prev & nxt))
    name = f"rare_event_adjacency.pool{pool_size}"
    if cond_pop == 0 or base == 0:
        return TestReport.make(name + "[no-marks]", 1.0, 1.0, 0.0)
    b = base / successors
    c = cond / cond_pop
    se_cond = math.sqrt(b * (1.0 - b) / cond_pop)
    return TestReport.make(name, c / b, 1.0, se_cond / b)


def cross_pool_correlation_fixed(cfg, pairs: int, probes=None, expect_composed_q: bool = False):
    """stats.cpp:260-307 with opts.fixed_transform: fresh Polar pools, one
    pinned pass each (device), reports against 0 or the composed q_{i,j}."""
    import paper_1005_2314_b200 as pb
    if pairs < 1000:
        raise ValueError("cross_pool_correlation: pool_pairs must be >= 1000")
    probes = default_probes(cfg.pool_size) if probes is None else list(probes)
    acc = pb.cross_pool_fixed_sums(cfg, pairs, probes)
    plan = pb.pass_plan()
    out = []
    for k, (oi, ij) in enumerate(probes):
        exp = pb.pass_coefficient(cfg, plan, oi, ij) if expect_composed_q else 0.0
        out.append(probe_report(acc[k], pairs, probe_name(oi, ij), exp))
    return out

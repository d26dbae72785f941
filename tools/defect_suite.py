"""Run the GPU-resident defect suite at scale (stats.cpp analyses at 2^34
samples) and print the reports and throughput.  Measurement helper:

    python tools/defect_suite.py [--pools 65536] [--emissions 256] [--passes 10000]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1005_2314_b200 as pb  # noqa: E402
from paper_1005_2314_b200 import stats  # noqa: E402


def moments_fast(x):
    """Two-pass fp64 moments for large sample arrays (the exact Welford
    restatement, stats.moments, is a Python loop)."""
    x = np.asarray(x, dtype=np.float64).ravel()
    n = x.size
    mean = x.mean()
    d = x - mean
    m2 = np.dot(d, d)
    m4 = np.sum(d ** 4)
    return n, mean, m2 / (n - 1), m4 * n / (m2 * m2) - 3.0


def sum_squares_reports(totals, nu):
    n, mean, var, kurt = moments_fast(totals)
    se_mean = np.sqrt(var / n)
    se_var = var * np.sqrt(max(kurt + 2.0, 0.0) / n)
    return (stats.TestReport.make("pool_sum_squares.mean", float(mean), nu, float(se_mean)),
            stats.TestReport.make("pool_sum_squares.variance", float(var), 2.0 * nu, float(se_var)))


def run(label, kw, pools, emissions, passes, probe_pools, thr):
    import torch
    out = {"config": label}
    n = kw["pool_size"]
    seeds = np.arange(1, pools + 1, dtype=np.uint64)
    b = pb.PoolBatch(pb.GeneratorConfig(**kw), n_pools=pools, seeds=seeds, dtype="f32")
    b.pool_defect_stats(2, thr)  # warm-up (module load, kernel attributes)
    torch.cuda.synchronize()
    t = time.perf_counter()
    totals, marks = b.pool_defect_stats(emissions, thr)
    dt = time.perf_counter() - t
    samples = pools * emissions * (n - 1)
    out["pool_stats"] = {"samples": samples, "seconds": dt, "samples_per_s": samples / dt}
    mr, vr = sum_squares_reports(totals, float(n))
    ra = stats.rare_event_adjacency_report(marks, n)
    out["reports"] = [r.__dict__ for r in (mr, vr, ra)]
    del b
    seeds = np.arange(1, probe_pools + 1, dtype=np.uint64)
    b = pb.PoolBatch(pb.GeneratorConfig(**kw), n_pools=probe_pools, seeds=seeds, dtype="f32")
    probes = stats.default_probes(n)
    b.cross_pool_probes(2, probes)  # warm-up
    torch.cuda.synchronize()
    t = time.perf_counter()
    acc = b.cross_pool_probes(passes, probes)
    dt = time.perf_counter() - t
    out["probes"] = {"pairs_per_probe": passes * probe_pools, "seconds": dt,
                     "pool_values_per_s": passes * probe_pools * n / dt}
    reps = stats.cross_pool_correlation_reports(acc, passes, probes)
    out["reports"] += [r.__dict__ for r in reps]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pools", type=int, default=65536)
    ap.add_argument("--emissions", type=int, default=256)
    ap.add_argument("--passes", type=int, default=10000)
    ap.add_argument("--probe-pools", type=int, default=16384)
    ap.add_argument("--threshold", type=float, default=4.0)
    ap.add_argument("--pool-size", type=int, default=1024)
    a = ap.parse_args()
    base = dict(pool_size=a.pool_size, discard_every=1)
    for label, kw in (("production (cubic_a chi2, random transforms)", base),
                      ("diag.disable_chi2", dict(base, disable_chi2=True)),
                      ("diag.fixed_transform", dict(base, fixed_transform=True))):
        r = run(label, kw, a.pools, a.emissions, a.passes, a.probe_pools, a.threshold)
        print(json.dumps(r))
        for rep in r["reports"]:
            print(f"  [{'PASS' if rep['passed'] else 'FAIL'}] {rep['name']:36s} stat={rep['statistic']:.6g} "
                  f"exp={rep['expected']:.6g} z={rep['z_score']:.2f}")
        sys.stdout.flush()


if __name__ == "__main__":
    main()

"""Generate tests/golden/golden.json from the UNMODIFIED reference library.

Run in the build container, where /root/reference exists:

    make -C oracle all ref && python tests/golden/make_golden.py

f64 cases come from oracle/_ref/libmaxent_ref.so (the reference's own
Generator compiled from its sources) — they are reference outputs.  f32
cases come from the pinned C oracle (the reference has no fp32 mode); they
freeze the fp32 restatement of DESIGN.md §3 against regressions.
The GPU box has no /root/reference: tests there read only this JSON.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Cfg, OracleGen, RefGen, uniform_words  # noqa: E402

CASES = [
    # name, cfg kwargs, count  (BASELINE.json configs 1-5 at a per-pool scale,
    # plus the reference test shapes of test_generator.cpp)
    ("cfg1_n1024_d1_seed1", dict(pool_size=1024, discard_every=1, seed=1), 1 << 20),
    ("cfg2_n4096_d2_nochi2_seed1", dict(pool_size=4096, discard_every=2, disable_chi2=True, seed=1), 1 << 18),
    ("cfg2_n4096_d2_nochi2_seed16384", dict(pool_size=4096, discard_every=2, disable_chi2=True, seed=16384), 1 << 18),
    ("cfg3_n4096_d2_seed1", dict(pool_size=4096, discard_every=2, seed=1), 1 << 18),
    ("cfg3_n4096_d2_seed777", dict(pool_size=4096, discard_every=2, seed=777), 1 << 18),
    ("cfg4_n2048_d3_seed1", dict(pool_size=2048, discard_every=3, seed=1), 1 << 17),
    ("cfg4_n2048_d3_seed8192", dict(pool_size=2048, discard_every=3, seed=8192), 1 << 17),
    ("cfg5_n1024_d1_seed65536", dict(pool_size=1024, discard_every=1, seed=65536), 1 << 18),
    ("n64_sqrtshift_seed5", dict(pool_size=64, chi2_method=0, seed=5), 100000),
    ("n128_wh_d3_seed9", dict(pool_size=128, chi2_method=1, discard_every=3, seed=9), 50000),
    ("n256_mean5_sigma2_seed99", dict(pool_size=256, out_mean=5.0, out_sigma=2.0, seed=99), 10000),
    ("n128_fixed_seed4", dict(pool_size=128, fixed_transform=True, seed=4), 5000),
    ("n32_d2_seed3", dict(pool_size=32, discard_every=2, seed=3), 20000),
    ("acc9_n1024_seed42", dict(pool_size=1024, seed=42), 1000000),  # acceptance criterion 9 stream
]


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    out = {"source": "oracle/_ref (reference library) for f64; pinned C oracle for f32",
           "xoshiro_seed1": [hex(int(w)) for w in uniform_words(1, 8)],
           "cases": []}
    for name, kw, cnt in CASES:
        c = Cfg(**kw)
        r = RefGen(c)
        vals = r.fill(cnt)
        st = r.stats()
        f32 = OracleGen(c, "f32")
        fv = f32.fill(cnt)
        fs = f32.stats()
        out["cases"].append(dict(
            name=name, cfg=kw, count=cnt,
            f64_sha256=digest(vals), f64_head=[float(x).hex() for x in vals[:16]],
            f64_tail=[float(x).hex() for x in vals[-4:]],
            f64_pool_sha256=digest(r.pool()),
            f64_stats={k: (float(v).hex() if isinstance(v, float) else v) for k, v in st.items()},
            f32_sha256=digest(fv), f32_head=[float(x).hex() for x in fv[:16].astype(np.float64)],
            f32_pool_sha256=digest(f32.pool()),
            f32_stats={k: (float(v).hex() if isinstance(v, float) else v) for k, v in fs.items()
                       if k != "buffered"},
            f32_vs_f64_maxabs=float(np.max(np.abs(fv.astype(np.float64) - vals))),
        ))
        print(name, out["cases"][-1]["f32_vs_f64_maxabs"])
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()

"""Benchmark built kernel variants (paper_1005_2314_b200/variants/lib_*.so)
on the GPU: a parity smoke per variant, then bench.py configs.  Prints one
summary line per (variant, config).  Measurement helper, not product code."""
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
libs = [os.path.join(ROOT, "paper_1005_2314_b200", "libwallace_b200.so")]
libs += sorted(glob.glob(os.path.join(ROOT, "paper_1005_2314_b200", "variants", "lib_*.so")))
configs = [int(c) for c in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["2", "4"])]
for lib in libs:
    env = dict(os.environ, WALLACE_B200_LIB=lib)
    name = os.path.basename(lib)
    smoke = subprocess.run([sys.executable, "-c", "import __graft_entry__ as g; g.smoke()"], cwd=ROOT,
                           env=env, capture_output=True, text=True)
    ok = smoke.returncode == 0
    for c in configs:
        r = subprocess.run([sys.executable, "bench.py", "--config", str(c), "--steps", "20",
                            "--no-e2e", "--no-cpu", "--no-configs", "--no-sustained"], cwd=ROOT, env=env, capture_output=True, text=True)
        try:
            d = json.loads(r.stdout.strip().splitlines()[-1])
            frac = (d.get("roofline") or {}).get("frac")
            kms = (d.get("roofline") or {}).get("kernel_ms")
            print(f"{name:24s} cfg{c} parity={'ok' if ok else 'FAIL'} ms={d['ms_per_step']:.3f} "
                  f"kernel_ms={kms if kms is None else round(kms, 3)} "
                  f"frac={frac if frac is None else round(frac, 3)} sm_mhz={d['clocks']['sm_mhz']}",
                  flush=True)
        except Exception:  # noqa: BLE001
            print(f"{name:24s} cfg{c} parity={'ok' if ok else 'FAIL'} bench failed: {r.stderr[-300:]}",
                  flush=True)

# For every built variant (paper_1005_2314_b200/variants/lib_*.so): a pytest
# selection ($TESTS, default: none) then quick device timings of configs ($@).
# Measurement helper: bash tools/var_run.sh 5 3   (TESTS="tests/x.py -k y")
cd "$(dirname "$0")/.." || exit 1
for lib in paper_1005_2314_b200/variants/lib_*.so; do
  n=$(basename "$lib" .so)
  if [ -n "$TESTS" ]; then
    r=$(WALLACE_B200_LIB=$PWD/$lib timeout 900 python -m pytest $TESTS -x -q 2>&1 | tail -1)
    echo "$n tests: $r"
  fi
  for c in "$@"; do
    WALLACE_B200_LIB=$PWD/$lib python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e --no-configs --no-sustained > /tmp/vr.json 2>/tmp/vr.err || { echo "$n cfg$c FAILED"; tail -3 /tmp/vr.err; continue; }
    python - "$n" "$c" <<'PY'
import json, sys
d = json.loads(open("/tmp/vr.json").read().strip().splitlines()[-1])
r = d["roofline"]
print(f"{sys.argv[1]:10s} cfg{sys.argv[2]}: {d['ms_per_step']:.3f} ms/step kernel {r['kernel_ms']:.3f} ms frac {r.get('frac') or 0:.3f} clocks {d['clocks']['sm_mhz']} {d['clocks']['reasons']}", flush=True)
PY
  done
done

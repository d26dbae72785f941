# quick device timings of configs ($@, default 2 3 4 5 1): ms per step and kernel ms
for c in ${@:-2 3 4 5 1}; do
  python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e --no-configs --no-sustained > /tmp/qb_$c.json 2>/tmp/qb_$c.err || { echo "cfg$c FAILED"; tail -5 /tmp/qb_$c.err; continue; }
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
d = json.loads(open(f"/tmp/qb_{c}.json").read().strip().splitlines()[-1])
r = d["roofline"]
print(f"cfg{c}: {d['ms_per_step']:.3f} ms/step kernel {r['kernel_ms']:.3f} ms frac {r.get('frac', 0):.3f} "
      f"value {d['value']:.4g} clocks {d['clocks']['sm_mhz']} {d['clocks']['reasons']}")
PY
done

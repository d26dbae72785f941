# cfg3 ablations: chain (a3), bulk read wait (a7), staging stores (a8), proxy fence (a9); register emission
python tools/tune_variants.py 3
WALLACE_B200_NO_STAGED=1 python bench.py --config 3 --steps 20 --no-e2e --no-cpu --no-configs --no-sustained | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('NO_STAGED cfg3', d['ms_per_step'], d['roofline']['kernel_ms'])"

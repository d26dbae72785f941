python -m pytest tests -q -m gpu -x > gpurun_out/r02g_all.log 2>&1
tail -5 gpurun_out/r02g_all.log
python bench.py > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r02g_bench.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['e2e']['s_per_step'], d.get('sustained',{}).get('ms_per_step'))
for k,v in d['configs'].items(): print(k, v['ms_per_step'], v['kernel_ms'], v.get('roofline_frac'), (v.get('e2e') or {}).get('s_per_step'))
"

set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for c in 2 3 4 1 5; do python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02a_cfg$c.json 2>gpurun_out/r02a_cfg$c.err; done
python bench.py --config 2 --steps 300 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02a_cfg2_sustained.json 2>&1

#!/bin/bash
# Run on the GPU box (gpurun): evidence for profiles/.  Each ncu run follows
# the same command run plainly (exit 0) first, per the profiling recipe.
set -u
O=gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
# 1. launch list of the bench command (cfg2): every kernel with its duration
$B > $O/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $O/launches_cfg2.csv $B > $O/ncu_launch.log 2>&1
# 2. full-size per-launch DRAM traffic of pool_kernel (application replay: no
#    16 GiB save/restore), cfg2 (bulk), cfg3 (staged), cfg4 (staged fp64)
for c in 2 3 4; do
  Bc="python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu"
  $Bc > $O/plain$c.log 2>&1 && \
  ncu --replay-mode application -k regex:pool_kernel -s 5 -c 1 \
      --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed \
      --clock-control none --csv --log-file $O/traffic_cfg$c.csv $Bc > $O/ncu_traffic$c.log 2>&1
done
# 3. --set full on 2048-pool jobs (same kernels, 2.3 waves) for stall/pipe analysis
for c in 2 3 4; do
  S="python bench.py --config $c --steps 2 --warmup 3 --pools 2048 --no-e2e --no-cpu"
  $S > $O/plain_s$c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:pool_kernel -s 4 -c 1 \
      -o $O/prof_cfg${c}_full $S > $O/ncu_full$c.log 2>&1
  # the reports are ~25 MB each (gpurun copies back <= 64 MiB): keep CSV pages
  ncu -i $O/prof_cfg${c}_full.ncu-rep --page raw --csv > $O/full_raw_cfg$c.csv 2>/dev/null
  ncu -i $O/prof_cfg${c}_full.ncu-rep --page source --csv --print-source sass > $O/full_sass_cfg$c.csv 2>/dev/null
  [ "$c" = 2 ] || rm -f $O/prof_cfg${c}_full.ncu-rep
done
tail -n 2 $O/ncu_launch.log $O/ncu_traffic2.log $O/ncu_traffic3.log $O/ncu_traffic4.log $O/ncu_full2.log

#!/bin/bash
# Round-2 evidence run on the GPU box: the GPU suite, the default bench line,
# the launch list of the bench command, full-size DRAM traffic of the pool
# kernels (cfg2/3/4), a --set full capture of the cfg2 bulk kernel.
set -u
O=gpurun_out; T=${1:-r02f}
python -m pytest tests -q -m gpu > $O/${T}_gpu_tests.log 2>&1; tail -1 $O/${T}_gpu_tests.log
python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err; tail -c 300 $O/${T}_bench.err
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-configs --no-sustained"
$B > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $O/${T}_launches_cfg2.csv $B > $O/${T}_ncu_launch.log 2>&1
for c in 2 3 4; do
  Bc="python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu --no-configs --no-sustained"
  $Bc > /dev/null 2>&1 && ncu --replay-mode application -k "regex:pool_kernel|pair_kernel" -s 5 -c 1 \
      --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed \
      --clock-control none --csv --log-file $O/${T}_traffic_cfg$c.csv $Bc > $O/${T}_ncu_traffic$c.log 2>&1
done
S="python bench.py --config 2 --steps 2 --warmup 3 --pools 2048 --no-e2e --no-cpu --no-configs --no-sustained"
$S > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k "regex:pool_kernel|pair_kernel" -s 4 -c 1 \
    -o /tmp/${T}_cfg2_full -f $S > $O/${T}_ncu_full2.log 2>&1
ncu -i /tmp/${T}_cfg2_full.ncu-rep --page raw --csv > $O/${T}_full_raw_cfg2.csv 2>/dev/null
ncu -i /tmp/${T}_cfg2_full.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $O/${T}_full_src_cfg2.csv.gz
python tools/launch_summary.py $O/${T}_launches_cfg2.csv | head -8

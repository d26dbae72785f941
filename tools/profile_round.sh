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
#    16 GiB save/restore)
ncu --replay-mode application -k regex:pool_kernel -s 5 -c 1 \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none --csv --log-file $O/traffic_cfg2.csv $B > $O/ncu_traffic.log 2>&1
B4="python bench.py --config 4 --steps 3 --warmup 3 --no-e2e --no-cpu"
$B4 > $O/plain4.log 2>&1 && \
ncu --replay-mode application -k regex:pool_kernel -s 5 -c 1 \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none --csv --log-file $O/traffic_cfg4.csv $B4 > $O/ncu_traffic4.log 2>&1
# 3. --set full on a 2048-pool job (same kernel, 2.3 waves) for stall/pipe analysis
S="python bench.py --steps 2 --warmup 3 --pools 2048 --no-e2e --no-cpu"
$S > $O/plain_s.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pool_kernel -s 4 -c 1 \
    -o $O/prof_cfg2_full $S > $O/ncu_full2.log 2>&1
S4="python bench.py --config 4 --steps 2 --warmup 3 --pools 2048 --no-e2e --no-cpu"
$S4 > $O/plain_s4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pool_kernel -s 4 -c 1 \
    -o $O/prof_cfg4_full $S4 > $O/ncu_full4.log 2>&1
tail -n 2 $O/ncu_launch.log $O/ncu_traffic.log $O/ncu_traffic4.log $O/ncu_full2.log $O/ncu_full4.log

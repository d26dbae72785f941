# --set full of one 2048-pass launch of the cfg1 latency kernel, warp sampling every 32 cycles
TAG=${1:-cfg1}
mkdir -p /tmp/prof gpurun_out
CMD="python bench.py --config 1 --steps 1 --warmup 3 --no-cpu --no-e2e --no-configs --no-sustained"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k "regex:pool_kernel" -s 40 -c 1 -o /tmp/prof/${TAG} -f $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo "rc=$?"
ncu -i /tmp/prof/${TAG}.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i /tmp/prof/${TAG}.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/${TAG}_src.csv.gz

TAG=$1; MODE=$2
export WALLACE_B200_PAIR_DEBUG=$MODE
mkdir -p /tmp/prof gpurun_out
CMD="python bench.py --config 3 --pools 2048 --steps 1 --warmup 3 --no-cpu --no-e2e --no-configs --no-sustained"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 3 -c 1 -o /tmp/prof/${TAG} -f $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo "rc=$?"
ncu -i /tmp/prof/${TAG}.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i /tmp/prof/${TAG}.ncu-rep --page source --csv --print-source sass > /tmp/prof/${TAG}_src.csv 2>/dev/null
gzip -c /tmp/prof/${TAG}_src.csv > gpurun_out/${TAG}_src.csv.gz

# --set full of one launch of a config's dominant kernel on a 2048-pool job:
# bash tools/dbg/prof_cfg.sh TAG CFG [kernel regex]
TAG=$1; CFG=$2; K=${3:-pool_kernel|pair_kernel}
mkdir -p /tmp/prof gpurun_out
CMD="python bench.py --config $CFG --pools 2048 --steps 1 --warmup 3 --no-cpu --no-e2e --no-configs --no-sustained"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k "regex:$K" -s 4 -c 1 -o /tmp/prof/${TAG} -f $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo "rc=$?"
ncu -i /tmp/prof/${TAG}.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i /tmp/prof/${TAG}.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/${TAG}_src.csv.gz

# ncu --set full captures of the pool kernel for each BASELINE config
# (reduced pool counts: same kernels, one launch per fill), exported on the
# box to CSV (raw metrics + per-instruction source page), gzipped.
#   bash tools/r02_prof.sh TAG "3 2 4 1 5"
TAG=${1:-r02}
CFGS=${2:-"3 2 4 1 5"}
EXTRA=${3:-}
mkdir -p gpurun_out /tmp/prof
for c in $CFGS; do
  case $c in
    1) P="" ;;
    *) P="--pools 2048" ;;
  esac
  CMD="python bench.py --config $c $P --steps 1 --warmup 3 --no-cpu --no-e2e"
  $CMD > gpurun_out/${TAG}_plain_cfg$c.log 2>&1 && \
  $EXTRA ncu --set full --clock-control none --import-source on -k regex:pool_kernel -s 3 -c 1 \
      -o /tmp/prof/${TAG}_cfg$c -f $CMD > gpurun_out/${TAG}_ncu_cfg$c.log 2>&1
  echo "cfg$c rc=$?"
  ncu -i /tmp/prof/${TAG}_cfg$c.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw_cfg$c.csv 2>/dev/null
  ncu -i /tmp/prof/${TAG}_cfg$c.ncu-rep --page source --csv --print-source sass > /tmp/prof/${TAG}_src_cfg$c.csv 2>/dev/null
  gzip -c /tmp/prof/${TAG}_src_cfg$c.csv > gpurun_out/${TAG}_src_cfg$c.csv.gz
done
ls -la gpurun_out/

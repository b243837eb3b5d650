#!/usr/bin/env bash
# Per-kernel duration and DRAM/L2 traffic with the caches as the frame
# pipeline leaves them (--cache-control none, single-pass metric set, so
# the first and only replay sees the real state).  GPU box only.
#   bash tools/ncu_warm.sh <tag> [bench args...]
set -u
TAG=${1:-warm}; shift || true
OUT=gpurun_out
mkdir -p "$OUT"
CMD="python bench.py --steps 3 --warmup 3 --profile-frames 0 --no-cpu-baseline --no-e2e $*"
if $CMD > "$OUT/${TAG}_plain.log" 2>&1; then
  ncu --cache-control none --clock-control none -k regex:"k_(walk|resolve|seg|scatter|update)" --csv \
      --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_write.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active \
      --log-file "$OUT/${TAG}_warm.csv" $CMD > "$OUT/${TAG}_ncu.log" 2>&1
fi

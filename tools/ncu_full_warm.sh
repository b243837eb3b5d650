#!/usr/bin/env bash
# One `ncu --set full` capture of a kernel with the caches as the pipeline
# leaves them (--cache-control none).  GPU box only.
#   bash tools/ncu_full_warm.sh <tag> <kernel-regex> [bench args...]
set -u
TAG=$1; KRE=$2; shift 2
OUT=gpurun_out
mkdir -p "$OUT"
CMD="python bench.py --steps 3 --warmup 3 --profile-frames 0 --no-cpu-baseline --no-e2e $*"
if $CMD > "$OUT/${TAG}_plain.log" 2>&1; then
  ncu --set full --cache-control none --clock-control none --import-source on -k "regex:${KRE}" -s 4 -c 1 \
      -o "$OUT/${TAG}_prof" -f $CMD > "$OUT/${TAG}_ncu.log" 2>&1
fi

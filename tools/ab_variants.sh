#!/usr/bin/env bash
# On the GPU box: kernel spans + wall per frame for every variants/libsvx_*.so
cd "$(dirname "$0")/.."
for lib in variants/libsvx_*.so; do
  v=$(basename "$lib" .so)
  SVX_LIB_PATH=$PWD/$lib python tools/host_overhead.py --frames 30 $AB_ARGS > gpurun_out/ab_$v.txt 2>&1
  echo "$v: $(grep '^kernel spans' gpurun_out/ab_$v.txt | head -1) | $(grep '^config' gpurun_out/ab_$v.txt | head -1 | sed 's/.*integrate wall/wall/;s/, device.*//')"
done

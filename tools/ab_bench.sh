#!/usr/bin/env bash
# On the GPU box: the default bench line (device pass only) for every
# variants/libsvx_*.so, twice each, interleaved.
cd "$(dirname "$0")/.."
for rep in 1 2; do
for lib in variants/libsvx_*.so; do
  v=$(basename "$lib" .so)
  SVX_LIB_PATH=$PWD/$lib timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline $AB_ARGS > gpurun_out/abb_${v}_$rep.json 2>/dev/null
  python3 -c "
import json,sys;d=json.loads(open('gpurun_out/abb_${v}_$rep.json').read().strip().splitlines()[-1]);s=d['stages_ms']
print('%-22s rep $rep  %.1f M/s  step %.4f  p50 %.4f  walk %.4f resolve %.4f update %.4f update_b %.4f frame %.4f e2e %s' % ('$v', d['value']/1e6, d['ms_per_step'], d['ms_per_frame_p50'], s['walk'], s['resolve'], s['update'], s['update_b'], s['frame'], (round(d['e2e']['value']/1e6,1) if d.get('e2e') else None)))"
done; done

#!/usr/bin/env bash
# On the GPU box: per-stage span sums (us) of cfg $CFG frames 0..NF-1 for
# every variants/libsvx_*.so (tools/mode_diag.py), one line per variant.
cd "$(dirname "$0")/.."
CFG=${CFG:-3}; NF=${NF:-10}
for lib in variants/libsvx_*.so; do
  v=$(basename "$lib" .so)
  SVX_LIB_PATH=$PWD/$lib timeout 600 python tools/mode_diag.py --config $CFG --mode auto --frames $NF > gpurun_out/abs_${CFG}_$v.txt 2>&1
  python3 - "$v" gpurun_out/abs_${CFG}_$v.txt <<'PY'
import re, sys
v, f = sys.argv[1], sys.argv[2]
fr = [l for l in open(f) if l.startswith("frame ")]
def g(l, k):
    m = re.search(r" %s ([0-9.]+)" % k, l)
    return float(m.group(1)) if m else 0.0
ks = ["walk", "resolve", "scatter", "update", "update_b", "frame"]
print(f"{v:18s} n {len(fr)} " + " ".join(f"{k} {sum(g(l, k) for l in fr):9.1f}" for k in ks))
PY
done

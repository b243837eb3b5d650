#!/usr/bin/env bash
# On the GPU box: open-set update stage times (cfg3 frames 0-9 by default) for
# every variants/libsvx_*.so; prints per-variant mean update / update_b (us)
# over the normal frames and the total over all frames.
cd "$(dirname "$0")/.."
CFG=${CFG:-3}; NF=${NF:-10}
for lib in variants/libsvx_*.so; do
  v=$(basename "$lib" .so)
  SVX_LIB_PATH=$PWD/$lib timeout 600 python tools/mode_diag.py --config $CFG --mode auto --frames $NF > gpurun_out/abo_$v.txt 2>&1
  python3 - "$v" gpurun_out/abo_$v.txt <<'PY'
import re, sys
v, f = sys.argv[1], sys.argv[2]
fr = [l for l in open(f) if l.startswith("frame ")]
def g(l, k):
    m = re.search(r" %s ([0-9.]+)" % k, l)
    return float(m.group(1)) if m else 0.0
up = [g(l, "update") for l in fr]; ub = [g(l, "update_b") for l in fr]; fs = [g(l, "frame") for l in fr]
print(f"{v:24s} frames {len(fr)}  update sum {sum(up):9.1f}  update_b sum {sum(ub):9.1f}  frame sum {sum(fs):9.1f} us")
PY
done

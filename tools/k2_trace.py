"""K2 (k_resolve) step anatomy on cfg2 frames (GPU box; needs a libsvx built
with -DSVX_RESOLVE_TRACE, e.g. variants/libsvx_trace.so via
tools/build_variants.sh trace=-DSVX_RESOLVE_TRACE):

    SVX_LIB_PATH=$PWD/variants/libsvx_trace.so python tools/k2_trace.py

For the last of a few frames, per CTA and step: phase durations (barrier
entry, hash lookups, bslot atomics, listing rank, writes) and the start /
end of every step relative to the kernel's first stamp.
"""

from __future__ import annotations

import ctypes
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch

    from paper_2512_12945_b200 import Mapper, _lib, scenes

    fn = _lib.lib.svx_debug_resolve_trace
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_void_p, ctypes.c_longlong]
    cap = fn(None, 0)
    wl = scenes.workload(2, device="cuda")
    frames = [wl.make_frame(i) for i in range(12)]
    m = Mapper(**wl.mapper_kwargs)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    buf = np.zeros(cap, dtype=np.uint64)
    for i, f in enumerate(frames):
        flush.zero_()
        torch.cuda.synchronize()
        m.integrate(f.points, f.pose, labels=f.labels).points_used
        torch.cuda.synchronize()
        fn(buf.ctypes.data, cap)
    tr = buf.reshape(2048, 4, 6).astype(np.int64)
    ran = tr[:, :, 0] > 0
    t0 = tr[ran][:, 0].min()
    names = ["enter barrier", "hash+leaf claims", "bslot atomics+claims", "list rank", "writes"]
    print(f"steps traced: {int(ran.sum())} over {int(ran.any(1).sum())} CTAs; kernel stamps span "
          f"{(tr[ran][:, 5].max() - t0) / 1e3:.1f} us")
    for j, nm in enumerate(names):
        d = (tr[:, :, j + 1] - tr[:, :, j])[ran] / 1e3
        print(f"  {nm:22s} median {np.median(d):6.2f} us  p90 {np.percentile(d, 90):6.2f}  max {d.max():6.2f}")
    for s in range(4):
        r = ran[:, s]
        if not r.any():
            continue
        st = (tr[r, s, 0] - t0) / 1e3
        en = (tr[r, s, 5] - t0) / 1e3
        print(f"  step {s}: {int(r.sum())} CTAs, start median {np.median(st):6.2f} us "
              f"[{st.min():.2f}, {st.max():.2f}], end median {np.median(en):6.2f} [{en.min():.2f}, {en.max():.2f}]")
    # CTA first-step start distribution (launch / PDL wait / second wave)
    first = (tr[ran.any(1), 0, 0] - t0) / 1e3
    print("  first-step start percentiles (us):", [round(float(np.percentile(first, q)), 2) for q in (0, 10, 50, 75, 90, 100)])


if __name__ == "__main__":
    main()

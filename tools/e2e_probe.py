"""Anatomy of the bench's e2e step (GPU box only).

    SVX_TRACE_HOST=1 python tools/e2e_probe.py [--config 2] [--frames 20]

Per step, as bench.py's e2e pass: L2 flush, then CUDA events around
Mapper.integrate on pinned host arrays plus the read of the report; prints
the event time, the host time of the call (H2D copy enqueue + wait, graph
launch) and of the report read (wait for the frame).
"""

from __future__ import annotations

import argparse
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--frames", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    args = ap.parse_args()
    import torch

    from paper_2512_12945_b200 import Mapper, scenes

    wl = scenes.workload(args.config, device="cuda")
    n = args.warmup + args.frames
    frames = [wl.make_frame(i % wl.n_frames) for i in range(n)]
    host = []
    for f in frames:
        p = torch.empty(f.points.shape, dtype=f.points.dtype, pin_memory=True)
        p.copy_(f.points)
        lab = None
        if f.labels is not None:
            lab = torch.empty(f.labels.shape, dtype=f.labels.dtype, pin_memory=True)
            lab.copy_(f.labels)
        host.append((p.numpy(), None if lab is None else lab.numpy()))
    m = Mapper(**wl.mapper_kwargs)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    rows = []
    for i, (f, (p, lab)) in enumerate(zip(frames, host)):
        flush.fill_(i & 255)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        t0 = time.perf_counter()
        r = m.integrate(p, f.pose, labels=lab)
        t1 = time.perf_counter()
        used = r.points_used
        t2 = time.perf_counter()
        b.record(s)
        b.synchronize()
        ev = a.elapsed_time(b)
        if i >= args.warmup:
            rows.append((ev, 1e3 * (t1 - t0), 1e3 * (t2 - t1), r.kernel_ms))
        print(f"step {i}: event {ev:.4f} ms  call {1e3 * (t1 - t0):.4f} ms  report {1e3 * (t2 - t1):.4f} ms  "
              f"kernel_ms {r.kernel_ms:.4f}  used {used}", flush=True)
    med = [statistics.median(c) for c in zip(*rows)]
    print("median: event %.4f call %.4f report %.4f kernel_ms %.4f" % tuple(med))


if __name__ == "__main__":
    main()

"""Where a depth frame's step time goes (GPU box only).

    SVX_TRACE_HOST=1 python tools/depth_overhead.py [--config 3] [--frames 10]

Per frame: the bench's step (CUDA events around Mapper.integrate_depth on the
current stream, L2 flushed before), the wall time of the Python call, and
the library's device time (report.kernel_ms); with SVX_TRACE_HOST the
library prints its own host spans to stderr.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--frames", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    import torch

    from paper_2512_12945_b200 import Mapper, scenes

    wl = scenes.workload(args.config, device="cuda")
    n = args.warmup + args.frames
    frames = [wl.make_frame(i % wl.n_frames) for i in range(n)]
    m = Mapper(**wl.mapper_kwargs)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    for i, f in enumerate(frames):
        h, w = f.camera["height"], f.camera["width"]
        pay = f.labels.reshape(h, w) if f.features is None else f.features.reshape(h, w, -1)
        flush.fill_(i & 255)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        t0 = time.perf_counter()
        r = m.integrate_depth(f.depth, pay, f.camera, pose=f.pose)
        t1 = time.perf_counter()
        b.record(s)
        b.synchronize()
        print(f"frame {i}: step {a.elapsed_time(b):.3f} ms  python wall {1e3 * (t1 - t0):.3f} ms  "
              f"kernel_ms {r.kernel_ms:.3f}  used {r.points_used}", flush=True)
        print(f"frame {i} --", file=sys.stderr, flush=True)


if __name__ == "__main__":
    main()

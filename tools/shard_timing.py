"""Loopback timing of the sharded frame plans on one GPU.

    python tools/shard_timing.py [--config 2] [--frames 12] [--G 1 2 4 8]

G in-process shards integrate the same BASELINE frames through
``integrate_loopback`` in the host plan (sizes, headers and reports read back
after each phase) and in the device plan (one host synchronisation per frame,
svx_shard_*_async).  All shards share the GPU, so a frame's time is the sum of
the G ranks' kernels plus the host work between them; the growth with G is the
per-rank overhead a real G-GPU run pays once per rank (its kernels then run in
parallel).  Prints one JSON line per (G, plan): ms per frame (median, wall
clock around the frame with a device synchronisation on both sides), host
synchronisations per frame, and the bytes each rank sent.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--frames", type=int, default=12)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--G", type=int, nargs="+", default=[1, 2, 4, 8])
    args = ap.parse_args()
    import torch

    from paper_2512_12945_b200 import scenes
    from paper_2512_12945_b200.sharded import ShardedMapper, integrate_loopback

    wl = scenes.workload(args.config, device="cuda")
    kw = dict(wl.mapper_kwargs)
    frames = [wl.make_frame(i) for i in range(args.warmup + args.frames)]
    for G in args.G:
        for plan in (False, True):
            shards = [ShardedMapper(rank=r, world=G, **kw) for r in range(G)]
            ms, syncs = [], []
            for i, f in enumerate(frames):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                integrate_loopback(shards, f.points_world, origin=f.origin, labels=f.labels,
                                   features=f.features, device_plan=plan)
                torch.cuda.synchronize()
                if i >= args.warmup:
                    ms.append((time.perf_counter() - t0) * 1e3)
                    syncs.append(shards[0].host_syncs if plan else None)
            print(json.dumps({
                "config": f"cfg{args.config}", "G": G, "plan": "device" if plan else "host",
                "ms_per_frame": round(statistics.median(ms), 3),
                "points_per_frame": int(frames[0].points_world.shape[0]),
                "host_syncs_per_frame": (statistics.median(syncs) if plan else "~7 (march, summary, plan, "
                                         "sizes, headers, report, report sum)"),
                "section_cap_bytes": shards[0]._cap if plan else None,
                "timing": "wall clock per frame, torch.cuda.synchronize before and after; G shards on one GPU",
            }), flush=True)
            del shards


if __name__ == "__main__":
    main()

"""Per-frame device times and stage spans of a workload (GPU box only).

    python tools/frame_times.py --config 3 [--depth] [--frames 20]
"""

from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--depth", action="store_true")
    ap.add_argument("--frames", type=int, default=20)
    args = ap.parse_args()
    import torch

    from paper_2512_12945_b200 import Mapper, scenes

    wl = scenes.workload(args.config, device="cuda")
    m = Mapper(**wl.mapper_kwargs)
    m.set_profiling(True)
    for i in range(args.frames):
        f = wl.make_frame(i % wl.n_frames)
        torch.cuda.synchronize()
        if args.depth:
            pay = f.labels.reshape(f.depth.shape) if f.labels is not None else \
                f.features.reshape(f.depth.shape[0], f.depth.shape[1], -1)
            r = m.integrate_depth(f.depth, pay, f.camera, f.pose)
        elif f.features is not None:
            r = m.integrate_world(f.points_world, f.origin, features=f.features)
        else:
            r = m.integrate(f.points, f.pose, labels=f.labels)
        st = m.stage_times()
        es = m.engine_stats()
        print(f"frame {i:3d} kernel_ms {r.kernel_ms:8.3f} touched {r.touched_voxels:8d} "
              f"band {r.band_hits:9d} " + " ".join(f"{k} {v:.3f}" for k, v in st.items())
              + f" reruns {es.get('slot_overflow_reruns', 0)}", flush=True)


if __name__ == "__main__":
    main()

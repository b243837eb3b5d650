"""Ray-march rendering (render / Mapper.render) throughput on one GPU.

    python tools/bench_render.py [--config 2] [--frames 20] [--width 640 --height 480]

Integrates `frames` frames of a BASELINE workload, then renders the map from
the last sensor pose (looking forward, slightly down) and times, per mode:
  * gpu_ms -- svx_render into a device buffer (CUDA events)
  * e2e_ms -- Mapper.render as a user calls it (numpy image out)
  * reference_ms -- the reference's own render (baseline/_ref, numpy) on the
    same map read back from this map's .slvg snapshot, once per mode
and checks the images are identical.  One JSON line per mode.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import tempfile
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--frames", type=int, default=20)
    ap.add_argument("--width", type=int, default=640)
    ap.add_argument("--height", type=int, default=480)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--no-ref", action="store_true")
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_2512_12945_b200 import Mapper, RenderCamera, scenes
    from paper_2512_12945_b200._lib import check, lib
    from paper_2512_12945_b200.render import _MODE_CODE
    from paper_2512_12945_b200.surface import default_palette

    wl = scenes.workload(args.config, device="cuda")
    kw = dict(wl.mapper_kwargs)
    m = Mapper(**kw)
    f = None
    for i in range(args.frames):
        f = wl.make_frame(i % wl.n_frames)
        if f.features is not None:
            m.integrate_world(f.points_world, f.origin, features=f.features)
        else:
            m.integrate(f.points, f.pose, labels=f.labels)
    pose = np.asarray(f.pose, np.float64).copy()
    if args.config in (2, 4):          # LiDAR: sensor +x forward -> camera +z
        c, s = np.cos(0.2), np.sin(0.2)
        pose[:3, :3] = pose[:3, :3] @ np.array([[0, -s, c], [-1, 0, 0], [0, -c, -s]], np.float64)
        pose[2, 3] += 0.5
    W, H = args.width, args.height
    cam = RenderCamera(pose=pose, fx=0.8 * W, fy=0.8 * W, cx=W / 2.0, cy=H / 2.0, width=W,
                       height=H, near=0.1, far=40.0 if args.config in (2, 4) else 8.0)
    cam.validate()
    ref = None
    if not args.no_ref and os.path.isdir(os.path.join(REPO, "baseline", "_ref", "semvox")):
        sys.path.insert(0, os.path.join(REPO, "baseline", "_ref"))
        import semvox

        with tempfile.TemporaryDirectory() as td:
            p = os.path.join(td, "m.slvg")
            m.save(p)
            grids = semvox.load_grids(p)
        ref = (semvox, grids[0], grids[1] if len(grids) > 1 else None)
    P = kw.get("num_classes") or kw.get("feature_dim") or 1
    pal = default_palette(P)
    for mode in ("depth", "semantic", "normal"):
        if mode == "semantic" and m.sem_kind is None:
            continue
        nbytes = W * H * (8 if mode == "depth" else 24 if mode == "normal" else 3)
        out = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        c = cam._c()

        def gpu():
            check(lib.svx_render(m._handle, ctypes.byref(c), _MODE_CODE[mode], None, 0, 0.0, 0.0,
                                 pal.ctypes.data, pal.shape[0], out.data_ptr(), None))

        gpu()
        torch.cuda.synchronize()
        g_ms, e_ms = [], []
        img = None
        for _ in range(args.reps):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            gpu()
            b.record()
            b.synchronize()
            g_ms.append(a.elapsed_time(b))
            t0 = time.perf_counter()
            img = m.render(cam, mode=mode)
            e_ms.append((time.perf_counter() - t0) * 1e3)
        rec = {"metric": "render", "mode": mode, "config": f"cfg{args.config}",
               "frames": args.frames, "active_voxels": m.active_count(), "width": W,
               "height": H, "hit_pixels": int((img.reshape(H * W, -1) != 0).any(axis=1).sum()),
               "gpu_ms": statistics.median(g_ms), "e2e_ms": statistics.median(e_ms),
               "gpu_fps": 1e3 / statistics.median(g_ms),
               "timing": "gpu_ms: CUDA events around svx_render (device output); e2e_ms: wall "
                         "time of Mapper.render into numpy"}
        if ref is not None:
            sv, rt, rs = ref
            rc = sv.RenderCamera(pose=cam.pose.copy(), fx=cam.fx, fy=cam.fy, cx=cam.cx, cy=cam.cy,
                                 width=W, height=H, near=cam.near, far=cam.far)
            t0 = time.perf_counter()
            rimg = sv.render(rt, rs, rc, mode=mode)
            rec["reference_ms"] = (time.perf_counter() - t0) * 1e3
            rec["identical"] = bool(np.array_equal(rimg, img))
            rec["speedup_e2e_vs_reference"] = rec["reference_ms"] / rec["e2e_ms"]
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()

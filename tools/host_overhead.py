"""Where a frame's wall time goes on the host side (GPU box only).

    python tools/host_overhead.py [--config 2] [--frames 30]

Prints, per frame averaged over the timed frames: wall time of
Mapper.integrate, the library's own device time (report.kernel_ms: events
around the frame inside svx_integrate), the time of the raw C call
(svx_integrate through ctypes, no Python validation), and the Python
argument handling alone.
"""

from __future__ import annotations

import argparse
import ctypes
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--frames", type=int, default=30)
    ap.add_argument("--mode", default="auto")
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_2512_12945_b200 import Mapper, _lib, scenes
    from paper_2512_12945_b200.mapper import _check_pose

    wl = scenes.workload(args.config, device="cuda")
    frames = [wl.make_frame(i % wl.n_frames) for i in range(args.frames + 5)]
    m = Mapper(**wl.mapper_kwargs)
    m.set_update_mode(args.mode)
    for f in frames[:5]:
        m.integrate(f.points, f.pose, labels=f.labels)
    st = m.engine_stats()
    m.reserve(st["active_voxels"] * 4, st["leaf_count"] * 4)
    torch.cuda.synchronize()
    wall, dev = [], []
    for f in frames[5:]:
        t0 = time.perf_counter()
        r = m.integrate(f.points, f.pose, labels=f.labels)
        wall.append((time.perf_counter() - t0) * 1e3)
        dev.append(r.kernel_ms)
    # python-side argument handling only
    py = []
    for f in frames[5:]:
        t0 = time.perf_counter()
        pts = m._points_arg(f.points)
        pose = _check_pose(f.pose, 0)
        m._payload_args(int(pts.shape[0]), f.labels, None, 0)
        py.append((time.perf_counter() - t0) * 1e3)
    # raw C call on a second map
    m2 = Mapper(**wl.mapper_kwargs)
    m2.set_update_mode(args.mode)
    for f in frames[:5]:
        m2.integrate(f.points, f.pose, labels=f.labels)
    m2.reserve(st["active_voxels"] * 4, st["leaf_count"] * 4)
    lib = _lib.lib
    raw = []
    rep = _lib.SvxReport()
    for f in frames[5:]:
        pose = np.ascontiguousarray(np.asarray(f.pose, np.float64).reshape(-1))
        pp = pose.ctypes.data
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _lib.check(lib.svx_integrate(m2._handle, f.points.data_ptr(), _lib.DEVICE_INPUTS,
                                     f.points.shape[0], pp,
                                     f.labels.data_ptr(), None, 0, None, ctypes.byref(rep)))
        raw.append((time.perf_counter() - t0) * 1e3)
    med = statistics.median
    # kernel spans inside the frame graph (profiling mode)
    m.set_profiling(True)
    spans = []
    for f in frames[5:]:
        m.integrate(f.points, f.pose, labels=f.labels)
        spans.append(m.stage_times())
    m.set_profiling(False)
    # pinned host inputs (the e2e path): spans and wall
    hp = []
    for f in frames[5:]:
        pt = torch.empty(f.points.shape, dtype=f.points.dtype, pin_memory=True)
        pt.copy_(f.points)
        lb = torch.empty(f.labels.shape, dtype=f.labels.dtype, pin_memory=True)
        lb.copy_(f.labels)
        hp.append((pt.numpy(), lb.numpy()))
    m.set_profiling(True)
    hspans, hwall = [], []
    for f, (pt, lb) in zip(frames[5:], hp):
        t0 = time.perf_counter()
        m.integrate(pt, f.pose, labels=lb)
        hwall.append((time.perf_counter() - t0) * 1e3)
        hspans.append(m.stage_times())
    print("pinned host inputs: wall %.4f ms; kernel spans (median us): " % med(hwall) + ", ".join(
        f"{k} {1e3 * med([sp[k] for sp in hspans]):.1f}" for k in _lib.STAGES))
    print("kernel spans (median us): " + ", ".join(
        f"{k} {1e3 * med([sp[k] for sp in spans]):.1f}" for k in _lib.STAGES))
    print(f"config {args.config} mode {args.mode}: per frame (median ms) "
          f"integrate wall {med(wall):.4f}, device (kernel_ms) {med(dev):.4f}, "
          f"raw C call {med(raw):.4f}, python arg handling {med(py):.4f}; "
          f"slot frames {m.engine_stats()['frames_slot_mode']}")


if __name__ == "__main__":
    main()

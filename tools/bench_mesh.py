"""Surface extraction (Mapper.extract) throughput on one GPU.

    python tools/bench_mesh.py [--config 2] [--frames 20] [--reps 10]

Integrates `frames` frames of a BASELINE workload, then times:
  * gpu_ms   -- svx_extract_mesh alone (CUDA events; mesh stays on the device)
  * e2e_ms   -- Mapper.extract as a user calls it (extraction + copies of
               vertices / triangles / labels / colours into numpy arrays)
  * reference_ms -- the reference's own extract_mesh (baseline/_ref, numpy)
               on the same map, read back from this map's .slvg snapshot
  * oracle_ms -- the oracle restatement (numpy) on the exported map
and checks the three meshes are identical.  One JSON line.
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
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import numpy as np
    import torch

    from oracle import mesh as om
    from paper_2512_12945_b200 import Mapper, _lib, scenes

    wl = scenes.workload(args.config, device="cuda")
    kw = dict(wl.mapper_kwargs)
    m = Mapper(**kw)
    for i in range(args.frames):
        f = wl.make_frame(i % wl.n_frames)
        if f.features is not None:
            m.integrate_world(f.points_world, f.origin, features=f.features)
        else:
            m.integrate(f.points, f.pose, labels=f.labels)
    lib = _lib.lib
    nv, nt = ctypes.c_int64(), ctypes.c_int64()

    def gpu():
        _lib.check(lib.svx_extract_mesh(m._handle, 0.5, None, 0, 0.0, 0.0, ctypes.byref(nv),
                                        ctypes.byref(nt), None))

    for _ in range(2):
        gpu()
    torch.cuda.synchronize()
    g_ms, e_ms = [], []
    for _ in range(args.reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        gpu()
        b.record()
        b.synchronize()
        g_ms.append(a.elapsed_time(b))
        t0 = time.perf_counter()
        mesh = m.extract()
        e_ms.append((time.perf_counter() - t0) * 1e3)
    out = {"metric": "mesh extraction", "config": f"cfg{args.config}", "frames": args.frames,
           "active_voxels": m.active_count(), "vertices": mesh.n_vertices,
           "triangles": mesh.n_triangles, "gpu_ms": statistics.median(g_ms),
           "e2e_ms": statistics.median(e_ms),
           "timing": "gpu_ms: CUDA events around svx_extract_mesh (host syncs for the "
                     "allocation sizes included); e2e_ms: wall time of Mapper.extract"}
    coords, d, w, s0, _ = m._export()
    psize = kw.get("num_classes") or kw.get("feature_dim") or 1
    t0 = time.perf_counter()
    want = om.extract(coords, d, w, kw["voxel_size"], 0.5, m.sem_kind, s0, palette_size=psize)
    out["oracle_ms"] = (time.perf_counter() - t0) * 1e3
    same = all(np.array_equal(a, b) for a, b in
               zip((mesh.vertices, mesh.triangles, mesh.labels, mesh.colors), want))
    ref = os.path.join(REPO, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "semvox")):
        sys.path.insert(0, ref)
        from semvox import extract_mesh, load_grids

        with tempfile.TemporaryDirectory() as td:
            p = os.path.join(td, "m.slvg")
            m.save(p)
            grids = load_grids(p)
        tsdf = grids[0]
        sem = grids[1] if len(grids) > 1 else None
        t0 = time.perf_counter()
        rm = extract_mesh(tsdf, sem, min_weight=0.5)
        out["reference_ms"] = (time.perf_counter() - t0) * 1e3
        same = same and all(np.array_equal(a, b) for a, b in
                            zip((mesh.vertices, mesh.triangles, mesh.labels, mesh.colors),
                                (rm.vertices, rm.triangles, rm.labels, rm.colors)))
        out["speedup_e2e_vs_reference"] = out["reference_ms"] / out["e2e_ms"]
    out["identical"] = bool(same)
    print(json.dumps(out))


if __name__ == "__main__":
    main()

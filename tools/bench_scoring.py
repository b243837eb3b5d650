"""Open-set query scoring (classify_means) throughput on one GPU.

    python tools/bench_scoring.py [--config 3|5] [--frames N] [--reps R]

Builds an open-set map from the BASELINE depth-camera workload (cfg3: D=512,
32 queries; cfg5: D=768, 128 queries), then times svx_classify with device
output buffers (CUDA events around the call, which includes the active-list
build).  Prints one JSON line: voxels scored per second, f64 GFLOP/s of the
scoring GEMM (2*V*D*k) and its fraction of the B200's nominal FP64 tensor-core
peak (40 TFLOP/s; the DMMA path), and the kernel's span.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

FP64_TENSOR_PEAK_TFLOPS = 40.0   # B200 nominal FP64 / FP64 tensor core


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--frames", type=int, default=4)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--path", default="auto", choices=["auto", "dmma", "tcgen05"])
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_2512_12945_b200 import Mapper, _lib, scenes

    wl = scenes.workload(args.config, device="cuda")
    kw = dict(wl.mapper_kwargs)
    D = kw["feature_dim"]
    k = 32 if args.config == 3 else 128
    m = Mapper(**kw)
    m.set_score_path(args.path)
    for i in range(args.frames):
        f = wl.make_frame(i * max(1, wl.n_frames // args.frames))
        m.integrate_world(f.points_world, f.origin, features=f.features)
    rng = np.random.default_rng(0)
    emb = rng.normal(size=(k, D))
    emb /= np.linalg.norm(emb, axis=1, keepdims=True)
    V = m.active_count()
    lab = torch.empty(V, dtype=torch.int32, device="cuda")
    best = torch.empty(V, dtype=torch.float64, device="cuda")
    embc = np.ascontiguousarray(emb)
    lib = _lib.lib

    def run():
        _lib.check(lib.svx_classify(m._handle, embc.ctypes.data, k, 0.01, 0.1, V, lab.data_ptr(),
                                    best.data_ptr(), None, None))

    for _ in range(2):
        run()
    torch.cuda.synchronize()
    ms = []
    for _ in range(args.reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        b.record()
        b.synchronize()
        ms.append(a.elapsed_time(b))
    t = statistics.median(ms) / 1e3
    flops = 2.0 * V * D * k
    print(json.dumps({
        "metric": "open-set voxels scored/sec", "config": f"cfg{args.config}",
        "voxels": V, "feature_dim": D, "queries": k, "ms": t * 1e3,
        "value": V / t, "gflops_f64": flops / t / 1e9,
        "frac_of_fp64_tensor_peak": flops / t / 1e12 / FP64_TENSOR_PEAK_TFLOPS,
        "peak_source": "nominal B200 FP64 tensor core 40 TFLOP/s",
        "path": ("tcgen05.mma.kind::i8 exact split GEMM (7 byte planes per operand, 34 plane pairs, "
                 "int32 TMEM accumulators) + softmax kernel"
                 if (args.path == "tcgen05" or (args.path == "auto" and k > 64))
                 else "mma.sync.m8n8k4.f64 (DMMA) fused GEMM + softmax epilogue"),
        "timing": "CUDA events around svx_classify (includes the active-list build)",
    }))


if __name__ == "__main__":
    main()

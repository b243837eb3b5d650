"""Open-set query scoring (classify_means) throughput on one GPU.

    python tools/bench_scoring.py [--config 3|5] [--frames N] [--reps R]

Builds an open-set map from the BASELINE depth-camera workload (cfg3: D=512,
32 queries; cfg5: D=768, 128 queries), then times svx_classify with device
output buffers (CUDA events around the call, which includes the active-list
build).  Prints one JSON line: voxels scored per second, the f64-equivalent
GFLOP/s of the scoring GEMM (2*V*D*k), and against measured peaks: the DMMA
path's fraction of the FP64 tensor rate, the tcgen05 path's int8 TOP/s (34
plane-pair GEMMs) against the dense int8 rate and the N=64 shared-memory rate.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

# measured on this pool's B200 by tools/tc_peaks.py (profiles/r02_tensor_peaks_measured.json)
FP64_TENSOR_PEAK_TFLOPS = 37.17   # mma.sync.m8n8k4.f64
I8_DENSE_PEAK_TOPS = 4494.9       # tcgen05 kind::i8, M=128 N=256 (tensor-bound)
I8_SS_N64_TOPS = 2893.9           # the scoring kernel's shape: N=64, both operands in smem (48 cycles/MMA)


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
    tc = args.path == "tcgen05" or (args.path == "auto" and k > 64)
    out = {
        "metric": "open-set voxels scored/sec", "config": f"cfg{args.config}",
        "voxels": V, "feature_dim": D, "queries": k, "ms": t * 1e3,
        "value": V / t, "gflops_f64_equiv": flops / t / 1e9,
        "timing": "CUDA events around svx_classify (includes the active-list build)",
    }
    if tc:
        tn = 32 if k <= 32 else 64
        kp = -(-k // tn) * tn
        dp = max(2, -(-D // 64)) * 64
        i8 = 34 * 2.0 * (-(-V // 128) * 128) * kp * dp   # 34 byte-plane pair GEMMs
        out.update({
            "path": "tcgen05.mma.kind::i8 exact split GEMM (7 byte planes per operand, 34 plane pairs, "
                    "int32 TMEM accumulators)" + (" + fused softmax" if k <= 32 else " + softmax kernel"),
            "int8_tops": i8 / t / 1e12,
            "frac_of_i8_dense_peak": i8 / t / 1e12 / I8_DENSE_PEAK_TOPS,
            "frac_of_i8_ss_n64_rate": i8 / t / 1e12 / I8_SS_N64_TOPS,
            "peak_source": "measured, profiles/r02_tensor_peaks_measured.json (whole call incl. prep and softmax)",
        })
    else:
        out.update({
            "path": "mma.sync.m8n8k4.f64 (DMMA) fused GEMM + softmax epilogue",
            "frac_of_fp64_tensor_peak": flops / t / 1e12 / FP64_TENSOR_PEAK_TFLOPS,
            "peak_source": "measured DMMA 37.17 TFLOP/s, profiles/r02_tensor_peaks_measured.json",
        })
    print(json.dumps(out))

if __name__ == "__main__":
    main()

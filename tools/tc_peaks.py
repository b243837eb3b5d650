"""Measured tensor-core rates for the scoring roofline (tools/tc_peaks.cu).

    python tools/tc_peaks.py          # on a GPU box; builds variants/libtcpeaks.so first

Prints one JSON line: FP64 tensor (DMMA) and FP64 FMA TFLOP/s, and the
tcgen05 kind::i8 dense rate and cycles per MMA for N = 32..256 with both
operands in shared memory (the scoring kernel's SS mode).
"""

from __future__ import annotations

import ctypes
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "variants", "libtcpeaks.so")


def main():
    if not os.path.exists(SO):
        os.makedirs(os.path.dirname(SO), exist_ok=True)
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                               "-Xcompiler", "-fPIC", os.path.join(ROOT, "tools", "tc_peaks.cu"), "-o", SO])
    lib = ctypes.CDLL(SO)
    lib.dmma_peak.restype = ctypes.c_double
    lib.dfma_peak.restype = ctypes.c_double
    lib.i8_rate.restype = ctypes.c_double
    lib.i8_rate.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
    out = {"dmma_fp64_tflops": round(lib.dmma_peak(20000), 2),
           "dfma_fp64_tflops": round(lib.dfma_peak(200000), 2), "i8": {}}
    for n in (32, 64, 128, 256):
        cyc = ctypes.c_double()
        tops = lib.i8_rate(n, 20000, ctypes.byref(cyc))
        out["i8"][f"N{n}"] = {"tops": round(tops, 1), "cycles_per_mma": round(cyc.value, 1)}
    out["how"] = ("DMMA: mma.sync.m8n8k4.f64, 8 independent chains per warp, 148x8 CTAs x 256 threads; DFMA: 8 "
                  "chains per thread; i8: one CTA per SM, one elected lane issuing back-to-back "
                  "tcgen05.mma.cta_group::1.kind::i8 M=128 K=32 with both operands in shared memory "
                  "(64B swizzle), CUDA events around the launch, clock64 per CTA for cycles per MMA")
    print(json.dumps(out))


if __name__ == "__main__":
    main()

"""Run the tcgen05 int8 MMA probe (tools/tc_probe.cu) and compare with numpy."""
import ctypes
import os
import sys

import numpy as np

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                               "variants", "libtcprobe.so"))
rng = np.random.default_rng(0)
for n in (32, 64):
    A = rng.integers(-64, 65, (128, 64)).astype(np.int8)
    B = rng.integers(-64, 65, (n, 64)).astype(np.int8)
    C = np.zeros((128, n), np.int32)
    rc = lib.tc_probe(A.ctypes.data, B.ctypes.data, C.ctypes.data, n)
    ref = A.astype(np.int64) @ B.astype(np.int64).T
    ok = np.array_equal(C, ref)
    print(f"n={n} rc={rc} exact={ok} max|diff|={np.abs(C - ref).max()}", flush=True)
    if not ok:
        bad = np.argwhere(C != ref)
        print(bad[:10], C[bad[0][0], :8], ref[bad[0][0], :8])
        sys.exit(1)

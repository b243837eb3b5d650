"""CPU restatement of the reference's ray-march renderer -- TEST
INFRASTRUCTURE ONLY (imported by tests/ as the checker; never by the
product path).

Follows render.py (pkg/src/semvox/render.py) one ray at a time in plain
Python floats (IEEE double, the same roundings as numpy's elementwise ops):
  * RenderCamera.rays (:70-85): ((u + .5 - cx) / fx, (v + .5 - cy) / fy, 1)
    over its norm, then `@ R.T` -- numpy hands the (H*W, 3) @ (3, 3) product
    to OpenBLAS dgemm, which fuses k = 0, 1, 2 from the k = 0 product (a
    1x1 image takes the one-row path: k = 1 product, then k = 0, k = 2);
  * sample_distance (:88-113), _skip_empty_leaves (:116-131), _march
    (:134-176), _refine (:179-211) and render's depth / normal / semantic
    outputs (:214-272), labels as voxel_labels (mesh.py:392-416).
Small images only (pure-Python loops).  Open-set labels by embeddings are
not restated here (they need classify_means; the GPU tests pin them to the
reference's own images).
"""

from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

from .mesh import default_palette


def _fma(a, b, c):
    return float(Fraction(a) * Fraction(b) + Fraction(c))


class VoxelState:
    """Active voxels of a map: coords (n, 3) -> d, plus per-voxel semantic rows."""

    def __init__(self, coords, d, w, voxel_size, truncation, kind=None, rows=None):
        coords = np.asarray(coords, np.int64)
        self.vox = {tuple(int(v) for v in c): i for i, c in enumerate(coords)}
        self.leaves = {(c[0] >> 3, c[1] >> 3, c[2] >> 3) for c in self.vox}
        self.d = [float(x) for x in np.asarray(d, np.float64)]
        self.w = [float(x) for x in np.asarray(w, np.float64)]
        self.h = float(voxel_size)
        self.trunc = float(truncation)
        self.kind = kind
        self.rows = None if rows is None else np.asarray(rows, np.float64)

    def sample(self, p):
        h = self.h
        q = [p[0] / h - 0.5, p[1] / h - 0.5, p[2] / h - 0.5]
        base = [math.floor(x) for x in q]
        frac = [q[k] - float(base[k]) for k in range(3)]
        val = 0.0
        for c in range(8):
            off = ((c >> 2) & 1, (c >> 1) & 1, c & 1)
            i = self.vox.get((base[0] + off[0], base[1] + off[1], base[2] + off[2]))
            if i is None:
                return math.nan, False
            w = 1.0
            for ax in range(3):
                w *= frac[ax] if off[ax] else 1.0 - frac[ax]
            val += w * self.d[i]
        return val, True

    def label(self, coord):
        i = self.vox.get(coord)
        if i is None or self.kind is None:
            return 0
        row = self.rows[i]
        arg = int(np.argmax(row))
        if self.kind == "closed":
            return 0 if row.sum() <= 0.0 else arg + 1
        return 0 if np.abs(row).sum() == 0.0 else arg + 1


def rays(pose, fx, fy, cx, cy, width, height):
    pose = np.asarray(pose, np.float64)
    R = [[float(pose[r, c]) for c in range(3)] for r in range(3)]
    o = [float(pose[r, 3]) for r in range(3)]
    single = width * height == 1
    out = []
    for v in range(height):
        for u in range(width):
            a = ((float(u) + 0.5) - cx) / fx
            b = ((float(v) + 0.5) - cy) / fy
            n = math.sqrt((a * a + b * b) + 1.0 * 1.0)
            dc = (a / n, b / n, 1.0 / n)
            d = []
            for r in range(3):
                acc = (_fma(R[r][0], dc[0], R[r][1] * dc[1]) if single
                       else _fma(R[r][1], dc[1], R[r][0] * dc[0]))
                d.append(_fma(R[r][2], dc[2], acc))
            out.append((o, d))
    return out


def _point(o, d, t):
    return [o[0] + t * d[0], o[1] + t * d[1], o[2] + t * d[2]]


def march(st, o, d, near, far):
    h = st.h
    step = 0.5 * h
    t, prev_d, prev_ok = float(near), 0.0, False
    while True:
        p = _point(o, d, t)
        vox = [math.floor(x / h) for x in p]
        lc = [v >> 3 for v in vox]
        if tuple(lc) not in st.leaves:
            t_exit = math.inf
            for k in range(3):
                if d[k] != 0.0:
                    e1 = (float(lc[k] << 3) * h - o[k]) / d[k]
                    e2 = (float((lc[k] + 1) << 3) * h - o[k]) / d[k]
                    t_exit = min(t_exit, max(e1, e2))
            t += max(step, (t_exit - t) + 1e-3 * h)
            prev_ok = False
        else:
            dv, ok = st.sample(p)
            if ok and prev_ok and prev_d > 0.0 and dv <= 0.0:
                return _refine(st, o, d, t - step, prev_d, t, dv)
            prev_ok, prev_d = ok, dv
            t += step
        if not t <= far:
            return None


def _refine(st, o, d, at, ad, bt, bd):
    tol = 1e-4 * st.trunc
    best = bt
    for _ in range(32):
        tm = bt - bd * (bt - at) / (bd - ad)
        dm, ok = st.sample(_point(o, d, tm))
        if not ok:
            dm = 0.0
        best = tm
        if not ok or abs(dm) < tol:
            break
        if dm > 0.0:
            at, ad = tm, dm
        else:
            bt, bd = tm, dm
    return best


def render(st, pose, fx, fy, cx, cy, width, height, near=0.05, far=10.0, mode="depth",
           palette=None, palette_size=1):
    h = st.h
    shape = (height, width) if mode == "depth" else (height, width, 3)
    out = np.zeros(shape, np.float64 if mode != "semantic" else np.uint8)
    flat = out.reshape(height * width, -1)
    pal = default_palette(palette_size) if palette is None else np.asarray(palette, np.uint8)
    for i, (o, d) in enumerate(rays(pose, fx, fy, cx, cy, width, height)):
        th = march(st, o, d, near, far)
        if th is None:
            continue
        p = _point(o, d, th)
        if mode == "depth":
            flat[i, 0] = th
        elif mode == "normal":
            g = [0.0, 0.0, 0.0]
            ok = True
            for ax in range(3):
                pp = list(p)
                pp[ax] = p[ax] + 0.5 * h
                dp, okp = st.sample(pp)
                pp[ax] = p[ax] - 0.5 * h
                dn, okn = st.sample(pp)
                ok = ok and okp and okn
                g[ax] = dp - dn if (okp and okn) else 0.0
            nrm = math.sqrt((g[0] * g[0] + g[1] * g[1]) + g[2] * g[2])
            ok = ok and nrm > 0.0
            flat[i] = [x / nrm for x in g] if ok else [0.0, 0.0, 0.0]
        else:
            near_vox = tuple(int(round(x / h - 0.5)) for x in p)
            lab = st.label(near_vox)
            row = 1 + (lab - 1) % (pal.shape[0] - 1) if lab > 0 else 0
            flat[i] = pal[row]
    return out

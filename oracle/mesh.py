"""CPU restatement of the reference's zero-level surface extraction -- TEST
INFRASTRUCTURE ONLY (imported by tests/ as the checker; never by the
product path).

Follows extract_mesh (pkg/src/semvox/mesh.py:419-545) and voxel_labels
(mesh.py:392-416) step for step on a map state given as arrays (active
coords, d, w, semantic rows), in numpy:

  1. keep voxels with w >= min_weight (mesh.py:452-456);
  2. bound the kept extent to 2^20 per axis, pack relative coords into a
     60-bit spatial key and sort by it (:458-476);
  3. a cell per kept voxel whose 7 +x/+y/+z neighbours are kept (:478-491);
     case bit c = d(corner c) < 0, live when some edge changes sign (:493-499);
  4. one vertex per (lower voxel, axis) edge of a live cell, numbered in key
     order, at (lower + 0.5) h + t h along the axis, t = d_lo / (d_lo - d_hi)
     (:501-513);
  5. table triangles per live cell, reversed, without zero-area ones (:515-535);
  6. drop vertices no triangle uses, renumber (:537-540); label each vertex
     from the nearer edge end (t < 0.5 -> lower), colour by palette row
     (:542-556, palette_colors :382-389).

The 256-case triangle table is read from the engine's packed copy
(csrc/svx_mesh.cu, c_tri); its correctness is pinned by the reference-made
mesh fixtures (tests/golden/mesh_*.npz) and, where /root/reference exists,
entry by entry against the reference's table (tests/test_mesh.py).
"""

from __future__ import annotations

import os
import re

import numpy as np

PACK = 20
_CORNERS = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0],
                     [0, 0, 1], [1, 0, 1], [1, 1, 1], [0, 1, 1]], np.int64)
_ELO = np.array([0, 1, 3, 0, 4, 5, 7, 4, 0, 1, 2, 3])
_EUP = np.array([1, 2, 2, 3, 5, 6, 6, 7, 4, 5, 6, 7])
_EAX = np.array([0, 1, 0, 1, 0, 1, 0, 1, 2, 2, 2, 2])
_SRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                    "paper_2512_12945_b200", "csrc", "svx_mesh.cu")
_TABLE = None


def tri_table() -> np.ndarray:
    """(256, 15) int edge indices, -1 padded, decoded from c_tri."""
    global _TABLE
    if _TABLE is None:
        src = open(_SRC).read()
        body = src[src.index("c_tri[256]"):]
        body = body[body.index("{") + 1:body.index("};")]
        words = [int(x, 16) for x in re.findall(r"0x([0-9a-fA-F]+)ULL", body)]
        assert len(words) == 256
        t = np.full((256, 15), -1, np.int64)
        for case, wd in enumerate(words):
            n = 3 * (wd >> 60)
            for i in range(n):
                t[case, i] = (wd >> (4 * i)) & 15
        _TABLE = t
    return _TABLE


def edge_table() -> np.ndarray:
    cases = np.arange(256)[:, None]
    return ((((cases >> _ELO) ^ (cases >> _EUP)) & 1) << np.arange(12)).sum(axis=1)


def default_palette(num_classes):
    import colorsys

    rows = [(128, 128, 128)]
    h = 0.0
    for _ in range(max(int(num_classes), 0)):
        h = (h + 0.618033988749895) % 1.0
        r, g, b = colorsys.hsv_to_rgb(h, 0.65, 0.95)
        rows.append((int(r * 255.0), int(g * 255.0), int(b * 255.0)))
    return np.array(rows, np.uint8)


def _labels(kind, rows, voxel_labels, idx):
    if voxel_labels is not None:
        return np.asarray(voxel_labels, np.int32)[idx]
    if kind is None:
        return np.zeros(idx.shape[0], np.int32)
    v = np.asarray(rows, np.float64)[idx]
    lab = np.argmax(v, axis=1).astype(np.int32) + 1
    if kind == "closed":
        lab[v.sum(axis=1) <= 0.0] = 0
    else:
        lab[np.abs(v).sum(axis=1) == 0.0] = 0
    return lab


def extract(coords, d, w, voxel_size, min_weight=0.5, kind=None, rows=None, voxel_labels=None,
            palette=None, palette_size=1):
    """(vertices, triangles, labels, colors) of the state's level set.
    kind None / "closed" / "open"; rows = counts or means per voxel (aligned
    with coords); voxel_labels = precomputed per-voxel labels (open-set with
    embeddings)."""
    empty = (np.zeros((0, 3)), np.zeros((0, 3), np.int32), np.zeros(0, np.int32),
             np.zeros((0, 3), np.uint8))
    coords = np.asarray(coords, np.int64)
    keep = np.asarray(w, np.float64) >= float(min_weight)
    vox = np.flatnonzero(keep)                      # indices into the state
    if vox.size == 0:
        return empty
    kc = coords[vox]
    lo = kc.min(axis=0)
    ext = kc.max(axis=0) - lo + 2
    if ext.max() > (1 << PACK):
        raise OverflowError("grid extent %s voxels exceeds the %d-per-axis mesh extraction limit"
                            % (ext.tolist(), 1 << PACK))
    rel = kc - lo
    key = (rel[:, 0] << (2 * PACK)) | (rel[:, 1] << PACK) | rel[:, 2]
    srt = np.argsort(key)
    key, vox = key[srt], vox[srt]
    dd = np.asarray(d, np.float64)[vox]
    n = key.shape[0]
    # corners of the cell anchored at every kept voxel
    corner = np.empty((n, 8), np.int64)
    full = np.ones(n, bool)
    for c in range(8):
        o = _CORNERS[c]
        want = key + ((o[0] << (2 * PACK)) | (o[1] << PACK) | o[2])
        pos = np.minimum(np.searchsorted(key, want), n - 1)
        full &= key[pos] == want
        corner[:, c] = pos
    corner = corner[full]
    if corner.shape[0] == 0:
        return empty
    case = ((dd[corner] < 0.0).astype(np.int64) << np.arange(8)).sum(axis=1)
    em = edge_table()[case]
    live = em != 0
    corner, case, em = corner[live], case[live], em[live]
    if corner.shape[0] == 0:
        return empty
    # vertices: crossed edges of live cells, numbered by (lower key, axis)
    cell_i, edge_i = np.nonzero((em[:, None] >> np.arange(12)) & 1)
    lower = corner[cell_i, _ELO[edge_i]]
    upper = corner[cell_i, _EUP[edge_i]]
    ekey = key[lower] * 4 + _EAX[edge_i]
    ukeys, first, vert_of = np.unique(ekey, return_index=True, return_inverse=True)
    vlo, vhi, vax = lower[first], upper[first], _EAX[edge_i[first]]
    t = dd[vlo] / (dd[vlo] - dd[vhi])
    h = float(voxel_size)
    pos = (coords[vox[vlo]].astype(np.float64) + 0.5) * h
    pos[np.arange(pos.shape[0]), vax] += t * h
    slot = np.full((corner.shape[0], 12), -1, np.int64)
    slot[cell_i, edge_i] = vert_of
    # triangles, table order within each cell, reversed winding
    tab = tri_table()[case].reshape(-1, 5, 3)
    tc, tj = np.nonzero(tab[:, :, 0] >= 0)
    e = tab[tc, tj]
    tri = np.stack([slot[tc, e[:, 2]], slot[tc, e[:, 1]], slot[tc, e[:, 0]]], axis=1)
    a = pos[tri[:, 1]] - pos[tri[:, 0]]
    b = pos[tri[:, 2]] - pos[tri[:, 0]]
    cr = np.stack([a[:, 1] * b[:, 2] - a[:, 2] * b[:, 1],
                   a[:, 2] * b[:, 0] - a[:, 0] * b[:, 2],
                   a[:, 0] * b[:, 1] - a[:, 1] * b[:, 0]], axis=1)
    area2 = (cr[:, 0] * cr[:, 0] + cr[:, 1] * cr[:, 1]) + cr[:, 2] * cr[:, 2]
    tri = tri[area2 > 0.0]
    used = np.unique(tri)
    tri = np.searchsorted(used, tri).astype(np.int32)
    verts = pos[used]
    near = np.where(t[used] < 0.5, vlo[used], vhi[used])
    labels = _labels(kind, rows, voxel_labels, vox[near])
    pal = default_palette(palette_size) if palette is None else np.asarray(palette, np.uint8)
    lab64 = labels.astype(np.int64)
    colors = pal[np.where(lab64 > 0, 1 + (lab64 - 1) % (pal.shape[0] - 1), 0)]
    if tri.shape[0] == 0:
        return empty
    return verts, tri, labels.astype(np.int32), colors

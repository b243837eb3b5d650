"""Surface meshes of the device map: the host-side record and palette of
``Mapper.extract`` (mesh.py:355-389 SemanticMesh / default_palette /
palette_colors).  The extraction itself runs in libsvx.so
(``svx_extract_mesh``, csrc/svx_mesh.cu); this module only holds the result
type and builds the default palette the device colours vertices with.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import SemvoxError


@dataclass
class SemanticMesh:
    """Triangle surface with one class label and colour per vertex
    (mesh.py:355-380): vertices (n, 3) f64 metres, triangles (m, 3) int32,
    labels (n,) int32 (0 = unknown / rejected), colors (n, 3) uint8."""

    vertices: np.ndarray
    triangles: np.ndarray
    labels: np.ndarray
    colors: np.ndarray

    @classmethod
    def empty(cls) -> "SemanticMesh":
        return cls(vertices=np.zeros((0, 3), np.float64), triangles=np.zeros((0, 3), np.int32),
                   labels=np.zeros(0, np.int32), colors=np.zeros((0, 3), np.uint8))

    @property
    def n_vertices(self) -> int:
        return int(self.vertices.shape[0])

    @property
    def n_triangles(self) -> int:
        return int(self.triangles.shape[0])

    def validate(self) -> None:
        """Shape and index checks (mesh.py SemanticMesh.validate semantics)."""
        n = self.n_vertices
        problems = []
        if self.vertices.shape != (n, 3):
            problems.append("vertex array must be (n, 3)")
        elif self.labels.shape != (n,) or self.colors.shape != (n, 3):
            problems.append("labels/colors must match vertex count")
        elif self.triangles.size and not (0 <= int(self.triangles.min()) and int(self.triangles.max()) < n):
            problems.append("triangle index out of range")
        if problems:
            raise SemvoxError(problems[0])

    def triangle_areas(self) -> np.ndarray:
        corners = self.vertices[self.triangles]            # (m, 3 corners, 3)
        edges = corners[:, 1:, :] - corners[:, :1, :]      # two edges from corner 0
        return 0.5 * np.sqrt((np.cross(edges[:, 0], edges[:, 1]) ** 2).sum(axis=1))


_GOLDEN = 0.618033988749895


def _hsv_rgb(h: np.ndarray, s: float, v: float) -> np.ndarray:
    """Vectorised HSV -> RGB in [0, 1] with the sector arithmetic of
    colorsys.hsv_to_rgb (same float operations, so identical values)."""
    sector = (h * 6.0).astype(np.int64)
    f = h * 6.0 - sector
    p = np.full_like(h, v * (1.0 - s))
    q = v * (1.0 - s * f)
    t = v * (1.0 - s * (1.0 - f))
    vv = np.full_like(h, v)
    table = {0: (vv, t, p), 1: (q, vv, p), 2: (p, vv, t), 3: (p, q, vv), 4: (t, p, vv), 5: (vv, p, q)}
    out = np.empty(h.shape + (3,), np.float64)
    for k, (r, g, b) in table.items():
        sel = (sector % 6) == k
        out[sel, 0], out[sel, 1], out[sel, 2] = r[sel], g[sel], b[sel]
    return out


def default_palette(num_classes: int) -> np.ndarray:
    """(num_classes + 1, 3) uint8: row 0 the unknown grey (128, 128, 128),
    row c the colour of hue frac(c * golden ratio) accumulated step by step
    (saturation 0.65, value 0.95) -- the reference's palette (mesh.py:382-395)."""
    k = max(int(num_classes), 0)
    hues = np.empty(k, np.float64)
    acc = 0.0
    for c in range(k):   # sequential accumulation: the rounding of each step matters
        acc = (acc + _GOLDEN) % 1.0
        hues[c] = acc
    pal = np.full((k + 1, 3), 128, np.uint8)
    if k:
        pal[1:] = (_hsv_rgb(hues, 0.65, 0.95) * 255.0).astype(np.int64).astype(np.uint8)
    return pal


def check_palette(palette) -> np.ndarray:
    """palette_colors' argument check (mesh.py:398-402)."""
    palette = np.ascontiguousarray(np.asarray(palette, np.uint8))
    if palette.ndim != 2 or palette.shape[1] != 3 or palette.shape[0] < 2:
        raise SemvoxError("palette must be (>=2, 3) uint8")
    return palette


def write_ply(mesh: SemanticMesh, path) -> None:
    """ASCII PLY with per-vertex colour and class label, the reference's
    layout (mesh.py:580-600): byte-identical files for identical meshes."""
    mesh.validate()
    with open(path, "w", encoding="ascii") as fh:
        fh.write("ply\nformat ascii 1.0\n")
        fh.write("element vertex %d\n" % mesh.n_vertices)
        fh.write("property float x\nproperty float y\nproperty float z\n")
        fh.write("property uchar red\nproperty uchar green\nproperty uchar blue\n")
        fh.write("property int label\n")
        fh.write("element face %d\n" % mesh.n_triangles)
        fh.write("property list uchar int vertex_indices\nend_header\n")
        rows = np.column_stack([mesh.vertices, mesh.colors.astype(np.float64),
                                mesh.labels.astype(np.float64)])
        np.savetxt(fh, rows, fmt=["%.9g"] * 3 + ["%d"] * 4)
        np.savetxt(fh, mesh.triangles, fmt="3 %d %d %d")


def read_ply(path) -> SemanticMesh:
    """Read meshes in write_ply's layout (ASCII, x y z r g b label vertices,
    then '3 i j k' faces; mesh.py:603-650).  The header is scanned for its
    element counts; the body is parsed in one pass with numpy."""
    with open(path, "rb") as fh:
        data = fh.read()
    try:
        text = data.decode("ascii")
    except UnicodeDecodeError:
        text = ""
    lines = text.split("\n")
    if not lines or lines[0].strip() != "ply":
        raise SemvoxError("%s: not a PLY file" % path)
    counts = {}
    body_at = None
    for i, line in enumerate(lines[1:], start=1):
        tok = line.split()
        if tok[:1] == ["format"] and tok[1:2] != ["ascii"]:
            raise SemvoxError("%s: only ASCII PLY is supported" % path)
        if tok[:1] == ["element"] and len(tok) == 3:
            counts[tok[1]] = int(tok[2])
        if tok[:1] == ["end_header"]:
            body_at = i + 1
            break
    if body_at is None:
        raise SemvoxError("%s: unterminated PLY header" % path)
    if "vertex" not in counts or "face" not in counts:
        raise SemvoxError("%s: missing vertex/face elements" % path)
    nv, nf = counts["vertex"], counts["face"]
    vrows = np.loadtxt(lines[body_at:body_at + nv], dtype=np.float64, ndmin=2).reshape(nv, 7) \
        if nv else np.zeros((0, 7))
    frows = np.loadtxt(lines[body_at + nv:body_at + nv + nf], dtype=np.int64, ndmin=2).reshape(nf, 4) \
        if nf else np.zeros((0, 4), np.int64)
    bad = np.flatnonzero(frows[:, 0] != 3)
    if bad.size:
        raise SemvoxError("%s: face %d is not a triangle" % (path, int(bad[0])))
    mesh = SemanticMesh(vertices=np.ascontiguousarray(vrows[:, :3]),
                        triangles=frows[:, 1:].astype(np.int32),
                        labels=vrows[:, 6].astype(np.int32),
                        colors=vrows[:, 3:6].astype(np.uint8))
    mesh.validate()
    return mesh


def palette_colors(labels, palette) -> np.ndarray:
    """Host restatement of the device colour lookup (label 0 -> row 0,
    others wrap over rows 1..), for callers colouring their own labels."""
    palette = check_palette(palette)
    labels = np.asarray(labels, np.int64)
    return palette[np.where(labels > 0, 1 + (labels - 1) % (palette.shape[0] - 1), 0)]

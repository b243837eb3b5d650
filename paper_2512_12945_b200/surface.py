"""Surface meshes of the device map: the host-side record and palette of
``Mapper.extract`` (mesh.py:355-389 SemanticMesh / default_palette /
palette_colors).  The extraction itself runs in libsvx.so
(``svx_extract_mesh``, csrc/svx_mesh.cu); this module only holds the result
type and builds the default palette the device colours vertices with.
"""

from __future__ import annotations

import colorsys
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
        n = self.n_vertices
        if self.vertices.shape != (n, 3):
            raise SemvoxError("vertex array must be (n, 3)")
        if self.labels.shape != (n,) or self.colors.shape != (n, 3):
            raise SemvoxError("labels/colors must match vertex count")
        t = self.triangles
        if t.size and (t.min() < 0 or t.max() >= n):
            raise SemvoxError("triangle index out of range")

    def triangle_areas(self) -> np.ndarray:
        v, t = self.vertices, self.triangles
        return 0.5 * np.linalg.norm(np.cross(v[t[:, 1]] - v[t[:, 0]], v[t[:, 2]] - v[t[:, 0]]),
                                    axis=1)


def default_palette(num_classes: int) -> np.ndarray:
    """(num_classes + 1, 3) uint8; row 0 = unknown grey, then hues stepping
    by the golden ratio (mesh.py:382-395)."""
    rows = [(128, 128, 128)]
    hue = 0.0
    for _ in range(max(int(num_classes), 0)):
        hue = (hue + 0.618033988749895) % 1.0
        r, g, b = colorsys.hsv_to_rgb(hue, 0.65, 0.95)
        rows.append((int(r * 255.0), int(g * 255.0), int(b * 255.0)))
    return np.array(rows, dtype=np.uint8)


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
    """Read meshes written by write_ply (mesh.py:603-650): ASCII, fixed layout."""
    with open(path, "r", encoding="ascii") as fh:
        if fh.readline().strip() != "ply":
            raise SemvoxError("%s: not a PLY file" % path)
        n_vert = n_face = -1
        while True:
            line = fh.readline()
            if not line:
                raise SemvoxError("%s: unterminated PLY header" % path)
            parts = line.split()
            if parts[:2] in (["format", "binary_little_endian"], ["format", "binary_big_endian"]):
                raise SemvoxError("%s: only ASCII PLY is supported" % path)
            if parts[:2] == ["element", "vertex"]:
                n_vert = int(parts[2])
            elif parts[:2] == ["element", "face"]:
                n_face = int(parts[2])
            elif parts[:1] == ["end_header"]:
                break
        if n_vert < 0 or n_face < 0:
            raise SemvoxError("%s: missing vertex/face elements" % path)
        verts = np.zeros((n_vert, 3), np.float64)
        labels = np.zeros(n_vert, np.int32)
        colors = np.zeros((n_vert, 3), np.uint8)
        for i in range(n_vert):
            f = fh.readline().split()
            verts[i] = [float(f[0]), float(f[1]), float(f[2])]
            colors[i] = [int(f[3]), int(f[4]), int(f[5])]
            labels[i] = int(f[6])
        tri = np.zeros((n_face, 3), np.int32)
        for i in range(n_face):
            f = fh.readline().split()
            if int(f[0]) != 3:
                raise SemvoxError("%s: face %d is not a triangle" % (path, i))
            tri[i] = [int(f[1]), int(f[2]), int(f[3])]
    mesh = SemanticMesh(vertices=verts, triangles=tri, labels=labels, colors=colors)
    mesh.validate()
    return mesh


def palette_colors(labels, palette) -> np.ndarray:
    """Host restatement of the device colour lookup (label 0 -> row 0,
    others wrap over rows 1..), for callers colouring their own labels."""
    palette = check_palette(palette)
    labels = np.asarray(labels, np.int64)
    return palette[np.where(labels > 0, 1 + (labels - 1) % (palette.shape[0] - 1), 0)]

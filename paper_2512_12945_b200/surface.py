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


def palette_colors(labels, palette) -> np.ndarray:
    """Host restatement of the device colour lookup (label 0 -> row 0,
    others wrap over rows 1..), for callers colouring their own labels."""
    palette = check_palette(palette)
    labels = np.asarray(labels, np.int64)
    return palette[np.where(labels > 0, 1 + (labels - 1) % (palette.shape[0] - 1), 0)]

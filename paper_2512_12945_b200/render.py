"""Ray-march rendering of the device map: the reference's render surface
(render.py:33-272: RenderCamera, sample_distance, render) over libsvx.so
(``svx_render`` / ``svx_sample_distance``, csrc/svx_render.cu).  Host side:
camera validation (the reference's messages) and the default palette; the
rays, the march, the secant refinement and the per-pixel outputs run on the
GPU and reproduce the reference's images bit for bit.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import surface
from ._lib import check, lib
from .errors import ConfigError, SemvoxError

_MODES = ("depth", "semantic", "normal")
_MODE_CODE = {"depth": 0, "semantic": 1, "normal": 2}


class SvxRenderCamera(ctypes.Structure):
    _fields_ = [("pose", ctypes.c_double * 16),
                ("fx", ctypes.c_double), ("fy", ctypes.c_double),
                ("cx", ctypes.c_double), ("cy", ctypes.c_double),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("near_plane", ctypes.c_double), ("far_plane", ctypes.c_double)]


@dataclass
class RenderCamera:
    """Pinhole camera: x right, y down, z forward (render.py:33-85)."""

    pose: np.ndarray  # (4, 4) camera-to-world
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    near: float = 0.05
    far: float = 10.0

    @classmethod
    def from_config(cls, cfg, pose, near: float = 0.05, far: float = 10.0) -> "RenderCamera":
        return cls(pose=np.asarray(pose, np.float64), fx=cfg.fx, fy=cfg.fy, cx=cfg.cx, cy=cfg.cy,
                   width=cfg.width, height=cfg.height, near=near, far=far)

    def validate(self) -> None:
        from .mapper import validate_rotation

        if self.near <= 0.0:
            raise ConfigError(f"near plane must be positive, got {self.near}")
        if self.far <= self.near:
            raise ConfigError(f"far plane {self.far} must exceed near {self.near}")
        if self.width <= 0 or self.height <= 0:
            raise ConfigError("image dimensions must be positive")
        if self.fx == 0.0 or self.fy == 0.0:
            raise ConfigError("focal lengths must be nonzero")
        pose = np.asarray(self.pose, np.float64)
        if pose.shape != (4, 4):
            raise ConfigError(f"camera pose must be 4x4, got {pose.shape}")
        if not np.allclose(pose[3], (0.0, 0.0, 0.0, 1.0), atol=1e-9):
            raise ConfigError("camera pose bottom row must be (0, 0, 0, 1)")
        self.pose = pose.copy()
        self.pose[:3, :3] = validate_rotation(pose[:3, :3])

    def _c(self) -> SvxRenderCamera:
        c = SvxRenderCamera()
        c.pose[:] = [float(x) for x in np.asarray(self.pose, np.float64).reshape(-1)]
        c.fx, c.fy, c.cx, c.cy = float(self.fx), float(self.fy), float(self.cx), float(self.cy)
        c.width, c.height = int(self.width), int(self.height)
        c.near_plane, c.far_plane = float(self.near), float(self.far)
        return c


def _mapper_of(grid):
    m = getattr(grid, "_m", None)
    if m is None:
        raise SemvoxError("expected a grid view of this engine's map")
    return m


def sample_distance(tsdf_grid, points):
    """Trilinear D at world points (render.py:88-113): (values (N,), valid (N,));
    NaN / False where a surrounding voxel centre is unobserved."""
    from .mapper import KIND_TSDF

    if tsdf_grid.kind != KIND_TSDF:
        raise SemvoxError("sample_distance needs a TSDF grid, got kind %d" % tsdf_grid.kind)
    m = _mapper_of(tsdf_grid)
    pts = np.ascontiguousarray(np.asarray(points, np.float64).reshape(-1, 3))
    n = pts.shape[0]
    vals = np.empty(n, np.float64)
    valid = np.empty(n, np.uint8)
    if n:
        check(lib.svx_sample_distance(m._handle, pts.ctypes.data, n, vals.ctypes.data,
                                      valid.ctypes.data, None))
    return vals, valid.astype(bool)


def render(tsdf_grid, semantic_grid, camera: RenderCamera, mode: str = "depth",
           embeddings=None, palette=None) -> np.ndarray:
    """render (render.py:214-272) on the GPU: "depth" (H, W) f64, "semantic"
    (H, W, 3) u8, "normal" (H, W, 3) f64; background 0 in every mode."""
    from .mapper import KIND_OPEN, KIND_TSDF, PayloadMismatchError

    if mode not in _MODES:
        raise ConfigError(f"render mode must be one of {_MODES}, got {mode!r}")
    if tsdf_grid.kind != KIND_TSDF:
        raise SemvoxError("render needs a TSDF grid, got kind %d" % tsdf_grid.kind)
    if mode == "semantic" and semantic_grid is None:
        raise ConfigError("semantic mode needs a semantic grid")
    m = _mapper_of(tsdf_grid)
    camera.validate()
    emb = None
    k = 0
    pal = None
    if mode == "semantic":
        if embeddings is not None and semantic_grid.kind == KIND_OPEN:
            emb = np.ascontiguousarray(embeddings, np.float64)
            if emb.ndim != 2 or emb.shape[1] != m._open.feature_dim:
                raise PayloadMismatchError(
                    f"embeddings shape {emb.shape} incompatible with feature dim "
                    f"{m._open.feature_dim}")
            k = emb.shape[0]
        if palette is None:
            if m._closed is not None:
                size = m._closed.num_classes
            else:
                size = k if emb is not None else m._open.feature_dim
            palette = surface.default_palette(size)
        pal = surface.check_palette(palette)
    h, w = int(camera.height), int(camera.width)
    out = (np.empty((h, w), np.float64) if mode == "depth" else
           np.empty((h, w, 3), np.uint8 if mode == "semantic" else np.float64))
    tau = m._open.temperature if m._open is not None else 0.0
    tp = m._open.confidence_threshold if m._open is not None else 0.0
    cam = camera._c()
    check(lib.svx_render(m._handle, ctypes.byref(cam), _MODE_CODE[mode],
                         emb.ctypes.data if emb is not None else None, k, tau, tp,
                         pal.ctypes.data if pal is not None else None,
                         pal.shape[0] if pal is not None else 0, out.ctypes.data, None))
    return out


"""``Mapper``: the drop-in mapping API over the B200 engine.

Mirrors ``semvox_bindings.Mapper`` (pkg/bindings/src/semvox_bindings/__init__.py:58-201):
flat-config routing and its errors, ``integrate(points, pose, labels=|features=)``
returning an ``IntegrationReport``, ``query``, ``stats``, ``config`` and
``grids``.  Host-side work is limited to what the reference does on the host
before its kernel (frame validation, fusion.py:31-92, 173-224); everything from
the world transform on runs in libsvx.so on the GPU.  Arrays may be numpy
arrays (copied by the engine) or CUDA torch tensors (used in place, on torch's
current stream).
"""

from __future__ import annotations

import collections
import ctypes
import dataclasses
import hashlib
import math
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import SEM_CLOSED, SEM_NONE, SEM_OPEN, SVX_F32, SVX_F64, check, lib
from .config import ClosedSetConfig, EngineConfig, FusionConfig, OpenSetConfig
from . import snapshot, surface
from .errors import (ConfigError, FormatError, OutOfRangeError, PayloadMismatchError,
                     UserInputError)

KIND_TSDF, KIND_CLOSED, KIND_OPEN = 0, 1, 2   # grid.py:26-28
KIND_NAMES = {KIND_TSDF: "tsdf", KIND_CLOSED: "closed", KIND_OPEN: "open"}
COORD_LIMIT = 1 << 30                          # coords.py:41
LEAF_LOG2, INTERNAL_LOG2 = 3, 4                # config.py:26-27
_MAGIC = b"SLVG"                               # grid.py:31

_FUSION_KEYS = {f.name for f in dataclasses.fields(FusionConfig)}
_CLOSED_KEYS = {f.name for f in dataclasses.fields(ClosedSetConfig)}
_OPEN_KEYS = {f.name for f in dataclasses.fields(OpenSetConfig)}
_ENGINE_KEYS = {f.name for f in dataclasses.fields(EngineConfig)}
_MAPPER_KEYS = {"threads", "backend", "map_bounds"}

_ROT_PASS, _ROT_FIX = 1e-4, 1e-3               # fusion.py:27-28


@dataclass
class IntegrationReport:
    """Per-frame counts (fusion.py:103-117) plus engine extras."""

    points_in: int = 0
    points_used: int = 0
    skipped_nonfinite: int = 0
    skipped_range: int = 0
    skipped_degenerate: int = 0
    skipped_bad_label: int = 0
    band_hits: int = 0
    touched_voxels: int = 0
    prep_ms: float = 0.0
    kernel_ms: float = 0.0
    new_blocks: int = 0
    new_voxels: int = 0

    def as_dict(self):
        return {f.name: getattr(self, f.name) for f in dataclasses.fields(IntegrationReport)}


_REPORT_FIELDS = frozenset(f.name for f in dataclasses.fields(IntegrationReport))
_RESOLVE_AFTER = 32   # pending reports older than this many frames are fetched (64 are held)


class _PendingReport(IntegrationReport):
    """The report of a frame still in flight (svx_integrate_async): its
    fields are fetched with svx_report_wait on first access, so reading one
    waits for that frame (and only for the frames before it)."""

    def __init__(self, mapper, ticket):
        object.__setattr__(self, "_mapper", mapper)
        object.__setattr__(self, "_ticket", ticket)

    def __getattribute__(self, name):
        if name in _REPORT_FIELDS and object.__getattribute__(self, "_mapper") is not None:
            object.__getattribute__(self, "_resolve")()
        return object.__getattribute__(self, name)

    def _resolve(self):
        m = object.__getattribute__(self, "_mapper")
        if m is None:
            return
        rep = _lib.SvxReport()
        check(lib.svx_report_wait(m._handle, object.__getattribute__(self, "_ticket"),
                                  ctypes.byref(rep)))
        for f in ("points_in", "points_used", "skipped_nonfinite", "skipped_range",
                  "skipped_degenerate", "skipped_bad_label", "band_hits", "touched_voxels",
                  "kernel_ms", "new_blocks", "new_voxels"):
            object.__setattr__(self, f, getattr(rep, f))
        object.__setattr__(self, "prep_ms", 0.0)
        object.__setattr__(self, "_mapper", None)


@dataclass
class MemoryStats:
    """grid.py:80-86."""

    leaf_count: int
    internal_count: int
    root_entries: int
    active_voxels: int
    resident_bytes: int


@dataclass
class TsdfPayload:
    truncation: float
    kind: int = KIND_TSDF


@dataclass
class ClosedPayload:
    cfg: ClosedSetConfig
    kind: int = KIND_CLOSED


@dataclass
class OpenPayload:
    cfg: OpenSetConfig
    kind: int = KIND_OPEN


def validate_rotation(R, context: str = "pose"):
    """Accept within 1e-4 of orthonormal, polar-fix within 1e-3, else reject
    (fusion.py:31-49)."""
    R = np.asarray(R, np.float64)
    if R.shape != (3, 3) or not np.isfinite(R).all():
        raise UserInputError(f"{context}: rotation block must be finite 3x3")
    err = float(np.abs(R @ R.T - np.eye(3)).max())
    if np.linalg.det(R) <= 0:
        raise UserInputError(f"{context}: rotation determinant not positive (mirrored)")
    if err <= _ROT_PASS:
        return R
    if err <= _ROT_FIX:
        u, _, vt = np.linalg.svd(R)
        fixed = u @ vt
        if np.linalg.det(fixed) <= 0:
            raise UserInputError(f"{context}: rotation not fixable by polar projection")
        return fixed
    raise UserInputError(f"{context}: rotation block off orthonormal by {err:.2e} (> 1e-3)")


def _check_pose(pose, frame_id):
    """Frame pose checks of fusion.py:68-77.  The common case (finite, exact
    bottom row, rotation within 1e-4 of orthonormal) is decided with scalar
    arithmetic; anything else takes the numpy path of validate_rotation."""
    pose = np.asarray(pose, np.float64)
    if pose.shape != (4, 4):
        raise UserInputError(f"pose must be 4x4, got {pose.shape}")
    f = pose.ravel().tolist()
    a0, a1, a2, _, b0, b1, b2, _, c0, c1, c2, _, z0, z1, z2, z3 = f
    if z0 == 0.0 and z1 == 0.0 and z2 == 0.0 and z3 == 1.0 and all(map(math.isfinite, f)):
        # |R R^T - I| entrywise, straight-line
        err = max(abs(a0 * a0 + a1 * a1 + a2 * a2 - 1.0), abs(b0 * b0 + b1 * b1 + b2 * b2 - 1.0),
                  abs(c0 * c0 + c1 * c1 + c2 * c2 - 1.0), abs(a0 * b0 + a1 * b1 + a2 * b2),
                  abs(a0 * c0 + a1 * c1 + a2 * c2), abs(b0 * c0 + b1 * c1 + b2 * c2))
        det = a0 * (b1 * c2 - b2 * c1) - a1 * (b0 * c2 - b2 * c0) + a2 * (b0 * c1 - b1 * c0)
        if err <= _ROT_PASS * 0.5 and det > 0.0:
            return pose.copy(order="C")
    if not np.isfinite(pose).all():
        raise UserInputError("pose contains non-finite values")
    if not np.allclose(pose[3], (0, 0, 0, 1), atol=1e-9):
        raise UserInputError("pose bottom row must be [0 0 0 1]")
    fixed = np.array(pose, np.float64, copy=True, order="C")
    fixed[:3, :3] = validate_rotation(pose[:3, :3], f"frame {frame_id} pose")
    return fixed


_TORCH = []


def _torch_mod():
    """torch if it is already imported (CUDA tensors imply it), else None."""
    if not _TORCH:
        import sys

        t = sys.modules.get("torch")
        if t is None:
            return None
        _TORCH.append(t)
    return _TORCH[0]


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


class _Arg:
    """A contiguous array handed to the C ABI: numpy (host) or CUDA tensor."""

    def __init__(self, x, kind: str):
        self.keep = None
        self.cuda = False
        if _is_torch(x):
            import torch

            if kind == "int32":
                t = x if x.dtype == torch.int32 else x.to(torch.int32)
                self.code = None
            elif kind == "depth" and x.dtype in (torch.float32, torch.float64, torch.uint16):
                t = x
                self.code = {torch.float32: SVX_F32, torch.float64: SVX_F64,
                             torch.uint16: _lib.SVX_U16}[x.dtype]
            elif x.dtype in (torch.float32, torch.float64):
                t = x
                self.code = SVX_F64 if x.dtype == torch.float64 else SVX_F32
            else:
                t = x.to(torch.float64)
                self.code = SVX_F64
            t = t.contiguous()
            if not t.is_cuda:
                t = t.numpy()
                self.keep = t
                self.ptr = t.ctypes.data if t.size else None
                self.shape = t.shape
                return
            self.keep = t
            self.cuda = True
            self.dev = t.get_device()
            self.ptr = t.data_ptr() if t.numel() else None
            self.shape = tuple(t.shape)
            return
        if kind == "int32":
            a = np.ascontiguousarray(x, np.int32)
            self.code = None
        elif kind == "depth":
            a = np.asarray(x)
            if a.dtype not in (np.float32, np.float64, np.uint16):
                a = a.astype(np.float64)
            a = np.ascontiguousarray(a)
            self.code = {np.dtype(np.float32): SVX_F32, np.dtype(np.float64): SVX_F64,
                         np.dtype(np.uint16): _lib.SVX_U16}[a.dtype]
        else:
            a = np.asarray(x)
            if a.dtype not in (np.float32, np.float64):
                a = a.astype(np.float64)
            a = np.ascontiguousarray(a)
            self.code = SVX_F64 if a.dtype == np.float64 else SVX_F32
        self.keep = a
        self.ptr = a.ctypes.data if a.size else None
        self.shape = a.shape

    def finite_host(self):
        return None if self.cuda else self.keep


def _camera_arg(camera):
    """CameraConfig fields (config.py:114-134) -> SvxCamera, validated with
    the reference's messages."""
    get = (lambda k, dflt: camera.get(k, dflt)) if isinstance(camera, dict) else \
        (lambda k, dflt: getattr(camera, k, dflt))
    c = _lib.SvxCamera()
    c.fx, c.fy = float(get("fx", 0.0)), float(get("fy", 0.0))
    c.cx, c.cy = float(get("cx", 0.0)), float(get("cy", 0.0))
    c.depth_scale = float(get("depth_scale", 1.0))
    c.width, c.height, c.stride = int(get("width", 0)), int(get("height", 0)), int(get("stride", 1))
    if c.fx <= 0 or c.fy <= 0:
        raise ConfigError("fx and fy must be positive")
    if c.width < 1 or c.height < 1:
        raise ConfigError("raster dimensions must be positive")
    if c.depth_scale <= 0:
        raise ConfigError("depth_scale must be positive")
    if c.stride < 1:
        raise ConfigError("stride must be >= 1")
    return c


def _is_float_raster(x) -> bool:
    if _is_torch(x):
        return x.dtype.is_floating_point
    return np.issubdtype(np.asarray(x).dtype, np.floating)


def _stream_for(args):
    """(stream handle, all inputs on `device`) for a call: torch's current
    stream of the inputs' device when any input is a CUDA tensor."""
    dev = None
    all_dev = True
    for a in args:
        if a is None:
            continue
        if a.cuda:
            dev = a.dev
        else:
            all_dev = False
    if dev is None:
        return None, False
    import torch

    return ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(dev)), all_dev


class Mapper:
    """One mapping run on one GPU: a TSDF grid plus an optional semantic grid.

    Configuration is one flat mapping (keyword arguments override it), routed
    by field name exactly like the reference (bindings/__init__.py:77-116).
    Extra engine keys: ``tsdf_dtype`` ("float64" reference layout, default, or
    "float32" compact), ``device``, ``reserve_voxels``, ``reserve_blocks``.
    ``backend`` accepts None/"auto"/"python"/"native" (there is one engine); ``threads``
    is validated and has no effect (device parallelism never changes bits).
    """

    def __init__(self, config=None, /, **overrides):
        self._handle = None
        merged = {}
        if config is not None:
            merged.update(config)
        merged.update(overrides)
        unknown = (set(merged) - _FUSION_KEYS - _CLOSED_KEYS - _OPEN_KEYS - _MAPPER_KEYS
                   - _ENGINE_KEYS)
        if unknown:
            raise ConfigError("unknown config keys: " + ", ".join(sorted(unknown)))
        threads = merged.pop("threads", 1)
        if not isinstance(threads, (int, np.integer)) or threads < 1:
            raise ConfigError(f"threads must be an integer >= 1, got {threads!r}")
        self._threads = int(threads)
        # get_backend's names (backend.py:25-37) are accepted so scripts that pin
        # one keep working; there is one engine here (the CUDA path), whichever
        # is named.  Unknown names fail with the reference's message.
        backend = merged.pop("backend", None)
        bname = backend.strip().lower() if isinstance(backend, str) else backend
        if bname not in (None, "auto", "python", "native", "cuda"):
            raise ConfigError(f"unknown backend {backend!r} (expected auto, python, or native)")
        self._map_bounds = merged.pop("map_bounds", None)

        fusion_kw = {k: v for k, v in merged.items() if k in _FUSION_KEYS}
        closed_kw = {k: v for k, v in merged.items() if k in _CLOSED_KEYS}
        open_kw = {k: v for k, v in merged.items() if k in _OPEN_KEYS}
        engine_kw = {k: v for k, v in merged.items() if k in _ENGINE_KEYS}
        closed = open_set = None
        if closed_kw.get("num_classes", 0):
            closed = ClosedSetConfig(**closed_kw)
        elif closed_kw:
            raise ConfigError("closed-set keys %s need num_classes >= 1"
                              % ", ".join(sorted(closed_kw)))
        if open_kw.get("feature_dim", 0):
            open_set = OpenSetConfig(**open_kw)
        elif open_kw:
            raise ConfigError("open-set keys %s need feature_dim >= 1"
                              % ", ".join(sorted(open_kw)))
        self._cfg = FusionConfig(**fusion_kw)
        self._cfg.validate()                                   # make_grids, fusion.py:304
        if closed is not None and open_set is not None:        # fusion.py:305-306
            raise UserInputError("a run is closed-set or open-set, not both")
        if closed is not None:
            closed.validate()
        if open_set is not None:
            open_set.validate()
        self._engine = EngineConfig(**engine_kw)
        self._engine.validate()
        self._closed, self._open = closed, open_set
        self._frames = 0

        c = _lib.SvxConfig()
        c.voxel_size = float(self._cfg.voxel_size)
        c.truncation = float(self._cfg.truncation)
        c.max_range = float(self._cfg.max_range)
        c.weight_fn = 0 if self._cfg.weight_fn == "constant_one" else 1
        c.space_carving = int(bool(self._cfg.space_carving))
        c.sem_kind = SEM_CLOSED if closed else (SEM_OPEN if open_set else SEM_NONE)
        if closed is not None:
            c.num_classes = int(closed.num_classes)
            c.last_wins = int(closed.fusion == "last_wins")
            c.count_dtype = SVX_F64 if np.dtype(closed.count_dtype) == np.float64 else SVX_F32
        if open_set is not None:
            c.feature_dim = int(open_set.feature_dim)
            c.state_dtype = SVX_F64 if np.dtype(open_set.state_dtype) == np.float64 else SVX_F32
            c.prior_beta = float(open_set.prior_beta)
            c.lambda_floor = float(open_set.lambda_floor)
        else:
            c.lambda_floor = 1e-3
        c.tsdf_dtype = SVX_F64 if np.dtype(self._engine.tsdf_dtype) == np.float64 else SVX_F32
        c.device = int(self._engine.device)
        self._device = c.device
        c.reserve_voxels = int(self._engine.reserve_voxels)
        c.reserve_blocks = int(self._engine.reserve_blocks)
        self._c = c
        h = ctypes.c_void_p()
        check(lib.svx_create(ctypes.byref(c), ctypes.byref(h)))
        self._handle = h
        self._rep = _lib.SvxReport()
        self._rep_ref = ctypes.byref(self._rep)
        # asynchronous frames (closed-set / geometry maps): Mapper.integrate's
        # fast paths submit the frame and return a report read on first use
        self._async = int(self._engine.async_frames) if open_set is None else 0
        check(lib.svx_set_async(h, self._async, int(self._engine.async_leaf_headroom)))
        self._pending = collections.deque()
        self._ticket = ctypes.c_uint64()
        self._ticket_ref = ctypes.byref(self._ticket)
        self._tsdf_view = GridView(self, KIND_TSDF)
        self._sem_view = None
        if closed is not None:
            self._sem_view = GridView(self, KIND_CLOSED)
        elif open_set is not None:
            self._sem_view = GridView(self, KIND_OPEN)

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and lib is not None:
            lib.svx_destroy(h)
            self._handle = None

    # -- reference surface ---------------------------------------------------

    @property
    def config(self) -> FusionConfig:
        return self._cfg

    @property
    def grids(self):
        """(tsdf, semantic) views over the device grids (semantic None for a
        geometry-only run); they read the live map, they are not copies."""
        return self._tsdf_view, self._sem_view

    @property
    def sem_kind(self) -> str | None:
        return "closed" if self._closed else ("open" if self._open else None)

    def _payload_args(self, n, labels, features, frame_id):
        if labels is not None and features is not None:
            raise PayloadMismatchError("frame carries both labels and features")
        lab = feat = None
        if labels is not None:
            lab = _Arg(labels, "int32")
            if tuple(lab.shape) != (n,):
                raise PayloadMismatchError(f"labels shape {tuple(lab.shape)} != point count {n}")
        if features is not None:
            feat = _Arg(features, "float")
            if len(feat.shape) != 2 or feat.shape[0] != n:
                raise PayloadMismatchError(
                    f"features shape {tuple(feat.shape)} incompatible with {n} points")
        # _check_grids (fusion.py:173-197)
        if self._closed is not None and lab is None:
            raise PayloadMismatchError("closed-set grid requires per-point labels")
        if self._open is not None:
            if feat is None:
                raise PayloadMismatchError("open-set grid requires per-point features")
            if feat.shape[1] != self._open.feature_dim:
                raise PayloadMismatchError(
                    f"feature dim {feat.shape[1]} != grid dim {self._open.feature_dim}")
        if self._closed is None:
            lab = None
        if self._open is None:
            feat = None
        return lab, feat

    def _points_arg(self, points):
        pts = _Arg(points, "float")
        if len(pts.shape) != 2 or pts.shape[1] != 3:
            raise UserInputError(f"points must be (n, 3), got {tuple(pts.shape)}")
        return pts

    def _run(self, fn, pts, vec, lab, feat):
        rep = self._rep
        stream, all_dev = _stream_for((pts, lab, feat))
        # every input already on the map's GPU: skip the library's pointer checks
        flag = _lib.DEVICE_INPUTS if all_dev and pts.dev == self._device else 0
        n = int(pts.shape[0])
        vec = np.ascontiguousarray(vec, np.float64)
        check(fn(self._handle, pts.ptr, pts.code | flag, n, vec.ctypes.data,
                 lab.ptr if lab is not None else None,
                 feat.ptr if feat is not None else None,
                 feat.code if feat is not None else SVX_F32, stream, self._rep_ref))
        self._frames += 1
        return IntegrationReport(
            points_in=rep.points_in, points_used=rep.points_used,
            skipped_nonfinite=rep.skipped_nonfinite, skipped_range=rep.skipped_range,
            skipped_degenerate=rep.skipped_degenerate, skipped_bad_label=rep.skipped_bad_label,
            band_hits=rep.band_hits, touched_voxels=rep.touched_voxels,
            kernel_ms=rep.kernel_ms, new_blocks=rep.new_blocks, new_voxels=rep.new_voxels)

    def integrate(self, points, pose, labels=None, features=None):
        """Fuse one frame of sensor-frame points (n, 3) under a 4x4
        sensor-to-world pose, with integer ``labels`` (closed-set) or float
        ``features`` (open-set).  Same contract as bindings/__init__.py:131-142
        and integrate_frame (fusion.py:200-293)."""
        if features is None and self._open is None:
            rep = self._integrate_fast(points, pose, labels)
            if rep is not None:
                return rep
        pts = self._points_arg(points)
        pose = _check_pose(pose, self._frames)
        lab, feat = self._payload_args(int(pts.shape[0]), labels, features, self._frames)
        return self._run(lib.svx_integrate, pts, pose.reshape(-1), lab, feat)

    def _integrate_fast(self, points, pose, labels):
        """The common call -- contiguous CUDA tensors on the map's GPU or
        contiguous numpy arrays (f32/f64 points, int32 labels for closed-set
        maps) and a C-contiguous float64 4x4 pose -- with the pose's fast
        acceptance test done by the library (SVX_POSE_CHECK).  Returns None
        when the call needs the general path (any other argument form, or a
        pose that needs full validation), so checks and error messages stay
        those of the general path."""
        if type(points) is np.ndarray:
            return self._integrate_fast_host(points, pose, labels)
        torch = _torch_mod()
        if torch is None or type(points) is not torch.Tensor or not points.is_cuda:
            return None
        dt = points.dtype
        if (dt is not torch.float32 and dt is not torch.float64) or points.dim() != 2 \
                or points.shape[1] != 3 or not points.is_contiguous() \
                or points.get_device() != self._device:
            return None
        n = points.shape[0]
        lab_ptr = None
        if self._closed is not None:
            if type(labels) is not torch.Tensor or labels.dtype is not torch.int32 \
                    or labels.dim() != 1 or labels.shape[0] != n or not labels.is_contiguous() \
                    or labels.get_device() != self._device:
                return None
            lab_ptr = labels.data_ptr() if n else None
        elif labels is not None:
            return None
        if type(pose) is not np.ndarray or pose.dtype != np.float64 or pose.shape != (4, 4) \
                or not pose.flags.c_contiguous:
            return None
        code = (SVX_F64 if dt is torch.float64 else SVX_F32) | _lib.DEVICE_INPUTS | _lib.POSE_CHECK
        stream = ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(self._device))
        if self._async:
            return self._submit(points.data_ptr() if n else None, code, n, pose, lab_ptr, stream)
        st = lib.svx_integrate(self._handle, points.data_ptr() if n else None, code, n,
                               pose.ctypes.data, lab_ptr, None, SVX_F32, stream, self._rep_ref)
        if st == _lib.POSE_NEEDS_HOST:
            return None
        check(st)
        self._frames += 1
        rep = self._rep
        return IntegrationReport(
            points_in=rep.points_in, points_used=rep.points_used,
            skipped_nonfinite=rep.skipped_nonfinite, skipped_range=rep.skipped_range,
            skipped_degenerate=rep.skipped_degenerate, skipped_bad_label=rep.skipped_bad_label,
            band_hits=rep.band_hits, touched_voxels=rep.touched_voxels,
            kernel_ms=rep.kernel_ms, new_blocks=rep.new_blocks, new_voxels=rep.new_voxels)

    def _submit(self, pts_ptr, code, n, pose, lab_ptr, stream):
        """svx_integrate_async: the frame is queued; its report is fetched on
        first use (or here, once it is _RESOLVE_AFTER frames old)."""
        st = lib.svx_integrate_async(self._handle, pts_ptr, code, n, pose.ctypes.data, lab_ptr,
                                     stream, self._ticket_ref)
        if st == _lib.POSE_NEEDS_HOST:
            return None
        check(st)
        self._frames += 1
        rep = _PendingReport(self, self._ticket.value)
        pend = self._pending
        pend.append(rep)
        while len(pend) > _RESOLVE_AFTER:
            pend.popleft()._resolve()
        return rep

    def _integrate_fast_host(self, points, pose, labels):
        """_integrate_fast for host numpy arrays: the library copies them to
        the GPU on the default stream (pinned memory goes by DMA)."""
        dt = points.dtype
        if (dt != np.float32 and dt != np.float64) or points.ndim != 2 or points.shape[1] != 3 \
                or not points.flags.c_contiguous:
            return None
        n = points.shape[0]
        lab_ptr = None
        if self._closed is not None:
            if type(labels) is not np.ndarray or labels.dtype != np.int32 or labels.ndim != 1 \
                    or labels.shape[0] != n or not labels.flags.c_contiguous:
                return None
            lab_ptr = labels.ctypes.data if n else None
        elif labels is not None:
            return None
        if type(pose) is not np.ndarray or pose.dtype != np.float64 or pose.shape != (4, 4) \
                or not pose.flags.c_contiguous:
            return None
        code = (SVX_F64 if dt == np.float64 else SVX_F32) | _lib.POSE_CHECK
        if self._async:
            return self._submit(points.ctypes.data if n else None, code, n, pose, lab_ptr, None)
        st = lib.svx_integrate(self._handle, points.ctypes.data if n else None, code, n,
                               pose.ctypes.data, lab_ptr, None, SVX_F32, None, self._rep_ref)
        if st == _lib.POSE_NEEDS_HOST:
            return None
        check(st)
        self._frames += 1
        rep = self._rep
        return IntegrationReport(
            points_in=rep.points_in, points_used=rep.points_used,
            skipped_nonfinite=rep.skipped_nonfinite, skipped_range=rep.skipped_range,
            skipped_degenerate=rep.skipped_degenerate, skipped_bad_label=rep.skipped_bad_label,
            band_hits=rep.band_hits, touched_voxels=rep.touched_voxels,
            kernel_ms=rep.kernel_ms, new_blocks=rep.new_blocks, new_voxels=rep.new_voxels)

    def integrate_depth(self, depth, payload, camera, pose=None):
        """Back-project a depth raster on the GPU and fuse it: the
        reference's ``ingest.project_depth(depth, payload, intr, pose)``
        (ingest.py:285-322) followed by ``integrate`` on the returned Frame.
        ``camera`` has the CameraConfig fields (fx, fy, cx, cy, width, height,
        depth_scale, stride; an object or a mapping); ``payload`` is an
        integer (H, W) label raster or a float (H, W[, l]) feature raster.
        Rasters may be numpy arrays or CUDA tensors."""
        cam = _camera_arg(camera)
        d = _Arg(depth, "depth")
        if tuple(d.shape) != (cam.height, cam.width):
            raise ConfigError(f"depth raster {tuple(d.shape)} does not match camera "
                              f"({cam.height}, {cam.width})")
        pshape = tuple(payload.shape)
        if pshape[:2] != tuple(d.shape):
            raise ConfigError(f"payload raster {pshape[:2]} does not match depth {tuple(d.shape)}")
        is_float = _is_float_raster(payload)
        lab = feat = None
        if is_float:
            feat = _Arg(payload, "float")
            dim = 1 if len(pshape) == 2 else pshape[2]
            if self._closed is not None:
                raise PayloadMismatchError("closed-set grid requires per-point labels")
            if self._open is not None and dim != self._open.feature_dim:
                raise PayloadMismatchError(
                    f"feature dim {dim} != grid dim {self._open.feature_dim}")
        else:
            lab = _Arg(payload, "int32")
            if self._open is not None:
                raise PayloadMismatchError("open-set grid requires per-point features")
        if self._closed is None:
            lab = None
        if self._open is None:
            feat = None
        pose = np.eye(4) if pose is None else pose
        pose = _check_pose(pose, self._frames)
        rep = self._rep
        stream, _ = _stream_for((d, lab, feat))
        vec = np.ascontiguousarray(pose.reshape(-1), np.float64)
        check(lib.svx_integrate_depth(
            self._handle, d.ptr, d.code, ctypes.byref(cam), vec.ctypes.data,
            lab.ptr if lab is not None else None, feat.ptr if feat is not None else None,
            feat.code if feat is not None else SVX_F32, stream, self._rep_ref))
        self._frames += 1
        return IntegrationReport(
            points_in=rep.points_in, points_used=rep.points_used,
            skipped_nonfinite=rep.skipped_nonfinite, skipped_range=rep.skipped_range,
            skipped_degenerate=rep.skipped_degenerate, skipped_bad_label=rep.skipped_bad_label,
            band_hits=rep.band_hits, touched_voxels=rep.touched_voxels,
            kernel_ms=rep.kernel_ms, new_blocks=rep.new_blocks, new_voxels=rep.new_voxels)

    def integrate_world(self, points_world, origin, labels=None, features=None):
        """Fuse world-frame points observed from ``origin``: the reference's
        backend seam (fusion.py:229-289 -> integrate_points) with
        delta = p - origin, t = |delta|, u = delta / t."""
        pts = self._points_arg(points_world)
        o = np.asarray(origin, np.float64).reshape(-1)
        if o.shape != (3,) or not np.isfinite(o).all():
            raise UserInputError("origin must be a finite 3-vector")
        lab, feat = self._payload_args(int(pts.shape[0]), labels, features, self._frames)
        return self._run(lib.svx_integrate_world, pts, o, lab, feat)

    def query(self, embedding):
        """Cosine of every active voxel mean against one embedding, in active
        order: (coords (n, 3) int64, sims (n,) float64); NaN for a zero mean
        (bindings/__init__.py:153-169)."""
        if self._open is None:
            raise PayloadMismatchError("embedding query needs an open-set map")
        q = np.ascontiguousarray(embedding, np.float64).reshape(-1)
        dim = self._open.feature_dim
        if q.shape[0] != dim:
            raise PayloadMismatchError(f"query vector has dim {q.shape[0]}, map stores {dim}")
        n = self.active_count()
        coords = self._tsdf_view.active_coords()
        sims = np.empty(n, np.float64)
        check(lib.svx_query_cosine(self._handle, q.ctypes.data, n,
                                   sims.ctypes.data if n else None, None))
        return coords, sims

    def classify(self, embeddings, temperature=None, confidence_threshold=None,
                 return_sims=False):
        """classify_means (gaussian.py:132-155) over all active voxels with the
        TSDF weight as the observation weight (mesh.py:419-445): (labels
        (n,) int32 with 0 = reject, best (n,) float64[, sims (n, k)])."""
        if self._open is None:
            raise PayloadMismatchError("classification needs an open-set map")
        emb = np.ascontiguousarray(embeddings, np.float64)
        if emb.ndim != 2 or emb.shape[1] != self._open.feature_dim:
            raise PayloadMismatchError(
                f"embeddings shape {emb.shape} incompatible with feature dim "
                f"{self._open.feature_dim}")
        tau = self._open.temperature if temperature is None else float(temperature)
        tp = (self._open.confidence_threshold if confidence_threshold is None
              else float(confidence_threshold))
        n = self.active_count()
        k = emb.shape[0]
        labels = np.empty(n, np.int32)
        best = np.empty(n, np.float64)
        sims = np.empty((n, k), np.float64) if return_sims else None
        check(lib.svx_classify(self._handle, emb.ctypes.data, k, tau, tp, n,
                               labels.ctypes.data if n else None,
                               best.ctypes.data if n else None,
                               sims.ctypes.data if (return_sims and n) else None, None))
        return (labels, best, sims) if return_sims else (labels, best)

    def label_map(self, zero_if_empty=False):
        """Closed-set argmax labels in active order: dirichlet.label_map
        (dirichlet.py:81-88), or evalbench.grid_labels (0 where no counts,
        evalbench.py:30-55) with ``zero_if_empty``.  Returns (coords, labels)."""
        if self._closed is None:
            raise PayloadMismatchError("label map needs a closed-set map")
        n = self.active_count()
        labels = np.empty(n, np.int32)
        check(lib.svx_label_map(self._handle, 1 if zero_if_empty else 0, n,
                                labels.ctypes.data if n else None, None))
        return self._tsdf_view.active_coords(), labels

    def reserve(self, voxels: int, blocks: int) -> None:
        """Pre-size the device pools for `voxels` active voxels in `blocks` leaves."""
        check(lib.svx_reserve(self._handle, int(voxels), int(blocks)))

    _UPDATE_MODES = {"auto": 0, "segments": 1, "slots": 2, "leaves": 3}

    def set_update_mode(self, mode: str = "auto") -> None:
        """Row-grouping strategy of closed-set / geometry maps
        (svx_set_update_mode): "auto", "segments", "slots" or "leaves".  All
        give bit-identical maps; the choice only changes speed."""
        if mode not in self._UPDATE_MODES:
            raise ValueError(f"update mode must be one of {sorted(self._UPDATE_MODES)}")
        check(lib.svx_set_update_mode(self._handle, self._UPDATE_MODES[mode]))

    _SCORE_PATHS = {"auto": 0, "dmma": 1, "tcgen05": 2}

    def set_score_path(self, path: str = "auto") -> None:
        """classify's kernel (svx_set_score_path): "auto", "dmma" (FP64 tensor
        cores) or "tcgen05" (exact int8 split GEMM on the 5th-gen tensor
        cores).  Same labels; scores within f64 rounding."""
        if path not in self._SCORE_PATHS:
            raise ValueError(f"score path must be one of {sorted(self._SCORE_PATHS)}")
        check(lib.svx_set_score_path(self._handle, self._SCORE_PATHS[path]))

    def set_profiling(self, enable: bool = True) -> None:
        """Record per-stage device times of each integrate (svx_set_profiling)."""
        check(lib.svx_set_profiling(self._handle, int(bool(enable))))

    def stage_times(self) -> dict:
        """Last frame's per-stage device milliseconds (needs set_profiling)."""
        buf = (ctypes.c_double * len(_lib.STAGES))()
        lib.svx_stage_times(self._handle, buf, len(_lib.STAGES))
        return {name: float(buf[i]) for i, name in enumerate(_lib.STAGES)}

    def frame_counters(self) -> dict:
        """Diagnostics: internal counters of the last finished frame."""
        buf = (ctypes.c_int64 * 6)()
        lib.svx_frame_counters(self._handle, buf, 6)
        return dict(zip(("rows", "touched", "leaves", "big_leaves", "long_voxels", "huge_voxels"),
                        (int(v) for v in buf)))

    def active_count(self) -> int:
        c = ctypes.c_int64()
        check(lib.svx_active_count(self._handle, ctypes.byref(c)))
        return int(c.value)

    def engine_stats(self) -> dict:
        s = _lib.SvxStats()
        check(lib.svx_stats_get(self._handle, ctypes.byref(s)))
        return {f: int(getattr(s, f)) for f, _ in s._fields_}

    def stats(self) -> dict:
        """sparsity_report of the TSDF grid (evalbench.py:297-327) plus
        frames_integrated and semantic_active_voxels (bindings/__init__.py:171-181)."""
        report = dict(_sparsity_report(self._tsdf_view, self._map_bounds))
        report["frames_integrated"] = self._frames
        if self._sem_view is not None:
            report["semantic_active_voxels"] = self._sem_view.memory_stats().active_voxels
        return report

    def save(self, path) -> None:
        """Write the map as a ``.slvg`` snapshot (bindings/__init__.py:183-187):
        the TSDF grid block, then the semantic one; byte-identical to the
        reference's file for the same map (snapshot.py)."""
        coords, d, w, sem0, sem1 = self._export()
        views = [v for v in (self._tsdf_view, self._sem_view) if v is not None]
        with open(path, "wb") as fh:
            for v in views:
                snapshot.write_block(fh, v.kind, v.voxel_size, _params_block(v.payload), coords,
                                     v._fields(d, w, sem0, sem1))

    def render(self, camera, mode: str = "depth", embeddings=None, palette=None):
        """render (render.py:214-272) of this map from `camera` (a RenderCamera),
        ray-marched on the GPU; see paper_2512_12945_b200.render.render."""
        from .render import render

        return render(self._tsdf_view, self._sem_view, camera, mode=mode, embeddings=embeddings,
                      palette=palette)

    @classmethod
    def from_snapshot(cls, path, config=None, /, **overrides):
        """A Mapper whose map is the snapshot's, ready to integrate further
        frames (engine extension; the reference only reads snapshots back as
        grids, grid.py:358-407).  Voxel size, truncation and the semantic
        payload parameters come from the file; the remaining configuration
        (max_range, weight_fn, space_carving, engine keys) from `config` /
        keyword arguments, which must not contradict the file."""
        blocks = snapshot.read_blocks(path)
        tsdf, sem = _split_blocks(blocks)
        merged = dict(config or {})
        merged.update(overrides)
        from_file = {"voxel_size": tsdf.voxel_size, "truncation": tsdf.params[0]}
        if sem is not None and sem.kind == KIND_CLOSED:
            c, alpha, mode, code = sem.params
            from_file.update(num_classes=c, prior_alpha=alpha,
                             fusion="bayes" if mode == 0 else "last_wins",
                             count_dtype=_CODE_NAMES[code])
        elif sem is not None:
            dim, beta, floor, conf, temp, code = sem.params
            from_file.update(feature_dim=dim, prior_beta=beta, lambda_floor=floor,
                             confidence_threshold=conf, temperature=temp,
                             state_dtype=_CODE_NAMES[code])
        for k, v in from_file.items():
            if k in merged and merged[k] != v and not (
                    isinstance(v, str) and np.dtype(merged[k]) == np.dtype(v)):
                raise ConfigError(f"{k}={merged[k]!r} contradicts the snapshot's {v!r}")
            merged[k] = v
        if sem is None and (merged.get("num_classes") or merged.get("feature_dim")):
            raise ConfigError("the snapshot holds geometry only")
        m = cls(merged)
        m._import_blocks(tsdf, sem)
        return m

    def _import_blocks(self, tsdf, sem):
        n = tsdf.active_count
        sem0 = sem1 = None
        if sem is not None:
            sem0 = np.ascontiguousarray(sem.fields[0])
            sem1 = np.ascontiguousarray(sem.fields[1]) if sem.kind == KIND_OPEN else None
        lc = np.ascontiguousarray(tsdf.leaf_coords, np.int32)
        vl = np.ascontiguousarray(tsdf.voxel_leaf, np.int32)
        vs = np.ascontiguousarray(tsdf.voxel_slot, np.int32)
        d = np.ascontiguousarray(tsdf.fields[0], np.float64)
        w = np.ascontiguousarray(tsdf.fields[1], np.float64)

        def p(a):
            return a.ctypes.data if (a is not None and a.size) else None

        check(lib.svx_import(self._handle, lc.shape[0], p(lc), n, p(vl), p(vs), p(d), p(w),
                             p(sem0), p(sem1), None))

    def extract(self, min_weight: float = 0.5, embeddings=None, palette=None):
        """Triangulate the current zero level set (bindings/__init__.py:144-151 ->
        extract_mesh, mesh.py:419-545) on the GPU: a SemanticMesh with
        vertices, triangles, per-vertex labels and colours, byte-identical to
        the reference's for the same map.  ``embeddings`` (k, D) labels
        open-set vertices by classify_means; otherwise closed-set maps use
        the count argmax and open-set maps the dominant feature axis."""
        emb = None
        k = 0
        if embeddings is not None and self._open is not None:
            emb = np.ascontiguousarray(embeddings, np.float64)
            if emb.ndim != 2 or emb.shape[1] != self._open.feature_dim:
                raise PayloadMismatchError(
                    f"embeddings shape {emb.shape} incompatible with feature dim "
                    f"{self._open.feature_dim}")
            k = emb.shape[0]
        tau = self._open.temperature if self._open is not None else 0.0
        tp = self._open.confidence_threshold if self._open is not None else 0.0
        nv, nt = ctypes.c_int64(), ctypes.c_int64()
        check(lib.svx_extract_mesh(self._handle, float(min_weight),
                                   emb.ctypes.data if emb is not None else None, k, tau, tp,
                                   ctypes.byref(nv), ctypes.byref(nt), None))
        nv, nt = int(nv.value), int(nt.value)
        if nt == 0:
            return surface.SemanticMesh.empty()
        if palette is None:
            if self._closed is not None:
                size = self._closed.num_classes
            elif self._open is not None:
                size = k if emb is not None else self._open.feature_dim
            else:
                size = 1
            palette = surface.default_palette(size)
        palette = surface.check_palette(palette)
        mesh = surface.SemanticMesh(vertices=np.empty((nv, 3), np.float64),
                                    triangles=np.empty((nt, 3), np.int32),
                                    labels=np.empty(nv, np.int32),
                                    colors=np.empty((nv, 3), np.uint8))
        check(lib.svx_mesh_read(self._handle, mesh.vertices.ctypes.data,
                                mesh.triangles.ctypes.data, mesh.labels.ctypes.data,
                                mesh.colors.ctypes.data, palette.ctypes.data, palette.shape[0],
                                None))
        return mesh

    # -- bulk export -----------------------------------------------------------

    def _export(self):
        """(coords, d, w, sem0, sem1) of all active voxels in active order."""
        n = self.active_count()
        tdt = np.float64 if self._c.tsdf_dtype == SVX_F64 else np.float32
        coords = np.empty((n, 3), np.int64)
        d = np.empty(n, tdt)
        w = np.empty(n, tdt)
        sem0 = sem1 = None
        if self._closed is not None:
            sem0 = np.empty((n, self._closed.num_classes), np.dtype(self._closed.count_dtype))
        if self._open is not None:
            sdt = np.dtype(self._open.state_dtype)
            sem0 = np.empty((n, self._open.feature_dim), sdt)
            sem1 = np.empty((n, self._open.feature_dim), sdt)

        def p(a):
            return a.ctypes.data if (a is not None and a.size) else None

        check(lib.svx_export_active(self._handle, n, p(coords), p(d), p(w), p(sem0), p(sem1),
                                    None))
        return coords, d, w, sem0, sem1

    def _probe(self, coords):
        coords = np.ascontiguousarray(np.atleast_2d(coords), np.int64)
        if coords.size and np.abs(coords).max() >= COORD_LIMIT:
            raise OutOfRangeError("voxel coordinate beyond +/-2^30 addressable range")
        m = coords.shape[0]
        tdt = np.float64 if self._c.tsdf_dtype == SVX_F64 else np.float32
        d = np.empty(m, tdt)
        w = np.empty(m, tdt)
        active = np.empty(m, np.uint8)
        sem0 = sem1 = None
        if self._closed is not None:
            sem0 = np.empty((m, self._closed.num_classes), np.dtype(self._closed.count_dtype))
        if self._open is not None:
            sdt = np.dtype(self._open.state_dtype)
            sem0 = np.empty((m, self._open.feature_dim), sdt)
            sem1 = np.empty((m, self._open.feature_dim), sdt)

        def p(a):
            return a.ctypes.data if (a is not None and a.size) else None

        check(lib.svx_probe(self._handle, p(coords), m, p(d), p(w), p(sem0), p(sem1),
                            p(active), None))
        return d, w, sem0, sem1, active.astype(bool)


class GridView:
    """Read-only SparseGrid-like view (grid.py:89-215) of one payload of a
    Mapper's device map.  TSDF fields are returned as float64 like the
    reference's payload (grid.py:45-47)."""

    def __init__(self, mapper: Mapper, kind: int):
        self._m = mapper
        self.kind = kind
        self.voxel_size = float(mapper._cfg.voxel_size)
        if kind == KIND_TSDF:
            self.payload = TsdfPayload(float(mapper._cfg.truncation))
        elif kind == KIND_CLOSED:
            self.payload = ClosedPayload(mapper._closed)
        else:
            self.payload = OpenPayload(mapper._open)

    @property
    def kind_name(self):
        return KIND_NAMES[self.kind]

    def _fields(self, d, w, sem0, sem1):
        if self.kind == KIND_TSDF:
            return [np.asarray(d, np.float64), np.asarray(w, np.float64)]
        if self.kind == KIND_CLOSED:
            return [sem0]
        return [sem0, sem1]

    def active_values(self):
        coords, d, w, sem0, sem1 = self._m._export()
        return coords, self._fields(d, w, sem0, sem1)

    def active_coords(self):
        return self._m._export()[0]

    def probe_many(self, coords):
        d, w, sem0, sem1, active = self._m._probe(coords)
        return self._fields(d, w, sem0, sem1), active

    def get(self, coord):
        vals, _ = self.probe_many(np.asarray(coord, np.int64).reshape(1, 3))
        return tuple(v[0] for v in vals)

    def memory_stats(self) -> MemoryStats:
        st = self._m.engine_stats()
        coords = self.active_coords()
        internal = 0
        if coords.shape[0]:
            internal = int(np.unique(coords >> (LEAF_LOG2 + INTERNAL_LOG2), axis=0).shape[0])
        te = 8 if self._m._c.tsdf_dtype == SVX_F64 else 4
        per_tsdf = 2 * te
        per_sem = st["payload_bytes_per_voxel"] - per_tsdf
        leaf_bytes = st["leaf_count"] * (16 + 64 + 4 * 512)
        hash_bytes = st["hash_capacity"] * 16
        if self.kind == KIND_TSDF:
            resident = leaf_bytes + hash_bytes + st["active_voxels"] * per_tsdf
        else:
            resident = st["active_voxels"] * per_sem
        return MemoryStats(leaf_count=st["leaf_count"], internal_count=internal,
                           root_entries=internal, active_voxels=st["active_voxels"],
                           resident_bytes=int(resident))

    def content_hash(self):
        """Order-independent digest with the reference's layout (grid.py:204-215)."""
        coords, vals = self.active_values()
        return content_hash_of(coords, vals, self.payload, self.voxel_size)


_CODE_NAMES = {0: "float32", 1: "float64"}


def _split_blocks(blocks):
    """(tsdf, semantic) blocks of a snapshot (load_grid,
    bindings/__init__.py:189-201: the first of each kind), checked to share
    one active set: the engine keeps TSDF and semantic payloads of a voxel in
    one record, as every Mapper-written snapshot has them."""
    tsdf = sem = None
    for b in blocks:
        if b.kind == KIND_TSDF and tsdf is None:
            tsdf = b
        elif b.kind != KIND_TSDF and sem is None:
            sem = b
    if tsdf is None:
        raise FormatError("snapshot holds no TSDF grid block")
    if sem is not None:
        if sem.voxel_size != tsdf.voxel_size:
            raise FormatError("TSDF and semantic blocks disagree on the voxel size")
        if not (np.array_equal(sem.leaf_coords, tsdf.leaf_coords)
                and np.array_equal(sem.voxel_leaf, tsdf.voxel_leaf)
                and np.array_equal(sem.voxel_slot, tsdf.voxel_slot)):
            raise FormatError("semantic block's active set differs from the TSDF block's")
    return tsdf, sem


def load_grid(path, backend=None, **engine):
    """Read a snapshot written by Mapper.save (bindings/__init__.py:189-201).

    Returns (tsdf, semantic) grid views over a device map holding the
    snapshot (semantic None for geometry only); the views keep that map
    alive.  `engine` takes EngineConfig keys (device, tsdf_dtype, ...)."""
    if backend not in (None, "auto", "cuda"):
        raise ConfigError(f"unknown backend {backend!r} (expected auto or cuda)")
    m = Mapper.from_snapshot(path, **engine)
    return m.grids


def grids_equal(a, b, exact=True, rtol=0.0, atol=0.0) -> bool:
    """grid.py:428-447 over any two grids with ``kind``, ``voxel_size`` and
    ``active_values()`` (engine views, or the reference's SparseGrid)."""
    if a.kind != b.kind or a.voxel_size != b.voxel_size:
        return False
    ca, va = a.active_values()
    cb, vb = b.active_values()
    if ca.shape != cb.shape:
        return False
    oa = np.lexsort((ca[:, 2], ca[:, 1], ca[:, 0]))
    ob = np.lexsort((cb[:, 2], cb[:, 1], cb[:, 0]))
    if not np.array_equal(ca[oa], cb[ob]):
        return False
    for fa, fb in zip(va, vb):
        if exact:
            if not np.array_equal(fa[oa], fb[ob]):
                return False
        elif not np.allclose(fa[oa], fb[ob], rtol=rtol, atol=atol):
            return False
    return True


def content_hash_of(coords, vals, payload, voxel_size: float) -> str:
    """content_hash (grid.py:204-215) of active coords + field arrays."""
    order = np.lexsort((coords[:, 2], coords[:, 1], coords[:, 0]))
    hs = hashlib.sha256()
    hs.update(_MAGIC)
    hs.update(_params_block(payload))
    hs.update(struct.pack("<dBB", voxel_size, LEAF_LOG2, INTERNAL_LOG2))
    hs.update(np.ascontiguousarray(coords[order]).tobytes())
    for v in vals:
        hs.update(np.ascontiguousarray(v[order]).tobytes())
    return hs.hexdigest()


def _dtype_code(name) -> int:
    return 1 if np.dtype(name) == np.float64 else 0


def _params_block(payload) -> bytes:
    """Payload parameter bytes hashed by content_hash (grid.py:276-295)."""
    if payload.kind == KIND_TSDF:
        return struct.pack("<d", payload.truncation)
    cfg = payload.cfg
    if payload.kind == KIND_CLOSED:
        return struct.pack("<IdBB", cfg.num_classes, cfg.prior_alpha,
                           0 if cfg.fusion == "bayes" else 1, _dtype_code(cfg.count_dtype))
    return struct.pack("<IddddB", cfg.feature_dim, cfg.prior_beta, cfg.lambda_floor,
                       cfg.confidence_threshold, cfg.temperature, _dtype_code(cfg.state_dtype))


def _sparsity_report(view: GridView, map_bounds=None) -> dict:
    """evalbench.sparsity_report (evalbench.py:297-327) over a device grid."""
    stats = view.memory_stats()
    te = 8 if view._m._c.tsdf_dtype == SVX_F64 else 4
    per_voxel = 2 * te
    out = {
        "active_voxels": stats.active_voxels,
        "leaf_count": stats.leaf_count,
        "internal_count": stats.internal_count,
        "resident_bytes": stats.resident_bytes,
        "payload_bytes_per_voxel": per_voxel,
    }
    coords = view.active_coords()
    if coords.shape[0]:
        ext = coords.max(axis=0) - coords.min(axis=0) + 1
        dense_bbox = int(np.prod(ext.astype(np.float64)) * per_voxel)
        out["dense_bbox_bytes"] = dense_bbox
        out["ratio_bbox"] = stats.resident_bytes / dense_bbox if dense_bbox else np.inf
    if map_bounds is not None:
        lo, hi = np.asarray(map_bounds, np.float64)
        nvox = np.prod(np.ceil((hi - lo) / view.voxel_size))
        dense_bounds = int(nvox * per_voxel)
        out["dense_bounds_bytes"] = dense_bounds
        out["ratio_bounds"] = stats.resident_bytes / dense_bounds if dense_bounds else np.inf
    return out

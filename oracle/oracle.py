"""ctypes wrapper of the CPU oracle (liboracle.so, built from svx_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU legs as the parity checker / CPU baseline, never by the
product package.  See svx_oracle.c for the reference lines each step restates.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")


class OrcConfig(ctypes.Structure):
    _fields_ = [
        ("voxel_size", ctypes.c_double), ("truncation", ctypes.c_double),
        ("max_range", ctypes.c_double), ("weight_fn", ctypes.c_int32),
        ("space_carving", ctypes.c_int32), ("sem_kind", ctypes.c_int32),
        ("num_classes", ctypes.c_int32), ("last_wins", ctypes.c_int32),
        ("feature_dim", ctypes.c_int32), ("prior_beta", ctypes.c_double),
        ("lambda_floor", ctypes.c_double), ("tsdf_f32", ctypes.c_int32),
        ("sem_f32", ctypes.c_int32), ("threads", ctypes.c_int32),
    ]


class OrcReport(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "points_in", "points_used", "skipped_nonfinite", "skipped_range", "skipped_degenerate",
        "skipped_bad_label", "band_hits", "touched_voxels", "new_blocks", "new_voxels")] + [
        (n, ctypes.c_double) for n in (
            "t_emit_ms", "t_sort_ms", "t_group_ms", "t_ensure_ms", "t_update_ms")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


def build():
    """Compile liboracle.so (gcc, -ffp-contract=off, OpenMP)."""
    import subprocess

    cc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
    subprocess.check_call(["make", "-s", "-C", HERE, f"CC={cc}"])


def _load():
    if not os.path.exists(LIB_PATH):
        build()
    lib = ctypes.CDLL(LIB_PATH)
    P, I64, I32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
    sig = {
        "orc_create": ([ctypes.POINTER(OrcConfig)], P),
        "orc_destroy": ([P], None),
        "orc_integrate": ([P, P, I64, P, I32, P, P, ctypes.POINTER(OrcReport)], I32),
        "orc_raycast_band": ([P, P, D, D, I32, P, I64], I64),
        "orc_active_count": ([P], I64),
        "orc_leaf_count": ([P], I64),
        "orc_export": ([P, P, P, P, P, P], I64),
        "orc_probe": ([P, P, I64, P, P, P, P, P], None),
        "orc_cosine": ([P, P, P], None),
        "orc_classify": ([P, P, I32, D, D, P, P], None),
        "orc_label_map": ([P, I32, P], None),
        "orc_last_error": ([], ctypes.c_char_p),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = _load()
    return _lib


class OracleError(Exception):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _p(a):
    return a.ctypes.data if a is not None and a.size else None


class OracleMap:
    """CPU restatement of one mapping run (TSDF + optional semantics)."""

    def __init__(self, voxel_size=0.05, truncation=0.1, max_range=15.0, weight_fn="constant_one",
                 space_carving=False, num_classes=0, fusion="bayes", feature_dim=0,
                 prior_beta=1e-3, lambda_floor=1e-3, tsdf_dtype="float64", sem_dtype="float32",
                 threads=0):
        c = OrcConfig()
        c.voxel_size, c.truncation, c.max_range = voxel_size, truncation, max_range
        c.weight_fn = 0 if weight_fn == "constant_one" else 1
        c.space_carving = int(bool(space_carving))
        c.sem_kind = 1 if num_classes else (2 if feature_dim else 0)
        c.num_classes, c.feature_dim = int(num_classes), int(feature_dim)
        c.last_wins = int(fusion == "last_wins")
        c.prior_beta, c.lambda_floor = prior_beta, lambda_floor
        c.tsdf_f32 = int(np.dtype(tsdf_dtype) == np.float32)
        c.sem_f32 = int(np.dtype(sem_dtype) == np.float32)
        c.threads = int(threads)
        self.cfg = c
        self.tsdf_dtype = np.dtype(tsdf_dtype)
        self.sem_dtype = np.dtype(sem_dtype)
        self._h = lib().orc_create(ctypes.byref(c))
        if not self._h:
            raise MemoryError("oracle map allocation failed")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.orc_destroy(h)
            self._h = None

    @property
    def kind(self):
        return {0: None, 1: "closed", 2: "open"}[self.cfg.sem_kind]

    def _integrate(self, points, pose16, sensor, labels, features):
        pts = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
        lab = np.ascontiguousarray(labels, np.int32) if labels is not None else None
        feat = np.ascontiguousarray(features, np.float64) if features is not None else None
        pose = np.ascontiguousarray(pose16, np.float64).reshape(16)
        rep = OrcReport()
        st = lib().orc_integrate(self._h, _p(pts), pts.shape[0], pose.ctypes.data, int(sensor),
                                 _p(lab), _p(feat), ctypes.byref(rep))
        if st:
            raise OracleError(st, lib().orc_last_error().decode())
        return rep

    def integrate(self, points, pose, labels=None, features=None):
        """Sensor-frame points + 4x4 pose (transform ((R0x+R1y)+R2z)+t)."""
        return self._integrate(points, np.asarray(pose, np.float64), True, labels, features)

    def integrate_world(self, points_world, origin, labels=None, features=None):
        pose = np.eye(4)
        pose[:3, 3] = np.asarray(origin, np.float64)
        return self._integrate(points_world, pose, False, labels, features)

    def active_count(self):
        return int(lib().orc_active_count(self._h))

    def leaf_count(self):
        return int(lib().orc_leaf_count(self._h))

    def export(self):
        """(coords, d, w, sem0, sem1) in active order; values as stored
        (rounded to the configured dtypes), returned in those dtypes."""
        n = self.active_count()
        P = self.cfg.num_classes or self.cfg.feature_dim
        coords = np.empty((n, 3), np.int64)
        d = np.empty(n)
        w = np.empty(n)
        s0 = np.empty((n, P)) if self.cfg.sem_kind else None
        s1 = np.empty((n, P)) if self.cfg.sem_kind == 2 else None
        lib().orc_export(self._h, _p(coords), _p(d), _p(w), _p(s0), _p(s1))
        d = d.astype(self.tsdf_dtype)
        w = w.astype(self.tsdf_dtype)
        if s0 is not None:
            s0 = s0.astype(self.sem_dtype)
        if s1 is not None:
            s1 = s1.astype(self.sem_dtype)
        return coords, d, w, s0, s1

    def probe(self, coords):
        coords = np.ascontiguousarray(np.atleast_2d(coords), np.int64)
        m = coords.shape[0]
        P = self.cfg.num_classes or self.cfg.feature_dim
        d, w = np.empty(m), np.empty(m)
        s0 = np.empty((m, P)) if self.cfg.sem_kind else None
        s1 = np.empty((m, P)) if self.cfg.sem_kind == 2 else None
        act = np.empty(m, np.uint8)
        lib().orc_probe(self._h, _p(coords), m, _p(d), _p(w), _p(s0), _p(s1), _p(act))
        return d, w, s0, s1, act.astype(bool)

    def cosine(self, q):
        q = np.ascontiguousarray(q, np.float64).reshape(-1)
        out = np.empty(self.active_count())
        lib().orc_cosine(self._h, q.ctypes.data, _p(out))
        return out

    def classify(self, emb, temperature=0.01, confidence_threshold=0.1):
        emb = np.ascontiguousarray(emb, np.float64)
        n = self.active_count()
        labels = np.empty(n, np.int32)
        best = np.empty(n)
        lib().orc_classify(self._h, emb.ctypes.data, emb.shape[0], float(temperature),
                           float(confidence_threshold), _p(labels), _p(best))
        return labels, best

    def label_map(self, zero_if_empty=False):
        labels = np.empty(self.active_count(), np.int32)
        lib().orc_label_map(self._h, 1 if zero_if_empty else 0, _p(labels))
        return labels


def raycast_band(origin, endpoint, voxel_size, truncation, space_carving=False):
    """Ordered band voxels of one ray (int64 (M, 3))."""
    o = np.ascontiguousarray(origin, np.float64)
    e = np.ascontiguousarray(endpoint, np.float64)
    cap = 1 << 16
    out = np.empty((cap, 3), np.int64)
    n = lib().orc_raycast_band(o.ctypes.data, e.ctypes.data, float(voxel_size), float(truncation),
                               int(bool(space_carving)), out.ctypes.data, cap)
    if n < 0:
        raise OracleError(6, "ray band exceeds step budget")
    return out[:n].copy()


def project_depth(depth, payload, camera):
    """Depth raster -> sensor-frame points + payload, restating
    ingest.project_depth (ingest.py:285-322): pixels sampled every `stride`
    from (0, 0) in row-major order; d > 0 and finite only; point
    ((u - cx) * d / fx, (v - cy) * d / fy, d) * depth_scale in f64; integer
    payloads give int32 labels, float payloads (n, l) f64 features.
    `camera` is a mapping with the CameraConfig fields."""
    s = int(camera.get("stride", 1))
    d = np.asarray(depth)[::s, ::s].astype(np.float64)
    us = np.arange(0, camera["width"], s, dtype=np.float64)
    vs = np.arange(0, camera["height"], s, dtype=np.float64)
    uu, vv = np.meshgrid(us, vs)
    with np.errstate(invalid="ignore"):
        ok = (d > 0) & np.isfinite(d)
    d, uu, vv = d[ok], uu[ok], vv[ok]
    pts = np.stack([(uu - camera["cx"]) * d / camera["fx"],
                    (vv - camera["cy"]) * d / camera["fy"],
                    d], axis=1) * camera.get("depth_scale", 1.0)
    pay = np.asarray(payload)[::s, ::s]
    if np.issubdtype(pay.dtype, np.floating):
        feats = pay[ok].astype(np.float64)
        if feats.ndim == 1:
            feats = feats[:, None]
        return pts, None, feats
    return pts, pay[ok].astype(np.int32), None

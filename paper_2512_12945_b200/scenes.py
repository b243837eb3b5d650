"""Seeded synthetic sensor streams for the BASELINE.json configurations.

The paper's datasets (SemanticKITTI, SceneNet) are not available; these
analytic scenes stand in for them with the shapes, sizes and value
distributions BASELINE.json states.  Everything is
torch so generation runs on the GPU for the benchmark and on the CPU in tests.
Generation is not part of any timed region.

Scenes are unions of labelled primitives (half-space floor, axis-aligned boxes,
vertical capped cylinders, spheres, inward room walls).  Rays return the
nearest hit; LiDAR rays with no return yield NaN points (a real driver's "no
return"), which the integrator counts as skipped_nonfinite.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch


@dataclass
class Scene:
    boxes: torch.Tensor          # (B, 6) xmin ymin zmin xmax ymax zmax
    box_cls: torch.Tensor        # (B,) int64 object ids
    cyls: torch.Tensor           # (Y, 5) cx cy r zmin zmax
    cyl_cls: torch.Tensor
    spheres: torch.Tensor        # (S, 4) cx cy cz r
    sph_cls: torch.Tensor
    ground_cls: int = 1          # z = 0 plane (facing +z); <= 0 disables
    room: tuple | None = None    # (xmin, ymin, zmin, xmax, ymax, zmax) inward walls
    room_cls: tuple = (1, 2, 3)  # walls, floor, ceiling
    n_objects: int = 0           # object ids are 1..n_objects
    extra: dict = field(default_factory=dict)

    def to(self, device):
        kw = {k: (v.to(device) if torch.is_tensor(v) else v) for k, v in self.__dict__.items()}
        return Scene(**kw)


def _ray_boxes(o, d, boxes, t_best, c_best, cls):
    if boxes.shape[0] == 0:
        return
    inv = 1.0 / torch.where(d == 0, torch.full_like(d, 1e-30), d)        # (N, 3)
    lo = boxes[None, :, :3]
    hi = boxes[None, :, 3:]
    t1 = (lo - o[:, None, :]) * inv[:, None, :]
    t2 = (hi - o[:, None, :]) * inv[:, None, :]
    tmin = torch.minimum(t1, t2).amax(dim=2)
    tmax = torch.maximum(t1, t2).amin(dim=2)
    hit = (tmax >= tmin) & (tmin > 1e-6)
    t = torch.where(hit, tmin, torch.full_like(tmin, math.inf))
    tb, ib = t.min(dim=1)
    better = tb < t_best
    t_best[better] = tb[better]
    c_best[better] = cls[ib[better]]


def _ray_cylinders(o, d, cyl, t_best, c_best, cls):
    if cyl.shape[0] == 0:
        return
    ox = o[:, None, 0] - cyl[None, :, 0]
    oy = o[:, None, 1] - cyl[None, :, 1]
    dx, dy, dz = d[:, None, 0], d[:, None, 1], d[:, None, 2]
    r = cyl[None, :, 2]
    a = dx * dx + dy * dy
    b = 2 * (ox * dx + oy * dy)
    c = ox * ox + oy * oy - r * r
    disc = b * b - 4 * a * c
    sq = torch.sqrt(torch.clamp(disc, min=0))
    a_safe = torch.where(a > 1e-12, a, torch.ones_like(a))
    t_side = (-b - sq) / (2 * a_safe)
    z_side = o[:, None, 2] + t_side * dz
    ok = (disc >= 0) & (a > 1e-12) & (t_side > 1e-6) & (z_side >= cyl[None, :, 3]) & (z_side <= cyl[None, :, 4])
    t = torch.where(ok, t_side, torch.full_like(t_side, math.inf))
    # top cap
    dz_safe = torch.where(dz.abs() > 1e-12, dz, torch.full_like(dz, 1e-12))
    t_cap = (cyl[None, :, 4] - o[:, None, 2]) / dz_safe
    px = ox + t_cap * dx
    py = oy + t_cap * dy
    ok_cap = (t_cap > 1e-6) & (px * px + py * py <= r * r)
    t = torch.minimum(t, torch.where(ok_cap, t_cap, torch.full_like(t_cap, math.inf)))
    tb, ib = t.min(dim=1)
    better = tb < t_best
    t_best[better] = tb[better]
    c_best[better] = cls[ib[better]]


def _ray_spheres(o, d, sph, t_best, c_best, cls):
    if sph.shape[0] == 0:
        return
    oc = o[:, None, :] - sph[None, :, :3]
    b = (oc * d[:, None, :]).sum(-1)
    c = (oc * oc).sum(-1) - sph[None, :, 3] ** 2
    disc = b * b - c
    t = -b - torch.sqrt(torch.clamp(disc, min=0))
    ok = (disc >= 0) & (t > 1e-6)
    t = torch.where(ok, t, torch.full_like(t, math.inf))
    tb, ib = t.min(dim=1)
    better = tb < t_best
    t_best[better] = tb[better]
    c_best[better] = cls[ib[better]]


def raycast(scene: Scene, o, d, chunk=1 << 16):
    """Nearest hit distance (inf if none) and object id (0 if none) per ray."""
    n = d.shape[0]
    t_out = torch.full((n,), math.inf, dtype=d.dtype, device=d.device)
    c_out = torch.zeros(n, dtype=torch.int64, device=d.device)
    o = o.expand(n, 3) if o.dim() == 1 or o.shape[0] == 1 else o
    for s in range(0, n, chunk):
        oo, dd = o[s:s + chunk], d[s:s + chunk]
        tb = t_out[s:s + chunk]
        cb = c_out[s:s + chunk]
        if scene.ground_cls > 0:
            dz = dd[:, 2]
            tg = torch.where(dz < -1e-12, -oo[:, 2] / torch.where(dz < -1e-12, dz, -torch.ones_like(dz)),
                             torch.full_like(dz, math.inf))
            better = tg < tb
            tb[better] = tg[better]
            cb[better] = scene.ground_cls
        if scene.room is not None:
            lo = torch.tensor(scene.room[:3], dtype=d.dtype, device=d.device)
            hi = torch.tensor(scene.room[3:], dtype=d.dtype, device=d.device)
            inv = 1.0 / torch.where(dd == 0, torch.full_like(dd, 1e-30), dd)
            t_exit = torch.maximum((lo - oo) * inv, (hi - oo) * inv)       # (N, 3)
            tw, axis = t_exit.min(dim=1)
            wall_cls = torch.tensor(scene.room_cls, device=d.device)
            cls = torch.where(axis == 2, torch.where(dd[:, 2] < 0, wall_cls[1], wall_cls[2]), wall_cls[0])
            better = tw < tb
            tb[better] = tw[better]
            cb[better] = cls[better]
        _ray_boxes(oo, dd, scene.boxes, tb, cb, scene.box_cls)
        _ray_cylinders(oo, dd, scene.cyls, tb, cb, scene.cyl_cls)
        _ray_spheres(oo, dd, scene.spheres, tb, cb, scene.sph_cls)
    return t_out, c_out


def look_at(eye, target, up=(0.0, 0.0, 1.0)):
    """Camera-to-world rotation (columns x right, y down, z forward)."""
    eye, target, up = (np.asarray(v, np.float64) for v in (eye, target, up))
    z = target - eye
    z /= np.linalg.norm(z)
    x = np.cross(z, up)
    x /= np.linalg.norm(x)
    y = np.cross(z, x)
    return np.stack([x, y, z], axis=1)


# -- scenes ---------------------------------------------------------------------

def room_scene(seed, size=(6.0, 6.0, 3.0), n_boxes=5, n_spheres=3, device="cpu"):
    """Box room with random axis-aligned boxes and spheres (cfg1 / cfg3)."""
    g = np.random.default_rng(seed)
    sx, sy, sz = size
    boxes, spheres = [], []
    for _ in range(n_boxes):
        w = g.uniform(0.3, 1.0, 2)
        h = g.uniform(0.3, 1.5)
        c = g.uniform([-sx / 2 + 0.6, -sy / 2 + 0.6], [sx / 2 - 0.6, sy / 2 - 0.6])
        boxes.append([c[0] - w[0] / 2, c[1] - w[1] / 2, 0.0, c[0] + w[0] / 2, c[1] + w[1] / 2, h])
    for _ in range(n_spheres):
        r = g.uniform(0.15, 0.4)
        c = g.uniform([-sx / 2 + 0.5, -sy / 2 + 0.5, r], [sx / 2 - 0.5, sy / 2 - 0.5, 1.5])
        spheres.append([c[0], c[1], c[2], r])
    n_obj = 3 + n_boxes + n_spheres
    f64 = dict(dtype=torch.float64, device=device)
    return Scene(
        boxes=torch.tensor(boxes, **f64).reshape(-1, 6),
        box_cls=torch.arange(4, 4 + n_boxes, device=device),
        cyls=torch.zeros((0, 5), **f64), cyl_cls=torch.zeros(0, dtype=torch.int64, device=device),
        spheres=torch.tensor(spheres, **f64).reshape(-1, 4),
        sph_cls=torch.arange(4 + n_boxes, 4 + n_boxes + n_spheres, device=device),
        ground_cls=0, room=(-sx / 2, -sy / 2, 0.0, sx / 2, sy / 2, sz), room_cls=(1, 2, 3),
        n_objects=n_obj)


def street_scene(seed, n_buildings=40, n_poles=60, length=200.0, device="cpu"):
    """Straight road along +x with box buildings and pole cylinders (cfg2)."""
    g = np.random.default_rng(seed)
    boxes, cyls = [], []
    for _ in range(n_buildings):
        side = g.choice([-1.0, 1.0])
        x0 = g.uniform(-20.0, length)
        w = g.uniform(6.0, 20.0)
        dpt = g.uniform(6.0, 15.0)
        y0 = side * g.uniform(8.0, 14.0)
        y1 = y0 + side * dpt
        boxes.append([x0, min(y0, y1), 0.0, x0 + w, max(y0, y1), g.uniform(4.0, 25.0)])
    for _ in range(n_poles):
        side = g.choice([-1.0, 1.0])
        cyls.append([g.uniform(-20.0, length), side * g.uniform(5.0, 7.5), g.uniform(0.08, 0.3),
                     0.0, g.uniform(3.0, 9.0)])
    f64 = dict(dtype=torch.float64, device=device)
    return Scene(
        boxes=torch.tensor(boxes, **f64), box_cls=torch.full((n_buildings,), 2, device=device),
        cyls=torch.tensor(cyls, **f64), cyl_cls=torch.full((n_poles,), 3, device=device),
        spheres=torch.zeros((0, 4), **f64), sph_cls=torch.zeros(0, dtype=torch.int64, device=device),
        ground_cls=1, n_objects=3)


def city_scene(seed, extent=1000.0, block=50.0, n_poles=400, device="cpu"):
    """Grid city of box buildings with streets and poles (cfg4)."""
    g = np.random.default_rng(seed)
    boxes, cyls = [], []
    half = extent / 2
    street = 16.0
    for bx in np.arange(-half, half, block):
        for by in np.arange(-half, half, block):
            if g.uniform() < 0.15:
                continue
            x0, y0 = bx + street / 2, by + street / 2
            boxes.append([x0, y0, 0.0, x0 + block - street, y0 + block - street, g.uniform(6, 60)])
    for _ in range(n_poles):
        cx = (np.floor(g.uniform(-half, half) / block) * block + g.choice([2.0, -2.0]) + street / 2)
        cy = g.uniform(-half, half)
        cyls.append([cx, cy, g.uniform(0.1, 0.3), 0.0, g.uniform(3.0, 10.0)])
    f64 = dict(dtype=torch.float64, device=device)
    nb = len(boxes)
    cls_b = torch.tensor(g.integers(2, 30, nb), device=device)
    cls_c = torch.tensor(g.integers(30, 41, len(cyls)), device=device)
    return Scene(
        boxes=torch.tensor(boxes, **f64), box_cls=cls_b, cyls=torch.tensor(cyls, **f64),
        cyl_cls=cls_c, spheres=torch.zeros((0, 4), **f64),
        sph_cls=torch.zeros(0, dtype=torch.int64, device=device), ground_cls=1, n_objects=40)


def floor_scene(seed, size=(20.0, 20.0, 4.0), n_objects=200, device="cpu"):
    """Multi-room floor: outer walls, interior partition boxes and objects (cfg5)."""
    g = np.random.default_rng(seed)
    sx, sy, sz = size
    boxes = []
    for k in range(1, 4):   # partition walls with door gaps
        x = -sx / 2 + k * sx / 4
        boxes.append([x - 0.05, -sy / 2, 0.0, x + 0.05, -1.0, sz])
        boxes.append([x - 0.05, 1.0, 0.0, x + 0.05, sy / 2, sz])
    n_box = n_objects // 2
    for _ in range(n_box):
        w = g.uniform(0.2, 1.2, 2)
        c = g.uniform([-sx / 2 + 0.5, -sy / 2 + 0.5], [sx / 2 - 0.5, sy / 2 - 0.5])
        boxes.append([c[0] - w[0] / 2, c[1] - w[1] / 2, 0.0, c[0] + w[0] / 2, c[1] + w[1] / 2,
                      g.uniform(0.3, 2.0)])
    sph = []
    for _ in range(n_objects - n_box):
        r = g.uniform(0.1, 0.35)
        c = g.uniform([-sx / 2 + 0.5, -sy / 2 + 0.5, r], [sx / 2 - 0.5, sy / 2 - 0.5, 2.5])
        sph.append([c[0], c[1], c[2], r])
    f64 = dict(dtype=torch.float64, device=device)
    nb = len(boxes)
    return Scene(
        boxes=torch.tensor(boxes, **f64), box_cls=torch.arange(4, 4 + nb, device=device),
        cyls=torch.zeros((0, 5), **f64), cyl_cls=torch.zeros(0, dtype=torch.int64, device=device),
        spheres=torch.tensor(sph, **f64).reshape(-1, 4),
        sph_cls=torch.arange(4 + nb, 4 + nb + len(sph), device=device),
        ground_cls=0, room=(-sx / 2, -sy / 2, 0.0, sx / 2, sy / 2, sz), room_cls=(1, 2, 3),
        n_objects=3 + nb + len(sph))


# -- sensors --------------------------------------------------------------------

def depth_camera_dirs(width, height, fx, fy, cx=None, cy=None, device="cpu"):
    """Unit ray directions (camera frame, z forward) and per-pixel z scale."""
    cx = (width / 2.0) if cx is None else cx
    cy = (height / 2.0) if cy is None else cy
    u = torch.arange(width, dtype=torch.float64, device=device)
    v = torch.arange(height, dtype=torch.float64, device=device)
    vv, uu = torch.meshgrid(v, u, indexing="ij")
    d = torch.stack([(uu - cx) / fx, (vv - cy) / fy, torch.ones_like(uu)], dim=-1).reshape(-1, 3)
    norm = d.norm(dim=1, keepdim=True)
    return d / norm, 1.0 / norm[:, 0]


def lidar_dirs(rows, cols, fov_deg, device="cpu"):
    """Spinning-LiDAR beam directions (sensor frame, z up)."""
    el = torch.linspace(-fov_deg, fov_deg, rows, dtype=torch.float64, device=device) * math.pi / 180
    az = torch.arange(cols, dtype=torch.float64, device=device) * (2 * math.pi / cols)
    ee, aa = torch.meshgrid(el, az, indexing="ij")
    return torch.stack([torch.cos(ee) * torch.cos(aa), torch.cos(ee) * torch.sin(aa),
                        torch.sin(ee)], dim=-1).reshape(-1, 3)


@dataclass
class FrameData:
    """One frame: sensor-frame points (n,3) f32, pose 4x4 f64, world points
    f32, payload (labels int32 (n,) or features f32 (n,D)), true object ids."""

    points: torch.Tensor
    pose: np.ndarray
    points_world: torch.Tensor
    labels: torch.Tensor | None
    features: torch.Tensor | None
    truth: torch.Tensor
    depth: torch.Tensor | None = None    # depth cameras: (H, W) f32 z-depth, NaN = no return
    camera: dict | None = None           # CameraConfig fields of that raster

    @property
    def origin(self):
        return self.pose[:3, 3].copy()


def closed_labels(truth, num_classes, alpha, boost, wrong_frac, gen, device):
    """Per-point softmax drawn Dirichlet(alpha) with the true class boosted to
    ~boost; a `wrong_frac` fraction gets a uniformly random wrong peak.
    Returns argmax+1 (np.argmax tie rule) as int32 labels, the payload the
    reference's closed-set path consumes (fusion.py:244-250)."""
    n = truth.shape[0]
    conc = torch.full((n, num_classes), float(alpha), device=device, dtype=torch.float32)
    # torch's Dirichlet sampler has no generator argument: seed the global
    # stream from this frame's generator so frames stay reproducible
    torch.manual_seed(int(torch.randint(0, 2**62, (1,), generator=gen, device=device).item()))
    p = torch.distributions.Dirichlet(conc).sample() * (1.0 - boost)
    peak = (truth.clamp(1, num_classes) - 1).clone()
    if wrong_frac > 0:
        flip = torch.rand(n, generator=gen, device=device) < wrong_frac
        shift = torch.randint(1, num_classes, (n,), generator=gen, device=device)
        peak = torch.where(flip, (peak + shift) % num_classes, peak)
    p[torch.arange(n, device=device), peak] += boost
    return (torch.argmax(p, dim=1) + 1).to(torch.int32)


def object_embeddings(n_objects, dim, seed, device):
    g = torch.Generator(device="cpu").manual_seed(seed)
    c = torch.randn(n_objects + 1, dim, generator=g, dtype=torch.float32)
    return (c / c.norm(dim=1, keepdim=True)).to(device)


def open_features(truth, centres, noise, gen, device):
    z = centres[truth] + noise * torch.randn(truth.shape[0], centres.shape[1], generator=gen,
                                             device=device, dtype=torch.float32)
    return z / z.norm(dim=1, keepdim=True)


@dataclass
class Workload:
    """A BASELINE config: map settings plus a frame generator."""

    name: str
    n_frames: int
    points_per_frame: int
    mapper_kwargs: dict
    make_frame: object = None
    queries: torch.Tensor | None = None
    info: dict = field(default_factory=dict)

    def frames(self, start=0, stop=None):
        stop = self.n_frames if stop is None else min(stop, self.n_frames)
        for i in range(start, stop):
            yield self.make_frame(i)


def _camera_workload(name, scene, width, height, f, n_frames, radius, height_m, noise, seed,
                     mapper_kwargs, payload, device, num_classes=0, dim=0, n_queries=0,
                     wrong_frac=0.0, scale=1.0):
    dirs_cam, zscale = depth_camera_dirs(width, height, f, f, device=device)
    centres = object_embeddings(scene.n_objects, dim, seed + 7, device) if dim else None

    def make_frame(i):
        gen = torch.Generator(device=device).manual_seed(seed * 100003 + i)
        ang = 2 * math.pi * i / max(n_frames, 1)
        eye = np.array([radius * math.cos(ang), radius * math.sin(ang), height_m])
        R = look_at(eye, np.array([0.0, 0.0, 1.0 * scale]))
        pose = np.eye(4)
        pose[:3, :3] = R
        pose[:3, 3] = eye
        Rt = torch.tensor(R, dtype=torch.float64, device=device)
        o = torch.tensor(eye, dtype=torch.float64, device=device)
        dw = dirs_cam @ Rt.T
        t, cls = raycast(scene, o[None, :], dw)
        # depth noise on the z-depth, carried along the ray
        depth = t * zscale + noise * torch.randn(t.shape[0], generator=gen, device=device,
                                                 dtype=torch.float64)
        rng = depth / zscale
        pw = (o[None, :] + rng[:, None] * dw).to(torch.float32)
        pw[~torch.isfinite(t)] = float("nan")
        ps = ((pw.to(torch.float64) - o[None, :]) @ Rt).to(torch.float32)
        truth = cls
        labels = feats = None
        if payload == "closed":
            labels = closed_labels(truth, num_classes, 0.5, 0.7, wrong_frac, gen, device)
        else:
            feats = open_features(truth, centres, 0.05, gen, device)
        depth_raster = depth.to(torch.float32).reshape(height, width)
        depth_raster[~torch.isfinite(t).reshape(height, width)] = float("nan")
        camera = dict(fx=float(f), fy=float(f), cx=width / 2.0, cy=height / 2.0, width=width,
                      height=height, depth_scale=1.0, stride=1)
        return FrameData(ps, pose, pw, labels, feats, truth, depth_raster, camera)

    queries = None
    if n_queries:
        g = torch.Generator(device="cpu").manual_seed(seed + 11)
        q = torch.randn(n_queries, dim, generator=g, dtype=torch.float64)
        queries = (q / q.norm(dim=1, keepdim=True)).to(device)
    return Workload(name, n_frames, width * height, mapper_kwargs, make_frame, queries)


def _lidar_workload(name, scene, rows, cols, fov, max_range, n_frames, step, height_m, noise,
                    seed, mapper_kwargs, num_classes, alpha, wrong_frac, device, loop_radius=None):
    dirs = lidar_dirs(rows, cols, fov, device=device)

    def make_frame(i):
        gen = torch.Generator(device=device).manual_seed(seed * 100003 + i)
        if loop_radius is None:
            eye = np.array([step * i, 0.0, height_m])
            R = np.eye(3)
        else:
            ang = step * i / loop_radius
            eye = np.array([loop_radius * math.cos(ang), loop_radius * math.sin(ang), height_m])
            yaw = ang + math.pi / 2
            R = np.array([[math.cos(yaw), -math.sin(yaw), 0.0],
                          [math.sin(yaw), math.cos(yaw), 0.0], [0.0, 0.0, 1.0]])
        pose = np.eye(4)
        pose[:3, :3] = R
        pose[:3, 3] = eye
        Rt = torch.tensor(R, dtype=torch.float64, device=device)
        o = torch.tensor(eye, dtype=torch.float64, device=device)
        dw = dirs @ Rt.T
        t, cls = raycast(scene, o[None, :], dw)
        t = torch.where(t <= max_range, t, torch.full_like(t, math.inf))
        rng = t + noise * torch.randn(t.shape[0], generator=gen, device=device, dtype=torch.float64)
        # sensor-frame points: with an identity rotation the world points are
        # exactly ps + t in float64, which is what the reference computes
        ps = (rng[:, None] * dirs).to(torch.float32)
        ps[~torch.isfinite(t)] = float("nan")
        pw = (ps.to(torch.float64) @ Rt.T + o[None, :]).to(torch.float32)
        labels = closed_labels(cls, num_classes, alpha, 0.7, wrong_frac, gen, device)
        return FrameData(ps, pose, pw, labels, None, cls)

    return Workload(name, n_frames, rows * cols, mapper_kwargs, make_frame)


def workload(cfg: int, device="cpu", seed=None, scale_frames=None, small=False,
             dim=None) -> Workload:
    """BASELINE.json configs[cfg-1] (1-based cfg).  `small` shrinks sensors
    for CPU tests (same geometry and value distributions); `dim` overrides the
    open-set embedding dimension (small sensors with the BASELINE D = 512 /
    768 for reference-generated fixtures)."""
    if cfg == 1:
        s = 1 if seed is None else seed
        scene = room_scene(s, device=device)
        w, h, f = (80, 60, 75.0) if small else (320, 240, 300.0)
        return _camera_workload("cfg1_closed_room_320x240", scene, w, h, f, 20, 1.5, 1.2, 0.01, s,
                                dict(voxel_size=0.05, truncation=0.15, max_range=15.0,
                                     num_classes=20), "closed", device, num_classes=20)
    if cfg == 2:
        s = 2 if seed is None else seed
        scene = street_scene(s, device=device)
        rows, cols = (16, 256) if small else (64, 1024)
        return _lidar_workload("cfg2_closed_lidar_64x1024", scene, rows, cols, 15.0, 80.0, 100, 1.0,
                               1.73, 0.02, s,
                               dict(voxel_size=0.1, truncation=0.3, max_range=80.0,
                                    num_classes=20), 20, 0.5, 0.10, device)
    if cfg == 3:
        s = 3 if seed is None else seed
        scene = room_scene(s, size=(8.0, 8.0, 3.0), n_boxes=8, n_spheres=4, device=device)
        w, h, f = (64, 48, 52.5) if small else (640, 480, 525.0)
        dim = dim or (32 if small else 512)
        return _camera_workload("cfg3_open_room_640x480_D512", scene, w, h, f, 50, 2.0, 1.2, 0.01,
                                s, dict(voxel_size=0.04, truncation=0.12, max_range=15.0,
                                        feature_dim=dim), "open", device, dim=dim, n_queries=32)
    if cfg == 4:
        s = 4 if seed is None else seed
        scene = city_scene(s, device=device)
        rows, cols = (16, 256) if small else (128, 2048)
        return _lidar_workload("cfg4_closed_lidar_128x2048", scene, rows, cols, 22.5, 120.0, 200,
                               1.0, 1.73, 0.02, s,
                               dict(voxel_size=0.05, truncation=0.15, max_range=120.0,
                                    num_classes=40), 40, 0.3, 0.0, device, loop_radius=150.0)
    if cfg == 5:
        s = 5 if seed is None else seed
        scene = floor_scene(s, device=device)
        w, h, f = (64, 36, 45.0) if small else (1280, 720, 900.0)
        dim = dim or (32 if small else 768)
        return _camera_workload("cfg5_open_floor_1280x720_D768", scene, w, h, f, 300, 6.0, 1.4,
                                0.01, s, dict(voxel_size=0.03, truncation=0.09, max_range=30.0,
                                              feature_dim=dim), "open", device, dim=dim,
                                n_queries=128)
    raise ValueError(f"unknown config {cfg}")

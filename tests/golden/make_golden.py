"""Generate the golden fixtures that pin the oracle and the engine to the
reference implementation itself.

Runs ONLY in the build container, where the read-only reference package is
importable (it does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/bindings/src \
        python tests/golden/make_golden.py

Each scenario stores its inputs (so tests never depend on re-generating
them) and the reference's outputs:

  api_*   drive ``semvox_bindings.Mapper.integrate`` (the reference's public
          API, bindings/__init__.py:131-142) with identity-rotation poses, for
          which the reference's BLAS world transform is exact;
  seam_*  drive the reference backend seam ``integrate_points``
          (fusion.py:278-289) with world-frame float32 points and the frame
          prep of fusion.py:228-275 restated here (delta, t, masks, u), for
          rotated trajectories whose BLAS transform is not reproducible.

Outputs: per-frame IntegrationReport counts, active coords in the
reference's active order, TSDF d/w (f64), semantic fields, content hashes,
and readouts (label_map / grid_labels, cosine query, classify_means).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

REF = os.environ.get("SEMVOX_REF", "/root/reference/pkg")
for sub in ("src", "bindings/src"):
    p = os.path.join(REF, sub)
    if p not in sys.path:
        sys.path.insert(0, p)

import semvox  # noqa: E402
import semvox_bindings as sb  # noqa: E402
from semvox.dirichlet import label_map  # noqa: E402
from semvox.evalbench import grid_labels  # noqa: E402
from semvox.gaussian import classify_means, cosine_to_embeddings  # noqa: E402

REPORT_KEYS = ("points_in", "points_used", "skipped_nonfinite", "skipped_range",
               "skipped_degenerate", "skipped_bad_label", "band_hits", "touched_voxels")


def _reports_array(reps):
    return np.array([[getattr(r, k) if hasattr(r, k) else r[k] for k in REPORT_KEYS]
                     for r in reps], np.int64)


def _sha(a):
    import hashlib

    return np.array(hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest())


def _dump_state(out, tsdf, sem, sem_kind, queries=None, tau=0.01, tp=0.1, digest=False):
    coords, (d, w) = tsdf.active_values()
    out["coords"] = np.asarray(coords, np.int64)
    out["d"] = d
    out["w"] = w
    out["tsdf_hash"] = np.array(tsdf.content_hash())
    if sem is None:
        return
    scoords, svals = sem.active_values()
    assert np.array_equal(scoords, coords)
    out["sem_hash"] = np.array(sem.content_hash())
    if sem_kind == "closed":
        out["counts"] = svals[0]
        out["label_map"] = label_map(sem)[1].astype(np.int32)
        out["grid_labels"] = grid_labels(sem)[1]
    else:
        if digest:   # large D: SHA-256 of the exact arrays + the first rows for diagnostics
            out["mean_sha256"], out["beta_sha256"] = _sha(svals[0]), _sha(svals[1])
            out["mean_head"], out["beta_head"] = svals[0][:32], svals[1][:32]
        else:
            out["mean"], out["beta"] = svals
        if queries is not None:
            out["queries"] = queries
            out["cosine_q0"] = cosine_to_embeddings(svals[0], queries[:1])[:, 0]
            lab, best = classify_means(svals[0], w, queries, tau, tp)
            out["classify_labels"] = lab
            out["classify_best"] = best


def api_scenario(name, frames, mapper_kw, queries=None, feat_store=None):
    """frames: list of (points_sensor, pose, labels|None, feats|None).
    feat_store: None (features stored as given), "f16" (the features are
    exactly float16-representable and stored as float16), or ("basis", B,
    idx_list) (each frame's features are rows B[idx]; only B and idx are
    stored) -- keeps the large-D fixtures small; the loader rebuilds the
    exact float32 inputs (tests/helpers.py load_golden)."""
    m = sb.Mapper(**mapper_kw)
    reps = []
    for pts, pose, lab, feat in frames:
        reps.append(m.integrate(pts, pose, labels=lab, features=feat))
    tsdf, sem = m.grids
    kind = "closed" if mapper_kw.get("num_classes") else ("open" if mapper_kw.get("feature_dim") else None)
    out = {"mode": np.array("api"), "reports": _reports_array(reps)}
    for i, (pts, pose, lab, feat) in enumerate(frames):
        out[f"points_{i}"] = pts
        out[f"pose_{i}"] = pose
        if lab is not None:
            out[f"labels_{i}"] = lab
        if feat is not None:
            if feat_store == "f16":
                f16 = feat.astype(np.float16)
                assert np.array_equal(f16.astype(feat.dtype), feat)
                out[f"features16_{i}"] = f16
            elif isinstance(feat_store, tuple):
                basis, idxs = feat_store[1], feat_store[2]
                assert np.array_equal(basis[idxs[i]], feat)
                out["featbasis"] = basis
                out[f"featidx_{i}"] = idxs[i]
            else:
                out[f"features_{i}"] = feat
    out["n_frames"] = np.array(len(frames))
    out["mapper_kw"] = np.array(repr(mapper_kw))
    _dump_state(out, tsdf, sem, kind, queries, digest=feat_store is not None)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, "frames", len(frames), "active", out["coords"].shape[0])


def seam_integrate(tsdf, sem, kind, fusion, pw, origin, labels, feats):
    """fusion.py:228-293 from the world points on, then the backend seam."""
    pw = np.asarray(pw, np.float64)
    origin = np.asarray(origin, np.float64)
    rep = {k: 0 for k in REPORT_KEYS}
    rep["points_in"] = pw.shape[0]
    finite = np.isfinite(pw).all(axis=1)
    rep["skipped_nonfinite"] = int((~finite).sum())
    delta = pw - origin
    with np.errstate(invalid="ignore"):
        t = np.sqrt((delta * delta).sum(axis=1))
    t = np.where(np.isfinite(t), t, np.inf)
    degenerate = finite & (t == 0.0)
    rep["skipped_degenerate"] = int(degenerate.sum())
    in_range = t <= fusion.max_range
    rep["skipped_range"] = int((finite & ~degenerate & ~in_range).sum())
    keep = finite & ~degenerate & in_range
    if kind == "closed":
        k = sem.payload.cfg.num_classes
        good = (labels >= 1) & (labels <= k)
        rep["skipped_bad_label"] = int((keep & ~good).sum())
        keep &= good
    elif kind == "open":
        good = np.isfinite(feats).all(axis=1)
        rep["skipped_bad_label"] = int((keep & ~good).sum())
        keep &= good
    idx = np.flatnonzero(keep)
    rep["points_used"] = int(idx.shape[0])
    if idx.shape[0] == 0:
        return rep
    tk = t[idx]
    u = delta[idx] / tk[:, None]
    params = {
        "voxel_size": fusion.voxel_size, "truncation": fusion.truncation,
        "weight_fn": 0 if fusion.weight_fn == "constant_one" else 1,
        "space_carving": fusion.space_carving,
        "num_classes": sem.payload.cfg.num_classes if kind == "closed" else 0,
        "lambda_floor": sem.payload.cfg.lambda_floor if kind == "open" else 1e-3,
        "last_wins": kind == "closed" and sem.payload.cfg.fusion == "last_wins",
    }
    kr = tsdf.backend.integrate_points(
        tsdf.core, sem.core if sem is not None else None, kind, origin, u, tk,
        np.ascontiguousarray(labels[idx], np.int32) if kind == "closed" else None,
        np.ascontiguousarray(feats[idx], np.float64) if kind == "open" else None, params, 1)
    rep["band_hits"] = kr["band_hits"]
    rep["touched_voxels"] = kr["touched_voxels"]
    return rep


def seam_scenario(name, frames, mapper_kw, queries=None):
    """frames: list of (points_world f32, origin, labels|None, feats|None)."""
    fkw = {k: v for k, v in mapper_kw.items()
           if k in ("voxel_size", "truncation", "weight_fn", "space_carving", "max_range")}
    fusion = semvox.FusionConfig(**fkw)
    closed = open_set = None
    kind = None
    if mapper_kw.get("num_classes"):
        kind = "closed"
        closed = semvox.ClosedSetConfig(num_classes=mapper_kw["num_classes"],
                                        fusion=mapper_kw.get("fusion", "bayes"))
    if mapper_kw.get("feature_dim"):
        kind = "open"
        open_set = semvox.OpenSetConfig(feature_dim=mapper_kw["feature_dim"])
    tsdf, sem = semvox.make_grids(fusion, closed=closed, open_set=open_set)
    reps = []
    out = {"mode": np.array("seam")}
    for i, (pw, origin, lab, feat) in enumerate(frames):
        reps.append(seam_integrate(tsdf, sem, kind, fusion, pw, origin, lab, feat))
        out[f"points_{i}"] = pw
        out[f"origin_{i}"] = np.asarray(origin, np.float64)
        if lab is not None:
            out[f"labels_{i}"] = lab
        if feat is not None:
            out[f"features_{i}"] = feat
    out["reports"] = _reports_array(reps)
    out["n_frames"] = np.array(len(frames))
    out["mapper_kw"] = np.array(repr(mapper_kw))
    _dump_state(out, tsdf, sem, kind, queries, digest=feat_store is not None)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, "frames", len(frames), "active", out["coords"].shape[0])


def plane_frames(seed, n, frames, labels_k=0, feat_dim=0, with_bad=True):
    """Sensor-frame points of the z = 0 square seen from above (identity
    rotation), plus invalid rows exercising every skip counter."""
    rng = np.random.default_rng(seed)
    out = []
    for i in range(frames):
        origin = np.array([0.1 * i, -0.05 * i, 2.0])
        world = np.column_stack([rng.uniform(-1.0, 1.0, (n, 2)), rng.normal(0, 0.01, n)])
        pts = world - origin
        if with_bad:
            pts[0] = np.nan                      # nonfinite
            pts[1] = (0.0, 0.0, 0.0)             # degenerate
            pts[2] = (50.0, 0.0, 0.0)            # out of range
        pose = np.eye(4)
        pose[:3, 3] = origin
        lab = feat = None
        if labels_k:
            lab = rng.integers(1, labels_k + 1, n).astype(np.int32)
            if with_bad:
                lab[3] = 0
                lab[4] = labels_k + 1
        if feat_dim:
            feat = rng.normal(size=(n, feat_dim)).astype(np.float32)
            if with_bad:
                feat[5, 0] = np.inf
        out.append((pts, pose, lab, feat))
    return out


def depth_scenario(name, mapper_kw, camera, frames):
    """The reference's depth path: ingest.project_depth (ingest.py:285-322)
    then Mapper.integrate on the Frame (identity rotations: exact BLAS).
    frames: list of (depth raster, payload raster, pose)."""
    from semvox.config import CameraConfig
    from semvox.ingest import project_depth

    intr = CameraConfig(**camera)
    m = sb.Mapper(**mapper_kw)
    reps = []
    out = {"mode": np.array("depth"), "camera": np.array(repr(camera))}
    for i, (depth, payload, pose) in enumerate(frames):
        fr = project_depth(depth, payload, intr, pose=pose, frame_id=i)
        out[f"depth_{i}"] = depth
        out[f"payload_{i}"] = payload
        out[f"pose_{i}"] = pose
        out[f"ref_points_{i}"] = fr.points
        reps.append(m.integrate(fr.points, pose, labels=fr.labels, features=fr.features))
    tsdf, sem = m.grids
    kind = "closed" if mapper_kw.get("num_classes") else ("open" if mapper_kw.get("feature_dim") else None)
    out["reports"] = _reports_array(reps)
    out["n_frames"] = np.array(len(frames))
    out["mapper_kw"] = np.array(repr(mapper_kw))
    _dump_state(out, tsdf, sem, kind)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, "frames", len(frames), "active", out["coords"].shape[0])


def depth_frames(seed, H, W, frames, labels_k=0, feat_dim=0, dtype=np.float32, scale=1.0):
    """A tilted wall seen by a camera translating along x (identity
    rotation), with zero, negative and non-finite depth pixels."""
    rng = np.random.default_rng(seed)
    out = []
    vv, uu = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
    for i in range(frames):
        z = 1.5 + 0.4 * uu / W + 0.2 * vv / H + rng.normal(0, 0.005, (H, W))
        raw = z / scale
        if np.issubdtype(dtype, np.integer):
            raw = np.round(raw).astype(dtype)
            raw[rng.random((H, W)) < 0.03] = 0
        else:
            raw = raw.astype(dtype)
            raw[rng.random((H, W)) < 0.03] = 0.0
            raw[rng.random((H, W)) < 0.02] = np.nan
            raw[rng.random((H, W)) < 0.01] = -1.0
        if labels_k:
            pay = rng.integers(0, labels_k + 1, (H, W)).astype(np.int64)
        else:
            pay = rng.normal(size=(H, W, feat_dim)).astype(np.float32)
        pose = np.eye(4)
        pose[:3, 3] = [0.05 * i, 0.0, 0.0]
        out.append((raw, pay, pose))
    return out


def main_depth():
    # -- depth frames (project_depth + integrate) ---------------------------------
    cam = dict(fx=50.0, fy=52.0, cx=31.5, cy=23.0, width=64, height=48, depth_scale=1.0, stride=1)
    depth_scenario("depth_closed_f32", dict(voxel_size=0.05, truncation=0.15, num_classes=5),
                   cam, depth_frames(11, 48, 64, 3, labels_k=5))
    cam2 = dict(cam, stride=2, depth_scale=0.001)
    depth_scenario("depth_closed_u16_stride2", dict(voxel_size=0.05, truncation=0.15, num_classes=5),
                   cam2, depth_frames(12, 48, 64, 2, labels_k=5, dtype=np.uint16, scale=0.001))
    depth_scenario("depth_open_f32_stride2", dict(voxel_size=0.05, truncation=0.15, feature_dim=4),
                   dict(cam, stride=2), depth_frames(13, 48, 64, 2, feat_dim=4))


def main_rotated():
    # -- rotated poses through the public API ---------------------------------------
    # Frame.points_world = points @ R.T + t goes through numpy/OpenBLAS; the
    # engine and the oracle evaluate it in the same fused-multiply-add order
    # (svx_internal.cuh world_coord), so rotated trajectories are pinned bit
    # for bit through Mapper.integrate too.  First check that order here.
    from fractions import Fraction

    def fma(a, b, c):
        return float(Fraction(a) * Fraction(b) + Fraction(c))

    rng = np.random.default_rng(21)
    for n in (1, 2, 3, 7, 64):
        q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
        pts = rng.normal(size=(n, 3)) * 5.0
        t = rng.normal(size=3)
        ref = pts @ q.T + t
        for i in range(n):
            for j in range(3):
                x, y, z = pts[i]
                acc = fma(q[j, 0], x, q[j, 1] * y) if n == 1 else fma(q[j, 1], y, q[j, 0] * x)
                assert fma(q[j, 2], z, acc) + t[j] == ref[i, j], (n, i, j)
    from paper_2512_12945_b200 import scenes

    wl = scenes.workload(1, small=True)
    fr = []
    for i in range(3):
        f = wl.make_frame(i)
        fr.append((f.points.numpy(), f.pose, f.labels.numpy(), None))
    api_scenario("api_closed_room_rotated", fr, wl.mapper_kwargs)
    wl = scenes.workload(4, small=True)
    fr = []
    for i in range(2):
        f = wl.make_frame(i)
        fr.append((f.points.numpy(), f.pose, f.labels.numpy(), None))
    api_scenario("api_closed_city_rotated", fr, wl.mapper_kwargs)
    wl = scenes.workload(3, small=True)
    fr = []
    dim = 16
    for i in range(2):
        f = wl.make_frame(i)
        fr.append((f.points.numpy()[::2], f.pose, None,
                   np.ascontiguousarray(f.features.numpy()[::2, :dim])))
    api_scenario("api_open_room_rotated", fr, dict(wl.mapper_kwargs, feature_dim=dim),
                 queries=np.ascontiguousarray(wl.queries[:4, :dim].numpy()))
    # tiny frames (1, 2, 3 points): numpy's one-row product takes another path
    rng = np.random.default_rng(22)
    fr = []
    for i in range(12):
        n = 1 + i % 3
        q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
        if np.linalg.det(q) < 0:
            q[:, 0] = -q[:, 0]
        pose = np.eye(4)
        pose[:3, :3] = q
        pose[:3, 3] = rng.uniform(-1.0, 1.0, 3)
        pts = rng.normal(size=(n, 3)) * 1.5
        fr.append((pts, pose, rng.integers(1, 4, n).astype(np.int32), None))
    api_scenario("api_closed_tiny_frames_rotated", fr,
                 dict(voxel_size=0.05, truncation=0.15, num_classes=3))


def main_snapshot():
    # -- .slvg snapshots written by the reference's Mapper.save -------------------
    # Re-runs the api_* fixtures' own inputs through the reference Mapper and
    # saves its snapshot (bindings/__init__.py:183-187), so the engine's
    # Mapper.save output can be compared byte for byte.
    for name in ("api_closed_plane", "api_open_plane", "api_geometry_carving_dropoff",
                 "api_closed_lastwins_dropoff"):
        g = np.load(os.path.join(HERE, name + ".npz"))
        kw = eval(str(g["mapper_kw"]))  # noqa: S307 -- our own repr() of a dict literal
        m = sb.Mapper(**kw)
        for i in range(int(g["n_frames"])):
            m.integrate(g[f"points_{i}"], g[f"pose_{i}"],
                        labels=g[f"labels_{i}"] if f"labels_{i}" in g else None,
                        features=g[f"features_{i}"] if f"features_{i}" in g else None)
        tsdf, sem = m.grids
        assert tsdf.content_hash() == str(g["tsdf_hash"])
        _save_gz(m, "snap_" + name[4:])
    _save_gz(sb.Mapper(voxel_size=0.1, truncation=0.2), "snap_empty")


def _mesh_out(out, prefix, mesh):
    out[prefix + "vertices"] = mesh.vertices
    out[prefix + "triangles"] = mesh.triangles
    out[prefix + "labels"] = mesh.labels
    out[prefix + "colors"] = mesh.colors


def _band_grid(cfg_kw, sdf, span, sem=None, seed=0, permute=False, weight=1.0):
    """A reference grid pair filled directly (no integration): every voxel
    whose centre is within the truncation of sdf's zero set."""
    from semvox import ClosedSetConfig, FusionConfig, OpenSetConfig, make_grids

    cfg = FusionConfig(**cfg_kw)
    kw = {}
    if sem and sem[0] == "closed":
        kw["closed"] = ClosedSetConfig(num_classes=sem[1])
    elif sem:
        kw["open_set"] = OpenSetConfig(feature_dim=sem[1])
    tsdf, sg = make_grids(cfg, **kw)
    g = np.stack(np.meshgrid(*[np.arange(-span, span + 1)] * 3, indexing="ij"), -1).reshape(-1, 3)
    d = sdf((g + 0.5) * cfg.voxel_size)
    keep = np.abs(d) <= cfg.truncation
    coords, d = g[keep], d[keep]
    rng = np.random.default_rng(seed)
    if permute:
        p = rng.permutation(len(d))
        coords, d = coords[p], d[p]
    w = np.where(rng.random(len(d)) < 0.1, 0.3, weight)      # some voxels below min_weight
    tsdf.set_many(coords, [d, w])
    if sg is not None and sem[0] == "closed":
        counts = rng.integers(0, 3, (len(d), sem[1])).astype(np.float32)
        counts[rng.random(len(d)) < 0.1] = 0.0                # some voxels without counts
        sg.set_many(coords, [counts])
    elif sg is not None:
        mean = rng.normal(size=(len(d), sem[1])).astype(np.float32)
        mean[rng.random(len(d)) < 0.05] = 0.0
        sg.set_many(coords, [mean, np.ones_like(mean)])
    return tsdf, sg


def main_mesh():
    # -- surface extraction (extract_mesh, mesh.py:419-545) -------------------------
    from semvox import extract_mesh, save_grids

    # maps integrated by the api_* fixtures
    for name, variants in (("api_closed_plane", [dict()]),
                           ("api_open_plane", [dict(), dict(emb=True)]),
                           ("api_geometry_carving_dropoff", [dict(), dict(min_weight=0.0),
                                                             dict(min_weight=2.0)])):
        g = np.load(os.path.join(HERE, name + ".npz"))
        kw = eval(str(g["mapper_kw"]))  # noqa: S307 -- our own repr() of a dict literal
        m = sb.Mapper(**kw)
        for i in range(int(g["n_frames"])):
            m.integrate(g[f"points_{i}"], g[f"pose_{i}"],
                        labels=g[f"labels_{i}"] if f"labels_{i}" in g else None,
                        features=g[f"features_{i}"] if f"features_{i}" in g else None)
        out = {}
        for j, v in enumerate(variants):
            emb = g["queries"] if v.get("emb") else None
            mesh = m.extract(min_weight=v.get("min_weight", 0.5), embeddings=emb)
            _mesh_out(out, f"v{j}_", mesh)
            out[f"v{j}_min_weight"] = np.array(v.get("min_weight", 0.5))
            out[f"v{j}_emb"] = np.array(bool(v.get("emb")))
            print(name, j, mesh.n_vertices, mesh.n_triangles)
        out["n_variants"] = np.array(len(variants))
        np.savez_compressed(os.path.join(HERE, "mesh_" + name[4:] + ".npz"), **out)

    # grids filled directly, loaded through their snapshots
    cfg = dict(voxel_size=0.05, truncation=0.15)
    c = np.array([0.013, -0.004, 0.021])
    sphere = lambda p: np.linalg.norm(p - c, axis=-1) - 0.5              # noqa: E731
    # a level set through voxel centres: corners exactly on it collapse edges
    lattice = lambda p: p[:, 2] - 0.025 - 0.0 * p[:, 0]                   # noqa: E731
    wavy = lambda p: p[:, 2] - 0.1 * np.sin(7.0 * p[:, 0]) * np.cos(5.0 * p[:, 1])  # noqa: E731
    scenes = [("sphere_closed", sphere, 14, ("closed", 4), {}),
              ("sphere_open", sphere, 14, ("open", 5), {}),
              ("lattice_plane", lattice, 10, None, {}),
              ("wavy_closed_permuted", wavy, 12, ("closed", 3), dict(permute=True))]
    import tempfile

    for stem, sdf, span, sem, extra in scenes:
        tsdf, sg = _band_grid(cfg, sdf, span, sem, seed=len(stem), **extra)
        with tempfile.TemporaryDirectory() as td:
            tmp = os.path.join(td, "g.slvg")
            save_grids(tmp, [x for x in (tsdf, sg) if x is not None])
            with open(tmp, "rb") as fh:
                raw = fh.read()
        import gzip

        with gzip.GzipFile(os.path.join(HERE, f"meshsnap_{stem}.slvg.gz"), "wb", mtime=0) as fh:
            fh.write(raw)
        out = {}
        variants = [dict(), dict(min_weight=0.1)]
        if sem and sem[0] == "open":
            q = np.random.default_rng(9).normal(size=(3, sem[1]))
            out["queries"] = q
            variants.append(dict(emb=True))
        for j, v in enumerate(variants):
            mesh = extract_mesh(tsdf, sg, min_weight=v.get("min_weight", 0.5),
                                embeddings=out["queries"] if v.get("emb") else None)
            _mesh_out(out, f"v{j}_", mesh)
            out[f"v{j}_min_weight"] = np.array(v.get("min_weight", 0.5))
            out[f"v{j}_emb"] = np.array(bool(v.get("emb")))
            if j == 0:   # the reference's PLY text of this mesh (write_ply, mesh.py:580-600)
                from semvox import write_ply

                with tempfile.TemporaryDirectory() as td2:
                    pp = os.path.join(td2, "m.ply")
                    write_ply(mesh, pp)
                    out["ply_v0"] = np.frombuffer(open(pp, "rb").read(), np.uint8)
            print(stem, j, mesh.n_vertices, mesh.n_triangles, len(raw))
        out["n_variants"] = np.array(len(variants))
        np.savez_compressed(os.path.join(HERE, f"mesh_{stem}.npz"), **out)


def main_render():
    # -- ray-march rendering (render.py:214-272) -------------------------------------
    import gzip

    from semvox import RenderCamera, load_grids, render

    from cameras import RENDER_CAMERAS

    def cam(name):
        pose, w, h, f, near, far = RENDER_CAMERAS[name]
        return RenderCamera(pose=pose.copy(), fx=f, fy=f * 1.05, cx=w / 2.0 - 0.3,
                            cy=h / 2.0 + 0.2, width=w, height=h, near=near, far=far)

    def shoot(out, tsdf, sem, cams, emb=None):
        for c in cams:
            out[f"{c}_depth"] = render(tsdf, sem, cam(c), mode="depth")
            out[f"{c}_normal"] = render(tsdf, sem, cam(c), mode="normal")
            if sem is not None:
                out[f"{c}_semantic"] = render(tsdf, sem, cam(c), mode="semantic")
                if emb is not None:
                    out[f"{c}_semantic_emb"] = render(tsdf, sem, cam(c), mode="semantic",
                                                      embeddings=emb)
            print("render", c, int((out[f"{c}_depth"] > 0).sum()), "hits")
        out["cameras"] = np.array(list(cams))

    # grids from the mesh snapshots
    for stem, cams in (("sphere_closed", ["front", "oblique"]),
                       ("sphere_open", ["front"]),
                       ("lattice_plane", ["down", "down_far_cut", "down_near_skip"])):
        with gzip.open(os.path.join(HERE, f"meshsnap_{stem}.slvg.gz"), "rb") as fh:
            raw = fh.read()
        import tempfile

        with tempfile.TemporaryDirectory() as td:
            p = os.path.join(td, "g.slvg")
            with open(p, "wb") as fh:
                fh.write(raw)
            grids = load_grids(p)
        tsdf, sem = grids[0], (grids[1] if len(grids) > 1 else None)
        out = {}
        emb = None
        if stem == "sphere_open":
            emb = np.random.default_rng(9).normal(size=(3, 5))
            out["queries"] = emb
        shoot(out, tsdf, sem, cams, emb)
        np.savez_compressed(os.path.join(HERE, f"render_{stem}.npz"), **out)
    # an integrated map (api_closed_plane) seen from above
    g = np.load(os.path.join(HERE, "api_closed_plane.npz"))
    kw = eval(str(g["mapper_kw"]))  # noqa: S307 -- our own repr() of a dict literal
    m = sb.Mapper(**kw)
    for i in range(int(g["n_frames"])):
        m.integrate(g[f"points_{i}"], g[f"pose_{i}"], labels=g[f"labels_{i}"])
    tsdf, sem = m.grids
    out = {}
    shoot(out, tsdf, sem, ["down", "oblique"])
    np.savez_compressed(os.path.join(HERE, "render_closed_plane.npz"), **out)


def _save_gz(mapper, stem):
    import gzip
    import tempfile

    with tempfile.TemporaryDirectory() as td:
        tmp = os.path.join(td, "map.slvg")
        mapper.save(tmp)
        with open(tmp, "rb") as fh:
            raw = fh.read()
    path = os.path.join(HERE, stem + ".slvg.gz")
    with gzip.GzipFile(path, "wb", mtime=0) as fh:
        fh.write(raw)
    print(path, len(raw), "bytes,", os.path.getsize(path), "compressed")


def main_bigdim():
    """Open-set fixtures at the BASELINE embedding dims (cfg3 D = 512 with its
    32 queries, cfg5 D = 768 with its 128 queries) and a close wall at D = 768
    whose band voxels collect > 8192 rows each (the engine's dimension-sliced
    huge-voxel path, 24 slices of 32 dims)."""
    from paper_2512_12945_b200 import scenes

    for cfg, stem, step in ((3, "api_open_room_d512", 6), (5, "api_open_floor_d768", 6)):
        wl = scenes.workload(cfg, small=True, dim=512 if cfg == 3 else 768)
        fr = []
        for i in range(2):
            f = wl.make_frame(i * 3)
            feats = f.features.numpy()[::step].astype(np.float16).astype(np.float32)
            fr.append((np.ascontiguousarray(f.points.numpy()[::step]), f.pose, None,
                       np.ascontiguousarray(feats)))
        api_scenario(stem, fr, wl.mapper_kwargs, queries=np.ascontiguousarray(wl.queries.numpy()),
                     feat_store="f16")
    rng = np.random.default_rng(768)
    D = 768
    basis = rng.normal(size=(8, D)).astype(np.float32)
    fr, idxs = [], []
    for f in range(2):
        n = 9000 + 1500 * f
        pts = np.column_stack([1.0 + rng.normal(0.0, 0.002, n), rng.uniform(-0.012, 0.012, n),
                               rng.uniform(-0.012, 0.012, n)])
        pose = np.eye(4)
        pose[:3, 3] = [0.015 + 0.002 * f, 0.015, 0.015]
        idx = rng.integers(0, 8, n).astype(np.uint8)
        idxs.append(idx)
        fr.append((pts, pose, None, basis[idx]))
    q = rng.normal(size=(128, D))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    api_scenario("api_open_wall_d768", fr, dict(voxel_size=0.03, truncation=0.09, feature_dim=D,
                                                max_range=5.0),
                 queries=q, feat_store=("basis", basis, idxs))


def main():
    from paper_2512_12945_b200 import scenes

    if "bigdim" in sys.argv[1:]:
        main_bigdim()
        return

    if "depth" in sys.argv[1:]:   # only the depth scenarios
        main_depth()
        return
    if "snapshot" in sys.argv[1:]:
        main_snapshot()
        return
    if "mesh" in sys.argv[1:]:
        main_mesh()
        return
    if "rotated" in sys.argv[1:]:
        main_rotated()
        return
    if "render" in sys.argv[1:]:
        main_render()
        return
    main_depth()

    # -- API level ------------------------------------------------------------
    api_scenario("api_closed_plane", plane_frames(0, 600, 4, labels_k=4),
                 dict(voxel_size=0.05, truncation=0.15, num_classes=4))
    api_scenario("api_open_plane", plane_frames(1, 400, 3, feat_dim=6),
                 dict(voxel_size=0.05, truncation=0.15, feature_dim=6),
                 queries=np.random.default_rng(5).normal(size=(4, 6)))
    api_scenario("api_geometry_carving_dropoff", plane_frames(2, 300, 2),
                 dict(voxel_size=0.05, truncation=0.15, space_carving=True,
                      weight_fn="linear_dropoff"))
    api_scenario("api_closed_lastwins_dropoff", plane_frames(3, 400, 3, labels_k=5),
                 dict(voxel_size=0.04, truncation=0.12, num_classes=5, fusion="last_wins",
                      weight_fn="linear_dropoff"))
    wl = scenes.workload(2, small=True)
    fr = []
    for i in range(3):
        f = wl.make_frame(i)
        fr.append((f.points.numpy(), f.pose, f.labels.numpy(), None))
    api_scenario("api_closed_lidar_small", fr, wl.mapper_kwargs)
    # -- backend seam, rotated trajectories --------------------------------------
    wl = scenes.workload(1, small=True)
    fr = []
    for i in range(3):
        f = wl.make_frame(i)
        fr.append((f.points_world.numpy(), f.origin, f.labels.numpy(), None))
    seam_scenario("seam_closed_room_small", fr, wl.mapper_kwargs)
    wl = scenes.workload(3, small=True)
    fr = []
    dim = 16   # keep the fixture small: first 16 embedding dims, every 2nd pixel
    for i in range(2):
        f = wl.make_frame(i)
        fr.append((f.points_world.numpy()[::2], f.origin, None,
                   np.ascontiguousarray(f.features.numpy()[::2, :dim])))
    kw = dict(wl.mapper_kwargs, feature_dim=dim)
    seam_scenario("seam_open_room_small", fr, kw,
                  queries=np.ascontiguousarray(wl.queries[:4, :dim].numpy()))
    wl = scenes.workload(4, small=True)
    fr = []
    for i in range(2):
        f = wl.make_frame(i)
        fr.append((f.points_world.numpy(), f.origin, f.labels.numpy(), None))
    seam_scenario("seam_closed_city_small", fr, wl.mapper_kwargs)
    main_rotated()
    main_bigdim()
    main_snapshot()
    main_mesh()
    main_render()


if __name__ == "__main__":
    main()

"""Ray-march rendering: render / sample_distance
(render.py:88-272) on the GPU.

Fixtures (tests/golden/render_*.npz, make_golden.py render) hold images the
reference's own render() produced -- depth, normal and semantic modes, from
head-on, oblique (rotated) and top-down cameras, with far / near planes that
cut and skip the band -- for grids loaded from reference snapshots and for an
integrated map.  Bar: bit-exact images.  CPU tests pin the oracle
restatement (oracle/render.py) to them; GPU tests check the engine against
both.
"""

import gzip
import os

import numpy as np
import pytest

from helpers import GOLDEN, load_golden, replay_mapper

RENDERS = ["sphere_closed", "sphere_open", "lattice_plane", "closed_plane"]


def cameras():
    import importlib.util

    spec = importlib.util.spec_from_file_location("mg_cams", os.path.join(GOLDEN, "cameras.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def render_golden(stem):
    z = np.load(os.path.join(GOLDEN, f"render_{stem}.npz"))
    return {k: z[k] for k in z.files}


def cam_args(name):
    pose, w, h, f, near, far = cameras().RENDER_CAMERAS[name]
    return dict(pose=pose.copy(), fx=f, fy=f * 1.05, cx=w / 2.0 - 0.3, cy=h / 2.0 + 0.2,
                width=w, height=h, near=near, far=far)


def snap_raw(stem):
    with gzip.open(os.path.join(GOLDEN, f"meshsnap_{stem}.slvg.gz"), "rb") as fh:
        return fh.read()


def oracle_state(stem):
    from oracle.render import VoxelState
    from paper_2512_12945_b200 import snapshot
    from paper_2512_12945_b200.mapper import _split_blocks

    if stem == "closed_plane":
        g = load_golden("api_closed_plane")
        kw = g["mapper_kw"]
        return VoxelState(g["coords"], g["d"], g["w"], kw["voxel_size"], kw["truncation"],
                          "closed", g["counts"]), kw["num_classes"]
    t, s = _split_blocks(snapshot.parse(snap_raw(stem)))
    kind = None if s is None else ("closed" if s.kind == 1 else "open")
    return (VoxelState(t.coords(), t.fields[0], t.fields[1], t.voxel_size, t.params[0], kind,
                       None if s is None else s.fields[0]),
            1 if s is None else int(s.params[0]))


# ---- CPU ----------------------------------------------------------------------------------------


@pytest.mark.parametrize("stem", RENDERS)
def test_oracle_matches_reference_images(stem):
    from oracle import render as orc

    g = render_golden(stem)
    st, psize = oracle_state(stem)
    for cam in g["cameras"]:
        for mode in ("depth", "normal", "semantic"):
            key = f"{cam}_{mode}"
            if key not in g:
                continue
            a = cam_args(str(cam))
            got = orc.render(st, a["pose"], a["fx"], a["fy"], a["cx"], a["cy"], a["width"],
                             a["height"], a["near"], a["far"], mode=mode, palette_size=psize)
            assert np.array_equal(got, g[key]), key


def test_camera_validation():
    from paper_2512_12945_b200 import ConfigError, RenderCamera, UserInputError

    def cam(**kw):
        a = dict(pose=np.eye(4), fx=60.0, fy=60.0, cx=24.0, cy=18.0, width=48, height=36)
        a.update(kw)
        return RenderCamera(**a)

    for kw, msg in ((dict(near=0.0), "near"), (dict(near=2.0, far=1.0), "far"),
                    (dict(width=0), "dimensions"), (dict(fx=0.0), "focal")):
        with pytest.raises(ConfigError, match=msg):
            cam(**kw).validate()
    with pytest.raises(ConfigError, match="4x4"):
        cam(pose=np.zeros((3, 3))).validate()
    bad = np.eye(4)
    bad[3, 0] = 0.5
    with pytest.raises(ConfigError, match="bottom row"):
        cam(pose=bad).validate()
    mirror = np.eye(4)
    mirror[0, 0] = -1.0
    with pytest.raises(UserInputError, match="mirrored"):
        cam(pose=mirror).validate()


# ---- GPU ----------------------------------------------------------------------------------------


def engine_grids(stem, tmp_path):
    from paper_2512_12945_b200 import Mapper, load_grid

    if stem == "closed_plane":
        g = load_golden("api_closed_plane")
        m = Mapper(**g["mapper_kw"])
        replay_mapper(g, m)
        return m.grids
    p = tmp_path / "g.slvg"
    p.write_bytes(snap_raw(stem))
    return load_grid(p)


@pytest.mark.gpu
@pytest.mark.parametrize("stem", RENDERS)
def test_engine_matches_reference_images(stem, tmp_path):
    from paper_2512_12945_b200 import RenderCamera, render

    g = render_golden(stem)
    tsdf, sem = engine_grids(stem, tmp_path)
    for cam in g["cameras"]:
        for mode in ("depth", "normal", "semantic", "semantic_emb"):
            key = f"{cam}_{mode}"
            if key not in g:
                continue
            emb = g["queries"] if mode == "semantic_emb" else None
            img = render(tsdf, sem, RenderCamera(**cam_args(str(cam))),
                         mode="semantic" if emb is not None else mode, embeddings=emb)
            assert img.dtype == g[key].dtype and np.array_equal(img, g[key]), key


@pytest.mark.gpu
def test_render_checks_and_background(tmp_path):
    from paper_2512_12945_b200 import (ConfigError, Mapper, RenderCamera, SemvoxError, render,
                                       sample_distance)

    m = Mapper(voxel_size=0.05, truncation=0.15)
    cam = RenderCamera(**cam_args("front"))
    img = m.render(cam)
    assert img.shape == (30, 40) and not img.any()               # empty map: background
    with pytest.raises(ConfigError, match="mode"):
        m.render(cam, mode="albedo")
    with pytest.raises(ConfigError, match="semantic mode needs"):
        m.render(cam, mode="semantic")
    tsdf, sem = engine_grids("sphere_closed", tmp_path)
    with pytest.raises(SemvoxError, match="TSDF"):
        render(sem, None, cam)
    h0 = tsdf.content_hash()
    render(tsdf, sem, cam, mode="normal")
    assert tsdf.content_hash() == h0                              # rendering is read-only
    vals, valid = sample_distance(tsdf, np.array([[0.0, 0.0, 5.0], [0.013, -0.004, 0.521]]))
    assert not valid[0] and np.isnan(vals[0])
    assert valid[1] and abs(vals[1]) < 0.01


@pytest.mark.gpu
def test_sample_distance_matches_oracle(tmp_path):
    from paper_2512_12945_b200 import sample_distance

    tsdf, _ = engine_grids("wavy_closed_permuted", tmp_path)
    st, _ = oracle_state("wavy_closed_permuted")
    rng = np.random.default_rng(5)
    pts = rng.uniform([-0.6, -0.6, -0.2], [0.6, 0.6, 0.2], (3000, 3))
    vals, valid = sample_distance(tsdf, pts)
    want = [st.sample(list(p)) for p in pts]
    assert np.array_equal(valid, np.array([w[1] for w in want]))
    assert valid.sum() > 500
    assert np.array_equal(vals[valid], np.array([w[0] for w in want])[valid])


@pytest.mark.gpu
def test_render_full_size_map_vs_oracle():
    """A BASELINE cfg2 map (several frames of 64x1024 LiDAR) rendered from a
    rotated camera: every mode equals the oracle's image."""
    from oracle import render as orc
    from oracle.render import VoxelState
    from paper_2512_12945_b200 import Mapper, RenderCamera, scenes

    wl = scenes.workload(2, device="cuda")
    kw = dict(wl.mapper_kwargs)
    m = Mapper(**kw)
    f = None
    for i in range(4):
        f = wl.make_frame(i)
        m.integrate(f.points, f.pose, labels=f.labels)
    coords, d, w, s0, _ = m._export()
    st = VoxelState(coords, d, w, kw["voxel_size"], kw["truncation"], "closed", s0)
    pose = np.asarray(f.pose, np.float64).copy()
    # look along the sensor's +x (forward), tilted down a little
    c, s = np.cos(0.2), np.sin(0.2)
    cam_to_sensor = np.array([[0, -s, c], [-1, 0, 0], [0, -c, -s]], np.float64)
    pose[:3, :3] = pose[:3, :3] @ cam_to_sensor
    pose[2, 3] += 0.5
    cam = RenderCamera(pose=pose, fx=40.0, fy=40.0, cx=31.7, cy=23.6, width=64, height=48,
                       near=0.1, far=40.0)
    for mode in ("depth", "normal", "semantic"):
        img = m.render(cam, mode=mode)
        want = orc.render(st, cam.pose, cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height,
                          cam.near, cam.far, mode=mode, palette_size=kw["num_classes"])
        if mode == "depth":
            assert (img > 0).sum() > 300
        assert np.array_equal(img, want), mode


@pytest.mark.gpu
def test_compact_f32_map_queries_vs_oracle(tmp_path):
    """The compact layout (tsdf_dtype float32): marching cubes and rendering
    read the stored f32 pair as f64, exactly like the oracle run on the
    exported state; a snapshot of it stores f64 and loads back unchanged."""
    from oracle import mesh as om
    from oracle import render as orc
    from oracle.render import VoxelState
    from paper_2512_12945_b200 import Mapper, RenderCamera

    g = load_golden("api_closed_plane")
    kw = dict(g["mapper_kw"], tsdf_dtype="float32")
    m = Mapper(**kw)
    replay_mapper(g, m)
    coords, d, w, s0, _ = m._export()
    mesh = m.extract()
    want = om.extract(coords, d, w, kw["voxel_size"], 0.5, "closed", s0,
                      palette_size=kw["num_classes"])
    assert mesh.n_triangles > 100
    for a, b in zip((mesh.vertices, mesh.triangles, mesh.labels, mesh.colors), want):
        assert np.array_equal(a, b)
    st = VoxelState(coords, d, w, kw["voxel_size"], kw["truncation"], "closed", s0)
    cam = RenderCamera(**cam_args("down"))
    for mode in ("depth", "semantic"):
        img = m.render(cam, mode=mode)
        ref = orc.render(st, cam.pose, cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height,
                         cam.near, cam.far, mode=mode, palette_size=kw["num_classes"])
        assert np.array_equal(img, ref), mode
    p = tmp_path / "f32.slvg"
    m.save(p)
    m2 = Mapper.from_snapshot(p, tsdf_dtype="float32")
    c2, d2, w2, s2, _ = m2._export()
    assert np.array_equal(c2, coords) and np.array_equal(d2, d) and np.array_equal(w2, w)
    assert np.array_equal(s2, s0)


@pytest.mark.gpu
def test_absurd_far_plane_is_an_error_not_a_hang():
    from paper_2512_12945_b200 import Mapper, RenderCamera, UserInputError

    m = Mapper(voxel_size=0.05, truncation=0.15)
    cam = RenderCamera(pose=np.eye(4), fx=8.0, fy=8.0, cx=4.0, cy=3.0, width=8, height=6,
                       near=0.05, far=1e12)
    with pytest.raises(UserInputError, match="march steps"):
        m.render(cam)
    cam.far = 50.0
    assert not m.render(cam).any()

"""GPU parity: the CUDA engine (through the C ABI / Mapper) against the
reference's own outputs (golden fixtures) and against the CPU oracle.

Bar (north star): active voxel set + argmax labels bit-exact; TSDF, weights
and semantic statistics within 1e-5 relative.  With the reference TSDF layout
(tsdf_dtype="float64") the engine is in fact bit-exact everywhere, including
the reference's content hashes; the compact fp32 TSDF layout is bit-exact
against the oracle's fp32 mode and within tolerance of the reference.
"""

import numpy as np
import pytest

from helpers import (RTOL, assert_close_rel, golden_names, load_golden, open_state_matches,
                     oracle_for, replay_mapper, replay_oracle, report_rows)

pytestmark = pytest.mark.gpu
NAMES = golden_names()


def mapper_for(g, **extra):
    from paper_2512_12945_b200 import Mapper

    kw = dict(g["mapper_kw"])
    kw.update(extra)
    return Mapper(**kw)


@pytest.mark.parametrize("device_inputs", [False, True], ids=["host", "device"])
@pytest.mark.parametrize("name", NAMES)
def test_engine_matches_reference_fixture(name, device_inputs):
    g = load_golden(name)
    m = mapper_for(g)
    reps = replay_mapper(g, m, device_inputs=device_inputs)
    assert np.array_equal(report_rows(reps), g["reports"])
    tsdf, sem = m.grids
    coords, (d, w) = tsdf.active_values()
    assert np.array_equal(coords, g["coords"])           # active set and order
    assert np.array_equal(d, g["d"]) and np.array_equal(w, g["w"])
    assert tsdf.content_hash() == str(g["tsdf_hash"])     # the reference's own digest
    if sem is not None:
        assert sem.content_hash() == str(g["sem_hash"])
        _, vals = sem.active_values()
        if "counts" in g:
            assert np.array_equal(vals[0], g["counts"])
            assert np.array_equal(m.label_map()[1], g["label_map"])
            assert np.array_equal(m.label_map(zero_if_empty=True)[1], g["grid_labels"])
        else:
            assert open_state_matches(g, vals[0], vals[1])
    if "queries" in g:
        q = g["queries"]
        qc, sims = m.query(q[0])
        assert np.array_equal(qc, g["coords"])
        np.testing.assert_allclose(sims, g["cosine_q0"], rtol=1e-12, atol=1e-15)
        lab, best = m.classify(q)
        assert np.array_equal(lab, g["classify_labels"])
        np.testing.assert_allclose(best, g["classify_best"], rtol=1e-12)


@pytest.mark.parametrize("mode", ["auto", "slots", "segments", "leaves"])
@pytest.mark.parametrize("name", [n for n in NAMES if "open" not in n])
def test_pinned_host_inputs(name, mode):
    """Page-locked host arrays: slot-mode frames read them in place
    (zero-copy walk), segment-mode frames copy them first; same bits."""
    g = load_golden(name)
    m = mapper_for(g)
    m.set_update_mode(mode)
    reps = replay_mapper(g, m, pinned=True)
    assert np.array_equal(report_rows(reps), g["reports"])
    tsdf, sem = m.grids
    assert tsdf.content_hash() == str(g["tsdf_hash"])
    if sem is not None:
        assert sem.content_hash() == str(g["sem_hash"])


@pytest.mark.parametrize("name", NAMES)
def test_compact_tsdf_vs_oracle_and_reference(name):
    g = load_golden(name)
    m = mapper_for(g, tsdf_dtype="float32")
    replay_mapper(g, m)
    om = oracle_for(g, tsdf_dtype="float32")
    replay_oracle(g, om)
    coords, d, w, s0, s1 = m._export()
    oc, od, ow, os0, os1 = om.export()
    assert np.array_equal(coords, oc) and np.array_equal(coords, g["coords"])
    assert np.array_equal(d, od) and np.array_equal(w, ow)   # bit-exact vs fp32 oracle
    trunc = float(g["mapper_kw"].get("truncation", 0.1))
    assert_close_rel(w, g["w"], what="w")
    assert_close_rel(d, g["d"], atol=1e-5 * trunc, what="d")
    if "counts" in g:
        assert np.array_equal(s0, g["counts"])
    if "mean" in g:
        assert_close_rel(s0, g["mean"], atol=1e-7, what="mean")
        assert_close_rel(s1, g["beta"], what="beta")
    elif "mean_sha256" in g:   # large-D fixture: exact vs the fp32-TSDF oracle
        assert np.array_equal(s0, os0) and np.array_equal(s1, os1)


def test_probe_and_background():
    g = load_golden("api_open_plane")
    m = mapper_for(g)
    replay_mapper(g, m)
    tsdf, sem = m.grids
    coords = g["coords"]
    rng = np.random.default_rng(0)
    q = np.concatenate([coords[::7], rng.integers(-500, 500, (300, 3)),
                        np.array([[10**6, -10**6, 5]])])
    (d, w), act = tsdf.probe_many(q)
    om = oracle_for(g)
    replay_oracle(g, om)
    od, ow, os0, os1, oact = om.probe(q)
    assert np.array_equal(act, oact)
    assert np.array_equal(d, od) and np.array_equal(w, ow)
    (mm, bb), act2 = sem.probe_many(q)
    assert np.array_equal(act2, oact)
    assert np.array_equal(mm.astype(np.float64), os0)
    assert np.array_equal(bb.astype(np.float64), os1)
    # backgrounds (grid.py:37-77): d = +trunc, w = 0, m = 0, beta = prior_beta
    inactive = ~act
    assert np.all(d[inactive] == 0.15) and np.all(w[inactive] == 0.0)
    assert np.all(bb[inactive] == np.float32(1e-3))


def test_stats_and_counts():
    g = load_golden("api_closed_plane")
    m = mapper_for(g)
    replay_mapper(g, m)
    st = m.stats()
    assert st["active_voxels"] == g["coords"].shape[0]
    assert st["semantic_active_voxels"] == g["coords"].shape[0]
    assert st["frames_integrated"] == g["n_frames"]
    leaves = np.unique(g["coords"] >> 3, axis=0).shape[0]
    assert st["leaf_count"] == leaves
    assert st["internal_count"] == np.unique(g["coords"] >> 7, axis=0).shape[0]


def _random_world_frames(seed, n, frames, h):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(frames):
        origin = rng.uniform(-1, 1, 3)
        pts = origin + rng.normal(size=(n, 3)) * rng.uniform(0.5, 6.0, (n, 1))
        out.append((pts.astype(np.float32), origin))
    return out


@pytest.mark.parametrize("carving", [False, True])
@pytest.mark.parametrize("wfn", ["constant_one", "linear_dropoff"])
def test_random_world_frames_vs_oracle(carving, wfn):
    from paper_2512_12945_b200 import Mapper
    from oracle.oracle import OracleMap

    kw = dict(voxel_size=0.07, truncation=0.21, space_carving=carving, weight_fn=wfn,
              num_classes=7, max_range=10.0)
    m = Mapper(**kw)
    om = OracleMap(**kw)
    rng = np.random.default_rng(1)
    for pts, origin in _random_world_frames(3 + carving, 3000, 3, 0.07):
        lab = rng.integers(0, 9, pts.shape[0]).astype(np.int32)
        r1 = m.integrate_world(pts, origin, labels=lab)
        r2 = om.integrate_world(pts, origin, labels=lab)
        assert np.array_equal(report_rows([r1]), report_rows([r2]))
    c, d, w, s0, _ = m._export()
    oc, od, ow, os0, _ = om.export()
    assert np.array_equal(c, oc) and np.array_equal(d, od) and np.array_equal(w, ow)
    assert np.array_equal(s0, os0)


# Frames per config: cfg3 frame 6 faces a wall at close range (about 200
# band voxels collecting ~10^4 rows each), which takes the open-set update's
# dimension-sliced giant-voxel kernels (k_huge_prep / k_huge_items, 16 slices
# of 32 dims at D = 512); the other frames take the per-voxel kernels.
WORKLOAD_FRAMES = {1: (0, 3), 2: (0, 3), 3: (0, 6), 4: (0, 3), 5: (0, 3)}


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_workload_frames_vs_oracle(cfg):
    """Full-resolution BASELINE frames at the BASELINE dims (C = 20/40,
    D = 512/768) through integrate_world, bit-exact vs the oracle; for the
    open-set configs also classify_means against the config's own queries
    (cfg3: k = 32 at D = 512; cfg5: k = 128 at D = 768): labels exact, best
    within 1e-12 relative (only the dot products' summation order differs)."""
    from paper_2512_12945_b200 import Mapper, scenes
    from oracle.oracle import OracleMap

    wl = scenes.workload(cfg, device="cuda")
    kw = dict(wl.mapper_kwargs)
    m = Mapper(**kw)
    om = OracleMap(**kw)
    for i in WORKLOAD_FRAMES[cfg]:
        f = wl.make_frame(i)
        pw = f.points_world
        r1 = m.integrate_world(pw, f.origin, labels=f.labels, features=f.features)
        r2 = om.integrate_world(pw.cpu().numpy(), f.origin,
                                labels=f.labels.cpu().numpy() if f.labels is not None else None,
                                features=f.features.cpu().numpy() if f.features is not None else None)
        assert np.array_equal(report_rows([r1]), report_rows([r2]))
    c, d, w, s0, s1 = m._export()
    oc, od, ow, os0, os1 = om.export()
    assert np.array_equal(c, oc)
    assert np.array_equal(d, od) and np.array_equal(w, ow)
    assert np.array_equal(s0, os0)
    if s1 is not None:
        assert np.array_equal(s1, os1)
    if wl.queries is not None:
        q = wl.queries.cpu().numpy()
        assert q.shape == ((32, 512) if cfg == 3 else (128, 768))
        olab, obest = om.classify(q)
        for path in ("dmma", "tcgen05"):   # FP64 DMMA and the int8 split GEMM on tcgen05
            m.set_score_path(path)
            lab, best = m.classify(q)
            assert lab.shape[0] == c.shape[0] > 100000
            assert np.array_equal(lab, olab), path
            np.testing.assert_allclose(best, obest, rtol=1e-12, atol=1e-300, err_msg=path)


@pytest.mark.parametrize("variant", ["bayes", "last_wins_dropoff", "geometry"])
@pytest.mark.parametrize("cfg", [1, 2, 4])
@pytest.mark.parametrize("mode", ["segments", "slots", "auto", "leaves"])
def test_update_modes_vs_oracle(mode, cfg, variant):
    """Every row-grouping strategy (svx_set_update_mode) on full BASELINE
    frames, bit-exact vs the oracle.  cfg1 (depth camera, ~17 rows per voxel)
    forced into slot mode overflows the 16 slots and must re-run the frame in
    segment mode without leaving a trace; forced into leaf mode it runs its
    leaves of up to 8192 rows through the CTA path."""
    from paper_2512_12945_b200 import Mapper, scenes
    from oracle.oracle import OracleMap

    wl = scenes.workload(cfg, device="cuda")
    kw = dict(wl.mapper_kwargs)
    if variant == "last_wins_dropoff":
        kw.update(fusion="last_wins", weight_fn="linear_dropoff")
    elif variant == "geometry":
        kw.pop("num_classes", None)
    m = Mapper(**kw)
    m.set_update_mode(mode)
    om = OracleMap(**kw)
    for i in range(3):
        f = wl.make_frame(i * 2)
        lab = f.labels if variant != "geometry" else None
        r1 = m.integrate_world(f.points_world, f.origin, labels=lab)
        r2 = om.integrate_world(f.points_world.cpu().numpy(), f.origin,
                                labels=lab.cpu().numpy() if lab is not None else None)
        assert np.array_equal(report_rows([r1]), report_rows([r2]))
    st = m.engine_stats()
    if mode == "segments":
        assert st["frames_slot_mode"] == 0 and st["frames_leaf_mode"] == 0
    elif mode == "slots" and cfg == 1:   # depth camera: slot mode overflows, re-run with segments
        assert st["frames_slot_mode"] == 0 and st["slot_overflow_reruns"] >= 1
    elif mode == "slots":                # LiDAR: every frame fits the slots
        assert st["frames_slot_mode"] == 3 and st["slot_overflow_reruns"] == 0
    elif mode == "leaves":
        assert st["frames_leaf_mode"] + st["slot_overflow_reruns"] == 3
    elif cfg != 1:                       # auto: LiDAR frames go to slot mode
        assert st["frames_slot_mode"] == 3
    c, d, w, s0, _ = m._export()
    oc, od, ow, os0, _ = om.export()
    assert np.array_equal(c, oc)
    assert np.array_equal(d, od) and np.array_equal(w, ow)
    if variant != "geometry":
        assert np.array_equal(s0, os0)
        assert np.array_equal(m.label_map()[1], om.label_map())


@pytest.mark.parametrize("mode", ["slots", "segments", "leaves"])
def test_pinned_host_inputs_match_device_inputs(mode):
    """Pinned host arrays are read in place by the walk in slot mode (no
    staging copy); the map must equal the one built from device tensors."""
    import torch

    from paper_2512_12945_b200 import Mapper, scenes

    wl = scenes.workload(2, device="cuda")
    a = Mapper(**wl.mapper_kwargs)
    b = Mapper(**wl.mapper_kwargs)
    a.set_update_mode(mode)
    b.set_update_mode(mode)
    for i in range(3):
        f = wl.make_frame(i)
        pts = torch.empty(f.points.shape, dtype=f.points.dtype, pin_memory=True)
        pts.copy_(f.points)
        lab = torch.empty(f.labels.shape, dtype=f.labels.dtype, pin_memory=True)
        lab.copy_(f.labels)
        ra = a.integrate(pts, f.pose, labels=lab)
        rb = b.integrate(f.points, f.pose, labels=f.labels)
        assert np.array_equal(report_rows([ra]), report_rows([rb]))
    assert a.grids[0].content_hash() == b.grids[0].content_hash()
    assert a.grids[1].content_hash() == b.grids[1].content_hash()


def test_cuda_fast_path_pose_fallbacks():
    """CUDA-tensor calls take the library-side pose check; poses outside its
    fast acceptance set (polar fix needed, non-finite, bad bottom row) must
    behave exactly like the general path."""
    import torch

    from paper_2512_12945_b200 import Mapper
    from paper_2512_12945_b200.errors import UserInputError

    rng = np.random.default_rng(5)
    pts = rng.normal(size=(4000, 3)).astype(np.float32) * 3.0
    lab = rng.integers(1, 5, 4000).astype(np.int32)
    tp, tl = torch.from_numpy(pts).cuda(), torch.from_numpy(lab).cuda()
    kw = dict(voxel_size=0.1, truncation=0.3, num_classes=4, max_range=20.0)
    pose = np.eye(4)
    pose[:3, :3] += 1.2e-4 * rng.normal(size=(3, 3))   # needs validate_rotation's polar fix
    pose[:3, 3] = [0.5, -0.2, 0.1]
    r = pose[:3, :3]
    assert 1e-4 < np.abs(r @ r.T - np.eye(3)).max() <= 1e-3
    a, b, c = Mapper(**kw), Mapper(**kw), Mapper(**kw)
    ra = a.integrate(tp, pose, labels=tl)            # CUDA fast path -> host fallback
    rb = b.integrate(pts, pose, labels=lab)          # numpy fast path -> host fallback
    rc = c.integrate(pts, pose, labels=lab.astype(np.int64))   # general path
    for r in (ra, rb):
        assert r.touched_voxels == rc.touched_voxels and r.band_hits == rc.band_hits
    assert a.grids[0].content_hash() == c.grids[0].content_hash()
    assert b.grids[0].content_hash() == c.grids[0].content_hash()
    # a pose inside the fast acceptance set: all three paths agree too
    good = np.eye(4)
    good[:3, 3] = [0.1, 0.2, -0.3]
    ra, rb, rc = (a.integrate(tp, good, labels=tl), b.integrate(pts, good, labels=lab),
                  c.integrate(pts.astype(np.float64).tolist(), good, labels=lab.tolist()))
    assert a.grids[0].content_hash() == c.grids[0].content_hash() == b.grids[0].content_hash()
    for bad in (np.full((4, 4), np.nan), np.diag([1.0, 1.0, 1.0, 2.0])):
        with pytest.raises(UserInputError):
            a.integrate(tp, bad, labels=tl)
        with pytest.raises(UserInputError):
            b.integrate(pts, bad, labels=lab)


@pytest.mark.parametrize("path", ["dmma", "tcgen05"])
@pytest.mark.parametrize("k", [5, 32, 100, 160])
def test_classify_fp64_tensor_core_vs_oracle(k, path):
    """classify_means on the FP64 tensor cores (DMMA, k <= 128; the CUDA-core
    kernel beyond) and on the tcgen05 int8 split GEMM (any k) against the
    oracle's sequential f64 scoring: labels exact, best and similarities
    within 1e-12 (only the rounding of the dot products differs)."""
    from paper_2512_12945_b200 import Mapper, scenes
    from oracle.oracle import OracleMap

    wl = scenes.workload(3, device="cuda")
    kw = dict(wl.mapper_kwargs)
    kw["feature_dim"] = 96                     # keeps the oracle fast; not a multiple of 16
    m = Mapper(**kw)
    m.set_score_path(path)
    om = OracleMap(**kw)
    for i in range(2):
        f = wl.make_frame(i * 5)
        feats = f.features[:, :96].contiguous()
        m.integrate_world(f.points_world, f.origin, features=feats)
        om.integrate_world(f.points_world.cpu().numpy(), f.origin, features=feats.cpu().numpy())
    rng = np.random.default_rng(k)
    emb = rng.normal(size=(k, 96))
    emb /= np.linalg.norm(emb, axis=1, keepdims=True)
    lab, best, sims = m.classify(emb, return_sims=True)
    olab, obest = om.classify(emb)
    assert lab.shape[0] > 1000
    assert np.array_equal(lab, olab)
    np.testing.assert_allclose(best, obest, rtol=1e-12, atol=1e-300)
    # similarities of the first query against the single-query cosine path
    _, s0 = m.query(emb[0])
    np.testing.assert_allclose(sims[:, 0], s0, rtol=1e-12, atol=1e-14, equal_nan=True)


@pytest.mark.parametrize("mode", ["slots", "segments", "leaves"])
def test_capacity_retries_vs_oracle(mode):
    """Tiny initial pools: frames run out of leaves and voxels mid-flight, are
    cleaned up, grown and re-run (recover_capacity / k_cleanup(_slots));
    the map must still equal the oracle's bit for bit."""
    from paper_2512_12945_b200 import Mapper, scenes
    from oracle.oracle import OracleMap

    wl = scenes.workload(2, device="cuda")
    m = Mapper(**wl.mapper_kwargs, reserve_voxels=64, reserve_blocks=4)
    m.set_update_mode(mode)
    om = OracleMap(**wl.mapper_kwargs)
    for i in range(3):
        f = wl.make_frame(i * 7)
        r1 = m.integrate(f.points, f.pose, labels=f.labels)
        r2 = om.integrate(f.points.cpu().numpy(), f.pose, labels=f.labels.cpu().numpy())
        assert np.array_equal(report_rows([r1]), report_rows([r2]))
    c, d, w, s0, _ = m._export()
    oc, od, ow, os0, _ = om.export()
    assert np.array_equal(c, oc)
    assert np.array_equal(d, od) and np.array_equal(w, ow)
    assert np.array_equal(s0, os0)
    # retries grow the pools to the frame's measured demand, not by repeated
    # doubling (a city frame once asked for 49 GB of slots this way)
    st = m.engine_stats()
    rows = 64 * 1024 * 24 + 4096
    assert st["block_capacity"] <= 8 * st["leaf_count"] + 65536
    assert st["voxel_capacity"] <= 4 * (st["active_voxels"] + rows) + 65536


def test_update_mode_argument():
    from paper_2512_12945_b200 import Mapper

    m = Mapper(voxel_size=0.1, truncation=0.3, num_classes=3)
    with pytest.raises(ValueError):
        m.set_update_mode("bogus")


def test_sensor_frame_identity_pose_lidar_full():
    """cfg2 (straight road, identity rotation) through Mapper.integrate: the
    reference's own API path, bit-exact vs the oracle."""
    from paper_2512_12945_b200 import Mapper, scenes
    from oracle.oracle import OracleMap

    wl = scenes.workload(2, device="cuda")
    m = Mapper(**wl.mapper_kwargs)
    om = OracleMap(**wl.mapper_kwargs)
    for i in range(3):
        f = wl.make_frame(i)
        r1 = m.integrate(f.points, f.pose, labels=f.labels)
        r2 = om.integrate(f.points.cpu().numpy(), f.pose, labels=f.labels.cpu().numpy())
        assert np.array_equal(report_rows([r1]), report_rows([r2]))
    c, d, w, s0, _ = m._export()
    oc, od, ow, os0, _ = om.export()
    assert np.array_equal(c, oc) and np.array_equal(d, od) and np.array_equal(w, ow)
    assert np.array_equal(s0, os0)
    _, lab = m.label_map()
    assert np.array_equal(lab, om.label_map())


class TestReferenceKnownAnswers:
    """Known-answer cases of the reference's own tests, re-expressed through
    the engine (test_raycast.py:26-69, test_tsdf.py:152-210)."""

    def band(self, origin, endpoint, h, trunc, carving=False):
        from paper_2512_12945_b200 import Mapper

        m = Mapper(voxel_size=h, truncation=trunc, space_carving=carving, max_range=50.0)
        m.integrate_world(np.array([endpoint], np.float64), origin)
        return sorted(map(tuple, m.grids[0].active_coords().tolist()))

    def test_axis_ray_half_open(self):
        assert self.band((0, 0, 0), (1.0, 0, 0), 0.25, 0.25) == [(3, 0, 0), (4, 0, 0)]

    def test_axis_ray_carving(self):
        assert self.band((0, 0, 0), (1.0, 0, 0), 0.25, 0.25, True) == [(i, 0, 0) for i in range(5)]

    def test_positive_overlap_included(self):
        assert self.band((0, 0, 0), (1.0, 0, 0), 0.25, 0.26) == [(i, 0, 0) for i in range(2, 6)]

    def test_negative_direction(self):
        assert self.band((0, 0, 0), (-1.0, 0, 0), 0.25, 0.25) == [(-5, 0, 0), (-4, 0, 0)]

    def test_corner_tie_lowest_axis_first(self):
        got = self.band((0.05, 0.05, 0.05), (0.25, 0.25, 0.05), 0.1, 0.2, True)
        assert got == sorted([(0, 0, 0), (1, 0, 0), (1, 1, 0), (2, 1, 0), (2, 2, 0), (3, 2, 0),
                              (3, 3, 0)])

    def test_same_frame_twice_doubles_weight(self):
        from paper_2512_12945_b200 import Mapper

        rng = np.random.default_rng(11)
        pts = rng.uniform(0.4, 1.3, (40, 3))
        once = Mapper(voxel_size=0.05, truncation=0.15)
        twice = Mapper(voxel_size=0.05, truncation=0.15)
        once.integrate(pts, np.eye(4))
        twice.integrate(pts, np.eye(4))
        twice.integrate(pts, np.eye(4))
        c1, (d1, w1) = once.grids[0].active_values()
        c2, (d2, w2) = twice.grids[0].active_values()
        assert np.array_equal(c1, c2)
        assert np.array_equal(w2, 2.0 * w1)
        assert np.array_equal(d1, d2)


class TestErrors:
    def test_step_budget(self):
        from paper_2512_12945_b200 import Mapper, SemvoxError

        m = Mapper(voxel_size=1e-5, truncation=3e-5, space_carving=True, max_range=50.0)
        with pytest.raises(SemvoxError, match="step budget"):
            m.integrate_world(np.array([[12.0, 0.0, 0.0]]), (0.0, 0.0, 0.0))
        assert m.active_count() == 0

    def test_frame_extent(self):
        from paper_2512_12945_b200 import Mapper, SemvoxError

        m = Mapper(voxel_size=1e-6, truncation=3e-6, max_range=50.0)
        pts = np.array([[3.0, 0.0, 0.0], [-3.0, 0.0, 0.0]])
        with pytest.raises(SemvoxError, match="2\\^21"):
            m.integrate_world(pts, (0.0, 0.0, 0.0))

    def test_out_of_range(self):
        from paper_2512_12945_b200 import Mapper, OutOfRangeError

        m = Mapper(voxel_size=1.0, truncation=3.0, max_range=50.0)
        o = np.array([2.0**30 + 5, 0.0, 0.0])
        with pytest.raises(OutOfRangeError):
            m.integrate_world(o[None, :] + [[2.0, 0.0, 0.0]], o)

    def test_payload_errors(self):
        from paper_2512_12945_b200 import Mapper, PayloadMismatchError

        m = Mapper(voxel_size=0.05, num_classes=3)
        with pytest.raises(PayloadMismatchError, match="labels"):
            m.integrate(np.zeros((2, 3)), np.eye(4))
        m2 = Mapper(voxel_size=0.05, feature_dim=4)
        with pytest.raises(PayloadMismatchError, match="feature dim"):
            m2.integrate(np.ones((2, 3)), np.eye(4), features=np.zeros((2, 5)))

    def test_empty_frame(self):
        from paper_2512_12945_b200 import Mapper

        m = Mapper(voxel_size=0.05)
        r = m.integrate(np.zeros((0, 3)), np.eye(4))
        assert r.points_in == 0 and r.touched_voxels == 0
        assert m.stats()["leaf_count"] == 0


@pytest.mark.parametrize("feat_dtype", ["float32", "float64"])
@pytest.mark.parametrize("D", [40, 96, 512, 768])
def test_open_huge_voxels_vs_oracle(D, feat_dtype):
    """Open-set voxels with thousands of rows (every ray of a frame crosses
    the same few band voxels, like a depth camera facing a close wall): the
    dimension-sliced huge-voxel kernels (k_huge_prep / k_huge_items) against
    the oracle's sequential point-ordered sums, bit for bit; D not a
    multiple of the 32-dimension slice, the BASELINE D = 512 / 768 (16 / 24
    slices), f32 and f64 features."""
    from oracle.oracle import OracleMap
    from paper_2512_12945_b200 import Mapper

    rng = np.random.default_rng(D)
    kw = dict(voxel_size=0.05, truncation=0.15, feature_dim=D, max_range=5.0)
    m, om = Mapper(**kw), OracleMap(**kw)
    for f, n in enumerate((6000, 8000, 10000, 30000)):
        pts = np.column_stack([1.0 + rng.normal(0.0, 0.003, n), rng.uniform(-0.03, 0.03, n),
                               rng.uniform(-0.03, 0.03, n)])
        origin = np.array([0.01 * f, 0.005 * f, -0.004 * f])
        feats = rng.normal(size=(n, D)).astype(feat_dtype)
        r1 = m.integrate_world(pts + origin, origin, features=feats)
        r2 = om.integrate_world(pts + origin, origin, features=feats)
        assert r1.touched_voxels == r2.touched_voxels and r1.band_hits == r2.band_hits
        if n == 30000:   # this frame alone gives some voxels > 8192 rows (giant path)
            one = OracleMap(voxel_size=0.05, truncation=0.15, max_range=5.0)
            one.integrate_world(pts + origin, origin)
            assert one.export()[2].max() > 8192
    assert m.engine_stats()["active_voxels"] < 200    # few voxels, thousands of rows each
    c1, d1, w1, m1, b1 = m._export()
    c2, d2, w2, m2, b2 = om.export()
    assert np.array_equal(c1, c2)
    assert np.array_equal(d1, d2) and np.array_equal(w1, w2)
    assert np.array_equal(m1, m2) and np.array_equal(b1, b2)


@pytest.mark.parametrize("D", [4, 6, 512])
def test_nonfinite_features_vs_oracle(D):
    """Open-set frames whose feature rows carry NaN / inf at scattered rows
    and positions (first and last element, several per warp, a ragged tail of
    points): the walk's feature scan must mask exactly the rows the reference
    masks (fusion.py:246-256).  D = 4 and 512 take the contiguous block scan,
    D = 6 the row-by-row loop."""
    from paper_2512_12945_b200 import Mapper
    from oracle.oracle import OracleMap

    kw = dict(voxel_size=0.1, truncation=0.3, feature_dim=D, max_range=12.0)
    m = Mapper(**kw)
    om = OracleMap(**kw)
    rng = np.random.default_rng(7)
    for pts, origin in _random_world_frames(3, 1000 + 37, 3, 0.1):
        n = pts.shape[0]
        feat = rng.normal(size=(n, D)).astype(np.float32)
        bad = rng.choice(n, size=n // 20, replace=False)
        pos = rng.integers(0, D, bad.size)
        pos[: bad.size // 3] = D - 1
        pos[bad.size // 3: 2 * bad.size // 3] = 0
        vals = np.array([np.nan, np.inf, -np.inf], np.float32)[rng.integers(0, 3, bad.size)]
        feat[bad, pos] = vals
        feat[n - 1, D - 1] = np.nan                   # last element of the array
        feat[32:40, D // 2] = np.inf                   # a run inside one warp
        r1 = m.integrate_world(pts, origin, features=feat)
        r2 = om.integrate_world(pts, origin, features=feat)
        assert np.array_equal(report_rows([r1]), report_rows([r2]))
        assert r1.skipped_bad_label > 0   # the reference counts bad feature rows as bad payload
    c, d, w, s0, s1 = m._export()
    oc, od, ow, os0, os1 = om.export()
    assert np.array_equal(c, oc) and np.array_equal(d, od) and np.array_equal(w, ow)
    assert np.array_equal(s0, os0) and np.array_equal(s1, os1)

"""``.slvg`` snapshots: the reference's grid-block file
format (grid.py:298-426), Mapper.save (bindings/__init__.py:183-187) and
load_grid (:189-201), mirroring the reference's TestGridSnapshots
(pkg/tests/test_io.py:425-484).

Fixtures: tests/golden/snap_*.slvg.gz are files the reference's own
Mapper.save wrote for the api_* fixtures' inputs (make_golden.py snapshot).
CPU tests pin the format code against them (decode = the fixture's active
values, encode = the same bytes, also from the oracle's map); GPU tests check
the engine's Mapper.save bytes, the device import and resuming a map.
"""

import gzip
import io
import os
import struct

import numpy as np
import pytest

from helpers import GOLDEN, load_golden, oracle_for, replay_mapper, replay_oracle

SNAPS = ["closed_plane", "open_plane", "geometry_carving_dropoff", "closed_lastwins_dropoff"]


def snap_bytes(stem):
    with gzip.open(os.path.join(GOLDEN, f"snap_{stem}.slvg.gz"), "rb") as fh:
        return fh.read()


def views_of(mkw):
    """(kind, params bytes, field selector) per block, as Mapper.save writes them."""
    from paper_2512_12945_b200.config import ClosedSetConfig, OpenSetConfig
    from paper_2512_12945_b200.mapper import (ClosedPayload, OpenPayload, TsdfPayload,
                                              _params_block)

    out = [(0, _params_block(TsdfPayload(mkw.get("truncation"))), lambda d, w, s0, s1: [d, w])]
    if mkw.get("num_classes"):
        keys = {k: v for k, v in mkw.items() if k in ("num_classes", "prior_alpha", "fusion",
                                                      "count_dtype")}
        out.append((1, _params_block(ClosedPayload(ClosedSetConfig(**keys))),
                    lambda d, w, s0, s1: [s0]))
    if mkw.get("feature_dim"):
        keys = {k: v for k, v in mkw.items() if k in ("feature_dim", "prior_beta", "lambda_floor",
                                                      "confidence_threshold", "temperature",
                                                      "state_dtype")}
        out.append((2, _params_block(OpenPayload(OpenSetConfig(**keys))),
                    lambda d, w, s0, s1: [s0, s1]))
    return out


@pytest.mark.parametrize("stem", SNAPS)
def test_decode_reference_snapshot(stem):
    from paper_2512_12945_b200 import snapshot
    from paper_2512_12945_b200.mapper import _split_blocks

    g = load_golden("api_" + stem)
    blocks = snapshot.parse(snap_bytes(stem))
    tsdf, sem = _split_blocks(blocks)
    assert len(blocks) == (2 if sem is not None else 1)
    assert np.array_equal(tsdf.coords(), g["coords"])      # active order = file order
    assert np.array_equal(tsdf.fields[0], g["d"]) and np.array_equal(tsdf.fields[1], g["w"])
    assert tsdf.voxel_size == g["mapper_kw"]["voxel_size"]
    if "counts" in g:
        assert sem.kind == 1 and np.array_equal(sem.fields[0], g["counts"])
    elif "mean" in g:
        assert sem.kind == 2
        assert np.array_equal(sem.fields[0], g["mean"]) and np.array_equal(sem.fields[1], g["beta"])
    else:
        assert sem is None


@pytest.mark.parametrize("stem", SNAPS)
def test_encode_matches_reference_bytes(stem):
    """Writing the decoded blocks back gives the reference's bytes."""
    from paper_2512_12945_b200 import snapshot

    raw = snap_bytes(stem)
    blocks = snapshot.parse(raw)
    fh = io.BytesIO()
    for b in blocks:
        snapshot.write_block(fh, b.kind, b.voxel_size, snapshot.pack_params(b.kind, b.params),
                             b.coords(), b.fields)
    assert fh.getvalue() == raw


@pytest.mark.parametrize("stem", SNAPS)
def test_oracle_map_encodes_to_reference_bytes(stem):
    """The oracle's map of the fixture's frames, written by the engine's
    writer, is the reference's snapshot byte for byte (pins the writer on a
    map state that did not come from the file)."""
    from paper_2512_12945_b200 import snapshot

    g = load_golden("api_" + stem)
    om = oracle_for(g)
    replay_oracle(g, om)
    coords, d, w, s0, s1 = om.export()
    fh = io.BytesIO()
    for kind, params, sel in views_of(g["mapper_kw"]):
        snapshot.write_block(fh, kind, g["mapper_kw"]["voxel_size"], params, coords,
                             sel(d, w, s0, s1))
    assert fh.getvalue() == snap_bytes(stem)


def test_empty_snapshot():
    from paper_2512_12945_b200 import snapshot

    raw = snap_bytes("empty")
    (b,) = snapshot.parse(raw)
    assert b.kind == 0 and b.active_count == 0 and b.leaf_coords.shape == (0, 3)
    fh = io.BytesIO()
    snapshot.write_block(fh, 0, b.voxel_size, snapshot.pack_params(0, b.params),
                         np.zeros((0, 3), np.int64), [np.zeros(0), np.zeros(0)])
    assert fh.getvalue() == raw


def test_format_errors():
    from paper_2512_12945_b200 import FormatError, snapshot

    with pytest.raises(FormatError, match="no grid blocks"):
        snapshot.parse(b"")
    with pytest.raises(FormatError, match="magic"):
        snapshot.parse(b"WHAT" + b"\0" * 40)
    raw = snap_bytes("closed_plane")
    with pytest.raises(FormatError, match="truncated"):
        snapshot.parse(raw[:-5])
    with pytest.raises(FormatError, match="version"):
        snapshot.parse(raw[:4] + struct.pack("<I", 2) + raw[8:])
    bad = bytearray(raw)
    bad[4 + 4 + 8 + 2] = 7                                  # kind byte
    with pytest.raises(FormatError, match="kind"):
        snapshot.parse(bytes(bad))
    # header active count disagreeing with the masks
    n = struct.unpack_from("<Q", raw, 4 + 4 + 8 + 3)[0]
    bad = raw[:4 + 4 + 8 + 3] + struct.pack("<Q", n + 1) + raw[4 + 4 + 8 + 3 + 8:]
    with pytest.raises(FormatError, match="active count"):
        snapshot.parse(bad)


def test_split_leaves_groups_by_leaf():
    from paper_2512_12945_b200 import snapshot

    coords = np.array([[0, 0, 1], [0, 0, 7], [8, 0, 0], [-1, -1, -1], [-8, -8, -8]], np.int64)
    lc, vl, sl = snapshot.split_leaves(coords)
    assert lc.tolist() == [[0, 0, 0], [1, 0, 0], [-1, -1, -1]]
    assert vl.tolist() == [0, 0, 1, 2, 2]
    assert sl.tolist() == [1, 7, 0, 511, 0]


# ---- GPU: the engine's Mapper.save / load_grid / from_snapshot ---------------------------


def mapper_for(g, **extra):
    from paper_2512_12945_b200 import Mapper

    kw = dict(g["mapper_kw"])
    kw.update(extra)
    return Mapper(**kw)


@pytest.mark.gpu
@pytest.mark.parametrize("stem", SNAPS)
def test_engine_save_is_reference_bytes(stem, tmp_path):
    g = load_golden("api_" + stem)
    m = mapper_for(g)
    replay_mapper(g, m)
    p = tmp_path / "map.slvg"
    m.save(str(p))
    assert p.read_bytes() == snap_bytes(stem)


@pytest.mark.gpu
@pytest.mark.parametrize("stem", SNAPS + ["empty"])
def test_load_grid_round_trip(stem, tmp_path):
    """load_grid of the reference's file: same active values, same content
    hashes, and saving it again gives the same bytes."""
    from paper_2512_12945_b200 import load_grid

    p = tmp_path / "ref.slvg"
    p.write_bytes(snap_bytes(stem))
    tsdf, sem = load_grid(str(p))
    if stem == "empty":
        assert sem is None and tsdf.active_values()[0].shape == (0, 3)
        assert tsdf.memory_stats().leaf_count == 0
    else:
        g = load_golden("api_" + stem)
        coords, (d, w) = tsdf.active_values()
        assert np.array_equal(coords, g["coords"])
        assert np.array_equal(d, g["d"]) and np.array_equal(w, g["w"])
        assert tsdf.content_hash() == str(g["tsdf_hash"])
        if sem is not None:
            assert sem.content_hash() == str(g["sem_hash"])
        # probe through the device hash of the imported leaves
        vals, active = tsdf.probe_many(g["coords"][::7])
        assert active.all() and np.array_equal(vals[0], g["d"][::7])
    q = tmp_path / "again.slvg"
    tsdf._m.save(str(q))
    assert q.read_bytes() == snap_bytes(stem)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["auto", "segments"])
@pytest.mark.parametrize("stem", SNAPS)
def test_resume_from_snapshot(stem, mode, tmp_path):
    """save after k frames -> from_snapshot -> remaining frames == the map of
    all frames in one run (and the reference's: its snapshot bytes)."""
    from paper_2512_12945_b200 import Mapper

    g = load_golden("api_" + stem)
    n = g["n_frames"]
    k = max(1, n // 2)
    first = dict(g, n_frames=k)
    m = mapper_for(g)
    replay_mapper(first, m)
    p = tmp_path / "part.slvg"
    m.save(str(p))
    kw = {k2: v for k2, v in g["mapper_kw"].items()
          if k2 in ("max_range", "weight_fn", "space_carving")}
    m2 = Mapper.from_snapshot(str(p), **kw)
    m2.set_update_mode(mode)
    rest = {f"{key}_{i - k}": g[f"{key}_{i}"] for i in range(k, n)
            for key in ("points", "pose", "labels", "features") if f"{key}_{i}" in g}
    replay_mapper(dict(rest, mode=g["mode"], n_frames=n - k), m2)
    q = tmp_path / "full.slvg"
    m2.save(str(q))
    assert q.read_bytes() == snap_bytes(stem)


@pytest.mark.gpu
def test_from_snapshot_config_checks(tmp_path):
    from paper_2512_12945_b200 import ConfigError, Mapper

    p = tmp_path / "ref.slvg"
    p.write_bytes(snap_bytes("closed_plane"))
    with pytest.raises(ConfigError, match="contradicts"):
        Mapper.from_snapshot(str(p), voxel_size=0.2)
    with pytest.raises(ConfigError, match="contradicts"):
        Mapper.from_snapshot(str(p), num_classes=9)
    m = Mapper.from_snapshot(str(p), tsdf_dtype="float32")     # compact layout loads too
    g = load_golden("api_closed_plane")
    coords, (d, w) = m.grids[0].active_values()
    assert np.array_equal(coords, g["coords"])
    assert np.array_equal(d, g["d"].astype(np.float32).astype(np.float64))
    g2 = tmp_path / "geom.slvg"
    g2.write_bytes(snap_bytes("geometry_carving_dropoff"))
    with pytest.raises(ConfigError, match="geometry only"):
        Mapper.from_snapshot(str(g2), num_classes=4)
    # a map that already holds frames does not take a snapshot
    m3 = Mapper(voxel_size=0.05, truncation=0.15, num_classes=4)
    replay_mapper(dict(g, n_frames=1), m3)
    from paper_2512_12945_b200.mapper import _split_blocks
    from paper_2512_12945_b200 import UserInputError, snapshot

    t, s = _split_blocks(snapshot.read_blocks(str(p)))
    with pytest.raises(UserInputError, match="empty map"):
        m3._import_blocks(t, s)


@pytest.mark.gpu
@pytest.mark.parametrize("config", [2, 3])
def test_resume_full_size(config, tmp_path):
    """BASELINE-size frames (cfg2 LiDAR closed-set, cfg3 depth camera
    open-set): a map resumed from its snapshot integrates the next frames to
    the same bytes as the map that never left the GPU."""
    from paper_2512_12945_b200 import Mapper, scenes

    wl = scenes.workload(config, device="cuda")
    kw = dict(wl.mapper_kwargs)
    m = Mapper(**kw)

    def feed(mapper, i):
        f = wl.make_frame(i)
        if f.features is not None:
            mapper.integrate_world(f.points_world, f.origin, features=f.features)
        else:
            mapper.integrate(f.points, f.pose, labels=f.labels)

    for i in range(2):
        feed(m, i)
    p = tmp_path / "a.slvg"
    m.save(str(p))
    m2 = Mapper.from_snapshot(str(p), **{k: v for k, v in kw.items()
                                         if k in ("max_range", "weight_fn", "space_carving")})
    assert m2.grids[0].content_hash() == m.grids[0].content_hash()
    for i in range(2, 4):
        feed(m, i)
        feed(m2, i)
    qa, qb = tmp_path / "b.slvg", tmp_path / "c.slvg"
    m.save(str(qa))
    m2.save(str(qb))
    assert qa.read_bytes() == qb.read_bytes()


def test_missing_and_empty_files(tmp_path):
    """test_bindings.py TestSnapshots: empty file -> FormatError, missing -> OSError
    (both raised before any device work)."""
    from paper_2512_12945_b200 import FormatError, load_grid

    bad = tmp_path / "empty.slvg"
    bad.write_bytes(b"")
    with pytest.raises(FormatError):
        load_grid(bad)
    with pytest.raises(OSError):
        load_grid(tmp_path / "nope.slvg")


@pytest.mark.gpu
def test_grids_equal_and_path_objects(tmp_path):
    from paper_2512_12945_b200 import grids_equal, load_grid

    g = load_golden("api_closed_plane")
    m = mapper_for(g)
    replay_mapper(g, m)
    snap = tmp_path / "run.slvg"
    m.save(snap)                                  # pathlib paths, like the reference
    tsdf, sem = load_grid(snap)
    assert grids_equal(tsdf, m.grids[0]) and grids_equal(sem, m.grids[1])
    assert not grids_equal(tsdf, sem)
    m2 = mapper_for(g)
    replay_mapper(dict(g, n_frames=1), m2)
    assert not grids_equal(tsdf, m2.grids[0])


def test_parser_rejects_corruption_cleanly():
    """Truncations and byte flips of a reference snapshot either parse or
    raise FormatError -- never another exception (the parser validates every
    length and count before using it)."""
    from paper_2512_12945_b200 import FormatError, snapshot

    raw = snap_bytes("closed_plane")
    rng = np.random.default_rng(11)
    cuts = sorted(set(rng.integers(0, len(raw), 60).tolist()) | {1, 3, 4, 8, 20, 40})
    for cut in cuts:
        try:
            snapshot.parse(raw[:cut])
        except FormatError:
            pass
    for _ in range(150):
        b = bytearray(raw)
        for pos in rng.integers(0, 200, 3):      # header, parameters, first leaves
            b[pos] = int(rng.integers(0, 256))
        try:
            snapshot.parse(bytes(b))
        except FormatError:
            pass


@pytest.mark.gpu
def test_device_import_rejects_bad_arrays():
    """svx_import validates what it is given (C-ABI callers need not come
    through the parser): a repeated slot, a leaf index out of range or a
    repeated leaf fails with FormatError and leaves the map empty and usable."""
    from types import SimpleNamespace

    from paper_2512_12945_b200 import FormatError, Mapper

    g = load_golden("api_closed_plane")

    def block(lc, vl, vs):
        n = len(vs)
        return SimpleNamespace(leaf_coords=np.array(lc, np.int32).reshape(-1, 3),
                               voxel_leaf=np.array(vl, np.int32), voxel_slot=np.array(vs, np.int32),
                               active_count=n, fields=[np.zeros(n), np.ones(n)])

    bad = [block([[0, 0, 0]], [0, 0], [5, 5]),                   # repeated slot
           block([[0, 0, 0]], [0, 1], [5, 6]),                   # leaf index out of range
           block([[0, 0, 0], [0, 0, 0]], [0, 1], [5, 6]),        # repeated leaf
           block([[1 << 28, 0, 0]], [0], [5])]                   # beyond +/-2^30 voxels
    for b in bad:
        m = Mapper(**{k: v for k, v in g["mapper_kw"].items() if k != "num_classes"})
        with pytest.raises(FormatError):
            m._import_blocks(b, None)
        assert m.active_count() == 0
        replay_mapper(dict(g, labels_0=None, labels_1=None, labels_2=None, labels_3=None), m)
        ref = Mapper(**{k: v for k, v in g["mapper_kw"].items() if k != "num_classes"})
        replay_mapper(dict(g, labels_0=None, labels_1=None, labels_2=None, labels_3=None), ref)
        assert m.grids[0].content_hash() == ref.grids[0].content_hash()

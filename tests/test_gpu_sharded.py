"""Sharded integration on one GPU.

G in-process shards are driven by ``integrate_loopback``: the per-rank march /
plan / pack / apply phases and the exchange buffers of the multi-process NCCL
driver, with the all-reduce and all-to-all done in-process (one GPU cannot
host ranks whose kernels wait on each other).  Bar: the union of the shards,
merged by leaf stamps, equals the single-GPU map bit for bit -- active set,
global active order, TSDF, weights, semantic state, content hashes and the
frame reports -- and the oracle where it is run directly.
"""

import numpy as np
import pytest

from helpers import report_rows

pytestmark = pytest.mark.gpu

CASES = {
    "closed": dict(voxel_size=0.07, truncation=0.21, num_classes=7, max_range=10.0),
    "last_wins": dict(voxel_size=0.07, truncation=0.21, num_classes=5, fusion="last_wins",
                      max_range=10.0),
    "carving_dropoff": dict(voxel_size=0.07, truncation=0.21, space_carving=True,
                            weight_fn="linear_dropoff", max_range=10.0),
    "open": dict(voxel_size=0.07, truncation=0.21, feature_dim=16, max_range=10.0),
}


def _shards(G, **kw):
    from paper_2512_12945_b200.sharded import ShardedMapper

    return [ShardedMapper(rank=r, world=G, **kw) for r in range(G)]


def _merged(shards):
    from paper_2512_12945_b200.sharded import merge_by_stamps

    return merge_by_stamps([s.local_export() for s in shards])


def _frames(seed, n, count):
    rng = np.random.default_rng(seed)
    for _ in range(count):
        origin = rng.uniform(-1, 1, 3)
        pts = origin + rng.normal(size=(n, 3)) * rng.uniform(0.5, 6.0, (n, 1))
        yield pts.astype(np.float32), origin


def _payload(kw, rng, n):
    lab = feat = None
    if "num_classes" in kw:
        lab = rng.integers(0, kw["num_classes"] + 2, n).astype(np.int32)
    if "feature_dim" in kw:
        feat = rng.normal(size=(n, kw["feature_dim"])).astype(np.float32)
    return lab, feat


def _assert_union_equals(single, shards):
    from paper_2512_12945_b200.sharded import merged_content_hash

    ref = single._export()
    got = _merged(shards)
    for a, b in zip(ref, got):
        assert (a is None) == (b is None)
        if a is not None:
            assert a.dtype == b.dtype and np.array_equal(a, b)
    for k, view in enumerate(shards[0].grids):
        if view is not None:
            assert merged_content_hash(got, view) == single.grids[k].content_hash()


def _assert_owned(shards):
    from paper_2512_12945_b200.sharded import leaf_owner

    G = len(shards)
    for s in shards:
        coords = s._export()[0]
        leaves = np.unique(coords >> 3, axis=0)
        assert all(leaf_owner(*b, G) == s.rank for b in leaves)


@pytest.mark.parametrize("G", [1, 2, 3, 4])
@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("plan", [False, True], ids=["host_plan", "device_plan"])
def test_loopback_shards_equal_single_gpu(case, G, plan):
    from paper_2512_12945_b200 import Mapper
    from paper_2512_12945_b200.sharded import integrate_loopback

    kw = CASES[case]
    single = Mapper(**kw)
    shards = _shards(G, **kw)
    rng = np.random.default_rng(7)
    for pts, origin in _frames(11, 2500, 3):
        lab, feat = _payload(kw, rng, pts.shape[0])
        r1 = single.integrate_world(pts, origin, labels=lab, features=feat)
        r2 = integrate_loopback(shards, pts, origin=origin, labels=lab, features=feat, device_plan=plan)
        assert np.array_equal(report_rows([r1]), report_rows([r2]))
        assert (r1.new_blocks, r1.new_voxels) == (r2.new_blocks, r2.new_voxels)
    _assert_union_equals(single, shards)
    _assert_owned(shards)
    assert sum(s.active_count() for s in shards) == single.active_count()


@pytest.mark.parametrize("plan", [False, True], ids=["host_plan", "device_plan"])
def test_loopback_workload_vs_oracle(plan):
    """Full cfg2 LiDAR frames (65,536 points, sensor pose) on 4 shards,
    bit-exact against the oracle."""
    from oracle.oracle import OracleMap
    from paper_2512_12945_b200 import scenes
    from paper_2512_12945_b200.sharded import integrate_loopback

    wl = scenes.workload(2, device="cuda")
    kw = dict(wl.mapper_kwargs)
    shards = _shards(4, **kw)
    om = OracleMap(**kw)
    for i in range(2):
        f = wl.make_frame(i * 3)
        r1 = integrate_loopback(shards, f.points_world, origin=f.origin, labels=f.labels, device_plan=plan)
        r2 = om.integrate_world(f.points_world.cpu().numpy(), f.origin,
                                labels=f.labels.cpu().numpy())
        assert np.array_equal(report_rows([r1]), report_rows([r2]))
    got = _merged(shards)
    ref = om.export()
    for a, b in zip(ref, got):
        if a is not None:
            assert np.array_equal(a, b)
    _assert_owned(shards)


@pytest.mark.parametrize("plan", [False, True], ids=["host_plan", "device_plan"])
def test_loopback_sensor_pose_and_device_inputs(plan):
    """Mapper.integrate semantics (sensor points + pose) with CUDA inputs."""
    import torch

    from paper_2512_12945_b200 import Mapper
    from paper_2512_12945_b200.sharded import integrate_loopback

    kw = dict(voxel_size=0.05, truncation=0.15, num_classes=4, max_range=8.0)
    single = Mapper(**kw)
    shards = _shards(3, **kw)
    rng = np.random.default_rng(3)
    for k in range(3):
        pose = np.eye(4)
        pose[:3, 3] = [0.3 * k, -0.2 * k, 0.1]
        pts = torch.as_tensor(rng.normal(size=(4000, 3)) * 2.0, dtype=torch.float32).cuda()
        lab = torch.as_tensor(rng.integers(1, 5, 4000), dtype=torch.int32).cuda()
        r1 = single.integrate(pts, pose, labels=lab)
        r2 = integrate_loopback(shards, pts, pose=pose, labels=lab, device_plan=plan)
        assert np.array_equal(report_rows([r1]), report_rows([r2]))
    _assert_union_equals(single, shards)


@pytest.mark.parametrize("plan", [False, True], ids=["host_plan", "device_plan"])
def test_global_queries_merge_in_active_order(plan):
    from paper_2512_12945_b200 import Mapper
    from paper_2512_12945_b200.sharded import integrate_loopback, merge_by_stamps

    kw = CASES["open"]
    single = Mapper(**kw)
    shards = _shards(3, **kw)
    rng = np.random.default_rng(5)
    for pts, origin in _frames(2, 2000, 2):
        _, feat = _payload(kw, rng, pts.shape[0])
        single.integrate_world(pts, origin, features=feat)
        integrate_loopback(shards, pts, origin=origin, features=feat, device_plan=plan)
    q = rng.normal(size=kw["feature_dim"])
    c1, s1 = single.query(q)
    c2, s2 = merge_by_stamps([s.local_query(q) for s in shards])
    assert np.array_equal(c1, c2)
    assert np.array_equal(np.isnan(s1), np.isnan(s2))
    assert np.array_equal(s1[~np.isnan(s1)], s2[~np.isnan(s2)])

    kwc = CASES["closed"]
    single = Mapper(**kwc)
    shards = _shards(2, **kwc)
    for pts, origin in _frames(4, 2000, 2):
        lab, _ = _payload(kwc, rng, pts.shape[0])
        single.integrate_world(pts, origin, labels=lab)
        integrate_loopback(shards, pts, origin=origin, labels=lab, device_plan=plan)
    for zero in (False, True):
        c1, l1 = single.label_map(zero)
        c2, l2 = merge_by_stamps([s.local_label_map(zero) for s in shards])
        assert np.array_equal(c1, c2) and np.array_equal(l1, l2)


def test_device_plan_one_sync_and_capacity_redo():
    """The device plan takes one host synchronisation per frame; sections
    over their capacity abort the frame on every shard before any change and
    it is redone with the capacity the device reported."""
    from paper_2512_12945_b200 import Mapper
    from paper_2512_12945_b200.sharded import integrate_loopback

    kw = CASES["closed"]
    single = Mapper(**kw)
    shards = _shards(3, **kw)
    rng = np.random.default_rng(5)
    for i, (pts, origin) in enumerate(_frames(13, 3000, 4)):
        lab, _ = _payload(kw, rng, pts.shape[0])
        if i == 2:
            for s in shards:
                s._cap = 1024   # far below one section
        r1 = single.integrate_world(pts, origin, labels=lab)
        r2 = integrate_loopback(shards, pts, origin=origin, labels=lab, device_plan=True)
        assert np.array_equal(report_rows([r1]), report_rows([r2]))
        assert shards[0].host_syncs == (2 if i == 2 else 1)
        if i == 2:
            assert shards[0]._cap > 1024
    _assert_union_equals(single, shards)
    assert all(s.stats()["frames_integrated"] == 4 for s in shards)


@pytest.mark.parametrize("plan", [False, True], ids=["host_plan", "device_plan"])
def test_key_window_rebase_is_global(plan):
    """Rows beyond the default packed-key window (2^20 voxels from the
    sensor) make every rank re-march with the frame's minimum as key base."""
    from oracle.oracle import OracleMap
    from paper_2512_12945_b200 import Mapper
    from paper_2512_12945_b200.sharded import integrate_loopback

    kw = dict(voxel_size=1e-3, truncation=3e-3, max_range=2000.0, num_classes=3)
    single = Mapper(**kw)
    shards = _shards(2, **kw)
    om = OracleMap(**kw)
    pts = np.array([[0.5, 0.0, 0.0], [0.6, 0.1, 0.0], [1100.0, 0.2, 0.0], [1100.4, 0.1, 0.3]])
    lab = np.array([1, 2, 3, 1], np.int32)
    r1 = single.integrate_world(pts, (0.0, 0.0, 0.0), labels=lab)
    r2 = integrate_loopback(shards, pts, origin=(0.0, 0.0, 0.0), labels=lab, device_plan=plan)
    r3 = om.integrate_world(pts, (0.0, 0.0, 0.0), labels=lab)
    assert np.array_equal(report_rows([r1]), report_rows([r2]))
    assert np.array_equal(report_rows([r2]), report_rows([r3]))
    _assert_union_equals(single, shards)


@pytest.mark.parametrize("plan", [False, True], ids=["host_plan", "device_plan"])
def test_frame_errors_fail_on_every_shard_before_mutation(plan):
    from paper_2512_12945_b200 import SemvoxError
    from paper_2512_12945_b200.sharded import integrate_loopback

    # each slice alone fits the 2^21 extent; the frame does not
    shards = _shards(2, voxel_size=1e-6, truncation=3e-6, max_range=50.0)
    pts = np.array([[3.0, 0.0, 0.0], [-3.0, 0.0, 0.0]])
    with pytest.raises(SemvoxError, match="2\\^21"):
        integrate_loopback(shards, pts, origin=(0.0, 0.0, 0.0), device_plan=plan)
    assert all(s.active_count() == 0 for s in shards)
    shards = _shards(3, voxel_size=1e-5, truncation=3e-5, space_carving=True, max_range=50.0)
    with pytest.raises(SemvoxError, match="step budget"):
        integrate_loopback(shards, np.array([[12.0, 0.0, 0.0]] * 3), origin=(0.0, 0.0, 0.0), device_plan=plan)
    assert all(s.active_count() == 0 for s in shards)
    # the shards stay usable after a rejected frame
    r = integrate_loopback(shards, np.array([[0.001, 0.0, 0.0]]), origin=(0.0, 0.0, 0.0), device_plan=plan)
    assert r.points_used == 1 and sum(s.active_count() for s in shards) > 0


@pytest.mark.parametrize("plan", [False, True], ids=["host_plan", "device_plan"])
def test_empty_and_tiny_frames(plan):
    from paper_2512_12945_b200 import Mapper
    from paper_2512_12945_b200.sharded import integrate_loopback

    kw = dict(voxel_size=0.05, truncation=0.15, num_classes=3)
    single = Mapper(**kw)
    shards = _shards(4, **kw)
    for pts, lab in [(np.zeros((0, 3)), np.zeros(0, np.int32)),
                     (np.array([[1.0, 0.5, 0.2], [0.3, -1.0, 0.4]]), np.array([1, 3], np.int32)),
                     (np.array([[np.nan, 0.0, 0.0]]), np.array([2], np.int32))]:
        r1 = single.integrate_world(pts, (0.0, 0.0, 0.0), labels=lab)
        r2 = integrate_loopback(shards, pts, origin=(0.0, 0.0, 0.0), labels=lab, device_plan=plan)
        assert np.array_equal(report_rows([r1]), report_rows([r2]))
    _assert_union_equals(single, shards)
    assert all(s.stats()["frames_integrated"] == 3 for s in shards)


def _dist_worker(rank, world, port, kw, seed, out, plan=False):
    import os

    import torch
    import torch.distributed as dist

    from paper_2512_12945_b200.sharded import DistTransport, ShardedMapper

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = ShardedMapper(**kw, rank=rank, world=world, transport=DistTransport())
        m.device_plan = plan
        rng = np.random.default_rng(seed)
        reps = []
        for pts, origin in _frames(seed, 3000, 3):
            lab, _ = _payload(kw, rng, pts.shape[0])
            reps.append(m.integrate_world(pts, origin, labels=lab))
        merged = m.global_export()
        out.put((rank, report_rows(reps).tolist(),
                 None if merged is None else [a.tobytes() for a in merged if a is not None]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("plan", [False, True], ids=["host_plan", "device_plan"])
def test_dist_driver_two_processes_gloo(plan):
    """ShardedMapper.integrate through DistTransport in two processes (gloo
    collectives; both ranks on cuda:0, kernels independent) == one Mapper."""
    import socket

    import torch.multiprocessing as mp

    from paper_2512_12945_b200 import Mapper

    kw = CASES["closed"]
    seed = 21
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dist_worker, args=(r, 2, port, kw, seed, q, plan)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r[0], r[1:]) for r in (q.get(timeout=300) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    single = Mapper(**kw)
    rng = np.random.default_rng(seed)
    reps = []
    for pts, origin in _frames(seed, 3000, 3):
        lab, _ = _payload(kw, rng, pts.shape[0])
        reps.append(single.integrate_world(pts, origin, labels=lab))
    for r in range(2):
        assert res[r][0] == report_rows(reps).tolist()
    assert res[0][1] == [a.tobytes() for a in single._export() if a is not None]
    assert res[1][1] is None

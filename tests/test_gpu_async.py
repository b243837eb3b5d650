"""Asynchronous frames (svx_integrate_async, Mapper(async_frames=N)).

Mapper.integrate queues closed-set / geometry frames without waiting for
them; the report is read on first use and every other call sees the map
after all submitted frames.  The map must be bit-identical to the
synchronous engine and to the oracle, including when a frame in flight
overflows a pool or its row slots and is re-run -- with the frames queued
behind it -- from the frame's own copy of its inputs, even after the caller
has overwritten its buffers.
"""

import numpy as np
import pytest

from helpers import report_rows

pytestmark = pytest.mark.gpu


def _maps_equal(a, b):
    ca, da, wa, sa, _ = a._export()
    cb, db, wb, sb, _ = b._export()
    assert np.array_equal(ca, cb)
    assert np.array_equal(da, db) and np.array_equal(wa, wb)
    if sa is not None or sb is not None:
        assert np.array_equal(sa, sb)


@pytest.mark.parametrize("depth", [1, 2, 4])
@pytest.mark.parametrize("mode", ["auto", "slots", "segments", "leaves"])
def test_async_equals_sync_lidar(mode, depth):
    from paper_2512_12945_b200 import Mapper, scenes

    wl = scenes.workload(2, device="cuda")
    a = Mapper(**wl.mapper_kwargs, async_frames=depth)
    b = Mapper(**wl.mapper_kwargs, async_frames=0)
    a.set_update_mode(mode)
    b.set_update_mode(mode)
    ra, rb = [], []
    for i in range(6):
        f = wl.make_frame(i)
        ra.append(a.integrate(f.points, f.pose, labels=f.labels))
        rb.append(b.integrate(f.points, f.pose, labels=f.labels))
    assert np.array_equal(report_rows(ra), report_rows(rb))
    assert [r.new_voxels for r in ra] == [r.new_voxels for r in rb]
    assert [r.new_blocks for r in ra] == [r.new_blocks for r in rb]
    _maps_equal(a, b)
    assert a.grids[0].content_hash() == b.grids[0].content_hash()
    assert a.grids[1].content_hash() == b.grids[1].content_hash()


def test_async_reports_read_late_and_out_of_order():
    """Reports are held per ticket: reading them late, or newest first,
    gives each frame its own counts."""
    from paper_2512_12945_b200 import Mapper, scenes

    wl = scenes.workload(2, device="cuda")
    a = Mapper(**wl.mapper_kwargs, async_frames=4)
    b = Mapper(**wl.mapper_kwargs, async_frames=0)
    ra = [a.integrate(wl.make_frame(i).points, wl.make_frame(i).pose, labels=wl.make_frame(i).labels)
          for i in range(5)]
    rb = [b.integrate(wl.make_frame(i).points, wl.make_frame(i).pose, labels=wl.make_frame(i).labels)
          for i in range(5)]
    for r1, r2 in zip(reversed(ra), reversed(rb)):
        assert r1.touched_voxels == r2.touched_voxels and r1.new_voxels == r2.new_voxels
    assert a.stats()["frames_integrated"] == 5


@pytest.mark.parametrize("host", [False, True], ids=["device", "host"])
def test_async_capacity_rerun_from_own_copy(host):
    """Tiny leaf pool: frames in flight overflow it and are re-run (with the
    frames queued behind them) from their own input copies -- the caller's
    buffers are overwritten right after each call, so a re-run that read
    them would differ.  Map == oracle bit for bit."""
    import torch

    from oracle.oracle import OracleMap
    from paper_2512_12945_b200 import Mapper, scenes

    wl = scenes.workload(2, device="cuda")
    m = Mapper(**wl.mapper_kwargs, async_frames=4, reserve_voxels=64, reserve_blocks=4,
               async_leaf_headroom=512)
    om = OracleMap(**wl.mapper_kwargs)
    n = wl.points_per_frame
    if host:
        pts_buf = torch.empty((n, 3), dtype=torch.float32, pin_memory=True)
        lab_buf = torch.empty((n,), dtype=torch.int32, pin_memory=True)
    else:
        pts_buf = torch.empty((n, 3), dtype=torch.float32, device="cuda")
        lab_buf = torch.empty((n,), dtype=torch.int32, device="cuda")
    reps, oreps = [], []
    for i in range(5):
        f = wl.make_frame(i * 5)
        pts_buf.copy_(f.points)
        lab_buf.copy_(f.labels)
        if host:
            reps.append(m.integrate(pts_buf.numpy(), f.pose, labels=lab_buf.numpy()))
        else:
            reps.append(m.integrate(pts_buf, f.pose, labels=lab_buf))
        pts_buf.fill_(0.5)          # the caller reuses its buffers at once
        lab_buf.fill_(1)
        oreps.append(om.integrate(f.points.cpu().numpy(), f.pose, labels=f.labels.cpu().numpy()))
    assert np.array_equal(report_rows(reps), report_rows(oreps))
    st = m.engine_stats()
    assert st["async_reruns"] >= 1
    c, d, w, s0, _ = m._export()
    oc, od, ow, os0, _ = om.export()
    assert np.array_equal(c, oc)
    assert np.array_equal(d, od) and np.array_equal(w, ow)
    assert np.array_equal(s0, os0)


@pytest.mark.parametrize("mode", ["slots", "leaves"])
def test_async_slot_overflow_rerun(mode):
    """Depth-camera frames forced into slot mode overflow the 16 row slots
    of close-up voxels while in flight: they are re-run in segment mode from
    their own copies (leaf mode: leaves past 8192 rows do the same).  Map ==
    oracle."""
    from oracle.oracle import OracleMap
    from paper_2512_12945_b200 import Mapper, scenes

    wl = scenes.workload(1, device="cuda")
    m = Mapper(**wl.mapper_kwargs, async_frames=2)
    m.set_update_mode(mode)
    om = OracleMap(**wl.mapper_kwargs)
    reps, oreps = [], []
    for i in range(3):
        f = wl.make_frame(i * 2)
        reps.append(m.integrate(f.points, f.pose, labels=f.labels))
        oreps.append(om.integrate(f.points.cpu().numpy(), f.pose, labels=f.labels.cpu().numpy()))
    assert np.array_equal(report_rows(reps), report_rows(oreps))
    st = m.engine_stats()
    if mode == "slots":
        assert st["slot_overflow_reruns"] >= 1 and st["async_reruns"] >= 1
    c, d, w, s0, _ = m._export()
    oc, od, ow, os0, _ = om.export()
    assert np.array_equal(c, oc)
    assert np.array_equal(d, od) and np.array_equal(w, ow)
    assert np.array_equal(s0, os0)


def test_async_falls_back_when_errors_possible():
    """An infinite max_range leaves the reference's frame errors possible:
    the frame runs synchronously and raises at the call, as the reference
    does, with nothing applied."""
    from paper_2512_12945_b200 import Mapper, SemvoxError

    m = Mapper(voxel_size=1e-6, truncation=3e-6, max_range=float("inf"), async_frames=2)
    pts = np.array([[3.0, 0.0, 0.0], [-3.0, 0.0, 0.0]])
    with pytest.raises(SemvoxError, match="2\\^21"):
        m.integrate(pts, np.eye(4))
    assert m.active_count() == 0
    # the map still works afterwards
    m2 = Mapper(voxel_size=0.05, truncation=0.15, async_frames=2)
    r = m2.integrate(np.array([[1.0, 0.0, 0.0]]), np.eye(4))
    assert r.touched_voxels > 0 and m2.active_count() == r.new_voxels


@pytest.mark.parametrize("backend", [None, "auto", "python", "native", "NATIVE"])
def test_backend_names_accepted(backend):
    """A script that pins a reference backend keeps working: one engine."""
    from paper_2512_12945_b200 import Mapper

    m = Mapper(voxel_size=0.1, truncation=0.3, num_classes=3, backend=backend)
    r = m.integrate(np.array([[1.0, 0.0, 0.0]]), np.eye(4), labels=np.array([2], np.int32))
    assert r.touched_voxels > 0

"""Depth frames: the reference's ingest.project_depth
(ingest.py:285-322) + integrate, against fixtures made by the reference
itself (tests/golden/make_golden.py main_depth).

CPU: the oracle's restatement of project_depth reproduces the reference's
point clouds bit for bit, and the oracle map fed with them reproduces the
reference's map.  GPU: Mapper.integrate_depth (back-projection on the GPU)
reproduces the reference's reports, active set, TSDF, payload statistics and
content hashes bit for bit, from host and from device rasters.
"""

import ast

import numpy as np
import pytest

from helpers import depth_names, load_golden, report_rows

NAMES = depth_names()


def _camera(g):
    return ast.literal_eval(str(g["camera"]))


def _payload_kw(payload):
    if np.issubdtype(payload.dtype, np.floating):
        f = payload.astype(np.float64)
        return dict(features=f.reshape(-1, f.shape[-1]) if f.ndim == 3 else f[:, None])
    return dict(labels=payload.astype(np.int32))


@pytest.mark.parametrize("name", NAMES)
def test_oracle_project_depth_matches_reference(name):
    from oracle.oracle import OracleMap, project_depth

    g = load_golden(name)
    cam = _camera(g)
    om = OracleMap(**g["mapper_kw"])
    reps = []
    for i in range(g["n_frames"]):
        pts, lab, feat = project_depth(g[f"depth_{i}"], g[f"payload_{i}"], cam)
        assert np.array_equal(pts, g[f"ref_points_{i}"])      # bit for bit
        reps.append(om.integrate(pts, g[f"pose_{i}"], labels=lab, features=feat))
    assert np.array_equal(report_rows(reps), g["reports"])
    c, d, w, s0, s1 = om.export()
    assert np.array_equal(c, g["coords"])
    assert np.array_equal(d, g["d"]) and np.array_equal(w, g["w"])


@pytest.mark.gpu
@pytest.mark.parametrize("device_inputs", [False, True], ids=["host", "device"])
@pytest.mark.parametrize("name", NAMES)
def test_gpu_integrate_depth_matches_reference(name, device_inputs):
    import torch

    from paper_2512_12945_b200 import Mapper

    g = load_golden(name)
    cam = _camera(g)
    m = Mapper(**g["mapper_kw"])
    reps = []
    for i in range(g["n_frames"]):
        depth, pay = g[f"depth_{i}"], g[f"payload_{i}"]
        if device_inputs:
            depth = torch.from_numpy(np.ascontiguousarray(depth)).cuda()
            pay = torch.from_numpy(np.ascontiguousarray(pay)).cuda()
        reps.append(m.integrate_depth(depth, pay, cam, pose=g[f"pose_{i}"]))
    assert np.array_equal(report_rows(reps), g["reports"])
    # host-link bytes the library reports for the last call (bench e2e)
    io = m.engine_stats()
    last_d = np.asarray(g[f"depth_{g['n_frames'] - 1}"])
    last_p = np.asarray(g[f"payload_{g['n_frames'] - 1}"])
    pay_bytes = last_p.size * 4   # labels go in as int32, features as float32 here
    want = 0 if device_inputs else last_d.nbytes + pay_bytes
    assert io["last_h2d_bytes"] == want
    assert io["last_d2h_bytes"] > 0
    tsdf, sem = m.grids
    coords, (d, w) = tsdf.active_values()
    assert np.array_equal(coords, g["coords"])
    assert np.array_equal(d, g["d"]) and np.array_equal(w, g["w"])
    assert tsdf.content_hash() == str(g["tsdf_hash"])
    if sem is not None:
        assert sem.content_hash() == str(g["sem_hash"])


@pytest.mark.gpu
def test_integrate_depth_errors():
    from paper_2512_12945_b200 import Mapper
    from paper_2512_12945_b200.errors import ConfigError, PayloadMismatchError

    m = Mapper(voxel_size=0.05, truncation=0.15, num_classes=3)
    cam = dict(fx=50.0, fy=50.0, cx=8.0, cy=6.0, width=16, height=12)
    depth = np.ones((12, 16), np.float32)
    with pytest.raises(ConfigError):
        m.integrate_depth(np.ones((10, 16), np.float32), np.ones((10, 16), np.int32), cam)
    with pytest.raises(ConfigError):
        m.integrate_depth(depth, np.ones((12, 15), np.int32), cam)
    with pytest.raises(ConfigError):
        m.integrate_depth(depth, np.ones((12, 16), np.int32), dict(cam, fx=0.0))
    with pytest.raises(PayloadMismatchError):
        m.integrate_depth(depth, np.ones((12, 16), np.float32), cam)
    r = m.integrate_depth(np.zeros((12, 16), np.float32), np.ones((12, 16), np.int32), cam)
    assert r.points_in == 0 and r.touched_voxels == 0


@pytest.mark.gpu
@pytest.mark.parametrize("stride", [1, 2])
@pytest.mark.parametrize("cfg", [1, 3])
def test_gpu_depth_workload_vs_oracle(cfg, stride):
    """Full-resolution depth frames of the BASELINE camera configs (rotated
    poses) through integrate_depth, bit-exact vs the oracle fed with its own
    project_depth restatement (same world-transform order as the engine)."""
    from oracle.oracle import OracleMap, project_depth
    from paper_2512_12945_b200 import Mapper, scenes

    wl = scenes.workload(cfg, device="cuda")
    kw = dict(wl.mapper_kwargs)
    dim = kw.get("feature_dim")   # cfg3: the BASELINE D = 512
    m = Mapper(**kw)
    om = OracleMap(**kw)
    for i in range(2):
        f = wl.make_frame(i * 4)
        cam = dict(f.camera, stride=stride)
        if dim:
            pay = f.features.reshape(cam["height"], cam["width"], dim).contiguous()
        else:
            pay = f.labels.reshape(cam["height"], cam["width"])
        r1 = m.integrate_depth(f.depth, pay, cam, pose=f.pose)
        pts, lab, feat = project_depth(f.depth.cpu().numpy(), pay.cpu().numpy(), cam)
        r2 = om.integrate(pts, f.pose, labels=lab, features=feat)
        assert np.array_equal(report_rows([r1]), report_rows([r2]))
    c, d, w, s0, s1 = m._export()
    oc, od, ow, os0, os1 = om.export()
    assert np.array_equal(c, oc)
    assert np.array_equal(d, od) and np.array_equal(w, ow)
    assert np.array_equal(s0, os0)
    if s1 is not None:
        assert np.array_equal(s1, os1)

"""The oracle against the reference's own known-answer tests and an
independent interval (slab) oracle, on the CPU.

KATs re-expressed from pkg/tests/test_raycast.py:26-140 and
pkg/tests/test_tsdf.py:35-210; the slab oracle restates the idea of
pkg/tests/raycast_oracle.py:20-56 (dense candidate sampling + half-open
interval overlap) in this repo's own code.
"""

import numpy as np
import pytest

from oracle.oracle import OracleMap, raycast_band


def rows(a):
    return [tuple(int(v) for v in r) for r in np.asarray(a)]


def test_axis_ray_half_open():
    assert rows(raycast_band((0, 0, 0), (1.0, 0, 0), 0.25, 0.25)) == [(3, 0, 0), (4, 0, 0)]


def test_axis_ray_carving():
    assert rows(raycast_band((0, 0, 0), (1.0, 0, 0), 0.25, 0.25, True)) == \
        [(0, 0, 0), (1, 0, 0), (2, 0, 0), (3, 0, 0), (4, 0, 0)]


def test_positive_overlap():
    assert rows(raycast_band((0, 0, 0), (1.0, 0, 0), 0.25, 0.26)) == \
        [(2, 0, 0), (3, 0, 0), (4, 0, 0), (5, 0, 0)]


def test_negative_direction():
    assert rows(raycast_band((0, 0, 0), (-1.0, 0, 0), 0.25, 0.25)) == [(-4, 0, 0), (-5, 0, 0)]


def test_corner_tie_x_first():
    got = rows(raycast_band((0.05, 0.05, 0.05), (0.25, 0.25, 0.05), 0.1, 0.2, True))
    assert got == [(0, 0, 0), (1, 0, 0), (1, 1, 0), (2, 1, 0), (2, 2, 0), (3, 2, 0), (3, 3, 0)]


def slab_band(origin, endpoint, h, trunc, carving):
    """Independent band: every voxel whose [t_enter, t_exit) overlaps
    [t_lo, t_hi), ordered by t_enter (valid for rays in generic position)."""
    origin = np.asarray(origin, np.float64)
    endpoint = np.asarray(endpoint, np.float64)
    delta = endpoint - origin
    ts = float(np.linalg.norm(delta))
    u = delta / ts
    t_lo = 0.0 if carving else max(0.0, ts - trunc)
    t_hi = ts + trunc
    samples = np.arange(0.0, t_hi + h, h / 5.0)
    base = np.floor((origin + samples[:, None] * u) / h).astype(np.int64)
    offs = np.array([(i, j, k) for i in (-1, 0, 1) for j in (-1, 0, 1) for k in (-1, 0, 1)])
    cand = np.unique((base[:, None, :] + offs[None]).reshape(-1, 3), axis=0)
    lo, hi = cand * h, cand * h + h
    with np.errstate(divide="ignore", invalid="ignore"):
        ta = (lo - origin) / u
        tb = (hi - origin) / u
    par = u == 0
    tmin = np.where(par, -np.inf, np.minimum(ta, tb)).max(axis=1)
    tmax = np.where(par, np.inf, np.maximum(ta, tb)).min(axis=1)
    inside = np.all(~par | ((origin >= lo) & (origin < hi)), axis=1)
    keep = inside & (tmax > tmin) & (tmax > t_lo) & (tmin < t_hi)
    order = np.argsort(tmin[keep], kind="stable")
    return rows(cand[keep][order])


@pytest.mark.parametrize("carving", [False, True])
def test_random_rays_vs_slab_oracle(carving):
    rng = np.random.default_rng(2024 + carving)
    checked = 0
    for _ in range(150):
        h = float(rng.choice([0.04, 0.1, 0.25]))
        trunc = h * float(rng.uniform(1.0, 4.0))
        o = rng.uniform(-2.0, 2.0, 3)
        e = o + rng.uniform(-1.5, 1.5, 3)
        if np.linalg.norm(e - o) < 1e-3:
            continue
        got = rows(raycast_band(o, e, h, trunc, carving))
        assert got == slab_band(o, e, h, trunc, carving)
        assert len(set(got)) == len(got)
        checked += 1
    assert checked > 100


def test_identical_updates_never_drift():
    # test_tsdf.py:35-63 / :163-177: the same frame twice doubles the weight
    # exactly and leaves distances unchanged
    rng = np.random.default_rng(11)
    pts = rng.uniform(0.4, 1.3, (40, 3))
    once, twice = OracleMap(0.05, 0.15), OracleMap(0.05, 0.15)
    once.integrate(pts, np.eye(4))
    twice.integrate(pts, np.eye(4))
    twice.integrate(pts, np.eye(4))
    c1, d1, w1, _, _ = once.export()
    c2, d2, w2, _, _ = twice.export()
    assert np.array_equal(c1, c2) and np.array_equal(w2, 2 * w1) and np.array_equal(d1, d2)


def test_skip_counters():
    # test_tsdf.py:222-301
    om = OracleMap(0.05, 0.15, max_range=1.0, num_classes=3)
    pts = np.array([[0.8, 0.1, 0.2], [np.nan, 0, 0], [0, 0, 0], [5.0, 0, 0], [0.7, 0.1, 0.1],
                    [0.6, 0.1, 0.1]])
    r = om.integrate(pts, np.eye(4), labels=np.array([1, 1, 1, 1, 0, 7]))
    assert (r.points_in, r.skipped_nonfinite, r.skipped_degenerate, r.skipped_range,
            r.skipped_bad_label, r.points_used) == (6, 1, 1, 1, 2, 1)


def test_closed_counts_and_ties():
    # dirichlet: exact integer counts, ties to the lowest id (dirichlet.py:38-41)
    om = OracleMap(0.05, 0.15, num_classes=3)
    p = np.array([[1.0, 0.0, 0.0]] * 4)
    om.integrate(p, np.eye(4), labels=np.array([3, 2, 3, 2]))
    _, _, _, counts, _ = om.export()
    assert np.all(counts.sum(axis=1) == 4)
    assert np.all(om.label_map() == 2)


def test_open_hand_example():
    # test_gaussian.py:32-35 style: one voxel, batch of features
    om = OracleMap(0.05, 0.15, feature_dim=2, prior_beta=1e-3, lambda_floor=1e-3,
                   sem_dtype="float64")
    z = np.array([[1.0, 2.0], [3.0, 2.0]])
    p = np.array([[0.5, 0.0, 0.0], [0.5, 0.0, 0.0]])
    om.integrate(p, np.eye(4), features=z)
    _, _, w, m, b = om.export()
    lam = 1e-3
    zbar = z.mean(axis=0)
    want_m = (lam * 0 + z.sum(axis=0)) / (lam + 2)
    ss = ((z - zbar) ** 2).sum(axis=0)
    want_b = 1e-3 + 0.5 * ss + (lam * 2 / (lam + 2)) * zbar ** 2 * 0.5
    np.testing.assert_allclose(m[0], want_m, rtol=1e-15)
    np.testing.assert_allclose(b[0], want_b, rtol=1e-12)

"""Shared test helpers: golden fixtures, replay on the oracle or the engine,
and the comparators (bit-exact where the reference is exact, tolerance
written out where it is not)."""

from __future__ import annotations

import ast
import glob
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")

REPORT_KEYS = ("points_in", "points_used", "skipped_nonfinite", "skipped_range",
               "skipped_degenerate", "skipped_bad_label", "band_hits", "touched_voxels")

# Tolerances (north star: TSDF / weights / semantic statistics within 1e-5
# relative; the absolute floor is 1e-5 * truncation for |d| -> 0).
RTOL = 1e-5


def golden_names():
    """Point-cloud fixtures (api_* / seam_*); depth_* fixtures: depth_names()."""
    return sorted(os.path.splitext(os.path.basename(p))[0]
                  for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                  if os.path.basename(p).startswith(("api_", "seam_")))


def depth_names():
    return sorted(os.path.splitext(os.path.basename(p))[0]
                  for p in glob.glob(os.path.join(GOLDEN, "depth_*.npz")))


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)
    g = {k: z[k] for k in z.files}
    g["mapper_kw"] = ast.literal_eval(str(g["mapper_kw"]))
    g["mode"] = str(g["mode"])
    g["n_frames"] = int(g["n_frames"])
    for i in range(g["n_frames"]):   # compact feature storage (make_golden.api_scenario)
        if f"features16_{i}" in g:
            g[f"features_{i}"] = g.pop(f"features16_{i}").astype(np.float32)
        elif f"featidx_{i}" in g:
            g[f"features_{i}"] = g["featbasis"][g.pop(f"featidx_{i}")]
    return g


def frames_of(g):
    for i in range(g["n_frames"]):
        yield (g[f"points_{i}"], g.get(f"pose_{i}"), g.get(f"origin_{i}"), g.get(f"labels_{i}"),
               g.get(f"features_{i}"))


def oracle_for(g, **extra):
    from oracle.oracle import OracleMap

    kw = dict(g["mapper_kw"])
    kw.update(extra)
    return OracleMap(**kw)


def replay_oracle(g, om):
    reps = []
    for pts, pose, origin, lab, feat in frames_of(g):
        if g["mode"] == "api":
            reps.append(om.integrate(pts, pose, labels=lab, features=feat))
        else:
            reps.append(om.integrate_world(pts, origin, labels=lab, features=feat))
    return reps


def _pinned(a):
    """A copy of numpy array `a` in page-locked host memory (numpy view)."""
    import torch

    if a is None:
        return None
    t = torch.empty(a.shape, dtype=torch.from_numpy(np.ascontiguousarray(a)).dtype,
                    pin_memory=True)
    t.copy_(torch.from_numpy(np.ascontiguousarray(a)))
    return t.numpy()


def replay_mapper(g, mapper, device_inputs=False, pinned=False):
    """Feed a fixture through the engine's Mapper (host numpy arrays -- pageable,
    or page-locked when pinned -- or CUDA tensors when device_inputs)."""
    reps = []
    for pts, pose, origin, lab, feat in frames_of(g):
        if pinned:
            pts, lab, feat = _pinned(pts), _pinned(lab), _pinned(feat)
        if device_inputs:
            import torch

            pts = torch.as_tensor(np.ascontiguousarray(pts)).cuda()
            lab = torch.as_tensor(lab).cuda() if lab is not None else None
            feat = torch.as_tensor(np.ascontiguousarray(feat)).cuda() if feat is not None else None
        if g["mode"] == "api":
            reps.append(mapper.integrate(pts, pose, labels=lab, features=feat))
        else:
            reps.append(mapper.integrate_world(pts, origin, labels=lab, features=feat))
    return reps


def report_rows(reps):
    out = []
    for r in reps:
        get = (lambda k: getattr(r, k))
        out.append([int(get(k)) for k in REPORT_KEYS])
    return np.array(out, np.int64)


def open_state_matches(g, mean, beta):
    """Open-set state vs a fixture: exact arrays, or (large-D fixtures) the
    SHA-256 of the exact float32 arrays in active order."""
    import hashlib

    if "mean" in g:
        return np.array_equal(mean, g["mean"]) and np.array_equal(beta, g["beta"])
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a, np.float32).tobytes()).hexdigest()
    ok_head = (np.array_equal(mean[:32], g["mean_head"]) and np.array_equal(beta[:32], g["beta_head"]))
    return ok_head and sha(mean) == str(g["mean_sha256"]) and sha(beta) == str(g["beta_sha256"])


def assert_close_rel(a, b, rtol=RTOL, atol=0.0, what=""):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    err = np.abs(a - b)
    tol = atol + rtol * np.abs(b)
    bad = err > tol
    assert not bad.any(), f"{what}: {int(bad.sum())} of {a.size} beyond rtol={rtol} atol={atol}; " \
                          f"max err {err.max():.3e}"

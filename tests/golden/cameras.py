"""Render-fixture cameras shared by make_golden.py (which renders the
reference with them) and tests/test_render.py."""

import numpy as np


def _look_at(eye, target, up=(0.0, 0.0, 1.0)):
    """Camera-to-world pose (x right, y down, z forward) looking at target."""
    eye = np.asarray(eye, np.float64)
    z = np.asarray(target, np.float64) - eye
    z /= np.linalg.norm(z)
    x = np.cross(z, np.asarray(up, np.float64))
    if np.linalg.norm(x) < 1e-9:
        x = np.cross(z, np.array([0.0, 1.0, 0.0]))
    x /= np.linalg.norm(x)
    y = np.cross(z, x)
    pose = np.eye(4)
    pose[:3, :3] = np.stack([x, y, z], axis=1)
    pose[:3, 3] = eye
    return pose


RENDER_CAMERAS = {
    # name: (pose, width, height, fx, near, far)
    "front": (np.array([[1, 0, 0, 0.02], [0, 1, 0, -0.01], [0, 0, 1, -1.6], [0, 0, 0, 1.0]]),
              40, 30, 30.0, 0.05, 10.0),
    "oblique": (_look_at([1.1, -0.9, 1.3], [0.0, 0.0, 0.0]), 36, 28, 28.0, 0.05, 10.0),
    "down": (_look_at([0.05, 0.02, 2.0], [0.0, 0.0, 0.0], up=(0.0, 1.0, 0.0)), 40, 30, 30.0,
             0.05, 10.0),
    "down_far_cut": (_look_at([0.05, 0.02, 2.0], [0.0, 0.0, 0.0], up=(0.0, 1.0, 0.0)), 24, 18,
                     18.0, 0.05, 1.9),
    "down_near_skip": (_look_at([0.05, 0.02, 2.0], [0.0, 0.0, 0.0], up=(0.0, 1.0, 0.0)), 24, 18,
                       18.0, 1.99, 10.0),
}

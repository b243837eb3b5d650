"""CPU tests of the boundary: the C-ABI library loads and exports every
symbol include/svx.h declares; the Mapper's config routing and validation
fail exactly like semvox_bindings.Mapper (bindings/__init__.py:77-116,
config.py:44-110) before any device work."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2512_12945_b200 import (ConfigError, Mapper, PayloadMismatchError, SemvoxError,
                                   UserInputError, _lib)
from paper_2512_12945_b200.mapper import _check_pose, validate_rotation

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    h = open(os.path.join(REPO, "include", "svx.h")).read()
    h = re.sub(r"/\*.*?\*/", "", h, flags=re.S)
    return sorted(set(re.findall(r"\b(svx_[a-z_]+)\s*\(", h)))


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(syms) == sorted(_lib.EXPORTED)


def test_abi_version_and_counters():
    assert _lib.lib.svx_abi_version() == 1
    assert _lib.kernel_launches() >= 0


def test_struct_layout_matches_header():
    # svx_config: 3 doubles, 8 int32, 2 doubles, 2 int32, 2 int64
    assert ctypes.sizeof(_lib.SvxConfig) == 3 * 8 + 8 * 4 + 2 * 8 + 2 * 4 + 2 * 8
    assert ctypes.sizeof(_lib.SvxReport) == 10 * 8 + 8
    assert ctypes.sizeof(_lib.SvxStats) == 14 * 8


def test_status_codes_map_to_semvox_classes():
    from paper_2512_12945_b200.errors import OutOfRangeError, STATUS_CLASSES

    assert STATUS_CLASSES[1] is ConfigError
    assert STATUS_CLASSES[2] is PayloadMismatchError
    assert STATUS_CLASSES[3] is UserInputError
    assert STATUS_CLASSES[4] is OutOfRangeError
    assert issubclass(ConfigError, UserInputError) and issubclass(UserInputError, SemvoxError)


class TestConfigRouting:
    def test_unknown_key(self):
        with pytest.raises(ConfigError, match="voxal_size"):
            Mapper(voxal_size=0.1)

    def test_closed_and_open_together(self):
        with pytest.raises(UserInputError, match="not both"):
            Mapper(num_classes=2, feature_dim=3)

    def test_semantic_keys_need_mode(self):
        with pytest.raises(ConfigError, match="num_classes"):
            Mapper(prior_alpha=0.01)
        with pytest.raises(ConfigError, match="feature_dim"):
            Mapper(prior_beta=1.0)

    def test_values_validated(self):
        with pytest.raises(ConfigError):
            Mapper(voxel_size=-1.0)
        with pytest.raises(ConfigError, match="fusion"):
            Mapper(num_classes=2, fusion="bogus")
        with pytest.raises(ConfigError, match="weight_fn"):
            Mapper(weight_fn="gaussian")
        with pytest.raises(ConfigError, match="temperature"):
            Mapper(feature_dim=3, temperature=0.0)
        with pytest.raises(ConfigError, match="tsdf_dtype"):
            Mapper(tsdf_dtype="float16")

    def test_threads_validated(self):
        with pytest.raises(ConfigError, match="threads"):
            Mapper(threads=0)

    def test_backend_key(self):
        """get_backend's names are accepted (backend.py:25-37); others fail
        with the reference's message."""
        with pytest.raises(ConfigError, match=r"unknown backend 'cupy' \(expected auto, python, or native\)"):
            Mapper(backend="cupy")


class TestPoseValidation:
    def test_bottom_row(self):
        T = np.eye(4)
        T[3, 0] = 0.5
        with pytest.raises(UserInputError, match="bottom row"):
            _check_pose(T, 0)

    def test_reorthonormalised(self):
        T = np.eye(4)
        T[0, 1] = 5e-4
        R = _check_pose(T, 0)[:3, :3]
        assert np.abs(R @ R.T - np.eye(3)).max() < 1e-12

    def test_badly_off(self):
        T = np.eye(4)
        T[0, 1] = 0.05
        with pytest.raises(UserInputError, match="orthonormal"):
            _check_pose(T, 0)

    def test_mirrored(self):
        with pytest.raises(UserInputError, match="determinant"):
            validate_rotation(np.diag([-1.0, 1.0, 1.0]))

    def test_shape(self):
        with pytest.raises(UserInputError, match="4x4"):
            _check_pose(np.eye(3), 0)

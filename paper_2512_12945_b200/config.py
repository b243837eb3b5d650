"""Configuration records accepted by :class:`Mapper`.

Field names, defaults and validation messages follow the reference's
dataclasses (pkg/src/semvox/config.py:36-110) so a flat config mapping written
for ``semvox_bindings.Mapper`` routes and fails identically here.  Only what
the integration path consumes is modelled; the tree shape is fixed at the
reference default (8^3 leaves, config.py:26-27).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigError

WEIGHT_FNS = ("constant_one", "linear_dropoff")
CLOSED_FUSION_MODES = ("bayes", "last_wins")
TSDF_DTYPES = ("float64", "float32")


def _float_dtype(name) -> np.dtype:
    """Parse a payload dtype (config.py:146-153 semantics)."""
    try:
        dt = np.dtype(name)
    except TypeError as exc:
        raise ConfigError(f"unknown dtype {name!r}") from exc
    if dt.kind != "f":
        raise ConfigError(f"state dtype must be floating point, got {name!r}")
    return dt


def _engine_dtype(name, what: str) -> np.dtype:
    """Payload dtypes the CUDA engine stores (f32 and f64)."""
    dt = _float_dtype(name)
    if dt not in (np.dtype(np.float32), np.dtype(np.float64)):
        raise ConfigError(f"{what} {name!r} is not supported by the B200 engine (float32/float64)")
    return dt


@dataclass
class FusionConfig:
    """Geometry of the band integration (config.py:36-52)."""

    voxel_size: float = 0.05
    truncation: float = 0.1
    weight_fn: str = "constant_one"
    space_carving: bool = False
    max_range: float = 15.0

    def validate(self) -> None:
        if not self.voxel_size > 0:
            raise ConfigError(f"voxel_size must be positive, got {self.voxel_size}")
        if not self.truncation > 0:
            raise ConfigError(f"truncation must be positive, got {self.truncation}")
        if self.weight_fn not in WEIGHT_FNS:
            raise ConfigError(f"weight_fn must be one of {WEIGHT_FNS}, got {self.weight_fn!r}")
        if not self.max_range > 0:
            raise ConfigError(f"max_range must be positive, got {self.max_range}")


@dataclass
class ClosedSetConfig:
    """Dirichlet class counts over labels 1..num_classes (config.py:55-78)."""

    num_classes: int = 0
    prior_alpha: float = 0.001
    fusion: str = "bayes"
    count_dtype: str = "float32"

    def validate(self) -> None:
        if self.num_classes < 1:
            raise ConfigError(f"num_classes must be >= 1, got {self.num_classes}")
        if not self.prior_alpha > 0:
            raise ConfigError(f"prior_alpha must be positive, got {self.prior_alpha}")
        if self.fusion not in CLOSED_FUSION_MODES:
            raise ConfigError(f"fusion must be one of {CLOSED_FUSION_MODES}, got {self.fusion!r}")
        _engine_dtype(self.count_dtype, "count_dtype")


@dataclass
class OpenSetConfig:
    """Normal-Inverse-Gamma embedding state (config.py:81-110)."""

    feature_dim: int = 0
    prior_beta: float = 1e-3
    lambda_floor: float = 1e-3
    confidence_threshold: float = 0.1
    temperature: float = 0.01
    state_dtype: str = "float32"

    def validate(self) -> None:
        if self.feature_dim < 1:
            raise ConfigError(f"feature_dim must be >= 1, got {self.feature_dim}")
        if not self.prior_beta > 0:
            raise ConfigError(f"prior_beta must be positive, got {self.prior_beta}")
        if not self.lambda_floor > 0:
            raise ConfigError(f"lambda_floor must be positive, got {self.lambda_floor}")
        if not 0.0 <= self.confidence_threshold <= 1.0:
            raise ConfigError(
                f"confidence_threshold must be in [0,1], got {self.confidence_threshold}")
        if not self.temperature > 0:
            raise ConfigError(f"temperature must be positive, got {self.temperature}")
        _engine_dtype(self.state_dtype, "state_dtype")


@dataclass
class EngineConfig:
    """B200-engine knobs that have no reference counterpart.

    tsdf_dtype: "float64" keeps the reference's TSDF layout (grid.py:45-47) and
    makes d/w bit-identical to it; "float32" stores d/w in fp32 (update math
    stays fp64) and halves TSDF traffic.
    async_frames: how many closed-set / geometry frames ``Mapper.integrate``
    may leave in flight on the GPU (0-4; 0 = every call waits for its frame).
    Reports are read when first used; every other call sees the map after
    all submitted frames (svx_integrate_async, include/svx.h).
    async_leaf_headroom: leaf-pool room kept per frame in flight (0 =
    automatic); a frame that runs out anyway is re-run (svx_set_async).
    """

    tsdf_dtype: str = "float64"
    device: int = 0
    reserve_voxels: int = 0
    reserve_blocks: int = 0
    async_frames: int = 2
    async_leaf_headroom: int = 0

    def validate(self) -> None:
        if str(np.dtype(self.tsdf_dtype)) not in TSDF_DTYPES:
            raise ConfigError(f"tsdf_dtype must be one of {TSDF_DTYPES}, got {self.tsdf_dtype!r}")
        if int(self.device) < 0:
            raise ConfigError(f"device must be >= 0, got {self.device}")
        if int(self.reserve_voxels) < 0 or int(self.reserve_blocks) < 0:
            raise ConfigError("reserve_voxels / reserve_blocks must be >= 0")
        if not 0 <= int(self.async_frames) <= 4:
            raise ConfigError(f"async_frames must be in [0, 4], got {self.async_frames}")
        if int(self.async_leaf_headroom) < 0:
            raise ConfigError("async_leaf_headroom must be >= 0")

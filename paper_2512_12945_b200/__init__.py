"""B200-native SLIM-VDB integration engine (arxiv 2512.12945 hot path).

Public surface mirrors the reference's scripting facade
(pkg/bindings/src/semvox_bindings/__init__.py) for the integration path:
``Mapper`` plus the semvox error classes and config records.  The compute
path is libsvx.so (hand-written sm_100a CUDA behind a C ABI, include/svx.h).
"""

from .config import ClosedSetConfig, EngineConfig, FusionConfig, OpenSetConfig
from .errors import (
    ConfigError,
    FormatError,
    OutOfRangeError,
    PayloadMismatchError,
    SemvoxError,
    UserInputError,
)
from .mapper import (GridView, IntegrationReport, Mapper, grids_equal, load_grid,
                     validate_rotation)

from .render import RenderCamera, render, sample_distance
from .surface import SemanticMesh, default_palette, palette_colors, read_ply, write_ply

__version__ = "0.1.0"

__all__ = [
    "Mapper", "load_grid", "grids_equal", "RenderCamera", "render", "sample_distance",
    "SemanticMesh", "default_palette", "palette_colors", "write_ply", "read_ply", "GridView", "IntegrationReport", "validate_rotation",
    "FusionConfig", "ClosedSetConfig", "OpenSetConfig", "EngineConfig",
    "SemvoxError", "UserInputError", "ConfigError", "PayloadMismatchError",
    "FormatError", "OutOfRangeError",
]

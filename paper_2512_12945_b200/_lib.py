"""ctypes binding of libsvx.so (include/svx.h).

The library is built in-tree by ``build.py`` (``__graft_entry__.build()``).
There is no fallback: importing this module without the built library raises,
so no CPU path can silently stand in for the CUDA engine.
"""

from __future__ import annotations

import ctypes
import os

from .errors import STATUS_CLASSES, SemvoxError

LIB_PATH = os.environ.get("SVX_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsvx.so")

SVX_F32, SVX_F64 = 0, 1
SEM_NONE, SEM_CLOSED, SEM_OPEN = 0, 1, 2


class SvxConfig(ctypes.Structure):
    _fields_ = [
        ("voxel_size", ctypes.c_double),
        ("truncation", ctypes.c_double),
        ("max_range", ctypes.c_double),
        ("weight_fn", ctypes.c_int32),
        ("space_carving", ctypes.c_int32),
        ("sem_kind", ctypes.c_int32),
        ("num_classes", ctypes.c_int32),
        ("last_wins", ctypes.c_int32),
        ("count_dtype", ctypes.c_int32),
        ("feature_dim", ctypes.c_int32),
        ("state_dtype", ctypes.c_int32),
        ("prior_beta", ctypes.c_double),
        ("lambda_floor", ctypes.c_double),
        ("tsdf_dtype", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("reserve_voxels", ctypes.c_int64),
        ("reserve_blocks", ctypes.c_int64),
    ]


class SvxReport(ctypes.Structure):
    _fields_ = [
        ("points_in", ctypes.c_int64),
        ("points_used", ctypes.c_int64),
        ("skipped_nonfinite", ctypes.c_int64),
        ("skipped_range", ctypes.c_int64),
        ("skipped_degenerate", ctypes.c_int64),
        ("skipped_bad_label", ctypes.c_int64),
        ("band_hits", ctypes.c_int64),
        ("touched_voxels", ctypes.c_int64),
        ("new_blocks", ctypes.c_int64),
        ("new_voxels", ctypes.c_int64),
        ("kernel_ms", ctypes.c_double),
    ]


class SvxCamera(ctypes.Structure):
    _fields_ = [
        ("fx", ctypes.c_double), ("fy", ctypes.c_double),
        ("cx", ctypes.c_double), ("cy", ctypes.c_double),
        ("depth_scale", ctypes.c_double),
        ("width", ctypes.c_int32), ("height", ctypes.c_int32),
        ("stride", ctypes.c_int32), ("pad", ctypes.c_int32),
    ]


SVX_U16 = 2


class SvxStats(ctypes.Structure):
    _fields_ = [
        ("leaf_count", ctypes.c_int64),
        ("active_voxels", ctypes.c_int64),
        ("resident_bytes", ctypes.c_int64),
        ("payload_bytes_per_voxel", ctypes.c_int64),
        ("frames_integrated", ctypes.c_int64),
        ("hash_capacity", ctypes.c_int64),
        ("voxel_capacity", ctypes.c_int64),
        ("block_capacity", ctypes.c_int64),
        ("frames_slot_mode", ctypes.c_int64),
        ("slot_overflow_reruns", ctypes.c_int64),
        ("async_reruns", ctypes.c_int64),
        ("frames_leaf_mode", ctypes.c_int64),
        ("last_h2d_bytes", ctypes.c_int64),
        ("last_d2h_bytes", ctypes.c_int64),
    ]


MAX_SHARDS = 16


class SvxShardSummary(ctypes.Structure):
    """svx_shard_summary: one rank's march counters, reduced across ranks."""

    _fields_ = [
        ("points_in", ctypes.c_int64),
        ("nonfinite", ctypes.c_int64),
        ("range", ctypes.c_int64),
        ("degenerate", ctypes.c_int64),
        ("bad_label", ctypes.c_int64),
        ("used", ctypes.c_int64),
        ("band_hits", ctypes.c_int64),
        ("rows", ctypes.c_int64),
        ("bbox_min", ctypes.c_int64 * 3),
        ("bbox_max", ctypes.c_int64 * 3),
        ("err_budget", ctypes.c_int64),
        ("err_pack", ctypes.c_int64),
    ]


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_D = ctypes.c_double

# name -> argtypes; every entry point returns svx_status (int32)
_SIGNATURES = {
    "svx_create": [ctypes.POINTER(SvxConfig), ctypes.POINTER(_P)],
    "svx_destroy": [_P],
    # pose / origin as a raw address (a numpy array's .ctypes.data)
    "svx_integrate": [_P, _P, _I32, _I64, _P, _P, _P, _I32, _P, ctypes.POINTER(SvxReport)],
    "svx_integrate_world": [_P, _P, _I32, _I64, _P, _P, _P, _I32, _P,
                            ctypes.POINTER(SvxReport)],
    "svx_integrate_async": [_P, _P, _I32, _I64, _P, _P, _P, ctypes.POINTER(ctypes.c_uint64)],
    "svx_report_wait": [_P, ctypes.c_uint64, ctypes.POINTER(SvxReport)],
    "svx_set_async": [_P, _I32, _I64],
    "svx_integrate_depth": [_P, _P, _I32, ctypes.POINTER(SvxCamera), _P, _P, _P, _I32, _P,
                            ctypes.POINTER(SvxReport)],
    "svx_stats_get": [_P, ctypes.POINTER(SvxStats)],
    "svx_active_count": [_P, ctypes.POINTER(_I64)],
    "svx_export_active": [_P, _I64, _P, _P, _P, _P, _P, _P],
    "svx_probe": [_P, _P, _I64, _P, _P, _P, _P, _P, _P],
    "svx_query_cosine": [_P, _P, _I64, _P, _P],
    "svx_classify": [_P, _P, _I32, _D, _D, _I64, _P, _P, _P, _P],
    "svx_label_map": [_P, _I32, _I64, _P, _P],
    "svx_set_profiling": [_P, _I32],
    "svx_extract_mesh": [_P, ctypes.c_double, _P, _I32, ctypes.c_double, ctypes.c_double, _P, _P,
                         _P],
    "svx_mesh_read": [_P, _P, _P, _P, _P, _P, _I32, _P],
    "svx_render": [_P, _P, _I32, _P, _I32, ctypes.c_double, ctypes.c_double, _P, _I32, _P, _P],
    "svx_sample_distance": [_P, _P, _I64, _P, _P, _P],
    "svx_import": [_P, _I64, _P, _I64, _P, _P, _P, _P, _P, _P, _P],
    "svx_set_update_mode": [_P, _I32],
    "svx_set_score_path": [_P, _I32],
    "svx_reserve": [_P, _I64, _I64],
    "svx_shard_march": [_P, _P, _I32, _I64, ctypes.POINTER(_D), ctypes.POINTER(_D), _P, _P, _I32,
                        ctypes.POINTER(_I64), _P, ctypes.POINTER(SvxShardSummary)],
    "svx_shard_plan": [_P, ctypes.POINTER(SvxShardSummary), _I32, _I32, ctypes.POINTER(_I64),
                       ctypes.POINTER(_I32)],
    "svx_shard_pack": [_P, _P, _I64, _P],
    "svx_shard_apply": [_P, _P, ctypes.POINTER(_I64), _I32, _P, ctypes.POINTER(SvxReport)],
    "svx_export_leaf_stamps": [_P, _I64, _P, _P, _P, ctypes.POINTER(_I64), _P],
    "svx_shard_march_async": [_P, _P, _I32, _I64, ctypes.POINTER(_D), ctypes.POINTER(_D), _P, _P, _I32,
                              ctypes.POINTER(_I64), _P, _P],
    "svx_shard_plan_async": [_P, _P, _I32, _I32, _I64, _P, _P],
    "svx_shard_pack_async": [_P, _P, _I64, _P, _P],
    "svx_shard_apply_async": [_P, _P, _I64, _I32, _P, _I64, _P, _P],
    "svx_shard_finish": [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.POINTER(_I64),
                         ctypes.POINTER(SvxReport), ctypes.POINTER(_I32), ctypes.POINTER(_I64)],
}

SHARD_SUM_WORDS = 10        # svx.h SVX_SHARD_SUM_WORDS
SHARD_SUMMARY_WORDS = 18    # svx.h SVX_SHARD_SUMMARY_WORDS
SHARD_ABORT_WORDS = 8       # svx.h SVX_SHARD_ABORT_WORDS

DEVICE_INPUTS = 0x100   # svx.h SVX_DEVICE_INPUTS
POSE_CHECK = 0x200      # svx.h SVX_POSE_CHECK
POSE_NEEDS_HOST = 8     # svx.h SVX_POSE_NEEDS_HOST

STAGES = ("walk", "resolve", "seg", "scatter", "update", "update_b", "frame")
KERNEL_STAGES = STAGES[:-1]

# every symbol include/svx.h declares (checked by tests/test_abi_and_config.py)
EXPORTED = sorted(list(_SIGNATURES) + ["svx_last_error", "svx_abi_version",
                                       "svx_kernel_launches", "svx_stage_times", "svx_frame_counters",
                                       "svx_leaf_owner"])


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libsvx.so not built at {LIB_PATH}; run `python -c 'import __graft_entry__ as g; "
            f"g.build()'` (the CUDA engine has no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, args in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int32
    lib.svx_last_error.argtypes = []
    lib.svx_last_error.restype = ctypes.c_char_p
    lib.svx_abi_version.argtypes = []
    lib.svx_abi_version.restype = ctypes.c_int32
    lib.svx_kernel_launches.argtypes = []
    lib.svx_kernel_launches.restype = ctypes.c_int64
    lib.svx_stage_times.argtypes = [_P, ctypes.POINTER(_D), _I32]
    lib.svx_stage_times.restype = ctypes.c_int32
    lib.svx_frame_counters.argtypes = [_P, ctypes.POINTER(_I64), _I32]
    lib.svx_frame_counters.restype = ctypes.c_int32
    lib.svx_leaf_owner.argtypes = [_I64, _I64, _I64, _I32]
    lib.svx_leaf_owner.restype = ctypes.c_int32
    return lib


lib = _load()


def check(status: int) -> None:
    """Raise the semvox-equivalent exception for a non-zero svx_status."""
    if status == 0:
        return
    msg = lib.svx_last_error().decode("utf-8", "replace")
    raise STATUS_CLASSES.get(int(status), SemvoxError)(msg)


def kernel_launches() -> int:
    return int(lib.svx_kernel_launches())

"""``.slvg`` map snapshots: the reference's grid-block file format.

A snapshot is a sequence of grid blocks (grid.py:298-356 write_grid_block /
read_grid_block, save_grids / load_grids :410-426); ``Mapper.save`` writes the
TSDF block then the semantic block (bindings/__init__.py:183-187).  One block:

    b"SLVG" | <IdBBBQ version=1, voxel_size, leaf_log2=3, internal_log2=4,
             kind (0 tsdf / 1 closed / 2 open), active_count>
    | payload parameters (tsdf <d truncation>; closed <IdBB C, prior_alpha,
      fusion 0 bayes / 1 last_wins, count dtype code>; open <IddddB D,
      prior_beta, lambda_floor, confidence_threshold, temperature, state dtype
      code>; dtype codes f32 0 / f64 1)
    | <Q n_leaves> | per leaf, in allocation order: <iii origin = leaf << 3>,
      the 512-bit activity mask (8 little-endian u64, bit = slot
      (x&7)<<6 | (y&7)<<3 | (z&7)), then each field's active values in slot
      order (tsdf: d f64 then w f64; closed: counts (n, C); open: mean (n, D)
      then beta (n, D)).

This module is the host side of the format only: the writer takes a map's
active list (``svx_export_active``, leaf-allocation then slot order = the
order the file stores), the reader produces the leaf table + per-voxel
arrays that ``svx_import`` loads onto the GPU.  Files are byte-identical to
the reference's for the same map (tests/test_snapshot.py checks that against
files the reference wrote).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from .errors import FormatError

MAGIC = b"SLVG"                         # grid.py:31
FORMAT_VERSION = 1                      # grid.py:32
KIND_TSDF, KIND_CLOSED, KIND_OPEN = 0, 1, 2
LEAF_LOG2, INTERNAL_LOG2 = 3, 4
LEAF_VOLUME = 1 << (3 * LEAF_LOG2)
MASK_WORDS = LEAF_VOLUME // 64
_HEAD = struct.Struct("<IdBBBQ")
_PARAM_FMT = {KIND_TSDF: "<d", KIND_CLOSED: "<IdBB", KIND_OPEN: "<IddddB"}
_CODE_DTYPES = {0: np.dtype(np.float32), 1: np.dtype(np.float64)}


@dataclass
class GridBlock:
    """One decoded grid block.  ``params`` is the unpacked parameter tuple
    (see the module docstring); ``fields`` the per-voxel arrays in file order
    (tsdf [d, w]; closed [counts]; open [mean, beta])."""

    kind: int
    voxel_size: float
    params: tuple
    leaf_coords: np.ndarray      # (nl, 3) int32, leaf coordinates (voxel >> 3)
    voxel_leaf: np.ndarray       # (nv,) int32, leaf index of each voxel
    voxel_slot: np.ndarray       # (nv,) int32, slot within its leaf
    fields: list

    @property
    def active_count(self) -> int:
        return int(self.voxel_slot.shape[0])

    def coords(self) -> np.ndarray:
        """(nv, 3) int64 voxel coordinates in file order."""
        s = self.voxel_slot.astype(np.int64)
        local = np.stack([(s >> 6) & 7, (s >> 3) & 7, s & 7], axis=1)
        return (self.leaf_coords.astype(np.int64)[self.voxel_leaf] << LEAF_LOG2) + local

    def dtype(self):
        if self.kind == KIND_TSDF:
            return np.dtype(np.float64)
        return _CODE_DTYPES[self.params[-1]]

    def width(self) -> int:
        return 1 if self.kind == KIND_TSDF else int(self.params[0])


def pack_params(kind: int, params: tuple) -> bytes:
    return struct.pack(_PARAM_FMT[kind], *params)


def split_leaves(coords: np.ndarray):
    """Active coords in leaf-then-slot order -> (leaf_coords (nl,3) int64,
    voxel_leaf (n,) int64, voxel_slot (n,) int64).  Consecutive runs of one
    leaf coordinate are one leaf (active order keeps each leaf's voxels
    together, _core.pyx:424-444)."""
    coords = np.asarray(coords, np.int64).reshape(-1, 3)
    n = coords.shape[0]
    lc = coords >> LEAF_LOG2
    s = coords & ((1 << LEAF_LOG2) - 1)
    slot = (s[:, 0] << 6) | (s[:, 1] << 3) | s[:, 2]
    if n == 0:
        return np.zeros((0, 3), np.int64), np.zeros(0, np.int64), slot
    starts = np.ones(n, bool)
    starts[1:] = np.any(lc[1:] != lc[:-1], axis=1)
    voxel_leaf = np.cumsum(starts) - 1
    return lc[starts], voxel_leaf, slot


def write_block(fh, kind: int, voxel_size: float, params: bytes, coords: np.ndarray,
                fields) -> None:
    """write_grid_block (grid.py:325-355) from a map's active list; `params`
    is the packed parameter block (grid.py:276-295)."""
    leaf_coords, voxel_leaf, slot = split_leaves(coords)
    nl = leaf_coords.shape[0]
    n = slot.shape[0]
    if nl and (np.unique(leaf_coords, axis=0).shape[0] != nl
               or np.any(np.diff(voxel_leaf) < 0)):
        raise FormatError("active list is not grouped by leaf")
    fh.write(MAGIC)
    fh.write(_HEAD.pack(FORMAT_VERSION, float(voxel_size), LEAF_LOG2, INTERNAL_LOG2, kind, n))
    if len(params) != struct.calcsize(_PARAM_FMT[kind]):
        raise FormatError("parameter block size does not match the payload kind")
    fh.write(params)
    fh.write(struct.pack("<Q", nl))
    if nl == 0:
        return
    counts = np.bincount(voxel_leaf, minlength=nl)
    off = np.zeros(nl + 1, np.int64)
    np.cumsum(counts, out=off[1:])
    masks = np.zeros((nl, MASK_WORDS), np.uint64)
    np.bitwise_or.at(masks, (voxel_leaf, slot >> 6),
                     np.left_shift(np.uint64(1), (slot & 63).astype(np.uint64)))
    origins = (leaf_coords << LEAF_LOG2).astype(np.int32)
    fields = [np.ascontiguousarray(f) for f in fields]
    row_bytes = [f.reshape(n, -1).view(np.uint8) for f in fields]
    parts = []
    for leaf in range(nl):
        a, b = off[leaf], off[leaf + 1]
        parts.append(origins[leaf].tobytes())
        parts.append(masks[leaf].tobytes())
        for rb in row_bytes:
            parts.append(rb[a:b].tobytes())
        if len(parts) > 4096:
            fh.write(b"".join(parts))
            parts.clear()
    fh.write(b"".join(parts))


def read_block(buf: memoryview, pos: int):
    """read_grid_block (grid.py:358-407) over an in-memory file; returns
    (GridBlock, next offset) or (None, pos) at end of file."""
    if pos == len(buf):
        return None, pos
    head = bytes(buf[pos:pos + 4])
    if head != MAGIC:
        raise FormatError(f"bad grid magic {head!r}")
    pos += 4
    if pos + _HEAD.size > len(buf):
        raise FormatError("truncated grid block header")
    version, voxel_size, ll, il, kind, active = _HEAD.unpack_from(buf, pos)
    pos += _HEAD.size
    if version != FORMAT_VERSION:
        raise FormatError(f"unsupported grid format version {version}")
    if kind not in _PARAM_FMT:
        raise FormatError(f"unknown payload kind {kind}")
    if (ll, il) != (LEAF_LOG2, INTERNAL_LOG2):
        raise FormatError(f"tree shape leaf_log2={ll} internal_log2={il} is not the engine's "
                          f"({LEAF_LOG2}, {INTERNAL_LOG2})")
    pf = struct.Struct(_PARAM_FMT[kind])
    if pos + pf.size + 8 > len(buf):
        raise FormatError("truncated grid block parameters")
    params = pf.unpack_from(buf, pos)
    pos += pf.size
    if kind != KIND_TSDF and params[-1] not in _CODE_DTYPES:
        raise FormatError(f"unknown dtype code {params[-1]}")
    (nl,) = struct.unpack_from("<Q", buf, pos)
    pos += 8
    if nl > (len(buf) - pos) // (12 + 8 * MASK_WORDS):
        raise FormatError(f"leaf count {nl} exceeds the rest of the file")
    if kind != KIND_TSDF and not 1 <= params[0] <= (1 << 20):
        raise FormatError(f"payload width {params[0]} out of range")
    block = GridBlock(kind, voxel_size, params, None, None, None, [])
    dt = block.dtype()
    width = block.width()
    nfield = {KIND_TSDF: 2, KIND_CLOSED: 1, KIND_OPEN: 2}[kind]
    row = width * dt.itemsize
    origins = np.empty((nl, 3), np.int32)
    leaf_of, slot_of, chunks = [], [], [[] for _ in range(nfield)]
    for leaf in range(nl):
        if pos + 12 + 8 * MASK_WORDS > len(buf):
            raise FormatError("truncated leaf record")
        origins[leaf] = np.frombuffer(buf, np.int32, 3, pos)
        mask = np.frombuffer(buf, np.uint8, 8 * MASK_WORDS, pos + 12)
        pos += 12 + 8 * MASK_WORDS
        slots = np.flatnonzero(np.unpackbits(mask, bitorder="little"))
        k = slots.shape[0]
        end = pos + nfield * k * row
        if end > len(buf):
            raise FormatError("truncated leaf payload")
        for fi in range(nfield):
            chunks[fi].append(np.frombuffer(buf, dt, k * width, pos + fi * k * row))
        pos = end
        leaf_of.append(np.full(k, leaf, np.int32))
        slot_of.append(slots.astype(np.int32))
    if np.any(origins & ((1 << LEAF_LOG2) - 1)):
        raise FormatError("leaf origin not aligned to the leaf size")
    block.leaf_coords = (origins >> LEAF_LOG2).astype(np.int32)
    block.voxel_leaf = np.concatenate(leaf_of) if nl else np.zeros(0, np.int32)
    block.voxel_slot = np.concatenate(slot_of) if nl else np.zeros(0, np.int32)
    n = block.voxel_slot.shape[0]
    for fi in range(nfield):
        v = np.concatenate(chunks[fi]) if nl else np.zeros(0, dt)
        block.fields.append(v.reshape(n) if kind == KIND_TSDF else v.reshape(n, width))
    if n != active:
        raise FormatError(f"grid block active count mismatch: header {active}, decoded {n}")
    if nl and np.unique(block.leaf_coords, axis=0).shape[0] != nl:
        raise FormatError("duplicate leaf in grid block")
    return block, pos


def read_blocks(path):
    """load_grids (grid.py:416-426): every block of a snapshot file."""
    with open(path, "rb") as fh:
        return parse(fh.read(), str(path))


def parse(data: bytes, name: str = "snapshot"):
    """Every grid block of an in-memory snapshot."""
    buf = memoryview(data)
    out, pos = [], 0
    while True:
        b, pos = read_block(buf, pos)
        if b is None:
            break
        out.append(b)
    if not out:
        raise FormatError(f"{name}: no grid blocks found")
    return out

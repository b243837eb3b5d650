"""Leaf-sharded integration over G ranks.

The map is split by leaf ownership (``svx_leaf_owner``: high bits of the leaf
hash modulo G).  A frame is cut into G contiguous point slices; rank r marches
slice r, the ranks all-reduce the march summaries (the reference's frame
checks run on the global numbers, so a bad frame fails on every rank before
any shard changes), then each rank sends every owner the points and rows that
fall in its leaves (one all-to-all) and the owners run the usual
resolve/group/update.  Slices are concatenated in rank order, so each voxel's
rows are reduced in the reference's (voxel, point) order and the union of the
shards is the single-GPU map bit for bit (include/svx.h, "sharded
integration").

Two drivers share the per-rank phases:

* ``ShardedMapper.integrate`` -- one process per GPU, collectives through
  ``torch.distributed`` (NCCL over NVLink for CUDA tensors; gloo works for the
  host-side collectives on CPU).
* ``integrate_loopback`` -- all G shards in one process (one GPU), the
  exchange done by device copies; used by the single-GPU parity tests.

Queries gather per-shard results and merge them into the reference's global
active order with the leaf stamps (creation frame, smallest packed key).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import MAX_SHARDS, SVX_F32, SvxShardSummary, check, lib
from .errors import UserInputError
from .mapper import IntegrationReport, Mapper, _check_pose, content_hash_of

_SUM_FIELDS = ("points_in", "nonfinite", "range", "degenerate", "bad_label", "used",
               "band_hits", "rows")
_INT64_MAX = np.iinfo(np.int64).max
_INT64_MIN = np.iinfo(np.int64).min


def slice_bounds(n: int, rank: int, world: int) -> tuple[int, int]:
    """Rank's contiguous slice [lo, hi) of an n-point frame."""
    return (n * rank) // world, (n * (rank + 1)) // world


def leaf_owner(bx: int, by: int, bz: int, world: int) -> int:
    """Owning rank of leaf (bx, by, bz) (svx_leaf_owner)."""
    return int(lib.svx_leaf_owner(int(bx), int(by), int(bz), int(world)))


def summary_to_vectors(s: SvxShardSummary) -> tuple[np.ndarray, np.ndarray]:
    """(sum-reduced, max-reduced) int64 vectors of a summary; bbox minima are
    negated so one MAX reduction covers them."""
    sums = np.array([getattr(s, f) for f in _SUM_FIELDS], np.int64)
    mn = np.array(list(s.bbox_min), np.int64)
    maxes = np.concatenate([np.where(mn == _INT64_MAX, _INT64_MIN, -mn),
                            np.array(list(s.bbox_max), np.int64),
                            np.array([s.err_budget, s.err_pack], np.int64)])
    return sums, maxes


def summary_from_vectors(sums: np.ndarray, maxes: np.ndarray) -> SvxShardSummary:
    s = SvxShardSummary()
    for f, v in zip(_SUM_FIELDS, sums):
        setattr(s, f, int(v))
    for a in range(3):
        nm = int(maxes[a])
        s.bbox_min[a] = _INT64_MAX if nm == _INT64_MIN else -nm
        s.bbox_max[a] = int(maxes[3 + a])
    s.err_budget = int(maxes[6])
    s.err_pack = int(maxes[7])
    return s


def reduce_summaries(parts) -> SvxShardSummary:
    """Host reduction of per-rank summaries (the loopback all-reduce)."""
    vs = [summary_to_vectors(p) for p in parts]
    return summary_from_vectors(np.sum([v[0] for v in vs], axis=0),
                                np.max([v[1] for v in vs], axis=0))


class DistTransport:
    """The two collectives of a sharded frame over ``torch.distributed``."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist

        self._torch, self._dist, self.group = torch, dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        backend = dist.get_backend(group)
        if device is None:
            device = (torch.device("cuda", torch.cuda.current_device()) if backend == "nccl"
                      else torch.device("cpu"))
        self.device = torch.device(device)

    def allreduce_summary(self, s: SvxShardSummary) -> SvxShardSummary:
        torch, dist = self._torch, self._dist
        sums, maxes = summary_to_vectors(s)
        ts = torch.from_numpy(sums).to(self.device)
        tm = torch.from_numpy(maxes).to(self.device)
        dist.all_reduce(ts, op=dist.ReduceOp.SUM, group=self.group)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX, group=self.group)
        return summary_from_vectors(ts.cpu().numpy(), tm.cpu().numpy())

    def allreduce_ints(self, values) -> np.ndarray:
        torch, dist = self._torch, self._dist
        t = torch.tensor(np.asarray(values, np.int64), device=self.device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t.cpu().numpy()

    def exchange(self, send, send_sizes):
        """All-to-all of variable-size byte sections (rank order both ways).
        Returns (recv uint8 tensor, recv sizes)."""
        torch, dist = self._torch, self._dist
        ssz = torch.tensor(list(send_sizes), dtype=torch.int64, device=self.device)
        rsz = torch.empty_like(ssz)
        dist.all_to_all_single(rsz, ssz, group=self.group)
        recv_sizes = [int(v) for v in rsz.cpu().tolist()]
        recv = torch.empty(sum(recv_sizes), dtype=torch.uint8, device=self.device)
        dist.all_to_all_single(recv, send, output_split_sizes=recv_sizes,
                               input_split_sizes=list(int(v) for v in send_sizes),
                               group=self.group)
        return recv, recv_sizes

    def gather_objects(self, obj, dst: int = 0):
        out = [None] * self.world if self.rank == dst else None
        self._dist.gather_object(obj, out, dst=dst, group=self.group)
        return out


class ShardedMapper(Mapper):
    """This rank's shard of a map sharded over ``world`` ranks.

    Construct one per rank with the same configuration; every rank then calls
    ``integrate`` with the same frame (each marches only its own slice; with
    host inputs only the slice is copied to the device).  The readouts
    inherited from ``Mapper`` (grids, query, label_map, active_count, stats)
    read this shard only; the ``global_*`` methods gather the whole map on one
    rank in the reference's active order (collective: every rank calls them).
    """

    def __init__(self, config=None, /, *, rank: int = 0, world: int = 1, transport=None,
                 **overrides):
        if not (1 <= int(world) <= MAX_SHARDS) or not (0 <= int(rank) < int(world)):
            raise UserInputError(f"invalid shard rank {rank} of {world} (1..{MAX_SHARDS} ranks)")
        super().__init__(config, **overrides)
        self.rank, self.world = int(rank), int(world)
        self.transport = transport

    # -- per-rank phases (shared by both drivers) ----------------------------

    def _march(self, pts, vec, sensor, lab, feat, key_base=None):
        s = SvxShardSummary()
        stream = self._stream_handle()
        n = int(pts.shape[0])
        v = np.ascontiguousarray(vec, np.float64)
        vp = v.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        kb = None
        if key_base is not None:
            kba = np.ascontiguousarray(key_base, np.int64)
            kb = kba.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
        check(lib.svx_shard_march(self._handle, pts.ptr, pts.code, n, vp if sensor else None,
                                  None if sensor else vp,
                                  lab.ptr if lab is not None else None,
                                  feat.ptr if feat is not None else None,
                                  feat.code if feat is not None else SVX_F32, kb, stream,
                                  ctypes.byref(s)))
        return s

    def _plan(self, g: SvxShardSummary):
        sizes = (ctypes.c_int64 * self.world)()
        remarch = ctypes.c_int32()
        check(lib.svx_shard_plan(self._handle, ctypes.byref(g), self.rank, self.world, sizes,
                                 ctypes.byref(remarch)))
        return bool(remarch.value), [int(x) for x in sizes]

    def _pack(self, sizes, device):
        import torch

        send = torch.empty(max(sum(sizes), 16), dtype=torch.uint8, device=device)
        check(lib.svx_shard_pack(self._handle, ctypes.c_void_p(send.data_ptr()), send.numel(),
                                 self._stream_handle()))
        return send[: sum(sizes)]

    def _apply(self, recv, recv_sizes, device):
        rep = _lib.SvxReport()
        rs = (ctypes.c_int64 * self.world)(*recv_sizes)
        check(lib.svx_shard_apply(self._handle, ctypes.c_void_p(recv.data_ptr()), rs,
                                  self.world, self._stream_handle(), ctypes.byref(rep)))
        self._frames += 1
        return rep

    def _stream_handle(self):
        """All four calls of a frame run on the current torch stream of the
        map's device."""
        import torch

        return ctypes.c_void_p(torch.cuda.current_stream(int(self._c.device)).cuda_stream)

    def _slice_inputs(self, points, labels, features):
        pts = self._points_arg(points)
        n = int(pts.shape[0])
        lab, feat = self._payload_args(n, labels, features, self._frames)
        lo, hi = slice_bounds(n, self.rank, self.world)
        return _slice_arg(pts, lo, hi), _slice_arg(lab, lo, hi), _slice_arg(feat, lo, hi)

    # -- distributed driver --------------------------------------------------

    def _integrate_dist(self, pts, vec, sensor, lab, feat, reduce_report):
        import torch

        t = self.transport
        if t is None:
            raise UserInputError("ShardedMapper.integrate needs a transport (DistTransport)")
        device = torch.device("cuda", torch.cuda.current_device())
        key_base = None
        while True:
            local = self._march(pts, vec, sensor, lab, feat, key_base)
            g = t.allreduce_summary(local)
            remarch, sizes = self._plan(g)
            if not remarch:
                break
            key_base = list(g.bbox_min)
        send = self._pack(sizes, device)
        if t.device.type != "cuda":   # host transport (gloo): stage through host memory
            recv, recv_sizes = t.exchange(send.cpu(), sizes)
            recv = recv.to(device)
        else:
            recv, recv_sizes = t.exchange(send, sizes)
        rep = self._apply(recv, recv_sizes, device)
        return _report(rep, t.allreduce_ints([rep.touched_voxels, rep.new_blocks,
                                              rep.new_voxels]) if reduce_report else None)

    def integrate(self, points, pose, labels=None, features=None, reduce_report=True):
        """Fuse one frame (the whole frame, passed identically on every rank)
        into the sharded map; see Mapper.integrate.  ``reduce_report`` sums
        touched/new counts over ranks (one small all-reduce)."""
        pose = _check_pose(pose, self._frames)
        pts, lab, feat = self._slice_inputs(points, labels, features)
        return self._integrate_dist(pts, pose.reshape(-1), True, lab, feat, reduce_report)

    def integrate_world(self, points_world, origin, labels=None, features=None,
                        reduce_report=True):
        o = np.asarray(origin, np.float64).reshape(-1)
        if o.shape != (3,) or not np.isfinite(o).all():
            raise UserInputError("origin must be a finite 3-vector")
        pts, lab, feat = self._slice_inputs(points_world, labels, features)
        return self._integrate_dist(pts, o, False, lab, feat, reduce_report)

    # -- shard-local readouts and the merged global view -----------------------

    def leaf_stamps(self):
        """(frame, key, count) per leaf of this shard, in its active order."""
        n = self.engine_stats()["leaf_count"]
        frame = np.empty(n, np.int32)
        key = np.empty(n, np.uint64)
        count = np.empty(n, np.int32)
        nl = ctypes.c_int64()

        def p(a):
            return a.ctypes.data if a.size else None

        check(lib.svx_export_leaf_stamps(self._handle, n, p(frame), p(key), p(count),
                                         ctypes.byref(nl), None))
        return frame[: nl.value], key[: nl.value], count[: nl.value]

    def _stamps_per_voxel(self):
        frame, key, count = self.leaf_stamps()
        return np.repeat(frame, count), np.repeat(key, count)

    def local_export(self):
        """This shard's (coords, d, w, sem0, sem1) in its active order plus the
        per-voxel leaf stamps (frame, key)."""
        return self._export() + self._stamps_per_voxel()

    def local_query(self, embedding):
        """Mapper.query on this shard plus per-voxel leaf stamps."""
        return self.query(embedding) + self._stamps_per_voxel()

    def local_label_map(self, zero_if_empty=False):
        """Mapper.label_map on this shard plus per-voxel leaf stamps."""
        return self.label_map(zero_if_empty) + self._stamps_per_voxel()

    def _gather(self, part, dst):
        if self.transport is None:
            raise UserInputError("global readouts need a transport (DistTransport)")
        parts = self.transport.gather_objects(part, dst)
        return merge_by_stamps(parts) if parts is not None else None

    def global_export(self, dst: int = 0):
        """Whole-map (coords, d, w, sem0, sem1) in the reference's active
        order on rank ``dst`` (None elsewhere)."""
        return self._gather(self.local_export(), dst)

    def global_query(self, embedding, dst: int = 0):
        """Mapper.query over the whole map: (coords, sims) on rank ``dst``.
        Scoring runs on each shard; only the results are gathered."""
        return self._gather(self.local_query(embedding), dst)

    def global_label_map(self, zero_if_empty=False, dst: int = 0):
        """Mapper.label_map over the whole map: (coords, labels) on ``dst``."""
        return self._gather(self.local_label_map(zero_if_empty), dst)


def _slice_arg(a, lo, hi):
    if a is None:
        return None
    import copy

    b = copy.copy(a)
    if a.cuda:
        b.keep = a.keep[lo:hi]
        b.ptr = b.keep.data_ptr() if b.keep.numel() else None
    else:
        b.keep = a.keep[lo:hi]
        b.ptr = b.keep.ctypes.data if b.keep.size else None
    b.shape = (hi - lo,) + tuple(a.shape[1:])
    return b


def _report(rep, sums=None):
    touched, nb, nv = (rep.touched_voxels, rep.new_blocks, rep.new_voxels) if sums is None \
        else (int(sums[0]), int(sums[1]), int(sums[2]))
    return IntegrationReport(
        points_in=rep.points_in, points_used=rep.points_used,
        skipped_nonfinite=rep.skipped_nonfinite, skipped_range=rep.skipped_range,
        skipped_degenerate=rep.skipped_degenerate, skipped_bad_label=rep.skipped_bad_label,
        band_hits=rep.band_hits, touched_voxels=touched, kernel_ms=rep.kernel_ms,
        new_blocks=nb, new_voxels=nv)


def merge_by_stamps(parts):
    """Merge per-shard readouts into the reference's global active order.

    Each part is a tuple of per-voxel arrays in its shard's active order whose
    last two entries are the voxel's leaf stamps (creation frame, smallest
    packed key of that frame); entries may be None.  Leaves sort by stamp
    (the reference allocates a frame's new leaves in first-occurrence order of
    its sorted voxel keys, _core.pyx:377-420); the stable sort keeps each
    leaf's slot order.  Returns the tuple without the stamps."""
    parts = [p for p in parts if p is not None]
    width = len(parts[0])
    cat = [np.concatenate([p[i] for p in parts]) if parts[0][i] is not None else None
           for i in range(width)]
    order = np.lexsort((cat[-1], cat[-2]))
    return tuple(c[order] if c is not None else None for c in cat[:-2])


def integrate_loopback(shards, points, pose=None, origin=None, labels=None, features=None):
    """Integrate one frame into G in-process shards (one GPU): the same phases
    as the distributed driver, with the summary reduction and the all-to-all
    done in-process.  Returns the frame's IntegrationReport."""
    import torch

    G = len(shards)
    if any(s.world != G or s.rank != r for r, s in enumerate(shards)):
        raise UserInputError("shards must be ranks 0..G-1 of a G-rank map")
    device = torch.device("cuda", torch.cuda.current_device())
    sensor = pose is not None
    vec = (_check_pose(pose, shards[0]._frames).reshape(-1) if sensor
           else np.asarray(origin, np.float64).reshape(-1))
    inputs = [s._slice_inputs(points, labels, features) for s in shards]
    key_base = None
    while True:
        locals_ = [s._march(inp[0], vec, sensor, inp[1], inp[2], key_base)
                   for s, inp in zip(shards, inputs)]
        g = reduce_summaries(locals_)
        plans = [s._plan(g) for s in shards]
        if not plans[0][0]:
            break
        key_base = list(g.bbox_min)
    sends = [s._pack(p[1], device) for s, p in zip(shards, plans)]
    reps = []
    for q, s in enumerate(shards):
        pieces, sizes = [], []
        for src in range(G):
            off = sum(plans[src][1][:q])
            sz = plans[src][1][q]
            pieces.append(sends[src][off: off + sz])
            sizes.append(sz)
        recv = torch.cat(pieces) if pieces else torch.empty(0, dtype=torch.uint8, device=device)
        reps.append(s._apply(recv, sizes, device))
    sums = np.sum([[r.touched_voxels, r.new_blocks, r.new_voxels] for r in reps], axis=0)
    return _report(reps[0], sums)


def merged_content_hash(export, view) -> str:
    """content_hash (grid.py:204-215) of a merged export for the payload of
    ``view`` (one shard's GridView: TSDF or semantic)."""
    coords, d, w, s0, s1 = export
    return content_hash_of(coords, view._fields(d, w, s0, s1), view.payload, view.voxel_size)

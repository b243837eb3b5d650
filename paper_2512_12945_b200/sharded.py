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

Each driver runs a frame in one of two plans.  The host plan reads every
phase's result back (summaries, section sizes, headers, report: about seven
host synchronisations per frame).  The device plan (``device_plan=True``, the
default with NCCL) keeps sizes and checks on the device: fixed-capacity
sections, all-to-all of equal blocks, abort words reduced on the device, and
one host synchronisation after the last collective (``svx_shard_*_async``).

Queries gather per-shard results and merge them into the reference's global
active order with the leaf stamps (creation frame, smallest packed key).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import (MAX_SHARDS, SHARD_ABORT_WORDS, SHARD_SUM_WORDS, SHARD_SUMMARY_WORDS, SVX_F32,
                   SvxShardSummary, check, lib)
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

    # -- device-plan collectives (device tensors in, in place; gloo stages through host) --

    def all_reduce(self, tensor, op: str):
        dist = self._dist
        rop = dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX
        if self.device.type == "cuda":
            dist.all_reduce(tensor, op=rop, group=self.group)
        else:
            t = tensor.cpu()
            dist.all_reduce(t, op=rop, group=self.group)
            tensor.copy_(t)

    def all_to_all_equal(self, recv, send):
        """Equal-size blocks: send[q*cap:(q+1)*cap] to rank q, in rank order."""
        if self.device.type == "cuda":
            self._dist.all_to_all_single(recv, send, group=self.group)
        else:
            r = recv.new_empty(recv.shape, device="cpu")
            self._dist.all_to_all_single(r, send.cpu(), group=self.group)
            recv.copy_(r)

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
        self.device_plan = None      # None: device plan when the transport is on CUDA
        self._cap = 0                # device plan: section capacity per destination (bytes)
        self._bufs = {}
        self.host_syncs = 0          # device plan: host synchronisations of the last frame

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

    # -- device-plan phases (one host synchronisation per frame) ---------------

    def _buf(self, name, nbytes, device):
        import torch

        b = self._bufs.get(name)
        if b is None or b.numel() < nbytes:
            b = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=device)
            self._bufs[name] = b
        return b[:nbytes]

    def _initial_cap(self, n_frame):
        pay = 0
        if self._c.sem_kind == _lib.SEM_CLOSED:
            pay = 4
        elif self._c.sem_kind == _lib.SEM_OPEN:
            pay = 8 * int(self._c.feature_dim)
        # a slice's points and ~8 rows each, twice over for an uneven split
        per = -(-int(n_frame) // self.world)
        cap = 2 * per * (32 + pay + 8 * 12) + 65536
        return (cap + 15) // 16 * 16

    def _march_async(self, pts, vec, sensor, lab, feat, key_base, summary):
        v = np.ascontiguousarray(vec, np.float64)
        vp = v.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        kb = None
        if key_base is not None:
            kba = np.ascontiguousarray(key_base, np.int64)
            kb = kba.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
        n = int(pts.shape[0])
        check(lib.svx_shard_march_async(self._handle, pts.ptr, pts.code, n, vp if sensor else None,
                                        None if sensor else vp,
                                        lab.ptr if lab is not None else None,
                                        feat.ptr if feat is not None else None,
                                        feat.code if feat is not None else SVX_F32, kb,
                                        self._stream_handle(), ctypes.c_void_p(summary.data_ptr())))

    def _plan_async(self, gsum, cap, abort):
        check(lib.svx_shard_plan_async(self._handle, ctypes.c_void_p(gsum.data_ptr()), self.rank, self.world,
                                       int(cap), self._stream_handle(), ctypes.c_void_p(abort.data_ptr())))

    def _pack_async(self, send, cap, abort):
        check(lib.svx_shard_pack_async(self._handle, ctypes.c_void_p(send.data_ptr()), int(cap),
                                       self._stream_handle(), ctypes.c_void_p(abort.data_ptr())))

    def _apply_async(self, recv, cap, abort, n_frame, rep):
        check(lib.svx_shard_apply_async(self._handle, ctypes.c_void_p(recv.data_ptr()), int(cap), self.world,
                                        ctypes.c_void_p(abort.data_ptr()), int(n_frame),
                                        self._stream_handle(), ctypes.c_void_p(rep.data_ptr())))

    def _finish(self, summary, abort, rep_sum):
        """After the frame's host synchronisation: (action, need, SvxReport)."""
        sm = np.ascontiguousarray(summary, np.int64)
        ab = np.ascontiguousarray(abort, np.int64)
        rs = None if rep_sum is None else np.ascontiguousarray(rep_sum, np.int64)
        P = ctypes.POINTER(ctypes.c_int64)
        rep = _lib.SvxReport()
        action, need = ctypes.c_int32(), ctypes.c_int64()
        check(lib.svx_shard_finish(self._handle, sm.ctypes.data_as(P), ab.ctypes.data_as(P),
                                   rs.ctypes.data_as(P) if rs is not None else None, ctypes.byref(rep),
                                   ctypes.byref(action), ctypes.byref(need)))
        if action.value == 0 or action.value == 3:
            self._frames += 1
        return action.value, int(need.value), rep

    def _redo_setup(self, host, need):
        """Frame-level redo (action 1): larger sections or the rebased key window."""
        if need:
            self._cap = (need + need // 4 + 15) // 16 * 16
        ab = host[SHARD_SUMMARY_WORDS:SHARD_SUMMARY_WORDS + SHARD_ABORT_WORDS]
        if ab[3]:   # key window: the frame's minimum as key base
            return [-int(host[SHARD_SUM_WORDS + 3 + a]) for a in range(3)]
        return None

    def _integrate_dev(self, pts, vec, sensor, lab, feat, n_frame):
        import torch

        t = self.transport
        device = torch.device("cuda", torch.cuda.current_device())
        G, S, A = self.world, SHARD_SUMMARY_WORDS, SHARD_ABORT_WORDS
        if self._cap == 0:
            self._cap = self._initial_cap(n_frame)
        key_base = None
        self.host_syncs = 0
        while True:
            cap = self._cap
            words = torch.empty(S + A + 4, dtype=torch.int64, device=device)
            summ, abort, rep = words[:S], words[S:S + A], words[S + A:]
            self._march_async(pts, vec, sensor, lab, feat, key_base, summ)
            t.all_reduce(summ[:SHARD_SUM_WORDS], "sum")
            t.all_reduce(summ[SHARD_SUM_WORDS:], "max")
            self._plan_async(summ, cap, abort)
            send = self._buf("send", G * cap, device)
            self._pack_async(send, cap, abort)
            t.all_reduce(abort, "max")
            recv = self._buf("recv", G * cap, device)
            t.all_to_all_equal(recv, send)
            self._apply_async(recv, cap, abort, n_frame, rep)
            mine = rep.clone()
            t.all_reduce(rep, "sum")
            host = words.cpu().numpy()      # the frame's one host synchronisation
            self.host_syncs += 1
            action, need, r = self._finish(host[:S], host[S:S + A], host[S + A:])
            while action in (2, 3):          # a rank re-runs its apply (scratch or pools grown)
                if action == 2:
                    self._apply_async(recv, cap, abort, n_frame, mine)
                rs = mine.clone()
                t.all_reduce(rs, "sum")
                hr = rs.cpu().numpy()
                self.host_syncs += 1
                if action == 2:
                    action, need, r = self._finish(host[:S], host[S:S + A], hr)
                else:
                    r.touched_voxels, r.new_blocks, r.new_voxels = int(hr[0]), int(hr[1]), int(hr[2])
                    action = 3 if hr[3] > 0 else 0
            if action == 0:
                return r
            key_base = self._redo_setup(host, need)

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

    def _integrate_dist(self, pts, vec, sensor, lab, feat, reduce_report, n_frame=None):
        import torch

        t = self.transport
        if t is None:
            raise UserInputError("ShardedMapper.integrate needs a transport (DistTransport)")
        dev_plan = self.device_plan if self.device_plan is not None else t.device.type == "cuda"
        if dev_plan:
            return _report(self._integrate_dev(pts, vec, sensor, lab, feat, n_frame))
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
        n_frame = int(self._points_arg(points).shape[0])
        pts, lab, feat = self._slice_inputs(points, labels, features)
        return self._integrate_dist(pts, pose.reshape(-1), True, lab, feat, reduce_report, n_frame)

    def integrate_world(self, points_world, origin, labels=None, features=None,
                        reduce_report=True):
        o = np.asarray(origin, np.float64).reshape(-1)
        if o.shape != (3,) or not np.isfinite(o).all():
            raise UserInputError("origin must be a finite 3-vector")
        n_frame = int(self._points_arg(points_world).shape[0])
        pts, lab, feat = self._slice_inputs(points_world, labels, features)
        return self._integrate_dist(pts, o, False, lab, feat, reduce_report, n_frame)

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


def integrate_loopback(shards, points, pose=None, origin=None, labels=None, features=None,
                       device_plan=False):
    """Integrate one frame into G in-process shards (one GPU): the same phases
    as the distributed driver, with the summary reduction and the all-to-all
    done in-process.  Returns the frame's IntegrationReport.  ``device_plan``
    runs the one-synchronisation plan (svx_shard_*_async)."""
    import torch

    G = len(shards)
    if any(s.world != G or s.rank != r for r, s in enumerate(shards)):
        raise UserInputError("shards must be ranks 0..G-1 of a G-rank map")
    device = torch.device("cuda", torch.cuda.current_device())
    sensor = pose is not None
    vec = (_check_pose(pose, shards[0]._frames).reshape(-1) if sensor
           else np.asarray(origin, np.float64).reshape(-1))
    inputs = [s._slice_inputs(points, labels, features) for s in shards]
    if device_plan:
        n_frame = int(shards[0]._points_arg(points).shape[0])
        return _report(_loopback_dev(shards, inputs, vec, sensor, n_frame, device))
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


def _loopback_dev(shards, inputs, vec, sensor, n_frame, device):
    """integrate_loopback's device plan: the G shards' phases in lock step,
    the collectives as device reductions and block copies, one host
    synchronisation per frame (plus one per rare apply re-run)."""
    import torch

    G, S, A, SW = len(shards), SHARD_SUMMARY_WORDS, SHARD_ABORT_WORDS, SHARD_SUM_WORDS
    for s in shards:
        if s._cap == 0:
            s._cap = s._initial_cap(n_frame)
    key_base = None
    syncs = 0
    while True:
        cap = max(s._cap for s in shards)
        words = torch.empty((G, S + A + 4), dtype=torch.int64, device=device)
        for s, inp, w in zip(shards, inputs, words):
            s._march_async(inp[0], vec, sensor, inp[1], inp[2], key_base, w[:S])
        words[:, :SW] = words[:, :SW].sum(0)
        words[:, SW:S] = words[:, SW:S].max(0).values
        sends = []
        for s, w in zip(shards, words):
            s._plan_async(w[:S], cap, w[S:S + A])
            send = s._buf("send", G * cap, device)
            s._pack_async(send, cap, w[S:S + A])
            sends.append(send)
        words[:, S:S + A] = words[:, S:S + A].max(0).values
        for q, (s, w) in enumerate(zip(shards, words)):
            recv = s._buf("recv", G * cap, device)
            for src in range(G):
                recv[src * cap:(src + 1) * cap].copy_(sends[src][q * cap:(q + 1) * cap])
            s._apply_async(recv, cap, w[S:S + A], n_frame, w[S + A:])
        mine = words[:, S + A:].clone()
        words[:, S + A:] = words[:, S + A:].sum(0)
        host = words.cpu().numpy()           # the frame's one host synchronisation
        syncs += 1
        res = [s._finish(h[:S], h[S:S + A], h[S + A:]) for s, h in zip(shards, host)]
        while any(a in (2, 3) for a, _, _ in res):
            for i, (s, (a, _, _)) in enumerate(zip(shards, res)):
                if a == 2:
                    s._apply_async(s._bufs["recv"][:G * cap], cap, words[i, S:S + A], n_frame, mine[i])
            hr = mine.sum(0).cpu().numpy()
            syncs += 1
            new = []
            for s, h, (a, need, r) in zip(shards, host, res):
                if a == 2:
                    new.append(s._finish(h[:S], h[S:S + A], hr))
                else:
                    r.touched_voxels, r.new_blocks, r.new_voxels = int(hr[0]), int(hr[1]), int(hr[2])
                    new.append((3 if hr[3] > 0 else 0, need, r))
            res = new
        for s in shards:
            s.host_syncs = syncs
        if all(a == 0 for a, _, _ in res):
            return res[0][2]
        need = max(n for _, n, _ in res)
        kb = [s._redo_setup(host[0], need) for s in shards]
        key_base = kb[0]


def merged_content_hash(export, view) -> str:
    """content_hash (grid.py:204-215) of a merged export for the payload of
    ``view`` (one shard's GridView: TSDF or semantic)."""
    coords, d, w, s0, s1 = export
    return content_hash_of(coords, view._fields(d, w, s0, s1), view.payload, view.voxel_size)

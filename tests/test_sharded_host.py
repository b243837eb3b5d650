"""Host side of the sharded path on CPU: slicing, the summary
all-reduce, leaf ownership, the stamp merge into the reference's active order,
and the collectives themselves over ``torch.distributed`` with gloo at
world_size 2 (the GPU data path is covered by tests/test_gpu_sharded.py)."""

import os
import socket

import numpy as np
import pytest

M64 = (1 << 64) - 1


def _block_hash(a, b, c):
    """block_hash (svx_internal.cuh) restated with Python integers."""
    h = ((a & 0xFFFFFFFF) * 0xD6E8FEB86659FD93) & M64
    h = (h + (b & 0xFFFFFFFF) * 0xA0761D6478BD642F) & M64
    h ^= h >> 31
    h = (h + (c & 0xFFFFFFFF) * 0xE7037ED1A0B428DB) & M64
    h ^= h >> 29
    h = (h * 0x94D049BB133111EB) & M64
    h ^= h >> 32
    return h


def test_block_hash_restatement_matches_header():
    src = open(os.path.join(os.path.dirname(__file__), "..", "paper_2512_12945_b200", "csrc",
                            "svx_internal.cuh")).read()
    body = src[src.index("inline uint64_t block_hash"):]
    body = body[:body.index("}")]
    for const in ("0xD6E8FEB86659FD93", "0xA0761D6478BD642F", "0xE7037ED1A0B428DB",
                  "0x94D049BB133111EB", ">> 31", ">> 29", ">> 32"):
        assert const in body


def test_leaf_owner_formula_and_balance():
    from paper_2512_12945_b200.sharded import leaf_owner

    rng = np.random.default_rng(0)
    leaves = rng.integers(-2**20, 2**20, size=(2000, 3))
    for G in (1, 2, 3, 8, 16):
        got = np.array([leaf_owner(*b, G) for b in leaves])
        want = np.array([(_block_hash(*map(int, b)) >> 32) % G for b in leaves])
        assert np.array_equal(got, want)
    counts = np.bincount(np.array([leaf_owner(*b, 8) for b in leaves]), minlength=8)
    assert counts.min() > 2000 / 8 * 0.75 and counts.max() < 2000 / 8 * 1.25
    assert leaf_owner(0, 0, 0, 0) == -1


def test_slice_bounds_partition():
    from paper_2512_12945_b200.sharded import slice_bounds

    for n in (0, 1, 5, 65536, 921600):
        for G in (1, 2, 3, 7, 8):
            b = [slice_bounds(n, r, G) for r in range(G)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[r][1] == b[r + 1][0] for r in range(G - 1))
            assert max(hi - lo for lo, hi in b) - min(hi - lo for lo, hi in b) <= 1


def _summary(rank):
    from paper_2512_12945_b200._lib import SvxShardSummary

    s = SvxShardSummary()
    s.points_in, s.used, s.rows, s.band_hits = 10 + rank, 7 + rank, 100 * (rank + 1), 55
    s.nonfinite, s.range, s.degenerate, s.bad_label = rank, 2, 0, 3 * rank
    if rank == 2:   # no rows: sentinels
        s.rows = 0
        for a in range(3):
            s.bbox_min[a] = np.iinfo(np.int64).max
            s.bbox_max[a] = np.iinfo(np.int64).min
    else:
        for a in range(3):
            s.bbox_min[a] = -5 * (rank + 1) + a
            s.bbox_max[a] = 3 * rank - a
    s.err_budget = 0
    s.err_pack = 1 if rank == 1 else 0
    return s


def test_summary_vectors_and_reduction():
    from paper_2512_12945_b200.sharded import (reduce_summaries, summary_from_vectors,
                                               summary_to_vectors)

    parts = [_summary(r) for r in range(3)]
    for p in parts:
        q = summary_from_vectors(*summary_to_vectors(p))
        assert bytes(q) == bytes(p)
    g = reduce_summaries(parts)
    assert g.points_in == 33 and g.used == 24 and g.rows == 300 and g.band_hits == 165
    assert list(g.bbox_min) == [-10, -9, -8] and list(g.bbox_max) == [3, 2, 1]
    assert g.err_pack == 1 and g.err_budget == 0
    empty = reduce_summaries([_summary(2)])
    assert list(empty.bbox_min) == [np.iinfo(np.int64).max] * 3


def _global_order_and_shards(seed, G):
    """A global active list (leaves in stamp order, slots ascending) and its
    split over G shards, each in its own stamp order."""
    rng = np.random.default_rng(seed)
    nleaves = 300
    frame = np.sort(rng.integers(0, 6, nleaves)).astype(np.int32)
    key = np.zeros(nleaves, np.uint64)
    for f in np.unique(frame):
        idx = np.nonzero(frame == f)[0]
        key[idx] = np.sort(rng.choice(2**40, idx.size, replace=False)).astype(np.uint64)
    counts = rng.integers(1, 9, nleaves)
    vox_leaf = np.repeat(np.arange(nleaves), counts)
    vox_slot = np.concatenate([np.sort(rng.choice(512, c, replace=False)) for c in counts])
    owner = rng.integers(0, G, nleaves)
    parts = []
    for r in range(G):
        sel = owner[vox_leaf] == r
        ids = np.nonzero(sel)[0]
        perm = np.lexsort((key[vox_leaf[ids]], frame[vox_leaf[ids]]))   # shard's own order
        ids = ids[perm]
        parts.append((vox_leaf[ids], vox_slot[ids], frame[vox_leaf[ids]], key[vox_leaf[ids]]))
    return (vox_leaf, vox_slot), parts


@pytest.mark.parametrize("G", [1, 2, 5])
def test_merge_by_stamps_recovers_global_order(G):
    from paper_2512_12945_b200.sharded import merge_by_stamps

    (leaf, slot), parts = _global_order_and_shards(G, G)
    ml, ms = merge_by_stamps(parts)
    assert np.array_equal(ml, leaf) and np.array_equal(ms, slot)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    from paper_2512_12945_b200.sharded import DistTransport, merge_by_stamps

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = DistTransport()
        g = t.allreduce_summary(_summary(rank))
        # variable sections, one of them empty: rank r sends (r+1)*16 bytes
        # of value 10*r+dst to each dst != r+1, nothing to dst == r+1
        sizes = [0 if d == rank + 1 else 16 * (rank + 1) for d in range(world)]
        send = torch.cat([torch.full((sz,), 10 * rank + d, dtype=torch.uint8)
                          for d, sz in enumerate(sizes)])
        recv, rsz = t.exchange(send, sizes)
        got = []
        off = 0
        for src, sz in enumerate(rsz):
            got.append((src, sz, sorted(set(recv[off:off + sz].tolist()))))
            off += sz
        _, parts = _global_order_and_shards(9, world)
        merged = t.gather_objects(parts[rank], dst=0)
        merged = merge_by_stamps(merged) if merged is not None else None
        ints = t.allreduce_ints([rank + 1, 2])
        out.put((rank, bytes(g), got, None if merged is None else [m.tolist() for m in merged],
                 ints.tolist()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_collectives():
    import torch.multiprocessing as mp

    from paper_2512_12945_b200.sharded import reduce_summaries

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, g, got, merged, ints = q.get(timeout=120)
        res[rank] = (g, got, merged, ints)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = bytes(reduce_summaries([_summary(r) for r in range(world)]))
    for rank in range(world):
        g, got, merged, ints = res[rank]
        assert g == want
        assert ints == [3, 4]
        for src, sz, vals in got:
            exp = 0 if rank == src + 1 else 16 * (src + 1)
            assert sz == exp
            assert vals == ([] if exp == 0 else [10 * src + rank])
    (leaf, slot), _ = _global_order_and_shards(9, world)
    assert res[0][2] == [leaf.tolist(), slot.tolist()]
    assert res[1][2] is None

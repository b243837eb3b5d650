// svx_resolve.cu -- K2: rows -> persistent voxel ids (leaf find-or-insert,
// voxel activation) and per-voxel row counts; K3: row segments.
//
// This is where the reference's grouping (_core.pyx:707-753) and allocation
// (ensure_coords, _core.pyx:377-420; _resolve_leaf_alloc :248-280) happen.
// Rows are grouped by the voxel's persistent id rather than by a per-frame
// key table: each row resolves its voxel once (lanes of a warp that hit the
// same voxel, or the same leaf, share one lookup), counts itself in the
// voxel's vcnt and the voxel's first toucher appends it to the frame's
// touched list.  Only voxels with several rows need a segment (their rows
// are re-sorted by point index later); single-row voxels of closed/geometry
// maps are finished in ray order by the scatter.
//
// Leaf order: new leaves take arrival-order ids and record (creation frame,
// smallest frame key of their voxels); frame keys are x-major offsets from
// one base, so that stamp is the reference's first-occurrence order and
// queries recover the reference's allocation order from it (svx_query.cu).
//
// Capacity: pools are sized before the frame from the previous frames; a
// pool that still runs out sets err_cap, rolls its claim back, and the host
// cleans up (launch_cleanup), grows and re-runs the frame.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "svx_internal.cuh"

namespace svx {
namespace {

constexpr int kResolveThreads = 256;
constexpr int kSegThreads = 256;
constexpr int kSegTile = kSegThreads * 4;
constexpr int kSegBlocks = 148 * 4;

__device__ __forceinline__ int slot_of(long long x, long long y, long long z) {
    return (int)(((x & 7) << 6) | ((y & 7) << 3) | (z & 7));
}

// counter += 1 for every converged lane, one atomic per warp; returns this
// lane's ticket.
__device__ __forceinline__ unsigned long long warp_ticket(unsigned long long* counter) {
    const unsigned mask = __activemask();
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(mask) - 1;
    const unsigned rank = __popc(mask & ((1u << lane) - 1u));
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(counter, (unsigned long long)__popc(mask));
    base = __shfl_sync(mask, base, leader);
    return base + rank;
}

// 16-byte volatile store / load of a hash slot (one transaction each).
__device__ __forceinline__ void st_slot(int4* p, int4 v) {
    asm volatile("st.volatile.global.v4.s32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

__device__ __forceinline__ int4 ld_slot(const int4* p) {
    int4 v;
    asm volatile("ld.volatile.global.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}

// Leaf find-or-insert.  A claimed slot stays BUSY until the new leaf's id,
// coordinates and creation frame are written; then the id is published.
// Returns -1 (and sets err_cap) when the leaf pool is full.
__device__ int leaf_find_or_insert(int4* table, long long mask, int a, int b, int c, int frame,
                                   long long bcap, int4* bcoord, FrameCtr* ctr) {
    long long pos = (long long)(block_hash(a, b, c) & (unsigned long long)mask);
    while (true) {
        // Fast path: one 16-byte L2 read.  Key and id are published together
        // by one 16-byte store, so a matching key is final -- almost every
        // lookup ends here.
        const int4 sv = __ldcg(table + pos);
        if (sv.w >= 0) {
            if (sv.x == a && sv.y == b && sv.z == c) return sv.w;
            pos = (pos + 1) & mask;
            continue;
        }
        volatile int* vw = &table[pos].w;
        int v = sv.w;
        if (v == kHashEmpty) {
            int old = atomicCAS((int*)&table[pos].w, kHashEmpty, kHashBusy);
            if (old == kHashEmpty) {
                const long long id = (long long)warp_ticket(&ctr->nblocks);
                if (id >= bcap) {
                    atomicExch((int*)&table[pos].w, kHashEmpty);
                    atomicOr(&ctr->err_cap, 1);
                    return -1;
                }
                bcoord[id] = make_int4(a, b, c, frame);
                // publish key and id with one 16-byte store: a reader sees the
                // slot either BUSY or complete (no fence on the creating side)
                st_slot(table + pos, make_int4(a, b, c, (int)id));
                return (int)id;
            }
            v = old;
        }
        while (v == kHashBusy) {
            __nanosleep(20);
            v = *vw;
        }
        if (v == kHashEmpty) {   // a creator rolled back (pool full)
            atomicOr(&ctr->err_cap, 1);
            return -1;
        }
        const int4 full = ld_slot(table + pos);
        if (full.x == a && full.y == b && full.z == c) return full.w;
        pos = (pos + 1) & mask;
    }
}

// K2: rows -> voxel ids, in CTA-synchronous tiles of 256 rows so that every
// allocation counter (leaves, voxels, touched list) is bumped once per tile
// after a block scan -- never per thread.  Within a warp, lanes that hit the
// same voxel elect one leader (one lookup, one count of popc(peers)), and
// voxel leaders that share a leaf elect one leaf lookup.  A slot claimed by
// another CTA (BUSY) is waited for after this tile's own claims are
// published, so no thread ever waits across a barrier.
__global__ void __launch_bounds__(kResolveThreads) k_resolve(
    const unsigned long long* __restrict__ rowkey, const int* __restrict__ rowray,
    const double* __restrict__ rowd, const int* __restrict__ rowlab,
    int* __restrict__ rowvid, RowSlot* __restrict__ vslot, int4* table, int4* bcoord,
    unsigned long long* bkey, unsigned long long* bmask, int* bslot, VoxFrame* rec,
    int* __restrict__ tlist, FrameCtr* ctr) {
    grid_dep_wait();
    using Scan = cub::BlockScan<int, kResolveThreads>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ unsigned long long s_base;
    if (ctr->abort) return;
    const FrameParams& fp = ctr->p;
    const long long total = (long long)ctr->rows;
    const KeyPack kp = fp.kp;
    const long long hmask = fp.hmask, bcap = fp.bcap, vcap = fp.vcap, nblocks0 = fp.nblocks0;
    const int frame = fp.frame;
    const bool slots = fp.slots != 0;
    const int lane = threadIdx.x & 31;
    const unsigned full = 0xffffffffu;
    for (long long tile = blockIdx.x; tile * kResolveThreads < total; tile += gridDim.x) {
        const long long t = tile * kResolveThreads + threadIdx.x;
        const bool valid = t < total;
        const unsigned long long key = valid ? rowkey[t] : kKeyEmpty;
        RowSlot rsl{0, 0, 0.0};
        if (valid && slots) {
            rsl.point = rowray[t];
            rsl.label = rowlab[t];
            rsl.d = rowd[t];
        }
        long long x = 0, y = 0, z = 0;
        if (valid) unpack_key(key, kp, x, y, z);
        const unsigned vpeers = __match_any_sync(full, valid ? key : (kKeyEmpty ^ (unsigned long long)lane));
        const int vleader = __ffs(vpeers) - 1;
        const bool is_vl = valid && lane == vleader;
        // exact leaf identity: leaf coords relative to the base's leaf, 19 bits each
        const int la = (int)(x >> kLeafLog2), lb = (int)(y >> kLeafLog2), lc = (int)(z >> kLeafLog2);
        const unsigned long long lkey =
            is_vl ? (((unsigned long long)(la - (kp.base[0] >> kLeafLog2)) << 38) |
                     ((unsigned long long)(lb - (kp.base[1] >> kLeafLog2)) << 19) |
                     (unsigned long long)(lc - (kp.base[2] >> kLeafLog2)))
                  : (~0ULL ^ (unsigned long long)lane);
        const unsigned lpeers = __match_any_sync(full, lkey);
        const int lleader = __ffs(lpeers) - 1;
        const bool is_ll = is_vl && lane == lleader;

        // ---- leaves: find, or claim an empty slot; ids for the tile's claims
        int id = -1, lstate = 0;   // 1 = claimed here, 2 = another CTA's claim
        long long lpos = 0;
        if (is_ll) {
            lpos = (long long)(block_hash(la, lb, lc) & (unsigned long long)hmask);
            while (true) {
                const int4 sv = __ldcg(table + lpos);
                if (sv.w >= 0) {
                    if (sv.x == la && sv.y == lb && sv.z == lc) { id = sv.w; break; }
                    lpos = (lpos + 1) & hmask;
                    continue;
                }
                if (sv.w == kHashBusy) { lstate = 2; break; }
                const int old = atomicCAS(&table[lpos].w, kHashEmpty, kHashBusy);
                if (old == kHashEmpty) { lstate = 1; break; }
                // lost the race for this slot: look at it again
            }
        }
        int rank, cnt;
        Scan(scan_tmp).ExclusiveSum(lstate == 1 ? 1 : 0, rank, cnt);
        if (threadIdx.x == 0 && cnt) s_base = atomicAdd(&ctr->nblocks, (unsigned long long)cnt);
        __syncthreads();
        if (lstate == 1) {
            const long long nid = (long long)s_base + rank;
            if (nid >= bcap) {
                atomicExch(&table[lpos].w, kHashEmpty);
                atomicOr(&ctr->err_cap, 1);
            } else {
                bcoord[nid] = make_int4(la, lb, lc, frame);
                st_slot(table + lpos, make_int4(la, lb, lc, (int)nid));   // key + id in one store
                id = (int)nid;
            }
        }
        __syncthreads();
        if (lstate == 2) {   // another CTA is publishing this slot (maybe another key)
            volatile int* vw = &table[lpos].w;
            int v = *vw;
            while (v == kHashBusy) {
                __nanosleep(32);
                v = *vw;
            }
            const int4 sv = ld_slot(table + lpos);
            if (v >= 0 && sv.x == la && sv.y == lb && sv.z == lc) id = v;
            else id = leaf_find_or_insert(table, hmask, la, lb, lc, frame, bcap, bcoord, ctr);
        }
        id = __shfl_sync(full, id, lleader);

        // ---- voxels: find, or claim an inactive slot; ids for the tile's claims
        int vid = -1, vstate = 0;
        int* sp = nullptr;
        const int slot = slot_of(x, y, z);   // GridCore.activate_slot, _core.pyx:312-322
        if (is_vl && id >= 0) {
            if (id >= nblocks0) atomicMin(&bkey[id], key);
            sp = &bslot[(long long)id * kLeafVolume + slot];
            int v = __ldcg(sp);
            if (v == -1) {
                v = atomicCAS(sp, -1, -2);
                if (v == -1) vstate = 1;
            }
            if (vstate == 0) {
                if (v >= 0) vid = v;
                else vstate = 2;   // another CTA claimed it
            }
        }
        Scan(scan_tmp).ExclusiveSum(vstate == 1 ? 1 : 0, rank, cnt);
        if (threadIdx.x == 0 && cnt) s_base = atomicAdd(&ctr->nvox, (unsigned long long)cnt);
        __syncthreads();
        bool created = false;
        if (vstate == 1) {
            const long long nv = (long long)s_base + rank;
            if (nv >= vcap) {
                atomicExch(sp, -1);
                atomicOr(&ctr->err_cap, 1);
            } else {
                atomicOr(&bmask[(long long)id * kMaskWords + (slot >> 6)], 1ULL << (slot & 63));
                atomicExch(sp, (int)nv);
                vid = (int)nv;
                created = true;
            }
        }
        __syncthreads();
        if (vstate == 2) {
            volatile int* vsp = sp;
            int v = *vsp;
            while (v == -2) {
                __nanosleep(32);
                v = *vsp;
            }
            if (v >= 0) vid = v;
            else atomicOr(&ctr->err_cap, 1);
        }

        // ---- counts; the voxel's first toucher this frame lists it
        bool first = false;
        unsigned cbase = 0;
        if (is_vl && vid >= 0) {
            const unsigned c = atomicAdd(&rec[vid].cnt, (unsigned)__popc(vpeers) + (created ? kNewBit : 0u));
            cbase = c & ~kNewBit;
            first = cbase == 0u;
        }
        Scan(scan_tmp).ExclusiveSum(first ? 1 : 0, rank, cnt);
        if (threadIdx.x == 0 && cnt) s_base = atomicAdd(&ctr->n_touched, (unsigned long long)cnt);
        __syncthreads();
        if (first) {
            rec[vid].key = key;
            tlist[s_base + rank] = vid;
        }
        vid = __shfl_sync(full, vid, vleader);
        if (slots) {
            // this row's rank among the voxel's rows = its slot (order is
            // restored by point index in k_update_slots)
            cbase = __shfl_sync(full, cbase, vleader) + __popc(vpeers & ((1u << lane) - 1u));
            if (valid && vid >= 0) {
                if (cbase < (unsigned)kSlots) vslot[(long long)vid * kSlots + cbase] = rsl;
                else ctr->err_slots = 1;
            }
        } else if (valid) {
            rowvid[t] = vid;
        }
        __syncthreads();
    }
}

// K3: one pass over the touched list with a decoupled look-back scan.
// Listed voxels (multi-row ones, or all for open-set maps) go to mlist in
// touched-list order and get contiguous row segments (vseg).  Tiles are
// claimed in order from a frame counter, so a tile only ever waits on tiles
// already running.  Tile status words are 16-byte {tag, value} records
// written and read with one transaction; tag = seq << 2 | flag (1 = tile
// aggregate, 2 = inclusive prefix), so records of earlier launches never
// match and the array needs no clearing.  value = listed << 40 | rows.
struct alignas(16) SegStatus {
    unsigned long long tag, val;
};

__device__ __forceinline__ void st_status(SegStatus* p, unsigned long long tag, unsigned long long v) {
    asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(tag), "l"(v) : "memory");
}

__device__ __forceinline__ void ld_status(const SegStatus* p, unsigned long long& tag,
                                          unsigned long long& v) {
    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(tag), "=l"(v) : "l"(p) : "memory");
}

__global__ void __launch_bounds__(kSegThreads) k_seg(const int* __restrict__ tlist,
                                                     VoxFrame* __restrict__ rec,
                                                     int* __restrict__ mlist,
                                                     SegStatus* __restrict__ status, FrameCtr* ctr) {
    grid_dep_wait();
    using Scan = cub::BlockScan<unsigned long long, kSegThreads>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ unsigned long long s_prefix;
    __shared__ long long s_tile;
    if (ctr->abort | ctr->err_cap) return;
    const long long n = (long long)ctr->n_touched;
    const int singles = ctr->p.inline_singles;
    const unsigned long long seq = ctr->p.seq;
    const unsigned long long low40 = (1ULL << 40) - 1;
    const long long ntiles = (n + kSegTile - 1) / kSegTile;
    const int lane = threadIdx.x & 31;
    while (true) {
        if (threadIdx.x == 0) s_tile = (long long)atomicAdd(&ctr->seg_tiles, 1u);
        __syncthreads();
        const long long tile = s_tile;
        if (tile >= ntiles) break;
        const long long e0 = tile * kSegTile + (long long)threadIdx.x * 4;
        int vv[4];
        unsigned cc[4];
        bool li[4];
        unsigned cnt = 0, rows = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const long long e = e0 + q;
            vv[q] = e < n ? tlist[e] : -1;
            cc[q] = vv[q] >= 0 ? (rec[vv[q]].cnt & ~kNewBit) : 0u;
            li[q] = vv[q] >= 0 && (!singles || cc[q] > 1u);
            cnt += li[q];
            rows += li[q] ? cc[q] : 0u;
        }
        unsigned long long pre, agg;
        Scan(scan_tmp).ExclusiveSum(((unsigned long long)cnt << 40) | rows, pre, agg);
        if (threadIdx.x < 32) {
            unsigned long long prefix = 0;
            if (tile == 0) {
                if (lane == 0) st_status(status, seq << 2 | 2, agg);
            } else {
                if (lane == 0) st_status(status + tile, seq << 2 | 1, agg);
                // look back 32 tiles at a time until an inclusive prefix
                long long hi = tile - 1;
                while (true) {
                    const long long p = hi - lane;
                    unsigned long long tag = seq << 2 | 2, v = 0;
                    if (p >= 0) ld_status(status + p, tag, v);
                    const unsigned ready = __ballot_sync(0xffffffffu, (tag >> 2) == seq && (tag & 3) != 0);
                    const unsigned incl = __ballot_sync(0xffffffffu, (tag >> 2) == seq && (tag & 3) == 2);
                    // lanes up to the first inclusive one must all be ready
                    const unsigned upto = incl ? (incl & (0u - incl)) * 2u - 1u : 0xffffffffu;
                    if ((ready & upto) != upto) continue;   // a predecessor not yet published
                    unsigned long long part = ((upto >> lane) & 1u) ? v : 0ULL;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
                    prefix += part;
                    if (incl) break;
                    hi -= 32;
                }
                if (lane == 0) st_status(status + tile, seq << 2 | 2, prefix + agg);
            }
            if (lane == 0) {
                s_prefix = prefix;
                if (tile == ntiles - 1) {
                    ctr->n_list = (prefix + agg) >> 40;
                    ctr->rows_seg = (prefix + agg) & low40;
                }
            }
        }
        __syncthreads();
        const unsigned long long base = s_prefix + pre;
        unsigned long long u = base >> 40, r = base & low40;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (!li[q]) continue;
            mlist[u] = vv[q];
            rec[vv[q]].seg = (unsigned)r;
            ++u;
            r += cc[q];
        }
    }
}

// After a capacity abort: give the voxels activated by the failed attempt
// their background state (they stay active and are found again by the
// retry) and clear the per-voxel frame counts.
template <class TD, class TS>
__global__ void k_cleanup(const int* __restrict__ tlist, VoxFrame* rec, TD* vt,
                          TS* mean, TS* beta, int D, double trunc, double prior_beta,
                          const FrameCtr* __restrict__ ctr) {
    const long long n = (long long)ctr->n_touched;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x) {
        const int vid = tlist[e];
        if (rec[vid].cnt & kNewBit) {
            vt[2 * (long long)vid] = (TD)trunc;
            vt[2 * (long long)vid + 1] = (TD)0;
            if (mean) {
                for (int c = 0; c < D; ++c) {
                    mean[(long long)vid * D + c] = (TS)0;
                    beta[(long long)vid * D + c] = (TS)prior_beta;
                }
            }
        }
        rec[vid].cnt = 0u;
        rec[vid].cur = 0u;
    }
}

template <class TD, class TS>
svx_status cleanup_t(svx_map* m, cudaStream_t s) {
    const bool open = m->cfg.sem_kind == SVX_SEM_OPEN;
    k_cleanup<TD, TS><<<kPersistentBlocks, 256, 0, s>>>(
        ptr<int>(m->tlist), ptr<VoxFrame>(m->vrec), ptr<TD>(m->vt),
        open ? ptr<TS>(m->s0) : nullptr, open ? ptr<TS>(m->s1) : nullptr, m->payload_d,
        m->cfg.truncation, m->cfg.prior_beta, ptr<FrameCtr>(m->ctr));
    SVX_LAUNCHED();
    return SVX_OK;
}

}  // namespace

svx_status launch_resolve(svx_map* m, cudaStream_t s) {
    SVX_CUDA(launch_pdl(k_resolve, kPersistentBlocks, kResolveThreads, 0, s, 
        ptr<unsigned long long>(m->rowkey), ptr<int>(m->rowray), ptr<double>(m->rowd), ptr<int>(m->rowlab),
        ptr<int>(m->rowvid), ptr<RowSlot>(m->vslot),
        ptr<int4>(m->hash), ptr<int4>(m->bcoord),
        ptr<unsigned long long>(m->bkey), ptr<unsigned long long>(m->bmask), ptr<int>(m->bslot),
        ptr<VoxFrame>(m->vrec), ptr<int>(m->tlist),
        ptr<FrameCtr>(m->ctr)));
    SVX_LAUNCHED();
    return SVX_OK;
}

svx_status launch_segments(svx_map* m, cudaStream_t s) {
    SegStatus* status =
        reinterpret_cast<SegStatus*>(ptr<char>(m->partials) + partials_bytes());
    SVX_CUDA(launch_pdl(k_seg, kSegBlocks, kSegThreads, 0, s, ptr<int>(m->tlist), ptr<VoxFrame>(m->vrec),
                                             ptr<int>(m->mlist), status,
                                             ptr<FrameCtr>(m->ctr)));
    SVX_LAUNCHED();
    return SVX_OK;
}

svx_status launch_cleanup(svx_map* m, cudaStream_t s) {
    const bool t64 = m->cfg.tsdf_dtype == SVX_F64, s64 = m->cfg.state_dtype == SVX_F64;
    if (t64) return s64 ? cleanup_t<double, double>(m, s) : cleanup_t<double, float>(m, s);
    return s64 ? cleanup_t<float, double>(m, s) : cleanup_t<float, float>(m, s);
}

size_t segment_status_bytes(unsigned long long ucap) {
    return sizeof(SegStatus) * (ucap / kSegTile + 2);
}

}  // namespace svx

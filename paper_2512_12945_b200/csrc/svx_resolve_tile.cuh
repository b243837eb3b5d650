// svx_resolve_tile.cuh -- one CTA-synchronous resolve step (K2 logic) for
// k_resolve, and the leaf hash helpers the leaf-mode binning kernel
// (svx_leaf.cu) shares with it.
//
// Rows -> voxel ids: within a warp, lanes that hit the same voxel elect one
// leader (one lookup, one count of popc(peers)), and voxel leaders that share
// a leaf elect one leaf lookup; every allocation counter (leaves, voxels,
// touched list) is bumped once per step after a block scan.  A slot claimed
// by another CTA (BUSY) is waited for after this step's own claims are
// published, so no thread ever waits across a barrier.  This is the
// reference's grouping + allocation (_core.pyx:707-753, ensure_coords
// :377-420, _resolve_leaf_alloc :248-280).
#pragma once

#include <cub/block/block_scan.cuh>

#include "svx_internal.cuh"

#ifndef SVX_RESOLVE_PREFETCH
#define SVX_RESOLVE_PREFETCH 1
#endif

namespace svx {
namespace rt {

// -DSVX_RESOLVE_TRACE: thread 0 of each K2 CTA stamps the phases of its first
// kTraceSteps steps (%globaltimer) into g_rtrace (read by svx_debug_resolve_trace).
// (only svx_resolve.cu, which defines SVX_RT_TRACE_HOST, holds the buffer)
#if defined(SVX_RESOLVE_TRACE) && defined(SVX_RT_TRACE_HOST)
constexpr int kTraceSteps = 4, kTraceMarks = 6, kTraceCtas = 2048;
__device__ unsigned long long g_rtrace[kTraceCtas][kTraceSteps][kTraceMarks];
#define RT_MARK(i)                                                                         \
    do {                                                                                   \
        if (threadIdx.x == 0 && blockIdx.x < kTraceCtas && tstep < kTraceSteps)              \
            g_rtrace[blockIdx.x][tstep][i] = globaltimer();                                 \
    } while (0)
#else
#define RT_MARK(i) do { } while (0)
#endif

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
__device__ inline int leaf_find_or_insert(int4* table, long long mask, int a, int b, int c, int frame,
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
                // (a plain atomic: this lane may be alone on this path while other
                // lanes of its warp spin on slots it has not published yet)
                const long long id = (long long)atomicAdd(&ctr->nblocks, 1ULL);
                if (id >= bcap) {
                    atomicExch((int*)&table[pos].w, kHashEmpty);
                    atomicOr(&ctr->err_cap, 1);
                    return -1;
                }
                bcoord[id] = make_int4(a, b, c, frame);
                // the leaf's coordinates are visible before its id is published
                // (key and id go out in one 16-byte store: a reader sees the slot
                // BUSY or complete)
                __threadfence();
                st_slot(table + pos, make_int4(a, b, c, (int)id));
                return (int)id;
            }
            v = old;
        }
        int spins = 0;
        while (v == kHashBusy) {
            __nanosleep(20);
            v = *vw;
            SVX_SPIN_GUARD(spins, ctr, 11)
        }
        if (v == kHashBusy) return -1;
        if (v == kHashEmpty) {   // a creator rolled back (pool full)
            atomicOr(&ctr->err_cap, 1);
            return -1;
        }
        const int4 full = ld_slot(table + pos);
        if (full.x == a && full.y == b && full.z == c) return full.w;
        pos = (pos + 1) & mask;
    }
}

// CTA-wide exclusive rank of a predicate (warp ballots + one shared-memory
// round); every thread gets the total.  s_warp holds kThreads/32 counts and
// must not be rewritten before every thread has passed the next barrier.
template <int kThreads>
__device__ __forceinline__ int cta_rank(bool pred, int& total, int* s_warp) {
    constexpr int kWarps = kThreads / 32;
    const unsigned b = __ballot_sync(0xffffffffu, pred);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) s_warp[w] = __popc(b);
    __syncthreads();
    int off = 0, tot = 0;
#pragma unroll
    for (int i = 0; i < kWarps; ++i) {
        const int c = s_warp[i];
        off += i < w ? c : 0;
        tot += c;
    }
    total = tot;
    return off + __popc(b & ((1u << lane) - 1u));
}

struct ResolveArgs {
    int4* table;
    int4* bcoord;
    unsigned long long* bkey;
    unsigned long long* bmask;
    unsigned long long* bslot;   // {vid (low 32), frame row count (high 32, slot mode)}
    VoxFrame* rec;
    int* tlist;                  // segment mode: touched voxel ids
    TouchEntry* tent;            // slot mode: per-CTA touched regions
    unsigned* rcount;            // slot mode: entries per region
    RowSlot* vslot;              // slot mode
    int* rowvid;                 // segment mode
    FrameCtr* ctr;
    KeyPack kp;
    long long hmask, bcap, vcap, nblocks0;
    long long region;            // slot mode: touched entries per CTA region
    // slot mode: the first toucher prefetches the voxel's TSDF pair and its
    // own label's count into L2 for the update kernel (no registers held)
    const char* vt;
    int vt_bytes;                // bytes per voxel in vt
    const char* counts;
    int count_bytes;             // bytes per count
    int ncounts;                 // counts per voxel (C), 0 = none
    int frame;
    bool slots;
};

// One step over kThreads rows (one per thread; every thread of the CTA must
// call it).  `t` is the row's index in the global row arrays (segment mode
// writes rowvid[t]); `rsl` is the row's slot record (slot mode).
// Slot mode: the voxel's bslot word carries its frame row count in the high
// half, so one 64-bit atomicAdd returns both the voxel id and the row's rank
// among the voxel's rows (one dependent round trip instead of a load plus a
// count atomic).  An inactive voxel (-1) is claimed by the row that sees
// count 0; it publishes the new id with an atomicAnd on the low half (which
// was all ones), or -2 when the pool is full; rows that arrive meanwhile wait
// for the publish.  The first toucher lists the voxel in this CTA's touched
// region (shared-memory counter, no global atomic).
template <int kThreads>
__device__ __forceinline__ void resolve_step(const ResolveArgs& ra, bool valid,
                                             unsigned long long key, const RowSlot& rsl,
                                             long long t,
                                             int* s_warp, unsigned long long& s_base,
                                             unsigned& tcount, int tstep = 0) {
    const KeyPack& kp = ra.kp;
    const long long hmask = ra.hmask, bcap = ra.bcap, vcap = ra.vcap, nblocks0 = ra.nblocks0;
    const int frame = ra.frame;
    const bool slots = ra.slots;
    const int lane = threadIdx.x & 31;
    const unsigned full = 0xffffffffu;
    FrameCtr* ctr = ra.ctr;
    int4* table = ra.table;
    int4* bcoord = ra.bcoord;
    unsigned long long* bkey = ra.bkey;
    unsigned long long* bmask = ra.bmask;
    unsigned long long* bslot = ra.bslot;
    VoxFrame* rec = ra.rec;
    int* tlist = ra.tlist;
    RowSlot* vslot = ra.vslot;
    int* rowvid = ra.rowvid;
    // No thread claims a slot in this step while another thread of its CTA
    // may still wait (previous step) on another CTA's claim: that CTA could
    // itself be held at its claim barrier by a thread waiting on ours.
    RT_MARK(0);
    __syncthreads();
    RT_MARK(1);
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
    int rank = 0, cnt = 0;
    // leaf claims are rare: the rank/publish round only runs when this step has any
    const bool lclaims = __syncthreads_or(lstate == 1);
    RT_MARK(2);
    if (lclaims) {
        rank = cta_rank<kThreads>(lstate == 1, cnt, s_warp);
        if (threadIdx.x == 0) s_base = atomicAdd(&ctr->nblocks, (unsigned long long)cnt);
        __syncthreads();
    }
    if (lstate == 1) {
        const long long nid = (long long)s_base + rank;
        if (nid >= bcap) {
            atomicExch(&table[lpos].w, kHashEmpty);
            atomicOr(&ctr->err_cap, 1);
        } else {
            bcoord[nid] = make_int4(la, lb, lc, frame);
            __threadfence();   // coordinates visible before the id (see leaf_find_or_insert)
            st_slot(table + lpos, make_int4(la, lb, lc, (int)nid));   // key + id in one store
            id = (int)nid;
        }
    }
    if (lclaims) __syncthreads();   // this step's claims are published before anyone waits
    if (lstate == 2) {   // another CTA is publishing this slot (maybe another key)
        volatile int* vw = &table[lpos].w;
        int v = *vw;
        int spins = 0;
        while (v == kHashBusy) {
            __nanosleep(32);
            v = *vw;
            SVX_SPIN_GUARD(spins, ctr, 12)
        }
        const int4 sv = ld_slot(table + lpos);
        if (v == kHashBusy) id = -1;
        else if (v >= 0 && sv.x == la && sv.y == lb && sv.z == lc) id = v;
        else id = leaf_find_or_insert(table, hmask, la, lb, lc, frame, bcap, bcoord, ctr);
    }
    id = __shfl_sync(full, id, lleader);

    // ---- voxels: find, or claim an inactive slot; ids for the tile's claims
    int vid = -1, vstate = 0;   // 1 = claimed here, 2 = wait for another claim
    unsigned long long* sp = nullptr;
    unsigned j0 = 0;            // slot mode: rows of this voxel before this warp's
    const int slot = slot_of(x, y, z);   // GridCore.activate_slot, _core.pyx:312-322
    if (is_vl && id >= 0) {
        if (id >= nblocks0) atomicMin(&bkey[id], key);
        sp = &bslot[(long long)id * kLeafVolume + slot];
        if (slots) {
            const unsigned long long old = atomicAdd(sp, (unsigned long long)__popc(vpeers) << 32);
            const int v = (int)(unsigned)old;
            j0 = (unsigned)(old >> 32);
            if (v >= 0) vid = v;
            else if (v == -1 && j0 == 0u) vstate = 1;
            else vstate = 2;
        } else {
            unsigned long long v = __ldcg(sp);
            if (v == kSlotInactive) {
                v = atomicCAS(sp, kSlotInactive, kSlotClaim);
                if (v == kSlotInactive) vstate = 1;
            }
            if (vstate == 0) {
                if ((int)(unsigned)v >= 0) vid = (int)(unsigned)v;
                else vstate = 2;   // another CTA claimed it
            }
        }
    }
    const bool vclaims = __syncthreads_or(vstate == 1);
    RT_MARK(3);
    if (vclaims) {
        rank = cta_rank<kThreads>(vstate == 1, cnt, s_warp);
        if (threadIdx.x == 0) s_base = atomicAdd(&ctr->nvox, (unsigned long long)cnt);
        __syncthreads();
    }
    bool created = false;
    if (vstate == 1) {
        const long long nv = (long long)s_base + rank;
        if (nv >= vcap) {
            if (slots) atomicAnd(sp, 0xFFFFFFFFFFFFFFFEULL);   // low half := -2 (failed)
            else atomicExch(sp, kSlotInactive);
            atomicOr(&ctr->err_cap, 1);
        } else {
            atomicOr(&bmask[(long long)id * kMaskWords + (slot >> 6)], 1ULL << (slot & 63));
            if (slots) atomicAnd(sp, 0xFFFFFFFF00000000ULL | (unsigned long long)(unsigned)nv);
            else atomicExch(sp, (unsigned long long)(unsigned)nv);
            vid = (int)nv;
            created = true;
        }
    }
    if (vclaims) __syncthreads();
    if (vstate == 2) {
        volatile unsigned* vsp = reinterpret_cast<volatile unsigned*>(sp);   // low half
        const int pending = slots ? -1 : -2;
        int v = (int)*vsp;
        int spins = 0;
        while (v == pending) {
            __nanosleep(32);
            v = (int)*vsp;
            SVX_SPIN_GUARD(spins, ctr, 13)
        }
        if (v >= 0) vid = v;
        else atomicOr(&ctr->err_cap, 1);
    }

    // ---- counts; the voxel's first toucher this frame lists it
    bool first = false;
    unsigned cbase = 0;
    if (slots) {
        first = sp != nullptr && j0 == 0u;   // failed claims are listed too (cleanup)
        cbase = j0;
    } else if (is_vl && vid >= 0) {
        const unsigned c = atomicAdd(&rec[vid].cnt, (unsigned)__popc(vpeers) + (created ? kNewBit : 0u));
        cbase = c & ~kNewBit;
        first = cbase == 0u;
    }
    rank = cta_rank<kThreads>(first, cnt, s_warp);
    RT_MARK(4);
    if (slots) {
        if (first) {
            if (SVX_RESOLVE_PREFETCH && vid >= 0) {
                const char* pv = ra.vt + (long long)vid * ra.vt_bytes;
                asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(pv));
                if (ra.ncounts && rsl.label >= 1) {
                    const char* pc = ra.counts + ((long long)vid * ra.ncounts + (rsl.label - 1)) * ra.count_bytes;
                    asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(pc));
                }
            }
            TouchEntry te;
            te.vid = vid >= 0 ? ((unsigned)vid | (created ? kNewBit : 0u)) : 0xFFFFFFFFu;
            te.bidx = (unsigned)(sp - bslot);
            const long long pos = (long long)tcount + rank;
            if (pos < ra.region) ra.tent[(long long)blockIdx.x * ra.region + pos] = te;
            else atomicOr(&ctr->err_cap, 1);   // region sized from the row capacity: cannot happen
        }
        tcount += (unsigned)cnt;   // every thread keeps the same running count
    } else {
        if (threadIdx.x == 0 && cnt) s_base = atomicAdd(&ctr->n_touched, (unsigned long long)cnt);
        __syncthreads();
        if (first) {
            rec[vid].key = key;
            tlist[s_base + rank] = vid;
        }
    }
    vid = __shfl_sync(full, vid, vleader);
    if (slots) {
        // this row's rank among the voxel's rows = its slot (order is
        // restored by point index in k_update_slots)
        cbase = __shfl_sync(full, cbase, vleader) + __popc(vpeers & ((1u << lane) - 1u));
        if (valid && vid >= 0) {
            if (cbase < (unsigned)kSlots) {
                RowSlot* dst = vslot + ((long long)vid * kSlots + cbase) * kSlotStride;
                dst[0] = rsl;
                if (kSlotStride == 2) dst[1] = RowSlot{0, 0, 0.0};
            }
            else ctr->err_slots = 1;
        }
    } else if (valid) {
        rowvid[t] = vid;
    }
    RT_MARK(5);
}

}  // namespace rt

// The map's resolve arguments (pointers; per-frame values are filled on the
// device from FrameParams).  svx_resolve.cu.
rt::ResolveArgs resolve_args(svx_map* m);

}  // namespace svx

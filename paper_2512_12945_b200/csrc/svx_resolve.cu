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
#define SVX_RT_TRACE_HOST 1
#include "svx_resolve_tile.cuh"

namespace svx {
namespace {

constexpr int kResolveThreads = kResolveTile;
#ifndef SVX_ROW_DISCARD
#define SVX_ROW_DISCARD 1
#endif
constexpr int kSegThreads = 256;
constexpr int kSegTile = kSegThreads * 4;
constexpr int kSegBlocks = 148 * 4;

// K2: rows -> voxel ids over CTA-synchronous tiles of 256 rows
// (svx_resolve_tile.cuh).
#ifndef SVX_RESOLVE_MINB
#define SVX_RESOLVE_MINB 6
#endif
__global__ void __launch_bounds__(kResolveThreads, SVX_RESOLVE_MINB) k_resolve(
    const unsigned long long* __restrict__ rowkey, const int* __restrict__ rowray,
    const double* __restrict__ rowd, const int* __restrict__ rowlab, rt::ResolveArgs ra) {
    grid_dep_wait();
    __shared__ int s_warp[kResolveThreads / 32];
    __shared__ unsigned long long s_base;
    FrameCtr* ctr = ra.ctr;
    KSpan _ks(ctr, kSpanResolve);
    __shared__ FrameCtr s_ctr_;
    snapshot_ctr(ctr, s_ctr_);
    const FrameCtr* cv = &s_ctr_;
    unsigned tcount = 0u;   // this CTA's touched entries (same value in every thread)
    if (cv->abort) {
        // (a poisoned frame keeps the failed frame's touched regions for its cleanup)
        if (threadIdx.x == 0 && !cv->poison) ra.rcount[blockIdx.x] = 0u;
        return;
    }
    const FrameParams& fp = cv->p;
    const long long total = (long long)cv->rows;
    ra.kp = fp.kp;
    ra.hmask = fp.hmask;
    ra.bcap = fp.bcap;
    ra.vcap = fp.vcap;
    ra.nblocks0 = fp.nblocks0;
    ra.frame = fp.frame;
    ra.slots = fp.slots != 0;
    ra.region = fp.region;
    __syncthreads();
    int tstep = 0;
    for (long long tile = blockIdx.x; tile * kResolveThreads < total; tile += gridDim.x, ++tstep) {
        const long long t = tile * kResolveThreads + threadIdx.x;
        const bool valid = t < total;
        // row arrays are dead after this read: evict-first
        const unsigned long long key = valid ? __ldcs(rowkey + t) : kKeyEmpty;
        RowSlot rsl{0, 0, 0.0};
        if (valid && ra.slots) {
            rsl.point = __ldcs(rowray + t);
            rsl.label = __ldcs(rowlab + t);
            rsl.d = __ldcs(rowd + t);
        }
        // (each step starts with a barrier: see resolve_step)
        rt::resolve_step<kResolveThreads>(ra, valid, key, rsl, t, s_warp, s_base, tcount, tstep);
#if SVX_ROW_DISCARD
        // slot mode: the tile's rows are dead once every thread used them (the
        // step's barriers): drop their 48 L2 lines without write-back
        if (ra.slots && threadIdx.x < 48) {
            const long long t0 = tile * kResolveThreads;
            const int q = threadIdx.x;
            const char* line = q < 16 ? (const char*)(rowkey + t0) + 128 * q
                             : q < 32 ? (const char*)(rowd + t0) + 128 * (q - 16)
                             : q < 40 ? (const char*)(rowray + t0) + 128 * (q - 32)
                                      : (const char*)(rowlab + t0) + 128 * (q - 40);
            asm volatile("discard.global.L2 [%0], 128;" ::"l"(line) : "memory");
        }
#endif
    }
    if (ra.slots && threadIdx.x == 0) {   // this CTA's touched region
        ra.rcount[blockIdx.x] = tcount;
        if (tcount) atomicAdd(&ctr->n_touched, (unsigned long long)tcount);
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
    KSpan _ks(ctr, kSpanSeg);
    __shared__ FrameCtr s_ctr_;
    snapshot_ctr(ctr, s_ctr_);
    const FrameCtr* cv = &s_ctr_;
    using Scan = cub::BlockScan<unsigned long long, kSegThreads>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ unsigned long long s_prefix;
    __shared__ long long s_tile;
    if (cv->abort | cv->err_cap) return;
    const long long n = (long long)cv->n_touched;
    const int singles = cv->p.inline_singles;
    const unsigned long long seq = cv->p.seq;
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
                int spins = 0;
                while (true) {
                    const long long p = hi - lane;
                    unsigned long long tag = seq << 2 | 2, v = 0;
                    if (p >= 0) ld_status(status + p, tag, v);
                    const unsigned ready = __ballot_sync(0xffffffffu, (tag >> 2) == seq && (tag & 3) != 0);
                    const unsigned incl = __ballot_sync(0xffffffffu, (tag >> 2) == seq && (tag & 3) == 2);
                    // lanes up to the first inclusive one must all be ready
                    const unsigned upto = incl ? (incl & (0u - incl)) * 2u - 1u : 0xffffffffu;
                    if ((ready & upto) != upto) {   // a predecessor not yet published
                        bool stuck = false;
                        if (lane == 0 && ++spins > kSpinLimit) {
                            atomicCAS(&ctr->err_internal, 0ULL, 15ULL);
                            stuck = true;
                        }
                        if (__shfl_sync(0xffffffffu, stuck, 0)) break;
                        continue;
                    }
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
__global__ void k_cleanup(long long n, const int* __restrict__ tlist, VoxFrame* rec, TD* vt,
                          TS* mean, TS* beta, int D, double trunc, double prior_beta) {
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

// Slot mode: reset every listed voxel's bslot word (frame count 0; a failed
// claim back to inactive) and give voxels created by the attempt their
// background TSDF state (slot mode is closed/geometry: counts are untouched).
template <class TD>
__global__ void k_cleanup_slots(const TouchEntry* __restrict__ tent, const unsigned* __restrict__ rcount,
                                long long region, unsigned long long* bslot, TD* vt, double trunc) {
    const unsigned cnt = rcount[blockIdx.x];
    const TouchEntry* te = tent + (long long)blockIdx.x * region;
    for (unsigned e = threadIdx.x; e < cnt; e += blockDim.x) {
        const TouchEntry en = te[e];
        if (en.vid == 0xFFFFFFFFu) {
            bslot[en.bidx] = kSlotInactive;
            continue;
        }
        const unsigned vid = en.vid & ~kNewBit;
        bslot[en.bidx] = (unsigned long long)vid;
        if (en.vid & kNewBit) {
            vt[2 * (long long)vid] = (TD)trunc;
            vt[2 * (long long)vid + 1] = (TD)0;
        }
    }
}

template <class TD, class TS>
svx_status cleanup_t(svx_map* m, cudaStream_t s) {
    if (m->frame_leaf) return launch_leaf_cleanup(m, s);   // no voxel changed
    if (m->frame_slots) {
        k_cleanup_slots<TD><<<kPersistentBlocks, 256, 0, s>>>(
            ptr<TouchEntry>(m->tlist), ptr<unsigned>(m->rcount), slot_region(m->rcap),
            ptr<unsigned long long>(m->bslot), ptr<TD>(m->vt), m->cfg.truncation);
        SVX_LAUNCHED();
        return SVX_OK;
    }
    const bool open = m->cfg.sem_kind == SVX_SEM_OPEN;
    k_cleanup<TD, TS><<<kPersistentBlocks, 256, 0, s>>>(
        (long long)m->h_ctr->n_touched, ptr<int>(m->tlist), ptr<VoxFrame>(m->vrec), ptr<TD>(m->vt),
        open ? ptr<TS>(m->s0) : nullptr, open ? ptr<TS>(m->s1) : nullptr, m->payload_d,
        m->cfg.truncation, m->cfg.prior_beta);
    SVX_LAUNCHED();
    return SVX_OK;
}

}  // namespace

#ifdef SVX_RESOLVE_TRACE
// Debug build only: the last K2's per-CTA step stamps (kTraceCtas x
// kTraceSteps x kTraceMarks u64, zero where no step ran).
extern "C" int svx_debug_resolve_trace(unsigned long long* out, long long n) {
    const long long cap = (long long)sizeof(rt::g_rtrace) / 8;
    if (!out) return (int)cap;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, rt::g_rtrace, (size_t)(n < cap ? n : cap) * 8);
    void* p = nullptr;
    cudaGetSymbolAddress(&p, rt::g_rtrace);
    cudaMemset(p, 0, sizeof(rt::g_rtrace));
    cudaDeviceSynchronize();
    return (int)cap;
}
#endif

rt::ResolveArgs resolve_args(svx_map* m) {
    rt::ResolveArgs ra{};
    ra.table = ptr<int4>(m->hash);
    ra.bcoord = ptr<int4>(m->bcoord);
    ra.bkey = ptr<unsigned long long>(m->bkey);
    ra.bmask = ptr<unsigned long long>(m->bmask);
    ra.bslot = ptr<unsigned long long>(m->bslot);
    ra.rec = ptr<VoxFrame>(m->vrec);
    ra.tlist = ptr<int>(m->tlist);
    ra.tent = ptr<TouchEntry>(m->tlist);   // slot mode reuses the touched-list buffer
    ra.rcount = ptr<unsigned>(m->rcount);
    ra.vslot = ptr<RowSlot>(m->vslot);
    ra.rowvid = ptr<int>(m->rowvid);
    ra.ctr = ptr<FrameCtr>(m->ctr);
    ra.vt = ptr<const char>(m->vt);
    ra.vt_bytes = (int)(2 * tsdf_elem(m));
    ra.counts = m->cfg.sem_kind == SVX_SEM_CLOSED ? ptr<const char>(m->s0) : nullptr;
    ra.count_bytes = (int)sem_elem(m);
    ra.ncounts = m->cfg.sem_kind == SVX_SEM_CLOSED ? m->payload_d : 0;
    return ra;
}

svx_status launch_resolve(svx_map* m, cudaStream_t s) {
    SVX_CUDA(launch_pdl(k_resolve, kPersistentBlocks, kResolveThreads, 0, s,
        ptr<unsigned long long>(m->rowkey), ptr<int>(m->rowray), ptr<double>(m->rowd),
        ptr<int>(m->rowlab), resolve_args(m)));
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

// svx_update.cu -- K4 scatter (+ single-row voxel updates) and K5 the fused
// TSDF + semantic update of the voxels with several rows.
//
// Compiled with -fmad=false.  Every voxel's rows are reduced in ascending
// point order -- the reference's (voxel, point, step) order, since a ray
// visits a voxel at most once -- with sequential fp64 sums exactly like
// _core.pyx:759-843; the apply arithmetic restates apply_tsdf /
// apply_closed / apply_open (_pycore.py:399-446) operation for operation,
// so stored values round identically.
//
// Execution shapes by rows per voxel:
//   1      (closed/geometry)  finished by the scatter thread, in ray order
//   <= 16                      one thread per voxel, register insertion sort
//   <= 1024                    one warp per voxel, shared-memory bitonic sort
//   larger                     one warp per voxel, point-index bitmap in global
//                              scratch streamed in ascending chunks (space
//                              carving sends every ray through the origin voxel)
// Open-set voxels always take the warp shapes (lanes own feature dims).
#include <math.h>

#include <algorithm>

#include <cub/block/block_scan.cuh>
#include <cuda_pipeline.h>

#include "svx_internal.cuh"

namespace svx {
namespace {

constexpr int kSmemMax = 1024;                   // rows per warp buffer (4 KB)
constexpr int kWarpsPerCta = 8;
#ifndef SVX_DYN_LONG
#define SVX_DYN_LONG 1   // K5 long / open: warps take voxels from a frame counter
#endif
constexpr int kHugeWarps = 296;                  // bitmap scratch slots (huge segments)

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

// Clamped projective distance and weight of one row (row_distances_weights,
// _pycore.py:384-396; identical to _core.pyx:553-566).
__device__ __forceinline__ void row_dw(double cxv, double cyv, double czv, double4 r, double trunc,
                                       int wfn, double& d, double& w) {
    double proj = cxv * r.x + cyv * r.y + czv * r.z;
    d = r.w - proj;
    if (d < -trunc) d = -trunc;
    if (d > trunc) d = trunc;
    w = (wfn == 1) ? (d >= 0.0 ? 1.0 : (trunc + d) / trunc) : 1.0;
}

template <class TD>
__device__ __forceinline__ bool equals_stored(TD stored, double v) {
    return stored == (TD)v;
}

// apply_tsdf (_pycore.py:399-417) for one voxel; vt holds {d, w} pairs.
// Returns w_old.
template <class TD>
__device__ __forceinline__ double apply_tsdf(TD* vt, int vid, bool isnew, double trunc, double sw,
                                             double swd, double mind, double maxd) {
    using P2 = typename Pair<TD>::type;
    P2* slot = reinterpret_cast<P2*>(vt) + vid;
    P2 st;
    if (isnew) {
        st.x = (TD)trunc;
        st.y = (TD)0;
    } else {
        st = *slot;
    }
    double w_old = (double)st.y;
    double d_old = (double)st.x;
    double w_new = w_old + sw;
    double d_new = w_new > 0.0 ? (w_old * d_old + swd) / w_new : d_old;
    bool cst = (mind == maxd) && (w_old == 0.0 || equals_stored<TD>(st.x, mind));
    if (cst) d_new = mind;
    P2 out;
    out.x = (TD)d_new;
    out.y = (TD)w_new;
    *slot = out;
    return w_old;
}

struct Center {
    double x, y, z;
};

__device__ __forceinline__ Center center_of(unsigned long long key, const KeyPack& kp, double h,
                                            const PoseParams& pp) {
    long long x, y, z;
    unpack_key(key, kp, x, y, z);
    Center c;
    c.x = ((double)x + 0.5) * h - pp.t[0];
    c.y = ((double)y + 0.5) * h - pp.t[1];
    c.z = ((double)z + 0.5) * h - pp.t[2];
    return c;
}

struct UpdateArgs {
    const int* mlist;
    VoxFrame* rec;
    const int* srid;
    const double4* ray;
    int* longlist;
    int* hugelist;
    TouchEntry* hugelist2;   // slot mode: voxels of 5..16 rows
    unsigned* bitmap;     // kHugeWarps * bm_words
    long long bm_words;
    double h, trunc;
    int wfn;
    int sem_kind, last_wins, C;   // closed
    int D;                        // open
    double lambda_floor, prior_beta;
    FrameCtr* ctr;
};

__device__ __forceinline__ void clear_voxel_frame(const UpdateArgs& a, int vid) {
    a.rec[vid].cnt = 0u;
    a.rec[vid].cur = 0u;
}

// ---- K4: scatter, single-row voxels finished in ray order --------------------------
#ifndef SVX_SCATTER_AGG
#define SVX_SCATTER_AGG 1   // warp-aggregated segment cursors
#endif
// One thread per row.  A voxel with exactly one row needs no ordering: its
// sums are the row's own (0.0 + w * d exactly as the reference's sequential
// sum, _core.pyx:793-795), so closed/geometry maps update it right here;
// rows of other voxels go to their voxel's segment.
template <class TD, class TC>
#if defined(SVX_SCATTER_MINB)
#define SVX_LB_SCATTER __launch_bounds__(256, SVX_SCATTER_MINB)
#else
#define SVX_LB_SCATTER __launch_bounds__(256)
#endif
__global__ void SVX_LB_SCATTER k_scatter(UpdateArgs a, const int* __restrict__ rcnt,
                                                 const int* __restrict__ rowray,
                                                 const unsigned long long* __restrict__ rowkey,
                                                 const int* __restrict__ rowvid,
                                                 int* __restrict__ srid, TD* vt, TC* counts) {
    grid_dep_wait();
    FrameCtr* ctr = a.ctr;
    KSpan _ks(ctr, kSpanScatter);
    __shared__ FrameCtr s_ctr_;
    snapshot_ctr(ctr, s_ctr_);
    const FrameCtr* cv = &s_ctr_;
    if (cv->abort | cv->err_cap) return;
    const FrameParams& fp = cv->p;
    RowSpace rs;
    rs.maxrows = 0;   // rows are dense in every mode
    rs.rcnt = rcnt;
    rs.rowray = rowray;
    rs.total = (long long)cv->rows;
    const KeyPack kp = fp.kp;
    const PoseParams pp = fp.pp;
    const int32_t* __restrict__ labels = fp.labels;
    const bool singles = fp.inline_singles;
    const bool closed = a.sem_kind == SVX_SEM_CLOSED;
    const bool open_set = a.sem_kind == SVX_SEM_OPEN;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < rs.total;
         t += (long long)gridDim.x * blockDim.x) {
        long long i;
        if (!row_ray(rs, t, i)) continue;
        const int vid = rowvid[t];
        const unsigned c = a.rec[vid].cnt;
        if (!singles || (c & ~kNewBit) > 1u) {
#if SVX_SCATTER_AGG
            // open-set maps: lanes here with the same voxel take consecutive
            // places with one atomic (neighbouring rays share voxels; a camera
            // close to a wall sends ~10^4 rows into each of a few voxels): the
            // segment's order is irrelevant, the update sorts it by point index.
            // (Closed-set depth frames measured 1 us/frame slower with it.)
            if (!open_set) {
                const unsigned pos = a.rec[vid].seg + atomicAdd(&a.rec[vid].cur, 1u);
                srid[pos] = (int)i;
                continue;
            }
            const unsigned act = __activemask();
            const unsigned peers = __match_any_sync(act, vid);
            const int lane = threadIdx.x & 31;
            const int leader = __ffs(peers) - 1;
            unsigned off = 0u;
            if (lane == leader) off = atomicAdd(&a.rec[vid].cur, (unsigned)__popc(peers));
            off = __shfl_sync(peers, off, leader) + (unsigned)__popc(peers & ((1u << lane) - 1u));
            srid[a.rec[vid].seg + off] = (int)i;
#else
            const unsigned pos = a.rec[vid].seg + atomicAdd(&a.rec[vid].cur, 1u);
            srid[pos] = (int)i;
#endif
            continue;
        }
        const unsigned long long key = rowkey[t];
        const double4 ry = a.ray[i];
        const Center cc = center_of(key, kp, a.h, pp);
        double d, w;
        row_dw(cc.x, cc.y, cc.z, ry, a.trunc, a.wfn, d, w);
        apply_tsdf<TD>(vt, vid, (c & kNewBit) != 0u, a.trunc, 0.0 + w, 0.0 + w * d, d, d);
        if (closed) {
            const int lab = labels[i];
            TC* crow = counts + (long long)vid * a.C;
            if (a.last_wins) {
                for (int q = 0; q < a.C; ++q) crow[q] = (TC)(q == lab - 1 ? 1 : 0);
            } else {
                atomicAdd(&crow[lab - 1], (TC)1);   // integer count: fire-and-forget
            }
        }
        a.rec[vid].cnt = 0u;
    }
}

// ---- K5 short: one thread per multi-row voxel (closed / geometry) ----------------

template <class TD, class TC>
#if defined(SVX_SHORT_MINB)
#define SVX_LB_SHORT __launch_bounds__(256, SVX_SHORT_MINB)
#else
#define SVX_LB_SHORT __launch_bounds__(256)
#endif
__global__ void SVX_LB_SHORT k_update_short(UpdateArgs a, TD* vt, TC* counts) {
    grid_dep_wait();
    FrameCtr* ctr = a.ctr;
    KSpan _ks(ctr, kSpanUpdate);
    __shared__ FrameCtr s_ctr_;
    snapshot_ctr(ctr, s_ctr_);
    const FrameCtr* cv = &s_ctr_;
    if (cv->abort | cv->err_cap) return;
    const long long L = (long long)cv->n_list;
    const KeyPack kp = cv->p.kp;
    const PoseParams pp = cv->p.pp;
    const int32_t* __restrict__ labels = cv->p.labels;
    const bool closed = a.sem_kind == SVX_SEM_CLOSED;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < L;
         e += (long long)gridDim.x * blockDim.x) {
        const int vid = a.mlist[e];
        const unsigned c = a.rec[vid].cnt;
        const unsigned k = c & ~kNewBit;
        if (k > (unsigned)kShortMax) {
            if (k > (unsigned)kSmemMax) a.hugelist[warp_ticket(&ctr->n_huge)] = (int)e;
            else a.longlist[warp_ticket(&ctr->n_long)] = (int)e;
            continue;
        }
        const unsigned base = a.rec[vid].seg;
        int r[kShortMax];
        for (unsigned j = 0; j < k; ++j) {
            int v = a.srid[base + j];
            int p = (int)j;
            while (p > 0 && r[p - 1] > v) {
                r[p] = r[p - 1];
                --p;
            }
            r[p] = v;
        }
        const Center cc = center_of(a.rec[vid].key, kp, a.h, pp);
        double sw = 0.0, swd = 0.0, mind = INFINITY, maxd = -INFINITY;
        int last_lab = 0;
        TC* crow = counts + (long long)vid * a.C;
        for (unsigned j = 0; j < k; ++j) {
            const int rid = r[j];
            double d, w;
            row_dw(cc.x, cc.y, cc.z, a.ray[rid], a.trunc, a.wfn, d, w);
            sw += w;
            swd += w * d;
            mind = d < mind ? d : mind;
            maxd = d > maxd ? d : maxd;
            if (closed) {
                const int lab = labels[rid];
                if (a.last_wins) last_lab = lab;
                else atomicAdd(&crow[lab - 1], (TC)1);
            }
        }
        apply_tsdf<TD>(vt, vid, (c & kNewBit) != 0u, a.trunc, sw, swd, mind, maxd);
        if (closed && a.last_wins) {
            for (int q = 0; q < a.C; ++q) crow[q] = (TC)(q == last_lab - 1 ? 1 : 0);
        }
        clear_voxel_frame(a, vid);
    }
}

// ---- K5 slot mode: one thread per touched voxel (closed / geometry) --------------
// Each voxel's rows sit in its slots as {point, label, d} (d computed by the
// walk), so a voxel needs its count, its TSDF pair and its slots -- three
// independent loads, no gathers.  Rows are folded in ascending point order
// (the reference's (voxel, point) order) with the sequential sums of
// k_update_short; two rows need no sort for the sums (IEEE addition is
// commutative) but are ordered anyway for last-wins.

struct RowAcc {
    double sw = 0.0, swd = 0.0, mind = INFINITY, maxd = -INFINITY;
    int last = 0;
};

template <class TC>
__device__ __forceinline__ void fold_row(const UpdateArgs& a, double d, int lab, TC* crow,
                                         bool closed, RowAcc& acc) {
    // weight of row_dw (_pycore.py:384-396) from the stored clamped distance
    const double w = (a.wfn == 1) ? (d >= 0.0 ? 1.0 : (a.trunc + d) / a.trunc) : 1.0;
    acc.sw += w;
    acc.swd += w * d;
    acc.mind = d < acc.mind ? d : acc.mind;
    acc.maxd = d > acc.maxd ? d : acc.maxd;
    if (closed) {
        if (a.last_wins) acc.last = lab;
        else atomicAdd(&crow[lab - 1], (TC)1);   // integer count: order-free
    }
}

__device__ __forceinline__ RowSlot ld_slot16(const RowSlot* p) {
    const int4 v = __ldcs(reinterpret_cast<const int4*>(p));   // dead after this frame: evict-first
    RowSlot r;
    r.point = v.x;
    r.label = v.y;
    r.d = __hiloint2double(v.w, v.z);
    return r;
}

// The first two slots of a voxel share one 32-byte sector: loaded together,
// issued before the voxel's row count is known (asm volatile keeps the load
// where it is written, next to the count and TSDF loads it overlaps).
__device__ __forceinline__ void ld_slot_pair(const RowSlot* p, RowSlot& a, RowSlot& b) {
    int x0, y0, z0, w0, x1, y1, z1, w1;
    asm volatile("ld.global.cs.v4.s32 {%0, %1, %2, %3}, [%8];\n\t"
                 "ld.global.cs.v4.s32 {%4, %5, %6, %7}, [%8+16];"
                 : "=r"(x0), "=r"(y0), "=r"(z0), "=r"(w0), "=r"(x1), "=r"(y1), "=r"(z1), "=r"(w1)
                 : "l"(p));
    a.point = x0;
    a.label = y0;
    a.d = __hiloint2double(w0, z0);
    b.point = x1;
    b.label = y1;
    b.d = __hiloint2double(w1, z1);
}

// 9..16 rows in-thread: 16 (point << 4 | slot) keys through a bitonic
// network in registers, then the rows in that order.
template <class TC>
__device__ __forceinline__ void sorted_fold16(const UpdateArgs& a, const RowSlot* sl, unsigned k,
                                              TC* crow, bool closed, RowAcc& acc) {
    unsigned long long key[16];
#pragma unroll
    for (int j = 0; j < 16; ++j)
        key[j] = (unsigned)j < k ? (((unsigned long long)(unsigned)sl[j * kSlotStride].point << 4) | (unsigned)j)
                                 : ~0ULL;
#pragma unroll
    for (int kk = 2; kk <= 16; kk <<= 1) {
#pragma unroll
        for (int jj = kk >> 1; jj > 0; jj >>= 1) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int l = i ^ jj;
                if (l > i) {
                    const unsigned long long x = key[i], y = key[l];
                    const bool up = (i & kk) == 0;
                    key[i] = up ? (x < y ? x : y) : (x > y ? x : y);
                    key[l] = up ? (x > y ? x : y) : (x < y ? x : y);
                }
            }
        }
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        if ((unsigned)j < k) {
            const RowSlot r = ld_slot16(sl + (int)(key[j] & 15u) * kSlotStride);
            fold_row<TC>(a, r.d, r.label, crow, closed, acc);
        }
    }
}

#ifndef SVX_UPD_MINB
#define SVX_UPD_MINB 3
#endif
#ifndef SVX_SLOT_PAIR
#define SVX_SLOT_PAIR 1
#endif
#ifndef SVX_SLOT_DISCARD
#define SVX_SLOT_DISCARD 1
#endif
template <class TD, class TC, bool kInlineLong>
__device__ __forceinline__ void k_update_slots_body(UpdateArgs a, const TouchEntry* __restrict__ tent,
                                                      const unsigned* __restrict__ rcount,
                                                      unsigned long long* __restrict__ bslot,
                                                      const RowSlot* __restrict__ vslot, TD* vt,
                                                      TC* counts) {
    grid_dep_wait();
    FrameCtr* ctr = a.ctr;
    KSpan _ks(ctr, kSpanUpdate);
    __shared__ FrameCtr s_ctr_;
    snapshot_ctr(ctr, s_ctr_);
    const FrameCtr* cv = &s_ctr_;
    if (cv->abort | cv->err_cap | cv->err_slots) return;
    const bool closed = a.sem_kind == SVX_SEM_CLOSED;
    const long long region = cv->p.region;
    using P2 = typename Pair<TD>::type;
    // K2 CTA b listed its touched voxels in region b; this grid has the same size
    const unsigned cnt = rcount[blockIdx.x];
    const TouchEntry* te = tent + (long long)blockIdx.x * region;
    for (unsigned e = threadIdx.x; e < cnt; e += blockDim.x) {
        const unsigned long long raw = __ldcs(reinterpret_cast<const unsigned long long*>(te + e));
        TouchEntry en;
        en.vid = (unsigned)raw;
        en.bidx = (unsigned)(raw >> 32);
        const int vid = (int)(en.vid & ~kNewBit);
        const unsigned c = (unsigned)(bslot[en.bidx] >> 32) | (en.vid & kNewBit);
        P2 st = reinterpret_cast<const P2*>(vt)[vid];
        const RowSlot* sl = vslot + (long long)vid * kSlots * kSlotStride;
#if SVX_SLOT_PAIR
        RowSlot p0, p1;
        ld_slot_pair(sl, p0, p1);   // overlaps the count load: most voxels have 1-2 rows
#endif
        const unsigned k = c & ~kNewBit;
        if (!kInlineLong && k > 8u) {   // 9..16 rows (rare): one warp per voxel in k_update_slots_long
            a.hugelist2[warp_ticket(&ctr->n_long)] = en;
            continue;
        }
        TC* crow = counts + (long long)vid * a.C;
        RowAcc acc;
        if (kInlineLong && k > 8u) {
            sorted_fold16<TC>(a, sl, k, crow, closed, acc);
        } else if (k > 4u) {
            // 5..8 rows: sort (point, slot) keys in registers, then fold the rows
            // in that order (their slots were just read: L1/L2 hits)
            unsigned long long key[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
                key[j] = (unsigned)j < k ? (((unsigned long long)(unsigned)sl[j * kSlotStride].point << 3) | (unsigned)j)
                                         : ~0ULL;
#pragma unroll
            for (int kk = 2; kk <= 8; kk <<= 1) {
#pragma unroll
                for (int jj = kk >> 1; jj > 0; jj >>= 1) {
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int l = i ^ jj;
                        if (l > i) {
                            const unsigned long long x = key[i], y = key[l];
                            const bool up = (i & kk) == 0;
                            key[i] = up ? (x < y ? x : y) : (x > y ? x : y);
                            key[l] = up ? (x > y ? x : y) : (x < y ? x : y);
                        }
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if ((unsigned)j < k) {
                    const RowSlot r = ld_slot16(sl + (int)(key[j] & 7u) * kSlotStride);
                    fold_row<TC>(a, r.d, r.label, crow, closed, acc);
                }
            }
        } else {
        // rows in registers; only slots that exist are read (no partial-sector reads)
#if SVX_SLOT_PAIR
        RowSlot q0 = p0, q1 = p1, q2, q3;
        q2.point = q3.point = 0x7fffffff;
        if (k <= 1u) q1.point = 0x7fffffff;
#else
        RowSlot q0 = ld_slot16(sl), q1, q2, q3;
        q1.point = q2.point = q3.point = 0x7fffffff;
        if (k > 1u) q1 = ld_slot16(sl + 1 * kSlotStride);
#endif
        if (k > 2u) q2 = ld_slot16(sl + 2 * kSlotStride);
        if (k > 3u) q3 = ld_slot16(sl + 3 * kSlotStride);
        // 4-element sorting network on the point index (5 compare-exchanges)
        auto cx = [](RowSlot& x, RowSlot& y) {
            if (y.point < x.point) {
                const RowSlot t = x;
                x = y;
                y = t;
            }
        };
        cx(q0, q1);
        cx(q2, q3);
        cx(q0, q2);
        cx(q1, q3);
        cx(q1, q2);
        fold_row<TC>(a, q0.d, q0.label, crow, closed, acc);
        if (k > 1u) fold_row<TC>(a, q1.d, q1.label, crow, closed, acc);
        if (k > 2u) fold_row<TC>(a, q2.d, q2.label, crow, closed, acc);
        if (k > 3u) fold_row<TC>(a, q3.d, q3.label, crow, closed, acc);
        }
        // apply_tsdf (_pycore.py:399-417) on the pre-loaded pair
        if (c & kNewBit) {
            st.x = (TD)a.trunc;
            st.y = (TD)0;
        }
        const double w_old = (double)st.y, d_old = (double)st.x;
        const double w_new = w_old + acc.sw;
        double d_new = w_new > 0.0 ? (w_old * d_old + acc.swd) / w_new : d_old;
        if ((acc.mind == acc.maxd) && (w_old == 0.0 || equals_stored<TD>(st.x, acc.mind)))
            d_new = acc.mind;
        P2 out;
        out.x = (TD)d_new;
        out.y = (TD)w_new;
        reinterpret_cast<P2*>(vt)[vid] = out;
        if (closed && a.last_wins)
            for (int t = 0; t < a.C; ++t) crow[t] = (TC)(t == acc.last - 1 ? 1 : 0);
        bslot[en.bidx] = (unsigned long long)(unsigned)vid;   // frame count back to 0
#if SVX_SLOT_DISCARD
        // the voxel's row slots are dead until K2 of a later frame rewrites them:
        // drop their L2 lines without writing them back (k <= 8 here: one line)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(sl) : "memory");
#endif
    }
}

template <class TD, class TC, bool kInlineLong>
__global__ void __launch_bounds__(256, SVX_UPD_MINB) k_update_slots(UpdateArgs a, const TouchEntry* __restrict__ tent,
                                                                  const unsigned* __restrict__ rcount,
                                                                  unsigned long long* __restrict__ bslot,
                                                                  const RowSlot* __restrict__ vslot, TD* vt,
                                                                  TC* counts) {
    k_update_slots_body<TD, TC, kInlineLong>(a, tent, rcount, bslot, vslot, vt, counts);
    if (kInlineLong) frame_epilogue(a.ctr, a.ctr->p.epilogue, a.ctr->p.mirror);
}

// Slot-mode voxels of 9..16 rows: one warp per voxel; lanes own rows, a
// shuffle bitonic sort on (point, lane) orders them, the sums run in that
// order through shuffles.
template <class TD, class TC>
__device__ __forceinline__ void k_update_slots_long_body(UpdateArgs a,
                                                           unsigned long long* __restrict__ bslot,
                                                           const RowSlot* __restrict__ vslot, TD* vt,
                                                           TC* counts) {
    grid_dep_wait();
    FrameCtr* ctr = a.ctr;
    KSpan _ks(ctr, kSpanUpdateB);
    __shared__ FrameCtr s_ctr_;
    snapshot_ctr(ctr, s_ctr_);
    const FrameCtr* cv = &s_ctr_;
    if (cv->abort | cv->err_cap | cv->err_slots) return;
    const bool closed = a.sem_kind == SVX_SEM_CLOSED;
    const int lane = threadIdx.x & 31;
    using P2 = typename Pair<TD>::type;
    const long long L = (long long)cv->n_long;
    for (long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < L;
         w += ((long long)gridDim.x * blockDim.x) >> 5) {
        const TouchEntry en = a.hugelist2[w];
        const int vid = (int)(en.vid & ~kNewBit);
        const unsigned k = (unsigned)(bslot[en.bidx] >> 32);
        RowSlot r{0x7fffffff, 0, 0.0};
        if ((unsigned)lane < k) r = ld_slot16(vslot + ((long long)vid * kSlots + lane) * kSlotStride);
        unsigned long long key = ((unsigned long long)(unsigned)r.point << 32) | (unsigned)lane;
#pragma unroll
        for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
            for (int jj = kk >> 1; jj > 0; jj >>= 1) {
                const unsigned long long o = __shfl_xor_sync(0xffffffffu, key, jj);
                const bool up = (lane & kk) == 0;
                const bool lower = (lane & jj) == 0;
                key = (lower == up) ? (key < o ? key : o) : (key > o ? key : o);
            }
        }
        const int src = (int)(key & 31u);   // lane holding the lane-th smallest row
        const double d = __shfl_sync(0xffffffffu, r.d, src);
        const int lab = __shfl_sync(0xffffffffu, r.label, src);
        const double w_row = (a.wfn == 1) ? (d >= 0.0 ? 1.0 : (a.trunc + d) / a.trunc) : 1.0;
        RowAcc acc;
        for (unsigned q = 0; q < k; ++q) {
            const double wq = __shfl_sync(0xffffffffu, w_row, q);
            const double dq = __shfl_sync(0xffffffffu, d, q);
            acc.sw += wq;
            acc.swd += wq * dq;
            acc.mind = dq < acc.mind ? dq : acc.mind;
            acc.maxd = dq > acc.maxd ? dq : acc.maxd;
        }
        TC* crow = counts + (long long)vid * a.C;
        if (closed && !a.last_wins && (unsigned)lane < k) atomicAdd(&crow[lab - 1], (TC)1);
        const int last = __shfl_sync(0xffffffffu, lab, k - 1);
        if (lane == 0) {
            P2 st = reinterpret_cast<const P2*>(vt)[vid];
            if (en.vid & kNewBit) {
                st.x = (TD)a.trunc;
                st.y = (TD)0;
            }
            const double w_old = (double)st.y, d_old = (double)st.x;
            const double w_new = w_old + acc.sw;
            double d_new = w_new > 0.0 ? (w_old * d_old + acc.swd) / w_new : d_old;
            if ((acc.mind == acc.maxd) && (w_old == 0.0 || equals_stored<TD>(st.x, acc.mind)))
                d_new = acc.mind;
            P2 out;
            out.x = (TD)d_new;
            out.y = (TD)w_new;
            reinterpret_cast<P2*>(vt)[vid] = out;
            bslot[en.bidx] = (unsigned long long)(unsigned)vid;
        }
        if (closed && a.last_wins)
            for (int t = lane; t < a.C; t += 32) crow[t] = (TC)(t == last - 1 ? 1 : 0);
    }
}

template <class TD, class TC>
__global__ void __launch_bounds__(256) k_update_slots_long(UpdateArgs a, unsigned long long* __restrict__ bslot, const RowSlot* __restrict__ vslot, TD* vt, TC* counts) {
    k_update_slots_long_body(a, bslot, vslot, vt, counts);
    frame_epilogue(a.ctr, a.ctr->p.epilogue, a.ctr->p.mirror);
}

// ---- warp helpers ---------------------------------------------------------------

// Sort one segment's point indices ascending into buf (k <= kSmemMax).
__device__ __forceinline__ void warp_sort_segment(const int* __restrict__ srid, unsigned base, int k,
                                                  int* buf) {
    const int lane = threadIdx.x & 31;
    if (k <= 32) {
        // one element per lane: bitonic sort through shuffles
        int v = lane < k ? srid[base + lane] : 0x7fffffff;
        for (int kk = 2; kk <= 32; kk <<= 1) {
            for (int jj = kk >> 1; jj > 0; jj >>= 1) {
                int o = __shfl_xor_sync(0xffffffffu, v, jj);
                bool up = (lane & kk) == 0;
                bool lower = (lane & jj) == 0;
                v = (lower == up) ? min(v, o) : max(v, o);
            }
        }
        buf[lane] = v;
        __syncwarp();
        return;
    }
    int P = 64;
    while (P < k) P <<= 1;
    for (int j = lane; j < P; j += 32) buf[j] = j < k ? srid[base + j] : 0x7fffffff;
    __syncwarp();
    for (int kk = 2; kk <= P; kk <<= 1) {
        for (int jj = kk >> 1; jj > 0; jj >>= 1) {
            for (int i = lane; i < P; i += 32) {
                const int ixj = i ^ jj;
                if (ixj > i) {
                    const int x = buf[i], y = buf[ixj];
                    const bool up = (i & kk) == 0;
                    if ((x > y) == up) {
                        buf[i] = y;
                        buf[ixj] = x;
                    }
                }
            }
            __syncwarp();
        }
    }
}

// Next ascending chunk (<= 1024 rows) of a huge segment from its point bitmap.
__device__ __forceinline__ int bitmap_chunk(const unsigned* bm, long long w0, long long nwords,
                                            int minr, int* buf) {
    const int lane = threadIdx.x & 31;
    const long long w = w0 + lane;
    unsigned bits = w < nwords ? __ldcg(bm + w) : 0u;
    int cnt = __popc(bits);
    int incl = cnt;
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    int pos = incl - cnt;
    while (bits) {
        int b = __ffs(bits) - 1;
        bits &= bits - 1;
        buf[pos++] = minr + (int)(w * 32 + b);
    }
    int total = __shfl_sync(0xffffffffu, incl, 31);
    __syncwarp();
    return total;
}

// Build the point bitmap of a huge segment in this warp's scratch.
__device__ __forceinline__ void bitmap_build(const int* __restrict__ srid, unsigned base, unsigned k,
                                             unsigned* bm, int& minr, long long& nwords) {
    const int lane = threadIdx.x & 31;
    int mn = 0x7fffffff, mx = -1;
    for (unsigned j = lane; j < k; j += 32) {
        int v = srid[base + j];
        mn = min(mn, v);
        mx = max(mx, v);
    }
    for (int o = 16; o > 0; o >>= 1) {
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    minr = mn;
    nwords = ((long long)(mx - mn) >> 5) + 1;
    for (long long w = lane; w < nwords; w += 32) bm[w] = 0u;
    __threadfence();
    __syncwarp();
    for (unsigned j = lane; j < k; j += 32) {
        int v = srid[base + j] - mn;
        atomicOr(&bm[v >> 5], 1u << (v & 31));
    }
    __threadfence();
    __syncwarp();
}

struct TsdfAcc {
    double sw, swd, mind, maxd;
    int last_lab;
};

// Fold an ordered chunk of rows into the TSDF sums (all lanes end with the
// same sums); closed-set counts are integer increments (order-free).
template <class TC>
__device__ __forceinline__ void warp_tsdf_chunk(const UpdateArgs& a, const int32_t* labels,
                                                const int* buf, int cnt, const Center& c,
                                                TsdfAcc& acc, TC* crow, bool count_labels) {
    const int lane = threadIdx.x & 31;
    for (int c0 = 0; c0 < cnt; c0 += 32) {
        const int j = c0 + lane;
        double d = 0.0, w = 0.0;
        int lab = 0;
        if (j < cnt) {
            const int rid = buf[j];
            row_dw(c.x, c.y, c.z, a.ray[rid], a.trunc, a.wfn, d, w);
            if (count_labels) {
                lab = labels[rid];
                if (!a.last_wins) atomicAdd(&crow[lab - 1], (TC)1);
            }
        }
        const int nv = min(32, cnt - c0);
        for (int q = 0; q < nv; ++q) {
            const double wq = __shfl_sync(0xffffffffu, w, q);
            const double dq = __shfl_sync(0xffffffffu, d, q);
            acc.sw += wq;
            acc.swd += wq * dq;
            acc.mind = dq < acc.mind ? dq : acc.mind;
            acc.maxd = dq > acc.maxd ? dq : acc.maxd;
        }
        if (count_labels) acc.last_lab = __shfl_sync(0xffffffffu, lab, nv - 1);
    }
}

template <class TD, class TC>
__device__ __forceinline__ void finish_closed(const UpdateArgs& a, TD* vt, TC* crow, int vid,
                                              bool isnew, const TsdfAcc& acc) {
    const int lane = threadIdx.x & 31;
    if (lane == 0) apply_tsdf<TD>(vt, vid, isnew, a.trunc, acc.sw, acc.swd, acc.mind, acc.maxd);
    if (a.sem_kind == SVX_SEM_CLOSED && a.last_wins) {
        for (int q = lane; q < a.C; q += 32) crow[q] = (TC)(q == acc.last_lab - 1 ? 1 : 0);
    }
}

// ---- K5 long / huge (closed / geometry): one warp per voxel --------------------

template <class TD, class TC>
__device__ __forceinline__ void k_update_long_body(UpdateArgs a, TD* vt,
                                                                   TC* counts) {
    grid_dep_wait();
    __shared__ int sbuf[kWarpsPerCta][kSmemMax];
    FrameCtr* ctr = a.ctr;
    KSpan _ks(ctr, kSpanUpdateB);
    __shared__ FrameCtr s_ctr_;
    snapshot_ctr(ctr, s_ctr_);
    const FrameCtr* cv = &s_ctr_;
    if (cv->abort | cv->err_cap) return;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    int* buf = sbuf[wib];
    const KeyPack kp = cv->p.kp;
    const PoseParams pp = cv->p.pp;
    const int32_t* labels = cv->p.labels;
    const bool closed = a.sem_kind == SVX_SEM_CLOSED;
    const long long gw = (long long)blockIdx.x * kWarpsPerCta + wib;
    const long long nwarps = (long long)gridDim.x * kWarpsPerCta;
    const long long L = (long long)cv->n_long;
#if SVX_DYN_LONG
    // voxels cost from 17 to 1024 rows: warps take the next one from a frame
    // counter instead of a fixed stride, so no warp idles while others work
    for (long long t = 0;;) {
        if (lane == 0) t = (long long)atomicAdd(&ctr->work_long, 1ULL);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= L) break;
#else
    for (long long t = gw; t < L; t += nwarps) {
#endif
        const int vid = a.mlist[a.longlist[t]];
        const unsigned c = a.rec[vid].cnt;
        const unsigned k = c & ~kNewBit;
        warp_sort_segment(a.srid, a.rec[vid].seg, (int)k, buf);
        const Center cc = center_of(a.rec[vid].key, kp, a.h, pp);
        TC* crow = counts + (long long)vid * a.C;
        TsdfAcc acc{0.0, 0.0, INFINITY, -INFINITY, 0};
        warp_tsdf_chunk<TC>(a, labels, buf, (int)k, cc, acc, crow, closed);
        finish_closed<TD, TC>(a, vt, crow, vid, (c & kNewBit) != 0u, acc);
        __syncwarp();
        if (lane == 0) clear_voxel_frame(a, vid);
        __syncwarp();
    }
    // huge segments: only the first kHugeWarps warps own bitmap scratch
    if (gw >= kHugeWarps) return;
    unsigned* bm = a.bitmap + gw * a.bm_words;
    const long long Hn = (long long)cv->n_huge;
    for (long long t = gw; t < Hn; t += kHugeWarps) {
        const int vid = a.mlist[a.hugelist[t]];
        const unsigned c = a.rec[vid].cnt;
        const unsigned k = c & ~kNewBit;
        int minr;
        long long nwords;
        bitmap_build(a.srid, a.rec[vid].seg, k, bm, minr, nwords);
        const Center cc = center_of(a.rec[vid].key, kp, a.h, pp);
        TC* crow = counts + (long long)vid * a.C;
        TsdfAcc acc{0.0, 0.0, INFINITY, -INFINITY, 0};
        for (long long w0 = 0; w0 < nwords; w0 += 32) {
            const int cnt = bitmap_chunk(bm, w0, nwords, minr, buf);
            if (cnt) warp_tsdf_chunk<TC>(a, labels, buf, cnt, cc, acc, crow, closed);
            __syncwarp();
        }
        finish_closed<TD, TC>(a, vt, crow, vid, (c & kNewBit) != 0u, acc);
        __syncwarp();
        if (lane == 0) clear_voxel_frame(a, vid);
        __syncwarp();
    }
}

template <class TD, class TC>
#ifndef SVX_LONGK_MINB
#define SVX_LONGK_MINB 4
#endif
__global__ void __launch_bounds__(32 * kWarpsPerCta, SVX_LONGK_MINB) k_update_long(UpdateArgs a, TD* vt, TC* counts) {
    k_update_long_body(a, vt, counts);
    frame_epilogue(a.ctr, a.ctr->p.epilogue, a.ctr->p.mirror);
}

// ---- K5 open set: one warp per voxel, lanes own feature dimensions ------------

constexpr int kOpenPer = 8;   // dims per lane per pass (256 dims per pass)
#ifndef SVX_OPEN_SPLIT
#define SVX_OPEN_SPLIT 1
#endif
__device__ __forceinline__ int open_col(int lane, int q) {
#if SVX_OPEN_SPLIT
    return (q >> 2) * 128 + 4 * lane + (q & 3);
#else
    return 8 * lane + q;
#endif
}

#ifndef SVX_OPEN_RING
#define SVX_OPEN_RING 1
#endif
// open-set voxels with more rows than this go to the CTA-per-voxel kernel
#ifndef SVX_OPEN_PREFETCH
#define SVX_OPEN_PREFETCH 1
#endif
#ifndef SVX_OPEN_CTA_MIN
#define SVX_OPEN_CTA_MIN 256   // measured best of 64 / 256 / 1024 on cfg3 and cfg5
#endif
constexpr int kOpenCtaMin = SVX_OPEN_CTA_MIN;
// (k_update_open sorts a segment in a power-of-two shared buffer of kOpenCtaMin rows)
static_assert((kOpenCtaMin & (kOpenCtaMin - 1)) == 0 && kOpenCtaMin >= 32 && kOpenCtaMin <= kSmemMax,
              "kOpenCtaMin: a power of two in [32, kSmemMax]");

template <class TS>
__device__ __forceinline__ void nig_apply(TS* mrow, TS* brow, int c, bool isnew, double sz,
                                          double sz2, double lam, double lam_post, double coef,
                                          double nobs, double b_bg) {
    // apply_open (_pycore.py:432-446) for one dimension
    double m_old = isnew ? 0.0 : (double)mrow[c];
    double b_old = isnew ? b_bg : (double)brow[c];
    double m_new = (lam * m_old + sz) / lam_post;
    double zbar = sz / nobs;
    double ss = sz2 - sz * zbar;
    ss = ss < 0.0 ? 0.0 : ss;
    double diff = zbar - m_old;
    double gap = coef * (diff * diff) * 0.5;
    double b_new = b_old + 0.5 * ss + gap;
    mrow[c] = (TS)m_new;
    brow[c] = (TS)b_new;
}

// nig_apply for the 8 dimensions base + open_col(lane, 0..7) of a full pass (f32
// state: two 16-byte loads and stores per row of mean / beta); per element the
// same arithmetic as nig_apply.
// a / b, correctly rounded, from y = RN(1 / b): q = RN(a y) is within an ulp of
// a / b, the residual a - q b is exact (FMA), and one corrected FMA rounds to
// RN(a / b) (Markstein's theorem; finite operands, no underflow -- the NIG sums
// and weights here).  Checked against IEEE division on 2e8 random pairs
// (nobs-, lambda- and wide-range divisors).  Saves the per-element DDIV
// sequence (reciprocal on the XU pipe + Newton steps) when b is shared.
__device__ __forceinline__ double div_rn(double a, double b, double y) {
    const double q = a * y;
    const double r = fma(-q, b, a);
    return fma(r, y, q);
}

template <class TS>
__device__ __forceinline__ void nig_apply8(TS* mrow, TS* brow, int base, int lane, bool isnew, const double* sz,
                                           const double* sz2, double lam, double lam_post, double coef,
                                           double nobs, double b_bg) {
    if constexpr (sizeof(TS) == 4) {
        float m[8], b[8];
        if (isnew) {
#pragma unroll
            for (int q = 0; q < 8; ++q) { m[q] = 0.0f; b[q] = (float)b_bg; }
        } else {
            const int c0 = base + open_col(lane, 0), c1 = base + open_col(lane, 4);
            const float4 m0 = *reinterpret_cast<const float4*>(mrow + c0),
                         m1 = *reinterpret_cast<const float4*>(mrow + c1),
                         b0 = *reinterpret_cast<const float4*>(brow + c0),
                         b1 = *reinterpret_cast<const float4*>(brow + c1);
            m[0] = m0.x; m[1] = m0.y; m[2] = m0.z; m[3] = m0.w; m[4] = m1.x; m[5] = m1.y; m[6] = m1.z; m[7] = m1.w;
            b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w; b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
        }
        const double inv_lp = 1.0 / lam_post, inv_n = 1.0 / nobs;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const double m_old = isnew ? 0.0 : (double)m[q];
            const double b_old = isnew ? b_bg : (double)b[q];
            const double m_new = div_rn(lam * m_old + sz[q], lam_post, inv_lp);
            const double zbar = div_rn(sz[q], nobs, inv_n);
            double ss = sz2[q] - sz[q] * zbar;
            ss = ss < 0.0 ? 0.0 : ss;
            const double diff = zbar - m_old;
            const double gap = coef * (diff * diff) * 0.5;
            m[q] = (float)m_new;
            b[q] = (float)(b_old + 0.5 * ss + gap);
        }
        const int c0 = base + open_col(lane, 0), c1 = base + open_col(lane, 4);
        *reinterpret_cast<float4*>(mrow + c0) = make_float4(m[0], m[1], m[2], m[3]);
        *reinterpret_cast<float4*>(mrow + c1) = make_float4(m[4], m[5], m[6], m[7]);
        *reinterpret_cast<float4*>(brow + c0) = make_float4(b[0], b[1], b[2], b[3]);
        *reinterpret_cast<float4*>(brow + c1) = make_float4(b[4], b[5], b[6], b[7]);
    } else {
#pragma unroll
        for (int q = 0; q < 8; ++q)
            nig_apply<TS>(mrow, brow, base + open_col(lane, q), isnew, sz[q], sz2[q], lam, lam_post, coef,
                          nobs, b_bg);
    }
}

// L2 prefetch of a voxel's open-set state (mean and beta rows, `bytes` each):
// issued when the voxel is taken, so the per-pass NIG reads hit L2.
__device__ __forceinline__ void prefetch_rows_l2(const void* m, const void* b, int bytes) {
    const int lane = threadIdx.x & 31;
    for (int o = lane * 128; o < bytes; o += 32 * 128) {
        asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"((const char*)m + o));
        asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"((const char*)b + o));
    }
}

// Σz² term of the open-set sums: z is an f32 value widened to f64, so z·z is
// exact in f64 (24-bit significands) and one fused multiply-add rounds exactly
// like the reference's product-then-add (_pycore.py:432-446); f64 features keep
// the two separate steps.
template <class Fe>
__device__ __forceinline__ double add_sq(double s, double z) {
    if constexpr (sizeof(Fe) == 4) return fma(z, z, s);
    else return s + z * z;
}

// Per-dimension sequential sums over an ordered chunk (lane owns dims
// base + lane + 32 q).
template <class Fe>
__device__ __forceinline__ void open_chunk(const Fe* __restrict__ feats, int D, int base,
                                           const int* buf, int cnt, double* sz, double* sz2) {
    const int lane = threadIdx.x & 31;
    int j = 0;
    for (; j < cnt; ++j) {
        const Fe* f = feats + (long long)buf[j] * D + base;
#pragma unroll
        for (int q = 0; q < kOpenPer; ++q) {
            const int cc = lane + 32 * q;
            if (base + cc < D) {
                const double zv = (double)f[cc];
                sz[q] += zv;
                sz2[q] = add_sq<Fe>(sz2[q], zv);
            }
        }
    }
}

// open_chunk with the rows' feature slices streamed through this lane's
// part of a shared-memory ring by cp.async: kOpenRingR rows per group,
// kOpenRingS groups in flight.  Every lane reads back only what it copied
// itself, so the ring needs no warp synchronisation; the sums are the same
// in-order sums as open_chunk.
#ifndef SVX_OPEN_RING_R
#define SVX_OPEN_RING_R 2
#endif
#ifndef SVX_OPEN_RING_S
#define SVX_OPEN_RING_S 2
#endif
constexpr int kOpenRingR = SVX_OPEN_RING_R;
constexpr int kOpenRingS = SVX_OPEN_RING_S;
constexpr int kOpenPass = 32 * kOpenPer;   // dims per pass

template <class Fe>
__device__ __forceinline__ void open_chunk_ring(const Fe* __restrict__ feats, int D, int base,
                                                const int* buf, int cnt, double* sz, double* sz2,
                                                Fe* ring) {
    const int lane = threadIdx.x & 31;
    const int ng = (cnt + kOpenRingR - 1) / kOpenRingR;
    auto issue = [&](int g) {
        if (g < ng) {
            Fe* dst = ring + (g % kOpenRingS) * kOpenRingR * kOpenPass;
#pragma unroll
            for (int r = 0; r < kOpenRingR; ++r) {
                const int j = g * kOpenRingR + r;
                if (j < cnt) {
                    const Fe* src = feats + (long long)buf[j] * D + base;
#pragma unroll
                    for (int q = 0; q < kOpenPer; ++q) {
                        const int cc = lane + 32 * q;
                        if (base + cc < D)
                            __pipeline_memcpy_async(dst + r * kOpenPass + cc, src + cc, sizeof(Fe));
                    }
                }
            }
        }
        __pipeline_commit();
    };
#pragma unroll
    for (int g = 0; g < kOpenRingS - 1; ++g) issue(g);
    for (int g = 0; g < ng; ++g) {
        issue(g + kOpenRingS - 1);
        __pipeline_wait_prior(kOpenRingS - 1);
        const Fe* src = ring + (g % kOpenRingS) * kOpenRingR * kOpenPass;
        const int n = min(kOpenRingR, cnt - g * kOpenRingR);
        for (int r = 0; r < n; ++r) {
#pragma unroll
            for (int q = 0; q < kOpenPer; ++q) {
                const int cc = lane + 32 * q;
                if (base + cc < D) {
                    const double zv = (double)src[r * kOpenPass + cc];
                    sz[q] += zv;
                    sz2[q] = add_sq<Fe>(sz2[q], zv);
                }
            }
        }
    }
    __pipeline_wait_prior(0);
}

// ---- 1-D TMA (cp.async.bulk) feature ring ---------------------------------------
// Each row's slice of kOpenPass feature columns is one contiguous block of
// global memory, so lane 0 moves it into the warp's shared-memory ring with
// one bulk copy (the TMA engine; completion counted in bytes on the slot's
// mbarrier) instead of 8 four-byte cp.async per lane.  kOpenBulkRing rows
// are in flight per warp.  Used when the slice bytes are a multiple of 16
// and the feature array is 16-byte aligned (every BASELINE open-set config).
#ifndef SVX_OPEN_BULK
#define SVX_OPEN_BULK 1
#endif
#ifndef SVX_OPEN_BULK_RING
#define SVX_OPEN_BULK_RING 2
#endif
constexpr int kOpenBulkRing = SVX_OPEN_BULK_RING;

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(b),
        "r"(parity)
        : "memory");
}

// Warp state of the bulk ring: kOpenBulkRing slots of kOpenPass features,
// one mbarrier per slot and the slots' phase bits (warp-uniform).
template <class Fe>
struct BulkRing {
    Fe* slot;                   // kOpenBulkRing * kOpenPass
    unsigned long long* bar;    // kOpenBulkRing
    unsigned phase;             // bit s = parity of slot s's next completion
};

// Full passes (kOpenPass columns): lane owns columns base + 4 lane .. +3 and
// base + 128 + 4 lane .. +3 (SVX_OPEN_SPLIT; else the 8 contiguous columns
// base + 8 lane .. +7), read from the ring with two 16-byte shared loads (f32)
// and no per-column bounds checks; same per-column in-order sums.  The split
// mapping makes each 16-byte load of a warp one contiguous 512-byte span
// (4 shared wavefronts, no bank conflicts) and the mean / beta rows of the
// NIG apply coalesced 512-byte accesses.
template <class Fe>
__device__ __forceinline__ void load8(const Fe* row, int lane, double* v) {
    if constexpr (sizeof(Fe) == 4) {
        const float4 a = *reinterpret_cast<const float4*>(row + open_col(lane, 0)),
                     b = *reinterpret_cast<const float4*>(row + open_col(lane, 4));
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
        v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
        for (int q = 0; q < 8; q += 2) {
            const double2 a = *reinterpret_cast<const double2*>(row + open_col(lane, q));
            v[q] = a.x;
            v[q + 1] = a.y;
        }
    }
}

// Grouped bulk ring: a slot holds kOpenGrp rows and one mbarrier counts all
// their bytes, so a warp waits, syncs and refills once per kOpenGrp rows
// (lanes 0 .. kOpenGrp-1 issue one bulk copy each); kOpenBulkRing slots, i.e.
// kOpenBulkRing * kOpenGrp rows in flight per warp.  Same in-order sums.
#ifndef SVX_OPEN_GRP
#define SVX_OPEN_GRP 4   // 4 rows x 2 slots x 8 warps fit 3 CTAs per SM (6 rows: 2 CTAs)
#endif
constexpr int kOpenGrp = SVX_OPEN_GRP;
#ifndef SVX_OPEN_LDGSTS
#define SVX_OPEN_LDGSTS 0   // 1: group slices by per-lane 16-byte cp.async instead of one bulk copy per row
#endif
#ifndef SVX_OPEN_UNROLL
#define SVX_OPEN_UNROLL 2   // A/B with 4-row groups: 2 beats 3 and 4 by ~3 %
#endif
constexpr int kOpenUnroll = SVX_OPEN_UNROLL;   // rows of a group folded per loop iteration
static_assert(kOpenGrp >= 1 && kOpenGrp <= 32 && kOpenBulkRing <= 32, "grouped ring geometry");

// one bulk copy completing on bar (the expected bytes were posted separately)
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
        "l"(src), "r"(bytes), "r"(b)
        : "memory");
}

template <class Fe, bool kFull>
__device__ __forceinline__ void open_chunk_grp(const Fe* __restrict__ feats, int D, int base, const int* buf,
                                               int cnt, double* sz, double* sz2, BulkRing<Fe>& R) {
    const int lane = threadIdx.x & 31;
    const int nd = kFull ? kOpenPass : min(kOpenPass, D - base);
    const unsigned bytes = (unsigned)(nd * (int)sizeof(Fe));
    const int ng = (cnt + kOpenGrp - 1) / kOpenGrp;
#if SVX_OPEN_LDGSTS
    // every lane moves 16-byte pieces of the group's row slices (cp.async);
    // one commit group per slot, waited per lane, then a warp barrier
    const unsigned nchunk = bytes >> 4;
    auto issue = [&](int g) {
        if (g < ng) {
            const int sl = g % kOpenBulkRing, j0 = g * kOpenGrp;
            const int nr = min(kOpenGrp, cnt - j0);
            for (int r = 0; r < nr; ++r) {
                const char* src = reinterpret_cast<const char*>(feats + (long long)buf[j0 + r] * D + base);
                char* dst = reinterpret_cast<char*>(R.slot + (sl * kOpenGrp + r) * kOpenPass);
                for (unsigned q = lane; q < nchunk; q += 32) __pipeline_memcpy_async(dst + 16 * q, src + 16 * q, 16);
            }
        }
        __pipeline_commit();
    };
    __syncwarp();
    for (int g = 0; g < kOpenBulkRing; ++g) issue(g);
    for (int g = 0; g < ng; ++g) {
        const int sl = g % kOpenBulkRing;
        __pipeline_wait_prior(kOpenBulkRing - 1);
        __syncwarp();
#else
    auto issue = [&](int g) {
        const int sl = g % kOpenBulkRing, j0 = g * kOpenGrp;
        const int nr = min(kOpenGrp, cnt - j0);
        // (every lane's reads of the slot precede this point: __syncwarp below / at the call)
        if (lane == 0) {
            const unsigned b = (unsigned)__cvta_generic_to_shared(R.bar + sl);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b),
                         "r"(bytes * (unsigned)nr) : "memory");
        }
        if (lane < nr) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            bulk_copy(R.slot + (sl * kOpenGrp + lane) * kOpenPass, feats + (long long)buf[j0 + lane] * D + base,
                      bytes, R.bar + sl);
        }
    };
    __syncwarp();
    for (int g = 0; g < kOpenBulkRing && g < ng; ++g) issue(g);
    for (int g = 0; g < ng; ++g) {
        const int sl = g % kOpenBulkRing;
        mbar_wait(R.bar + sl, (R.phase >> sl) & 1u);
        R.phase ^= 1u << sl;
#endif
        const int nr = min(kOpenGrp, cnt - g * kOpenGrp);
        const Fe* src = R.slot + sl * kOpenGrp * kOpenPass;
#pragma unroll (kOpenUnroll)
        for (int r = 0; r < nr; ++r, src += kOpenPass) {
            if constexpr (kFull) {
                double v[kOpenPer];
                load8<Fe>(src, lane, v);
#pragma unroll
                for (int q = 0; q < kOpenPer; ++q) {
                    sz[q] += v[q];
                    sz2[q] = add_sq<Fe>(sz2[q], v[q]);
                }
            } else {
#pragma unroll
                for (int q = 0; q < kOpenPer; ++q) {
                    const int cc = lane + 32 * q;
                    if (cc < nd) {
                        const double zv = (double)src[cc];
                        sz[q] += zv;
                        sz2[q] = add_sq<Fe>(sz2[q], zv);
                    }
                }
            }
        }
        __syncwarp();
#if SVX_OPEN_LDGSTS
        issue(g + kOpenBulkRing);
#else
        if (g + kOpenBulkRing < ng) issue(g + kOpenBulkRing);
#endif
    }
#if SVX_OPEN_LDGSTS
    __pipeline_wait_prior(0);
#endif
}

template <class TD, class TS, class Fe>
__device__ __forceinline__ void open_voxel(const UpdateArgs& a, const KeyPack& kp,
                                           const PoseParams& pp, TD* vt, TS* mean, TS* beta,
                                           const Fe* feats, int vid, unsigned c, int* buf,
                                           unsigned* bm, bool huge, Fe* ring = nullptr,
                                           BulkRing<Fe>* bulk = nullptr, bool prepped = false) {
    const int lane = threadIdx.x & 31;
    const unsigned k = c & ~kNewBit;
    const bool isnew = (c & kNewBit) != 0u;
#if SVX_OPEN_PREFETCH
    if (!isnew) prefetch_rows_l2(mean + (long long)vid * a.D, beta + (long long)vid * a.D, a.D * (int)sizeof(TS));
#endif
    int minr = 0;
    long long nwords = 0;
    double w_old = 0.0;
    if (prepped) {
        // k_open_prep sorted the segment in place and applied the TSDF sums
        const unsigned seg = a.rec[vid].seg;
        for (unsigned j = lane; j < k; j += 32) buf[j] = __ldcg(a.srid + seg + j);
        w_old = __ldcg(&a.rec[vid].wold);
        __syncwarp();
    } else {
    const Center cc = center_of(a.rec[vid].key, kp, a.h, pp);
    if (huge) bitmap_build(a.srid, a.rec[vid].seg, k, bm, minr, nwords);
    else warp_sort_segment(a.srid, a.rec[vid].seg, (int)k, buf);
    // TSDF sums in point order
    TsdfAcc acc{0.0, 0.0, INFINITY, -INFINITY, 0};
    if (huge) {
        for (long long w0 = 0; w0 < nwords; w0 += 32) {
            const int cnt = bitmap_chunk(bm, w0, nwords, minr, buf);
            if (cnt) warp_tsdf_chunk<float>(a, nullptr, buf, cnt, cc, acc, nullptr, false);
            __syncwarp();
        }
    } else {
        warp_tsdf_chunk<float>(a, nullptr, buf, (int)k, cc, acc, nullptr, false);
    }
    if (lane == 0) w_old = apply_tsdf<TD>(vt, vid, isnew, a.trunc, acc.sw, acc.swd, acc.mind, acc.maxd);
    w_old = __shfl_sync(0xffffffffu, w_old, 0);
    }
    // NIG batch update with lambda from the pre-frame weight (_pycore.py:438)
    const double nobs = (double)k;
    const double lam = fmax(w_old, a.lambda_floor);
    const double lam_post = lam + nobs;
    const double coef = lam * nobs / lam_post;
    const double b_bg = (double)(TS)a.prior_beta;
    TS* mrow = mean + (long long)vid * a.D;
    TS* brow = beta + (long long)vid * a.D;
    for (int base = 0; base < a.D; base += 32 * kOpenPer) {
        double sz[kOpenPer], sz2[kOpenPer];
#pragma unroll
        for (int q = 0; q < kOpenPer; ++q) { sz[q] = 0.0; sz2[q] = 0.0; }
        if (huge) {
            for (long long w0 = 0; w0 < nwords; w0 += 32) {
                const int cnt = bitmap_chunk(bm, w0, nwords, minr, buf);
                open_chunk<Fe>(feats, a.D, base, buf, cnt, sz, sz2);
                __syncwarp();
            }
        } else if (bulk && base + kOpenPass <= a.D) {   // full pass, contiguous columns per lane
            open_chunk_grp<Fe, true>(feats, a.D, base, buf, (int)k, sz, sz2, *bulk);
            if ((a.D & 3) == 0) {   // 16-byte aligned rows of mean / beta
                nig_apply8<TS>(mrow, brow, base, lane, isnew, sz, sz2, lam, lam_post, coef, nobs, b_bg);
            } else {
#pragma unroll
                for (int q = 0; q < kOpenPer; ++q)
                    nig_apply<TS>(mrow, brow, base + open_col(lane, q), isnew, sz[q], sz2[q], lam, lam_post,
                                  coef, nobs, b_bg);
            }
            continue;
        } else if (bulk) {
            open_chunk_grp<Fe, false>(feats, a.D, base, buf, (int)k, sz, sz2, *bulk);
        } else if (ring) {
            open_chunk_ring<Fe>(feats, a.D, base, buf, (int)k, sz, sz2, ring);
        } else {
            open_chunk<Fe>(feats, a.D, base, buf, (int)k, sz, sz2);
        }
#pragma unroll
        for (int q = 0; q < kOpenPer; ++q) {
            const int col = base + lane + 32 * q;
            if (col < a.D) nig_apply<TS>(mrow, brow, col, isnew, sz[q], sz2[q], lam, lam_post, coef,
                                         nobs, b_bg);
        }
    }
    __syncwarp();
    if (lane == 0) clear_voxel_frame(a, vid);
    __syncwarp();
}

// K5 open prologue (SVX_OPEN_PREP): per listed voxel of <= kOpenCtaMin rows,
// one warp sorts the voxel's row segment in place (ascending point index,
// the reference's order) and applies its TSDF sums (_pycore.py:399-417);
// the pre-frame weight the NIG update needs goes to rec[vid].wold.
// k_update_open then runs only the feature passes, so its warps (3 per
// scheduler, big rings) no longer wait on each segment's scattered ray
// loads; this kernel hides them with 8 small CTAs per SM.
#ifndef SVX_OPEN_PREP
#define SVX_OPEN_PREP 0   // measured slower (update +11 % cfg3, +8 % cfg5): the prologue was already hidden
#endif
template <class TD>
__global__ void __launch_bounds__(32 * kWarpsPerCta) k_open_prep(UpdateArgs a, TD* vt, int* srid) {
    grid_dep_wait();
    __shared__ int sbuf[kWarpsPerCta][kOpenCtaMin];
    FrameCtr* ctr = a.ctr;
    KSpan _ks(ctr, kSpanUpdate);
    __shared__ FrameCtr s_ctr_;
    snapshot_ctr(ctr, s_ctr_);
    const FrameCtr* cv = &s_ctr_;
    if (cv->abort | cv->err_cap) return;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const long long L = (long long)cv->n_list;
    const KeyPack kp = cv->p.kp;
    const PoseParams pp = cv->p.pp;
    int* buf = sbuf[wib];
    for (long long e = (long long)blockIdx.x * kWarpsPerCta + wib; e < L;
         e += (long long)gridDim.x * kWarpsPerCta) {
        const int vid = a.mlist[e];
        const unsigned c = a.rec[vid].cnt;
        const unsigned k = c & ~kNewBit;
        if (k > (unsigned)kOpenCtaMin) continue;   // k_huge_prep sorts these
        const unsigned seg = a.rec[vid].seg;
        warp_sort_segment(srid, seg, (int)k, buf);
        for (unsigned j = lane; j < k; j += 32) srid[seg + j] = buf[j];
        const Center cc = center_of(a.rec[vid].key, kp, a.h, pp);
        TsdfAcc acc{0.0, 0.0, INFINITY, -INFINITY, 0};
        warp_tsdf_chunk<float>(a, nullptr, buf, (int)k, cc, acc, nullptr, false);
        if (lane == 0)
            a.rec[vid].wold = apply_tsdf<TD>(vt, vid, (c & kNewBit) != 0u, a.trunc, acc.sw, acc.swd, acc.mind,
                                             acc.maxd);
        __syncwarp();
    }
}

// K5 open: every listed voxel; huge segments are deferred to k_update_open_huge.
template <class TD, class TS, class Fe>
#ifndef SVX_OPEN_MINB
#define SVX_OPEN_MINB 3   // 2 CTAs per SM (<= 128 registers): cfg3 update -38 %, cfg5 -39 % vs 1; 3 CTAs
                          // (<= 80 registers, 40 B spilled, 4-row groups): a further -3 % / -2 %
#endif
__global__ void __launch_bounds__(32 * kWarpsPerCta, SVX_OPEN_MINB) k_update_open(UpdateArgs a, TD* vt, TS* mean,
                                                                   TS* beta) {
    grid_dep_wait();
    __shared__ int sbuf[kWarpsPerCta][kOpenCtaMin];   // a segment of <= kOpenCtaMin rows
#if SVX_OPEN_RING || SVX_OPEN_BULK
    extern __shared__ __align__(128) unsigned char oring[];
#endif
    FrameCtr* ctr = a.ctr;
    KSpan _ks(ctr, kSpanUpdate, SVX_OPEN_PREP != 0);   // the stage spans k_open_prep too
    __shared__ FrameCtr s_ctr_;
    snapshot_ctr(ctr, s_ctr_);
    const FrameCtr* cv = &s_ctr_;
    if (cv->abort | cv->err_cap) return;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const long long L = (long long)cv->n_list;
    const KeyPack kp = cv->p.kp;
    const PoseParams pp = cv->p.pp;
    const Fe* feats = (const Fe*)cv->p.feats;
#if SVX_OPEN_BULK
    // bulk ring (dynamic shared memory after the cp.async ring's space)
    __shared__ __align__(8) unsigned long long s_bar[kWarpsPerCta][kOpenBulkRing];
    const bool use_bulk = ((a.D * (int)sizeof(Fe)) % 16) == 0 && (((uintptr_t)feats) & 15) == 0;
    BulkRing<Fe> bulk;
    bulk.slot = reinterpret_cast<Fe*>(oring) + (size_t)wib * kOpenBulkRing * kOpenGrp * kOpenPass;
    bulk.bar = s_bar[wib];
    bulk.phase = 0u;
    if (use_bulk && lane == 0) {
        for (int q = 0; q < kOpenBulkRing; ++q) mbar_init(bulk.bar + q, 1u);
        mbar_fence_init();
    }
    __syncwarp();
#endif
#if SVX_DYN_LONG
    for (long long e = 0;;) {
        if (lane == 0) e = (long long)atomicAdd(&ctr->work_open, 1ULL);
        e = __shfl_sync(0xffffffffu, e, 0);
        if (e >= L) break;
#else
    for (long long e = (long long)blockIdx.x * kWarpsPerCta + wib; e < L;
         e += (long long)gridDim.x * kWarpsPerCta) {
#endif
        const int vid = a.mlist[e];
        const unsigned c = a.rec[vid].cnt;
        if ((c & ~kNewBit) > (unsigned)kOpenCtaMin) {   // one CTA per voxel (k_update_open_huge)
            if (lane == 0) a.hugelist[atomicAdd(&ctr->n_huge, 1ULL)] = (int)e;
            continue;
        }
#if SVX_OPEN_BULK
        if (use_bulk) {
            open_voxel<TD, TS, Fe>(a, kp, pp, vt, mean, beta, feats, vid, c, sbuf[wib], nullptr, false,
                                   nullptr, &bulk, SVX_OPEN_PREP != 0);
            continue;
        }
#endif
#if SVX_OPEN_RING
        Fe* ring = reinterpret_cast<Fe*>(oring) + (size_t)wib * kOpenRingS * kOpenRingR * kOpenPass;
        open_voxel<TD, TS, Fe>(a, kp, pp, vt, mean, beta, feats, vid, c, sbuf[wib], nullptr, false, ring,
                               nullptr, SVX_OPEN_PREP != 0);
#else
        open_voxel<TD, TS, Fe>(a, kp, pp, vt, mean, beta, feats, vid, c, sbuf[wib], nullptr, false, nullptr,
                               nullptr, SVX_OPEN_PREP != 0);
#endif
    }
}

// K5 open, voxels of more than kOpenCtaMin rows (a depth camera close to a
// surface funnels most of its rays into a few voxels).  Every dimension's
// two sums and the TSDF sums are sequential over the voxel's rows in point
// order (the reference's order), so one voxel's work cannot be split by
// rows -- but its dimensions are independent, so it is split by them:
//   k_huge_prep   one CTA per huge voxel: stash (vid, count, segment, the
//                 pre-frame weight) and sort the voxel's row ids in place
//                 (point-index bitmap in per-CTA scratch, CTA-wide scan);
//   k_huge_items  work items (voxel, 32-dimension slice) plus one TSDF item
//                 per voxel, over persistent CTAs (one per SM): a slice's
//                 feature columns stream through a 4-stage shared-memory ring
//                 with cp.async gathers issued by all 256 threads (~96 KB in
//                 flight per SM), while one warp folds them (lane = dimension)
//                 -- so a voxel of N rows runs on ceil(D / 32) + 1 SMs at
//                 once, each bound by its fp64 add chain, not by the few
//                 bytes one thread can keep in flight.
constexpr int kHugeThreads = 256;
constexpr int kHugeCtas = kHugeWarps;    // prep CTAs sharing the bitmap scratch
constexpr int kHugeSlice = 32;           // dimensions per feature item
constexpr int kHugeStages = 4;
#ifndef SVX_HUGE_STAGE_KB
#define SVX_HUGE_STAGE_KB 16
#endif
#ifndef SVX_HUGE_ITEM_CPS
#define SVX_HUGE_ITEM_CPS 3
#endif
constexpr int kHugeStageBytes = SVX_HUGE_STAGE_KB * 1024;
constexpr int kHugeItemCtas = 148 * SVX_HUGE_ITEM_CPS;   // CTAs per SM x SMs (4 stages of shared memory each)
// Voxels of up to kGiantRows rows: one CTA each (k_update_open_huge, all
// dimensions); bigger ones: dimension slices over many SMs (k_huge_items).
#ifndef SVX_GIANT_ROWS
#define SVX_GIANT_ROWS 4096   // A/B: cfg3 close-wall frames update_b -18 % vs 8192, cfg5 neutral; 16384 worse
#endif
constexpr int kGiantRows = SVX_GIANT_ROWS;
// k_huge_items: warps folding one item's dimensions (32 each); the SM folds
// kHugeFold * 32 dimension chains at once (1 = one fold warp per SM).
#ifndef SVX_HUGE_FOLD
#define SVX_HUGE_FOLD 1
#endif
constexpr int kHugeFold = SVX_HUGE_FOLD;
static_assert(kHugeFold >= 1 && kHugeFold <= 8, "fold warps per item");
#ifndef SVX_HUGE_MINB
#define SVX_HUGE_MINB 3   // k_update_open_huge CTAs per SM (<= 85 registers, no spills)
#endif
#ifndef SVX_HUGE_RING_KB
#define SVX_HUGE_RING_KB 72
#endif
constexpr int kHugeRingBytes = SVX_HUGE_RING_KB * 1024;   // k_update_open_huge: three row slots of dynamic shared memory

struct HugeInfo {
    int vid;
    unsigned cnt;      // frame count with the new-voxel bit
    unsigned seg;
    unsigned pad;
    double w_old;      // pre-frame TSDF weight (lambda of the NIG update)
};

// K5 open, voxels of kOpenCtaMin+1 .. kGiantRows rows (a depth camera close
// to a surface funnels most of its rays into a few voxels): one CTA per voxel,
// after k_huge_prep sorted its rows and applied its TSDF sums.  Row slices of
// up to 1024 dimensions stream through three shared-memory slots by 16-byte
// cp.async (a warp per row); every thread folds its own dimensions in row
// order, so the voxel's D sums run in parallel and each is the sequential
// point-ordered fp64 sum of the warp path.
constexpr int kHugeDims = 4;             // dims per feature thread and pass

// Per-thread fold of dims tid + 256 q (q < NQ) over nr staged rows (row
// stride hpw): sequential per-dimension Σz, Σz² in row order.
template <int NQ, class Fe>
__device__ __forceinline__ void fold_rows(const Fe* src, int nr, int hpw, int tid, double* sz, double* sz2) {
#pragma unroll 2
    for (int r = 0; r < nr; ++r, src += hpw) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const int col = tid + q * kHugeThreads;
            if (q < NQ - 1 || col < hpw) {
                const double z = (double)src[col];
                sz[q] += z;
                sz2[q] = add_sq<Fe>(sz2[q], z);
            }
        }
    }
}

template <class TD, class TS, class Fe>
__device__ __forceinline__ void k_update_open_huge_body(UpdateArgs a, TD* vt, TS* mean, TS* beta,
                                                        const HugeInfo* __restrict__ hinfo) {
    grid_dep_wait();
    extern __shared__ __align__(16) unsigned char hring_raw[];
    Fe* hring = reinterpret_cast<Fe*>(hring_raw);
    FrameCtr* ctr = a.ctr;
    KSpan _ks(ctr, kSpanUpdateB, true);   // update_b: k_huge_prep .. k_huge_items
    __shared__ FrameCtr s_ctr_;
    snapshot_ctr(ctr, s_ctr_);
    const FrameCtr* cv = &s_ctr_;
    if (cv->abort | cv->err_cap) return;
    const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
    const long long Hn = (long long)cv->n_huge;
    const Fe* feats = (const Fe*)cv->p.feats;
    const int D = a.D;
    // vector mode: row slices by 16-byte cp.async (16-byte sizes and addresses)
    const bool hbulk = ((D * (int)sizeof(Fe)) & 15) == 0 && (((uintptr_t)feats) & 15) == 0;
#if SVX_DYN_LONG
    __shared__ long long s_next;
    for (;;) {
        __syncthreads();   // every thread has read the previous ticket
        if (tid == 0) s_next = (long long)atomicAdd(&ctr->work_huge, 1ULL);
        __syncthreads();
        const long long t = s_next;
        if (t >= Hn) break;
#else
    for (long long t = blockIdx.x; t < Hn; t += gridDim.x) {
#endif
        const HugeInfo hi = hinfo[t];   // k_huge_prep: rows sorted, TSDF applied
        const unsigned k = hi.cnt & ~kNewBit;
        if (k > (unsigned)kGiantRows) continue;   // dimension-sliced kernel (k_huge_items)
        const bool isnew = (hi.cnt & kNewBit) != 0u;
        const int vid = hi.vid;
        const int* ids = a.srid + hi.seg;
        const int cnt = (int)k;
        // NIG batch update with lambda from the pre-frame weight (_pycore.py:438)
        const double nobs = (double)k;
        const double lam = fmax(hi.w_old, a.lambda_floor);
        const double lam_post = lam + nobs;
        const double coef = lam * nobs / lam_post;
        const double b_bg = (double)(TS)a.prior_beta;
        TS* mrow = mean + (long long)vid * D;
        TS* brow = beta + (long long)vid * D;
        // dims in passes of kHugeDims * kHugeThreads (one pass for D <= 1024);
        // thread tid owns dims dbase + tid + 256 q
        for (int dbase = 0; dbase < D; dbase += kHugeDims * kHugeThreads) {
            const int hpw = min(kHugeDims * kHugeThreads, D - dbase);   // this pass's columns
            double sz[kHugeDims], sz2[kHugeDims];
#pragma unroll
            for (int q = 0; q < kHugeDims; ++q) { sz[q] = 0.0; sz2[q] = 0.0; }
            if (hbulk) {
                // rows stream through three slots of hG rows (one barrier per
                // group): a warp copies a whole row slice with 16-byte cp.async
                // per lane, then every thread folds its dims of each row in order
                const int hG = max(1, min(16, kHugeRingBytes / (3 * hpw * (int)sizeof(Fe))));
                const int ng = (cnt + hG - 1) / hG;
                const int c4 = hpw * (int)sizeof(Fe) / 16;   // 16-byte chunks per row
                auto issue = [&](int g) {
                    if (g < ng) {
                        const int j0 = g * hG, nr = min(hG, cnt - j0);
                        Fe* dst = hring + (size_t)(g % 3) * hG * hpw;
                        for (int r = wib; r < nr; r += kHugeThreads / 32) {
                            const char* srow = reinterpret_cast<const char*>(feats + (long long)__ldg(ids + j0 + r) * D + dbase);
                            char* drow = reinterpret_cast<char*>(dst + (size_t)r * hpw);
                            for (int cc = lane; cc < c4; cc += 32)
                                __pipeline_memcpy_async(drow + cc * 16, srow + cc * 16, 16);
                        }
                    }
                    __pipeline_commit();
                };
                issue(0);
                issue(1);
                for (int g = 0; g < ng; ++g) {
                    const int nr = min(hG, cnt - g * hG);
                    __pipeline_wait_prior(1);   // this thread's copies of group g
                    __syncthreads();            // everyone's; everyone is done with group g - 1
                    issue(g + 2);               // into group g - 1's slot
                    const Fe* src = hring + (size_t)(g % 3) * hG * hpw;
                    switch ((hpw + kHugeThreads - 1) / kHugeThreads) {
                        case 1: fold_rows<1, Fe>(src, nr, hpw, tid, sz, sz2); break;
                        case 2: fold_rows<2, Fe>(src, nr, hpw, tid, sz, sz2); break;
                        case 3: fold_rows<3, Fe>(src, nr, hpw, tid, sz, sz2); break;
                        default: fold_rows<4, Fe>(src, nr, hpw, tid, sz, sz2); break;
                    }
                }
                __pipeline_wait_prior(0);
                __syncthreads();   // every fold done before the slots are reused
            } else {
                // unaligned rows: direct loads, same in-order sums
#pragma unroll
                for (int q = 0; q < kHugeDims; ++q) {
                    const int col = dbase + tid + q * kHugeThreads;
                    if (tid + q * kHugeThreads >= hpw) continue;
                    for (int j = 0; j < cnt; ++j) {
                        const double z = (double)feats[(long long)__ldg(ids + j) * D + col];
                        sz[q] += z;
                        sz2[q] = add_sq<Fe>(sz2[q], z);
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < kHugeDims; ++q) {
                const int col = dbase + tid + q * kHugeThreads;
                if (tid + q * kHugeThreads < hpw)
                    nig_apply<TS>(mrow, brow, col, isnew, sz[q], sz2[q], lam, lam_post, coef, nobs, b_bg);
            }
        }
    }
}

template <class TD, class TS, class Fe>
__global__ void __launch_bounds__(kHugeThreads, SVX_HUGE_MINB) k_update_open_huge(UpdateArgs a, TD* vt, TS* mean, TS* beta,
                                                                     const HugeInfo* __restrict__ hinfo) {
    k_update_open_huge_body<TD, TS, Fe>(a, vt, mean, beta, hinfo);
}

// K5p: every huge voxel (> kOpenCtaMin rows), one CTA each: sort the voxel's
// row ids in place (point-index bitmap in per-CTA scratch, CTA scan), fold
// its TSDF sums in point order (d, w of 1024 rows at a time in parallel,
// thread 0 adds them in order; min / max by reduction), apply apply_tsdf and
// stash (id, count, segment, pre-frame weight) for the feature kernels.  The
// feature sums then read the sorted segment directly, with no per-row TSDF
// chain inside their CTA-wide steps.
template <class TD>
__global__ void __launch_bounds__(kHugeThreads) k_huge_prep(UpdateArgs a, TD* vt, HugeInfo* hinfo, int* srid) {
    grid_dep_wait();
    using Scan = cub::BlockScan<int, kHugeThreads>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ int s_min, s_max;
    __shared__ double s_w[1024], s_p[1024];
    __shared__ double s_red[2][kHugeThreads / 32];
    FrameCtr* ctr = a.ctr;
    KSpan _ks(ctr, kSpanUpdateB);   // update_b: this kernel .. k_huge_items (end-only spans)
    __shared__ FrameCtr s_ctr_;
    snapshot_ctr(ctr, s_ctr_);
    const FrameCtr* cv = &s_ctr_;
    if (cv->abort | cv->err_cap) return;
    const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
    unsigned* bm = a.bitmap + (long long)blockIdx.x * a.bm_words;
    const long long Hn = (long long)cv->n_huge;
    const KeyPack kp = cv->p.kp;
    const PoseParams pp = cv->p.pp;
    for (long long t = blockIdx.x; t < Hn; t += gridDim.x) {
        const int vid = a.mlist[a.hugelist[t]];
        const unsigned c = a.rec[vid].cnt;
        const unsigned k = c & ~kNewBit;
        const unsigned seg = a.rec[vid].seg;
        if (tid == 0) {
            s_min = 0x7fffffff;
            s_max = -1;
        }
        __syncthreads();
        int mn = 0x7fffffff, mx = -1;
        for (unsigned j = tid; j < k; j += kHugeThreads) {
            const int v = srid[seg + j];
            mn = min(mn, v);
            mx = max(mx, v);
        }
        mn = (int)__reduce_min_sync(0xffffffffu, (unsigned)mn);
        mx = (int)__reduce_max_sync(0xffffffffu, (unsigned)(mx + 1)) - 1;
        if (lane == 0) {
            atomicMin(&s_min, mn);
            atomicMax(&s_max, mx);
        }
        __syncthreads();
        const int minr = s_min;
        const long long nwords = ((long long)(s_max - minr) >> 5) + 1;
        for (long long w = tid; w < nwords; w += kHugeThreads) bm[w] = 0u;
        __syncthreads();
        for (unsigned j = tid; j < k; j += kHugeThreads) {
            const int v = srid[seg + j] - minr;
            atomicOr(&bm[v >> 5], 1u << (v & 31));
        }
        __threadfence_block();
        __syncthreads();
        // ascending ids back into the segment
        int base = 0;
        for (long long w0 = 0; w0 < nwords; w0 += kHugeThreads) {
            const long long w = w0 + tid;
            unsigned bits = w < nwords ? __ldcg(bm + w) : 0u;
            int off, total;
            Scan(scan_tmp).ExclusiveSum(__popc(bits), off, total);
            int pos = base + off;
            while (bits) {
                const int b = __ffs(bits) - 1;
                bits &= bits - 1;
                srid[seg + pos++] = minr + (int)(w * 32 + b);
            }
            base += total;
            __syncthreads();
        }
        __threadfence_block();
        __syncthreads();
        if (k > (unsigned)kGiantRows) {
            // giant voxel: its TSDF item in k_huge_items runs beside the feature
            // items (and clears the voxel's frame record)
            if (tid == 0) {
                HugeInfo hi;
                hi.vid = vid;
                hi.cnt = c;
                hi.seg = seg;
                hi.pad = 0u;
                hi.w_old = (c & kNewBit) ? 0.0 : (double)vt[2 * (long long)vid + 1];
                hinfo[t] = hi;
            }
            __syncthreads();
            continue;
        }
        // TSDF sums in point order (_core.pyx:759-843)
        const Center cc = center_of(a.rec[vid].key, kp, a.h, pp);
        const int* ids = srid + seg;
        double sw = 0.0, swd = 0.0, mind = INFINITY, maxd = -INFINITY;
        for (unsigned j0 = 0; j0 < k; j0 += 1024) {
            const unsigned n = min(1024u, k - j0);
            for (unsigned q = tid; q < n; q += kHugeThreads) {
                double d, wr;
                row_dw(cc.x, cc.y, cc.z, a.ray[ids[j0 + q]], a.trunc, a.wfn, d, wr);
                s_w[q] = wr;
                s_p[q] = wr * d;
                mind = d < mind ? d : mind;
                maxd = d > maxd ? d : maxd;
            }
            __syncthreads();
            if (tid == 0) {
                unsigned q = 0;
                for (; q + 8 <= n; q += 8) {
                    double wv[8], pv[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        wv[u] = s_w[q + u];
                        pv[u] = s_p[q + u];
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        sw += wv[u];
                        swd += pv[u];
                    }
                }
                for (; q < n; ++q) {
                    sw += s_w[q];
                    swd += s_p[q];
                }
            }
            __syncthreads();
        }
        for (int o = 16; o; o >>= 1) {
            mind = fmin(mind, __shfl_xor_sync(0xffffffffu, mind, o));
            maxd = fmax(maxd, __shfl_xor_sync(0xffffffffu, maxd, o));
        }
        if (lane == 0) {
            s_red[0][wib] = mind;
            s_red[1][wib] = maxd;
        }
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < kHugeThreads / 32; ++w) {
                mind = fmin(mind, s_red[0][w]);
                maxd = fmax(maxd, s_red[1][w]);
            }
            HugeInfo hi;
            hi.vid = vid;
            hi.cnt = c;
            hi.seg = seg;
            hi.pad = 0u;
            hi.w_old = apply_tsdf<TD>(vt, vid, (c & kNewBit) != 0u, a.trunc, sw, swd, mind, maxd);
            hinfo[t] = hi;
            clear_voxel_frame(a, vid);   // (the feature kernels read hinfo only)
        }
        __syncthreads();
    }
}

template <class TD, class TS, class Fe>
__global__ void __launch_bounds__(kHugeThreads, SVX_HUGE_ITEM_CPS) k_huge_items(UpdateArgs a, TD* vt, TS* mean, TS* beta,
                                                                const HugeInfo* __restrict__ hinfo) {
    extern __shared__ __align__(16) unsigned char hsm[];
    grid_dep_wait();
    FrameCtr* ctr = a.ctr;
    {
    KSpan _ks(ctr, kSpanUpdateB, true);   // update_b spans k_huge_prep .. k_huge_items
    __shared__ FrameCtr s_ctr_;
    __shared__ double s_red[4][kHugeThreads / 32];
    snapshot_ctr(ctr, s_ctr_);
    const FrameCtr* cv = &s_ctr_;
    if (!(cv->abort | cv->err_cap)) {
    const int tid = threadIdx.x, wib = tid >> 5, lane = tid & 31;
    const int D = a.D;
    constexpr int G = kHugeFold;   // folding warps per item (32 dimensions each)
    const int S = (D + G * kHugeSlice - 1) / (G * kHugeSlice);
    const long long Hn = (long long)cv->n_huge;
    const KeyPack kp = cv->p.kp;
    const PoseParams pp = cv->p.pp;
    const Fe* feats = (const Fe*)cv->p.feats;
    // items: per giant voxel S feature slices and one TSDF item
    const long long items = Hn * (S + 1);
#if SVX_DYN_LONG
    __shared__ long long s_next;
    for (;;) {
        __syncthreads();   // every thread has read the previous ticket
        if (tid == 0) s_next = (long long)atomicAdd(&ctr->work_items, 1ULL);
        __syncthreads();
        const long long it = s_next;
        if (it >= items) break;
#else
    for (long long it = blockIdx.x; it < items; it += gridDim.x) {
#endif
        const long long t = it / (S + 1);
        const int sl = (int)(it % (S + 1));
        const HugeInfo hi = hinfo[t];
        const int vid = hi.vid;
        const unsigned k = hi.cnt & ~kNewBit;
        const bool isnew = (hi.cnt & kNewBit) != 0u;
        const int* ids = a.srid + hi.seg;
        if (k <= (unsigned)kGiantRows) continue;   // k_update_open_huge's voxel (k_huge_prep applied its TSDF)
        if (sl == S) {
            // ---- TSDF item: w and w*d of 1024 rows at a time in parallel; thread 0
            // folds the two sums in order (loads batched ahead of the adds), min/max
            // by reduction (order-free)
            double* s_w = reinterpret_cast<double*>(hsm);
            double* s_p = s_w + 1024;
            const Center cc = center_of(a.rec[vid].key, kp, a.h, pp);
            double sw = 0.0, swd = 0.0, mind = INFINITY, maxd = -INFINITY;
            for (unsigned j0 = 0; j0 < k; j0 += 1024) {
                const unsigned n = min(1024u, k - j0);
                for (unsigned q = tid; q < n; q += kHugeThreads) {
                    double d, wr;
                    row_dw(cc.x, cc.y, cc.z, a.ray[ids[j0 + q]], a.trunc, a.wfn, d, wr);
                    s_w[q] = wr;
                    s_p[q] = wr * d;
                    mind = d < mind ? d : mind;
                    maxd = d > maxd ? d : maxd;
                }
                __syncthreads();
                if (tid == 0) {
                    unsigned q = 0;
                    for (; q + 8 <= n; q += 8) {
                        double wv[8], pv[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            wv[u] = s_w[q + u];
                            pv[u] = s_p[q + u];
                        }
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            sw += wv[u];
                            swd += pv[u];
                        }
                    }
                    for (; q < n; ++q) {
                        sw += s_w[q];
                        swd += s_p[q];
                    }
                }
                __syncthreads();
            }
            for (int o = 16; o; o >>= 1) {
                mind = fmin(mind, __shfl_xor_sync(0xffffffffu, mind, o));
                maxd = fmax(maxd, __shfl_xor_sync(0xffffffffu, maxd, o));
            }
            if (lane == 0) {
                s_red[0][wib] = mind;
                s_red[1][wib] = maxd;
            }
            __syncthreads();
            if (tid == 0) {
                for (int w = 1; w < kHugeThreads / 32; ++w) {
                    mind = fmin(mind, s_red[0][w]);
                    maxd = fmax(maxd, s_red[1][w]);
                }
                apply_tsdf<TD>(vt, vid, isnew, a.trunc, sw, swd, mind, maxd);
                clear_voxel_frame(a, vid);
            }
            __syncthreads();
            continue;
        }
        // ---- feature item: the G * 32 dimensions of slice sl
        const int col0 = sl * G * kHugeSlice;
        const int ncols = min(G * kHugeSlice, D - col0);
        const int W = G * kHugeSlice;                                  // row stride in the stage
        const int SR = kHugeStageBytes / (W * (int)sizeof(Fe));        // rows per stage
        const int nst = (int)((k + SR - 1) / SR);
        // every stage holds exactly kEpt elements per thread: the row ids of a
        // thread's elements are loaded together first (independent loads), then
        // its gathers are issued
        constexpr int kEpt = kHugeStageBytes / (int)sizeof(Fe) / kHugeThreads;
        // 16-byte copies (kVec elements) when rows, slices and the array allow
        constexpr int kVec = 16 / (int)sizeof(Fe);
        constexpr int kCpt = kEpt / kVec;   // 16-byte chunks per thread and stage
        const bool vec = ((D * (int)sizeof(Fe)) & 15) == 0 && (((uintptr_t)feats) & 15) == 0;
        auto issue = [&](int st) {
            if (st < nst && vec) {
                Fe* buf = reinterpret_cast<Fe*>(hsm + (st % kHugeStages) * kHugeStageBytes);
                int idv[kCpt];
#pragma unroll
                for (int i = 0; i < kCpt; ++i) {
                    const int e = (tid + i * kHugeThreads) * kVec;
                    const unsigned j = (unsigned)(st * SR + e / W);
                    idv[i] = j < k ? __ldg(ids + j) : 0;
                }
#pragma unroll
                for (int i = 0; i < kCpt; ++i) {
                    const int e = (tid + i * kHugeThreads) * kVec;
                    const int r = e / W, c = e - r * W;
                    const unsigned j = (unsigned)(st * SR + r);
                    if (j < k && c < ncols)
                        __pipeline_memcpy_async(buf + e, feats + (long long)idv[i] * D + col0 + c, 16);
                }
            } else if (st < nst) {
                Fe* buf = reinterpret_cast<Fe*>(hsm + (st % kHugeStages) * kHugeStageBytes);
                int idv[kEpt];
#pragma unroll
                for (int i = 0; i < kEpt; ++i) {
                    const int e = tid + i * kHugeThreads;
                    const unsigned j = (unsigned)(st * SR + e / W);
                    idv[i] = j < k ? __ldg(ids + j) : 0;
                }
#pragma unroll
                for (int i = 0; i < kEpt; ++i) {
                    const int e = tid + i * kHugeThreads;
                    const int r = e / W, c = e - r * W;
                    const unsigned j = (unsigned)(st * SR + r);
                    if (j < k && c < ncols)
                        __pipeline_memcpy_async(buf + e, feats + (long long)idv[i] * D + col0 + c,
                                                sizeof(Fe));
                }
            }
            __pipeline_commit();
        };
        for (int st = 0; st < kHugeStages - 1; ++st) issue(st);
        const int mycol = wib * kHugeSlice + lane;                     // this thread's dimension
        const bool folds = wib < G && mycol < ncols;
        double sz = 0.0, sz2 = 0.0;
        for (int st = 0; st < nst; ++st) {
            issue(st + kHugeStages - 1);   // into the buffer the previous iteration consumed
            __pipeline_wait_prior(kHugeStages - 1);
            __syncthreads();
            if (folds) {
                const Fe* buf = reinterpret_cast<const Fe*>(hsm + (st % kHugeStages) * kHugeStageBytes);
                const int n = min(SR, (int)(k - (unsigned)(st * SR)));
                int r = 0;
                for (; r + 8 <= n; r += 8) {
                    double z[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) z[u] = (double)buf[(r + u) * W + mycol];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        sz += z[u];
                        sz2 = add_sq<Fe>(sz2, z[u]);
                    }
                }
                for (; r < n; ++r) {
                    const double z = (double)buf[r * W + mycol];
                    sz += z;
                    sz2 = add_sq<Fe>(sz2, z);
                }
            }
            __syncthreads();
        }
        __pipeline_wait_prior(0);
        if (folds) {
            // NIG batch update with lambda from the pre-frame weight (_pycore.py:438)
            const double nobs = (double)k;
            const double lam = fmax(hi.w_old, a.lambda_floor);
            const double lam_post = lam + nobs;
            const double coef = lam * nobs / lam_post;
            const double b_bg = (double)(TS)a.prior_beta;
            nig_apply<TS>(mean + (long long)vid * D, beta + (long long)vid * D, col0 + mycol, isnew, sz,
                          sz2, lam, lam_post, coef, nobs, b_bg);
        }
        __syncthreads();
    }
    }
    }
    frame_epilogue(ctr, ctr->p.epilogue, ctr->p.mirror);
}

__global__ void k_rehash(int64_t nblocks, const int4* __restrict__ bcoord, int4* table,
                         int64_t mask) {
    int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= nblocks) return;
    int4 c = bcoord[id];
    int64_t pos = (int64_t)(block_hash(c.x, c.y, c.z) & (uint64_t)mask);
    while (true) {
        int old = atomicCAS(&table[pos].w, kHashEmpty, kHashBusy);
        if (old == kHashEmpty) {
            table[pos] = make_int4(c.x, c.y, c.z, (int)id);
            return;
        }
        pos = (pos + 1) & mask;
    }
}

__global__ void k_fill_u64(unsigned long long* p, long long n, unsigned long long v) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        p[i] = v;
}

UpdateArgs make_args(svx_map* m) {
    UpdateArgs a;
    a.mlist = ptr<int>(m->mlist);
    a.rec = ptr<VoxFrame>(m->vrec);
    a.srid = ptr<int>(m->srid);
    a.ray = ptr<double4>(m->ray);
    a.longlist = ptr<int>(m->longlist);
    a.hugelist = ptr<int>(m->longlist) + m->ucap;
    a.hugelist2 = ptr<TouchEntry>(m->longlist);
    a.bitmap = ptr<unsigned>(m->bitmap);
    a.bm_words = (m->npts_cap + 31) / 32 + 1;
    a.h = m->cfg.voxel_size;
    a.trunc = m->cfg.truncation;
    a.wfn = m->cfg.weight_fn;
    a.sem_kind = m->cfg.sem_kind;
    a.last_wins = m->cfg.last_wins;
    a.C = m->payload_d > 0 ? m->payload_d : 1;
    a.D = m->payload_d;
    a.lambda_floor = m->cfg.lambda_floor;
    a.prior_beta = m->cfg.prior_beta;
    a.ctr = ptr<FrameCtr>(m->ctr);
    return a;
}

constexpr int kShortBlocks = 148 * 8;
#ifndef SVX_LONG_BLOCKS
#define SVX_LONG_BLOCKS (148 * 4)
#endif
constexpr int kLongBlocks = SVX_LONG_BLOCKS;

template <class TD, class TC>
svx_status scatter_t(svx_map* m, cudaStream_t s) {
    SVX_CUDA(launch_pdl(k_scatter<TD, TC>, kPersistentBlocks * 2, 256, 0, s, 
        make_args(m), ptr<int>(m->rcnt), ptr<int>(m->rowray), ptr<unsigned long long>(m->rowkey),
        ptr<int>(m->rowvid), ptr<int>(m->srid), ptr<TD>(m->vt), ptr<TC>(m->s0)));
    SVX_LAUNCHED();
    return SVX_OK;
}

template <class TD, class TC>
svx_status closed_a(svx_map* m, cudaStream_t s) {
    SVX_CUDA(launch_pdl(k_update_short<TD, TC>, kShortBlocks, 256, 0, s, make_args(m), ptr<TD>(m->vt),
                                                        ptr<TC>(m->s0)));
    SVX_LAUNCHED();
    return SVX_OK;
}

template <class TD, class TC>
svx_status closed_b(svx_map* m, cudaStream_t s) {
    SVX_CUDA(launch_pdl(k_update_long<TD, TC>, kLongBlocks, 32 * kWarpsPerCta, 0, s, make_args(m), ptr<TD>(m->vt),
                                                                    ptr<TC>(m->s0)));
    SVX_LAUNCHED();
    return SVX_OK;
}

template <class TD, class TS, class Fe>
svx_status open_a(svx_map* m, cudaStream_t s) {
    if (SVX_OPEN_PREP) {
        SVX_CUDA(launch_pdl(k_open_prep<TD>, kLongBlocks, 32 * kWarpsPerCta, 0, s, make_args(m), ptr<TD>(m->vt),
                            ptr<int>(m->srid)));
        SVX_LAUNCHED();
    }
    int ring = SVX_OPEN_RING ? kWarpsPerCta * kOpenRingS * kOpenRingR * kOpenPass * (int)sizeof(Fe) : 0;
    if (SVX_OPEN_BULK) ring = std::max(ring, kWarpsPerCta * kOpenBulkRing * kOpenGrp * kOpenPass * (int)sizeof(Fe));
    if (ring > 0) {
        SVX_CUDA(cudaFuncSetAttribute(k_update_open<TD, TS, Fe>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      ring));
        SVX_CUDA(cudaFuncSetAttribute(k_update_open<TD, TS, Fe>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                      100));
    }
    SVX_CUDA(launch_pdl(k_update_open<TD, TS, Fe>, kLongBlocks, 32 * kWarpsPerCta, ring, s, 
        make_args(m), ptr<TD>(m->vt), ptr<TS>(m->s0), ptr<TS>(m->s1)));
    SVX_LAUNCHED();
    return SVX_OK;
}

template <class TD, class TS, class Fe>
svx_status open_b(svx_map* m, cudaStream_t s) {
    // sort + TSDF of every huge voxel first, then their feature sums
    SVX_CUDA(launch_pdl(k_huge_prep<TD>, kHugeCtas, kHugeThreads, 0, s, make_args(m), ptr<TD>(m->vt),
                        ptr<HugeInfo>(m->hinfo), ptr<int>(m->srid)));
    SVX_LAUNCHED();
    const int hsmem = kHugeRingBytes;
    SVX_CUDA(cudaFuncSetAttribute(k_update_open_huge<TD, TS, Fe>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  hsmem));
    // two CTAs per SM need the largest shared-memory carveout
    SVX_CUDA(cudaFuncSetAttribute(k_update_open_huge<TD, TS, Fe>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  100));
    SVX_CUDA(launch_pdl(k_update_open_huge<TD, TS, Fe>, 148 * SVX_HUGE_MINB, kHugeThreads, hsmem, s, make_args(m),
                        ptr<TD>(m->vt), ptr<TS>(m->s0), ptr<TS>(m->s1), ptr<HugeInfo>(m->hinfo)));
    SVX_LAUNCHED();
    const int smem = kHugeStages * kHugeStageBytes;
    SVX_CUDA(cudaFuncSetAttribute(k_huge_items<TD, TS, Fe>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  smem));
    SVX_CUDA(cudaFuncSetAttribute(k_huge_items<TD, TS, Fe>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    SVX_CUDA(launch_pdl(k_huge_items<TD, TS, Fe>, kHugeItemCtas, kHugeThreads, smem, s, make_args(m),
                        ptr<TD>(m->vt), ptr<TS>(m->s0), ptr<TS>(m->s1), ptr<HugeInfo>(m->hinfo)));
    SVX_LAUNCHED();
    return SVX_OK;
}

template <class TD, class TC>
svx_status slots_t(svx_map* m, cudaStream_t s) {
    constexpr bool inl = SVX_INLINE_LONG != 0;
    SVX_CUDA(launch_pdl(k_update_slots<TD, TC, inl>, kPersistentBlocks, 256, 0, s, make_args(m),
                        ptr<TouchEntry>(m->tlist), ptr<unsigned>(m->rcount),
                        ptr<unsigned long long>(m->bslot), ptr<RowSlot>(m->vslot), ptr<TD>(m->vt),
                        ptr<TC>(m->s0)));
    SVX_LAUNCHED();
    if (!inl) {   // voxels of 9..16 rows; this kernel publishes the frame counters
        SVX_CUDA(launch_pdl(k_update_slots_long<TD, TC>, 148 * 2, 256, 0, s, make_args(m),
                            ptr<unsigned long long>(m->bslot), ptr<RowSlot>(m->vslot), ptr<TD>(m->vt),
                            ptr<TC>(m->s0)));
        SVX_LAUNCHED();
    }
    return SVX_OK;
}

template <class TD>
svx_status stage_td(svx_map* m, int feats_f64, bool b, cudaStream_t s) {
    if (m->cfg.sem_kind == SVX_SEM_OPEN) {
        const bool s64 = m->cfg.state_dtype == SVX_F64;
        if (s64) {
            if (feats_f64) return b ? open_b<TD, double, double>(m, s) : open_a<TD, double, double>(m, s);
            return b ? open_b<TD, double, float>(m, s) : open_a<TD, double, float>(m, s);
        }
        if (feats_f64) return b ? open_b<TD, float, double>(m, s) : open_a<TD, float, double>(m, s);
        return b ? open_b<TD, float, float>(m, s) : open_a<TD, float, float>(m, s);
    }
    if (m->cfg.count_dtype == SVX_F64) return b ? closed_b<TD, double>(m, s) : closed_a<TD, double>(m, s);
    return b ? closed_b<TD, float>(m, s) : closed_a<TD, float>(m, s);
}

}  // namespace

svx_status launch_scatter(svx_map* m, cudaStream_t s) {
    const bool t64 = m->cfg.tsdf_dtype == SVX_F64, c64 = m->cfg.count_dtype == SVX_F64;
    if (t64) return c64 ? scatter_t<double, double>(m, s) : scatter_t<double, float>(m, s);
    return c64 ? scatter_t<float, double>(m, s) : scatter_t<float, float>(m, s);
}

svx_status launch_update_a(svx_map* m, int feats_f64, cudaStream_t s) {
    if (m->cfg.tsdf_dtype == SVX_F64) return stage_td<double>(m, feats_f64, false, s);
    return stage_td<float>(m, feats_f64, false, s);
}

svx_status launch_update_b(svx_map* m, int feats_f64, cudaStream_t s) {
    if (m->cfg.tsdf_dtype == SVX_F64) return stage_td<double>(m, feats_f64, true, s);
    return stage_td<float>(m, feats_f64, true, s);
}

svx_status launch_update_slots(svx_map* m, cudaStream_t s) {
    const bool t64 = m->cfg.tsdf_dtype == SVX_F64, c64 = m->cfg.count_dtype == SVX_F64;
    if (t64) return c64 ? slots_t<double, double>(m, s) : slots_t<double, float>(m, s);
    return c64 ? slots_t<float, double>(m, s) : slots_t<float, float>(m, s);
}

svx_status launch_rehash(svx_map* m, int4* new_table, int64_t new_cap, cudaStream_t s) {
    const int T = 256;
    if (m->nblocks == 0) return SVX_OK;
    k_rehash<<<grid_for(m->nblocks, T), T, 0, s>>>(m->nblocks, ptr<int4>(m->bcoord), new_table,
                                                   new_cap - 1);
    SVX_LAUNCHED();
    return SVX_OK;
}

svx_status launch_fill_u64(unsigned long long* p, int64_t n, unsigned long long v, cudaStream_t s) {
    if (n <= 0) return SVX_OK;
    k_fill_u64<<<(int)std::min<int64_t>((n + 255) / 256, kPersistentBlocks), 256, 0, s>>>(p, n, v);
    SVX_LAUNCHED();
    return SVX_OK;
}

int huge_warps() { return kHugeWarps; }
size_t huge_info_bytes() { return sizeof(HugeInfo); }
int open_cta_min() { return kOpenCtaMin; }

}  // namespace svx

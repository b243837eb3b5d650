// svx_leaf.cu -- leaf mode: rows grouped by their 8^3 leaf, each touched leaf
// updated by one warp (or one CTA) out of shared memory.
//
// The reference groups a frame's rows by voxel key (sort + segments,
// _core.pyx:707-753), allocates leaves in first-occurrence order
// (ensure_coords, :377-420) and folds each voxel's rows in point order
// (:759-843, apply _pycore.py:399-429).  Leaf mode keeps the persistent
// per-voxel state of the other modes (dense voxel ids, bslot, bmask) and
// regroups only the rows:
//
//   K2L k_leaf_bin      rows -> leaf (one hash lookup per leaf per warp step,
//                       leaf find-or-insert as in K2), a per-leaf frame row
//                       count whose atomic returns the row's rank in its leaf;
//                       the leaf's first row lists the leaf
//   K3L k_leaf_alloc    per listed leaf a contiguous bin (warp scan + one
//                       atomic per warp); leaves of > kWarpRows rows go to the
//                       CTA list, > kCtaRows stop the frame (segment re-run)
//   K4L k_leaf_scatter  rows into their bins as (slot << 23 | point)
//   K5L k_leaf_update   CTAs take big leaves (counting sort by slot in shared
//                       memory), then warps take the rest (bitonic sort of the
//                       leaf's keys): each voxel's rows end up in (slot, point)
//                       order, one lane per voxel reads its id from the leaf's
//                       bslot block (new voxels get consecutive ids per leaf),
//                       folds the rows with the sequential fp64 sums of
//                       k_update_short and applies apply_tsdf / apply_closed.
//
// Per touched voxel the update reads its bslot word, TSDF pair and the count
// of each label present (no per-voxel frame records, no row slots); per row
// it reads its point's ray and label, both L2-resident.  Compiled with
// -fmad=false like the rest: distances are the same expressions as the
// walk's and the segment kernels', so the map is bit-identical.
#include <math.h>

#include <cub/block/block_scan.cuh>

#include "svx_internal.cuh"
#include "svx_resolve_tile.cuh"

namespace svx {
namespace {

constexpr int kLeafThreads = 256;
constexpr int kLeafWarps = kLeafThreads / 32;
#ifndef SVX_LEAF_WARP_ROWS
#define SVX_LEAF_WARP_ROWS 256
#endif
// Leaves of up to kWarpRows rows go to one warp, bigger ones to a whole CTA:
// a warp folds its leaf's voxels 32 at a time, so a leaf of a few hundred
// voxels would keep one warp busy for many dependent passes.
constexpr int kWarpRows = SVX_LEAF_WARP_ROWS;
constexpr int kCtaRows = 8192;         // rows a CTA sorts (more: the frame re-runs in segment mode)
constexpr unsigned kPointBits = 23;    // binned row = slot << 23 | point (n < 2^23)
constexpr unsigned kPointMask = (1u << kPointBits) - 1u;

struct LeafArgs {
    int4* table;
    int4* bcoord;
    unsigned long long* bkey;
    unsigned long long* bmask;
    unsigned long long* bslot;
    unsigned long long* lcnt;   // per leaf: frame rows (low 32), bin base (high 32); 0 between frames
    int* tleaf;                 // listed leaves of the frame
    int* lbig;                  // leaves for the CTA path
    const double4* ray;
    FrameCtr* ctr;
    double h, trunc;
    int wfn, sem_kind, last_wins, C;
};

// ---- K2L ----------------------------------------------------------------------------
// One CTA-synchronous step over kLeafThreads rows: lanes with the same leaf
// elect one lookup; claims of new leaves are ranked per step (one atomic on
// the leaf counter) exactly like K2's resolve_step.
__device__ __forceinline__ int leaf_step(const LeafArgs& a, const FrameParams& fp, bool valid,
                                         unsigned long long key, int* s_warp,
                                         unsigned long long& s_base, unsigned& lpeers_out,
                                         long long& x, long long& y, long long& z) {
    const KeyPack& kp = fp.kp;
    const int lane = threadIdx.x & 31;
    const unsigned full = 0xffffffffu;
    // No thread claims a slot in this step while another thread of its CTA
    // may still wait (previous step) on another CTA's claim: that CTA could
    // itself be held at its claim barrier by a thread waiting on ours.
    __syncthreads();
    x = y = z = 0;
    if (valid) unpack_key(key, kp, x, y, z);
    const int la = (int)(x >> kLeafLog2), lb = (int)(y >> kLeafLog2), lc = (int)(z >> kLeafLog2);
    const unsigned long long lkey =
        valid ? (((unsigned long long)(la - (kp.base[0] >> kLeafLog2)) << 38) |
                 ((unsigned long long)(lb - (kp.base[1] >> kLeafLog2)) << 19) |
                 (unsigned long long)(lc - (kp.base[2] >> kLeafLog2)))
              : (~0ULL ^ (unsigned long long)lane);
    const unsigned lpeers = __match_any_sync(full, lkey);
    const int lleader = __ffs(lpeers) - 1;
    const bool is_ll = valid && lane == lleader;
    const long long hmask = fp.hmask;
    int4* table = a.table;
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
        }
    }
    int rank = 0, cnt = 0;
    const bool lclaims = __syncthreads_or(lstate == 1);
    if (lclaims) {
        rank = rt::cta_rank<kLeafThreads>(lstate == 1, cnt, s_warp);
        if (threadIdx.x == 0) s_base = atomicAdd(&a.ctr->nblocks, (unsigned long long)cnt);
        __syncthreads();
    }
    if (lstate == 1) {
        const long long nid = (long long)s_base + rank;
        if (nid >= fp.bcap) {
            atomicExch(&table[lpos].w, kHashEmpty);
            atomicOr(&a.ctr->err_cap, 1);
        } else {
            a.bcoord[nid] = make_int4(la, lb, lc, fp.frame);
            // coordinates visible before the id is published (same-kernel
            // readers go through the published slot)
            __threadfence();
            rt::st_slot(table + lpos, make_int4(la, lb, lc, (int)nid));
            id = (int)nid;
        }
    }
    if (lclaims) __syncthreads();
    if (lstate == 2) {
        volatile int* vw = &table[lpos].w;
        int v = *vw;
        int spins = 0;
        while (v == kHashBusy) {
            __nanosleep(32);
            v = *vw;
            SVX_SPIN_GUARD(spins, a.ctr, 14)
        }
        const int4 sv = rt::ld_slot(table + lpos);
        if (v == kHashBusy) id = -1;
        else if (v >= 0 && sv.x == la && sv.y == lb && sv.z == lc) id = v;
        else id = rt::leaf_find_or_insert(table, hmask, la, lb, lc, fp.frame, fp.bcap, a.bcoord, a.ctr);
    }
    lpeers_out = lpeers;
    return __shfl_sync(full, id, lleader);
}

__global__ void __launch_bounds__(kLeafThreads, 4) k_leaf_bin(const unsigned long long* __restrict__ rowkey,
                                                              const int* __restrict__ rowray,
                                                              unsigned long long* __restrict__ rowleaf,
                                                              unsigned* __restrict__ rowpk, LeafArgs a) {
    grid_dep_wait();
    __shared__ int s_warp[kLeafWarps];
    __shared__ unsigned long long s_base;
    FrameCtr* ctr = a.ctr;
    KSpan _ks(ctr, kSpanResolve);
    __shared__ FrameCtr s_ctr_;
    snapshot_ctr(ctr, s_ctr_);
    const FrameCtr* cv = &s_ctr_;
    if (cv->abort) return;
    const FrameParams& fp = cv->p;
    const long long total = (long long)cv->rows;
    const int lane = threadIdx.x & 31;
    for (long long tile = blockIdx.x; tile * kLeafThreads < total; tile += gridDim.x) {
        const long long t = tile * kLeafThreads + threadIdx.x;
        const bool valid = t < total;
        const unsigned long long key = valid ? __ldcs(rowkey + t) : kKeyEmpty;
        const int point = valid ? __ldcs(rowray + t) : 0;
        unsigned lpeers;
        long long x, y, z;
        const int id = leaf_step(a, fp, valid, key, s_warp, s_base, lpeers, x, y, z);
        // (the warp stays converged through the shuffles and ballots below)
        const bool ok = valid && id >= 0;   // id < 0: leaf pool full, err_cap set, frame stops
        // creation stamp of a new leaf: the smallest frame key among its voxels
        const unsigned vpeers = __match_any_sync(0xffffffffu, ok ? key : (kKeyEmpty ^ (unsigned long long)lane));
        if (ok && lane == __ffs(vpeers) - 1 && id >= fp.nblocks0) atomicMin(&a.bkey[id], key);
        const int lleader = __ffs(lpeers) - 1;
        unsigned base = 0;
        if (ok && lane == lleader) base = (unsigned)atomicAdd(&a.lcnt[id], (unsigned long long)__popc(lpeers));
        // the leaf's first rows this frame list it (one atomic per warp)
        const bool lst = ok && lane == lleader && base == 0u;
        const unsigned lb = __ballot_sync(0xffffffffu, lst);
        unsigned long long lpos = 0;
        if (lb && lane == __ffs(lb) - 1) lpos = atomicAdd(&ctr->n_leaves, (unsigned long long)__popc(lb));
        lpos = __shfl_sync(0xffffffffu, lpos, lb ? __ffs(lb) - 1 : 0);
        if (lst) a.tleaf[lpos + __popc(lb & ((1u << lane) - 1u))] = id;
        base = __shfl_sync(0xffffffffu, base, lleader);
        if (!valid) continue;
        if (!ok) {
            rowleaf[t] = ~0ULL;
            continue;
        }
        const unsigned rank = base + __popc(lpeers & ((1u << lane) - 1u));
        rowleaf[t] = ((unsigned long long)(unsigned)id << 32) | rank;
        rowpk[t] = ((unsigned)rt::slot_of(x, y, z) << kPointBits) | (unsigned)point;
    }
}

// ---- K3L ----------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_leaf_alloc(LeafArgs a) {
    grid_dep_wait();
    FrameCtr* ctr = a.ctr;
    KSpan _ks(ctr, kSpanSeg);
    __shared__ FrameCtr s_ctr_;
    snapshot_ctr(ctr, s_ctr_);
    const FrameCtr* cv = &s_ctr_;
    if (cv->abort | cv->err_cap) return;
    const long long L = (long long)cv->n_leaves;
    const int lane = threadIdx.x & 31;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long e0 = (long long)blockIdx.x * blockDim.x; e0 < L; e0 += stride) {
        const long long e = e0 + threadIdx.x;
        const bool has = e < L;
        const int id = has ? a.tleaf[e] : 0;
        const unsigned c = has ? (unsigned)a.lcnt[id] : 0u;
        if (c > (unsigned)kCtaRows) ctr->err_slots = 1;   // re-run in segment mode
        unsigned incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        unsigned long long wb = 0;
        const unsigned tot = __shfl_sync(0xffffffffu, incl, 31);
        if (lane == 31 && tot) wb = atomicAdd(&ctr->bin_cursor, (unsigned long long)tot);
        wb = __shfl_sync(0xffffffffu, wb, 31);
        if (has) reinterpret_cast<unsigned*>(a.lcnt + id)[1] = (unsigned)(wb + incl - c);
        const bool big = has && c > (unsigned)kWarpRows;
        const unsigned bb = __ballot_sync(0xffffffffu, big);
        unsigned long long bpos = 0;
        if (bb && lane == __ffs(bb) - 1) bpos = atomicAdd(&ctr->n_bigleaf, (unsigned long long)__popc(bb));
        bpos = __shfl_sync(0xffffffffu, bpos, bb ? __ffs(bb) - 1 : 0);
        if (big) a.lbig[bpos + __popc(bb & ((1u << lane) - 1u))] = id;
    }
}

// ---- K4L ----------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_leaf_scatter(const unsigned long long* __restrict__ rowleaf,
                                                      const unsigned* __restrict__ rowpk,
                                                      unsigned* __restrict__ binrow, LeafArgs a) {
    grid_dep_wait();
    FrameCtr* ctr = a.ctr;
    KSpan _ks(ctr, kSpanScatter);
    __shared__ FrameCtr s_ctr_;
    snapshot_ctr(ctr, s_ctr_);
    const FrameCtr* cv = &s_ctr_;
    if (cv->abort | cv->err_cap | cv->err_slots) return;
    const long long total = (long long)cv->rows;
    const unsigned* lbase = reinterpret_cast<const unsigned*>(a.lcnt);
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const unsigned long long rl = __ldcs(rowleaf + t);
        const unsigned id = (unsigned)(rl >> 32);
        const unsigned base = __ldcg(lbase + 2 * (size_t)id + 1);
        binrow[base + (unsigned)rl] = __ldcs(rowpk + t);
    }
}

// ---- K5L ----------------------------------------------------------------------------

__device__ __forceinline__ double4 ldg_ray(const double4* p) {
    const double2* q = reinterpret_cast<const double2*>(p);
    const double2 u = __ldg(q), v = __ldg(q + 1);
    return make_double4(u.x, u.y, v.x, v.y);
}

// Fold one voxel's rows (points in ascending order) and apply the update:
// the sums of k_update_short (_core.pyx:759-843), apply_tsdf (_pycore.py:
// 399-417), apply_closed (:420-429).
template <class TD, class TC, class GetPoint>
__device__ __forceinline__ void fold_voxel(const LeafArgs& a, const FrameParams& fp, int4 lc, int slot,
                                           int k, GetPoint&& pt, int vid, bool isnew, TD* vt,
                                           TC* counts) {
    using P2 = typename Pair<TD>::type;
    P2 st = isnew ? P2{(TD)a.trunc, (TD)0} : reinterpret_cast<const P2*>(vt)[vid];
    const long long x = (long long)lc.x * 8 + (slot >> 6), y = (long long)lc.y * 8 + ((slot >> 3) & 7),
                    z = (long long)lc.z * 8 + (slot & 7);
    const double cx = ((double)x + 0.5) * a.h - fp.pp.t[0];
    const double cy = ((double)y + 0.5) * a.h - fp.pp.t[1];
    const double cz = ((double)z + 0.5) * a.h - fp.pp.t[2];
    const bool closed = a.sem_kind == SVX_SEM_CLOSED;
    TC* crow = counts + (long long)vid * a.C;
    double sw = 0.0, swd = 0.0, mind = INFINITY, maxd = -INFINITY;
    int last = 0;
#pragma unroll 4
    for (int j = 0; j < k; ++j) {
        const int p = pt(j);
        const double4 r = ldg_ray(a.ray + p);   // read-only: loads of later rows can issue early
        const double proj = cx * r.x + cy * r.y + cz * r.z;
        double d = r.w - proj;
        if (d < -a.trunc) d = -a.trunc;
        if (d > a.trunc) d = a.trunc;
        const double w = (a.wfn == 1) ? (d >= 0.0 ? 1.0 : (a.trunc + d) / a.trunc) : 1.0;
        sw += w;
        swd += w * d;
        mind = d < mind ? d : mind;
        maxd = d > maxd ? d : maxd;
        if (closed) {
            const int lab = __ldg(fp.labels + p);
            if (a.last_wins) last = lab;
            else atomicAdd(&crow[lab - 1], (TC)1);   // integer-valued count: order-free
        }
    }
    const double w_old = (double)st.y, d_old = (double)st.x;
    const double w_new = w_old + sw;
    double d_new = w_new > 0.0 ? (w_old * d_old + swd) / w_new : d_old;
    if ((mind == maxd) && (w_old == 0.0 || st.x == (TD)mind)) d_new = mind;
    P2 out;
    out.x = (TD)d_new;
    out.y = (TD)w_new;
    reinterpret_cast<P2*>(vt)[vid] = out;
    if (closed && a.last_wins)
        for (int q = 0; q < a.C; ++q) crow[q] = (TC)(q == last - 1 ? 1 : 0);
}

// Ascending insertion sort of a voxel's point indices (a handful of rows).
__device__ __forceinline__ void sort_points(unsigned* p, int k) {
    for (int i = 1; i < k; ++i) {
        const unsigned v = p[i];
        int j = i - 1;
        while (j >= 0 && p[j] > v) {
            p[j + 1] = p[j];
            --j;
        }
        p[j + 1] = v;
    }
}

// Shared memory of K5L.  Both paths counting-sort the leaf's rows by slot
// (binned rows are read twice from L2: histogram, then scatter), so only the
// point indices are kept.  Warp path: 16-bit per-slot counts packed in pairs
// (one 32-bit atomic per row), the list of the leaf's voxels (slots).
struct alignas(16) LeafSmem {
    union {
        struct {   // CTA path
            unsigned pts[kCtaRows];
            unsigned cnt[kLeafVolume];   // counts, then ends
        } c;
        struct {   // warp path, per warp
            unsigned pts[kLeafWarps][kWarpRows];
            unsigned cnt2[kLeafWarps][kLeafVolume / 2];   // two 16-bit counts per word
            unsigned short vox[kLeafWarps][kLeafVolume];
        } w;
    };
};

__device__ __forceinline__ unsigned cnt16(const unsigned* c2, int s) {
    return (c2[s >> 1] >> ((s & 1) * 16)) & 0xFFFFu;
}

#ifndef SVX_LEAF_UPD_MINB
#define SVX_LEAF_UPD_MINB 4   // CTAs per SM (64 registers; 3 = 80 registers, no spills)
#endif
template <class TD, class TC>
__global__ void __launch_bounds__(kLeafThreads, SVX_LEAF_UPD_MINB) k_leaf_update(const unsigned* __restrict__ binrow, LeafArgs a,
                                                              TD* vt, TC* counts) {
    grid_dep_wait();
    FrameCtr* ctr = a.ctr;
    {
    KSpan _ks(ctr, kSpanUpdate);
    __shared__ FrameCtr s_ctr_;
    snapshot_ctr(ctr, s_ctr_);
    const FrameCtr* cv = &s_ctr_;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    LeafSmem& S = *reinterpret_cast<LeafSmem*>(smem_raw);
    __shared__ long long s_item;
    __shared__ int s_warp[kLeafWarps];
    __shared__ unsigned long long s_vbase;
    __shared__ unsigned s_touched;
    if (!(cv->abort | cv->err_cap | cv->err_slots)) {
    const FrameParams& fp = cv->p;
    const long long vcap = fp.vcap;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned touched = 0;   // voxels this thread (lane) finished
    // -- CTA path: leaves of kWarpRows+1 .. kCtaRows rows ----------------------------
    const long long NB = (long long)cv->n_bigleaf;
    while (true) {
        if (threadIdx.x == 0) s_item = (long long)atomicAdd(&ctr->work_huge, 1ULL);
        __syncthreads();
        const long long e = s_item;
        if (e >= NB) break;
        const int id = a.lbig[e];
        const unsigned long long lw = a.lcnt[id];
        const unsigned c = (unsigned)lw, base = (unsigned)(lw >> 32);
        const int4 lc = a.bcoord[id];
        for (int s = threadIdx.x; s < kLeafVolume; s += kLeafThreads) S.c.cnt[s] = 0u;
        __syncthreads();
        for (unsigned j = threadIdx.x; j < c; j += kLeafThreads)
            atomicAdd(&S.c.cnt[__ldcg(binrow + base + j) >> kPointBits], 1u);
        __syncthreads();
        unsigned k2[2];
        {   // exclusive scan of the 512 slot counts (2 per thread) -> slot starts
            using Scan = cub::BlockScan<unsigned, kLeafThreads>;
            __shared__ typename Scan::TempStorage scan_tmp;
            k2[0] = S.c.cnt[2 * threadIdx.x];
            k2[1] = S.c.cnt[2 * threadIdx.x + 1];
            unsigned o2[2];
            Scan(scan_tmp).ExclusiveSum(k2, o2);
            __syncthreads();
            S.c.cnt[2 * threadIdx.x] = o2[0];
            S.c.cnt[2 * threadIdx.x + 1] = o2[1];
        }
        __syncthreads();
        for (unsigned j = threadIdx.x; j < c; j += kLeafThreads) {   // cursors advance to the slot ends
            const unsigned v = __ldcs(binrow + base + j);
            S.c.pts[atomicAdd(&S.c.cnt[v >> kPointBits], 1u)] = v & kPointMask;
        }
        __syncthreads();
        // voxels: slots 2*tid, 2*tid+1; new ones get consecutive ids
        int vidv[2];
        bool newv[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int s = 2 * threadIdx.x + q;
            vidv[q] = -1;
            if (k2[q]) vidv[q] = (int)(unsigned)a.bslot[(long long)id * kLeafVolume + s];
            newv[q] = k2[q] && vidv[q] < 0;
        }
        {
            int tot = 0, tot1 = 0;
            const int r0 = rt::cta_rank<kLeafThreads>(newv[0], tot, s_warp);
            __syncthreads();
            const int r1 = rt::cta_rank<kLeafThreads>(newv[1], tot1, s_warp);
            if (threadIdx.x == 0 && tot + tot1) s_vbase = atomicAdd(&ctr->nvox, (unsigned long long)(tot + tot1));
            __syncthreads();
            if (newv[0]) vidv[0] = (int)(s_vbase + r0);
            if (newv[1]) vidv[1] = (int)(s_vbase + tot + r1);
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            if (!k2[q]) continue;
            const int s = 2 * threadIdx.x + q;
            const int k = (int)k2[q];
            unsigned* pp = S.c.pts + (S.c.cnt[s] - k2[q]);
            sort_points(pp, k);
            if ((long long)vidv[q] >= vcap) {
                ctr->err_internal = 1;
                continue;
            }
            if (newv[q]) {
                a.bslot[(long long)id * kLeafVolume + s] = (unsigned long long)(unsigned)vidv[q];
                atomicOr(&a.bmask[(long long)id * kMaskWords + (s >> 6)], 1ULL << (s & 63));
            }
            fold_voxel<TD, TC>(a, fp, lc, s, k, [&](int j) { return (int)pp[j]; }, vidv[q], newv[q], vt,
                               counts);
            ++touched;
        }
        __syncthreads();
        if (threadIdx.x == 0) a.lcnt[id] = 0ULL;
    }
    // -- warp path: leaves of <= kWarpRows rows ---------------------------------------
    const long long L = (long long)cv->n_leaves;
    unsigned* pts = S.w.pts[warp];
    unsigned* cnt2 = S.w.cnt2[warp];
    unsigned short* vox = S.w.vox[warp];
    while (true) {
        unsigned long long e = 0;
        if (lane == 0) e = atomicAdd(&ctr->work_long, 1ULL);
        e = __shfl_sync(0xffffffffu, e, 0);
        if ((long long)e >= L) break;
        const int id = a.tleaf[e];
        const unsigned long long lw = a.lcnt[id];
        const unsigned c = (unsigned)lw, base = (unsigned)(lw >> 32);
        if (c > (unsigned)kWarpRows) continue;   // the CTA path's
        const int4 lc = a.bcoord[id];
#pragma unroll
        for (int q = 0; q < kLeafVolume / 64; ++q) cnt2[lane + 32 * q] = 0u;
        __syncwarp();
        for (unsigned j = lane; j < c; j += 32) {
            const unsigned s = __ldcg(binrow + base + j) >> kPointBits;
            atomicAdd(&cnt2[s >> 1], (s & 1u) ? 0x10000u : 1u);
        }
        __syncwarp();
        // lane owns slots 16*lane .. 16*lane+15: local counts, a warp scan of
        // rows and of voxels, then slot starts written back (16-bit) and the
        // lane's voxels appended to the list in slot order
        unsigned cl[16];
        unsigned rows_l = 0, vox_l = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const unsigned w2 = cnt2[8 * lane + q];
            cl[2 * q] = w2 & 0xFFFFu;
            cl[2 * q + 1] = w2 >> 16;
            rows_l += cl[2 * q] + cl[2 * q + 1];
            vox_l += (cl[2 * q] != 0u) + (cl[2 * q + 1] != 0u);
        }
        unsigned r_incl = rows_l, v_incl = vox_l;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned rr = __shfl_up_sync(0xffffffffu, r_incl, o);
            const unsigned vv = __shfl_up_sync(0xffffffffu, v_incl, o);
            if (lane >= o) {
                r_incl += rr;
                v_incl += vv;
            }
        }
        const int nv = (int)__shfl_sync(0xffffffffu, v_incl, 31);
        unsigned off = r_incl - rows_l, vo = v_incl - vox_l;
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 8; ++q) {   // slot starts (16-bit) overwrite the counts
            const unsigned lo = off, hi = off + cl[2 * q];
            off = hi + cl[2 * q + 1];
            cnt2[8 * lane + q] = lo | (hi << 16);
        }
#pragma unroll
        for (int q = 0; q < 16; ++q)
            if (cl[q]) vox[vo++] = (unsigned short)(16 * lane + q);
        __syncwarp();
        for (unsigned j = lane; j < c; j += 32) {   // starts advance to the slot ends
            const unsigned v = __ldcs(binrow + base + j);
            const unsigned s = v >> kPointBits;
            const unsigned old = atomicAdd(&cnt2[s >> 1], (s & 1u) ? 0x10000u : 1u);
            pts[(old >> ((s & 1u) * 16)) & 0xFFFFu] = v & kPointMask;
        }
        __syncwarp();
        for (int v0 = 0; v0 < nv; v0 += 32) {
            const int v = v0 + lane;
            const bool has = v < nv;
            int slot = 0, vid = -1, k = 0;
            unsigned* pp = pts;
            if (has) {
                slot = vox[v];
                vid = (int)(unsigned)a.bslot[(long long)id * kLeafVolume + slot];
                const unsigned end = cnt16(cnt2, slot);
                const unsigned st0 = slot ? cnt16(cnt2, slot - 1) : 0u;
                // (an empty slot's end equals its start; the previous slot's end
                // is this slot's start)
                k = (int)(end - st0);
                pp = pts + st0;
            }
            const bool isnew = has && vid < 0;
            const unsigned nb = __ballot_sync(0xffffffffu, isnew);
            unsigned long long vb = 0;
            if (nb && lane == __ffs(nb) - 1) vb = atomicAdd(&ctr->nvox, (unsigned long long)__popc(nb));
            if (nb) vb = __shfl_sync(0xffffffffu, vb, __ffs(nb) - 1);
            if (isnew) vid = (int)(vb + __popc(nb & ((1u << lane) - 1u)));
            if (!has) continue;
            sort_points(pp, k);
            if ((long long)vid >= vcap) {
                ctr->err_internal = 1;
                continue;
            }
            if (isnew) {
                a.bslot[(long long)id * kLeafVolume + slot] = (unsigned long long)(unsigned)vid;
                atomicOr(&a.bmask[(long long)id * kMaskWords + (slot >> 6)], 1ULL << (slot & 63));
            }
            fold_voxel<TD, TC>(a, fp, lc, slot, k, [&](int j) { return (int)pp[j]; }, vid, isnew, vt, counts);
            ++touched;
        }
        __syncwarp();
        if (lane == 0) a.lcnt[id] = 0ULL;
    }
    // touched voxels of the frame (report)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) touched += __shfl_xor_sync(0xffffffffu, touched, o);
    if (threadIdx.x == 0) s_touched = 0u;
    __syncthreads();
    if (lane == 0 && touched) atomicAdd(&s_touched, touched);
    __syncthreads();
    if (threadIdx.x == 0 && s_touched) atomicAdd(&ctr->n_touched, (unsigned long long)s_touched);
    }
    }
    frame_epilogue(ctr, ctr->p.epilogue, ctr->p.mirror);
}

// After an aborted leaf-mode attempt (leaf pool full, or a leaf too big for
// shared memory): no voxel changed; the listed leaves' frame counts go back
// to zero.
__global__ void k_leaf_cleanup(long long n, const int* __restrict__ tleaf, unsigned long long* lcnt) {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x)
        lcnt[tleaf[e]] = 0ULL;
}

LeafArgs leaf_args(svx_map* m) {
    LeafArgs a;
    a.table = ptr<int4>(m->hash);
    a.bcoord = ptr<int4>(m->bcoord);
    a.bkey = ptr<unsigned long long>(m->bkey);
    a.bmask = ptr<unsigned long long>(m->bmask);
    a.bslot = ptr<unsigned long long>(m->bslot);
    a.lcnt = ptr<unsigned long long>(m->lcnt);
    a.tleaf = ptr<int>(m->tlist);
    a.lbig = ptr<int>(m->longlist);
    a.ray = ptr<double4>(m->ray);
    a.ctr = ptr<FrameCtr>(m->ctr);
    a.h = m->cfg.voxel_size;
    a.trunc = m->cfg.truncation;
    a.wfn = m->cfg.weight_fn;
    a.sem_kind = m->cfg.sem_kind;
    a.last_wins = m->cfg.last_wins;
    a.C = m->payload_d > 0 ? m->payload_d : 1;
    return a;
}

template <class TD, class TC>
svx_status leaf_t(svx_map* m, cudaStream_t s) {
    const LeafArgs a = leaf_args(m);
    SVX_CUDA(launch_pdl(k_leaf_bin, kPersistentBlocks, kLeafThreads, 0, s, ptr<unsigned long long>(m->rowkey),
                        ptr<int>(m->rowray), ptr<unsigned long long>(m->rowleaf), ptr<unsigned>(m->rowpk), a));
    SVX_LAUNCHED();
    SVX_CUDA(launch_pdl(k_leaf_alloc, 148 * 2, 256, 0, s, a));
    SVX_LAUNCHED();
    SVX_CUDA(launch_pdl(k_leaf_scatter, kPersistentBlocks, 256, 0, s, ptr<unsigned long long>(m->rowleaf),
                        ptr<unsigned>(m->rowpk), ptr<unsigned>(m->binrow), a));
    SVX_LAUNCHED();
    const int smem = (int)sizeof(LeafSmem);
    SVX_CUDA(cudaFuncSetAttribute(k_leaf_update<TD, TC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    SVX_CUDA(launch_pdl(k_leaf_update<TD, TC>, 148 * SVX_LEAF_UPD_MINB, kLeafThreads, smem, s, ptr<unsigned>(m->binrow), a,
                        ptr<TD>(m->vt), ptr<TC>(m->s0)));
    SVX_LAUNCHED();
    return SVX_OK;
}

}  // namespace

svx_status launch_leaf(svx_map* m, cudaStream_t s) {
    const bool t64 = m->cfg.tsdf_dtype == SVX_F64, c64 = m->cfg.count_dtype == SVX_F64;
    if (t64) return c64 ? leaf_t<double, double>(m, s) : leaf_t<double, float>(m, s);
    return c64 ? leaf_t<float, double>(m, s) : leaf_t<float, float>(m, s);
}

svx_status launch_leaf_cleanup(svx_map* m, cudaStream_t s) {
    const long long n = (long long)m->h_ctr->n_leaves;
    if (n <= 0) return SVX_OK;
    k_leaf_cleanup<<<grid_for(n, 256) < kPersistentBlocks ? grid_for(n, 256) : kPersistentBlocks, 256, 0, s>>>(
        n, ptr<int>(m->tlist), ptr<unsigned long long>(m->lcnt));
    SVX_LAUNCHED();
    return SVX_OK;
}

bool leaf_mode_fits(int64_t n) { return n < (int64_t)(1u << kPointBits); }

}  // namespace svx

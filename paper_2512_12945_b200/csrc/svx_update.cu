// svx_update.cu -- leaf allocation (K4) and the fused TSDF + semantic update
// (K5/K6).
//
// Compiled with -fmad=false.  Every voxel's rows are put back into point
// order (the reference's (voxel, point, step) order) and reduced
// sequentially in fp64 exactly like _core.pyx:759-843; the apply arithmetic
// restates apply_tsdf / apply_closed / apply_open (_pycore.py:399-446)
// operation for operation, so stored values round identically.
//
// Segment lengths decide the execution shape:
//   short  (<= kShortMax rows)   one thread per voxel, register insertion sort
//   long   (<= kSmemMax rows)    one warp per voxel, shared-memory bitonic sort
//   huge   (> kSmemMax rows)     one warp per voxel, point-index bitmap in global
//                                scratch streamed in ascending chunks (space
//                                carving sends every ray through the origin voxel)
// Open-set voxels always take the warp shapes (lanes own feature dimensions).
#include <math.h>

#include "svx_internal.cuh"

namespace svx {
namespace {

constexpr int kSmemMax = 1024;                   // rows per warp buffer (4 KB)
constexpr int kWarpsPerCta = 8;
constexpr int kHugeWarps = 128;                  // warps that share the bitmap scratch

__device__ __forceinline__ int slot_of(long long x, long long y, long long z) {
    return (int)(((x & 7) << 6) | ((y & 7) << 3) | (z & 7));
}

__device__ __forceinline__ bool frame_aborted(const FrameCtr* ctr) {
    return *(volatile const int*)&ctr->abort != 0;
}

// counter += 1 for every converged lane, one atomic per warp; returns this
// lane's ticket.
__device__ __forceinline__ unsigned long long warp_aggregate_add(unsigned long long* counter,
                                                                 unsigned long long /*one*/) {
    const unsigned mask = __activemask();
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(mask) - 1;
    const unsigned rank = __popc(mask & ((1u << lane) - 1u));
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(counter, (unsigned long long)__popc(mask));
    base = __shfl_sync(mask, base, leader);
    return base + rank;
}

// Leaf find-or-insert.  A claimed slot stays BUSY until the new leaf's id,
// coordinates and creation frame are written; then the id is published.
__device__ int leaf_find_or_insert(int4* table, long long mask, int a, int b, int c, int frame,
                                   int4* bcoord, FrameCtr* ctr) {
    long long pos = (long long)(block_hash(a, b, c) & (unsigned long long)mask);
    while (true) {
        volatile int* vw = &table[pos].w;
        int v = *vw;
        if (v == kHashEmpty) {
            int old = atomicCAS((int*)&table[pos].w, kHashEmpty, kHashBusy);
            if (old == kHashEmpty) {
                table[pos].x = a;
                table[pos].y = b;
                table[pos].z = c;
                int id = (int)warp_aggregate_add(&ctr->nblocks, 1ULL);
                bcoord[id] = make_int4(a, b, c, frame);
                __threadfence();
                atomicExch((int*)&table[pos].w, id);
                return id;
            }
            v = old;
        }
        while (v == kHashBusy) {
            __nanosleep(20);
            v = *vw;
        }
        __threadfence();
        volatile int* key = &table[pos].x;
        if (key[0] == a && key[1] == b && key[2] == c) return v;
        pos = (pos + 1) & mask;
    }
}

// K4: per touched voxel -- leaf lookup/allocation, creation stamp for leaves
// created this frame (their first-occurrence key), voxel activation.
__global__ void __launch_bounds__(256) k_voxels(
    const int* __restrict__ ulist, const unsigned long long* __restrict__ ukey, KeyPack kp,
    int4* table, long long hmask, int frame, int4* bcoord, unsigned long long* bkey,
    unsigned long long* bmask, int* bslot, int* __restrict__ gvid, FrameCtr* ctr) {
    if (frame_aborted(ctr)) return;
    const long long U = (long long)ctr->n_groups;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < U;
         i += (long long)gridDim.x * blockDim.x) {
        const unsigned long long key = ukey[i];
        long long x, y, z;
        unpack_key(key, kp, x, y, z);
        const int id = leaf_find_or_insert(table, hmask, (int)(x >> kLeafLog2),
                                           (int)(y >> kLeafLog2), (int)(z >> kLeafLog2), frame,
                                           bcoord, ctr);
        if (__ldcg(&bcoord[id].w) == frame) atomicMin(&bkey[id], key);
        const int slot = slot_of(x, y, z);
        int* sp = &bslot[(long long)id * kLeafVolume + slot];
        int vid = *sp;
        int isnew = vid < 0;
        if (isnew) {
            vid = (int)warp_aggregate_add(&ctr->nvox, 1ULL);
            *sp = vid;
            atomicOr(&bmask[(long long)id * kMaskWords + (slot >> 6)], 1ULL << (slot & 63));
        }
        gvid[i] = vid | (isnew ? (int)0x80000000 : 0);
    }
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

// apply_tsdf (_pycore.py:399-417) for one voxel; returns w_old.
template <class TD>
__device__ __forceinline__ double apply_tsdf(TD* vd, TD* vw, int vid, bool isnew, double trunc,
                                             double sw, double swd, double mind, double maxd) {
    TD d_st = isnew ? (TD)trunc : vd[vid];
    TD w_st = isnew ? (TD)0 : vw[vid];
    double w_old = (double)w_st;
    double d_old = (double)d_st;
    double w_new = w_old + sw;
    double d_new = w_new > 0.0 ? (w_old * d_old + swd) / w_new : d_old;
    bool cst = (mind == maxd) && (w_old == 0.0 || equals_stored<TD>(d_st, mind));
    if (cst) d_new = mind;
    vd[vid] = (TD)d_new;
    vw[vid] = (TD)w_new;
    return w_old;
}

struct Center {
    double x, y, z;
};

__device__ __forceinline__ Center voxel_center(unsigned long long key, const KeyPack& kp, double h,
                                               const PoseParams& pp) {
    long long x, y, z;
    unpack_key(key, kp, x, y, z);
    Center c;
    c.x = ((double)x + 0.5) * h - pp.t[0];
    c.y = ((double)y + 0.5) * h - pp.t[1];
    c.z = ((double)z + 0.5) * h - pp.t[2];
    return c;
}

__device__ __forceinline__ void clear_frame_slot(unsigned long long* fkey, unsigned* fcount,
                                                 unsigned* fcur, int s) {
    fkey[s] = kKeyEmpty;
    fcount[s] = 0u;
    fcur[s] = 0u;
}

struct UpdateArgs {
    const int* ulist;
    const unsigned long long* ukey;
    const int* gvid;
    unsigned long long* fkey;
    unsigned* fcount;
    const unsigned* foff;
    unsigned* fcur;
    const int* srid;
    const double4* ray;
    int* longlist;
    int* hugelist;
    unsigned* bitmap;     // kHugeWarps * bm_words
    long long bm_words;
    KeyPack kp;
    PoseParams pp;
    double h, trunc;
    int wfn;
    // closed
    int sem_kind, last_wins, C;
    const int32_t* labels;
    // open
    int D;
    double lambda_floor, prior_beta;
    FrameCtr* ctr;
};

// ---- short segments: one thread per voxel -------------------------------------

template <class TD, class TC>
__global__ void __launch_bounds__(256) k_update_short(UpdateArgs a, TD* vd, TD* vw, TC* counts) {
    if (frame_aborted(a.ctr)) return;
    const long long U = (long long)a.ctr->n_groups;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < U;
         i += (long long)gridDim.x * blockDim.x) {
        const int s = a.ulist[i];
        const unsigned k = a.fcount[s];
        if (k > (unsigned)kShortMax) {
            if (k > (unsigned)kSmemMax) a.hugelist[warp_aggregate_add(&a.ctr->n_huge, 1ULL)] = (int)i;
            else a.longlist[warp_aggregate_add(&a.ctr->n_long, 1ULL)] = (int)i;
            continue;
        }
        const unsigned base = a.foff[s];
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
        const Center c = voxel_center(a.ukey[i], a.kp, a.h, a.pp);
        const int g = a.gvid[i];
        const int vid = g & 0x7fffffff;
        const bool isnew = g < 0;
        double sw = 0.0, swd = 0.0, mind = INFINITY, maxd = -INFINITY;
        int last_lab = 0;
        TC* crow = counts + (long long)vid * a.C;
        for (unsigned j = 0; j < k; ++j) {
            const int rid = r[j];
            double d, w;
            row_dw(c.x, c.y, c.z, a.ray[rid], a.trunc, a.wfn, d, w);
            sw += w;
            swd += w * d;
            mind = d < mind ? d : mind;
            maxd = d > maxd ? d : maxd;
            if (a.sem_kind == SVX_SEM_CLOSED) {
                const int lab = a.labels[rid];
                if (a.last_wins) last_lab = lab;
                else crow[lab - 1] += (TC)1;
            }
        }
        apply_tsdf<TD>(vd, vw, vid, isnew, a.trunc, sw, swd, mind, maxd);
        if (a.sem_kind == SVX_SEM_CLOSED && a.last_wins) {
            for (int q = 0; q < a.C; ++q) crow[q] = (TC)(q == last_lab - 1 ? 1 : 0);
        }
        clear_frame_slot(a.fkey, a.fcount, a.fcur, s);
    }
}

// ---- warp helpers ---------------------------------------------------------------

// Sort one segment's point indices ascending into buf (k <= kSmemMax).
__device__ __forceinline__ int warp_sort_segment(const int* __restrict__ srid, unsigned base, int k,
                                                 int* buf) {
    const int lane = threadIdx.x & 31;
    int P = 32;
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
    return k;
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

// Build the point bitmap of a huge segment in this warp's scratch; returns
// (minr, nwords).
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
__device__ __forceinline__ void warp_tsdf_chunk(const UpdateArgs& a, const int* buf, int cnt,
                                                const Center& c, TsdfAcc& acc, TC* crow,
                                                bool count_labels) {
    const int lane = threadIdx.x & 31;
    for (int c0 = 0; c0 < cnt; c0 += 32) {
        const int j = c0 + lane;
        double d = 0.0, w = 0.0;
        int lab = 0;
        if (j < cnt) {
            const int rid = buf[j];
            row_dw(c.x, c.y, c.z, a.ray[rid], a.trunc, a.wfn, d, w);
            if (count_labels) {
                lab = a.labels[rid];
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
__device__ __forceinline__ void finish_closed(const UpdateArgs& a, TD* vd, TD* vw, TC* crow, int vid,
                                              bool isnew, const TsdfAcc& acc) {
    const int lane = threadIdx.x & 31;
    if (lane == 0) apply_tsdf<TD>(vd, vw, vid, isnew, a.trunc, acc.sw, acc.swd, acc.mind, acc.maxd);
    if (a.sem_kind == SVX_SEM_CLOSED && a.last_wins) {
        for (int q = lane; q < a.C; q += 32) crow[q] = (TC)(q == acc.last_lab - 1 ? 1 : 0);
    }
}

// ---- long segments (TSDF / closed): one warp per voxel ---------------------------

template <class TD, class TC>
__global__ void __launch_bounds__(32 * kWarpsPerCta) k_update_long(UpdateArgs a, TD* vd, TD* vw,
                                                                   TC* counts) {
    __shared__ int sbuf[kWarpsPerCta][kSmemMax];
    if (frame_aborted(a.ctr)) return;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    int* buf = sbuf[wib];
    const long long L = (long long)a.ctr->n_long;
    for (long long t = (long long)blockIdx.x * kWarpsPerCta + wib; t < L;
         t += (long long)gridDim.x * kWarpsPerCta) {
        const int i = a.longlist[t];
        const int s = a.ulist[i];
        const unsigned k = a.fcount[s];
        warp_sort_segment(a.srid, a.foff[s], (int)k, buf);
        const Center c = voxel_center(a.ukey[i], a.kp, a.h, a.pp);
        const int g = a.gvid[i];
        const int vid = g & 0x7fffffff;
        TC* crow = counts + (long long)vid * a.C;
        TsdfAcc acc{0.0, 0.0, INFINITY, -INFINITY, 0};
        warp_tsdf_chunk<TC>(a, buf, (int)k, c, acc, crow, a.sem_kind == SVX_SEM_CLOSED);
        finish_closed<TD, TC>(a, vd, vw, crow, vid, g < 0, acc);
        if (lane == 0) clear_frame_slot(a.fkey, a.fcount, a.fcur, s);
        __syncwarp();
    }
}

// ---- huge segments (TSDF / closed): bitmap-ordered streaming --------------------

template <class TD, class TC>
__global__ void __launch_bounds__(32 * kWarpsPerCta) k_update_huge(UpdateArgs a, TD* vd, TD* vw,
                                                                   TC* counts) {
    __shared__ int sbuf[kWarpsPerCta][kSmemMax];
    if (frame_aborted(a.ctr)) return;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    int* buf = sbuf[wib];
    const long long gw = (long long)blockIdx.x * kWarpsPerCta + wib;
    unsigned* bm = a.bitmap + gw * a.bm_words;
    const long long Hn = (long long)a.ctr->n_huge;
    for (long long t = gw; t < Hn; t += (long long)gridDim.x * kWarpsPerCta) {
        const int i = a.hugelist[t];
        const int s = a.ulist[i];
        const unsigned k = a.fcount[s];
        int minr;
        long long nwords;
        bitmap_build(a.srid, a.foff[s], k, bm, minr, nwords);
        const Center c = voxel_center(a.ukey[i], a.kp, a.h, a.pp);
        const int g = a.gvid[i];
        const int vid = g & 0x7fffffff;
        TC* crow = counts + (long long)vid * a.C;
        TsdfAcc acc{0.0, 0.0, INFINITY, -INFINITY, 0};
        for (long long w0 = 0; w0 < nwords; w0 += 32) {
            const int cnt = bitmap_chunk(bm, w0, nwords, minr, buf);
            if (cnt) warp_tsdf_chunk<TC>(a, buf, cnt, c, acc, crow, a.sem_kind == SVX_SEM_CLOSED);
            __syncwarp();
        }
        finish_closed<TD, TC>(a, vd, vw, crow, vid, g < 0, acc);
        if (lane == 0) clear_frame_slot(a.fkey, a.fcount, a.fcur, s);
        __syncwarp();
    }
}

// ---- open set: one warp per voxel, lanes own feature dimensions ------------------

constexpr int kOpenPer = 8;   // dims per lane per pass (256 dims per pass)

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

// Per-dimension sequential sums over an ordered chunk (every lane owns
// dims base + lane + 32 q).
template <class Fe>
__device__ __forceinline__ void open_chunk(const Fe* __restrict__ feats, int D, int base,
                                           const int* buf, int cnt, double* sz, double* sz2) {
    const int lane = threadIdx.x & 31;
    for (int j = 0; j < cnt; ++j) {
        const Fe* f = feats + (long long)buf[j] * D + base;
#pragma unroll
        for (int q = 0; q < kOpenPer; ++q) {
            const int cc = lane + 32 * q;
            if (base + cc < D) {
                const double zv = (double)f[cc];
                sz[q] += zv;
                sz2[q] += zv * zv;
            }
        }
    }
}

template <class TD, class TS, class Fe>
__device__ __forceinline__ void open_voxel(const UpdateArgs& a, TD* vd, TD* vw, TS* mean, TS* beta,
                                           const Fe* feats, int i, int s, unsigned k, int* buf,
                                           unsigned* bm, bool huge) {
    const int lane = threadIdx.x & 31;
    const Center c = voxel_center(a.ukey[i], a.kp, a.h, a.pp);
    const int g = a.gvid[i];
    const int vid = g & 0x7fffffff;
    const bool isnew = g < 0;
    int minr = 0;
    long long nwords = 0;
    if (huge) bitmap_build(a.srid, a.foff[s], k, bm, minr, nwords);
    else warp_sort_segment(a.srid, a.foff[s], (int)k, buf);
    // TSDF sums in point order
    TsdfAcc acc{0.0, 0.0, INFINITY, -INFINITY, 0};
    if (huge) {
        for (long long w0 = 0; w0 < nwords; w0 += 32) {
            const int cnt = bitmap_chunk(bm, w0, nwords, minr, buf);
            if (cnt) warp_tsdf_chunk<float>(a, buf, cnt, c, acc, nullptr, false);
            __syncwarp();
        }
    } else {
        warp_tsdf_chunk<float>(a, buf, (int)k, c, acc, nullptr, false);
    }
    double w_old = 0.0;
    if (lane == 0) w_old = apply_tsdf<TD>(vd, vw, vid, isnew, a.trunc, acc.sw, acc.swd, acc.mind, acc.maxd);
    w_old = __shfl_sync(0xffffffffu, w_old, 0);
    // NIG batch update with lambda from the pre-frame weight
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
        } else {
            open_chunk<Fe>(feats, a.D, base, buf, (int)k, sz, sz2);
        }
#pragma unroll
        for (int q = 0; q < kOpenPer; ++q) {
            const int cc = base + lane + 32 * q;
            if (cc < a.D) nig_apply<TS>(mrow, brow, cc, isnew, sz[q], sz2[q], lam, lam_post, coef,
                                        nobs, b_bg);
        }
    }
    if (lane == 0) clear_frame_slot(a.fkey, a.fcount, a.fcur, s);
    __syncwarp();
}

template <class TD, class TS, class Fe>
__global__ void __launch_bounds__(32 * kWarpsPerCta) k_update_open(UpdateArgs a, TD* vd, TD* vw,
                                                                   TS* mean, TS* beta,
                                                                   const Fe* __restrict__ feats) {
    __shared__ int sbuf[kWarpsPerCta][kSmemMax];
    if (frame_aborted(a.ctr)) return;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const long long U = (long long)a.ctr->n_groups;
    for (long long i = (long long)blockIdx.x * kWarpsPerCta + wib; i < U;
         i += (long long)gridDim.x * kWarpsPerCta) {
        const int s = a.ulist[i];
        const unsigned k = a.fcount[s];
        if (k > (unsigned)kSmemMax) {
            if (lane == 0) a.hugelist[atomicAdd(&a.ctr->n_huge, 1ULL)] = (int)i;
            continue;
        }
        open_voxel<TD, TS, Fe>(a, vd, vw, mean, beta, feats, (int)i, s, k, sbuf[wib], nullptr, false);
    }
}

template <class TD, class TS, class Fe>
__global__ void __launch_bounds__(32 * kWarpsPerCta) k_update_open_huge(UpdateArgs a, TD* vd, TD* vw,
                                                                        TS* mean, TS* beta,
                                                                        const Fe* __restrict__ feats) {
    __shared__ int sbuf[kWarpsPerCta][kSmemMax];
    if (frame_aborted(a.ctr)) return;
    const int wib = threadIdx.x >> 5;
    const long long gw = (long long)blockIdx.x * kWarpsPerCta + wib;
    unsigned* bm = a.bitmap + gw * a.bm_words;
    const long long Hn = (long long)a.ctr->n_huge;
    for (long long t = gw; t < Hn; t += (long long)gridDim.x * kWarpsPerCta) {
        const int i = a.hugelist[t];
        const int s = a.ulist[i];
        open_voxel<TD, TS, Fe>(a, vd, vw, mean, beta, feats, i, s, a.fcount[s], sbuf[wib], bm, true);
    }
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

UpdateArgs make_args(svx_map* m, const KeyPack& kp, const PoseParams& pp, const int32_t* labels,
                     int64_t n) {
    UpdateArgs a;
    a.ulist = ptr<int>(m->ulist);
    a.ukey = ptr<unsigned long long>(m->ukey);
    a.gvid = ptr<int>(m->gvid);
    a.fkey = ptr<unsigned long long>(m->fkey);
    a.fcount = ptr<unsigned>(m->fcount);
    a.foff = ptr<unsigned>(m->foff);
    a.fcur = ptr<unsigned>(m->fcur);
    a.srid = ptr<int>(m->srid);
    a.ray = ptr<double4>(m->ray);
    a.longlist = ptr<int>(m->longlist);
    a.hugelist = ptr<int>(m->longlist) + m->ucap;
    a.bitmap = ptr<unsigned>(m->bitmap);
    a.bm_words = (n + 31) / 32 + 1;
    a.kp = kp;
    a.pp = pp;
    a.h = m->cfg.voxel_size;
    a.trunc = m->cfg.truncation;
    a.wfn = m->cfg.weight_fn;
    a.sem_kind = m->cfg.sem_kind;
    a.last_wins = m->cfg.last_wins;
    a.C = m->payload_d > 0 ? m->payload_d : 1;
    a.labels = labels;
    a.D = m->payload_d;
    a.lambda_floor = m->cfg.lambda_floor;
    a.prior_beta = m->cfg.prior_beta;
    a.ctr = ptr<FrameCtr>(m->ctr);
    return a;
}

constexpr int kShortBlocks = 148 * 8;
constexpr int kLongBlocks = 148 * 4;
constexpr int kHugeBlocks = kHugeWarps / kWarpsPerCta;

template <class TD, class TC>
svx_status update_closed_t(svx_map* m, const UpdateArgs& a, cudaStream_t s) {
    TD* vd = ptr<TD>(m->vd);
    TD* vw = ptr<TD>(m->vw);
    TC* cnt = ptr<TC>(m->s0);
    k_update_short<TD, TC><<<kShortBlocks, 256, 0, s>>>(a, vd, vw, cnt);
    SVX_LAUNCHED();
    k_update_long<TD, TC><<<kLongBlocks, 32 * kWarpsPerCta, 0, s>>>(a, vd, vw, cnt);
    SVX_LAUNCHED();
    k_update_huge<TD, TC><<<kHugeBlocks, 32 * kWarpsPerCta, 0, s>>>(a, vd, vw, cnt);
    SVX_LAUNCHED();
    return SVX_OK;
}

template <class TD, class TS, class Fe>
svx_status update_open_t(svx_map* m, const UpdateArgs& a, const Fe* feats, cudaStream_t s) {
    TD* vd = ptr<TD>(m->vd);
    TD* vw = ptr<TD>(m->vw);
    k_update_open<TD, TS, Fe><<<kLongBlocks, 32 * kWarpsPerCta, 0, s>>>(
        a, vd, vw, ptr<TS>(m->s0), ptr<TS>(m->s1), feats);
    SVX_LAUNCHED();
    k_update_open_huge<TD, TS, Fe><<<kHugeBlocks, 32 * kWarpsPerCta, 0, s>>>(
        a, vd, vw, ptr<TS>(m->s0), ptr<TS>(m->s1), feats);
    SVX_LAUNCHED();
    return SVX_OK;
}

template <class TD>
svx_status update_td(svx_map* m, const UpdateArgs& a, const void* feats, int feats_f64,
                     cudaStream_t s) {
    if (m->cfg.sem_kind == SVX_SEM_OPEN) {
        const bool s64 = m->cfg.state_dtype == SVX_F64;
        if (s64) {
            if (feats_f64) return update_open_t<TD, double, double>(m, a, (const double*)feats, s);
            return update_open_t<TD, double, float>(m, a, (const float*)feats, s);
        }
        if (feats_f64) return update_open_t<TD, float, double>(m, a, (const double*)feats, s);
        return update_open_t<TD, float, float>(m, a, (const float*)feats, s);
    }
    if (m->cfg.count_dtype == SVX_F64) return update_closed_t<TD, double>(m, a, s);
    return update_closed_t<TD, float>(m, a, s);
}

}  // namespace

svx_status launch_voxels(svx_map* m, const KeyPack& kp, const FrameCaps& fc, cudaStream_t s) {
    k_voxels<<<kPersistentBlocks, 256, 0, s>>>(
        ptr<int>(m->ulist), ptr<unsigned long long>(m->ukey), kp, ptr<int4>(m->hash), m->hcap - 1,
        fc.frame, ptr<int4>(m->bcoord), ptr<unsigned long long>(m->bkey),
        ptr<unsigned long long>(m->bmask), ptr<int>(m->bslot), ptr<int>(m->gvid),
        ptr<FrameCtr>(m->ctr));
    SVX_LAUNCHED();
    return SVX_OK;
}

svx_status launch_update(svx_map* m, const KeyPack& kp, const PoseParams& pp, const FrameCaps& fc,
                         const int32_t* labels, const void* feats, int feats_f64, int64_t n,
                         cudaStream_t s) {
    (void)fc;
    UpdateArgs a = make_args(m, kp, pp, labels, n);
    if (m->cfg.tsdf_dtype == SVX_F64) return update_td<double>(m, a, feats, feats_f64, s);
    return update_td<float>(m, a, feats, feats_f64, s);
}

svx_status launch_rehash(svx_map* m, int4* new_table, int64_t new_cap, cudaStream_t s) {
    const int T = 256;
    if (m->nblocks == 0) return SVX_OK;
    k_rehash<<<grid_for(m->nblocks, T), T, 0, s>>>(m->nblocks, ptr<int4>(m->bcoord), new_table,
                                                   new_cap - 1);
    SVX_LAUNCHED();
    return SVX_OK;
}

int huge_warps() { return kHugeWarps; }

}  // namespace svx

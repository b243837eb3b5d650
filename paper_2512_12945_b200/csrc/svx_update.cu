// svx_update.cu -- block allocation (K4) and the fused TSDF + semantic update
// (K5/K6).
//
// Compiled with -fmad=false.  Per voxel, rows arrive sorted by point index
// (the reference's (voxel, point, step) order) and are reduced sequentially in
// fp64 exactly like _core.pyx:759-837; the apply arithmetic restates
// apply_tsdf / apply_closed / apply_open (_pycore.py:399-446) operation for
// operation, so stored values round identically.
#include <math.h>

#include "svx_internal.cuh"

namespace svx {
namespace {

__device__ __forceinline__ void decode_key(unsigned long long key, const KeyPack& kp, long long& x,
                                           long long& y, long long& z) {
    const unsigned long long zm = (1ULL << kp.bz) - 1ULL;
    const unsigned long long ym = (1ULL << (kp.byz - kp.bz)) - 1ULL;
    x = (long long)(key >> kp.byz) + kp.mn[0];
    y = (long long)((key >> kp.bz) & ym) + kp.mn[1];
    z = (long long)(key & zm) + kp.mn[2];
}

__device__ __forceinline__ int slot_of(long long x, long long y, long long z) {
    return (int)(((x & 7) << 6) | ((y & 7) << 3) | (z & 7));
}

// Find-or-insert of a leaf coordinate.  A claimed slot is BUSY until its key
// is written, then PENDING(tmp) until the allocation pass assigns the final
// leaf id in first-occurrence order.
__device__ int hash_find_or_insert(int4* table, int64_t mask, int a, int b, int c,
                                   int4* newcoord, int* newpos,
                                   unsigned long long* n_new) {
    int64_t pos = (int64_t)(block_hash(a, b, c) & (uint64_t)mask);
    while (true) {
        volatile int* vw = &table[pos].w;
        int v = *vw;
        if (v == kHashEmpty) {
            int old = atomicCAS((int*)&table[pos].w, kHashEmpty, kHashBusy);
            if (old == kHashEmpty) {
                table[pos].x = a;
                table[pos].y = b;
                table[pos].z = c;
                unsigned long long tmp = atomicAdd(n_new, 1ULL);
                newcoord[tmp] = make_int4(a, b, c, 0);
                newpos[tmp] = (int)pos;
                __threadfence();
                int pend = kHashPendingBase - (int)tmp;
                atomicExch((int*)&table[pos].w, pend);
                return pend;
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

// One thread per unique voxel (group).  Leaders of runs that share a leaf do
// the hash operation; the rest of the run copies it through a shuffle.
__global__ void k_blocks(int64_t U, const unsigned long long* __restrict__ ukeys, KeyPack kp,
                         int4* table, int64_t mask, int* __restrict__ gblock,
                         int4* __restrict__ newcoord, int* __restrict__ newpos,
                         unsigned* __restrict__ newfirst, FrameCtr* ctr) {
    int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    long long x = 0, y = 0, z = 0;
    bool live = g < U;
    if (live) decode_key(ukeys[g], kp, x, y, z);
    int bx = (int)(x >> kLeafLog2), by = (int)(y >> kLeafLog2), bz = (int)(z >> kLeafLog2);
    int px = __shfl_up_sync(0xffffffffu, bx, 1);
    int py = __shfl_up_sync(0xffffffffu, by, 1);
    int pz = __shfl_up_sync(0xffffffffu, bz, 1);
    bool leader = live && (lane == 0 || px != bx || py != by || pz != bz);
    int val = 0;
    if (leader) {
        val = hash_find_or_insert(table, mask, bx, by, bz, newcoord, newpos, &ctr->n_new_blocks);
        if (val <= kHashPendingBase) atomicMin(&newfirst[kHashPendingBase - val], (unsigned)g);
    }
    unsigned leaders = __ballot_sync(0xffffffffu, leader);
    unsigned upto = leaders & (0xffffffffu >> (31 - lane));
    int src = upto ? 31 - __clz(upto) : 0;
    val = __shfl_sync(0xffffffffu, val, src);
    if (live) gblock[g] = val;
}

// New leaves, sorted by first occurrence, receive consecutive ids: the
// reference allocates leaves in first-occurrence order of the sorted unique
// voxels (_core.pyx:755, :377-420).
__global__ void k_assign_blocks(int64_t nnew, const unsigned* __restrict__ order,
                                const int4* __restrict__ newcoord, const int* __restrict__ newpos,
                                int64_t base, int frame, int4* table, int4* __restrict__ bcoord,
                                int* __restrict__ tmp2id) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nnew) return;
    unsigned tmp = order[r];
    int id = (int)(base + r);
    int4 c = newcoord[tmp];
    table[newpos[tmp]].w = id;
    bcoord[id] = make_int4(c.x, c.y, c.z, frame);
    tmp2id[tmp] = id;
}

__global__ void k_resolve(int64_t U, const unsigned long long* __restrict__ ukeys, KeyPack kp,
                          int* __restrict__ gblock, const int* __restrict__ tmp2id,
                          const int* __restrict__ bslot, int* __restrict__ gvid,
                          int* __restrict__ gnew, FrameCtr* ctr) {
    int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int isnew = 0;
    if (g < U) {
        int blk = gblock[g];
        if (blk <= kHashPendingBase) {
            blk = tmp2id[kHashPendingBase - blk];
            gblock[g] = blk;
        }
        long long x, y, z;
        decode_key(ukeys[g], kp, x, y, z);
        int vid = bslot[(int64_t)blk * kLeafVolume + slot_of(x, y, z)];
        isnew = vid < 0;
        gvid[g] = vid;
        gnew[g] = isnew;
    }
    unsigned a = __reduce_add_sync(0xffffffffu, (unsigned)isnew);
    if ((threadIdx.x & 31) == 0 && a) atomicAdd(&ctr->n_new_voxels, (unsigned long long)a);
}

__global__ void k_activate(int64_t U, const unsigned long long* __restrict__ ukeys, KeyPack kp,
                           const int* __restrict__ gblock, const int* __restrict__ gnew,
                           const int* __restrict__ grank, int64_t nvox, int* __restrict__ bslot,
                           unsigned long long* __restrict__ bmask, int* __restrict__ gvid) {
    int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= U || !gnew[g]) return;
    long long x, y, z;
    decode_key(ukeys[g], kp, x, y, z);
    int slot = slot_of(x, y, z);
    int blk = gblock[g];
    int vid = (int)(nvox + grank[g]);
    bslot[(int64_t)blk * kLeafVolume + slot] = vid;
    atomicOr(&bmask[(int64_t)blk * kMaskWords + (slot >> 6)], 1ULL << (slot & 63));
    gvid[g] = vid;
}

template <class TD>
__device__ __forceinline__ bool equals_stored(TD stored, double v) {
    return stored == (TD)v;
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

// TSDF (+ closed-set) update: one thread per unique voxel, rows reduced in
// sorted order (_core.pyx:789-817).
template <class TD, class TC>
__global__ void k_update_closed(int64_t U, const unsigned long long* __restrict__ ukeys, KeyPack kp,
                                const long long* __restrict__ gstart, const int* __restrict__ runlen,
                                const int* __restrict__ srid, const double4* __restrict__ ray,
                                const int* __restrict__ gvid, const int* __restrict__ gnew,
                                PoseParams pp, double h, double trunc, int wfn, int sem_kind,
                                int last_wins, const int32_t* __restrict__ labels, int C,
                                TD* __restrict__ vd, TD* __restrict__ vw, TC* __restrict__ counts) {
    int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= U) return;
    long long x, y, z;
    decode_key(ukeys[g], kp, x, y, z);
    const double cxv = ((double)x + 0.5) * h - pp.t[0];
    const double cyv = ((double)y + 0.5) * h - pp.t[1];
    const double czv = ((double)z + 0.5) * h - pp.t[2];
    const long long b = gstart[g];
    const long long e = b + runlen[g];
    const int vid = gvid[g];
    const bool isnew = gnew[g] != 0;
    double sw = 0.0, swd = 0.0, mind = INFINITY, maxd = -INFINITY;
    int last_lab = 0;
    TC* crow = counts + (int64_t)vid * C;
    for (long long s = b; s < e; ++s) {
        const int r = srid[s];
        double d, w;
        row_dw(cxv, cyv, czv, ray[r], trunc, wfn, d, w);
        sw += w;
        swd += w * d;
        mind = d < mind ? d : mind;
        maxd = d > maxd ? d : maxd;
        if (sem_kind == SVX_SEM_CLOSED) {
            int lab = labels[r];
            if (last_wins) last_lab = lab;
            else crow[lab - 1] += (TC)1;
        }
    }
    apply_tsdf<TD>(vd, vw, vid, isnew, trunc, sw, swd, mind, maxd);
    if (sem_kind == SVX_SEM_CLOSED && last_wins) {
        for (int c = 0; c < C; ++c) crow[c] = (TC)(c == last_lab - 1 ? 1 : 0);
    }
}

constexpr int kOpenPer = 8;  // dims per lane per pass (256 dims per pass)

// TSDF + open-set NIG update: one warp per unique voxel.  Lanes own feature
// dimensions; rows are walked in sorted order so every per-dimension sum is
// the reference's sequential fp64 sum (_core.pyx:827-837), then apply_open
// (_pycore.py:432-446) runs per dimension.
template <class TD, class TS, class Fe>
__global__ void k_update_open(int64_t U, const unsigned long long* __restrict__ ukeys, KeyPack kp,
                              const long long* __restrict__ gstart, const int* __restrict__ runlen,
                              const int* __restrict__ srid, const double4* __restrict__ ray,
                              const int* __restrict__ gvid, const int* __restrict__ gnew,
                              PoseParams pp, double h, double trunc, int wfn, double lambda_floor,
                              double prior_beta, const Fe* __restrict__ feats, int D,
                              TD* __restrict__ vd, TD* __restrict__ vw, TS* __restrict__ mean,
                              TS* __restrict__ beta) {
    const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (g >= U) return;
    long long x, y, z;
    decode_key(ukeys[g], kp, x, y, z);
    const double cxv = ((double)x + 0.5) * h - pp.t[0];
    const double cyv = ((double)y + 0.5) * h - pp.t[1];
    const double czv = ((double)z + 0.5) * h - pp.t[2];
    const long long b = gstart[g];
    const long long e = b + runlen[g];
    const int vid = gvid[g];
    const bool isnew = gnew[g] != 0;
    // TSDF sums: lanes evaluate 32 rows at a time, then every lane folds them
    // in row order so the fp64 sums keep the sequential association.
    double sw = 0.0, swd = 0.0, mind = INFINITY, maxd = -INFINITY;
    for (long long s0 = b; s0 < e; s0 += 32) {
        double d = 0.0, w = 0.0;
        long long s = s0 + lane;
        if (s < e) row_dw(cxv, cyv, czv, ray[srid[s]], trunc, wfn, d, w);
        const int nv = (int)min((long long)32, e - s0);
        for (int j = 0; j < nv; ++j) {
            double wj = __shfl_sync(0xffffffffu, w, j);
            double dj = __shfl_sync(0xffffffffu, d, j);
            sw += wj;
            swd += wj * dj;
            mind = dj < mind ? dj : mind;
            maxd = dj > maxd ? dj : maxd;
        }
    }
    // Lane 0 owns the TSDF write; every lane needs w_old.
    double w_old;
    if (lane == 0) w_old = apply_tsdf<TD>(vd, vw, vid, isnew, trunc, sw, swd, mind, maxd);
    w_old = __shfl_sync(0xffffffffu, w_old, 0);
    const double nobs = (double)(e - b);
    const double lam = fmax(w_old, lambda_floor);
    const double lam_post = lam + nobs;
    const double coef = lam * nobs / lam_post;
    const double b_bg = (double)(TS)prior_beta;
    TS* mrow = mean + (int64_t)vid * D;
    TS* brow = beta + (int64_t)vid * D;
    for (int base = 0; base < D; base += 32 * kOpenPer) {
        double sz[kOpenPer], sz2[kOpenPer];
#pragma unroll
        for (int q = 0; q < kOpenPer; ++q) { sz[q] = 0.0; sz2[q] = 0.0; }
        for (long long s = b; s < e; ++s) {
            const Fe* f = feats + (int64_t)srid[s] * D + base;
#pragma unroll
            for (int q = 0; q < kOpenPer; ++q) {
                int c = lane + 32 * q;
                if (base + c < D) {
                    double zv = (double)f[c];
                    sz[q] += zv;
                    sz2[q] += zv * zv;
                }
            }
        }
#pragma unroll
        for (int q = 0; q < kOpenPer; ++q) {
            int c = base + lane + 32 * q;
            if (c < D) {
                double m_old = isnew ? 0.0 : (double)mrow[c];
                double b_old = isnew ? b_bg : (double)brow[c];
                double m_new = (lam * m_old + sz[q]) / lam_post;
                double zbar = sz[q] / nobs;
                double ss = sz2[q] - sz[q] * zbar;
                ss = ss < 0.0 ? 0.0 : ss;
                double diff = zbar - m_old;
                double gap = coef * (diff * diff) * 0.5;
                double b_new = b_old + 0.5 * ss + gap;
                mrow[c] = (TS)m_new;
                brow[c] = (TS)b_new;
            }
        }
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

template <class TD, class TC>
svx_status update_closed_t(svx_map* m, int64_t U, const KeyPack& kp, const PoseParams& pp,
                           const int32_t* labels, cudaStream_t s) {
    const int T = 128;
    k_update_closed<TD, TC><<<grid_for(U, T), T, 0, s>>>(
        U, ptr<unsigned long long>(m->ukeys), kp, ptr<long long>(m->gstart), ptr<int>(m->runlen),
        m->srid, ptr<double4>(m->ray), ptr<int>(m->gvid), ptr<int>(m->gnew), pp,
        m->cfg.voxel_size, m->cfg.truncation, m->cfg.weight_fn, m->cfg.sem_kind,
        m->cfg.last_wins, labels, m->payload_d > 0 ? m->payload_d : 1, ptr<TD>(m->vd),
        ptr<TD>(m->vw), ptr<TC>(m->s0));
    SVX_LAUNCHED();
    return SVX_OK;
}

template <class TD, class TS, class Fe>
svx_status update_open_t(svx_map* m, int64_t U, const KeyPack& kp, const PoseParams& pp,
                         const Fe* feats, cudaStream_t s) {
    const int T = 256;  // 8 warps = 8 voxels per CTA
    k_update_open<TD, TS, Fe><<<grid_for(U * 32, T), T, 0, s>>>(
        U, ptr<unsigned long long>(m->ukeys), kp, ptr<long long>(m->gstart), ptr<int>(m->runlen),
        m->srid, ptr<double4>(m->ray), ptr<int>(m->gvid), ptr<int>(m->gnew), pp,
        m->cfg.voxel_size, m->cfg.truncation, m->cfg.weight_fn, m->cfg.lambda_floor,
        m->cfg.prior_beta, feats, m->payload_d, ptr<TD>(m->vd), ptr<TD>(m->vw), ptr<TS>(m->s0),
        ptr<TS>(m->s1));
    SVX_LAUNCHED();
    return SVX_OK;
}

template <class TD>
svx_status update_td(svx_map* m, int64_t U, const KeyPack& kp, const PoseParams& pp,
                     const int32_t* labels, const void* feats, int feats_f64, cudaStream_t s) {
    if (m->cfg.sem_kind == SVX_SEM_OPEN) {
        const bool s64 = m->cfg.state_dtype == SVX_F64;
        if (s64) {
            if (feats_f64) return update_open_t<TD, double, double>(m, U, kp, pp, (const double*)feats, s);
            return update_open_t<TD, double, float>(m, U, kp, pp, (const float*)feats, s);
        }
        if (feats_f64) return update_open_t<TD, float, double>(m, U, kp, pp, (const double*)feats, s);
        return update_open_t<TD, float, float>(m, U, kp, pp, (const float*)feats, s);
    }
    if (m->cfg.count_dtype == SVX_F64) return update_closed_t<TD, double>(m, U, kp, pp, labels, s);
    return update_closed_t<TD, float>(m, U, kp, pp, labels, s);
}

}  // namespace

svx_status launch_blocks(svx_map* m, int64_t U, const KeyPack& kp, cudaStream_t s) {
    const int T = 256;
    k_blocks<<<grid_for(U, T), T, 0, s>>>(U, ptr<unsigned long long>(m->ukeys), kp,
                                          ptr<int4>(m->hash), m->hcap - 1, ptr<int>(m->gblock),
                                          ptr<int4>(m->newcoord), ptr<int>(m->newpos),
                                          ptr<unsigned>(m->newfirst), ptr<FrameCtr>(m->ctr));
    SVX_LAUNCHED();
    return SVX_OK;
}

svx_status launch_assign_blocks(svx_map* m, int64_t nnew, const unsigned* order, cudaStream_t s) {
    const int T = 256;
    k_assign_blocks<<<grid_for(nnew, T), T, 0, s>>>(nnew, order, ptr<int4>(m->newcoord),
                                                    ptr<int>(m->newpos), m->nblocks,
                                                    (int)m->frames, ptr<int4>(m->hash),
                                                    ptr<int4>(m->bcoord), ptr<int>(m->tmp2id));
    SVX_LAUNCHED();
    return SVX_OK;
}

svx_status launch_resolve(svx_map* m, int64_t U, const KeyPack& kp, cudaStream_t s) {
    const int T = 256;
    k_resolve<<<grid_for(U, T), T, 0, s>>>(U, ptr<unsigned long long>(m->ukeys), kp,
                                           ptr<int>(m->gblock), ptr<int>(m->tmp2id),
                                           ptr<int>(m->bslot), ptr<int>(m->gvid),
                                           ptr<int>(m->gnew), ptr<FrameCtr>(m->ctr));
    SVX_LAUNCHED();
    return SVX_OK;
}

svx_status launch_activate(svx_map* m, int64_t U, const KeyPack& kp, cudaStream_t s) {
    const int T = 256;
    k_activate<<<grid_for(U, T), T, 0, s>>>(U, ptr<unsigned long long>(m->ukeys), kp,
                                            ptr<int>(m->gblock), ptr<int>(m->gnew),
                                            ptr<int>(m->grank), m->nvox, ptr<int>(m->bslot),
                                            ptr<unsigned long long>(m->bmask), ptr<int>(m->gvid));
    SVX_LAUNCHED();
    return SVX_OK;
}

svx_status launch_update(svx_map* m, int64_t U, const KeyPack& kp, const PoseParams& pp,
                         const int32_t* labels, const void* feats, int feats_f64, cudaStream_t s) {
    if (m->cfg.tsdf_dtype == SVX_F64)
        return update_td<double>(m, U, kp, pp, labels, feats, feats_f64, s);
    return update_td<float>(m, U, kp, pp, labels, feats, feats_f64, s);
}

svx_status launch_rehash(svx_map* m, int4* new_table, int64_t new_cap, cudaStream_t s) {
    const int T = 256;
    if (m->nblocks == 0) return SVX_OK;
    k_rehash<<<grid_for(m->nblocks, T), T, 0, s>>>(m->nblocks, ptr<int4>(m->bcoord), new_table,
                                                   new_cap - 1);
    SVX_LAUNCHED();
    return SVX_OK;
}

}  // namespace svx

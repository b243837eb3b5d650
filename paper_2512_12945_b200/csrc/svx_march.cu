// svx_march.cu -- per-point preparation, the fp64 band ray-march (K1), and
// the per-frame voxel grouping (counting sort by voxel: K2 compact, K3
// scatter).
//
// Compiled with -fmad=false: every double expression is evaluated with the
// operation order and IEEE round-to-nearest steps of the reference's
// -ffp-contract=off C++ (_core.pyx:478-579, pkg/setup.py:14) and its numpy
// twin (_pycore.py:326-396), so band membership and per-row distances are
// bit-identical.
//
// Grouping replaces the reference's global (voxel, point, step) sort
// (_core.pyx:707-753): each band row inserts its voxel key into a per-frame
// open-addressing table and bumps that voxel's row count (K1); one pass over
// the table compacts the touched voxels and assigns each a contiguous row
// segment (K2); a second march drops every row's point index into its
// voxel's segment (K3).  Rows inside a segment are put back into point order
// by the update kernels, which is all the reference's sort order is needed
// for (sequential per-voxel sums).
#include <math.h>

#include <cub/block/block_scan.cuh>

#include "svx_internal.cuh"

namespace svx {
namespace {

// Walk one ray's truncation band; calls on_cell(i, j, k) for each emitted
// voxel in near-to-far order.  Returns the emitted count, or -1 when the step
// budget is exhausted.  Follows _dda_ray (_core.pyx:478-579) step for step.
template <class F>
__device__ __forceinline__ long long dda_walk(double ox, double oy, double oz, double ux, double uy,
                                              double uz, double ts, const MarchParams& mp,
                                              F&& on_cell) {
    const double h = mp.h;
    double t_lo = mp.carving ? 0.0 : fmax(ts - mp.trunc, 0.0);
    double t_hi = ts + mp.trunc;
    double px = ox + ux * t_lo;
    double py = oy + uy * t_lo;
    double pz = oz + uz * t_lo;
    long long ci = (long long)floor(px / h);
    long long cj = (long long)floor(py / h);
    long long ck = (long long)floor(pz / h);
    int sx = ux == 0.0 ? 0 : (ux > 0.0 ? 1 : -1);
    int sy = uy == 0.0 ? 0 : (uy > 0.0 ? 1 : -1);
    int sz = uz == 0.0 ? 0 : (uz > 0.0 ? 1 : -1);
    double tmx, tmy, tmz, tdx, tdy, tdz;
    if (sx > 0) {
        tmx = t_lo + ((double)(ci + 1) * h - px) / ux;
        tdx = h / fabs(ux);
    } else if (sx < 0) {
        tmx = t_lo + ((double)ci * h - px) / ux;
        tdx = h / fabs(ux);
    } else {
        tmx = INFINITY;
        tdx = INFINITY;
    }
    if (sy > 0) {
        tmy = t_lo + ((double)(cj + 1) * h - py) / uy;
        tdy = h / fabs(uy);
    } else if (sy < 0) {
        tmy = t_lo + ((double)cj * h - py) / uy;
        tdy = h / fabs(uy);
    } else {
        tmy = INFINITY;
        tdy = INFINITY;
    }
    if (sz > 0) {
        tmz = t_lo + ((double)(ck + 1) * h - pz) / uz;
        tdz = h / fabs(uz);
    } else if (sz < 0) {
        tmz = t_lo + ((double)ck * h - pz) / uz;
        tdz = h / fabs(uz);
    } else {
        tmz = INFINITY;
        tdz = INFINITY;
    }
    double t_enter = t_lo;
    long long cnt = 0, k = 0;
    while (t_enter < t_hi) {
        if (k >= kStepBudget) return -1;
        int axis = 0;
        double tmin = tmx;
        if (tmy < tmin) { axis = 1; tmin = tmy; }
        if (tmz < tmin) { axis = 2; tmin = tmz; }
        if (tmin > t_lo) {
            on_cell(ci, cj, ck);
            ++cnt;
        }
        if (axis == 0) { ci += sx; tmx += tdx; }
        else if (axis == 1) { cj += sy; tmy += tdy; }
        else { ck += sz; tmz += tdz; }
        t_enter = tmin;
        ++k;
    }
    return cnt;
}

// Row weight under linear dropoff (row_distances_weights, _pycore.py:384-396).
__device__ __forceinline__ bool row_kept(long long ci, long long cj, long long ck, double ox,
                                         double oy, double oz, double4 r, const MarchParams& mp) {
    if (mp.wfn != 1) return true;
    double cx = ((double)ci + 0.5) * mp.h - ox;
    double cy = ((double)cj + 0.5) * mp.h - oy;
    double cz = ((double)ck + 0.5) * mp.h - oz;
    double proj = cx * r.x + cy * r.y + cz * r.z;
    double d = r.w - proj;
    if (d < -mp.trunc) d = -mp.trunc;
    if (d > mp.trunc) d = mp.trunc;
    double w = d >= 0.0 ? 1.0 : (mp.trunc + d) / mp.trunc;
    return w > 0.0;
}

// Frame-table insert; returns the slot or -1 when the table is full.
__device__ __forceinline__ long long frame_insert(unsigned long long* keys, long long mask,
                                                  unsigned long long key) {
    long long pos = (long long)(key_hash(key) & (unsigned long long)mask);
    for (long long probe = 0; probe <= mask; ++probe) {
        unsigned long long cur = keys[pos];
        if (cur == key) return pos;
        if (cur == kKeyEmpty) {
            cur = atomicCAS(&keys[pos], kKeyEmpty, key);
            if (cur == kKeyEmpty || cur == key) return pos;
        }
        pos = (pos + 1) & mask;
    }
    return -1;
}

__device__ __forceinline__ long long frame_find(const unsigned long long* __restrict__ keys,
                                                long long mask, unsigned long long key) {
    long long pos = (long long)(key_hash(key) & (unsigned long long)mask);
    while (true) {
        unsigned long long cur = keys[pos];
        if (cur == key) return pos;
        if (cur == kKeyEmpty) return -1;
        pos = (pos + 1) & mask;
    }
}

template <class P>
__device__ __forceinline__ void load_point(const P* pts, int64_t i, double& x, double& y, double& z) {
    x = (double)pts[3 * i];
    y = (double)pts[3 * i + 1];
    z = (double)pts[3 * i + 2];
}

// K1: validation masks (integrate_frame, fusion.py:228-256), ray setup
// (fusion.py:262-263), band walk, frame-table insert + per-voxel row count.
template <class P, class Fe>
__global__ void __launch_bounds__(256) k_march(
    const P* __restrict__ pts, int64_t n, PoseParams pp, MarchParams mp, KeyPack kp, long long fmask,
    int sem_kind, const int32_t* __restrict__ labels, int num_classes, const Fe* __restrict__ feats,
    int D, double4* __restrict__ ray, unsigned long long* fkey, unsigned* fcount,
    FrameCtr* __restrict__ ctr) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool live = i < n;
    unsigned c_nonfinite = 0, c_range = 0, c_degen = 0, c_badlab = 0, c_used = 0;
    unsigned long long c_hits = 0, c_rows = 0;
    long long mn0 = LLONG_MAX, mn1 = LLONG_MAX, mn2 = LLONG_MAX;
    long long mx0 = LLONG_MIN, mx1 = LLONG_MIN, mx2 = LLONG_MIN;
    int budget = 0, packerr = 0, probeerr = 0;
    if (live) {
        double x, y, z;
        load_point(pts, i, x, y, z);
        double wx, wy, wz;
        if (pp.sensor) {
            wx = ((pp.R[0] * x + pp.R[1] * y) + pp.R[2] * z) + pp.t[0];
            wy = ((pp.R[3] * x + pp.R[4] * y) + pp.R[5] * z) + pp.t[1];
            wz = ((pp.R[6] * x + pp.R[7] * y) + pp.R[8] * z) + pp.t[2];
        } else {
            wx = x; wy = y; wz = z;
        }
        const double ox = pp.t[0], oy = pp.t[1], oz = pp.t[2];
        bool finite = isfinite(wx) && isfinite(wy) && isfinite(wz);
        double dx = wx - ox, dy = wy - oy, dz = wz - oz;
        double ts = sqrt((dx * dx + dy * dy) + dz * dz);
        if (!isfinite(ts)) ts = INFINITY;
        bool degenerate = finite && ts == 0.0;
        bool in_range = ts <= mp.max_range;
        bool keep = finite && !degenerate && in_range;
        c_nonfinite = !finite;
        c_degen = degenerate;
        c_range = finite && !degenerate && !in_range;
        if (sem_kind == SVX_SEM_CLOSED) {
            int lab = labels[i];
            bool good = lab >= 1 && lab <= num_classes;
            c_badlab = keep && !good;
            keep = keep && good;
        } else if (sem_kind == SVX_SEM_OPEN) {
            bool good = true;
            const Fe* f = feats + (int64_t)i * D;
            for (int c = 0; c < D; ++c) good = good && isfinite((double)f[c]);
            c_badlab = keep && !good;
            keep = keep && good;
        }
        double4 r = make_double4(0.0, 0.0, 0.0, -1.0);
        if (keep) {
            c_used = 1;
            r = make_double4(dx / ts, dy / ts, dz / ts, ts);
            long long emitted = dda_walk(ox, oy, oz, r.x, r.y, r.z, ts, mp,
                [&](long long ci, long long cj, long long ck) {
                    if (!row_kept(ci, cj, ck, ox, oy, oz, r, mp)) return;
                    ++c_rows;
                    mn0 = min(mn0, ci); mn1 = min(mn1, cj); mn2 = min(mn2, ck);
                    mx0 = max(mx0, ci); mx1 = max(mx1, cj); mx2 = max(mx2, ck);
                    long long ox_ = ci - kp.base[0], oy_ = cj - kp.base[1], oz_ = ck - kp.base[2];
                    if (((ox_ | oy_ | oz_) & ~kPackMask) != 0) {
                        packerr = 1;
                        return;
                    }
                    long long s = frame_insert(fkey, fmask, pack_key(ox_, oy_, oz_));
                    if (s < 0) {
                        probeerr = 1;
                        return;
                    }
                    atomicAdd(&fcount[s], 1u);
                });
            if (emitted < 0) {
                budget = 1;
                r.w = -1.0;   // nothing of this frame is applied anyway
            } else {
                c_hits = (unsigned long long)emitted;
            }
        }
        ray[i] = r;
    }
    // warp-aggregated counters
    const unsigned full = 0xffffffffu;
    unsigned a_nf = __reduce_add_sync(full, c_nonfinite);
    unsigned a_rg = __reduce_add_sync(full, c_range);
    unsigned a_dg = __reduce_add_sync(full, c_degen);
    unsigned a_bl = __reduce_add_sync(full, c_badlab);
    unsigned a_us = __reduce_add_sync(full, c_used);
    unsigned a_er = __reduce_or_sync(full, (unsigned)(budget | (packerr << 1) | (probeerr << 2)));
    for (int o = 16; o > 0; o >>= 1) {
        c_hits += __shfl_xor_sync(full, c_hits, o);
        c_rows += __shfl_xor_sync(full, c_rows, o);
        mn0 = min(mn0, __shfl_xor_sync(full, mn0, o));
        mn1 = min(mn1, __shfl_xor_sync(full, mn1, o));
        mn2 = min(mn2, __shfl_xor_sync(full, mn2, o));
        mx0 = max(mx0, __shfl_xor_sync(full, mx0, o));
        mx1 = max(mx1, __shfl_xor_sync(full, mx1, o));
        mx2 = max(mx2, __shfl_xor_sync(full, mx2, o));
    }
    if ((threadIdx.x & 31) == 0) {
        if (a_nf) atomicAdd(&ctr->nonfinite, (unsigned long long)a_nf);
        if (a_rg) atomicAdd(&ctr->range, (unsigned long long)a_rg);
        if (a_dg) atomicAdd(&ctr->degenerate, (unsigned long long)a_dg);
        if (a_bl) atomicAdd(&ctr->bad_label, (unsigned long long)a_bl);
        if (a_us) atomicAdd(&ctr->used, (unsigned long long)a_us);
        if (c_hits) atomicAdd(&ctr->band_hits, c_hits);
        if (c_rows) {
            atomicAdd(&ctr->rows, c_rows);
            atomicMin(&ctr->bbox_min[0], mn0); atomicMin(&ctr->bbox_min[1], mn1);
            atomicMin(&ctr->bbox_min[2], mn2);
            atomicMax(&ctr->bbox_max[0], mx0); atomicMax(&ctr->bbox_max[1], mx1);
            atomicMax(&ctr->bbox_max[2], mx2);
        }
        if (a_er & 1) atomicOr(&ctr->err_budget, 1);
        if (a_er & 2) atomicOr(&ctr->err_pack, 1);
        if (a_er & 4) atomicOr(&ctr->err_probe, 1);
    }
}

constexpr int kCompactThreads = 256;
constexpr int kCompactPer = 4;

// K2: one pass over the frame table.  Touched voxels are compacted into
// ulist/ukey and each gets a contiguous segment of the row array; segment
// order follows CTA arrival (no observable effect).
__global__ void __launch_bounds__(kCompactThreads) k_compact(
    const unsigned long long* __restrict__ fkey, const unsigned* __restrict__ fcount,
    unsigned* __restrict__ foff, long long fcap, unsigned long long ucap, int* __restrict__ ulist,
    unsigned long long* __restrict__ ukey, FrameCtr* ctr) {
    using Scan = cub::BlockScan<unsigned long long, kCompactThreads>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ unsigned long long s_ubase, s_rbase;
    const long long base = ((long long)blockIdx.x * kCompactThreads + threadIdx.x) * kCompactPer;
    unsigned long long kk[kCompactPer];
    unsigned cc[kCompactPer];
    unsigned occ = 0, rows = 0;
#pragma unroll
    for (int q = 0; q < kCompactPer; ++q) {
        long long s = base + q;
        kk[q] = s < fcap ? fkey[s] : kKeyEmpty;
        cc[q] = kk[q] != kKeyEmpty ? fcount[s] : 0u;
        occ += kk[q] != kKeyEmpty;
        rows += cc[q];
    }
    // pack (occupied, rows) into one 64-bit scan
    unsigned long long packed = ((unsigned long long)occ << 40) | rows, pre, total;
    Scan(tmp).ExclusiveSum(packed, pre, total);
    if (threadIdx.x == 0) {
        unsigned long long tocc = total >> 40, trows = total & ((1ULL << 40) - 1);
        s_ubase = tocc ? atomicAdd(&ctr->n_groups, tocc) : 0ULL;
        s_rbase = trows ? atomicAdd(&ctr->rows_c, trows) : 0ULL;
    }
    __syncthreads();
    unsigned long long u = s_ubase + (pre >> 40);
    unsigned long long r = s_rbase + (pre & ((1ULL << 40) - 1));
#pragma unroll
    for (int q = 0; q < kCompactPer; ++q) {
        if (kk[q] == kKeyEmpty) continue;
        long long s = base + q;
        if (u < ucap) {
            ulist[u] = (int)s;
            ukey[u] = kk[q];
        }
        foff[s] = (unsigned)r;
        ++u;
        r += cc[q];
    }
}

// K3: second march; each kept row writes its point index into its voxel's
// segment (arbitrary order within the segment).
__global__ void __launch_bounds__(256) k_scatter(
    int64_t n, const double4* __restrict__ ray, PoseParams pp, MarchParams mp, KeyPack kp,
    long long fmask, const unsigned long long* __restrict__ fkey, const unsigned* __restrict__ foff,
    unsigned* fcur, int* __restrict__ srid, FrameCaps fc, const FrameCtr* __restrict__ ctr) {
    if (ctr->abort) return;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double4 r = ray[i];
    if (!(r.w >= 0.0)) return;
    const double ox = pp.t[0], oy = pp.t[1], oz = pp.t[2];
    dda_walk(ox, oy, oz, r.x, r.y, r.z, r.w, mp, [&](long long ci, long long cj, long long ck) {
        if (!row_kept(ci, cj, ck, ox, oy, oz, r, mp)) return;
        unsigned long long key = pack_key(ci - kp.base[0], cj - kp.base[1], ck - kp.base[2]);
        long long s = frame_find(fkey, fmask, key);
        unsigned pos = foff[s] + atomicAdd(&fcur[s], 1u);
        srid[pos] = (int)i;
    });
}

// Decide, once per frame on the device, whether the frame may mutate the map
// (mirrors the reference's checks before any allocation, _core.pyx:661-712,
// :386-387).
__global__ void k_gate(FrameCtr* ctr, FrameCaps fc) {
    int ab = ctr->err_budget | ctr->err_pack | ctr->err_probe;
    if (ctr->n_groups > fc.ucap || ctr->rows_c > fc.rcap) ab = 1;
    if (ctr->rows) {
        for (int a = 0; a < 3; ++a) {
            long long lo = ctr->bbox_min[a], hi = ctr->bbox_max[a];
            if (hi - lo >= (1LL << kPackBits)) ab = 1;
            if (llabs(lo) >= kCoordLimit || llabs(hi) >= kCoordLimit) ab = 1;
        }
    }
    ctr->abort = ab;
}

template <class P, class Fe>
svx_status march_t(svx_map* m, const P* pts, int64_t n, const PoseParams& pp, const MarchParams& mp,
                   const KeyPack& kp, const FrameCaps& fc, const int32_t* labels, const Fe* feats,
                   cudaStream_t s) {
    const int T = 256;
    k_march<P, Fe><<<grid_for(n, T), T, 0, s>>>(
        pts, n, pp, mp, kp, fc.fmask, m->cfg.sem_kind, labels, m->cfg.num_classes, feats,
        m->payload_d, ptr<double4>(m->ray), ptr<unsigned long long>(m->fkey),
        ptr<unsigned>(m->fcount), ptr<FrameCtr>(m->ctr));
    SVX_LAUNCHED();
    return SVX_OK;
}

MarchParams march_params(const svx_map* m) {
    MarchParams mp;
    mp.h = m->cfg.voxel_size;
    mp.trunc = m->cfg.truncation;
    mp.max_range = m->cfg.max_range;
    mp.carving = m->cfg.space_carving;
    mp.wfn = m->cfg.weight_fn;
    return mp;
}

}  // namespace

svx_status launch_march(svx_map* m, const void* pts, int pts_f64, int64_t n, const PoseParams& pp,
                        const KeyPack& kp, const FrameCaps& fc, const int32_t* labels,
                        const void* feats, int feats_f64, cudaStream_t s) {
    MarchParams mp = march_params(m);
    if (pts_f64) {
        if (feats_f64)
            return march_t(m, (const double*)pts, n, pp, mp, kp, fc, labels, (const double*)feats, s);
        return march_t(m, (const double*)pts, n, pp, mp, kp, fc, labels, (const float*)feats, s);
    }
    if (feats_f64)
        return march_t(m, (const float*)pts, n, pp, mp, kp, fc, labels, (const double*)feats, s);
    return march_t(m, (const float*)pts, n, pp, mp, kp, fc, labels, (const float*)feats, s);
}

svx_status launch_compact(svx_map* m, const FrameCaps& fc, cudaStream_t s) {
    const long long per_block = (long long)kCompactThreads * kCompactPer;
    const int blocks = (int)((m->fcap + per_block - 1) / per_block);
    k_compact<<<blocks, kCompactThreads, 0, s>>>(
        ptr<unsigned long long>(m->fkey), ptr<unsigned>(m->fcount), ptr<unsigned>(m->foff), m->fcap,
        fc.ucap, ptr<int>(m->ulist), ptr<unsigned long long>(m->ukey), ptr<FrameCtr>(m->ctr));
    SVX_LAUNCHED();
    k_gate<<<1, 1, 0, s>>>(ptr<FrameCtr>(m->ctr), fc);
    SVX_LAUNCHED();
    return SVX_OK;
}

svx_status launch_scatter(svx_map* m, int64_t n, const PoseParams& pp, const KeyPack& kp,
                          const FrameCaps& fc, cudaStream_t s) {
    MarchParams mp = march_params(m);
    const int T = 256;
    k_scatter<<<grid_for(n, T), T, 0, s>>>(n, ptr<double4>(m->ray), pp, mp, kp, fc.fmask,
                                           ptr<unsigned long long>(m->fkey),
                                           ptr<unsigned>(m->foff), ptr<unsigned>(m->fcur),
                                           ptr<int>(m->srid), fc, ptr<FrameCtr>(m->ctr));
    SVX_LAUNCHED();
    return SVX_OK;
}

}  // namespace svx

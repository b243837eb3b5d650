// svx_march.cu -- per-point preparation and the fp64 band ray-march (K1).
//
// Compiled with -fmad=false: every double expression below is evaluated with
// the same operation order and IEEE round-to-nearest steps as the reference's
// -ffp-contract=off C++ (_core.pyx:478-579, pkg/setup.py:14) and its numpy
// twin (_pycore.py:326-396), so band membership and per-row distances are
// bit-identical.
//
// Two passes over the rays (count, then fill after an exclusive scan) give
// rows in (point, step) order, which a stable radix sort on the voxel key then
// turns into the reference's canonical (voxel, point, step) order
// (_core.pyx:715-738).
#include <math.h>

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

// Per-row weight under linear dropoff (row_distances_weights, _pycore.py:384-396).
__device__ __forceinline__ double row_weight(long long ci, long long cj, long long ck, double ox,
                                             double oy, double oz, double ux, double uy, double uz,
                                             double ts, const MarchParams& mp) {
    double cx = ((double)ci + 0.5) * mp.h - ox;
    double cy = ((double)cj + 0.5) * mp.h - oy;
    double cz = ((double)ck + 0.5) * mp.h - oz;
    double proj = cx * ux + cy * uy + cz * uz;
    double d = ts - proj;
    if (d < -mp.trunc) d = -mp.trunc;
    if (d > mp.trunc) d = mp.trunc;
    return d >= 0.0 ? 1.0 : (mp.trunc + d) / mp.trunc;
}

template <class P>
__device__ __forceinline__ void load_point(const P* pts, int64_t i, double& x, double& y, double& z) {
    x = (double)pts[3 * i];
    y = (double)pts[3 * i + 1];
    z = (double)pts[3 * i + 2];
}

// Pass 1: validation masks (integrate_frame, fusion.py:228-256), ray setup
// (fusion.py:262-263), band row count and frame bbox of kept rows.
template <class P, class Fe>
__global__ void k_count(const P* __restrict__ pts, int64_t n, PoseParams pp, MarchParams mp,
                        int sem_kind, const int32_t* __restrict__ labels, int num_classes,
                        const Fe* __restrict__ feats, int D, double4* __restrict__ ray,
                        int* __restrict__ cnt, FrameCtr* __restrict__ ctr) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool live = i < n;
    unsigned c_nonfinite = 0, c_range = 0, c_degen = 0, c_badlab = 0, c_used = 0;
    unsigned long long c_hits = 0, c_rows = 0;
    long long mn0 = LLONG_MAX, mn1 = LLONG_MAX, mn2 = LLONG_MAX;
    long long mx0 = LLONG_MIN, mx1 = LLONG_MIN, mx2 = LLONG_MIN;
    int budget = 0;
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
        int rows = 0;
        if (keep) {
            c_used = 1;
            double ux = dx / ts, uy = dy / ts, uz = dz / ts;
            ray[i] = make_double4(ux, uy, uz, ts);
            long long emitted = dda_walk(ox, oy, oz, ux, uy, uz, ts, mp,
                [&](long long ci, long long cj, long long ck) {
                    if (mp.wfn == 1 &&
                        !(row_weight(ci, cj, ck, ox, oy, oz, ux, uy, uz, ts, mp) > 0.0))
                        return;
                    ++rows;
                    mn0 = min(mn0, ci); mn1 = min(mn1, cj); mn2 = min(mn2, ck);
                    mx0 = max(mx0, ci); mx1 = max(mx1, cj); mx2 = max(mx2, ck);
                });
            if (emitted < 0) {
                budget = 1;
                rows = 0;
            } else {
                c_hits = (unsigned long long)emitted;
            }
            c_rows = (unsigned long long)rows;
        }
        cnt[i] = rows;
    }
    // warp-aggregated counters
    const unsigned full = 0xffffffffu;
    unsigned a_nf = __reduce_add_sync(full, c_nonfinite);
    unsigned a_rg = __reduce_add_sync(full, c_range);
    unsigned a_dg = __reduce_add_sync(full, c_degen);
    unsigned a_bl = __reduce_add_sync(full, c_badlab);
    unsigned a_us = __reduce_add_sync(full, c_used);
    unsigned a_bu = __reduce_or_sync(full, (unsigned)budget);
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
        if (a_bu) atomicOr(&ctr->err_budget, 1);
    }
}

// Pass 2: write (voxel key, point index) rows at the ray's scanned offset.
__global__ void k_fill(int64_t n, const double4* __restrict__ ray, const int* __restrict__ cnt,
                       const long long* __restrict__ off, PoseParams pp, MarchParams mp, KeyPack kp,
                       unsigned long long* __restrict__ keys, int* __restrict__ rid) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || cnt[i] == 0) return;
    const double4 r = ray[i];
    const double ox = pp.t[0], oy = pp.t[1], oz = pp.t[2];
    long long o = off[i];
    dda_walk(ox, oy, oz, r.x, r.y, r.z, r.w, mp, [&](long long ci, long long cj, long long ck) {
        if (mp.wfn == 1 && !(row_weight(ci, cj, ck, ox, oy, oz, r.x, r.y, r.z, r.w, mp) > 0.0))
            return;
        unsigned long long dx = (unsigned long long)(ci - kp.mn[0]);
        unsigned long long dy = (unsigned long long)(cj - kp.mn[1]);
        unsigned long long dz = (unsigned long long)(ck - kp.mn[2]);
        keys[o] = (dx << kp.byz) | (dy << kp.bz) | dz;
        rid[o] = (int)i;
        ++o;
    });
}

template <class P, class Fe>
svx_status count_t(svx_map* m, const P* pts, int64_t n, const PoseParams& pp, const MarchParams& mp,
                   const int32_t* labels, const Fe* feats, cudaStream_t s) {
    const int T = 256;
    k_count<P, Fe><<<grid_for(n, T), T, 0, s>>>(pts, n, pp, mp, m->cfg.sem_kind, labels,
                                                m->cfg.num_classes, feats, m->payload_d,
                                                ptr<double4>(m->ray), ptr<int>(m->cnt),
                                                ptr<FrameCtr>(m->ctr));
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

svx_status launch_count(svx_map* m, const void* pts, int pts_f64, int64_t n, const PoseParams& pp,
                        const int32_t* labels, const void* feats, int feats_f64,
                        cudaStream_t s) {
    MarchParams mp = march_params(m);
    if (pts_f64) {
        if (feats_f64)
            return count_t(m, (const double*)pts, n, pp, mp, labels, (const double*)feats, s);
        return count_t(m, (const double*)pts, n, pp, mp, labels, (const float*)feats, s);
    }
    if (feats_f64)
        return count_t(m, (const float*)pts, n, pp, mp, labels, (const double*)feats, s);
    return count_t(m, (const float*)pts, n, pp, mp, labels, (const float*)feats, s);
}

svx_status launch_fill(svx_map* m, int64_t n, const PoseParams& pp, const KeyPack& kp,
                       cudaStream_t s) {
    MarchParams mp = march_params(m);
    const int T = 256;
    k_fill<<<grid_for(n, T), T, 0, s>>>(n, ptr<double4>(m->ray), ptr<int>(m->cnt),
                                        ptr<long long>(m->off), pp, mp, kp,
                                        ptr<unsigned long long>(m->keys0), ptr<int>(m->rid0));
    SVX_LAUNCHED();
    return SVX_OK;
}

}  // namespace svx

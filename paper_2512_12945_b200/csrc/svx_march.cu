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
// (_core.pyx:707-753): every band row inserts its voxel key into a per-frame
// open-addressing table and bumps that voxel's row count (K1); a pass over
// the table compacts the touched voxels and gives each a contiguous row
// segment (K2); every row then drops its point index into its voxel's
// segment (K3).  Rows inside a segment are put back into point order by the
// update kernels -- the sequential per-voxel sums are all the reference's
// sort order is needed for.
//
// Bounded bands (no space carving) split K1 into a compute-only walk that
// writes each row's key into a per-ray slot array (K1a) and a flat,
// fully parallel insert over all row slots (K1b); carving bands are
// unbounded, so their walk inserts as it goes and K3 re-walks them.
//
// All per-frame values are read from the device-side FrameCtr so one
// captured CUDA graph replays every frame; counters go to per-CTA partial
// records that the gate reduces (no same-address atomics).
#include <math.h>

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "svx_internal.cuh"

namespace svx {
namespace {

constexpr int kMarchThreads = 256;

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

// Frame-table insert: speculative CAS on the home slot, linear probing on a
// collision.  Returns the slot or -1 when the table is full.
__device__ __forceinline__ long long frame_insert(unsigned long long* keys, long long mask,
                                                  unsigned long long key) {
    long long pos = (long long)(key_hash(key) & (unsigned long long)mask);
    unsigned long long cur = atomicCAS(&keys[pos], kKeyEmpty, key);
    if (cur == kKeyEmpty || cur == key) return pos;
    for (long long probe = 0; probe < mask; ++probe) {
        pos = (pos + 1) & mask;
        cur = keys[pos];
        if (cur == key) return pos;
        if (cur == kKeyEmpty) {
            cur = atomicCAS(&keys[pos], kKeyEmpty, key);
            if (cur == kKeyEmpty || cur == key) return pos;
        }
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
__device__ __forceinline__ void load_point(const P* pts, long long i, double& x, double& y,
                                           double& z) {
    x = (double)pts[3 * i];
    y = (double)pts[3 * i + 1];
    z = (double)pts[3 * i + 2];
}

// Thread-local counters of the march; reduced per CTA at the end.
struct Tally {
    unsigned long long nonfinite = 0, range = 0, degenerate = 0, bad_label = 0, used = 0,
                       band_hits = 0, rows = 0;
    long long mn[3] = {LLONG_MAX, LLONG_MAX, LLONG_MAX};
    long long mx[3] = {LLONG_MIN, LLONG_MIN, LLONG_MIN};
    int errs = 0;
};

struct MaxOp {
    __device__ long long operator()(long long a, long long b) const { return a > b ? a : b; }
};
struct MinOp {
    __device__ long long operator()(long long a, long long b) const { return a < b ? a : b; }
};
struct OrOp {
    __device__ int operator()(int a, int b) const { return a | b; }
};

__device__ __forceinline__ void write_partial(const Tally& t, MarchPartial* out) {
    using RU = cub::BlockReduce<unsigned long long, kMarchThreads>;
    using RL = cub::BlockReduce<long long, kMarchThreads>;
    using RI = cub::BlockReduce<int, kMarchThreads>;
    __shared__ union {
        typename RU::TempStorage u;
        typename RL::TempStorage l;
        typename RI::TempStorage i;
    } tmp;
    __shared__ MarchPartial res;
    const unsigned long long uv[7] = {t.nonfinite, t.range, t.degenerate, t.bad_label,
                                      t.used, t.band_hits, t.rows};
    unsigned long long* ud[7] = {&res.nonfinite, &res.range, &res.degenerate, &res.bad_label,
                                 &res.used, &res.band_hits, &res.rows};
    for (int q = 0; q < 7; ++q) {
        unsigned long long v = RU(tmp.u).Sum(uv[q]);
        if (threadIdx.x == 0) *ud[q] = v;
        __syncthreads();
    }
    for (int a = 0; a < 3; ++a) {
        long long v = RL(tmp.l).Reduce(t.mn[a], MinOp());
        if (threadIdx.x == 0) res.bbox_min[a] = v;
        __syncthreads();
        v = RL(tmp.l).Reduce(t.mx[a], MaxOp());
        if (threadIdx.x == 0) res.bbox_max[a] = v;
        __syncthreads();
    }
    int e = RI(tmp.i).Reduce(t.errs, OrOp());
    if (threadIdx.x == 0) {
        res.errs = e;
        res.pad = 0;
        *out = res;
    }
}

// Shared front half of the march for one point: validation masks
// (integrate_frame, fusion.py:228-256) and ray setup (fusion.py:262-263).
// Returns true when the point is kept; r = (u, t_surf).
template <class P, class Fe>
__device__ __forceinline__ bool prepare_ray(long long i, const FrameParams& fp, double max_range,
                                            int sem_kind, int num_classes, int D, Tally& t,
                                            double4& r) {
    double x, y, z;
    load_point((const P*)fp.pts, i, x, y, z);
    const PoseParams& pp = fp.pp;
    double wx, wy, wz;
    if (pp.sensor) {
        wx = ((pp.R[0] * x + pp.R[1] * y) + pp.R[2] * z) + pp.t[0];
        wy = ((pp.R[3] * x + pp.R[4] * y) + pp.R[5] * z) + pp.t[1];
        wz = ((pp.R[6] * x + pp.R[7] * y) + pp.R[8] * z) + pp.t[2];
    } else {
        wx = x; wy = y; wz = z;
    }
    bool finite = isfinite(wx) && isfinite(wy) && isfinite(wz);
    double dx = wx - pp.t[0], dy = wy - pp.t[1], dz = wz - pp.t[2];
    double ts = sqrt((dx * dx + dy * dy) + dz * dz);
    if (!isfinite(ts)) ts = INFINITY;
    bool degenerate = finite && ts == 0.0;
    bool in_range = ts <= max_range;
    bool keep = finite && !degenerate && in_range;
    t.nonfinite += !finite;
    t.degenerate += degenerate;
    t.range += finite && !degenerate && !in_range;
    if (sem_kind == SVX_SEM_CLOSED) {
        int lab = fp.labels[i];
        bool good = lab >= 1 && lab <= num_classes;
        t.bad_label += keep && !good;
        keep = keep && good;
    } else if (sem_kind == SVX_SEM_OPEN) {
        bool good = true;
        const Fe* f = (const Fe*)fp.feats + i * D;
        for (int c = 0; c < D; ++c) good = good && isfinite((double)f[c]);
        t.bad_label += keep && !good;
        keep = keep && good;
    }
    r = make_double4(0.0, 0.0, 0.0, -1.0);
    if (keep) {
        t.used += 1;
        r = make_double4(dx / ts, dy / ts, dz / ts, ts);
    }
    return keep;
}

// K1a (bounded bands): compute-only walk; row keys go to rowkey[i*maxrows+j].
template <class P, class Fe>
__global__ void __launch_bounds__(kMarchThreads) k_walk(MarchParams mp, int sem_kind,
                                                        int num_classes, int D,
                                                        double4* __restrict__ ray,
                                                        int* __restrict__ rcnt,
                                                        unsigned long long* __restrict__ rowkey,
                                                        MarchPartial* __restrict__ partials,
                                                        const FrameCtr* __restrict__ ctr) {
    const FrameParams fp = ctr->p;
    const long long n = fp.n;
    const int maxrows = fp.maxrows;
    const double ox = fp.pp.t[0], oy = fp.pp.t[1], oz = fp.pp.t[2];
    Tally t;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double4 r;
        int rows = 0;
        if (prepare_ray<P, Fe>(i, fp, mp.max_range, sem_kind, num_classes, D, t, r)) {
            unsigned long long* rk = rowkey + i * maxrows;
            long long emitted = dda_walk(ox, oy, oz, r.x, r.y, r.z, r.w, mp,
                [&](long long ci, long long cj, long long ck) {
                    if (!row_kept(ci, cj, ck, ox, oy, oz, r, mp)) return;
                    t.rows += 1;
                    t.mn[0] = min(t.mn[0], ci); t.mn[1] = min(t.mn[1], cj); t.mn[2] = min(t.mn[2], ck);
                    t.mx[0] = max(t.mx[0], ci); t.mx[1] = max(t.mx[1], cj); t.mx[2] = max(t.mx[2], ck);
                    if (rows >= maxrows) {
                        t.errs |= 8;
                        return;
                    }
                    long long ox_ = ci - fp.kp.base[0], oy_ = cj - fp.kp.base[1], oz_ = ck - fp.kp.base[2];
                    unsigned long long key = kKeyEmpty;
                    if (((ox_ | oy_ | oz_) & ~kPackMask) != 0) t.errs |= 2;
                    else key = pack_key(ox_, oy_, oz_);
                    rk[rows++] = key;
                });
            if (emitted < 0) {
                t.errs |= 1;
                r.w = -1.0;
                rows = 0;
            } else {
                t.band_hits += (unsigned long long)emitted;
            }
        }
        ray[i] = r;
        rcnt[i] = rows;
    }
    write_partial(t, partials + blockIdx.x);
}

// K1b (bounded bands): one thread per row slot inserts the key and counts it.
__global__ void __launch_bounds__(256) k_insert(const int* __restrict__ rcnt,
                                                const unsigned long long* __restrict__ rowkey,
                                                int* __restrict__ rowslot, unsigned long long* fkey,
                                                unsigned* fcount, FrameCtr* ctr) {
    const long long n = ctr->p.n;
    const int maxrows = ctr->p.maxrows;
    const long long fmask = ctr->p.fmask;
    const long long total = n * maxrows;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long i = t / maxrows;
        const int j = (int)(t - i * maxrows);
        if (j >= rcnt[i]) continue;
        const unsigned long long key = rowkey[t];
        if (key == kKeyEmpty) continue;          // pack error: the frame is re-run
        const long long s = frame_insert(fkey, fmask, key);
        if (s < 0) {
            atomicOr(&ctr->err_probe, 1);
            continue;
        }
        atomicAdd(&fcount[s], 1u);
        rowslot[t] = (int)s;
    }
}

// K1 (space carving, unbounded bands): walk and insert in one pass.
template <class P, class Fe>
__global__ void __launch_bounds__(kMarchThreads) k_walk_insert(
    MarchParams mp, int sem_kind, int num_classes, int D, double4* __restrict__ ray,
    int* __restrict__ rcnt, unsigned long long* fkey, unsigned* fcount,
    MarchPartial* __restrict__ partials, const FrameCtr* __restrict__ ctr) {
    const FrameParams fp = ctr->p;
    const long long n = fp.n;
    const double ox = fp.pp.t[0], oy = fp.pp.t[1], oz = fp.pp.t[2];
    Tally t;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double4 r;
        int rows = 0;
        if (prepare_ray<P, Fe>(i, fp, mp.max_range, sem_kind, num_classes, D, t, r)) {
            long long emitted = dda_walk(ox, oy, oz, r.x, r.y, r.z, r.w, mp,
                [&](long long ci, long long cj, long long ck) {
                    if (!row_kept(ci, cj, ck, ox, oy, oz, r, mp)) return;
                    t.rows += 1;
                    t.mn[0] = min(t.mn[0], ci); t.mn[1] = min(t.mn[1], cj); t.mn[2] = min(t.mn[2], ck);
                    t.mx[0] = max(t.mx[0], ci); t.mx[1] = max(t.mx[1], cj); t.mx[2] = max(t.mx[2], ck);
                    long long ox_ = ci - fp.kp.base[0], oy_ = cj - fp.kp.base[1], oz_ = ck - fp.kp.base[2];
                    if (((ox_ | oy_ | oz_) & ~kPackMask) != 0) {
                        t.errs |= 2;
                        return;
                    }
                    if (t.errs & 4) return;   // table full: the frame is re-run anyway
                    long long s = frame_insert(fkey, fp.fmask, pack_key(ox_, oy_, oz_));
                    if (s < 0) {
                        t.errs |= 4;
                        return;
                    }
                    atomicAdd(&fcount[s], 1u);
                    ++rows;
                });
            if (emitted < 0) {
                t.errs |= 1;
                r.w = -1.0;
                rows = 0;
            } else {
                t.band_hits += (unsigned long long)emitted;
            }
        }
        ray[i] = r;
        rcnt[i] = rows;
    }
    write_partial(t, partials + blockIdx.x);
}

constexpr int kCompactThreads = 256;
constexpr int kCompactTile = kCompactThreads * 4;
constexpr int kCompactBlocks = 148 * 2;

// K2a: per-CTA totals over a contiguous table chunk: touched voxels, listed
// voxels (all, or only multi-row ones when single-row voxels are updated
// inline by the scatter) and the rows of the listed ones.
__global__ void __launch_bounds__(kCompactThreads) k_compact_count(
    const unsigned long long* __restrict__ fkey, const unsigned* __restrict__ fcount,
    long long fcap, long long chunk, int multi_only, unsigned long long* __restrict__ part) {
    using R = cub::BlockReduce<unsigned long long, kCompactThreads>;
    __shared__ typename R::TempStorage tmp;
    const long long lo = (long long)blockIdx.x * chunk;
    const long long hi = min(fcap, lo + chunk);
    unsigned long long occ = 0, listed = 0, rows = 0;
    for (long long s = lo + threadIdx.x; s < hi; s += kCompactThreads) {
        const unsigned long long k = fkey[s];
        if (k != kKeyEmpty) {
            occ += 1;
            const unsigned c = fcount[s];
            if (!multi_only || c > 1u) {
                listed += 1;
                rows += c;
            }
        }
    }
    unsigned long long packed = R(tmp).Sum((listed << 40) | rows);
    __syncthreads();
    unsigned long long o = R(tmp).Sum(occ);
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = packed;
        part[2 * blockIdx.x + 1] = o;
    }
}

__device__ void gate_body(const MarchPartial* __restrict__ parts, int nparts, FrameCtr* ctr);

// K2b: each CTA scans its chunk again with its exclusive base; listed
// voxels are compacted into ulist/ukey and get contiguous row segments.
__global__ void __launch_bounds__(kCompactThreads) k_compact_write(
    const unsigned long long* __restrict__ fkey, const unsigned* __restrict__ fcount,
    unsigned* __restrict__ foff, long long fcap, long long chunk, int multi_only,
    const unsigned long long* __restrict__ part, int* __restrict__ ulist,
    unsigned long long* __restrict__ ukey, const MarchPartial* __restrict__ mparts, int nmparts,
    FrameCtr* ctr) {
    using Scan = cub::BlockScan<unsigned long long, kCompactThreads>;
    using R = cub::BlockReduce<unsigned long long, kCompactThreads>;
    __shared__ union {
        typename Scan::TempStorage scan;
        typename R::TempStorage red;
    } tmp;
    __shared__ unsigned long long s_base, s_occ;
    const unsigned long long ucap = ctr->p.ucap;
    const unsigned long long low40 = (1ULL << 40) - 1;
    // exclusive base of this CTA: sum of the earlier CTAs' packed totals
    unsigned long long acc = 0, occ_all = 0;
    const bool last = blockIdx.x == gridDim.x - 1;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += kCompactThreads) {
        if (b < (int)blockIdx.x) acc += part[2 * b];
        if (last) occ_all += part[2 * b + 1];
    }
    acc = R(tmp.red).Sum(acc);
    __syncthreads();
    occ_all = R(tmp.red).Sum(occ_all);
    if (threadIdx.x == 0) {
        s_base = acc;
        s_occ = occ_all;
    }
    __syncthreads();
    unsigned long long base = s_base;
    const long long lo = (long long)blockIdx.x * chunk;
    const long long hi = min(fcap, lo + chunk);
    for (long long t0 = lo; t0 < hi; t0 += kCompactTile) {
        const long long s0 = t0 + (long long)threadIdx.x * 4;
        unsigned long long kk[4];
        unsigned cc[4];
        bool li[4];
        unsigned cnt = 0, rows = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const long long s = s0 + q;
            kk[q] = s < hi ? fkey[s] : kKeyEmpty;
            cc[q] = kk[q] != kKeyEmpty ? fcount[s] : 0u;
            li[q] = kk[q] != kKeyEmpty && (!multi_only || cc[q] > 1u);
            cnt += li[q];
            rows += li[q] ? cc[q] : 0u;
        }
        unsigned long long pre, total;
        __syncthreads();
        Scan(tmp.scan).ExclusiveSum(((unsigned long long)cnt << 40) | rows, pre, total);
        unsigned long long u = (base >> 40) + (pre >> 40);
        unsigned long long r = (base & low40) + (pre & low40);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (!li[q]) continue;
            const long long s = s0 + q;
            if (u < ucap) {
                ulist[u] = (int)s;
                ukey[u] = kk[q];
            }
            foff[s] = (unsigned)r;
            ++u;
            r += cc[q];
        }
        base += total;
    }
    if (last) {
        if (threadIdx.x == 0) {
            ctr->n_groups = s_occ;
            ctr->n_list = base >> 40;
            ctr->rows_c = base & low40;
        }
        __syncthreads();
        gate_body(mparts, nmparts, ctr);
    }
}

// Reduce the march partials and decide, once per frame on the device, whether
// the frame may mutate the map (the reference's checks before any
// allocation, _core.pyx:661-712, :386-387).  The host reports the reason.
// Run by the last CTA of the compaction (256 threads) once the totals are in.
__device__ void gate_body(const MarchPartial* __restrict__ parts, int nparts, FrameCtr* ctr) {
    using RU = cub::BlockReduce<unsigned long long, 256>;
    using RL = cub::BlockReduce<long long, 256>;
    __shared__ union {
        typename RU::TempStorage u;
        typename RL::TempStorage l;
    } tmp;
    unsigned long long v[7] = {0, 0, 0, 0, 0, 0, 0};
    long long mn[3] = {LLONG_MAX, LLONG_MAX, LLONG_MAX}, mx[3] = {LLONG_MIN, LLONG_MIN, LLONG_MIN};
    int errs = 0;
    for (int b = threadIdx.x; b < nparts; b += 256) {
        const MarchPartial& p = parts[b];
        v[0] += p.nonfinite; v[1] += p.range; v[2] += p.degenerate; v[3] += p.bad_label;
        v[4] += p.used; v[5] += p.band_hits; v[6] += p.rows;
        for (int a = 0; a < 3; ++a) {
            mn[a] = min(mn[a], p.bbox_min[a]);
            mx[a] = max(mx[a], p.bbox_max[a]);
        }
        errs |= p.errs;
    }
    unsigned long long* dst[7] = {&ctr->nonfinite, &ctr->range, &ctr->degenerate, &ctr->bad_label,
                                  &ctr->used, &ctr->band_hits, &ctr->rows};
    for (int q = 0; q < 7; ++q) {
        unsigned long long s = RU(tmp.u).Sum(v[q]);
        if (threadIdx.x == 0) *dst[q] = s;
        __syncthreads();
    }
    for (int a = 0; a < 3; ++a) {
        long long s = RL(tmp.l).Reduce(mn[a], MinOp());
        if (threadIdx.x == 0) ctr->bbox_min[a] = s;
        __syncthreads();
        s = RL(tmp.l).Reduce(mx[a], MaxOp());
        if (threadIdx.x == 0) ctr->bbox_max[a] = s;
        __syncthreads();
    }
    errs = __reduce_or_sync(0xffffffffu, (unsigned)errs);
    __shared__ int s_err[8];
    if ((threadIdx.x & 31) == 0) s_err[threadIdx.x >> 5] = errs;
    __syncthreads();
    if (threadIdx.x != 0) return;
    for (int w = 1; w < 8; ++w) errs |= s_err[w];
    if (errs & 1) ctr->err_budget = 1;
    if (errs & 2) ctr->err_pack = 1;
    if (errs & 4) ctr->err_probe = 1;
    if (errs & 8) ctr->err_rows = 1;
    int ab = ctr->err_budget | ctr->err_pack | ctr->err_probe | ctr->err_rows;
    if (ctr->n_list > ctr->p.ucap || ctr->n_groups > ctr->p.ucap || ctr->rows_c > ctr->p.rcap) ab = 1;
    if (ctr->rows) {
        for (int a = 0; a < 3; ++a) {
            long long lo = ctr->bbox_min[a], hi = ctr->bbox_max[a];
            if (hi - lo >= (1LL << kPackBits)) ab = 1;
            if (llabs(lo) >= kCoordLimit || llabs(hi) >= kCoordLimit) ab = 1;
        }
    }
    ctr->abort = ab;
}

// K3 (bounded bands): one thread per row slot -- fully parallel.
__global__ void __launch_bounds__(256) k_scatter_flat(const int* __restrict__ rcnt,
                                                      const int* __restrict__ rowslot,
                                                      const unsigned* __restrict__ foff,
                                                      unsigned* fcur, int* __restrict__ srid,
                                                      const FrameCtr* __restrict__ ctr) {
    if (ctr->abort) return;
    const long long n = ctr->p.n;
    const int maxrows = ctr->p.maxrows;
    const long long total = n * maxrows;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
        const long long i = t / maxrows;
        const int j = (int)(t - i * maxrows);
        if (j >= rcnt[i]) continue;
        const int s = rowslot[t];
        const unsigned pos = foff[s] + atomicAdd(&fcur[s], 1u);
        srid[pos] = (int)i;
    }
}

// K3 (space carving): re-walk each ray and look its voxels up again.
__global__ void __launch_bounds__(256) k_scatter_walk(const double4* __restrict__ ray,
                                                      MarchParams mp,
                                                      const unsigned long long* __restrict__ fkey,
                                                      const unsigned* __restrict__ foff,
                                                      unsigned* fcur, int* __restrict__ srid,
                                                      const FrameCtr* __restrict__ ctr) {
    if (ctr->abort) return;
    const long long n = ctr->p.n;
    const PoseParams pp = ctr->p.pp;
    const KeyPack kp = ctr->p.kp;
    const long long fmask = ctr->p.fmask;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double4 r = ray[i];
        if (!(r.w >= 0.0)) continue;
        const double ox = pp.t[0], oy = pp.t[1], oz = pp.t[2];
        dda_walk(ox, oy, oz, r.x, r.y, r.z, r.w, mp, [&](long long ci, long long cj, long long ck) {
            if (!row_kept(ci, cj, ck, ox, oy, oz, r, mp)) return;
            unsigned long long key = pack_key(ci - kp.base[0], cj - kp.base[1], ck - kp.base[2]);
            long long s = frame_find(fkey, fmask, key);
            unsigned pos = foff[s] + atomicAdd(&fcur[s], 1u);
            srid[pos] = (int)i;
        });
    }
}

template <class P, class Fe>
svx_status march_t(svx_map* m, cudaStream_t s) {
    const MarchParams mp = march_params(m);
    MarchPartial* parts = ptr<MarchPartial>(m->partials);
    if (m->maxrows > 0) {
        k_walk<P, Fe><<<kMarchBlocks, kMarchThreads, 0, s>>>(
            mp, m->cfg.sem_kind, m->cfg.num_classes, m->payload_d, ptr<double4>(m->ray),
            ptr<int>(m->rcnt), ptr<unsigned long long>(m->rowkey), parts, ptr<FrameCtr>(m->ctr));
        SVX_LAUNCHED();
        k_insert<<<kPersistentBlocks * 2, 256, 0, s>>>(
            ptr<int>(m->rcnt), ptr<unsigned long long>(m->rowkey), ptr<int>(m->rowslot),
            ptr<unsigned long long>(m->fkey), ptr<unsigned>(m->fcount), ptr<FrameCtr>(m->ctr));
        SVX_LAUNCHED();
    } else {
        k_walk_insert<P, Fe><<<kMarchBlocks, kMarchThreads, 0, s>>>(
            mp, m->cfg.sem_kind, m->cfg.num_classes, m->payload_d, ptr<double4>(m->ray),
            ptr<int>(m->rcnt), ptr<unsigned long long>(m->fkey), ptr<unsigned>(m->fcount), parts,
            ptr<FrameCtr>(m->ctr));
        SVX_LAUNCHED();
    }
    return SVX_OK;
}

}  // namespace

MarchParams march_params(const svx_map* m) {
    MarchParams mp;
    mp.h = m->cfg.voxel_size;
    mp.trunc = m->cfg.truncation;
    mp.max_range = m->cfg.max_range;
    mp.carving = m->cfg.space_carving;
    mp.wfn = m->cfg.weight_fn;
    return mp;
}

svx_status launch_march(svx_map* m, int pts_f64, int feats_f64, cudaStream_t s) {
    if (pts_f64) {
        if (feats_f64) return march_t<double, double>(m, s);
        return march_t<double, float>(m, s);
    }
    if (feats_f64) return march_t<float, double>(m, s);
    return march_t<float, float>(m, s);
}

svx_status launch_compact(svx_map* m, cudaStream_t s) {
    long long chunk = (m->fcap + kCompactBlocks - 1) / kCompactBlocks;
    chunk = (chunk + kCompactTile - 1) / kCompactTile * kCompactTile;
    const int blocks = (int)((m->fcap + chunk - 1) / chunk);
    unsigned long long* part = ptr<unsigned long long>(m->partials) +
                               (sizeof(MarchPartial) * kMarchBlocks) / sizeof(unsigned long long);
    const int multi_only = inline_singles(m);
    k_compact_count<<<blocks, kCompactThreads, 0, s>>>(
        ptr<unsigned long long>(m->fkey), ptr<unsigned>(m->fcount), m->fcap, chunk, multi_only, part);
    SVX_LAUNCHED();
    k_compact_write<<<blocks, kCompactThreads, 0, s>>>(
        ptr<unsigned long long>(m->fkey), ptr<unsigned>(m->fcount), ptr<unsigned>(m->foff), m->fcap,
        chunk, multi_only, part, ptr<int>(m->ulist), ptr<unsigned long long>(m->ukey),
        ptr<MarchPartial>(m->partials), kMarchBlocks, ptr<FrameCtr>(m->ctr));
    SVX_LAUNCHED();
    return SVX_OK;
}

svx_status launch_scatter(svx_map* m, bool flat, cudaStream_t s) {
    if (flat) {
        k_scatter_flat<<<kPersistentBlocks * 2, 256, 0, s>>>(
            ptr<int>(m->rcnt), ptr<int>(m->rowslot), ptr<unsigned>(m->foff), ptr<unsigned>(m->fcur),
            ptr<int>(m->srid), ptr<FrameCtr>(m->ctr));
    } else {
        k_scatter_walk<<<kPersistentBlocks, 256, 0, s>>>(
            ptr<double4>(m->ray), march_params(m), ptr<unsigned long long>(m->fkey),
            ptr<unsigned>(m->foff), ptr<unsigned>(m->fcur), ptr<int>(m->srid),
            ptr<FrameCtr>(m->ctr));
    }
    SVX_LAUNCHED();
    return SVX_OK;
}

size_t partials_bytes() {
    return sizeof(MarchPartial) * kMarchBlocks + sizeof(unsigned long long) * kCompactBlocks * 2;
}

}  // namespace svx

// svx_march.cu -- per-point preparation and the fp64 band ray-march (K1),
// plus the frame gate.
//
// Compiled with -fmad=false: every double expression is evaluated with the
// operation order and IEEE round-to-nearest steps of the reference's
// -ffp-contract=off C++ (_core.pyx:478-579, pkg/setup.py:14) and its numpy
// twin (_pycore.py:326-396), so band membership and per-row distances are
// bit-identical.
//
// The walk only computes: each kept row's voxel key and ray index are
// written to dense row arrays (bounded bands: 128-ray tiles staged in shared
// memory, one atomic per tile; unbounded bands, e.g. space carving: count,
// scan, re-walk).  The
// gate then applies the reference's pre-allocation checks before anything
// touches the map.  Grouping rows by voxel happens in svx_resolve.cu.
//
// All per-frame values are read from the device-side FrameCtr so one
// captured CUDA graph replays every frame; counters go to per-CTA partial
// records that the gate reduces (no same-address atomics).
#include <math.h>

#include <cub/block/block_reduce.cuh>
#include <cub/device/device_scan.cuh>

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

// Reduce the CTA's tallies (warp shuffles, one shared-memory round) and add
// them to the frame counters: sums by RED, the row bounding box by atomic
// min/max, error bits by atomic or.  No per-CTA partial records.
template <int kThreads>
__device__ __forceinline__ void publish_tally(const Tally& t, FrameCtr* ctr) {
    constexpr int kWarps = kThreads / 32;
    __shared__ unsigned long long s_sum[kWarps][7];
    __shared__ long long s_mn[kWarps][3], s_mx[kWarps][3];
    __shared__ int s_err[kWarps];
    unsigned long long v[7] = {t.nonfinite, t.range, t.degenerate, t.bad_label, t.used, t.band_hits, t.rows};
    long long mn[3] = {t.mn[0], t.mn[1], t.mn[2]}, mx[3] = {t.mx[0], t.mx[1], t.mx[2]};
    int e = t.errs;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int q = 0; q < 7; ++q) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            mn[a] = min(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
            mx[a] = max(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
        }
        e |= __shfl_xor_sync(0xffffffffu, e, o);
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int q = 0; q < 7; ++q) s_sum[w][q] = v[q];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            s_mn[w][a] = mn[a];
            s_mx[w][a] = mx[a];
        }
        s_err[w] = e;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int x = 1; x < kWarps; ++x) {
            for (int q = 0; q < 7; ++q) v[q] += s_sum[x][q];
            for (int a = 0; a < 3; ++a) {
                mn[a] = min(mn[a], s_mn[x][a]);
                mx[a] = max(mx[a], s_mx[x][a]);
            }
            e |= s_err[x];
        }
        unsigned long long* dst[7] = {&ctr->nonfinite, &ctr->range, &ctr->degenerate, &ctr->bad_label,
                                      &ctr->used, &ctr->band_hits, &ctr->rows};
        for (int q = 0; q < 7; ++q)
            if (v[q]) atomicAdd(dst[q], v[q]);
        if (v[6]) {
            for (int a = 0; a < 3; ++a) {
                atomicMin(&ctr->bbox_min[a], mn[a]);
                atomicMax(&ctr->bbox_max[a], mx[a]);
            }
        }
        if (e) {
            if (e & 1) atomicOr(&ctr->err_budget, 1);
            if (e & 2) atomicOr(&ctr->err_pack, 1);
            if (e & 8) atomicOr(&ctr->err_rows, 1);
        }
    }
}

// Open-set validation (features all finite), warp-cooperative.  The warp's
// points are consecutive (i = tile base + lane) and the valid ones a prefix,
// so their feature rows are one contiguous block: the lanes stream it with
// independent 16-byte loads, several in flight per lane, and collect a
// bit per bad row; one OR-reduction gives every lane its verdict.  (The
// features are the frame's largest input -- 2.8 GB at cfg5 -- and this scan
// is its first read.)  Other lane patterns take the row-by-row loop.  Called
// by all 32 lanes; `has` = this lane has a point to check.
#ifndef SVX_FEAT_UNROLL
#define SVX_FEAT_UNROLL 8
#endif
__device__ __forceinline__ bool finite4(const float4 v) {
    const unsigned e = 0x7f800000u;
    return ((__float_as_uint(v.x) & e) != e) & ((__float_as_uint(v.y) & e) != e) &
           ((__float_as_uint(v.z) & e) != e) & ((__float_as_uint(v.w) & e) != e);
}

template <class Fe>
__device__ __forceinline__ bool warp_feats_finite(const Fe* __restrict__ feats, int D, long long i,
                                                  bool has) {
    const int lane = threadIdx.x & 31;
    const unsigned todo = __ballot_sync(0xffffffffu, has);
    if (!todo) return true;
    if constexpr (sizeof(Fe) == 4) {
    const long long i0 = __shfl_sync(0xffffffffu, i, 0);
    const bool contiguous = __all_sync(0xffffffffu, i == i0 + lane) && (todo & (todo + 1u)) == 0u;
    if ((D & 3) == 0 && D < 46336 && contiguous) {
        const int nrows = __popc(todo);
        const unsigned d4 = (unsigned)D >> 2;
        const unsigned total = (unsigned)nrows * d4;       // float4 chunks of the block
        // row = c / d4 by a multiply-high: exact while c * d4 < 2^32 (c < 32 d4, D < 46336)
        const unsigned magic = d4 > 1u ? (unsigned)((0x100000000ULL + d4 - 1) / d4) : 0u;
        const float4* f4 = reinterpret_cast<const float4*>(feats + i0 * D);
        unsigned bad = 0u;
        for (unsigned c0 = lane; c0 < total; c0 += 32u * SVX_FEAT_UNROLL) {
            float4 v[SVX_FEAT_UNROLL];
#pragma unroll
            for (int u = 0; u < SVX_FEAT_UNROLL; ++u) {
                const unsigned c = c0 + 32u * u;
                v[u] = c < total ? __ldg(f4 + c) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < SVX_FEAT_UNROLL; ++u) {
                const unsigned c = c0 + 32u * u;
                if (!finite4(v[u])) bad |= 1u << (d4 > 1u ? __umulhi(c, magic) : c);
            }
        }
        bad = __reduce_or_sync(0xffffffffu, bad);
        return ((bad >> lane) & 1u) == 0u;
    }
    }
    bool mine = true;
    unsigned left = todo;
    while (left) {
        const int src = __ffs(left) - 1;
        left &= left - 1;
        const long long pi = __shfl_sync(0xffffffffu, i, src);
        const Fe* f = feats + pi * D;
        bool ok = true;
        if (sizeof(Fe) == 4 && (D & 3) == 0) {
            const float4* f4 = reinterpret_cast<const float4*>(f);
            for (int c = lane; c < (D >> 2); c += 32) ok = ok && finite4(__ldg(f4 + c));
        } else {
            for (int c = lane; c < D; c += 32) ok = ok && isfinite((double)f[c]);
        }
        ok = __all_sync(0xffffffffu, ok);
        if (lane == src) mine = ok;
    }
    return mine;
}

// Shared front half of the march for one point: validation masks
// (integrate_frame, fusion.py:228-256) and ray setup (fusion.py:262-263).
// Returns true when the point is kept; r = (u, t_surf).
template <class P, class Fe>
__device__ __forceinline__ bool prepare_ray(long long i, const FrameParams& fp, double max_range,
                                            int sem_kind, int num_classes, int D, Tally& t,
                                            double4& r, bool feats_ok = true,
                                            int* lab_out = nullptr) {
    double x, y, z;
    load_point((const P*)fp.pts, i, x, y, z);
    const PoseParams& pp = fp.pp;
    double wx, wy, wz;
    if (pp.sensor) {
        wx = world_coord(pp.R, pp.t[0], x, y, z, pp.single);
        wy = world_coord(pp.R + 3, pp.t[1], x, y, z, pp.single);
        wz = world_coord(pp.R + 6, pp.t[2], x, y, z, pp.single);
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
        const int lab = fp.labels[i];   // read once: may be zero-copy host memory
        if (lab_out) *lab_out = lab;
        bool good = lab >= 1 && lab <= num_classes;
        t.bad_label += keep && !good;
        keep = keep && good;
    } else if (sem_kind == SVX_SEM_OPEN) {
        const bool good = feats_ok;   // warp_feats_finite, evaluated by the caller
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

__device__ void gate_body(FrameCtr* ctr);
#ifndef SVX_WALK_FENCE1
#define SVX_WALK_FENCE1 1
#endif

// Every CTA of a walk adds its tallies; the last one to finish runs the gate.
template <int kThreads>
__device__ __forceinline__ void finish_walk(const Tally& t, MarchPartial*, FrameCtr* ctr) {
    publish_tally<kThreads>(t, ctr);
#if SVX_WALK_FENCE1
    // thread 0 published this CTA's tallies: it alone fences before counting
    // the CTA done (the rows reach the next kernel through the kernel boundary)
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&ctr->walk_done, 1u) == gridDim.x - 1) {
            __threadfence();
            gate_body(ctr);
        }
    }
#else
    __shared__ bool s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&ctr->walk_done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
        __threadfence();
        gate_body(ctr);
    }
#endif
}

// Asynchronous frames with device inputs: the frame's own copy of its
// points / labels (a frame that has to be re-run after a pool or slot
// overflow is re-run from it, whatever the caller did to its buffers since).
template <class P>
__device__ __forceinline__ void stage_inputs(const FrameParams& fp, int sem_kind) {
    const long long n = fp.n;
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const P* src = (const P*)fp.pts;
    P* dst = (P*)fp.stage_pts;
    for (long long e = t0; e < 3 * n; e += stride) dst[e] = src[e];
    if (sem_kind == SVX_SEM_CLOSED)
        for (long long e = t0; e < n; e += stride) fp.stage_lab[e] = fp.labels[e];
}

// K1 (bounded bands): compute-only walk over 128-ray tiles.  Each ray's row
// keys are staged in shared memory; a block scan packs the tile's rows and
// one atomic per tile reserves their place in the dense row arrays, which
// are then written coalesced (rowkey, rowray).
#ifndef SVX_TILE_RAYS
#define SVX_TILE_RAYS 128
#endif
#ifndef SVX_WALK_MINB
#define SVX_WALK_MINB 4
#endif
#ifndef SVX_WALK_PREFETCH
#define SVX_WALK_PREFETCH 0   // measured: +1.3 us walk, no resolve gain
#endif
constexpr int kTileRays = SVX_TILE_RAYS;

// Slot mode also writes each row's clamped distance d (row_distances_weights,
// _pycore.py:384-396, the same expression K5 would evaluate) and its point's
// label, so the slot update needs no gathers.
template <class P, class Fe>
__global__ void __launch_bounds__(kTileRays, SVX_WALK_MINB) k_walk(MarchParams mp, int sem_kind, int num_classes,
                                                    int D, double4* __restrict__ ray,
                                                    int* __restrict__ rcnt,
                                                    unsigned long long* __restrict__ rowkey,
                                                    int* __restrict__ rowray,
                                                    double* __restrict__ rowd,
                                                    int* __restrict__ rowlab,
                                                    MarchPartial* __restrict__ partials,
                                                    FrameCtr* __restrict__ ctr,
                                                    const int4* __restrict__ htab,
                                                    const __grid_constant__ FrameParams fpk) {
    grid_dep_wait();
    __shared__ FrameCtr s_ctr_;
    load_frame_params(ctr, s_ctr_, fpk);
    KSpan _ks(&s_ctr_, ctr, kSpanWalk);
    using Scan = cub::BlockScan<int, kTileRays>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ unsigned long long s_base;
    __shared__ int s_off[kTileRays];
    __shared__ double4 s_ray[kTileRays];
    __shared__ int s_lab[kTileRays];
    extern __shared__ unsigned long long s_keys[];   // kTileRays * maxrows keys, then row owners
    const FrameParams& fp = s_ctr_.p;
    const long long n = fp.n;
    const int maxrows = fp.maxrows;
    const bool slots = fp.slots != 0;
    const unsigned long long rcap = fp.rcap;
    unsigned char* s_own = reinterpret_cast<unsigned char*>(s_keys + (size_t)kTileRays * maxrows);
    const double ox = fp.pp.t[0], oy = fp.pp.t[1], oz = fp.pp.t[2];
    Tally t;
    if (fp.stage_pts) stage_inputs<P>(fp, sem_kind);
    // queued behind a frame that needs the host: stage only (the gate aborts)
    const long long tiles = s_ctr_.poison ? 0 : (n + kTileRays - 1) / kTileRays;
    for (long long tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const long long i = tile * kTileRays + threadIdx.x;
        int rows = 0;
        unsigned long long* rk = s_keys + (size_t)threadIdx.x * maxrows;
        const bool fok = sem_kind != SVX_SEM_OPEN ||
                         warp_feats_finite<Fe>((const Fe*)fp.feats, D, i, i < n);
        int lab_i = 0;
        if (i < n) {
            double4 r;
            if (prepare_ray<P, Fe>(i, fp, mp.max_range, sem_kind, num_classes, D, t, r, fok,
                                   &lab_i)) {
                long long f0 = 0, f1 = 0, f2 = 0, l0 = 0, l1 = 0, l2 = 0;
                int nk = 0;
                int pl0 = INT_MIN, pl1 = INT_MIN, pl2 = INT_MIN;   // last prefetched leaf
                long long emitted = dda_walk(ox, oy, oz, r.x, r.y, r.z, r.w, mp,
                    [&](long long ci, long long cj, long long ck) {
                        if (!row_kept(ci, cj, ck, ox, oy, oz, r, mp)) return;
                        t.rows += 1;
                        // cells are monotonic per axis along a ray: its first and
                        // last kept cells bound the band
                        if (nk == 0) { f0 = ci; f1 = cj; f2 = ck; }
                        l0 = ci; l1 = cj; l2 = ck;
                        ++nk;
                        if (rows >= maxrows) {
                            t.errs |= 8;
                            return;
                        }
                        long long ox_ = ci - fp.kp.base[0], oy_ = cj - fp.kp.base[1], oz_ = ck - fp.kp.base[2];
                        unsigned long long key = kKeyEmpty;
                        if (((ox_ | oy_ | oz_) & ~kPackMask) != 0) t.errs |= 2;
                        else key = pack_key(ox_, oy_, oz_);
                        rk[rows++] = key;
#if SVX_WALK_PREFETCH
                        // warm the leaf hash slot K2 will probe for this row (the walk
                        // is compute bound; its DRAM is idle)
                        {
                            const int la = (int)(ci >> kLeafLog2), lb = (int)(cj >> kLeafLog2),
                                      lc = (int)(ck >> kLeafLog2);
                            if (la != pl0 || lb != pl1 || lc != pl2) {
                                pl0 = la; pl1 = lb; pl2 = lc;
                                const int4* hs = htab + (block_hash(la, lb, lc) & (unsigned long long)fp.hmask);
                                asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(hs));
                            }
                        }
#endif
                    });
                if (emitted < 0) {
                    t.errs |= 1;
                    r.w = -1.0;
                    rows = 0;
                } else {
                    t.band_hits += (unsigned long long)emitted;
                }
                if (nk) {
                    t.mn[0] = min(t.mn[0], min(f0, l0)); t.mx[0] = max(t.mx[0], max(f0, l0));
                    t.mn[1] = min(t.mn[1], min(f1, l1)); t.mx[1] = max(t.mx[1], max(f1, l1));
                    t.mn[2] = min(t.mn[2], min(f2, l2)); t.mx[2] = max(t.mx[2], max(f2, l2));
                }
            }
            ray[i] = r;
            rcnt[i] = rows;
            if (slots) {
                s_ray[threadIdx.x] = r;
                s_lab[threadIdx.x] = lab_i;
            }
        }
        int off, total;
        Scan(scan_tmp).ExclusiveSum(rows, off, total);
        // packed row e of the tile belongs to the thread whose range holds it:
        // record the owner of each packed row, then copy out coalesced
        s_off[threadIdx.x] = off;
        if (threadIdx.x == 0) s_base = total ? atomicAdd(&ctr->rows_alloc, (unsigned long long)total) : 0ULL;
#pragma unroll 1
        for (int j = 0; j < rows; ++j) s_own[off + j] = (unsigned char)threadIdx.x;
        __syncthreads();
        const unsigned long long base = s_base;
        const long long ray0 = tile * kTileRays;
        if (base + (unsigned long long)total <= rcap) {
            for (int e = threadIdx.x; e < total; e += kTileRays) {
                const int o = s_own[e];
                const unsigned long long key = s_keys[(size_t)o * maxrows + (e - s_off[o])];
                rowkey[base + e] = key;
                rowray[base + e] = (int)(ray0 + o);
                if (slots) {
                    // d of this row exactly as row_dw evaluates it from the voxel centre
                    long long x, y, z;
                    unpack_key(key, fp.kp, x, y, z);
                    const double4 r = s_ray[o];
                    const double cx = ((double)x + 0.5) * mp.h - ox;
                    const double cy = ((double)y + 0.5) * mp.h - oy;
                    const double cz = ((double)z + 0.5) * mp.h - oz;
                    const double proj = cx * r.x + cy * r.y + cz * r.z;
                    double d = r.w - proj;
                    if (d < -mp.trunc) d = -mp.trunc;
                    if (d > mp.trunc) d = mp.trunc;
                    rowd[base + e] = d;
                    rowlab[base + e] = s_lab[o];
                }
            }
        } else if (threadIdx.x == 0) {
            atomicOr(&ctr->err_cap, 1);
        }
        __syncthreads();
    }
    finish_walk<kTileRays>(t, partials, ctr);
}


// K1 (dense mode, e.g. space carving's unbounded bands), pass 1: count kept
// rows per ray (rcnt is zero past n so a fixed-size scan covers it).
template <class P, class Fe>
__global__ void __launch_bounds__(kMarchThreads) k_walk_count(MarchParams mp, int sem_kind,
                                                              int num_classes, int D,
                                                              long long npts_cap,
                                                              double4* __restrict__ ray,
                                                              int* __restrict__ rcnt,
                                                              MarchPartial* __restrict__ partials,
                                                              FrameCtr* __restrict__ ctr,
                                                              const __grid_constant__ FrameParams fpk) {
    grid_dep_wait();
    __shared__ FrameCtr s_ctr_;
    load_frame_params(ctr, s_ctr_, fpk);
    KSpan _ks(&s_ctr_, ctr, kSpanWalk);
    const FrameParams& fp = s_ctr_.p;
    const long long n = fp.n;
    const double ox = fp.pp.t[0], oy = fp.pp.t[1], oz = fp.pp.t[2];
    Tally t;
    // warp-uniform trip count (warp_feats_finite needs every lane)
    for (long long i0 = (long long)blockIdx.x * blockDim.x; i0 < npts_cap;
         i0 += (long long)gridDim.x * blockDim.x) {
        const long long i = i0 + threadIdx.x;
        const bool fok = sem_kind != SVX_SEM_OPEN ||
                         warp_feats_finite<Fe>((const Fe*)fp.feats, D, i, i < n);
        if (i >= npts_cap) continue;
        if (i >= n) {
            rcnt[i] = 0;
            continue;
        }
        double4 r;
        int rows = 0;
        if (prepare_ray<P, Fe>(i, fp, mp.max_range, sem_kind, num_classes, D, t, r, fok)) {
            long long emitted = dda_walk(ox, oy, oz, r.x, r.y, r.z, r.w, mp,
                [&](long long ci, long long cj, long long ck) {
                    if (!row_kept(ci, cj, ck, ox, oy, oz, r, mp)) return;
                    t.rows += 1;
                    t.mn[0] = min(t.mn[0], ci); t.mn[1] = min(t.mn[1], cj); t.mn[2] = min(t.mn[2], ck);
                    t.mx[0] = max(t.mx[0], ci); t.mx[1] = max(t.mx[1], cj); t.mx[2] = max(t.mx[2], ck);
                    long long ox_ = ci - fp.kp.base[0], oy_ = cj - fp.kp.base[1], oz_ = ck - fp.kp.base[2];
                    if (((ox_ | oy_ | oz_) & ~kPackMask) != 0) t.errs |= 2;
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
    finish_walk<kMarchThreads>(t, partials, ctr);
}

// K1 (dense mode), pass 2: re-walk and write each kept row at its scanned offset.
__global__ void __launch_bounds__(kMarchThreads) k_walk_write(MarchParams mp,
                                                              const double4* __restrict__ ray,
                                                              const int* __restrict__ rcnt,
                                                              const long long* __restrict__ roff,
                                                              unsigned long long* __restrict__ rowkey,
                                                              int* __restrict__ rowray,
                                                              const FrameCtr* __restrict__ ctr) {
    grid_dep_wait();
    KSpan _ks(const_cast<FrameCtr*>(ctr), kSpanWalk);
    __shared__ FrameCtr s_ctr_;
    snapshot_ctr(ctr, s_ctr_);
    if (s_ctr_.abort) return;
    const FrameParams& fp = s_ctr_.p;
    const long long n = fp.n;
    const double ox = fp.pp.t[0], oy = fp.pp.t[1], oz = fp.pp.t[2];
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        if (rcnt[i] == 0) continue;
        const double4 r = ray[i];
        long long o = roff[i];
        dda_walk(ox, oy, oz, r.x, r.y, r.z, r.w, mp, [&](long long ci, long long cj, long long ck) {
            if (!row_kept(ci, cj, ck, ox, oy, oz, r, mp)) return;
            rowkey[o] = pack_key(ci - fp.kp.base[0], cj - fp.kp.base[1], ck - fp.kp.base[2]);
            rowray[o] = (int)i;
            ++o;
        });
    }
}

// Decide, once per frame on the device, whether the frame may mutate the map
// -- the reference's checks before any allocation (_core.pyx:661-712,
// :386-387) plus the dense row capacity.  Run by one thread of the last walk
// CTA, when every CTA's tallies are in the frame counters.  The host reports
// the reason after the frame.
__device__ void gate_body(FrameCtr* ctr) {
    volatile FrameCtr* c = ctr;
    int ab = c->err_budget | c->err_pack | c->err_rows | (c->poison ? 1 : 0);
    const unsigned long long rows = c->rows;
    if (rows > c->p.rcap) {
        ctr->err_cap = 1;
        ab = 1;
    }
    if (rows) {
        for (int a = 0; a < 3; ++a) {
            const long long lo = c->bbox_min[a], hi = c->bbox_max[a];
            if (hi - lo >= (1LL << kPackBits)) ab = 1;
            if (llabs(lo) >= kCoordLimit || llabs(hi) >= kCoordLimit) ab = 1;
        }
    }
    ctr->abort = ab;
}

template <class P, class Fe>
svx_status march_t(svx_map* m, cudaStream_t s) {
    const MarchParams mp = march_params(m);
    MarchPartial* parts = ptr<MarchPartial>(m->partials);
    FrameCtr* dc = ptr<FrameCtr>(m->ctr);
    if (m->maxrows > 0) {
        const size_t smem = (size_t)kTileRays * m->maxrows * (sizeof(unsigned long long) + 1);
        SVX_CUDA(launch_pdl(k_walk<P, Fe>, kMarchBlocks, kTileRays, smem, s, 
            mp, m->cfg.sem_kind, m->cfg.num_classes, m->payload_d, ptr<double4>(m->ray),
            ptr<int>(m->rcnt), ptr<unsigned long long>(m->rowkey), ptr<int>(m->rowray),
            ptr<double>(m->rowd), ptr<int>(m->rowlab), parts, dc, ptr<int4>(m->hash), m->h_ctr->p));
        m->first_nargs = 14;
        SVX_LAUNCHED();
        return SVX_OK;
    }
    SVX_CUDA(launch_pdl(k_walk_count<P, Fe>, kMarchBlocks, kMarchThreads, 0, s, 
        mp, m->cfg.sem_kind, m->cfg.num_classes, m->payload_d, m->npts_cap, ptr<double4>(m->ray),
        ptr<int>(m->rcnt), parts, dc, m->h_ctr->p));
    m->first_nargs = 10;
    SVX_LAUNCHED();
    size_t tmp = m->cubtmp.bytes;
    SVX_CUDA(cub::DeviceScan::ExclusiveSum(m->cubtmp.p, tmp, ptr<int>(m->rcnt),
                                           ptr<long long>(m->roff), (int)m->npts_cap, s));
    count_launch();
    SVX_CUDA(launch_pdl(k_walk_write, kMarchBlocks, kMarchThreads, 0, s, 
        mp, ptr<double4>(m->ray), ptr<int>(m->rcnt), ptr<long long>(m->roff),
        ptr<unsigned long long>(m->rowkey), ptr<int>(m->rowray), dc));
    SVX_LAUNCHED();
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

size_t partials_bytes() { return sizeof(MarchPartial) * kMarchBlocks; }

size_t scan_temp_bytes(int64_t n) {
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, (const int*)nullptr, (long long*)nullptr, (int)n);
    return tmp;
}

}  // namespace svx

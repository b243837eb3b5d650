// svx_render.cu -- ray-march rendering of the device map (render.py:88-272:
// RenderCamera.rays, sample_distance, _skip_empty_leaves, _march, _refine,
// render's depth / normal / semantic outputs).
//
// One thread per pixel ray, every step in f64 and in the reference's
// operation order (this file is compiled with -fmad=false, so no expression
// is contracted into an FMA unless written as fma()):
//   * directions: ((u + 0.5 - cx) / fx, (v + 0.5 - cy) / fy, 1) over its
//     norm, rotated as numpy's (N, 3) @ R.T (world_coord, dgemm order);
//   * steps of h / 2 from `near`; a probe whose voxel's leaf is not allocated
//     jumps to the leaf's AABB exit (+1e-3 h, at least one step) and forgets
//     the previous sample;
//   * a bracket is a valid sample > 0 followed by a valid sample <= 0, where
//     valid = all 8 voxel centres around the point active (trilinear weights
//     multiplied x, y, z; corner contributions summed in (x, y, z) bit order);
//   * up to 32 secant steps to |D| < 1e-4 truncation; a sample leaving
//     observed space stops there.
// The march is divergent by nature (rays end at different steps); each ray
// only reads the leaf hash, the bslot table and the TSDF pairs, all of which
// stay L2-resident for the map sizes of the BASELINE configs.
#include <cuda_runtime.h>

#include "svx_internal.cuh"

namespace svx {
namespace {

constexpr int kRefineIters = 32;           // render.py:30
constexpr double kRefineTolFrac = 1e-4;    // render.py:29

template <class TD>
struct RenderArgs {
    const int4* table;
    int64_t hmask;
    const unsigned long long* bslot;
    const TD* vt;
    double h, trunc;
    int* err;   // set when a ray exceeds kMarchMaxSteps (absurd far planes)
};

constexpr long long kMarchMaxSteps = 1LL << 22;   // 2^22 half-voxel steps or leaf jumps per ray

__device__ __forceinline__ long long floor_ll(double v) { return (long long)floor(v); }

template <class TD>
__device__ __forceinline__ int leaf_of(const RenderArgs<TD>& a, long long x, long long y, long long z) {
    return hash_find(a.table, a.hmask, (int)(x >> 3), (int)(y >> 3), (int)(z >> 3));
}

// vid of the active voxel (x, y, z), or -1 (GridCore.probe_coords).
template <class TD>
__device__ __forceinline__ int active_vid(const RenderArgs<TD>& a, long long x, long long y, long long z) {
    const int leaf = leaf_of(a, x, y, z);
    if (leaf < 0) return -1;
    const int slot = (int)(((x & 7) << 6) | ((y & 7) << 3) | (z & 7));
    return (int)(unsigned)a.bslot[(int64_t)leaf * kLeafVolume + slot];
}

// sample_distance (render.py:88-113) at one point: false where any of the 8
// surrounding voxel centres is inactive.
template <class TD>
__device__ bool sample(const RenderArgs<TD>& a, double px, double py, double pz, double* out) {
    const double qx = px / a.h - 0.5, qy = py / a.h - 0.5, qz = pz / a.h - 0.5;
    const double fbx = floor(qx), fby = floor(qy), fbz = floor(qz);
    const long long bx = (long long)fbx, by = (long long)fby, bz = (long long)fbz;
    const double fx = qx - fbx, fy = qy - fby, fz = qz - fbz;
    double v = 0.0;
    for (int c = 0; c < 8; ++c) {
        const int ox = (c >> 2) & 1, oy = (c >> 1) & 1, oz = c & 1;
        const int vid = active_vid(a, bx + ox, by + oy, bz + oz);
        if (vid < 0) return false;
        double w = 1.0;
        w *= ox ? fx : 1.0 - fx;
        w *= oy ? fy : 1.0 - fy;
        w *= oz ? fz : 1.0 - fz;
        v += w * (double)a.vt[2 * (int64_t)vid];
    }
    *out = v;
    return true;
}

struct Ray {
    double o[3], d[3];
};

__device__ __forceinline__ void ray_point(const Ray& r, double t, double* p) {
    p[0] = r.o[0] + t * r.d[0];
    p[1] = r.o[1] + t * r.d[1];
    p[2] = r.o[2] + t * r.d[2];
}

// _march + _refine (render.py:116-211) for one ray: returns hit, *t_hit.
template <class TD>
__device__ bool march(const RenderArgs<TD>& a, const Ray& r, double near, double far, double* t_hit) {
    const double h = a.h, step = 0.5 * h;
    double t = near, prev_d = 0.0;
    bool prev_ok = false;
    double t0 = 0.0, d0 = 0.0, t1 = 0.0, d1 = 0.0;
    bool hit = false;
    long long steps = 0;
    while (true) {
        if (++steps > kMarchMaxSteps) {   // a guard, not the reference's semantics
            if (a.err) atomicOr(a.err, 1);
            return false;
        }
        double p[3];
        ray_point(r, t, p);
        const long long vx = floor_ll(p[0] / h), vy = floor_ll(p[1] / h), vz = floor_ll(p[2] / h);
        if (leaf_of(a, vx, vy, vz) < 0) {
            // _skip_empty_leaves (render.py:116-131)
            const long long lc[3] = {vx >> 3, vy >> 3, vz >> 3};
            double t_exit = INFINITY;
            for (int k = 0; k < 3; ++k) {
                const double lo = (double)(lc[k] << 3) * h;
                const double hi = (double)((lc[k] + 1) << 3) * h;
                const double e1 = (lo - r.o[k]) / r.d[k];
                const double e2 = (hi - r.o[k]) / r.d[k];
                const double tf = r.d[k] != 0.0 ? fmax(e1, e2) : INFINITY;
                t_exit = fmin(t_exit, tf);
            }
            t += fmax(step, (t_exit - t) + 1e-3 * h);
            prev_ok = false;
        } else {
            double dv = NAN;
            const bool ok = sample(a, p[0], p[1], p[2], &dv);
            if (ok && prev_ok && prev_d > 0.0 && dv <= 0.0) {
                hit = true;
                t0 = t - step;
                d0 = prev_d;
                t1 = t;
                d1 = dv;
                break;
            }
            prev_ok = ok;
            prev_d = ok ? dv : NAN;
            t += step;
        }
        if (!(t <= far)) break;
    }
    if (!hit) return false;
    const double tol = kRefineTolFrac * a.trunc;
    double at = t0, ad = d0, bt = t1, bd = d1, best = t1;
    for (int it = 0; it < kRefineIters; ++it) {
        const double tm = bt - bd * (bt - at) / (bd - ad);
        double p[3], dm = 0.0;
        ray_point(r, tm, p);
        const bool ok = sample(a, p[0], p[1], p[2], &dm);
        if (!ok) dm = 0.0;
        best = tm;
        if (!ok || fabs(dm) < tol) break;
        if (dm > 0.0) {
            at = tm;
            ad = dm;
        } else {
            bt = tm;
            bd = dm;
        }
    }
    *t_hit = best;
    return true;
}

struct CamArgs {
    double R[9], t[3];
    double fx, fy, cx, cy, near, far;
    int width, height, single;
};

// RenderCamera.rays (render.py:70-85) for pixel (row v, column u).
__device__ __forceinline__ Ray camera_ray(const CamArgs& c, int u, int v) {
    const double a = ((double)u + 0.5 - c.cx) / c.fx;
    const double b = ((double)v + 0.5 - c.cy) / c.fy;
    const double one = 1.0;
    const double n = sqrt((a * a + b * b) + one * one);
    const double dc0 = a / n, dc1 = b / n, dc2 = one / n;
    Ray r;
    for (int k = 0; k < 3; ++k) {
        r.d[k] = world_coord(c.R + 3 * k, 0.0, dc0, dc1, dc2, c.single);
        r.o[k] = c.t[k];
    }
    return r;
}

template <class TD, class TS>
__global__ void __launch_bounds__(128) k_render(RenderArgs<TD> a, CamArgs c, int mode, int sem_kind, int P,
                                                const TS* __restrict__ s0, const int* __restrict__ vlab,
                                                const unsigned char* __restrict__ pal, int npal,
                                                void* __restrict__ out) {
    const int64_t npx = (int64_t)c.width * c.height;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npx;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int v = (int)(i / c.width), u = (int)(i % c.width);
        const Ray r = camera_ray(c, u, v);
        double th = 0.0;
        const bool hit = march(a, r, c.near, c.far, &th);
        if (mode == SVX_RENDER_DEPTH) {
            ((double*)out)[i] = hit ? th : 0.0;
            continue;
        }
        double p[3];
        ray_point(r, th, p);
        if (mode == SVX_RENDER_NORMAL) {
            double g[3] = {0.0, 0.0, 0.0};
            if (hit) {
                bool ok = true;
                for (int ax = 0; ax < 3; ++ax) {
                    double q[3] = {p[0], p[1], p[2]}, dp = 0.0, dn = 0.0;
                    q[ax] = p[ax] + 0.5 * a.h;
                    const bool okp = sample(a, q[0], q[1], q[2], &dp);
                    q[ax] = p[ax] - 0.5 * a.h;
                    const bool okn = sample(a, q[0], q[1], q[2], &dn);
                    ok = ok && okp && okn;
                    g[ax] = (okp && okn) ? dp - dn : 0.0;
                }
                const double nrm = sqrt((g[0] * g[0] + g[1] * g[1]) + g[2] * g[2]);
                ok = ok && nrm > 0.0;
                for (int ax = 0; ax < 3; ++ax) g[ax] = ok ? g[ax] / nrm : 0.0;
            }
            double* o = (double*)out + 3 * i;
            o[0] = g[0];
            o[1] = g[1];
            o[2] = g[2];
            continue;
        }
        // semantic: palette colour of the voxel nearest the hit point
        unsigned char* o = (unsigned char*)out + 3 * i;
        if (!hit) {
            o[0] = o[1] = o[2] = 0;
            continue;
        }
        const long long nx = (long long)rint(p[0] / a.h - 0.5);
        const long long ny = (long long)rint(p[1] / a.h - 0.5);
        const long long nz = (long long)rint(p[2] / a.h - 0.5);
        const int vid = active_vid(a, nx, ny, nz);
        int lab = 0;
        if (vid >= 0) {
            if (vlab) {
                lab = vlab[vid];
            } else {
                const TS* row = s0 + (int64_t)vid * P;
                int arg = 0;
                double best = (double)row[0], tot = 0.0;
                const bool open = sem_kind == SVX_SEM_OPEN;
                for (int k = 0; k < P; ++k) {
                    const double x = (double)row[k];
                    if (x != x) {
                        arg = k;
                        tot = x;
                        break;
                    }
                    if (x > best) {
                        best = x;
                        arg = k;
                    }
                    tot += open ? fabs(x) : x;
                }
                lab = open ? (tot == 0.0 ? 0 : arg + 1) : (tot <= 0.0 ? 0 : arg + 1);
            }
        }
        const long long row = lab > 0 ? 1 + (long long)(lab - 1) % (npal - 1) : 0;
        o[0] = pal[3 * row];
        o[1] = pal[3 * row + 1];
        o[2] = pal[3 * row + 2];
    }
}

template <class TD>
__global__ void k_sample_points(RenderArgs<TD> a, int64_t n, const double* __restrict__ pts,
                                double* __restrict__ vals, unsigned char* __restrict__ valid) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double v = NAN;
        const bool ok = sample(a, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], &v);
        vals[i] = ok ? v : NAN;
        valid[i] = ok;
    }
}

template <class TD>
RenderArgs<TD> render_args(svx_map* m) {
    return RenderArgs<TD>{ptr<int4>(m->hash), m->hcap - 1, ptr<unsigned long long>(m->bslot),
                          ptr<TD>(m->vt), m->cfg.voxel_size, m->cfg.truncation, nullptr};
}

template <class TD, class TS>
svx_status render_t(svx_map* m, const svx_render_camera& cam, int mode, const int* vlab,
                    const unsigned char* pal, int npal, void* out, cudaStream_t s) {
    CamArgs c;
    for (int r = 0; r < 3; ++r) {
        for (int k = 0; k < 3; ++k) c.R[3 * r + k] = cam.pose[4 * r + k];
        c.t[r] = cam.pose[4 * r + 3];
    }
    c.fx = cam.fx;
    c.fy = cam.fy;
    c.cx = cam.cx;
    c.cy = cam.cy;
    c.near = cam.near_plane;
    c.far = cam.far_plane;
    c.width = cam.width;
    c.height = cam.height;
    c.single = (int64_t)cam.width * cam.height == 1;
    const int64_t npx = (int64_t)cam.width * cam.height;
    const int T = 128;
    const int G = (int)std::min<int64_t>((npx + T - 1) / T, 148 * 16);
    RenderArgs<TD> ra = render_args<TD>(m);
    // one persistent error flag per map, cleared per call (nothing to free on
    // any exit path)
    SVX_TRY(ensure(m->render_err, sizeof(int), s));
    ra.err = ptr<int>(m->render_err);
    SVX_CUDA(cudaMemsetAsync(ra.err, 0, sizeof(int), s));
    k_render<TD, TS><<<G, T, 0, s>>>(ra, c, mode, m->cfg.sem_kind, m->payload_d, ptr<TS>(m->s0), vlab, pal,
                                     npal, out);
    SVX_LAUNCHED();
    int herr = 0;
    cudaError_t e = cudaMemcpyAsync(&herr, ra.err, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return fail(SVX_E_CUDA, std::string("render: ") + cudaGetErrorString(e));
    if (herr) return fail(SVX_E_INPUT, "render: a ray exceeded 2^22 march steps (far plane too far)");
    return SVX_OK;
}

}  // namespace

svx_status render_impl(svx_map* m, const svx_render_camera& cam, int mode, const int* vlab,
                       const unsigned char* pal, int npal, void* out, cudaStream_t s) {
    const bool t64 = m->cfg.tsdf_dtype == SVX_F64;
    const bool s64 = m->cfg.sem_kind == SVX_SEM_CLOSED ? m->cfg.count_dtype == SVX_F64
                                                        : m->cfg.state_dtype == SVX_F64;
    if (t64 && s64) return render_t<double, double>(m, cam, mode, vlab, pal, npal, out, s);
    if (t64) return render_t<double, float>(m, cam, mode, vlab, pal, npal, out, s);
    if (s64) return render_t<float, double>(m, cam, mode, vlab, pal, npal, out, s);
    return render_t<float, float>(m, cam, mode, vlab, pal, npal, out, s);
}

svx_status sample_impl(svx_map* m, int64_t n, const double* pts, double* vals, unsigned char* valid,
                       cudaStream_t s) {
    if (n == 0) return SVX_OK;
    const int G = grid_for(n, 256);
    if (m->cfg.tsdf_dtype == SVX_F64)
        k_sample_points<double><<<G, 256, 0, s>>>(render_args<double>(m), n, pts, vals, valid);
    else
        k_sample_points<float><<<G, 256, 0, s>>>(render_args<float>(m), n, pts, vals, valid);
    SVX_LAUNCHED();
    return SVX_OK;
}

}  // namespace svx

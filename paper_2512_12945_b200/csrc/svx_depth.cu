// svx_depth.cu -- depth frames on the GPU: back-projection of a depth raster
// (ingest.project_depth, ingest.py:285-322) straight into the integration
// path, replacing the host's f64 prep and its H2D copy of the point cloud.
//
// One thread per sampled pixel writes the sensor-frame point in f64 with the
// reference's operation order; pixels with d <= 0 or non-finite d become NaN
// points, which the walk skips.  Point indices follow the sampled raster in
// row-major order, so the valid points keep project_depth's relative order
// (the per-voxel reductions only depend on it); the report is corrected for
// the invalid pixels on the host (they are not points in the reference).
// Payload rasters are read in place at stride 1 and gathered at stride > 1.
#include <cuda_runtime.h>
#include <math.h>
#include <string.h>
#include <stdio.h>
#include <stdlib.h>
#include <time.h>

#include "svx_internal.cuh"

namespace svx {
namespace {

template <class DT, class Fe>
__global__ void k_backproject(const DT* __restrict__ depth, int W, int stride, int Ws, long long n,
                              double fx, double fy, double cx, double cy, double scale,
                              double* __restrict__ pts, const int32_t* __restrict__ lab_in,
                              int32_t* __restrict__ lab_out, const Fe* __restrict__ feat_in,
                              Fe* __restrict__ feat_out, int D, unsigned long long* __restrict__ n_invalid) {
    unsigned invalid = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long vi = i / Ws, ui = i - vi * Ws;
        const long long v = vi * stride, u = ui * stride;
        const long long src = v * W + u;
        const double d = (double)depth[src];
        double x = NAN, y = NAN, z = NAN;
        if (d > 0.0 && isfinite(d)) {
            // np.stack([(uu - cx) * d / fx, (vv - cy) * d / fy, d]) * depth_scale
            x = (((double)u - cx) * d / fx) * scale;
            y = (((double)v - cy) * d / fy) * scale;
            z = d * scale;
        } else {
            ++invalid;
        }
        pts[3 * i] = x;
        pts[3 * i + 1] = y;
        pts[3 * i + 2] = z;
        if (lab_out) lab_out[i] = lab_in[src];
        if (feat_out)
            for (int c = 0; c < D; ++c) feat_out[i * D + c] = feat_in[src * D + c];
    }
    invalid = __reduce_add_sync(0xffffffffu, invalid);
    if ((threadIdx.x & 31) == 0 && invalid) atomicAdd(n_invalid, (unsigned long long)invalid);
}

template <class DT, class Fe>
svx_status backproject_t(svx_map* m, const void* depth, const svx_camera& cam, int Hs, int Ws,
                         double* pts, const int32_t* lab_in, int32_t* lab_out, const void* feat_in,
                         void* feat_out, unsigned long long* n_invalid, cudaStream_t s) {
    const long long n = (long long)Hs * Ws;
    const int T = 256;
    const int grid = (int)std::min<long long>((n + T - 1) / T, (long long)kPersistentBlocks);
    k_backproject<DT, Fe><<<grid, T, 0, s>>>(
        (const DT*)depth, cam.width, cam.stride, Ws, n, cam.fx, cam.fy, cam.cx, cam.cy,
        cam.depth_scale, pts, lab_in, lab_out, (const Fe*)feat_in, (Fe*)feat_out, m->payload_d,
        n_invalid);
    SVX_LAUNCHED();
    return SVX_OK;
}

}  // namespace

static const bool g_trace_depth = getenv("SVX_TRACE_HOST") != nullptr;
static double depth_now_us() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e6 + ts.tv_nsec * 1e-3;
}

svx_status integrate_depth_impl(svx_map* m, const void* depth, int depth_dtype, const svx_camera& cam,
                                const PoseParams& pp, const int32_t* labels, const void* feats,
                                int feats_f64, cudaStream_t s, svx_report* rep) {
    if (!(cam.fx > 0) || !(cam.fy > 0)) return fail(SVX_E_CONFIG, "fx and fy must be positive");
    if (cam.width < 1 || cam.height < 1) return fail(SVX_E_CONFIG, "raster dimensions must be positive");
    if (!(cam.depth_scale > 0)) return fail(SVX_E_CONFIG, "depth_scale must be positive");
    if (cam.stride < 1) return fail(SVX_E_CONFIG, "stride must be >= 1");
    if (depth_dtype != SVX_F32 && depth_dtype != SVX_F64 && depth_dtype != SVX_U16)
        return fail(SVX_E_INPUT, "depth raster dtype must be float32, float64 or uint16");
    const int kind = m->cfg.sem_kind;
    if (kind == SVX_SEM_CLOSED && !labels) return fail(SVX_E_PAYLOAD, "closed-set grid requires per-point labels");
    if (kind == SVX_SEM_OPEN && !feats) return fail(SVX_E_PAYLOAD, "open-set grid requires per-point features");
    const double t0 = g_trace_depth ? depth_now_us() : 0.0;
    const int H = cam.height, W = cam.width, st = cam.stride;
    const int Hs = (H + st - 1) / st, Ws = (W + st - 1) / st;
    const long long npix = (long long)H * W, n = (long long)Hs * Ws;
    const size_t dsz = depth_dtype == SVX_F64 ? 8 : (depth_dtype == SVX_F32 ? 4 : 2);
    const size_t fsz = (size_t)m->payload_d * (feats_f64 ? 8 : 4);
    const void* dd;
    SVX_TRY(stage_in(depth, (size_t)npix * dsz, m->dp_depth, s, &dd));
    const void* ld = nullptr;
    const void* fd = nullptr;
    if (kind == SVX_SEM_CLOSED) SVX_TRY(stage_in(labels, (size_t)npix * 4, m->dp_lab_in, s, &ld));
    if (kind == SVX_SEM_OPEN) SVX_TRY(stage_in(feats, (size_t)npix * fsz, m->dp_feat_in, s, &fd));
    SVX_TRY(ensure(m->dp_pts, sizeof(double) * 3 * (size_t)n + sizeof(unsigned long long), s));
    int32_t* lab_out = nullptr;
    void* feat_out = nullptr;
    if (kind == SVX_SEM_CLOSED && st > 1) {
        SVX_TRY(ensure(m->dp_lab, (size_t)n * 4, s));
        lab_out = ptr<int32_t>(m->dp_lab);
    }
    if (kind == SVX_SEM_OPEN && st > 1) {
        SVX_TRY(ensure(m->dp_feat, (size_t)n * fsz, s));
        feat_out = m->dp_feat.p;
    }
    double* pts = ptr<double>(m->dp_pts);
    unsigned long long* d_inv = reinterpret_cast<unsigned long long*>(pts + 3 * n);
    SVX_CUDA(cudaMemsetAsync(d_inv, 0, sizeof(unsigned long long), s));
    const int32_t* lab_in = (const int32_t*)ld;
    svx_status bs;
    if (feats_f64) {
        bs = depth_dtype == SVX_F64 ? backproject_t<double, double>(m, dd, cam, Hs, Ws, pts, lab_in, lab_out, fd, feat_out, d_inv, s)
           : depth_dtype == SVX_F32 ? backproject_t<float, double>(m, dd, cam, Hs, Ws, pts, lab_in, lab_out, fd, feat_out, d_inv, s)
                                    : backproject_t<unsigned short, double>(m, dd, cam, Hs, Ws, pts, lab_in, lab_out, fd, feat_out, d_inv, s);
    } else {
        bs = depth_dtype == SVX_F64 ? backproject_t<double, float>(m, dd, cam, Hs, Ws, pts, lab_in, lab_out, fd, feat_out, d_inv, s)
           : depth_dtype == SVX_F32 ? backproject_t<float, float>(m, dd, cam, Hs, Ws, pts, lab_in, lab_out, fd, feat_out, d_inv, s)
                                    : backproject_t<unsigned short, float>(m, dd, cam, Hs, Ws, pts, lab_in, lab_out, fd, feat_out, d_inv, s);
    }
    SVX_TRY(bs);
    svx_report r;
    const int32_t* lab_use = kind == SVX_SEM_CLOSED ? (st > 1 ? lab_out : lab_in) : nullptr;
    const void* feat_use = kind == SVX_SEM_OPEN ? (st > 1 ? feat_out : fd) : nullptr;
    const double t1 = g_trace_depth ? depth_now_us() : 0.0;
    SVX_TRY(integrate_impl(m, pts, 1, n, pp, lab_use, feat_use, feats_f64, s, &r, 1));
    const double t2 = g_trace_depth ? depth_now_us() : 0.0;
    unsigned long long inv = 0;
    SVX_CUDA(cudaMemcpyAsync(&inv, d_inv, sizeof(inv), cudaMemcpyDeviceToHost, s));
    SVX_CUDA(cudaStreamSynchronize(s));
    // invalid pixels are not points of the reference's Frame
    // host-link bytes of this call: the rasters staged from host memory
    // (integrate_impl saw device pointers), the report mirror and `inv`
    int64_t h2d = 0;
    if (dd != depth) h2d += (int64_t)npix * (int64_t)dsz;
    if (ld && ld != (const void*)labels) h2d += (int64_t)npix * 4;
    if (fd && fd != feats) h2d += (int64_t)npix * (int64_t)fsz;
    m->io_h2d = h2d;
    m->io_d2h += (int64_t)sizeof(inv);
    if (g_trace_depth)
        fprintf(stderr, "svx depth us: backproject %.1f integrate %.1f tail %.1f\n", t1 - t0, t2 - t1,
                depth_now_us() - t2);
    r.points_in -= (int64_t)inv;
    r.skipped_nonfinite -= (int64_t)inv;
    if (rep) *rep = r;
    return SVX_OK;
}

}  // namespace svx

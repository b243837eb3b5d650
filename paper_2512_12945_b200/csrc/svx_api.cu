// svx_api.cu -- C ABI entry points and the per-frame orchestration.
//
// Frame pipeline on the caller's stream, one host synchronisation per frame
// (DESIGN.md "Per-frame pipeline"):
//   K1 march    masks, ray setup, fp64 band walk, frame-table insert + counts (svx_march.cu)
//   K2 compact  touched voxels -> list + row segments; device-side gate        (svx_march.cu)
//   K3 scatter  second walk: point index -> its voxel's segment                (svx_march.cu)
//   K4 voxels   leaf find-or-insert + creation stamp, voxel activation         (svx_update.cu)
//   K5 update   fused TSDF + closed/open update, rows re-sorted per voxel      (svx_update.cu)
// Kernels after K1 size themselves from device counters; a frame whose
// scratch was too small (or whose keys need a different base) is detected by
// the gate before any map mutation and re-run.
#include <cuda_runtime.h>
#include <limits.h>
#include <math.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <cub/cub.cuh>
#include <string>

#include <cmath>
#include <algorithm>

#include "svx_internal.cuh"

namespace svx {

static thread_local std::string g_error;
static std::atomic<long long> g_launches{0};

void set_error(const std::string& msg) { g_error = msg; }

svx_status fail(svx_status code, const std::string& msg) {
    g_error = msg;
    return code;
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

svx_status ensure(DevBuf& buf, size_t bytes, cudaStream_t s, bool keep, int fill) {
    if (bytes == 0) bytes = 16;
    if (buf.p && buf.bytes >= bytes) return SVX_OK;
    size_t nb = std::max(bytes, buf.bytes * 2);
    void* np = nullptr;
    cudaError_t e = cudaMalloc(&np, nb);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(SVX_E_CUDA, std::string("device allocation of ") + std::to_string(nb) +
                                    " bytes failed: " + cudaGetErrorString(e));
    }
    size_t old = 0;
    if (keep && buf.p && buf.bytes) {
        old = buf.bytes;
        SVX_CUDA(cudaMemcpyAsync(np, buf.p, old, cudaMemcpyDeviceToDevice, s));
    }
    if (fill >= 0) SVX_CUDA(cudaMemsetAsync((char*)np + old, fill, nb - old, s));
    if (buf.p) {
        SVX_CUDA(cudaStreamSynchronize(s));
        SVX_CUDA(cudaFree(buf.p));
    }
    buf.p = np;
    buf.bytes = nb;
    return SVX_OK;
}

void release(DevBuf& buf) {
    if (buf.p) cudaFree(buf.p);
    buf.p = nullptr;
    buf.bytes = 0;
}

namespace {

// Output staging: device pointers are written directly; host outputs go
// through device scratch and are copied back at the end of the call.
struct OutStage {
    DevBuf buf;
    void* user = nullptr;
    size_t bytes = 0;
    bool host = false;
};

svx_status out_prepare(OutStage& o, void* user, size_t bytes, cudaStream_t s, void** dev) {
    o.user = user;
    o.bytes = bytes;
    if (!user || bytes == 0) {
        *dev = user;
        return SVX_OK;
    }
    if (is_device_ptr(user)) {
        *dev = user;
        return SVX_OK;
    }
    o.host = true;
    SVX_TRY(ensure(o.buf, bytes, s));
    *dev = o.buf.p;
    return SVX_OK;
}

svx_status out_finish(OutStage& o, cudaStream_t s) {
    if (o.host && o.user && o.bytes) {
        SVX_CUDA(cudaMemcpyAsync(o.user, o.buf.p, o.bytes, cudaMemcpyDeviceToHost, s));
    }
    return SVX_OK;
}

void out_release(OutStage* o, int n) {
    for (int i = 0; i < n; ++i) release(o[i].buf);
}

// The fast acceptance test of the frame pose (fusion.py:31-77, mapper.py
// _check_pose): anything else goes back to the host's full validation.
bool pose_fast_ok(const double* f) {
    for (int i = 0; i < 16; ++i)
        if (!std::isfinite(f[i])) return false;
    if (f[12] != 0.0 || f[13] != 0.0 || f[14] != 0.0 || f[15] != 1.0) return false;
    const double a0 = f[0], a1 = f[1], a2 = f[2], b0 = f[4], b1 = f[5], b2 = f[6];
    const double c0 = f[8], c1 = f[9], c2 = f[10];
    double err = fabs(a0 * a0 + a1 * a1 + a2 * a2 - 1.0);
    err = std::max(err, fabs(b0 * b0 + b1 * b1 + b2 * b2 - 1.0));
    err = std::max(err, fabs(c0 * c0 + c1 * c1 + c2 * c2 - 1.0));
    err = std::max(err, fabs(a0 * b0 + a1 * b1 + a2 * b2));
    err = std::max(err, fabs(a0 * c0 + a1 * c1 + a2 * c2));
    err = std::max(err, fabs(b0 * c0 + b1 * c1 + b2 * c2));
    const double det = a0 * (b1 * c2 - b2 * c1) - a1 * (b0 * c2 - b2 * c0) + a2 * (b0 * c1 - b1 * c0);
    return err <= 0.5e-4 && det > 0.0;
}

svx_status set_device(const svx_map* m) {
    SVX_CUDA(cudaSetDevice(m->cfg.device));
    return SVX_OK;
}

}  // namespace
}  // namespace svx

using namespace svx;

extern "C" {

const char* svx_last_error(void) { return g_error.c_str(); }
int32_t svx_abi_version(void) { return SVX_ABI_VERSION; }
int64_t svx_kernel_launches(void) { return g_launches.load(); }

svx_status svx_create(const svx_config* cfg, svx_map** out) {
    if (!cfg || !out) return fail(SVX_E_INPUT, "null argument");
    *out = nullptr;
    if (!(cfg->voxel_size > 0)) return fail(SVX_E_CONFIG, "voxel_size must be positive");
    if (!(cfg->truncation > 0)) return fail(SVX_E_CONFIG, "truncation must be positive");
    if (!(cfg->max_range > 0)) return fail(SVX_E_CONFIG, "max_range must be positive");
    if (cfg->weight_fn != 0 && cfg->weight_fn != 1) return fail(SVX_E_CONFIG, "weight_fn must be 0 or 1");
    if (cfg->sem_kind == SVX_SEM_CLOSED && cfg->num_classes < 1)
        return fail(SVX_E_CONFIG, "num_classes must be >= 1");
    if (cfg->sem_kind == SVX_SEM_OPEN && cfg->feature_dim < 1)
        return fail(SVX_E_CONFIG, "feature_dim must be >= 1");
    if (cfg->sem_kind < 0 || cfg->sem_kind > 2) return fail(SVX_E_CONFIG, "unknown semantic kind");
    cudaError_t e = cudaSetDevice(cfg->device);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(SVX_E_CUDA, std::string("cudaSetDevice failed: ") + cudaGetErrorString(e));
    }
    svx_map* m = new svx_map();
    m->cfg = *cfg;
    m->payload_d = cfg->sem_kind == SVX_SEM_CLOSED ? cfg->num_classes
                   : cfg->sem_kind == SVX_SEM_OPEN ? cfg->feature_dim : 0;
    cudaStream_t s = 0;
    svx_status st = SVX_OK;
    auto bail = [&](svx_status code) {
        svx_destroy(m);
        return code;
    };
    if (cudaHostAlloc((void**)&m->h_ctr, sizeof(FrameCtr), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer((void**)&m->d_hctr, m->h_ctr, 0) != cudaSuccess) {
        cudaGetLastError();
        return bail(fail(SVX_E_CUDA, "pinned mapped allocation failed"));
    }
    memset(m->h_ctr, 0, sizeof(FrameCtr));
    m->h_ctr0 = m->h_ctr;
    m->d_hctr0 = m->d_hctr;
    if ((st = ensure(m->ctr, sizeof(FrameCtr), s)) != SVX_OK) return bail(st);
    if (cudaEventCreate(&m->ev0) != cudaSuccess || cudaEventCreate(&m->ev1) != cudaSuccess ||
        cudaEventCreateWithFlags(&m->ev_in, cudaEventDisableTiming) != cudaSuccess ||
        cudaStreamCreateWithFlags(&m->gstream, cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        return bail(fail(SVX_E_CUDA, "event/stream creation failed"));
    }
    int64_t rb = cfg->reserve_blocks > 0 ? cfg->reserve_blocks : 1024;
    int64_t rv = cfg->reserve_voxels > 0 ? cfg->reserve_voxels : 65536;
    if ((st = reserve_blocks(m, rb, s)) != SVX_OK) return bail(st);
    if ((st = reserve_voxels(m, rv, s)) != SVX_OK) return bail(st);
    if (cudaStreamSynchronize(s) != cudaSuccess) {
        cudaGetLastError();
        return bail(fail(SVX_E_CUDA, "initial allocation failed"));
    }
    *out = m;
    return SVX_OK;
}

svx_status svx_destroy(svx_map* m) {
    if (!m) return SVX_OK;
    cudaSetDevice(m->cfg.device);
    for (int i = 0; i < m->aq_count; ++i) {   // frames in flight finish first
        const AsyncFrame& f = m->aq[(m->aq_head + i) % kAsyncSlots];
        if (f.e1) cudaEventSynchronize(f.e1);
    }
    m->aq_count = 0;
    release_async(m);
    DevBuf* bufs[] = {&m->hash, &m->bcoord, &m->bkey, &m->bmask, &m->bslot, &m->vt,
                      &m->s0, &m->s1, &m->vrec, &m->vslot, &m->lcnt, &m->rowleaf, &m->rowpk,
                      &m->binrow, &m->render_err, &m->sc_q, &m->sc_o, &m->in_pts,
                      &m->in_lab, &m->in_feat, &m->dp_depth, &m->dp_lab_in, &m->dp_feat_in, &m->dp_pts, &m->dp_lab, &m->dp_feat, &m->ray, &m->rcnt, &m->roff, &m->rowkey,
                      &m->rowvid, &m->rowray, &m->rowd, &m->rowlab, &m->partials, &m->tlist, &m->mlist,
                      &m->longlist, &m->hinfo, &m->srid, &m->bitmap, &m->rcount, &m->cubtmp, &m->ctr, &m->ord0,
                      &m->ord1, &m->ordk0, &m->ordk1, &m->ordf0, &m->ordf1, &m->act_cnt,
                      &m->act_off, &m->act_vid, &m->act_coord, &m->q_buf, &m->out_buf,
                      &m->mesh_ctr, &m->mesh_k0, &m->mesh_k1, &m->mesh_i0, &m->mesh_i1,
                      &m->mesh_rec, &m->mesh_meta, &m->mesh_vmask, &m->mesh_cnt, &m->mesh_off,
                      &m->mesh_toff, &m->mesh_vk, &m->mesh_vv, &m->mesh_vidx, &m->mesh_v,
                      &m->mesh_l, &m->mesh_t, &m->mesh_col, &m->mesh_vlab, &m->mesh_cls_l,
                      &m->mesh_cls_b, &m->mesh_pal};
    for (DevBuf* b : bufs) release(*b);
    if (m->h_ctr0) cudaFreeHost(m->h_ctr0);
    if (m->h_kspan) cudaFreeHost(m->h_kspan);
    if (m->sh_hlocal) cudaFreeHost(m->sh_hlocal);
    release(m->kspan);
    if (m->ev0) cudaEventDestroy(m->ev0);
    if (m->ev1) cudaEventDestroy(m->ev1);
    if (m->ev_in) cudaEventDestroy(m->ev_in);
    for (auto& per_mode : m->gexec)
        for (cudaGraphExec_t g : per_mode)
            if (g) cudaGraphExecDestroy(g);
    for (cudaGraph_t g : m->graph)
        if (g) cudaGraphDestroy(g);
    if (m->gstream) cudaStreamDestroy(m->gstream);
    delete m;
    return SVX_OK;
}

svx_status svx_integrate(svx_map* m, const void* points, int32_t points_dtype, int64_t n,
                         const double pose[16], const int32_t* labels, const void* feats,
                         int32_t feats_dtype, void* stream, svx_report* report) {
    if (!m || !pose || (n > 0 && !points)) return fail(SVX_E_INPUT, "null argument");
    if ((points_dtype & SVX_POSE_CHECK) && !pose_fast_ok(pose)) return (svx_status)SVX_POSE_NEEDS_HOST;
    SVX_TRY(set_device(m));
    SVX_TRY(drain(m));
    PoseParams pp;
    for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) pp.R[3 * r + c] = pose[4 * r + c];
        pp.t[r] = pose[4 * r + 3];
    }
    pp.sensor = 1;
    pp.single = n == 1;
    const int dev = (points_dtype & SVX_DEVICE_INPUTS) ? 1 : 0;
    return integrate_impl(m, points, (points_dtype & 0xff) == SVX_F64, n, pp, labels, feats,
                          (feats_dtype & 0xff) == SVX_F64, (cudaStream_t)stream, report, dev);
}

svx_status svx_integrate_async(svx_map* m, const void* points, int32_t points_dtype, int64_t n,
                               const double pose[16], const int32_t* labels, void* stream,
                               uint64_t* ticket) {
    if (!m || !pose || !ticket || (n > 0 && !points)) return fail(SVX_E_INPUT, "null argument");
    if (m->cfg.sem_kind == SVX_SEM_OPEN)
        return fail(SVX_E_PAYLOAD, "open-set grid requires per-point features (use svx_integrate)");
    if ((points_dtype & SVX_POSE_CHECK) && !pose_fast_ok(pose)) return (svx_status)SVX_POSE_NEEDS_HOST;
    SVX_TRY(set_device(m));
    PoseParams pp;
    for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) pp.R[3 * r + c] = pose[4 * r + c];
        pp.t[r] = pose[4 * r + 3];
    }
    pp.sensor = 1;
    pp.single = n == 1;
    const int dev = (points_dtype & SVX_DEVICE_INPUTS) ? 1 : 0;
    return integrate_async_impl(m, points, (points_dtype & 0xff) == SVX_F64, n, pp, labels,
                                (cudaStream_t)stream, dev, ticket);
}

svx_status svx_report_wait(svx_map* m, uint64_t ticket, svx_report* report) {
    if (!m) return fail(SVX_E_INPUT, "null argument");
    SVX_TRY(set_device(m));
    return report_wait(m, ticket, report);
}

svx_status svx_set_async(svx_map* m, int32_t depth, int64_t leaf_headroom) {
    if (!m || depth < 0 || leaf_headroom < 0) return fail(SVX_E_INPUT, "invalid asynchronous settings");
    SVX_TRY(set_device(m));
    SVX_TRY(drain(m));
    m->async_depth = std::min<int32_t>(depth, kAsyncSlots);
    m->async_leaf_headroom = leaf_headroom;
    return SVX_OK;
}

svx_status svx_import(svx_map* m, int64_t nl, const int32_t* leaf_coords, int64_t nv,
                      const int32_t* voxel_leaf, const int32_t* voxel_slot, const double* d,
                      const double* w, const void* sem0, const void* sem1, void* stream) {
    if (!m || (nv > 0 && (!leaf_coords || !voxel_leaf || !voxel_slot || !d || !w)))
        return fail(SVX_E_INPUT, "null argument");
    SVX_TRY(set_device(m));
    SVX_TRY(drain(m));
    return import_impl(m, nl, leaf_coords, nv, voxel_leaf, voxel_slot, d, w, sem0, sem1,
                       (cudaStream_t)stream);
}

svx_status svx_integrate_depth(svx_map* m, const void* depth, int32_t depth_dtype,
                               const svx_camera* camera, const double pose[16],
                               const int32_t* labels, const void* feats, int32_t feats_dtype,
                               void* stream, svx_report* report) {
    if (!m || !depth || !camera || !pose) return fail(SVX_E_INPUT, "null argument");
    SVX_TRY(set_device(m));
    SVX_TRY(drain(m));
    PoseParams pp;
    for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) pp.R[3 * r + c] = pose[4 * r + c];
        pp.t[r] = pose[4 * r + 3];
    }
    pp.sensor = 1;
    pp.single = 0;   // (a raster with exactly one valid pixel would take numpy's 1-row path)
    return integrate_depth_impl(m, depth, depth_dtype & 0xff, *camera, pp, labels, feats,
                                (feats_dtype & 0xff) == SVX_F64, (cudaStream_t)stream, report);
}

svx_status svx_integrate_world(svx_map* m, const void* points_world, int32_t points_dtype,
                               int64_t n, const double origin[3], const int32_t* labels,
                               const void* feats, int32_t feats_dtype, void* stream,
                               svx_report* report) {
    if (!m || !origin || (n > 0 && !points_world)) return fail(SVX_E_INPUT, "null argument");
    SVX_TRY(set_device(m));
    SVX_TRY(drain(m));
    PoseParams pp;
    memset(&pp, 0, sizeof(pp));
    pp.R[0] = pp.R[4] = pp.R[8] = 1.0;
    for (int a = 0; a < 3; ++a) pp.t[a] = origin[a];
    pp.sensor = 0;
    pp.single = 0;
    const int dev = (points_dtype & SVX_DEVICE_INPUTS) ? 1 : 0;
    return integrate_impl(m, points_world, (points_dtype & 0xff) == SVX_F64, n, pp, labels, feats,
                          (feats_dtype & 0xff) == SVX_F64, (cudaStream_t)stream, report, dev);
}

svx_status svx_reserve(svx_map* m, int64_t voxels, int64_t blocks) {
    if (!m || voxels < 0 || blocks < 0) return fail(SVX_E_INPUT, "invalid reserve arguments");
    SVX_TRY(set_device(m));
    SVX_TRY(drain(m));
    cudaStream_t s = 0;
    SVX_TRY(reserve_blocks(m, std::max<int64_t>(blocks, m->nblocks), s));
    SVX_TRY(reserve_voxels(m, std::max<int64_t>(voxels, m->nvox), s));
    SVX_CUDA(cudaStreamSynchronize(s));
    return SVX_OK;
}

svx_status svx_set_profiling(svx_map* m, int32_t enable) {
    if (!m) return fail(SVX_E_INPUT, "null argument");
    SVX_TRY(set_device(m));
    SVX_TRY(drain(m));
    if (enable && !m->h_kspan) {
        const size_t n = (size_t)kSpanKernels * 2 * kSpanMaxCtas * sizeof(unsigned long long);
        SVX_TRY(ensure(m->kspan, n, 0));
        SVX_CUDA(cudaMallocHost((void**)&m->h_kspan, n));
    }
    m->prof = enable != 0;
    return SVX_OK;
}

svx_status svx_set_score_path(svx_map* m, int32_t path) {
    if (!m) return fail(SVX_E_INPUT, "null argument");
    if (path < 0 || path > 2) return fail(SVX_E_INPUT, "unknown score path");
    m->score_path = path;
    return SVX_OK;
}

svx_status svx_set_update_mode(svx_map* m, int32_t mode) {
    if (!m) return fail(SVX_E_INPUT, "null argument");
    if (mode < SVX_UPDATE_AUTO || mode > SVX_UPDATE_LEAVES) return fail(SVX_E_INPUT, "unknown update mode");
    m->mode_pref = mode;
    return SVX_OK;
}

int32_t svx_stage_times(svx_map* m, double* ms, int32_t n) {
    if (!m) return 0;
    for (int i = 0; i < n && i < SVX_N_STAGES; ++i) ms[i] = m->stage_ms[i];
    return SVX_N_STAGES;
}

int32_t svx_frame_counters(svx_map* m, int64_t* out, int32_t n) {
    if (!m || !out) return 0;
    if (drain(m) != SVX_OK) return 0;
    // the last finished frame's mirror: asynchronous frames keep their own
    const int64_t v[6] = {(int64_t)m->last_ctr.rows, (int64_t)m->last_ctr.n_touched,
                          (int64_t)m->last_ctr.n_leaves, (int64_t)m->last_ctr.n_bigleaf,
                          (int64_t)m->last_ctr.n_long, (int64_t)m->last_ctr.n_huge};
    for (int i = 0; i < n && i < 6; ++i) out[i] = v[i];
    return 6;
}

svx_status svx_stats_get(svx_map* m, svx_stats* out) {
    if (!m || !out) return fail(SVX_E_INPUT, "null argument");
    SVX_TRY(set_device(m));
    SVX_TRY(drain(m));
    const int64_t te = (int64_t)tsdf_elem(m), se = (int64_t)sem_elem(m);
    int64_t per_vox = 2 * te + se * m->payload_d * (m->cfg.sem_kind == SVX_SEM_OPEN ? 2 : 1);
    out->leaf_count = m->nblocks;
    out->active_voxels = m->nvox;
    out->resident_bytes = m->nblocks * (int64_t)(sizeof(int4) + 8 * kMaskWords + 8 * kLeafVolume) +
                          m->nvox * per_vox + m->hcap * (int64_t)sizeof(int4);
    out->payload_bytes_per_voxel = per_vox;
    out->frames_integrated = m->frames;
    out->hash_capacity = m->hcap;
    out->voxel_capacity = m->vcap;
    out->block_capacity = m->bcap;
    out->frames_slot_mode = m->n_slot_frames;
    out->slot_overflow_reruns = m->n_slot_reruns;
    out->async_reruns = m->n_async_reruns;
    out->frames_leaf_mode = m->n_leaf_frames;
    out->last_h2d_bytes = m->io_h2d;
    out->last_d2h_bytes = m->io_d2h;
    return SVX_OK;
}

svx_status svx_active_count(svx_map* m, int64_t* count) {
    if (!m || !count) return fail(SVX_E_INPUT, "null argument");
    SVX_TRY(set_device(m));
    SVX_TRY(drain(m));
    *count = m->nvox;
    return SVX_OK;
}

svx_status svx_export_active(svx_map* m, int64_t capacity, int64_t* coords, void* d, void* w,
                             void* sem0, void* sem1, void* stream) {
    if (!m) return fail(SVX_E_INPUT, "null argument");
    SVX_TRY(set_device(m));
    SVX_TRY(drain(m));
    cudaStream_t s = (cudaStream_t)stream;
    int64_t count = 0;
    SVX_TRY(build_active_list(m, &count, s));
    if (capacity < count) return fail(SVX_E_INPUT, "output capacity smaller than active count");
    const size_t te = tsdf_elem(m), se = sem_elem(m);
    OutStage o[5];
    void *dc, *dd, *dw, *ds0, *ds1;
    svx_status st = SVX_OK;
    if ((st = out_prepare(o[0], coords, 24 * count, s, &dc)) ||
        (st = out_prepare(o[1], d, te * count, s, &dd)) ||
        (st = out_prepare(o[2], w, te * count, s, &dw)) ||
        (st = out_prepare(o[3], sem0, se * m->payload_d * count, s, &ds0)) ||
        (st = out_prepare(o[4], m->cfg.sem_kind == SVX_SEM_OPEN ? sem1 : nullptr,
                          se * m->payload_d * count, s, &ds1)) ||
        (st = launch_export(m, count, (int64_t*)dc, dd, dw, ds0, ds1, s))) {
        out_release(o, 5);
        return st;
    }
    for (int i = 0; i < 5 && st == SVX_OK; ++i) st = out_finish(o[i], s);
    cudaError_t e = cudaStreamSynchronize(s);
    out_release(o, 5);
    if (st) return st;
    if (e != cudaSuccess) return fail(SVX_E_CUDA, std::string("export: ") + cudaGetErrorString(e));
    return SVX_OK;
}

svx_status svx_probe(svx_map* m, const int64_t* coords, int64_t cnt, void* d, void* w, void* sem0,
                     void* sem1, uint8_t* active, void* stream) {
    if (!m || (cnt > 0 && !coords)) return fail(SVX_E_INPUT, "null argument");
    SVX_TRY(set_device(m));
    SVX_TRY(drain(m));
    cudaStream_t s = (cudaStream_t)stream;
    if (cnt == 0) return SVX_OK;
    DevBuf cstage;
    const void* dcoords = nullptr;
    svx_status st = stage_in(coords, 24 * cnt, cstage, s, &dcoords);
    if (st) return st;
    const size_t te = tsdf_elem(m), se = sem_elem(m);
    OutStage o[5];
    void *dd, *dw, *ds0, *ds1, *da;
    if ((st = out_prepare(o[0], d, te * cnt, s, &dd)) ||
        (st = out_prepare(o[1], w, te * cnt, s, &dw)) ||
        (st = out_prepare(o[2], sem0, se * m->payload_d * cnt, s, &ds0)) ||
        (st = out_prepare(o[3], m->cfg.sem_kind == SVX_SEM_OPEN ? sem1 : nullptr,
                          se * m->payload_d * cnt, s, &ds1)) ||
        (st = out_prepare(o[4], active, cnt, s, &da)) ||
        (st = launch_probe(m, (const int64_t*)dcoords, cnt, dd, dw, ds0, ds1, (uint8_t*)da, s))) {
        out_release(o, 5);
        release(cstage);
        return st;
    }
    for (int i = 0; i < 5 && st == SVX_OK; ++i) st = out_finish(o[i], s);
    cudaError_t e = cudaStreamSynchronize(s);
    out_release(o, 5);
    release(cstage);
    if (st) return st;
    if (e != cudaSuccess) return fail(SVX_E_CUDA, std::string("probe: ") + cudaGetErrorString(e));
    return SVX_OK;
}

svx_status svx_query_cosine(svx_map* m, const double* query, int64_t capacity, double* sims,
                            void* stream) {
    if (!m || !query) return fail(SVX_E_INPUT, "null argument");
    if (m->cfg.sem_kind != SVX_SEM_OPEN)
        return fail(SVX_E_PAYLOAD, "embedding query needs an open-set map");
    SVX_TRY(set_device(m));
    SVX_TRY(drain(m));
    cudaStream_t s = (cudaStream_t)stream;
    const int D = m->payload_d;
    // query norm on the host (D doubles)
    double* hq = new double[D];
    if (is_device_ptr(query)) {
        cudaError_t e = cudaMemcpy(hq, query, 8 * D, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) { delete[] hq; return fail(SVX_E_CUDA, cudaGetErrorString(e)); }
    } else {
        memcpy(hq, query, 8 * D);
    }
    double nn = 0.0;
    for (int c = 0; c < D; ++c) nn += hq[c] * hq[c];
    const double qn = sqrt(nn);
    if (qn == 0.0) { delete[] hq; return fail(SVX_E_INTERNAL, "zero-norm label embedding"); }
    svx_status st = ensure(m->q_buf, 8 * D, s);
    if (st) { delete[] hq; return st; }
    cudaError_t e = cudaMemcpyAsync(m->q_buf.p, hq, 8 * D, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    delete[] hq;
    if (e != cudaSuccess) return fail(SVX_E_CUDA, cudaGetErrorString(e));
    int64_t count = 0;
    SVX_TRY(build_active_list(m, &count, s));
    if (capacity < count) return fail(SVX_E_INPUT, "output capacity smaller than active count");
    OutStage o;
    void* ds;
    if ((st = out_prepare(o, sims, 8 * count, s, &ds)) ||
        (st = launch_cosine(m, count, ptr<double>(m->q_buf), qn, (double*)ds, s)) ||
        (st = out_finish(o, s))) {
        release(o.buf);
        return st;
    }
    e = cudaStreamSynchronize(s);
    release(o.buf);
    if (e != cudaSuccess) return fail(SVX_E_CUDA, std::string("query: ") + cudaGetErrorString(e));
    return SVX_OK;
}

// classify_means' query block in device memory (m->q_buf): emb (k, D) then
// the k row norms (gaussian.py:132-155).
static svx_status upload_queries(svx_map* m, const double* emb, int k, cudaStream_t s) {
    const int D = m->payload_d;
    const size_t eb = (size_t)8 * D * k;
    double* he = new double[(size_t)D * k + k];
    if (is_device_ptr(emb)) {
        cudaError_t e = cudaMemcpy(he, emb, eb, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) { delete[] he; return fail(SVX_E_CUDA, cudaGetErrorString(e)); }
    } else {
        memcpy(he, emb, eb);
    }
    double* en = he + (size_t)D * k;
    for (int j = 0; j < k; ++j) {
        double nn = 0.0;
        for (int c = 0; c < D; ++c) nn += he[(size_t)j * D + c] * he[(size_t)j * D + c];
        en[j] = sqrt(nn);
        if (en[j] == 0.0) { delete[] he; return fail(SVX_E_INTERNAL, "zero-norm label embedding"); }
    }
    svx_status st = ensure(m->q_buf, eb + 8 * k, s);
    if (st) { delete[] he; return st; }
    cudaError_t e = cudaMemcpyAsync(m->q_buf.p, he, eb + 8 * k, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    delete[] he;
    if (e != cudaSuccess) return fail(SVX_E_CUDA, cudaGetErrorString(e));
    return SVX_OK;
}

// classify_means of every active voxel (TSDF weight as the observation
// weight), stored by voxel id: the open-set labels of mesh vertices and
// rendered pixels (voxel_labels, mesh.py:392-416).
static svx_status voxel_class_labels(svx_map* m, const double* emb, int k, double temperature,
                                     double confidence_threshold, cudaStream_t s, const int** out) {
    SVX_TRY(upload_queries(m, emb, k, s));
    int64_t count = 0;
    SVX_TRY(build_active_list(m, &count, s));
    SVX_TRY(ensure(m->mesh_cls_l, 4 * std::max<int64_t>(count, 1), s));
    SVX_TRY(ensure(m->mesh_cls_b, 8 * std::max<int64_t>(count, 1), s));
    SVX_TRY(ensure(m->mesh_vlab, 4 * std::max<int64_t>(m->nvox, 1), s));
    const double* q = ptr<double>(m->q_buf);
    SVX_TRY(launch_classify(m, count, q, q + (size_t)m->payload_d * k, k, temperature,
                            confidence_threshold, ptr<int32_t>(m->mesh_cls_l),
                            ptr<double>(m->mesh_cls_b), nullptr, s));
    SVX_TRY(scatter_active_labels(m, count, ptr<int>(m->mesh_cls_l), ptr<int>(m->mesh_vlab), s));
    *out = ptr<int>(m->mesh_vlab);
    return SVX_OK;
}

svx_status svx_render(svx_map* m, const svx_render_camera* cam, int32_t mode, const double* emb,
                      int32_t k, double temperature, double confidence_threshold,
                      const uint8_t* palette, int32_t npal, void* out, void* stream) {
    if (!m || !cam || !out || (emb && k < 1)) return fail(SVX_E_INPUT, "null argument");
    if (mode != SVX_RENDER_DEPTH && mode != SVX_RENDER_SEMANTIC && mode != SVX_RENDER_NORMAL)
        return fail(SVX_E_CONFIG, "render mode must be depth, semantic or normal");
    if (mode == SVX_RENDER_SEMANTIC && m->cfg.sem_kind == SVX_SEM_NONE)
        return fail(SVX_E_CONFIG, "semantic mode needs a semantic grid");
    if (mode == SVX_RENDER_SEMANTIC && (!palette || npal < 2))
        return fail(SVX_E_INPUT, "semantic mode needs a palette of >= 2 rows");
    if (cam->width <= 0 || cam->height <= 0) return fail(SVX_E_CONFIG, "image dimensions must be positive");
    if (!(cam->near_plane > 0.0) || !(cam->far_plane > cam->near_plane))
        return fail(SVX_E_CONFIG, "near/far planes must satisfy 0 < near < far");
    SVX_TRY(set_device(m));
    SVX_TRY(drain(m));
    cudaStream_t s = (cudaStream_t)stream;
    const int* vlab = nullptr;
    if (mode == SVX_RENDER_SEMANTIC && emb && m->cfg.sem_kind == SVX_SEM_OPEN)
        SVX_TRY(voxel_class_labels(m, emb, k, temperature, confidence_threshold, s, &vlab));
    const unsigned char* pal = nullptr;
    if (mode == SVX_RENDER_SEMANTIC) {
        SVX_TRY(ensure(m->mesh_pal, 3 * (size_t)npal, s));
        SVX_CUDA(cudaMemcpyAsync(m->mesh_pal.p, palette, 3 * (size_t)npal, cudaMemcpyDefault, s));
        pal = ptr<unsigned char>(m->mesh_pal);
    }
    const int64_t npx = (int64_t)cam->width * cam->height;
    const size_t bytes = (size_t)npx * (mode == SVX_RENDER_DEPTH ? 8 : mode == SVX_RENDER_NORMAL ? 24 : 3);
    OutStage o;
    void* dout = nullptr;
    svx_status st = out_prepare(o, out, bytes, s, &dout);
    if (!st) st = render_impl(m, *cam, mode, vlab, pal, npal, dout, s);
    if (!st) st = out_finish(o, s);
    cudaError_t e = cudaStreamSynchronize(s);
    out_release(&o, 1);
    if (st) return st;
    if (e != cudaSuccess) return fail(SVX_E_CUDA, std::string("render: ") + cudaGetErrorString(e));
    return SVX_OK;
}

svx_status svx_sample_distance(svx_map* m, const double* points, int64_t n, double* vals,
                               uint8_t* valid, void* stream) {
    if (!m || (n > 0 && (!points || !vals || !valid))) return fail(SVX_E_INPUT, "null argument");
    SVX_TRY(set_device(m));
    SVX_TRY(drain(m));
    cudaStream_t s = (cudaStream_t)stream;
    DevBuf stage;
    const void* dp = nullptr;
    SVX_TRY(stage_in(points, 24 * (size_t)n, stage, s, &dp));
    OutStage o[2];
    void *dv, *dk;
    svx_status st = SVX_OK;
    if (!(st = out_prepare(o[0], vals, 8 * (size_t)n, s, &dv)) &&
        !(st = out_prepare(o[1], valid, (size_t)n, s, &dk)) &&
        !(st = sample_impl(m, n, (const double*)dp, (double*)dv, (unsigned char*)dk, s))) {
        for (int i = 0; i < 2 && st == SVX_OK; ++i) st = out_finish(o[i], s);
    }
    cudaError_t e = cudaStreamSynchronize(s);
    out_release(o, 2);
    release(stage);
    if (st) return st;
    if (e != cudaSuccess) return fail(SVX_E_CUDA, std::string("sample: ") + cudaGetErrorString(e));
    return SVX_OK;
}

svx_status svx_extract_mesh(svx_map* m, double min_weight, const double* emb, int32_t k,
                            double temperature, double confidence_threshold, int64_t* n_vertices,
                            int64_t* n_triangles, void* stream) {
    if (!m || !n_vertices || !n_triangles || (emb && k < 1)) return fail(SVX_E_INPUT, "null argument");
    SVX_TRY(set_device(m));
    SVX_TRY(drain(m));
    cudaStream_t s = (cudaStream_t)stream;
    const int* vlab = nullptr;
    if (emb && m->cfg.sem_kind == SVX_SEM_OPEN)
        SVX_TRY(voxel_class_labels(m, emb, k, temperature, confidence_threshold, s, &vlab));
    SVX_TRY(mesh_impl(m, min_weight, vlab, s));
    *n_vertices = m->mesh_nv;
    *n_triangles = m->mesh_nt;
    return SVX_OK;
}

svx_status svx_mesh_read(svx_map* m, double* vertices, int32_t* triangles, int32_t* labels,
                         uint8_t* colors, const uint8_t* palette, int32_t npal, void* stream) {
    if (!m || (colors && (!palette || npal < 2))) return fail(SVX_E_INPUT, "null argument");
    SVX_TRY(set_device(m));
    SVX_TRY(drain(m));
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nv = m->mesh_nv, nt = m->mesh_nt;
    if (vertices && nv) SVX_CUDA(cudaMemcpyAsync(vertices, m->mesh_v.p, 24 * nv, cudaMemcpyDefault, s));
    if (triangles && nt) SVX_CUDA(cudaMemcpyAsync(triangles, m->mesh_t.p, 12 * nt, cudaMemcpyDefault, s));
    if (labels && nv) SVX_CUDA(cudaMemcpyAsync(labels, m->mesh_l.p, 4 * nv, cudaMemcpyDefault, s));
    if (colors && nv) {
        SVX_TRY(ensure(m->mesh_pal, 3 * (size_t)npal, s));
        SVX_CUDA(cudaMemcpyAsync(m->mesh_pal.p, palette, 3 * (size_t)npal, cudaMemcpyDefault, s));
        SVX_TRY(ensure(m->mesh_col, 3 * nv, s));
        SVX_TRY(mesh_colors(m, ptr<unsigned char>(m->mesh_pal), npal, ptr<unsigned char>(m->mesh_col), s));
        SVX_CUDA(cudaMemcpyAsync(colors, m->mesh_col.p, 3 * nv, cudaMemcpyDefault, s));
    }
    SVX_CUDA(cudaStreamSynchronize(s));
    return SVX_OK;
}

svx_status svx_classify(svx_map* m, const double* emb, int32_t k, double temperature,
                        double confidence_threshold, int64_t capacity, int32_t* labels,
                        double* best, double* sims, void* stream) {
    if (!m || !emb || !labels || !best || k < 1) return fail(SVX_E_INPUT, "null argument");
    if (m->cfg.sem_kind != SVX_SEM_OPEN)
        return fail(SVX_E_PAYLOAD, "classification needs an open-set map");
    SVX_TRY(set_device(m));
    SVX_TRY(drain(m));
    cudaStream_t s = (cudaStream_t)stream;
    SVX_TRY(upload_queries(m, emb, k, s));
    const int D = m->payload_d;
    svx_status st = SVX_OK;
    cudaError_t e = cudaSuccess;
    int64_t count = 0;
    SVX_TRY(build_active_list(m, &count, s));
    if (capacity < count) return fail(SVX_E_INPUT, "output capacity smaller than active count");
    OutStage o[3];
    void *dl, *db, *dsm;
    if ((st = out_prepare(o[0], labels, 4 * count, s, &dl)) ||
        (st = out_prepare(o[1], best, 8 * count, s, &db)) ||
        (st = out_prepare(o[2], sims, 8 * count * k, s, &dsm)) ||
        (st = launch_classify(m, count, ptr<double>(m->q_buf), ptr<double>(m->q_buf) + (size_t)D * k,
                              k, temperature, confidence_threshold, (int32_t*)dl, (double*)db,
                              (double*)dsm, s))) {
        out_release(o, 3);
        return st;
    }
    for (int i = 0; i < 3 && st == SVX_OK; ++i) st = out_finish(o[i], s);
    e = cudaStreamSynchronize(s);
    out_release(o, 3);
    if (st) return st;
    if (e != cudaSuccess) return fail(SVX_E_CUDA, std::string("classify: ") + cudaGetErrorString(e));
    return SVX_OK;
}

svx_status svx_label_map(svx_map* m, int32_t mode, int64_t capacity, int32_t* labels,
                         void* stream) {
    if (!m || !labels) return fail(SVX_E_INPUT, "null argument");
    if (m->cfg.sem_kind != SVX_SEM_CLOSED)
        return fail(SVX_E_PAYLOAD, "label map needs a closed-set map");
    SVX_TRY(set_device(m));
    SVX_TRY(drain(m));
    cudaStream_t s = (cudaStream_t)stream;
    int64_t count = 0;
    SVX_TRY(build_active_list(m, &count, s));
    if (capacity < count) return fail(SVX_E_INPUT, "output capacity smaller than active count");
    OutStage o;
    void* dl;
    svx_status st;
    if ((st = out_prepare(o, labels, 4 * count, s, &dl)) ||
        (st = launch_label_map(m, count, mode, (int32_t*)dl, s)) || (st = out_finish(o, s))) {
        release(o.buf);
        return st;
    }
    cudaError_t e = cudaStreamSynchronize(s);
    release(o.buf);
    if (e != cudaSuccess) return fail(SVX_E_CUDA, std::string("label map: ") + cudaGetErrorString(e));
    return SVX_OK;
}

// ---- sharded integration ---------------------------------------------------

int32_t svx_leaf_owner(int64_t bx, int64_t by, int64_t bz, int32_t nranks) {
    if (nranks < 1) return -1;
    return leaf_owner(bx, by, bz, nranks);
}

svx_status svx_shard_march(svx_map* m, const void* points, int32_t points_dtype, int64_t n,
                           const double pose[16], const double origin[3], const int32_t* labels,
                           const void* feats, int32_t feats_dtype, const int64_t key_base[3],
                           void* stream, svx_shard_summary* local) {
    if (!m || !local || (!pose && !origin) || (n > 0 && !points))
        return fail(SVX_E_INPUT, "null argument");
    SVX_TRY(set_device(m));
    SVX_TRY(drain(m));
    PoseParams pp;
    memset(&pp, 0, sizeof(pp));
    if (pose) {
        for (int r = 0; r < 3; ++r) {
            for (int c = 0; c < 3; ++c) pp.R[3 * r + c] = pose[4 * r + c];
            pp.t[r] = pose[4 * r + 3];
        }
        pp.sensor = 1;
    } else {
        pp.R[0] = pp.R[4] = pp.R[8] = 1.0;
        for (int a = 0; a < 3; ++a) pp.t[a] = origin[a];
        pp.sensor = 0;
    }
    return shard_march(m, points, points_dtype == SVX_F64, n, pp, labels, feats,
                       feats_dtype == SVX_F64, key_base, (cudaStream_t)stream, local);
}

svx_status svx_shard_plan(svx_map* m, const svx_shard_summary* global, int32_t rank,
                          int32_t nranks, int64_t* send_bytes, int32_t* remarch) {
    if (!m || !global || !send_bytes || !remarch) return fail(SVX_E_INPUT, "null argument");
    SVX_TRY(set_device(m));
    SVX_TRY(drain(m));
    int rm = 0;
    svx_status st = shard_plan(m, global, rank, nranks, send_bytes, &rm, (cudaStream_t)0);
    *remarch = rm;
    return st;
}

svx_status svx_shard_pack(svx_map* m, void* send, int64_t capacity, void* stream) {
    if (!m) return fail(SVX_E_INPUT, "null argument");
    SVX_TRY(set_device(m));
    SVX_TRY(drain(m));
    return shard_pack(m, send, capacity, (cudaStream_t)stream);
}

svx_status svx_shard_apply(svx_map* m, const void* recv, const int64_t* recv_bytes, int32_t nranks,
                           void* stream, svx_report* report) {
    if (!m || !recv_bytes) return fail(SVX_E_INPUT, "null argument");
    SVX_TRY(set_device(m));
    SVX_TRY(drain(m));
    return shard_apply(m, recv, recv_bytes, nranks, (cudaStream_t)stream, report);
}

static PoseParams shard_pose(const double pose[16], const double origin[3]) {
    PoseParams pp;
    memset(&pp, 0, sizeof(pp));
    if (pose) {
        for (int r = 0; r < 3; ++r) {
            for (int c = 0; c < 3; ++c) pp.R[3 * r + c] = pose[4 * r + c];
            pp.t[r] = pose[4 * r + 3];
        }
        pp.sensor = 1;
    } else {
        pp.R[0] = pp.R[4] = pp.R[8] = 1.0;
        for (int a = 0; a < 3; ++a) pp.t[a] = origin[a];
        pp.sensor = 0;
    }
    return pp;
}

svx_status svx_shard_march_async(svx_map* m, const void* points, int32_t points_dtype, int64_t n,
                                 const double pose[16], const double origin[3], const int32_t* labels,
                                 const void* feats, int32_t feats_dtype, const int64_t key_base[3],
                                 void* stream, int64_t* summary) {
    if (!m || !summary || (!pose && !origin) || (n > 0 && !points)) return fail(SVX_E_INPUT, "null argument");
    SVX_TRY(set_device(m));
    SVX_TRY(drain(m));
    return shard_march_async(m, points, points_dtype == SVX_F64, n, shard_pose(pose, origin), labels, feats,
                             feats_dtype == SVX_F64, key_base, (cudaStream_t)stream, summary);
}

svx_status svx_shard_plan_async(svx_map* m, const int64_t* global_summary, int32_t rank, int32_t nranks,
                                int64_t cap, void* stream, int64_t* abort_words) {
    if (!m || !global_summary || !abort_words) return fail(SVX_E_INPUT, "null argument");
    SVX_TRY(set_device(m));
    return shard_plan_async(m, global_summary, rank, nranks, cap, (cudaStream_t)stream, abort_words);
}

svx_status svx_shard_pack_async(svx_map* m, void* send, int64_t cap, void* stream, const int64_t* abort_words) {
    if (!m || !abort_words) return fail(SVX_E_INPUT, "null argument");
    SVX_TRY(set_device(m));
    return shard_pack_async(m, send, cap, (cudaStream_t)stream, abort_words);
}

svx_status svx_shard_apply_async(svx_map* m, const void* recv, int64_t cap, int32_t nranks,
                                 const int64_t* abort_words, int64_t frame_points, void* stream,
                                 int64_t* report_words) {
    if (!m || !abort_words || !report_words) return fail(SVX_E_INPUT, "null argument");
    SVX_TRY(set_device(m));
    return shard_apply_async(m, recv, cap, nranks, abort_words, frame_points, (cudaStream_t)stream,
                             report_words);
}

svx_status svx_shard_finish(svx_map* m, const int64_t* summary, const int64_t* abort_words,
                            const int64_t* report_sum, svx_report* report, int32_t* action, int64_t* need) {
    if (!m || !summary || !abort_words || !action || !need) return fail(SVX_E_INPUT, "null argument");
    SVX_TRY(set_device(m));
    return shard_finish(m, summary, abort_words, report_sum, report, action, need);
}

svx_status svx_export_leaf_stamps(svx_map* m, int64_t capacity, int32_t* frame, uint64_t* key,
                                  int32_t* count, int64_t* nleaves, void* stream) {
    if (!m || !nleaves) return fail(SVX_E_INPUT, "null argument");
    SVX_TRY(set_device(m));
    SVX_TRY(drain(m));
    cudaStream_t s = (cudaStream_t)stream;
    int64_t vox = 0;
    SVX_TRY(build_active_list(m, &vox, s));
    const int64_t nb = vox ? m->nblocks : 0;
    *nleaves = nb;
    if (capacity < nb) return fail(SVX_E_INPUT, "output capacity smaller than leaf count");
    OutStage o[3];
    void *df, *dk, *dn;
    svx_status st = SVX_OK;
    if ((st = out_prepare(o[0], frame, 4 * nb, s, &df)) ||
        (st = out_prepare(o[1], key, 8 * nb, s, &dk)) ||
        (st = out_prepare(o[2], count, 4 * nb, s, &dn)) ||
        (st = launch_leaf_stamps(m, (int32_t*)df, (uint64_t*)dk, (int32_t*)dn, s))) {
        out_release(o, 3);
        return st;
    }
    for (int i = 0; i < 3 && st == SVX_OK; ++i) st = out_finish(o[i], s);
    cudaError_t e = cudaStreamSynchronize(s);
    out_release(o, 3);
    if (st) return st;
    if (e != cudaSuccess) return fail(SVX_E_CUDA, std::string("leaf stamps: ") + cudaGetErrorString(e));
    return SVX_OK;
}

}  // extern "C"

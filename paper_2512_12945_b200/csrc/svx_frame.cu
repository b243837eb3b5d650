// svx_frame.cu -- per-frame orchestration of the integration path.
//
// A frame is a short kernel chain plus two small copies, all reading their
// per-frame values from the device-side FrameCtr (svx_internal.cuh):
//   H2D   frame parameters + zeroed counters (one pinned copy)
//   K1    march     masks, ray setup, fp64 band walk -> row keys     (svx_march.cu)
//         gate      the reference's pre-allocation checks            (svx_march.cu)
//   K2    resolve   rows -> leaf/voxel ids, per-voxel row counts     (svx_resolve.cu)
//   K3    segments  multi-row voxels -> row segments                 (svx_resolve.cu)
//   K4    scatter   rows -> segments; single-row voxels updated      (svx_update.cu)
//   K5    update    fused TSDF + closed/open update per voxel        (svx_update.cu)
//   D2H   counters (one pinned copy)
// The chain is captured once into a CUDA graph and replayed while buffer
// addresses stay the same; the host synchronises once per frame to read the
// report.  Error checks stop a frame before any map mutation; a frame whose
// pools or row slots turned out too small is cleaned up and re-run.
#include <cuda_runtime.h>
#include <limits.h>
#include <math.h>
#include <string.h>

#include <cmath>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "svx_internal.cuh"

namespace svx {

// SVX_TRACE_HOST=1: per-frame host-side phase times (us) on stderr.
static double now_us() {
    return std::chrono::duration<double, std::micro>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}
static const bool g_trace_host = getenv("SVX_TRACE_HOST") != nullptr;
static double g_t_launch0 = 0, g_t_launch1 = 0, g_t_synced = 0;

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Device address of page-locked host memory (mapped under UVA), else null.
static const void* pinned_device_ptr(const void* p) {
    if (!p) return nullptr;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

static const bool g_no_zero_copy = getenv("SVX_NO_ZERO_COPY") != nullptr;   // A/B switch

svx_status stage_in(const void* p, size_t bytes, DevBuf& stage, cudaStream_t s, const void** out) {
    if (!p || bytes == 0) {
        *out = p;
        return SVX_OK;
    }
    if (is_device_ptr(p)) {
        *out = p;
        return SVX_OK;
    }
    SVX_TRY(ensure(stage, bytes, s));
    SVX_CUDA(cudaMemcpyAsync(stage.p, p, bytes, cudaMemcpyHostToDevice, s));
    *out = stage.p;
    return SVX_OK;
}

size_t tsdf_elem(const svx_map* m) { return m->cfg.tsdf_dtype == SVX_F64 ? 8 : 4; }

size_t sem_elem(const svx_map* m) {
    if (m->cfg.sem_kind == SVX_SEM_CLOSED) return m->cfg.count_dtype == SVX_F64 ? 8 : 4;
    if (m->cfg.sem_kind == SVX_SEM_OPEN) return m->cfg.state_dtype == SVX_F64 ? 8 : 4;
    return 0;
}

// Voxel-pool capacity: grow by doubling.  Closed counts and open means are
// zero-filled (their background); the per-voxel frame counts start at zero.
svx_status reserve_voxels(svx_map* m, int64_t need, cudaStream_t s) {
    if (need <= m->vcap) return SVX_OK;
    int64_t cap = std::max<int64_t>(need, 2 * m->vcap);
    const size_t te = tsdf_elem(m), se = sem_elem(m);
    SVX_TRY(ensure(m->vt, 2 * te * cap, s, true));
    if (m->cfg.sem_kind != SVX_SEM_NONE)
        SVX_TRY(ensure(m->s0, se * (size_t)m->payload_d * cap, s, true, 0));
    if (m->cfg.sem_kind == SVX_SEM_OPEN)
        SVX_TRY(ensure(m->s1, se * (size_t)m->payload_d * cap, s, true, 0));
    SVX_TRY(ensure(m->vrec, sizeof(VoxFrame) * cap, s, true, 0));
    if (m->cfg.sem_kind != SVX_SEM_OPEN && !m->cfg.space_carving)   // per-frame contents only
        SVX_TRY(ensure(m->vslot, sizeof(RowSlot) * kSlots * kSlotStride * cap, s));
    m->vcap = cap;
    return SVX_OK;
}

svx_status reserve_blocks(svx_map* m, int64_t need, cudaStream_t s) {
    if (need > m->bcap) {
        int64_t cap = std::max<int64_t>(need, 2 * m->bcap);
        SVX_TRY(ensure(m->bcoord, sizeof(int4) * cap, s, true));
        SVX_TRY(ensure(m->bkey, sizeof(unsigned long long) * cap, s, true, 0xFF));
        SVX_TRY(ensure(m->bmask, sizeof(unsigned long long) * kMaskWords * cap, s, true, 0));
        const int64_t old = m->bcap;
        SVX_TRY(ensure(m->bslot, sizeof(unsigned long long) * kLeafVolume * cap, s, true));
        SVX_TRY(launch_fill_u64(ptr<unsigned long long>(m->bslot) + old * kLeafVolume,
                                (cap - old) * kLeafVolume, kSlotInactive, s));
        if (m->cfg.sem_kind != SVX_SEM_OPEN && !m->cfg.space_carving)   // leaf-mode frame counts
            SVX_TRY(ensure(m->lcnt, sizeof(unsigned long long) * cap, s, true, 0));
        m->bcap = cap;
    }
    // keep the leaf hash at <= 50% load when the pool is full
    int64_t want = 1024;
    while (want < 2 * m->bcap) want <<= 1;
    if (want > m->hcap) {
        DevBuf nt;
        SVX_TRY(ensure(nt, sizeof(int4) * want, s, false, 0xFF));
        SVX_TRY(launch_rehash(m, ptr<int4>(nt), want, s));
        SVX_CUDA(cudaStreamSynchronize(s));
        release(m->hash);
        m->hash = nt;
        m->hcap = want;
    }
    return SVX_OK;
}

// Per-frame scratch: per-ray arrays for npts_cap points, row arrays for the
// row space (slot mode: npts_cap * maxrows, dense: rcap), lists for ucap.
svx_status reserve_frame(svx_map* m, int64_t n, cudaStream_t s) {
    m->npts_cap = std::max<int64_t>(m->npts_cap, n);
    const int64_t rows = (int64_t)m->rcap;
    m->ucap = (uint64_t)rows;
    SVX_TRY(ensure(m->ray, sizeof(double4) * m->npts_cap, s));
    SVX_TRY(ensure(m->rcnt, sizeof(int) * m->npts_cap, s));
    SVX_TRY(ensure(m->partials, partials_bytes() + segment_status_bytes(m->ucap), s, false, 0));
    SVX_TRY(ensure(m->rowkey, sizeof(unsigned long long) * rows, s));
    SVX_TRY(ensure(m->rowvid, sizeof(int) * rows, s));
    SVX_TRY(ensure(m->tlist, std::max<size_t>(sizeof(int) * rows,
                                              sizeof(TouchEntry) * kPersistentBlocks * slot_region(rows)), s));
    SVX_TRY(ensure(m->rcount, sizeof(unsigned) * kPersistentBlocks, s));
    SVX_TRY(ensure(m->mlist, sizeof(int) * rows, s));
    SVX_TRY(ensure(m->longlist, 2 * sizeof(int) * rows, s));   // long list, then huge list
    SVX_TRY(ensure(m->srid, sizeof(int) * rows, s));
    SVX_TRY(ensure(m->bitmap, (size_t)4 * huge_warps() * ((m->npts_cap + 31) / 32 + 1), s));
    if (m->cfg.sem_kind == SVX_SEM_OPEN)   // huge voxels have > open_cta_min() rows each
        SVX_TRY(ensure(m->hinfo, huge_info_bytes() * (size_t)(rows / open_cta_min() + 2), s));
    SVX_TRY(ensure(m->rowray, sizeof(int) * rows, s));
    if (m->cfg.sem_kind != SVX_SEM_OPEN && !m->cfg.space_carving) {   // slot / leaf mode rows
        SVX_TRY(ensure(m->rowd, sizeof(double) * rows, s));
        SVX_TRY(ensure(m->rowlab, sizeof(int) * rows, s));
        SVX_TRY(ensure(m->rowleaf, sizeof(unsigned long long) * rows, s));
        SVX_TRY(ensure(m->rowpk, sizeof(unsigned) * rows, s));
        SVX_TRY(ensure(m->binrow, sizeof(unsigned) * rows, s));
    }
    if (m->maxrows == 0) {   // two-pass walk: per-ray offsets from a scan
        SVX_TRY(ensure(m->roff, sizeof(long long) * m->npts_cap, s));
        SVX_TRY(ensure(m->cubtmp, scan_temp_bytes(m->npts_cap), s));
    }
    m->rcap_sized = m->rcap;
    return SVX_OK;
}

// Everything a captured graph bakes in: buffer addresses, capacities that
// size grids or index scratch, and kernel template choices.
static unsigned long long graph_signature(const svx_map* m, int pts_f64, int feats_f64) {
    const void* ptrs[] = {m->ray.p,    m->rcnt.p,   m->roff.p,    m->rowkey.p, m->rowvid.p,
                          m->rowray.p, m->partials.p, m->tlist.p, m->mlist.p,  m->longlist.p, m->rcount.p,
                          m->srid.p,   m->bitmap.p, m->cubtmp.p,  m->hash.p,   m->bcoord.p,
                          m->bkey.p,   m->bmask.p,  m->bslot.p,   m->vt.p,     m->s0.p,
                          m->s1.p,     m->vrec.p,   m->vslot.p,   m->rowd.p,   m->rowlab.p,
                          m->ctr.p,    m->hinfo.p,  m->lcnt.p,    m->rowleaf.p, m->rowpk.p,
                          m->binrow.p};
    unsigned long long h = 1469598103934665603ULL;
    auto mix = [&](unsigned long long v) {
        h ^= v;
        h *= 1099511628211ULL;
    };
    for (const void* p : ptrs) mix((unsigned long long)(uintptr_t)p);
    mix(m->ucap);
    mix((unsigned long long)m->npts_cap);
    mix((unsigned long long)m->maxrows);
    mix((unsigned long long)(pts_f64 * 2 + feats_f64));
    return h;
}


// Enqueue one frame attempt on stream s (under graph capture).  No copy
// nodes: the first kernel reads the parameters from the mapped host
// FrameCtr, the last kernel's epilogue writes the counters back into it.
static svx_status enqueue_frame(svx_map* m, int pts_f64, int feats_f64, cudaStream_t s) {
    SVX_TRY(launch_march(m, pts_f64, feats_f64, s));
    if (m->frame_leaf) return launch_leaf(m, s);
    SVX_TRY(launch_resolve(m, s));
    if (m->frame_slots) return launch_update_slots(m, s);
    SVX_TRY(launch_segments(m, s));
    SVX_TRY(launch_scatter(m, s));
    SVX_TRY(launch_update_a(m, feats_f64, s));
    SVX_TRY(launch_update_b(m, feats_f64, s));
    return SVX_OK;
}

// Bring the device FrameCtr to the reset state the graph frames assume
// (after the sharded calls or a host-side change of the live pool counts).
svx_status clean_ctr(svx_map* m, cudaStream_t s) {
    if (m->ctr_clean) return SVX_OK;
    FrameCtr img;
    memset(&img, 0, sizeof(img));
    for (int a = 0; a < 3; ++a) {
        img.bbox_min[a] = LLONG_MAX;
        img.bbox_max[a] = LLONG_MIN;
    }
    img.nblocks = (unsigned long long)m->nblocks;
    img.nvox = (unsigned long long)m->nvox;
    SVX_CUDA(cudaMemcpyAsync(m->ctr.p, &img, sizeof(img), cudaMemcpyHostToDevice, s));
    SVX_CUDA(cudaStreamSynchronize(s));
    m->ctr_clean = true;
    return SVX_OK;
}

// Profiling: per-kernel spans recorded by the kernels themselves (KSpan),
// plus the frame span from the first kernel start to the last kernel end.
static svx_status collect_stage_times(svx_map* m) {
    const size_t n = (size_t)kSpanKernels * 2 * kSpanMaxCtas;
    SVX_CUDA(cudaMemcpy(m->h_kspan, m->kspan.p, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    unsigned long long t0 = ~0ULL, t1 = 0;
    for (int k = 0; k < kSpanKernels; ++k) {
        unsigned long long a = ~0ULL, b = 0;
        const unsigned long long* st = m->h_kspan + (size_t)k * 2 * kSpanMaxCtas;
        for (int c = 0; c < kSpanMaxCtas; ++c) {
            if (st[c] && st[c] < a) a = st[c];
            if (st[kSpanMaxCtas + c] > b) b = st[kSpanMaxCtas + c];
        }
        m->stage_ms[k] = (a != ~0ULL && b > a) ? (double)(b - a) * 1e-6 : 0.0;
        if (a != ~0ULL && b > a) {
            t0 = a < t0 ? a : t0;
            t1 = b > t1 ? b : t1;
        }
    }
    m->stage_ms[kSpanKernels] = t1 > t0 ? (double)(t1 - t0) * 1e-6 : 0.0;
    return SVX_OK;
}

// Launch one frame attempt: replay (or capture, on the map's own stream) the
// frame graph on the caller's stream; ev_end is recorded after it.  The
// frame's parameters are read from m->h_ctr->p (the mirror the attempt
// uses).
static const bool g_no_graph = getenv("SVX_NO_GRAPH") != nullptr;   // experiment: eager launches

static svx_status launch_frame(svx_map* m, int pts_f64, int feats_f64, cudaStream_t s,
                               cudaEvent_t ev_end) {
    if (g_no_graph) {
        if (m->prof) {
            const size_t n = (size_t)kSpanKernels * 2 * kSpanMaxCtas * sizeof(unsigned long long);
            SVX_CUDA(cudaMemsetAsync(m->kspan.p, 0, n, s));
        }
        SVX_TRY(clean_ctr(m, s));
        if (g_trace_host) g_t_launch0 = now_us();
        SVX_TRY(enqueue_frame(m, pts_f64, feats_f64, s));
        SVX_CUDA(cudaEventRecord(ev_end, s));
        if (g_trace_host) g_t_launch1 = now_us();
        return SVX_OK;
    }
    const unsigned long long sig = graph_signature(m, pts_f64, feats_f64);
    const int gm = m->frame_leaf ? 2 : (m->frame_slots ? 1 : 0);
    cudaGraphExec_t& gexec = m->gexec[gm][m->exec_slot];
    if (!m->graph[gm] || sig != m->gsig[gm]) {
        for (cudaGraphExec_t& g : m->gexec[gm])
            if (g) {
                cudaGraphExecDestroy(g);
                g = nullptr;
            }
        if (m->graph[gm]) {
            cudaGraphDestroy(m->graph[gm]);
            m->graph[gm] = nullptr;
        }
        SVX_CUDA(cudaStreamBeginCapture(m->gstream, cudaStreamCaptureModeThreadLocal));
        svx_status st = enqueue_frame(m, pts_f64, feats_f64, m->gstream);
        cudaGraph_t g = nullptr;
        cudaError_t e = cudaStreamEndCapture(m->gstream, &g);
        if (st != SVX_OK) {
            if (g) cudaGraphDestroy(g);
            return st;
        }
        if (e != cudaSuccess) return fail(SVX_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
        // the frame's first kernel is the graph's only root
        size_t nroots = 1;
        cudaGraphNode_t root = nullptr;
        e = cudaGraphGetRootNodes(g, &root, &nroots);
        cudaGraphNodeType ty;
        if (e != cudaSuccess || nroots != 1 || cudaGraphNodeGetType(root, &ty) != cudaSuccess ||
            ty != cudaGraphNodeTypeKernel) {
            cudaGraphDestroy(g);
            return fail(SVX_E_INTERNAL, "frame graph: expected one root kernel node");
        }
        m->graph[gm] = g;
        m->walk_node[gm] = root;
        m->walk_nargs[gm] = m->first_nargs;
        const int na = m->first_nargs;
        if (na < 1 || na > 16) return fail(SVX_E_INTERNAL, "frame graph: bad first-kernel arity");
        SVX_CUDA(cudaGraphKernelNodeGetParams(root, &m->walk_kp[gm]));
        for (int i = 0; i < na - 1; ++i) m->walk_args[gm][i] = m->walk_kp[gm].kernelParams[i];
        m->walk_kp[gm].kernelParams = m->walk_args[gm];
        m->walk_kp[gm].extra = nullptr;
        m->gsig[gm] = sig;
        size_t nn = 0;
        cudaGraphGetNodes(g, nullptr, &nn);
        std::vector<cudaGraphNode_t> nodes(nn);
        int nk = 0;
        if (nn && cudaGraphGetNodes(g, nodes.data(), &nn) == cudaSuccess)
            for (cudaGraphNode_t nd : nodes) {
                cudaGraphNodeType t;
                if (cudaGraphNodeGetType(nd, &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++nk;
            }
        m->graph_kernels[gm] = nk;
    }
    if (!gexec) {
        cudaError_t e = cudaGraphInstantiate(&gexec, m->graph[gm], 0);
        if (e != cudaSuccess) {
            gexec = nullptr;
            return fail(SVX_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
        }
    }
    // this frame's parameters (in the attempt's mirror) into the first kernel's
    // FrameParams argument; an instantiated graph copies them at this call, so
    // launches already queued keep theirs
    m->walk_args[gm][m->walk_nargs[gm] - 1] = &m->h_ctr->p;
    SVX_CUDA(cudaGraphExecKernelNodeSetParams(gexec, m->walk_node[gm], &m->walk_kp[gm]));
    if (m->prof) {
        const size_t n = (size_t)kSpanKernels * 2 * kSpanMaxCtas * sizeof(unsigned long long);
        SVX_CUDA(cudaMemsetAsync(m->kspan.p, 0, n, s));
    }
    SVX_TRY(clean_ctr(m, s));
    // the graph was captured on the map's own stream; it runs on the caller's
    if (g_trace_host) g_t_launch0 = now_us();
    SVX_CUDA(cudaGraphLaunch(gexec, s));
    count_launch(m->graph_kernels[gm]);   // the frame graph's kernel nodes
    SVX_CUDA(cudaEventRecord(ev_end, s));
    if (g_trace_host) g_t_launch1 = now_us();
    return SVX_OK;
}

// Run one frame attempt and wait for it (synchronous frames).
static svx_status run_frame(svx_map* m, int pts_f64, int feats_f64, cudaStream_t s) {
    SVX_TRY(launch_frame(m, pts_f64, feats_f64, s, m->ev1));
    SVX_CUDA(cudaEventSynchronize(m->ev1));
    if (g_trace_host) g_t_synced = now_us();
    if (m->prof) SVX_TRY(collect_stage_times(m));
    return SVX_OK;
}

// Row space.  A band of length L crosses at most 3 * (L / h + 1) voxels;
// without carving L = 2 * trunc, so each ray gets that many row slots.
// Carving bands are unbounded: rows are counted, scanned and packed.
void init_row_space(svx_map* m, int64_t n) {
    const double h = m->cfg.voxel_size;
    if (m->maxrows < 0) {
        const double bound = 3.0 * (2.0 * m->cfg.truncation / h + 1.0) + 3.0;
        m->maxrows = (m->cfg.space_carving || bound > 32.0) ? 0 : (int)bound;
    }
    if (m->rcap == 0)   // first frame: the bound (bounded bands) or a guess; adapted per frame
        m->rcap = m->maxrows > 0 ? (uint64_t)n * m->maxrows + 4096 : (uint64_t)n * 32 + 4096;
}

// Pool headroom: every row could open a voxel (closed/geometry), an eighth
// of them for open-set payloads; leaves get twice what recent frames
// created.  A shortfall is caught on the device and the frame re-run.
svx_status reserve_pools(svx_map* m, cudaStream_t s) {
    const int64_t rows_bound = (int64_t)m->ucap;
    const int64_t vhead = m->cfg.sem_kind == SVX_SEM_OPEN ? std::max<int64_t>(rows_bound / 8, 1 << 16)
                                                          : rows_bound;
    SVX_TRY(reserve_voxels(m, m->nvox + vhead, s));
    SVX_TRY(reserve_blocks(m, m->nblocks + std::max<int64_t>(m->new_leaves_cap, 4096), s));
    return SVX_OK;
}

// Zeroed counters with the live pool counts; FrameParams are filled by the caller.
void reset_ctr(svx_map* m, int64_t stamp) {
    FrameCtr* hc = m->h_ctr;
    memset(hc, 0, sizeof(FrameCtr));
    for (int a = 0; a < 3; ++a) {
        hc->bbox_min[a] = LLONG_MAX;
        hc->bbox_max[a] = LLONG_MIN;
    }
    hc->nblocks = (unsigned long long)m->nblocks;
    hc->nvox = (unsigned long long)m->nvox;
    FrameParams& p = hc->p;
    p.ucap = m->ucap;
    p.rcap = m->rcap;
    p.hmask = m->hcap - 1;
    p.bcap = m->bcap;
    p.vcap = m->vcap;
    p.frame = (int)stamp;
    p.maxrows = m->maxrows;
    p.inline_singles = inline_singles(m);
    p.slots = m->frame_slots;
    p.kspan = m->prof ? ptr<unsigned long long>(m->kspan) : nullptr;
    p.mirror = m->d_hctr;
    p.epilogue = 1;   // graph frames; the sharded calls copy explicitly and set 0
    p.region = slot_region(m->rcap);
    p.seq = ++m->seq;
}

// K2 ran out of leaf or voxel pool: give what it activated its background
// state, clear the frame counts and grow; the allocation counters carry over
// and the caller runs the frame again.
svx_status recover_capacity(svx_map* m, int64_t nblocks0, cudaStream_t s) {
    FrameCtr* hc = m->h_ctr;
    // the attempt's allocation counters kept counting past the pools: they
    // are the frame's demand (voxels of leaves that could not be created are
    // not in it yet, so a second retry can still be needed)
    const int64_t want_b = (int64_t)hc->nblocks, want_v = (int64_t)hc->nvox;
    SVX_TRY(launch_cleanup(m, s));
    SVX_CUDA(cudaStreamSynchronize(s));
    m->nblocks = std::min<int64_t>(want_b, m->bcap);
    m->nvox = std::min<int64_t>(want_v, m->vcap);
    m->ord_nblocks = std::min<int64_t>(m->ord_nblocks, nblocks0);
    m->ctr_clean = false;   // live counts may have been clamped to the pools
    m->new_leaves_cap = std::max<int64_t>(m->new_leaves_cap, 2 * (want_b - nblocks0) + 4096);
    if (want_b >= m->bcap) SVX_TRY(reserve_blocks(m, want_b + want_b / 2 + 4096, s));
    if (want_v >= m->vcap) SVX_TRY(reserve_voxels(m, want_v + want_v / 2 + 65536, s));
    return SVX_OK;
}

// Slot mode stopped before any payload change (a voxel got more than kSlots
// rows): same cleanup as a capacity abort, then the caller re-runs the frame
// in segment mode and stays there for a while.
svx_status recover_slots(svx_map* m, int64_t nblocks0, cudaStream_t s) {
    FrameCtr* hc = m->h_ctr;
    SVX_TRY(launch_cleanup(m, s));
    SVX_CUDA(cudaStreamSynchronize(s));
    m->nblocks = (int64_t)std::min<unsigned long long>(hc->nblocks, (unsigned long long)m->bcap);
    m->nvox = (int64_t)std::min<unsigned long long>(hc->nvox, (unsigned long long)m->vcap);
    m->ord_nblocks = std::min<int64_t>(m->ord_nblocks, nblocks0);
    m->ctr_clean = false;
    m->slot_hold = 32;
    m->frame_retry_segments = 1;
    m->n_slot_reruns++;
    return SVX_OK;
}

// Slot mode for bounded-band closed/geometry maps whose recent frames fit
// kSlots rows per voxel (LiDAR: ~1.6 rows per voxel); depth cameras (~17
// rows per voxel), open-set and carving maps use segments.
int choose_slots(const svx_map* m) {
    if (m->cfg.sem_kind == SVX_SEM_OPEN || m->cfg.space_carving || m->maxrows <= 0) return 0;
    if (m->mode_pref == SVX_UPDATE_SEGMENTS) return 0;
    if (m->mode_pref == SVX_UPDATE_SLOTS || m->mode_pref == SVX_UPDATE_LEAVES)
        return m->frame_retry_segments ? 0 : 1;
    if (m->slot_hold > 0) return 0;
    return m->last_rows <= 3 * m->last_touched ? 1 : 0;
}

// Slot and leaf mode serve the same frames (bounded-band closed/geometry
// maps whose recent frames fit few rows per voxel); auto picks slot mode
// (measured faster on cfg2: frame span 79 vs 130 us).
void choose_mode(svx_map* m, int64_t n) {
    const int lidar_like = choose_slots(m);
    m->frame_slots = 0;
    m->frame_leaf = 0;
    if (!lidar_like) return;
    if (m->mode_pref == SVX_UPDATE_LEAVES && leaf_mode_fits(n)) m->frame_leaf = 1;
    else m->frame_slots = 1;
}

// Report fields of the map side and the capacities for the next frame.
void finish_frame(svx_map* m, int64_t nblocks0, int64_t nvox0, svx_report& r) {
    FrameCtr* hc = m->h_ctr;
    m->last_ctr = *hc;
    r.touched_voxels = (int64_t)hc->n_touched;
    r.new_blocks = (int64_t)hc->nblocks - nblocks0;
    r.new_voxels = (int64_t)hc->nvox - nvox0;
    m->new_leaves_cap = std::max<int64_t>(m->new_leaves_cap, 2 * r.new_blocks + 1024);
    m->nblocks = (int64_t)hc->nblocks;
    m->nvox = (int64_t)hc->nvox;
    m->n_slot_frames += m->frame_slots;
    m->n_leaf_frames += m->frame_leaf;
    m->last_rows = (int64_t)hc->rows;
    m->last_touched = (int64_t)hc->n_touched;
    if (m->slot_hold > 0) --m->slot_hold;
    // row capacity for the next frame: 1.5x this one's rows
    const uint64_t need = hc->rows + hc->rows / 2 + 4096;
    if (hc->rows * 10 > m->rcap * 8 || need * 3 < m->rcap) m->rcap = need;
}

// Packed keys are offsets from the sensor's voxel minus 2^20 per axis.
KeyPack default_key_pack(const svx_map* m, const PoseParams& pp) {
    KeyPack kp;
    const long long half = 1LL << (kPackBits - 1);
    for (int a = 0; a < 3; ++a) kp.base[a] = (long long)floor(pp.t[a] / m->cfg.voxel_size) - half;
    return kp;
}

svx_status integrate_impl(svx_map* m, const void* pts_in, int pts_f64, int64_t n,
                          const PoseParams& pp, const int32_t* labels_in, const void* feats_in,
                          int feats_f64, cudaStream_t s, svx_report* rep, int device_inputs,
                          const FrameOpts* opt) {
    const double t_enter = g_trace_host ? now_us() : 0.0;
    const bool rerun = opt && opt->stamp >= 0;
    const int64_t stamp = rerun ? opt->stamp : m->frames;
    svx_report r;
    memset(&r, 0, sizeof(r));
    r.points_in = n;
    const int kind = m->cfg.sem_kind;
    // (an empty payload array arrives as NULL; presence is checked on the host)
    if (kind == SVX_SEM_CLOSED && !labels_in && n > 0)
        return fail(SVX_E_PAYLOAD, "closed-set grid requires per-point labels");
    if (kind == SVX_SEM_OPEN && !feats_in && n > 0)
        return fail(SVX_E_PAYLOAD, "open-set grid requires per-point features");
    if (n < 0) return fail(SVX_E_INPUT, "negative point count");
    if (n >= (int64_t)INT_MAX) return fail(SVX_E_INPUT, "point count exceeds 2^31-1");
    if (n == 0) {
        if (!rerun) m->frames++;
        if (rep) *rep = r;
        return SVX_OK;
    }
    m->h_ctr = m->h_ctr0;   // synchronous frames use the map's own mirror
    m->d_hctr = m->d_hctr0;
    SVX_CUDA(cudaEventRecord(m->ev0, s));
    const void* pts = pts_in;
    const void* feats = kind == SVX_SEM_OPEN ? feats_in : nullptr;
    const void* labv = kind == SVX_SEM_CLOSED ? (const void*)labels_in : nullptr;
    // Pinned host points/labels of closed-set and geometry frames are read
    // in place by the walk (zero-copy over the host link) when the frame
    // runs in slot mode: the walk is their only reader there, so the
    // transfer overlaps the band walk instead of preceding it.  Segment-mode
    // frames read labels again by point index and get a device copy.
    const void* zc_pts = nullptr;
    const void* zc_lab = nullptr;
    if (!device_inputs && kind != SVX_SEM_OPEN && !g_no_zero_copy) {
        zc_pts = pinned_device_ptr(pts_in);
        if (zc_pts && kind == SVX_SEM_CLOSED) {
            zc_lab = pinned_device_ptr(labels_in);
            if (!zc_lab) zc_pts = nullptr;
        }
    }
    bool staged = device_inputs != 0;
    auto stage_all = [&]() -> svx_status {
        SVX_TRY(stage_in(pts_in, (size_t)n * 3 * (pts_f64 ? 8 : 4), m->in_pts, s, &pts));
        if (kind == SVX_SEM_CLOSED) SVX_TRY(stage_in(labels_in, (size_t)n * 4, m->in_lab, s, &labv));
        if (kind == SVX_SEM_OPEN)
            SVX_TRY(stage_in(feats_in, (size_t)n * m->payload_d * (feats_f64 ? 8 : 4), m->in_feat, s,
                             &feats));
        staged = true;
        return SVX_OK;
    };
    if (!staged && !zc_pts) SVX_TRY(stage_all());
    if (!device_inputs && !rerun) {   // host-link bytes: inputs in (copied or read in place)
        const bool host_p = zc_pts || (pts != pts_in);
        m->io_h2d = host_p ? (int64_t)n * 3 * (pts_f64 ? 8 : 4) : 0;
        if (kind == SVX_SEM_CLOSED && (zc_lab || labv != (const void*)labels_in)) m->io_h2d += n * 4;
        if (kind == SVX_SEM_OPEN && feats != feats_in)
            m->io_h2d += (int64_t)n * m->payload_d * (feats_f64 ? 8 : 4);
    } else if (!rerun) {
        m->io_h2d = 0;
    }
    m->io_d2h = (int64_t)sizeof(FrameCtr);   // the counter mirror the last kernel writes
    init_row_space(m, n);
    KeyPack kp = default_key_pack(m, pp);
    FrameCtr* hc = m->h_ctr;
    // counts before this frame (stamps, report); m->nblocks / m->nvox stay the
    // live counts, including what a capacity-aborted attempt allocated
    const int64_t nblocks0 = opt && opt->nblocks0 >= 0 ? opt->nblocks0 : m->nblocks;
    const int64_t nvox0 = opt && opt->nvox0 >= 0 ? opt->nvox0 : m->nvox;
    m->frame_retry_segments = opt ? opt->force_segments : 0;
    for (int attempt = 0;; ++attempt) {
        if (attempt >= 8) return fail(SVX_E_INTERNAL, "frame scratch could not be sized");
        SVX_TRY(reserve_frame(m, n, s));
        SVX_TRY(reserve_pools(m, s));
        choose_mode(m, n);
        if (!staged && !m->frame_slots) SVX_TRY(stage_all());
        reset_ctr(m, stamp);
        FrameParams& p = hc->p;
        p.pts = staged ? pts : zc_pts;
        p.labels = (const int32_t*)(staged ? labv : zc_lab);
        p.feats = feats;
        p.n = n;
        p.pp = pp;
        p.kp = kp;
        p.nblocks0 = nblocks0;
        p.nvox0 = nvox0;

        SVX_TRY(run_frame(m, pts_f64, feats_f64, s));
        // a frame that ends needing the host leaves the device counters
        // poisoned for queued frames: clear them before the next attempt
        if (hc->abort | hc->err_cap | hc->err_slots) m->ctr_clean = false;
        if (hc->err_internal) {
            m->ctr_clean = false;
            return fail(SVX_E_INTERNAL, "engine invariant failed inside a frame (code " +
                                            std::to_string(hc->err_internal) + ")");
        }

        // the reference's pre-allocation checks, in its order (_core.pyx:661-712, :386-387)
        if (hc->err_budget)
            return fail(SVX_E_INTERNAL, "ray band exceeds step budget; shrink max_range or grow voxels");
        if (hc->rows) {
            bool extent = false, range = false;
            for (int a = 0; a < 3; ++a) {
                if (hc->bbox_max[a] - hc->bbox_min[a] >= (1LL << kPackBits)) extent = true;
                if (llabs(hc->bbox_min[a]) >= kCoordLimit || llabs(hc->bbox_max[a]) >= kCoordLimit)
                    range = true;
            }
            if (extent)
                return fail(SVX_E_INTERNAL,
                            "frame voxel extent exceeds 2^21 per axis; shrink max_range or grow voxels");
            if (range) return fail(SVX_E_RANGE, "voxel coordinate beyond +/-2^30 addressable range");
        }
        if (hc->abort) {
            // stopped by the gate before any mutation: re-based keys (pack),
            // dense rows (slot overflow) or a bigger dense row buffer
            if (hc->err_pack)
                for (int a = 0; a < 3; ++a) kp.base[a] = hc->bbox_min[a];
            if (hc->err_rows) {
                m->maxrows = 0;
                m->rcap = std::max<uint64_t>(m->rcap, hc->rows + hc->rows / 2 + 4096);
            }
            if (hc->err_cap) m->rcap = std::max<uint64_t>(2 * m->rcap, hc->rows + hc->rows / 2 + 4096);
            continue;
        }
        if (hc->err_cap) {
            SVX_TRY(recover_capacity(m, nblocks0, s));
            continue;
        }
        if (hc->err_slots) {
            SVX_TRY(recover_slots(m, nblocks0, s));
            continue;
        }
        break;
    }
    float ms = 0.f;
    SVX_CUDA(cudaEventElapsedTime(&ms, m->ev0, m->ev1));
    r.skipped_nonfinite = (int64_t)hc->nonfinite;
    r.skipped_range = (int64_t)hc->range;
    r.skipped_degenerate = (int64_t)hc->degenerate;
    r.skipped_bad_label = (int64_t)hc->bad_label;
    r.points_used = (int64_t)hc->used;
    r.band_hits = (int64_t)hc->band_hits;
    r.kernel_ms = ms;
    finish_frame(m, nblocks0, nvox0, r);
    if (!rerun) m->frames++;
    if (rep) *rep = r;
    if (g_trace_host) {
        const double t_exit = now_us();
        fprintf(stderr, "svx host us: prep %.1f launch %.1f wait %.1f finish %.1f total %.1f device %.1f\n",
                g_t_launch0 - t_enter, g_t_launch1 - g_t_launch0, g_t_synced - g_t_launch1,
                t_exit - g_t_synced, t_exit - t_enter, 1e3 * ms);
    }
    return SVX_OK;
}

// ---- asynchronous frames ---------------------------------------------------
//
// svx_integrate_async enqueues a frame and returns a ticket; the report is
// read later (svx_report_wait) and every other entry point first finishes
// the frames in flight (drain).  A frame goes asynchronous only when nothing
// it can meet needs the host before it mutates the map:
//   - the reference's frame errors cannot occur: with a finite max_range
//     every band lies within max_range + truncation of the sensor, so the
//     step budget, the 2^21 extent / key window and the +/-2^30 range checks
//     (_core.pyx:661-712, :386-387) are decided by the configuration and the
//     origin alone;
//   - bounded bands (no space carving): at most maxrows rows per point, so
//     the row buffers are sized for the worst case;
//   - closed-set or geometry payloads (open-set frames take milliseconds,
//     where one host round trip does not matter).
// What remains data-dependent -- a pool or slot overflow -- stops the frame
// on the device before any payload change (as for synchronous frames), and
// the frames queued behind it find the device counters poisoned and do
// nothing but keep their own copy of their inputs.  When the host finishes
// the failed frame it recovers as the synchronous path does and re-runs it,
// then the frames behind it, from those copies.

static bool async_eligible(const svx_map* m, int64_t n, const PoseParams& pp) {
    const svx_config& c = m->cfg;
    if (m->async_depth < 1 || m->prof || g_no_graph || n <= 0 || n >= (int64_t)INT_MAX) return false;
    if (c.sem_kind == SVX_SEM_OPEN || c.space_carving) return false;
    const double h = c.voxel_size;
    const double bound = 3.0 * (2.0 * c.truncation / h + 1.0) + 3.0;
    if (bound > 32.0) return false;   // dense rows (init_row_space)
    const double reach = (c.max_range + c.truncation) / h + 4.0;   // voxels from the sensor
    if (!std::isfinite(reach) || reach >= (double)(1LL << (kPackBits - 1))) return false;
    for (int a = 0; a < 3; ++a) {
        const double o = pp.t[a] / h;
        if (!std::isfinite(o) || fabs(o) + reach >= (double)kCoordLimit) return false;
    }
    return true;
}

static void store_report(svx_map* m, uint64_t ticket, const svx_report& r) {
    const int i = (int)(ticket % kDoneReports);
    m->done_rep[i] = r;
    m->done_tag[i] = ticket;
}

static svx_status ensure_async_slot(svx_map* m, AsyncFrame& f) {
    if (f.h) return SVX_OK;
    if (cudaHostAlloc((void**)&f.h, sizeof(FrameCtr), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer((void**)&f.d, f.h, 0) != cudaSuccess ||
        cudaEventCreate(&f.e0) != cudaSuccess || cudaEventCreate(&f.e1) != cudaSuccess ||
        cudaEventCreateWithFlags(&f.ecopy, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        return fail(SVX_E_CUDA, "asynchronous frame slot allocation failed");
    }
    memset(f.h, 0, sizeof(FrameCtr));
    return SVX_OK;
}

void release_async(svx_map* m) {
    for (AsyncFrame& f : m->aq) {
        if (f.h) cudaFreeHost(f.h);
        if (f.e0) cudaEventDestroy(f.e0);
        if (f.e1) cudaEventDestroy(f.e1);
        if (f.ecopy) cudaEventDestroy(f.ecopy);
        release(f.pts);
        release(f.lab);
        f = AsyncFrame();
    }
    if (m->cstream) cudaStreamDestroy(m->cstream);
    m->cstream = nullptr;
}

// Re-run asynchronous frame f synchronously from its own input copy.
static svx_status rerun_async(svx_map* m, const AsyncFrame& f, const FrameOpts& o, svx_report* r) {
    return integrate_impl(m, f.pts.p, f.pts_f64, f.n, f.pp,
                          m->cfg.sem_kind == SVX_SEM_CLOSED ? ptr<int32_t>(f.lab) : nullptr,
                          nullptr, 0, f.stream, r, 1, &o);
}

// Finish the oldest frame in flight: wait for it and take its report, or --
// when it stopped needing the host -- recover and re-run it and every frame
// queued behind it (those did nothing; see above).
static svx_status finalize_oldest(svx_map* m) {
    AsyncFrame& f = m->aq[m->aq_head];
    SVX_CUDA(cudaEventSynchronize(f.e1));
    FrameCtr* hc = f.h;
    if (hc->err_internal) {
        m->ctr_clean = false;
        return fail(SVX_E_INTERNAL, "engine invariant failed inside a frame (code " +
                                        std::to_string(hc->err_internal) + ")");
    }
    if (!(hc->abort | hc->err_cap | hc->err_slots)) {
        svx_report r;
        memset(&r, 0, sizeof(r));
        float ms = 0.f;
        SVX_CUDA(cudaEventElapsedTime(&ms, f.e0, f.e1));
        r.points_in = f.n;
        r.skipped_nonfinite = (int64_t)hc->nonfinite;
        r.skipped_range = (int64_t)hc->range;
        r.skipped_degenerate = (int64_t)hc->degenerate;
        r.skipped_bad_label = (int64_t)hc->bad_label;
        r.points_used = (int64_t)hc->used;
        r.band_hits = (int64_t)hc->band_hits;
        r.kernel_ms = ms;
        m->h_ctr = hc;
        m->frame_slots = f.slots;
        m->frame_leaf = f.leaf;
        finish_frame(m, hc->p.nblocks0, hc->p.nvox0, r);
        m->h_ctr = m->h_ctr0;
        store_report(m, f.ticket, r);
        m->aq_head = (m->aq_head + 1) % kAsyncSlots;
        m->aq_count--;
        return SVX_OK;
    }
    // recovery: everything queued behind f is a no-op; let it finish
    const int last = (m->aq_head + m->aq_count - 1) % kAsyncSlots;
    SVX_CUDA(cudaEventSynchronize(m->aq[last].e1));
    const int64_t nblocks0 = hc->p.nblocks0, nvox0 = hc->p.nvox0;
    cudaStream_t s = f.stream;
    m->h_ctr = hc;
    m->d_hctr = f.d;
    m->frame_slots = f.slots;
    m->frame_leaf = f.leaf;
    FrameOpts o;
    o.stamp = f.frame;
    o.nblocks0 = nblocks0;
    o.nvox0 = nvox0;
    svx_status st = SVX_OK;
    if (hc->abort) {   // gate abort: nothing changed (the row buffer only; cannot recur)
        if (hc->err_cap) m->rcap = std::max<uint64_t>(2 * m->rcap, hc->rows + hc->rows / 2 + 4096);
    } else if (hc->err_cap) {
        st = recover_capacity(m, nblocks0, s);
    } else {
        st = recover_slots(m, nblocks0, s);
        o.force_segments = 1;
    }
    m->ctr_clean = false;   // clears the poison
    m->n_async_reruns++;
    m->h_ctr = m->h_ctr0;
    m->d_hctr = m->d_hctr0;
    // re-run f, then the frames behind it, in order (the ring empties even on error)
    const int cnt = m->aq_count;
    const int head = m->aq_head;
    m->aq_count = 0;
    m->aq_head = (head + cnt) % kAsyncSlots;
    for (int i = 0; i < cnt && st == SVX_OK; ++i) {
        const AsyncFrame& g = m->aq[(head + i) % kAsyncSlots];
        FrameOpts go;
        go.stamp = g.frame;
        svx_report r;
        st = rerun_async(m, g, i == 0 ? o : go, &r);
        if (st == SVX_OK) store_report(m, g.ticket, r);
    }
    return st;
}

svx_status drain(svx_map* m) {
    while (m->aq_count > 0) SVX_TRY(finalize_oldest(m));
    return SVX_OK;
}

svx_status report_wait(svx_map* m, uint64_t ticket, svx_report* out) {
    if (ticket == 0 || ticket >= m->ticket_next) return fail(SVX_E_INPUT, "unknown frame ticket");
    while (m->aq_count > 0 && m->aq[m->aq_head].ticket <= ticket) SVX_TRY(finalize_oldest(m));
    const int i = (int)(ticket % kDoneReports);
    if (m->done_tag[i] != ticket) return fail(SVX_E_INPUT, "frame report no longer held (read it sooner)");
    if (out) *out = m->done_rep[i];
    return SVX_OK;
}

svx_status integrate_async_impl(svx_map* m, const void* pts_in, int pts_f64, int64_t n,
                                const PoseParams& pp, const int32_t* labels_in, cudaStream_t s,
                                int device_inputs, uint64_t* ticket) {
    const int kind = m->cfg.sem_kind;
    if (kind == SVX_SEM_CLOSED && !labels_in && n > 0)
        return fail(SVX_E_PAYLOAD, "closed-set grid requires per-point labels");
    if (!async_eligible(m, n, pp)) {   // synchronous frame, report kept the same way
        SVX_TRY(drain(m));
        svx_report r;
        SVX_TRY(integrate_impl(m, pts_in, pts_f64, n, pp, labels_in, nullptr, 0, s, &r, device_inputs));
        const uint64_t t = m->ticket_next++;
        store_report(m, t, r);
        *ticket = t;
        return SVX_OK;
    }
    const double ta0 = g_trace_host ? now_us() : 0.0;
    if (m->aq_count >= std::min(m->async_depth, kAsyncSlots)) SVX_TRY(finalize_oldest(m));
    const double ta1 = g_trace_host ? now_us() : 0.0;
    init_row_space(m, n);
    // worst-case rows (finish_frame may have lowered rcap to 1.5x the last
    // frame's rows: asynchronous frames always take the bound), and pool
    // headroom for every frame in flight; growing anything first finishes
    // the frames in flight
    const uint64_t rows_bound = (uint64_t)n * (uint64_t)m->maxrows + 4096;
    // voxel headroom per frame in flight: every row could open a voxel, but
    // sizing the pools for n * maxrows new voxels per frame costs gigabytes on
    // large frames; like the synchronous path, take 1.5x the last frame's rows
    // and let the rare overflow stop the frame and be re-run (recovery above)
    const int64_t vneed_per = m->last_rows > 0
                                  ? std::min<int64_t>((int64_t)rows_bound, m->last_rows + m->last_rows / 2 + 65536)
                                  : (int64_t)rows_bound;
    const int64_t bneed_per = m->async_leaf_headroom > 0 ? m->async_leaf_headroom
                                                         : std::max<int64_t>(m->new_leaves_cap, 4096);
    const int depth = std::min(m->async_depth, kAsyncSlots);
    const int q = m->aq_count + 1;
    const bool grow = n > m->npts_cap || rows_bound > m->rcap_sized ||
                      m->nvox + q * vneed_per > m->vcap || m->nblocks + q * bneed_per > m->bcap;
    if (grow) {
        SVX_TRY(drain(m));
        m->rcap = std::max<uint64_t>(m->rcap, rows_bound);
        SVX_TRY(reserve_frame(m, n, s));
        SVX_TRY(reserve_voxels(m, m->nvox + depth * vneed_per, s));
        SVX_TRY(reserve_blocks(m, m->nblocks + depth * bneed_per, s));
    }
    m->rcap = m->rcap_sized;   // the row space the scratch buffers were sized for (>= the bound)
    const int slot = (m->aq_head + m->aq_count) % kAsyncSlots;
    AsyncFrame& f = m->aq[slot];
    SVX_TRY(ensure_async_slot(m, f));
    const size_t pbytes = (size_t)n * 3 * (pts_f64 ? 8 : 4);
    SVX_TRY(ensure(f.pts, pbytes, s));
    if (kind == SVX_SEM_CLOSED) SVX_TRY(ensure(f.lab, (size_t)n * 4, s));
    const bool dev = device_inputs || is_device_ptr(pts_in);
    const void* pts = pts_in;
    const int32_t* lab = kind == SVX_SEM_CLOSED ? labels_in : nullptr;
    if (!dev) {
        // host inputs: copied into the frame's own buffers on the copy stream
        // (overlapping the frames in flight); on return the caller's arrays
        // have been read
        if (!m->cstream) SVX_CUDA(cudaStreamCreateWithFlags(&m->cstream, cudaStreamNonBlocking));
        SVX_CUDA(cudaMemcpyAsync(f.pts.p, pts_in, pbytes, cudaMemcpyHostToDevice, m->cstream));
        if (lab) SVX_CUDA(cudaMemcpyAsync(f.lab.p, lab, (size_t)n * 4, cudaMemcpyHostToDevice, m->cstream));
        SVX_CUDA(cudaEventRecord(f.ecopy, m->cstream));
        SVX_CUDA(cudaStreamWaitEvent(s, f.ecopy, 0));
        pts = f.pts.p;
        lab = lab ? ptr<int32_t>(f.lab) : nullptr;
    }
    m->h_ctr = f.h;
    m->d_hctr = f.d;
    m->frame_retry_segments = 0;
    choose_mode(m, n);
    reset_ctr(m, m->frames);
    FrameParams& p = f.h->p;
    p.pts = pts;
    p.labels = lab;
    p.feats = nullptr;
    p.n = n;
    p.pp = pp;
    p.kp = default_key_pack(m, pp);
    p.nblocks0 = -1;   // taken on the device at the frame's start
    p.nvox0 = -1;
    p.stage_pts = dev ? f.pts.p : nullptr;
    p.stage_lab = dev && kind == SVX_SEM_CLOSED ? ptr<int32_t>(f.lab) : nullptr;
    f.ticket = m->ticket_next;
    f.frame = m->frames;
    f.n = n;
    f.pts_f64 = pts_f64;
    f.slots = m->frame_slots;
    f.leaf = m->frame_leaf;
    f.pp = pp;
    f.stream = s;
    svx_status st = SVX_OK;
    if (cudaEventRecord(f.e0, s) != cudaSuccess) st = fail(SVX_E_CUDA, "event record failed");
    if (st == SVX_OK) st = launch_frame(m, pts_f64, 0, s, f.e1);
    m->h_ctr = m->h_ctr0;
    m->d_hctr = m->d_hctr0;
    if (st != SVX_OK) return st;
    if (!dev) SVX_CUDA(cudaEventSynchronize(f.ecopy));
    m->io_h2d = dev ? 0 : (int64_t)pbytes + (kind == SVX_SEM_CLOSED ? n * 4 : 0);
    m->io_d2h = (int64_t)sizeof(FrameCtr);
    m->aq_count++;
    m->frames++;
    *ticket = m->ticket_next++;
    if (g_trace_host) {
        const double ta2 = now_us();
        fprintf(stderr, "svx async us: finalize %.1f grow %d launch %.1f total %.1f in flight %d\n", ta1 - ta0,
                grow ? 1 : 0, ta2 - ta1, ta2 - ta0, m->aq_count);
    }
    return SVX_OK;
}

}  // namespace svx

// svx_internal.cuh -- shared definitions of the B200 integration engine.
//
// HBM layout:
//   leaf hash    int4[hcap]          {lx, ly, lz, id}; id = EMPTY / BUSY / leaf id
//   leaf pool    int4  bcoord[bcap]  leaf coords (voxel >> 3), w = creation frame
//                u64   bkey[bcap]    creation stamp: min frame-key of its voxels in
//                                    the creating frame (first-occurrence order)
//                u64   bmask[bcap*8] 512-bit active mask (GridCore.leaf_mask, _core.pyx:92)
//                i32   bslot[bcap*512] slot -> voxel id (-1 = inactive)
//   voxel pool   d[vcap], w[vcap]    TSDF (f64 reference layout or f32 compact)
//                sem0[vcap*C|D]      closed counts or open mean m
//                sem1[vcap*D]        open scale beta
//   frame hash   u64 fkey[fcap], u32 fcount/foff/fcur[fcap]  per-frame voxel groups
// Voxel ids are dense and never recycled, so a voxel's payload row is
// contiguous (the NanoVDB index-grid idea) and open-set means form a dense
// (V, D) matrix for query scoring.
#pragma once

#include <cuda_runtime.h>
#include <limits.h>
#include <stddef.h>
#include <stdint.h>

#include <string>

#include "../../include/svx.h"

namespace svx {

constexpr int kLeafLog2 = 3;                 // TreeConfig.leaf_log2 default (config.py:26)
constexpr int kLeafVolume = 512;             // 8^3
constexpr int kMaskWords = 8;                // 512 bits
constexpr int64_t kCoordLimit = int64_t(1) << 30;   // coords.py:41 COORD_LIMIT
constexpr int kPackBits = 21;                       // _core.pyx:34 PACK_BITS
constexpr long long kPackMask = (1LL << kPackBits) - 1;
constexpr int64_t kStepBudget = int64_t(1) << 20;   // _core.pyx:35 STEP_BUDGET
constexpr unsigned long long kKeyEmpty = ~0ULL;

constexpr int kHashEmpty = -1;
constexpr int kHashBusy = -2;

constexpr int kShortMax = 16;   // segments up to this many rows: thread-per-voxel update
// Slot mode (LiDAR-like frames, few rows per voxel): K2 writes each row's point
// index straight into its voxel's slot record (kSlots ints, one 64-byte line)
// and one thread per touched voxel finishes it -- no segment scan, no scatter.
// A voxel with more rows stops the attempt before any payload changes; the
// frame re-runs in segment mode.
constexpr int kSlots = 16;
// 1: slot-mode voxels of 9..16 rows sorted in-thread by the slot update;
// 0 (measured faster): a warp per such voxel in k_update_slots_long.
#ifndef SVX_INLINE_LONG
#define SVX_INLINE_LONG 0
#endif
// RowSlot spacing in vslot (2 = one 32-byte sector per row; measured: no gain).
constexpr int kSlotStride = 1;

struct PoseParams {
    double R[9];
    double t[3];
    int sensor;      // 1: transform points by (R, t); 0: points already world, origin = t
    int single;      // the frame has exactly one point (see world_point)
};

// Frame.points_world (fusion.py:98-100) = points @ R.T + t, evaluated the way
// the reference's numpy/OpenBLAS does it, so rotated poses reproduce bit for
// bit: a frame of n >= 2 points goes through dgemm, whose microkernel
// accumulates k = 0, 1, 2 with fused multiply-adds from the k = 0 product;
// a one-point frame goes through the vector-matrix path, which starts from
// the k = 1 product, then fuses k = 0 and k = 2 (both measured against
// numpy in the build container, tests/golden/make_golden.py rotated).
__host__ __device__ inline double world_coord(const double* Rrow, double t, double x, double y,
                                              double z, int single) {
    const double acc = single ? fma(Rrow[0], x, Rrow[1] * y) : fma(Rrow[1], y, Rrow[0] * x);
    return fma(Rrow[2], z, acc) + t;
}

// Frame key: voxel offsets from `base` packed 21 bits per axis, x-major, so
// key order is the reference's lexicographic voxel order (_core.pyx:727-732).
struct KeyPack {
    long long base[3];
};

// Everything that changes from frame to frame lives in device memory, so one
// captured CUDA graph replays every frame.
struct FrameParams {
    const void* pts;
    const int32_t* labels;
    const void* feats;
    long long n;
    PoseParams pp;
    KeyPack kp;
    unsigned long long ucap;   // touched voxels the per-frame lists hold
    unsigned long long rcap;   // rows the dense row arrays / segment buffer hold
    long long hmask;           // leaf hash capacity - 1
    long long nblocks0;        // leaves before this frame (ids >= it are new); < 0: the
                               // first kernel takes it (and nvox0) from the live counters
    long long nvox0;           // voxels before this frame (report only)
    long long bcap;            // leaf pool capacity
    long long vcap;            // voxel pool capacity
    int frame;                 // creation stamp for new leaves
    int maxrows;               // row slots per ray; 0 = dense rows (two-pass walk)
    int inline_singles;        // single-row voxels updated in the scatter (closed/geometry)
    int slots;                 // 1: slot mode (K2 fills vslot; K5 = k_update_slots)
    long long region;          // slot mode: touched entries per K2 CTA (svx::slot_region)
    unsigned long long* kspan; // profiling: per-CTA start/end times (KSpan), else null
    void* mirror;              // graph frames: device address of the mapped host FrameCtr
    int epilogue;              // 1: the frame's last kernel publishes + resets the counters
    unsigned seq;              // launch sequence number (epoch of the segment-scan status)
    // asynchronous frames with device inputs: the walk copies the frame's
    // points / labels here first (the frame's own copy, for a re-run)
    void* stage_pts;
    int32_t* stage_lab;
};

// Kernels with recorded spans in profiling mode (svx_stage_times order).
enum KSpanId { kSpanWalk = 0, kSpanResolve, kSpanSeg, kSpanScatter, kSpanUpdate, kSpanUpdateB, kSpanKernels };
constexpr int kSpanMaxCtas = 4096;   // per-CTA records per kernel and edge

// Per-CTA partial counters of the march, reduced by the gate (no
// same-address atomics on the hot path).
struct MarchPartial {
    unsigned long long nonfinite, range, degenerate, bad_label, used, band_hits, rows;
    long long bbox_min[3], bbox_max[3];
    int errs;      // bit 0 budget, 1 pack, 3 row-slot overflow
    int pad;
};

// Per-frame device counters and flags, copied back once per frame.
struct FrameCtr {
    FrameParams p;
    unsigned long long nonfinite;
    unsigned long long range;
    unsigned long long degenerate;
    unsigned long long bad_label;
    unsigned long long used;
    unsigned long long band_hits;   // rows emitted before the w <= 0 drop
    unsigned long long rows;        // rows kept (w > 0)
    unsigned long long rows_alloc;  // dense row slots handed out by the tile walk
    unsigned walk_done;             // walk CTAs finished (the last one runs the gate)
    unsigned seg_tiles;             // segment-scan tiles claimed
    unsigned long long n_touched;   // unique voxels of the frame (U)
    unsigned long long n_list;      // voxels listed for segment updates
    unsigned long long rows_seg;    // rows placed in segments
    unsigned long long n_long;      // voxels routed to the long-segment update
    unsigned long long n_huge;      // voxels routed to the huge-segment update
    unsigned long long nblocks;     // leaf allocation counter (device copy)
    unsigned long long nvox;        // voxel allocation counter (device copy)
    long long bbox_min[3];          // over kept rows
    long long bbox_max[3];
    int err_budget;                 // a ray exceeded the DDA step budget
    int err_pack;                   // a key offset left the 21-bit field (retry with bbox base)
    int err_cap;                    // a pool / list / row buffer was too small (grow, retry)
    int err_rows;                   // a band exceeded maxrows (retry with dense rows)
    int abort;                      // set by the gate: skip all mutation
    int err_slots;                  // slot mode: a voxel got more than kSlots rows (re-run in segment mode)
    unsigned epi_done;              // CTAs of the last kernel finished (frame_epilogue)
    unsigned pad_;
    unsigned long long work_long;   // K5 long / open: next listed voxel to take (dynamic scheduling)
    unsigned long long work_open;
    unsigned long long work_huge;   // K5h: next huge voxel; K5g: next (voxel, slice) item
    unsigned long long work_items;
    unsigned long long n_leaves;    // leaf mode: listed (touched) leaves
    unsigned long long bin_cursor;  // leaf mode: rows given bins so far
    unsigned long long n_bigleaf;   // leaf mode: leaves for the CTA path
    unsigned long long err_internal;   // an invariant the host relies on failed
    // Persistent (kept by the epilogue's reset, like nblocks / nvox): set when a
    // frame ends needing the host (pool overflow, slot overflow, gate abort).
    // Asynchronous frames queued behind it see it and do nothing but stage
    // their inputs; the host clears it after recovering (clean_ctr).
    unsigned long long poison;
};

// Per-voxel frame record (indexed by voxel id; cnt and cur are zero between
// frames).  One 32-byte sector, so K2's count atomic, the first toucher's key
// and the first slots land in one line, and the update reads it in one go.
//   cnt   rows this frame; bit 31 = voxel allocated this frame
//   seg   base of the voxel's row segment (segment mode)
//   key   the voxel's frame key (written by its first toucher)
//   cur   segment fill cursor (segment mode)
//   wold  open-set voxels: pre-frame TSDF weight (k_open_prep -> k_update_open)
// Slot mode keeps each voxel's rows in vslot[vid * kSlots + j] = RowSlot
// {point, label, d}: the row's distance was computed by the walk, so the
// update reads everything it needs from the slots (rows 0-1 share a sector).
constexpr unsigned kNewBit = 0x80000000u;
struct alignas(32) VoxFrame {
    unsigned cnt;
    unsigned seg;
    unsigned long long key;
    unsigned cur;
    unsigned pad;
    double wold;   // open-set: the pre-frame weight, left by k_open_prep for k_update_open
};
// Slot mode touched entry: the voxel id (bit 31 = created this frame;
// 0xFFFFFFFF = its claim failed) and its bslot index (leaf * 512 + slot).
struct TouchEntry {
    unsigned vid;
    unsigned bidx;
};
// bslot words: low half = voxel id, high half = slot-mode frame row count.
constexpr unsigned long long kSlotInactive = 0x00000000FFFFFFFFULL;   // id -1, count 0
constexpr unsigned long long kSlotClaim = 0x00000000FFFFFFFEULL;      // segment mode claim (-2)
struct alignas(16) RowSlot {
    int point;
    int label;
    double d;
};
static_assert(sizeof(VoxFrame) == 32, "VoxFrame must be one sector");

// Row addressing: slot mode (bounded bands: ray i owns slots [i*maxrows, +rcnt[i]))
// or dense mode (rows packed by a scan; rowray[r] = ray of row r).
struct RowSpace {
    int maxrows;
    const int* rcnt;
    const int* rowray;
    long long total;
};

__device__ __forceinline__ bool row_ray(const RowSpace& rs, long long t, long long& i) {
    if (rs.maxrows > 0) {
        i = t / rs.maxrows;
        return (int)(t - i * rs.maxrows) < rs.rcnt[i];
    }
    i = rs.rowray[t];
    return true;
}

// Growable device buffer.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
};

struct MarchParams {
    double h;        // voxel size
    double trunc;    // truncation
    double max_range;
    int carving;
    int wfn;         // 0 constant_one, 1 linear_dropoff
};

__host__ __device__ inline unsigned long long pack_key(long long dx, long long dy, long long dz) {
    return ((unsigned long long)dx << (2 * kPackBits)) | ((unsigned long long)dy << kPackBits) |
           (unsigned long long)dz;
}

__host__ __device__ inline void unpack_key(unsigned long long key, const KeyPack& kp, long long& x,
                                           long long& y, long long& z) {
    x = (long long)(key >> (2 * kPackBits)) + kp.base[0];
    y = (long long)((key >> kPackBits) & kPackMask) + kp.base[1];
    z = (long long)(key & kPackMask) + kp.base[2];
}

}  // namespace svx

namespace svx {
constexpr int kAsyncSlots = 4;     // most frames in flight (svx_set_async_depth)
constexpr int kDoneReports = 64;   // finished asynchronous reports kept for svx_report_wait
// One asynchronous frame in flight: its counter mirror, events and its own
// copy of its inputs (a frame that must be re-run is re-run from it).
struct AsyncFrame {
    FrameCtr* h = nullptr;        // mapped pinned counter mirror (host address)
    FrameCtr* d = nullptr;        // its device address
    cudaEvent_t e0 = nullptr, e1 = nullptr, ecopy = nullptr;
    DevBuf pts, lab;              // staged inputs
    uint64_t ticket = 0;
    int64_t frame = 0, n = 0;     // creation stamp, points
    int pts_f64 = 0, slots = 0, leaf = 0;   // update mode it was launched in
    PoseParams pp{};
    cudaStream_t stream = nullptr;
};
}  // namespace svx

struct svx_map {
    svx_config cfg;
    int payload_d = 0;     // C (closed) or D (open)
    // persistent state
    svx::DevBuf hash;  int64_t hcap = 0;
    svx::DevBuf bcoord, bkey, bmask, bslot;  int64_t bcap = 0, nblocks = 0;
    svx::DevBuf vt, s0, s1;                  int64_t vcap = 0, nvox = 0;  // vt: {d, w} per voxel
    svx::DevBuf vrec;                        // per-voxel frame records (svx::VoxFrame)
    svx::DevBuf vslot;                       // slot mode: kSlots RowSlots per voxel
    svx::DevBuf lcnt;                        // leaf mode: per leaf {frame rows, bin base}
    svx::DevBuf render_err;                  // renderer's step-budget flag
    svx::DevBuf sc_q, sc_o;                  // tcgen05 scoring scratch (svx_score.cu)
    int score_path = 0;                      // classify: 0 auto, 1 DMMA, 2 tcgen05 (svx_set_score_path)
    int64_t n_slot_frames = 0, n_slot_reruns = 0, n_async_reruns = 0, n_leaf_frames = 0;
    int64_t io_h2d = 0, io_d2h = 0;   // host-link bytes of the last frame (inputs in, report out)
    int mode_pref = 0;      // SVX_UPDATE_AUTO / SEGMENTS / SLOTS
    int slot_hold = 0;      // frames to stay in segment mode after a slot overflow
    int64_t last_rows = 0, last_touched = 0;   // previous frame's rows and touched voxels
    int frame_slots = 0;    // mode of the attempt being run: slots,
    int frame_leaf = 0;     //   leaves, or (both 0) segments
    int frame_retry_segments = 0;   // this frame overflowed its slots: re-run with segments
    int64_t frames = 0;
    unsigned seq = 0;   // frame launches so far (attempts included)
    // asynchronous frames (svx_integrate_async): ring of frames in flight,
    // finished in order; their reports are kept for svx_report_wait
    svx::AsyncFrame aq[svx::kAsyncSlots];
    int aq_head = 0, aq_count = 0;
    int async_depth = 2;
    int64_t async_leaf_headroom = 0;   // leaves kept free per frame in flight (0 = automatic)
    uint64_t ticket_next = 1;
    svx_report done_rep[svx::kDoneReports] = {};
    uint64_t done_tag[svx::kDoneReports] = {};
    cudaStream_t cstream = nullptr;   // host-input copies of asynchronous frames
    // per-frame scratch
    svx::DevBuf in_pts, in_lab, in_feat;
    svx::DevBuf dp_depth, dp_lab_in, dp_feat_in, dp_pts, dp_lab, dp_feat;   // depth frames
    svx::DevBuf ray, rcnt, roff, rowkey, rowvid, rowray, rowd, rowlab, partials;
    svx::DevBuf rowleaf, rowpk, binrow;      // leaf mode rows
    svx::DevBuf tlist, mlist, longlist, srid, bitmap, rcount, hinfo;
    uint64_t ucap = 0, rcap = 0;
    uint64_t rcap_sized = 0;      // rcap the frame scratch was last sized for (reserve_frame)
    int64_t new_leaves_cap = 0;   // leaf-pool headroom kept for one frame
    int maxrows = -1;      // row slots per ray; 0 = dense rows
    int64_t npts_cap = 0;  // points the per-ray scratch holds
    // captured frame graph (replayed while the layout is unchanged)
    cudaStream_t gstream = nullptr;
    // per mode (segments, slots, leaves) one captured graph and one executable
    // instance; updating the instance's first-kernel parameters does not touch
    // launches already queued, so frames in flight share it
    cudaGraphExec_t gexec[3][1] = {};
    int exec_slot = 0;
    cudaGraph_t graph[3] = {};       // kept: its first-kernel node is updated per frame
    cudaGraphNode_t walk_node[3] = {};
    int walk_nargs[3] = {};          // parameters of that kernel (FrameParams is the last)
    cudaKernelNodeParams walk_kp[3] = {};   // its captured launch parameters
    void* walk_args[3][16] = {};            // its argument pointers (graph-owned storage)
    int first_nargs = 0;             // set by launch_march for the kernel it launched first
    unsigned long long gsig[3] = {};
    int graph_kernels[3] = {0, 0, 0};   // kernel nodes of each frame graph (launch accounting)
    svx::DevBuf cubtmp;
    svx::DevBuf ctr;      // FrameCtr
    svx::FrameCtr* h_ctr = nullptr;  // pinned, mapped mirror of the frame being run (host side)
    svx::FrameCtr* d_hctr = nullptr; // its device address
    svx::FrameCtr last_ctr{};        // counters of the last finished frame (diagnostics)
    svx::FrameCtr* h_ctr0 = nullptr; // the mirror of synchronous frames (h_ctr points at it,
    svx::FrameCtr* d_hctr0 = nullptr;//   or at an asynchronous frame's own mirror)
    bool ctr_clean = false;          // device FrameCtr is in the reset state
    // query scratch
    svx::DevBuf ord0, ord1, ordk0, ordk1, ordf0, ordf1;  // leaf order (by creation stamp)
    int64_t ord_nblocks = -1;
    int* leaf_order = nullptr;
    svx::DevBuf act_cnt, act_off, act_vid, act_coord, q_buf, out_buf;
    // surface extraction (svx_mesh.cu)
    svx::DevBuf mesh_ctr, mesh_k0, mesh_k1, mesh_i0, mesh_i1, mesh_rec, mesh_meta, mesh_vmask,
        mesh_cnt, mesh_off, mesh_toff, mesh_vk, mesh_vv, mesh_vidx, mesh_v, mesh_l, mesh_t, mesh_col,
        mesh_vlab, mesh_cls_l, mesh_cls_b, mesh_pal;
    int64_t mesh_nv = 0, mesh_nt = 0;
    int64_t act_valid_frames = -1;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev_in = nullptr;
    // optional per-kernel timing (svx_set_profiling; FrameCtr.kspan)
    bool prof = false;
    double stage_ms[SVX_N_STAGES] = {};
    svx::DevBuf kspan;                       // kSpanKernels x 2 x kSpanMaxCtas u64
    unsigned long long* h_kspan = nullptr;   // host copy
    // sharded integration (svx_shard.cu): state between a frame's calls
    int shard_phase = 0;          // 0 idle, 1 marched, 2 planned, 3 packed
    int shard_g = 1, shard_rank = 0;
    int64_t shard_n = 0;          // points in this rank's slice
    int64_t shard_rows = 0;       // rows this rank marched
    int shard_pts_f64 = 0, shard_feats_f64 = 0;
    const void* shard_lab = nullptr;    // the slice's staged payload
    const void* shard_feat = nullptr;
    svx::PoseParams shard_pp{};
    svx::KeyPack shard_kp{};
    svx_shard_summary shard_sum{};      // the frame's global summary
    svx::DevBuf sh_mask, sh_pos, sh_tiles, sh_meta;
    int64_t sh_npts[SVX_MAX_SHARDS] = {}, sh_nrows[SVX_MAX_SHARDS] = {};
    int64_t sh_bytes[SVX_MAX_SHARDS] = {};
    // device-planned frames (svx_shard_*_async)
    int shard_async = 0;
    int64_t sh_cap = 0;
    int64_t sh_nblocks0 = 0, sh_nvox0 = 0;
    int64_t sh_last_rows = 0;           // rows of the last frame (global march / local apply, larger)
    svx::DevBuf sh_ao;                  // ApplyOffsets + local flags
    long long* sh_hlocal = nullptr;     // pinned copy of the local flags
};

namespace svx {

// ---- error plumbing ------------------------------------------------------
void set_error(const std::string& msg);
svx_status fail(svx_status code, const std::string& msg);
void count_launch(int n = 1);

#define SVX_CUDA(expr)                                                                \
    do {                                                                              \
        cudaError_t _e = (expr);                                                      \
        if (_e != cudaSuccess)                                                        \
            return ::svx::fail(SVX_E_CUDA, std::string("CUDA error: ") +              \
                                               cudaGetErrorString(_e) + " at " #expr); \
    } while (0)

#define SVX_TRY(expr)                     \
    do {                                  \
        svx_status _s = (expr);           \
        if (_s != SVX_OK) return _s;      \
    } while (0)

// Programmatic dependent launch: kernels of the frame pipeline are launched
// with programmatic stream serialization, so a kernel's CTAs are scheduled
// while its predecessor drains (hiding the launch gap inside the graph).
// Each such kernel calls grid_dep_wait() before it reads anything; that
// returns once the predecessor grid has completed and its writes are visible.
// The kernel first lets its successor be scheduled (launch_dependents), so
// the successor's launch overlaps this kernel's tail.
__device__ __forceinline__ void grid_dep_wait() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Spin-wait guard: a wait on another CTA's publish that has not finished
// after ~1 s is an engine bug; record which wait (err_internal) and give up
// instead of hanging the GPU.
constexpr int kSpinLimit = 1 << 25;
#define SVX_SPIN_GUARD(count, ctr, code)                                          \
    if (++(count) > ::svx::kSpinLimit) {                                          \
        atomicCAS(&(ctr)->err_internal, 0ULL, (unsigned long long)(code));        \
        break;                                                                    \
    }

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Profiling span of one kernel: construct after grid_dep_wait(); each CTA's
// thread 0 stores its start and (destructor, so early returns are covered)
// its end time into its own record -- plain stores, no contention; the host
// reduces them to [first start, last end].  One branch when profiling is off.
struct KSpan {
    unsigned long long* rec;
    __device__ __forceinline__ KSpan(FrameCtr* ctr, int k) : rec(ctr->p.kspan) { start(k); }
    // first kernel of a frame: parameters from its snapshot
    __device__ __forceinline__ KSpan(const FrameCtr* snap, FrameCtr*, int k) : rec(snap->p.kspan) {
        start(k);
    }
    // end_only: a later kernel of the same stage (its CTAs' end times replace
    // the first kernel's, whose start times stay): the stage spans both
    __device__ __forceinline__ KSpan(FrameCtr* ctr, int k, bool end_only) : rec(ctr->p.kspan) {
        start(k, end_only);
    }
    __device__ __forceinline__ void start(int k, bool end_only = false) {
        if (rec && threadIdx.x == 0 && blockIdx.x < kSpanMaxCtas) {
            rec += (size_t)k * 2 * kSpanMaxCtas + blockIdx.x;
            if (!end_only) rec[0] = globaltimer();
        } else {
            rec = nullptr;
        }
    }
    __device__ __forceinline__ ~KSpan() {
        if (rec) rec[kSpanMaxCtas] = globaltimer();
    }
};

// Per-CTA snapshot of the frame's counters and parameters in shared memory
// (after grid_dep_wait(), by all threads): kernels read them from there
// instead of every thread loading them from global memory.  Only fields that
// are final before the kernel starts may be read from the snapshot.
__device__ __forceinline__ void snapshot_ctr(const FrameCtr* g, FrameCtr& s) {
    static_assert(sizeof(FrameCtr) % 8 == 0, "FrameCtr must be a whole number of words");
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(g);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(&s);
    for (int i = threadIdx.x; i < (int)(sizeof(FrameCtr) / 8); i += blockDim.x) dst[i] = __ldcg(src + i);
    __syncthreads();
}

// First kernel of a frame: counters from the device FrameCtr (reset state),
// parameters from the kernel's own FrameParams argument (updated in the
// instantiated graph before each launch, cudaGraphExecKernelNodeSetParams);
// CTA 0 publishes them to the device FrameCtr for the later kernels.  All
// threads call it.
__device__ __forceinline__ void load_frame_params(FrameCtr* ctr, FrameCtr& s, const FrameParams& fpk) {
    snapshot_ctr(ctr, s);
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(&fpk);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(&s.p);
    static_assert(sizeof(FrameParams) % 8 == 0, "FrameParams must be a whole number of words");
    for (int i = threadIdx.x; i < (int)(sizeof(FrameParams) / 8); i += blockDim.x) dst[i] = src[i];
    __syncthreads();
    if (threadIdx.x == 0 && s.p.nblocks0 < 0) {   // asynchronous frame: pool counts at its start
        s.p.nblocks0 = (long long)s.nblocks;
        s.p.nvox0 = (long long)s.nvox;
    }
    __syncthreads();
    if (blockIdx.x == 0) {
        unsigned long long* g = reinterpret_cast<unsigned long long*>(&ctr->p);
        for (int i = threadIdx.x; i < (int)(sizeof(FrameParams) / 8); i += blockDim.x) g[i] = dst[i];
    }
}

// Graph frames have no copy nodes.  The first kernel gets the frame's
// parameters as its argument (load_frame_params) and publishes them to the
// device FrameCtr; the last kernel's last CTA copies the device
// FrameCtr to the mapped host FrameCtr (the host reads it after the frame's
// event) and resets the device counters for the next frame.  The live pool
// counters (nblocks, nvox) carry over.
__device__ __forceinline__ void reset_ctr_device(FrameCtr* ctr) {
    unsigned long long* w = reinterpret_cast<unsigned long long*>(ctr);
    const int first = (int)(offsetof(FrameCtr, nonfinite) / 8);
    const int total = (int)(sizeof(FrameCtr) / 8);
    const int keep0 = (int)(offsetof(FrameCtr, nblocks) / 8), keep1 = (int)(offsetof(FrameCtr, nvox) / 8);
    const int keep2 = (int)(offsetof(FrameCtr, poison) / 8);
    const int bb0 = (int)(offsetof(FrameCtr, bbox_min) / 8), bb1 = (int)(offsetof(FrameCtr, bbox_max) / 8);
    for (int i = first + (int)threadIdx.x; i < total; i += blockDim.x) {
        if (i == keep0 || i == keep1 || i == keep2) continue;
        unsigned long long v = 0ULL;
        if (i >= bb0 && i < bb0 + 3) v = (unsigned long long)LLONG_MAX;
        if (i >= bb1 && i < bb1 + 3) v = (unsigned long long)LLONG_MIN;
        w[i] = v;
    }
}

// Called by every thread of the frame's last kernel, after its work (no
// early returns before it).  `epi` = FrameParams.epilogue.
__device__ __forceinline__ void frame_epilogue(FrameCtr* ctr, int epi, void* mirror) {
    if (!epi) return;
    __shared__ bool s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&ctr->epi_done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(ctr);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(mirror);
    for (int i = threadIdx.x; i < (int)(sizeof(FrameCtr) / 8); i += blockDim.x) dst[i] = __ldcg(src + i);
    __syncthreads();
    if (threadIdx.x == 0 && (ctr->err_cap | ctr->err_slots | ctr->abort)) ctr->poison = 1ULL;
    reset_ctr_device(ctr);
    __threadfence_system();
}

template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), unsigned grid, unsigned block, size_t smem,
                              cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at{};
    at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

#define SVX_LAUNCHED()                                                                      \
    do {                                                                                    \
        ::svx::count_launch();                                                              \
        cudaError_t _e = cudaGetLastError();                                                \
        if (_e != cudaSuccess)                                                              \
            return ::svx::fail(SVX_E_CUDA, std::string("kernel launch: ") + cudaGetErrorString(_e)); \
    } while (0)

// Ensure `buf` holds at least `bytes`.  keep: preserve old contents (pool
// growth); fill >= 0: memset the grown tail (whole buffer when !keep) to that
// byte value.
svx_status ensure(DevBuf& buf, size_t bytes, cudaStream_t s, bool keep = false, int fill = -1);
void release(DevBuf& buf);

template <class T>
inline T* ptr(const DevBuf& b) { return static_cast<T*>(b.p); }

inline int grid_for(int64_t n, int threads) {
    int64_t g = (n + threads - 1) / threads;
    return (int)(g < 1 ? 1 : g);
}

constexpr int kPersistentBlocks = 148 * 8;   // grid-stride kernels over device-side counts
#ifndef SVX_RESOLVE_TILE
#define SVX_RESOLVE_TILE 256
#endif
constexpr int kResolveTile = SVX_RESOLVE_TILE;   // K2 rows per CTA step
// Slot mode: K2 CTA b lists its touched voxels in tent[b * region, ...); a CTA
// handles at most ceil(tiles / grid) tiles of kResolveTile rows.
inline long long slot_region(unsigned long long rows_cap) {
    const long long tiles = (long long)((rows_cap + kResolveTile - 1) / kResolveTile);
    return ((tiles + kPersistentBlocks - 1) / kPersistentBlocks) * kResolveTile;
}
#ifndef SVX_MARCH_BLOCKS
#define SVX_MARCH_BLOCKS (148 * 4)
#endif
constexpr int kMarchBlocks = SVX_MARCH_BLOCKS;   // march CTAs

// TSDF state of one voxel, {d, w} interleaved so an update touches one sector.
template <class T> struct Pair;
template <> struct Pair<double> { using type = double2; };
template <> struct Pair<float> { using type = float2; };

// ---- hashing -----------------------------------------------------------------
__host__ __device__ inline uint64_t block_hash(int a, int b, int c) {
    uint64_t h = (uint64_t)(uint32_t)a * 0xD6E8FEB86659FD93ULL;
    h += (uint64_t)(uint32_t)b * 0xA0761D6478BD642FULL;
    h ^= h >> 31;
    h += (uint64_t)(uint32_t)c * 0xE7037ED1A0B428DBULL;
    h ^= h >> 29;
    h *= 0x94D049BB133111EBULL;
    h ^= h >> 32;
    return h;
}

__host__ __device__ inline uint64_t key_hash(unsigned long long k) {
    k ^= k >> 33;
    k *= 0xFF51AFD7ED558CCDULL;
    k ^= k >> 33;
    k *= 0xC4CEB9FE1A85EC53ULL;
    k ^= k >> 33;
    return k;
}

// Read-only leaf lookup (no concurrent inserts).  Returns leaf id or -1.
__device__ inline int hash_find(const int4* __restrict__ table, int64_t mask, int a, int b, int c) {
    int64_t pos = (int64_t)(block_hash(a, b, c) & (uint64_t)mask);
    while (true) {
        int4 s = __ldg(table + pos);
        if (s.w == kHashEmpty) return -1;
        if (s.x == a && s.y == b && s.z == c) return s.w;
        pos = (pos + 1) & mask;
    }
}

// ---- svx_frame.cu ------------------------------------------------------------
bool is_device_ptr(const void* p);
svx_status stage_in(const void* p, size_t bytes, DevBuf& stage, cudaStream_t s, const void** out);
size_t tsdf_elem(const svx_map* m);
size_t sem_elem(const svx_map* m);
svx_status reserve_voxels(svx_map* m, int64_t need, cudaStream_t s);
svx_status reserve_blocks(svx_map* m, int64_t need, cudaStream_t s);
// Options of a frame run by integrate_impl for an asynchronous frame being
// re-run: its creation stamp and the pool counts at its first attempt.
struct FrameOpts {
    int64_t stamp = -1;          // < 0: a new frame (m->frames, then counted)
    int64_t nblocks0 = -1, nvox0 = -1;
    int force_segments = 0;
};
svx_status integrate_impl(svx_map* m, const void* pts_in, int pts_f64, int64_t n,
                          const PoseParams& pp, const int32_t* labels_in, const void* feats_in,
                          int feats_f64, cudaStream_t s, svx_report* rep, int device_inputs = 0,
                          const FrameOpts* opt = nullptr);
svx_status integrate_async_impl(svx_map* m, const void* pts_in, int pts_f64, int64_t n,
                                const PoseParams& pp, const int32_t* labels_in, cudaStream_t s,
                                int device_inputs, uint64_t* ticket);
svx_status report_wait(svx_map* m, uint64_t ticket, svx_report* out);
// Finish every asynchronous frame in flight (every other entry point calls
// it first, so the map it reads is the map after all submitted frames).
svx_status drain(svx_map* m);
void release_async(svx_map* m);

// ---- launchers implemented in the .cu files ---------------------------------
// svx_march.cu: K1 walk (+ dense-row scan) and the gate
MarchParams march_params(const svx_map* m);
svx_status launch_march(svx_map* m, int pts_f64, int feats_f64, cudaStream_t s);
size_t partials_bytes();
// svx_resolve.cu: K2 voxel resolution + per-voxel counts, K3 segments
svx_status launch_resolve(svx_map* m, cudaStream_t s);
svx_status launch_segments(svx_map* m, cudaStream_t s);
svx_status launch_cleanup(svx_map* m, cudaStream_t s);   // undo a capacity-aborted attempt
size_t segment_status_bytes(unsigned long long ucap);
size_t scan_temp_bytes(int64_t n);
// Single-row voxels of closed/geometry frames are updated inline by the
// scatter pass; open-set voxels always go through segments.
inline int inline_singles(const svx_map* m) { return m->cfg.sem_kind != SVX_SEM_OPEN; }
// svx_update.cu: K4 scatter (+ single-row updates), K5 segment updates
svx_status launch_scatter(svx_map* m, cudaStream_t s);
svx_status launch_update_a(svx_map* m, int feats_f64, cudaStream_t s);
svx_status launch_update_b(svx_map* m, int feats_f64, cudaStream_t s);
svx_status launch_update_slots(svx_map* m, cudaStream_t s);
// svx_leaf.cu: leaf mode (K2L bin, K3L alloc, K4L scatter, K5L update)
svx_status launch_leaf(svx_map* m, cudaStream_t s);
svx_status launch_leaf_cleanup(svx_map* m, cudaStream_t s);
bool leaf_mode_fits(int64_t n);
svx_status launch_rehash(svx_map* m, int4* new_table, int64_t new_cap, cudaStream_t s);
svx_status launch_fill_u64(unsigned long long* p, int64_t n, unsigned long long v, cudaStream_t s);
int huge_warps();
size_t huge_info_bytes();
int open_cta_min();   // open-set voxels above this many rows take the CTA kernels

// frame driver pieces shared by svx_integrate and the sharded calls (svx_frame.cu)
void init_row_space(svx_map* m, int64_t n);
svx_status reserve_frame(svx_map* m, int64_t n, cudaStream_t s);
svx_status reserve_pools(svx_map* m, cudaStream_t s);
void reset_ctr(svx_map* m, int64_t stamp);
svx_status recover_capacity(svx_map* m, int64_t nblocks0, cudaStream_t s);
svx_status recover_slots(svx_map* m, int64_t nblocks0, cudaStream_t s);
svx_status clean_ctr(svx_map* m, cudaStream_t s);
int choose_slots(const svx_map* m);
void choose_mode(svx_map* m, int64_t n);   // sets frame_slots / frame_leaf
void finish_frame(svx_map* m, int64_t nblocks0, int64_t nvox0, svx_report& r);
KeyPack default_key_pack(const svx_map* m, const PoseParams& pp);

// Owning rank of a leaf in a sharded map: high hash bits, independent of the
// low bits that place the leaf in its owner's hash table.
__host__ __device__ inline int leaf_owner(long long a, long long b, long long c, int g) {
    return (int)((block_hash((int)a, (int)b, (int)c) >> 32) % (uint64_t)g);
}
// svx_query.cu
svx_status build_active_list(svx_map* m, int64_t* count, cudaStream_t s);
svx_status launch_leaf_stamps(svx_map* m, int32_t* frame, uint64_t* key, int32_t* count,
                              cudaStream_t s);

// rendering (svx_render.cu)
svx_status render_impl(svx_map* m, const svx_render_camera& cam, int mode, const int* vlab,
                       const unsigned char* pal, int npal, void* out, cudaStream_t s);
svx_status sample_impl(svx_map* m, int64_t n, const double* pts, double* vals, unsigned char* valid,
                       cudaStream_t s);

// surface extraction (svx_mesh.cu)
svx_status mesh_impl(svx_map* m, double min_weight, const int* vlab, cudaStream_t s);
svx_status mesh_colors(svx_map* m, const unsigned char* pal, int npal, unsigned char* colors,
                       cudaStream_t s);
svx_status scatter_active_labels(svx_map* m, int64_t count, const int* labels, int* vlab,
                                 cudaStream_t s);
svx_status launch_classify(svx_map* m, int64_t count, const double* emb, const double* en, int k,
                           double tau, double tp, int32_t* labels, double* best, double* sims,
                           cudaStream_t s);

// snapshots (svx_import.cu)
svx_status import_impl(svx_map* m, int64_t nl, const int32_t* leaf_coords, int64_t nv,
                       const int32_t* voxel_leaf, const int32_t* voxel_slot, const double* d,
                       const double* w, const void* sem0, const void* sem1, cudaStream_t s);

// depth frames (svx_depth.cu)
svx_status integrate_depth_impl(svx_map* m, const void* depth, int depth_dtype, const svx_camera& cam,
                                const PoseParams& pp, const int32_t* labels, const void* feats,
                                int feats_f64, cudaStream_t s, svx_report* rep);

// sharded integration (svx_shard.cu)
svx_status shard_march(svx_map* m, const void* pts, int pts_f64, int64_t n, const PoseParams& pp,
                       const int32_t* labels, const void* feats, int feats_f64,
                       const int64_t* key_base, cudaStream_t s, svx_shard_summary* out);
svx_status shard_plan(svx_map* m, const svx_shard_summary* global, int rank, int nranks,
                      int64_t* send_bytes, int* remarch, cudaStream_t s);
svx_status shard_pack(svx_map* m, void* send, int64_t capacity, cudaStream_t s);
svx_status shard_apply(svx_map* m, const void* recv, const int64_t* recv_bytes, int nranks,
                       cudaStream_t s, svx_report* rep);
svx_status shard_march_async(svx_map* m, const void* pts, int pts_f64, int64_t n, const PoseParams& pp,
                             const int32_t* labels, const void* feats, int feats_f64,
                             const int64_t* key_base, cudaStream_t s, int64_t* summary);
svx_status shard_plan_async(svx_map* m, const int64_t* gsum, int rank, int G, int64_t cap, cudaStream_t s,
                            int64_t* abort);
svx_status shard_pack_async(svx_map* m, void* send, int64_t cap, cudaStream_t s, const int64_t* abort);
svx_status shard_apply_async(svx_map* m, const void* recv, int64_t cap, int G, const int64_t* abort,
                             int64_t frame_points, cudaStream_t s, int64_t* rep_words);
svx_status shard_finish(svx_map* m, const int64_t* g, const int64_t* abort, const int64_t* rsum,
                        svx_report* rep, int32_t* action, int64_t* need);
svx_status launch_export(svx_map* m, int64_t count, int64_t* coords, void* d, void* w, void* sem0,
                         void* sem1, cudaStream_t s);
svx_status launch_probe(svx_map* m, const int64_t* coords, int64_t cnt, void* d, void* w,
                        void* sem0, void* sem1, uint8_t* active, cudaStream_t s);
svx_status launch_cosine(svx_map* m, int64_t count, const double* q, double qn, double* sims,
                         cudaStream_t s);
svx_status launch_classify(svx_map* m, int64_t count, const double* emb, const double* en, int k,
                           double tau, double tp, int32_t* labels, double* best, double* sims,
                           cudaStream_t s);
svx_status launch_label_map(svx_map* m, int64_t count, int mode, int32_t* labels, cudaStream_t s);
// svx_score.cu: classify_means scores as an int8 split GEMM on tcgen05
svx_status classify_tc(svx_map* m, int64_t count, const int* act_vid, const double* emb, const double* en,
                       int k, double tau, double tp, int32_t* labels, double* best, double* sims,
                       cudaStream_t s);

}  // namespace svx

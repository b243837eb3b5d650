// svx_shard.cu -- integration of a map sharded over G ranks by leaf
// ownership (the reference is single-process, so this has no
// reference counterpart beyond the per-frame semantics it preserves).
//
// Per frame and rank (include/svx.h describes the calls):
//   march  K1 on this rank's contiguous slice of the frame's points (the
//          same walk and gate counters as svx_integrate); the host reduces
//          the summaries across ranks and applies the reference's frame
//          checks to the global one, so a bad frame fails on every rank
//          before any rank mutates its shard.
//   plan   rows -> owning rank of their leaf (leaf_owner); per point a bit
//          mask of the ranks its rows go to; per owner the point and row
//          counts and the byte size of its section of the send buffer.
//   pack   per owner section: header, the points (ray u + t_surf as one
//          double4, then the label or feature vector) in increasing point
//          order, then the rows (packed key, index into the section's
//          points).
//   apply  sections received from every rank are concatenated in rank
//          order, which keeps the frame's global point order; the rows then
//          go through K2-K5 exactly as in svx_integrate.  Every voxel's rows
//          land on one rank and are reduced in (voxel, point) order, so the
//          union of the shards is the single-GPU map bit for bit.
//
// Exchange volume per frame: 12 B per row plus (32 + payload) B per point
// and owner it has rows at -- a ray crosses few leaves, so a point is sent
// once or twice, never once per row.
#include <cub/block/block_scan.cuh>
#include <limits.h>
#include <string.h>

#include <algorithm>

#include "svx_internal.cuh"

namespace svx {
namespace {

constexpr int kPlanThreads = 256;

struct SectionHeader {
    unsigned npts, nrows, pay, magic;
};
constexpr unsigned kSectionMagic = 0x53565853u;   // "SXVS"

struct SectionLayout {
    long long rays, pay, keys, pts, size;
};

__host__ __device__ inline long long align16(long long b) { return (b + 15) & ~15LL; }

// Byte offsets inside one owner's section.
__host__ __device__ inline SectionLayout section_layout(long long npts, long long nrows,
                                                        long long pay) {
    SectionLayout L;
    L.rays = (long long)sizeof(SectionHeader);
    L.pay = L.rays + align16(npts * (long long)sizeof(double4));
    L.keys = L.pay + align16(npts * pay);
    L.pts = L.keys + align16(nrows * 8);
    L.size = L.pts + align16(nrows * 4);
    return L;
}

// Device-side plan: per owner point/row counts, section sizes, offsets and
// the row cursors of the pack.
struct ShardMeta {
    long long npts[SVX_MAX_SHARDS];
    long long nrows[SVX_MAX_SHARDS];
    long long size[SVX_MAX_SHARDS];
    long long off[SVX_MAX_SHARDS];
    unsigned long long cursor[SVX_MAX_SHARDS];
};

// Rows -> owning rank (kept in rowvid, unused until apply); the point's
// owner mask; per-owner row counts (one atomic per CTA and owner).
// Frame-level abort of a device-planned frame (svx_shard_*_async): any of the
// global checks, or (for the local pack) a section over its capacity.
__device__ __forceinline__ bool shard_aborted(const long long* abort, bool local) {
    if (!abort) return false;
    bool a = false;
    for (int i = 0; i < 5; ++i) a |= abort[i] != 0;
    return a || (local && abort[5] != 0);
}

__global__ void __launch_bounds__(kPlanThreads) k_shard_rows(
    long long R, int G, KeyPack kp, const unsigned long long* __restrict__ rowkey,
    const int* __restrict__ rowray, int* __restrict__ rowown, unsigned* __restrict__ ptmask,
    ShardMeta* meta, const FrameCtr* ctr, const long long* abort) {
    if (R < 0) R = (long long)ctr->rows;   // device-planned frames: the march's count
    if (shard_aborted(abort, false)) return;
    __shared__ unsigned s_cnt[SVX_MAX_SHARDS];
    if (threadIdx.x < SVX_MAX_SHARDS) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < R;
         t += (long long)gridDim.x * blockDim.x) {
        long long x, y, z;
        unpack_key(rowkey[t], kp, x, y, z);
        const int o = leaf_owner(x >> kLeafLog2, y >> kLeafLog2, z >> kLeafLog2, G);
        rowown[t] = o;
        atomicOr(&ptmask[rowray[t]], 1u << o);
        atomicAdd(&s_cnt[o], 1u);
    }
    __syncthreads();
    if (threadIdx.x < G && s_cnt[threadIdx.x])
        atomicAdd((unsigned long long*)&meta->nrows[threadIdx.x], (unsigned long long)s_cnt[threadIdx.x]);
}

// Per 256-point tile and owner: how many of the tile's points go there.
__global__ void __launch_bounds__(kPlanThreads) k_shard_tiles(long long n, int G,
                                                              const unsigned* __restrict__ ptmask,
                                                              long long* __restrict__ tiles) {
    __shared__ unsigned s_cnt[SVX_MAX_SHARDS];
    if (threadIdx.x < SVX_MAX_SHARDS) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    const long long i = (long long)blockIdx.x * kPlanThreads + threadIdx.x;
    unsigned mk = i < n ? ptmask[i] : 0u;
    while (mk) {
        const int o = __ffs(mk) - 1;
        mk &= mk - 1;
        atomicAdd(&s_cnt[o], 1u);
    }
    __syncthreads();
    if (threadIdx.x < G) tiles[(long long)blockIdx.x * G + threadIdx.x] = s_cnt[threadIdx.x];
}

// One warp: per owner, exclusive scan of the tile counts (in place), then
// section sizes and offsets in rank order.
__global__ void k_shard_plan(long long ntiles, int G, long long pay, long long* __restrict__ tiles,
                             ShardMeta* meta, long long cap, long long* abort) {
    const int o = threadIdx.x;
    if (o < G) {
        long long acc = 0;
        for (long long t = 0; t < ntiles; ++t) {
            const long long c = tiles[t * G + o];
            tiles[t * G + o] = acc;
            acc += c;
        }
        meta->npts[o] = acc;
        meta->cursor[o] = 0;
    }
    __syncwarp();
    if (o == 0) {
        long long off = 0, big = 0;
        for (int q = 0; q < G; ++q) {
            const SectionLayout L = section_layout(meta->npts[q], meta->nrows[q], pay);
            meta->size[q] = L.size;
            meta->off[q] = cap > 0 ? q * cap : off;   // fixed-capacity sections (device-planned frames)
            off += L.size;
            big = L.size > big ? L.size : big;
        }
        if (cap > 0 && abort) {
            abort[6] = big;                  // the capacity this frame needs
            if (big > cap) abort[5] = 1;     // pack skips; the frame is redone with a larger capacity
        }
    }
}

// Points -> every owner section they have rows in, in increasing point
// order (block scan per owner on top of the tile bases); labels ride along.
__global__ void __launch_bounds__(kPlanThreads) k_shard_pack_points(
    long long n, int G, const unsigned* __restrict__ ptmask, const long long* __restrict__ tiles,
    const double4* __restrict__ ray, const int32_t* __restrict__ labels, int* __restrict__ ptpos,
    const ShardMeta* __restrict__ meta, char* __restrict__ send, long long pay, const long long* abort) {
    if (shard_aborted(abort, true)) return;
    using Scan = cub::BlockScan<int, kPlanThreads>;
    __shared__ typename Scan::TempStorage tmp;
    const long long i = (long long)blockIdx.x * kPlanThreads + threadIdx.x;
    const unsigned mk = i < n ? ptmask[i] : 0u;
    for (int o = 0; o < G; ++o) {
        const int flag = (mk >> o) & 1u;
        int local, total;
        Scan(tmp).ExclusiveSum(flag, local, total);
        __syncthreads();
        if (!flag) continue;
        const long long pos = tiles[(long long)blockIdx.x * G + o] + local;
        ptpos[(long long)o * n + i] = (int)pos;
        const SectionLayout L = section_layout(meta->npts[o], meta->nrows[o], pay);
        char* sec = send + meta->off[o];
        reinterpret_cast<double4*>(sec + L.rays)[pos] = ray[i];
        if (labels) reinterpret_cast<int32_t*>(sec + L.pay)[pos] = labels[i];
    }
}

// Feature vectors (open-set payload): one warp per point, 16-byte words.
__global__ void k_shard_pack_feats(long long n, int G, const unsigned* __restrict__ ptmask,
                                   const int* __restrict__ ptpos, const char* __restrict__ feats,
                                   const ShardMeta* __restrict__ meta, char* __restrict__ send,
                                   long long pay, const long long* abort) {
    if (shard_aborted(abort, true)) return;
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    const long long words = pay / 4;
    for (long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
        unsigned mk = ptmask[i];
        const unsigned* src = reinterpret_cast<const unsigned*>(feats + i * pay);
        while (mk) {
            const int o = __ffs(mk) - 1;
            mk &= mk - 1;
            const long long pos = ptpos[(long long)o * n + i];
            const SectionLayout L = section_layout(meta->npts[o], meta->nrows[o], pay);
            unsigned* dst = reinterpret_cast<unsigned*>(send + meta->off[o] + L.pay + pos * pay);
            for (long long w = lane; w < words; w += 32) dst[w] = src[w];
        }
    }
}

// Rows -> their owner's section (key, index of the point in that section).
// Row order inside a section is free: K2-K5 do not depend on it.
__global__ void __launch_bounds__(kPlanThreads) k_shard_pack_rows(
    long long R, long long n, int G, const unsigned long long* __restrict__ rowkey,
    const int* __restrict__ rowray, const int* __restrict__ rowown, const int* __restrict__ ptpos,
    ShardMeta* meta, char* __restrict__ send, long long pay, const FrameCtr* ctr, const long long* abort) {
    if (R < 0) R = (long long)ctr->rows;
    if (shard_aborted(abort, true)) return;
    __shared__ unsigned s_cnt[SVX_MAX_SHARDS];
    __shared__ unsigned long long s_base[SVX_MAX_SHARDS];
    if (blockIdx.x == 0 && threadIdx.x < G) {
        SectionHeader hd;
        hd.npts = (unsigned)meta->npts[threadIdx.x];
        hd.nrows = (unsigned)meta->nrows[threadIdx.x];
        hd.pay = (unsigned)pay;
        hd.magic = kSectionMagic;
        *reinterpret_cast<SectionHeader*>(send + meta->off[threadIdx.x]) = hd;
    }
    for (long long t0 = (long long)blockIdx.x * kPlanThreads; t0 < R;
         t0 += (long long)gridDim.x * kPlanThreads) {
        if (threadIdx.x < SVX_MAX_SHARDS) s_cnt[threadIdx.x] = 0;
        __syncthreads();
        const long long t = t0 + threadIdx.x;
        int o = -1;
        unsigned local = 0;
        if (t < R) {
            o = rowown[t];
            local = atomicAdd(&s_cnt[o], 1u);
        }
        __syncthreads();
        if (threadIdx.x < G && s_cnt[threadIdx.x])
            s_base[threadIdx.x] = atomicAdd(&meta->cursor[threadIdx.x], (unsigned long long)s_cnt[threadIdx.x]);
        __syncthreads();
        if (o >= 0) {
            const long long pos = (long long)s_base[o] + local;
            const SectionLayout L = section_layout(meta->npts[o], meta->nrows[o], pay);
            char* sec = send + meta->off[o];
            reinterpret_cast<unsigned long long*>(sec + L.keys)[pos] = rowkey[t];
            reinterpret_cast<int*>(sec + L.pts)[pos] = ptpos[(long long)o * n + rowray[t]];
        }
        __syncthreads();
    }
}

// Received rows' point indices, shifted to the concatenated point list.
__global__ void k_shard_rowray(long long nrows, const int* __restrict__ src, int pt_off,
                               int* __restrict__ dst) {
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < nrows;
         t += (long long)gridDim.x * blockDim.x)
        dst[t] = src[t] + pt_off;
}

int grid_of(long long n, int threads, int cap) {
    long long g = (n + threads - 1) / threads;
    return (int)std::max<long long>(1, std::min<long long>(g, cap));
}

long long payload_bytes(const svx_map* m, int feats_f64) {
    if (m->cfg.sem_kind == SVX_SEM_CLOSED) return 4;
    if (m->cfg.sem_kind == SVX_SEM_OPEN) return (long long)m->payload_d * (feats_f64 ? 8 : 4);
    return 0;
}

void fill_summary(const svx_map* m, svx_shard_summary* out) {
    const FrameCtr* hc = m->h_ctr;
    memset(out, 0, sizeof(*out));
    out->points_in = m->shard_n;
    out->nonfinite = (int64_t)hc->nonfinite;
    out->range = (int64_t)hc->range;
    out->degenerate = (int64_t)hc->degenerate;
    out->bad_label = (int64_t)hc->bad_label;
    out->used = (int64_t)hc->used;
    out->band_hits = (int64_t)hc->band_hits;
    out->rows = (int64_t)hc->rows;
    for (int a = 0; a < 3; ++a) {
        out->bbox_min[a] = hc->rows ? hc->bbox_min[a] : LLONG_MAX;
        out->bbox_max[a] = hc->rows ? hc->bbox_max[a] : LLONG_MIN;
    }
    out->err_budget = hc->err_budget;
    out->err_pack = hc->err_pack;
}

// ---- device-planned frames (svx_shard_*_async): one host sync per frame ----
//
// Summary vector (int64, SVX_SHARD_SUMMARY_WORDS): kSumWords counters summed
// over ranks, then kMaxWords maxima (bbox_max, -bbox_min, and the slices'
// scratch overflows: err_rows, err_cap).
enum {
    kSumPoints, kSumNonfinite, kSumRange, kSumDegenerate, kSumBadLabel, kSumUsed, kSumBandHits, kSumRows,
    kSumErrBudget, kSumErrPack, kSumWords
};
constexpr int kMaxWords = 8;
constexpr int kMaxErrRows = kSumWords + 6, kMaxErrCap = kSumWords + 7;
static_assert(kSumWords == SVX_SHARD_SUM_WORDS && kSumWords + kMaxWords == SVX_SHARD_SUMMARY_WORDS,
              "summary layout");

__global__ void k_shard_summary(const FrameCtr* __restrict__ c, long long n, long long* __restrict__ v) {
    v[kSumPoints] = n;
    v[kSumNonfinite] = (long long)c->nonfinite;
    v[kSumRange] = (long long)c->range;
    v[kSumDegenerate] = (long long)c->degenerate;
    v[kSumBadLabel] = (long long)c->bad_label;
    v[kSumUsed] = (long long)c->used;
    v[kSumBandHits] = (long long)c->band_hits;
    v[kSumRows] = (long long)c->rows;
    v[kSumErrBudget] = c->err_budget ? 1 : 0;
    v[kSumErrPack] = c->err_pack ? 1 : 0;
    for (int a = 0; a < 3; ++a) {
        v[kSumWords + a] = c->rows ? c->bbox_max[a] : LLONG_MIN;
        v[kSumWords + 3 + a] = c->rows ? -c->bbox_min[a] : LLONG_MIN;
    }
    v[kMaxErrRows] = c->err_rows ? 1 : 0;   // this slice's scratch was too small
    v[kMaxErrCap] = c->err_cap ? 1 : 0;
}

// The reference's pre-allocation checks (_core.pyx:661-712, :386-387) on the
// global summary, in shard_plan's order; every rank computes the same flags.
//   abort[0] step budget  [1] extent  [2] coordinate range  [3] key window
//   (re-march with the frame's minimum as key base)  [4] a slice's scratch
//   overflowed  [5] a section over its capacity (this rank)  [6] largest
//   section  [7] unused
__global__ void k_shard_checks(const long long* __restrict__ g, long long* __restrict__ abort) {
    for (int i = 0; i < SVX_SHARD_ABORT_WORDS; ++i) abort[i] = 0;
    if (g[kMaxErrRows] | g[kMaxErrCap]) {
        abort[4] = 1;
        return;
    }
    if (g[kSumErrBudget]) {
        abort[0] = 1;
        return;
    }
    if (g[kSumRows]) {
        bool extent = false, range = false;
        for (int a = 0; a < 3; ++a) {
            const long long hi = g[kSumWords + a], lo = -g[kSumWords + 3 + a];
            if (hi - lo >= (1LL << kPackBits)) extent = true;
            if (llabs(lo) >= kCoordLimit || llabs(hi) >= kCoordLimit) range = true;
        }
        if (extent) {
            abort[1] = 1;
            return;
        }
        if (range) {
            abort[2] = 1;
            return;
        }
    }
    if (g[kSumErrPack]) abort[3] = 1;
}

// Received sections (fixed capacity each, rank order): validate the headers,
// concatenation offsets and totals; the frame's row count goes to the
// counters K2-K5 read, or the frame is dropped before any mutation (a global
// abort, a corrupt section, or this rank's scratch too small: local[0] = 1).
struct ApplyOffsets {
    long long pt_off[SVX_MAX_SHARDS + 1];
    long long row_off[SVX_MAX_SHARDS + 1];
    unsigned npts[SVX_MAX_SHARDS], nrows[SVX_MAX_SHARDS];
    int live;
};

__global__ void k_shard_apply_prep(const char* __restrict__ recv, long long cap, int G, long long pay,
                                   const long long* __restrict__ abort, long long pcap, long long rcap,
                                   FrameCtr* __restrict__ ctr, ApplyOffsets* __restrict__ ao,
                                   long long* __restrict__ local) {
    local[0] = local[1] = local[2] = 0;
    ao->live = 0;
    bool drop = shard_aborted(abort, false) || abort[5] != 0;
    long long P = 0, R = 0;
    ao->pt_off[0] = ao->row_off[0] = 0;
    if (!drop) {
        for (int q = 0; q < G; ++q) {
            const SectionHeader hd = *reinterpret_cast<const SectionHeader*>(recv + q * cap);
            if (hd.magic != kSectionMagic || (long long)hd.pay != pay ||
                section_layout(hd.npts, hd.nrows, pay).size > cap) {
                local[2] = 1;   // corrupt exchange
                drop = true;
                break;
            }
            ao->npts[q] = hd.npts;
            ao->nrows[q] = hd.nrows;
            P += hd.npts;
            R += hd.nrows;
            ao->pt_off[q + 1] = P;
            ao->row_off[q + 1] = R;
        }
    }
    if (!drop && (P > pcap || R > rcap)) {
        local[0] = 1;   // grow and re-run this rank's apply
        local[1] = R;
        drop = true;
    }
    if (drop) {
        ctr->abort = 1;
        ctr->rows = ctr->rows_alloc = 0;
        return;
    }
    ao->live = 1;
    ctr->rows = ctr->rows_alloc = (unsigned long long)R;
}

// Sections -> the frame's point and row arrays (block y = source rank).
__global__ void k_shard_apply_copy(const char* __restrict__ recv, long long cap, long long pay,
                                   const ApplyOffsets* __restrict__ ao, double4* __restrict__ ray,
                                   char* __restrict__ payload, unsigned long long* __restrict__ rowkey,
                                   int* __restrict__ rowray) {
    if (!ao->live) return;
    const int q = blockIdx.y;
    const long long np = ao->npts[q], nr = ao->nrows[q];
    const SectionLayout L = section_layout(np, nr, pay);
    const char* sec = recv + q * cap;
    const long long p0 = ao->pt_off[q], r0 = ao->row_off[q];
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const double4* rs = reinterpret_cast<const double4*>(sec + L.rays);
    for (long long i = t0; i < np; i += stride) ray[p0 + i] = rs[i];
    if (pay) {
        const long long words = np * pay / 4;   // payload rows are whole 4-byte words
        const unsigned* src = reinterpret_cast<const unsigned*>(sec + L.pay);
        unsigned* dst = reinterpret_cast<unsigned*>(payload + p0 * pay);
        for (long long i = t0; i < words; i += stride) dst[i] = src[i];
    }
    const unsigned long long* ks = reinterpret_cast<const unsigned long long*>(sec + L.keys);
    const int* ps = reinterpret_cast<const int*>(sec + L.pts);
    for (long long i = t0; i < nr; i += stride) {
        rowkey[r0 + i] = ks[i];
        rowray[r0 + i] = ps[i] + (int)p0;
    }
}

// Per-rank report words for the summed report: touched voxels, new leaves,
// new voxels, and 1 when this rank must re-run its apply (scratch or pool
// capacity; nothing was changed).
__global__ void k_shard_apply_report(const FrameCtr* __restrict__ c, long long nblocks0, long long nvox0,
                                     const long long* __restrict__ local, long long* __restrict__ rep) {
    const bool redo = local[0] != 0 || c->err_cap != 0;
    rep[0] = redo ? 0 : (long long)c->n_touched;
    rep[1] = redo ? 0 : (long long)c->nblocks - nblocks0;
    rep[2] = redo ? 0 : (long long)c->nvox - nvox0;
    rep[3] = redo ? 1 : 0;
}

}  // namespace

svx_status shard_march(svx_map* m, const void* pts_in, int pts_f64, int64_t n, const PoseParams& pp,
                       const int32_t* labels_in, const void* feats_in, int feats_f64,
                       const int64_t* key_base, cudaStream_t s, svx_shard_summary* out) {
    const int kind = m->cfg.sem_kind;
    if (kind == SVX_SEM_CLOSED && !labels_in && n > 0)
        return fail(SVX_E_PAYLOAD, "closed-set grid requires per-point labels");
    if (kind == SVX_SEM_OPEN && !feats_in && n > 0)
        return fail(SVX_E_PAYLOAD, "open-set grid requires per-point features");
    if (n < 0) return fail(SVX_E_INPUT, "negative point count");
    if (n >= (int64_t)INT_MAX) return fail(SVX_E_INPUT, "point count exceeds 2^31-1");
    m->shard_phase = 0;
    m->shard_async = 0;
    m->shard_n = n;
    m->shard_rows = 0;
    m->shard_pts_f64 = pts_f64;
    m->shard_feats_f64 = feats_f64;
    m->shard_pp = pp;
    KeyPack kp = default_key_pack(m, pp);
    if (key_base)
        for (int a = 0; a < 3; ++a) kp.base[a] = key_base[a];
    m->shard_kp = kp;
    m->shard_lab = nullptr;
    m->shard_feat = nullptr;
    FrameCtr* hc = m->h_ctr;
    if (n == 0) {
        reset_ctr(m, m->frames);
        fill_summary(m, out);
        m->shard_phase = 1;
        return SVX_OK;
    }
    const void* pts;
    const void* feats = nullptr;
    const void* labv = nullptr;
    SVX_TRY(stage_in(pts_in, (size_t)n * 3 * (pts_f64 ? 8 : 4), m->in_pts, s, &pts));
    if (kind == SVX_SEM_CLOSED) SVX_TRY(stage_in(labels_in, (size_t)n * 4, m->in_lab, s, &labv));
    if (kind == SVX_SEM_OPEN)
        SVX_TRY(stage_in(feats_in, (size_t)n * m->payload_d * (feats_f64 ? 8 : 4), m->in_feat, s,
                         &feats));
    init_row_space(m, n);
    for (int attempt = 0;; ++attempt) {
        if (attempt >= 8) return fail(SVX_E_INTERNAL, "frame scratch could not be sized");
        SVX_TRY(reserve_frame(m, n, s));
        m->frame_slots = 0;   // shard rows travel without d / labels; owners use segments
        reset_ctr(m, m->frames);
        FrameParams& p = hc->p;
        p.pts = pts;
        p.labels = (const int32_t*)labv;
        p.feats = feats;
        p.n = n;
        p.pp = pp;
        p.kp = kp;
        p.nblocks0 = m->nblocks;
        FrameCtr* dc = ptr<FrameCtr>(m->ctr);
        hc->p.epilogue = 0;   // explicit copies here, no graph epilogue
        m->ctr_clean = false;
        SVX_CUDA(cudaMemcpyAsync(dc, hc, sizeof(FrameCtr), cudaMemcpyHostToDevice, s));
        SVX_TRY(launch_march(m, pts_f64, feats_f64, s));
        SVX_CUDA(cudaMemcpyAsync(hc, dc, sizeof(FrameCtr), cudaMemcpyDeviceToHost, s));
        SVX_CUDA(cudaStreamSynchronize(s));
        // local row-space shortfalls are re-run here; key window, budget,
        // extent and range are decided on the global summary
        if (hc->err_rows) {
            m->maxrows = 0;
            m->rcap = std::max<uint64_t>(m->rcap, hc->rows + hc->rows / 2 + 4096);
            continue;
        }
        if (hc->err_cap) {
            m->rcap = std::max<uint64_t>(2 * m->rcap, hc->rows + hc->rows / 2 + 4096);
            continue;
        }
        break;
    }
    m->shard_rows = (int64_t)hc->rows;
    m->shard_lab = labv;
    m->shard_feat = feats;
    fill_summary(m, out);
    m->shard_phase = 1;
    return SVX_OK;
}

svx_status shard_plan(svx_map* m, const svx_shard_summary* g, int rank, int G, int64_t* send_bytes,
                      int* remarch, cudaStream_t s) {
    if (m->shard_phase != 1) return fail(SVX_E_INPUT, "svx_shard_plan: no marched frame");
    if (G < 1 || G > SVX_MAX_SHARDS || rank < 0 || rank >= G)
        return fail(SVX_E_INPUT, "invalid shard rank / count");
    *remarch = 0;
    // the reference's pre-allocation checks on the whole frame (_core.pyx:661-712, :386-387)
    if (g->err_budget) {
        m->shard_phase = 0;
        return fail(SVX_E_INTERNAL, "ray band exceeds step budget; shrink max_range or grow voxels");
    }
    if (g->rows) {
        bool extent = false, range = false;
        for (int a = 0; a < 3; ++a) {
            if (g->bbox_max[a] - g->bbox_min[a] >= (1LL << kPackBits)) extent = true;
            if (llabs(g->bbox_min[a]) >= kCoordLimit || llabs(g->bbox_max[a]) >= kCoordLimit)
                range = true;
        }
        m->shard_phase = 0;
        if (extent)
            return fail(SVX_E_INTERNAL,
                        "frame voxel extent exceeds 2^21 per axis; shrink max_range or grow voxels");
        if (range) return fail(SVX_E_RANGE, "voxel coordinate beyond +/-2^30 addressable range");
        m->shard_phase = 1;
    }
    if (g->err_pack) {   // re-march every slice with keys based at the frame's minimum
        *remarch = 1;
        m->shard_phase = 0;
        return SVX_OK;
    }
    m->shard_sum = *g;
    m->shard_g = G;
    m->shard_rank = rank;
    const long long n = m->shard_n, R = m->shard_rows;
    const long long pay = payload_bytes(m, m->shard_feats_f64);
    const long long ntiles = std::max<long long>(1, (n + kPlanThreads - 1) / kPlanThreads);
    SVX_TRY(ensure(m->sh_meta, sizeof(ShardMeta), s));
    SVX_TRY(ensure(m->sh_mask, sizeof(unsigned) * std::max<long long>(n, 1), s));
    SVX_TRY(ensure(m->sh_pos, sizeof(int) * std::max<long long>(n, 1) * G, s));
    SVX_TRY(ensure(m->sh_tiles, sizeof(long long) * ntiles * G, s));
    ShardMeta* meta = ptr<ShardMeta>(m->sh_meta);
    SVX_CUDA(cudaMemsetAsync(meta, 0, sizeof(ShardMeta), s));
    if (n > 0) SVX_CUDA(cudaMemsetAsync(m->sh_mask.p, 0, sizeof(unsigned) * n, s));
    if (R > 0) {
        k_shard_rows<<<grid_of(R, kPlanThreads, kPersistentBlocks * 2), kPlanThreads, 0, s>>>(
            R, G, m->shard_kp, ptr<unsigned long long>(m->rowkey), ptr<int>(m->rowray),
            ptr<int>(m->rowvid), ptr<unsigned>(m->sh_mask), meta, ptr<FrameCtr>(m->ctr), nullptr);
        SVX_LAUNCHED();
    }
    if (n > 0) {
        k_shard_tiles<<<(int)ntiles, kPlanThreads, 0, s>>>(n, G, ptr<unsigned>(m->sh_mask),
                                                           ptr<long long>(m->sh_tiles));
        SVX_LAUNCHED();
    } else {
        SVX_CUDA(cudaMemsetAsync(m->sh_tiles.p, 0, sizeof(long long) * ntiles * G, s));
    }
    k_shard_plan<<<1, 32, 0, s>>>(ntiles, G, pay, ptr<long long>(m->sh_tiles), meta, 0, nullptr);
    SVX_LAUNCHED();
    ShardMeta hm;
    SVX_CUDA(cudaMemcpyAsync(&hm, meta, sizeof(ShardMeta), cudaMemcpyDeviceToHost, s));
    SVX_CUDA(cudaStreamSynchronize(s));
    for (int o = 0; o < G; ++o) {
        m->sh_npts[o] = hm.npts[o];
        m->sh_nrows[o] = hm.nrows[o];
        m->sh_bytes[o] = hm.size[o];
        send_bytes[o] = hm.size[o];
    }
    m->shard_phase = 2;
    return SVX_OK;
}

svx_status shard_pack(svx_map* m, void* send, int64_t capacity, cudaStream_t s) {
    if (m->shard_phase != 2) return fail(SVX_E_INPUT, "svx_shard_pack: no planned frame");
    const int G = m->shard_g;
    int64_t total = 0;
    for (int o = 0; o < G; ++o) total += m->sh_bytes[o];
    if (!send || capacity < total) return fail(SVX_E_INPUT, "shard send buffer too small");
    if (((uintptr_t)send & 15) != 0) return fail(SVX_E_INPUT, "shard send buffer not 16-byte aligned");
    if (!is_device_ptr(send)) return fail(SVX_E_INPUT, "shard send buffer must be device memory");
    const long long n = m->shard_n, R = m->shard_rows;
    const long long pay = payload_bytes(m, m->shard_feats_f64);
    ShardMeta* meta = ptr<ShardMeta>(m->sh_meta);
    if (n > 0) {
        const long long ntiles = (n + kPlanThreads - 1) / kPlanThreads;
        k_shard_pack_points<<<(int)ntiles, kPlanThreads, 0, s>>>(
            n, G, ptr<unsigned>(m->sh_mask), ptr<long long>(m->sh_tiles), ptr<double4>(m->ray),
            m->cfg.sem_kind == SVX_SEM_CLOSED ? (const int32_t*)m->shard_lab : nullptr,
            ptr<int>(m->sh_pos), meta, (char*)send, pay, nullptr);
        SVX_LAUNCHED();
        if (m->cfg.sem_kind == SVX_SEM_OPEN) {
            k_shard_pack_feats<<<grid_of(n * 32, 256, kPersistentBlocks * 2), 256, 0, s>>>(
                n, G, ptr<unsigned>(m->sh_mask), ptr<int>(m->sh_pos), (const char*)m->shard_feat,
                meta, (char*)send, pay, nullptr);
            SVX_LAUNCHED();
        }
    }
    k_shard_pack_rows<<<grid_of(R, kPlanThreads, kPersistentBlocks * 2), kPlanThreads, 0, s>>>(
        R, n, G, ptr<unsigned long long>(m->rowkey), ptr<int>(m->rowray), ptr<int>(m->rowvid),
        ptr<int>(m->sh_pos), meta, (char*)send, pay, ptr<FrameCtr>(m->ctr), nullptr);
    SVX_LAUNCHED();
    m->shard_phase = 3;
    return SVX_OK;
}

svx_status shard_apply(svx_map* m, const void* recv, const int64_t* recv_bytes, int G,
                       cudaStream_t s, svx_report* rep) {
    if (m->shard_phase != 3) return fail(SVX_E_INPUT, "svx_shard_apply: no packed frame");
    if (G != m->shard_g) return fail(SVX_E_INPUT, "svx_shard_apply: rank count differs from plan");
    int64_t total = 0;
    for (int q = 0; q < G; ++q) {
        if (recv_bytes[q] < (int64_t)sizeof(SectionHeader))
            return fail(SVX_E_INTERNAL, "corrupt shard exchange: short section");
        total += recv_bytes[q];
    }
    if (!recv || ((uintptr_t)recv & 15) != 0 || !is_device_ptr(recv))
        return fail(SVX_E_INPUT, "shard receive buffer must be 16-byte aligned device memory");
    SVX_CUDA(cudaEventRecord(m->ev0, s));
    const long long pay = payload_bytes(m, m->shard_feats_f64);
    SectionHeader hd[SVX_MAX_SHARDS];
    long long off[SVX_MAX_SHARDS], pt_off[SVX_MAX_SHARDS], row_off[SVX_MAX_SHARDS];
    {
        long long o = 0;
        for (int q = 0; q < G; ++q) {
            off[q] = o;
            SVX_CUDA(cudaMemcpyAsync(&hd[q], (const char*)recv + o, sizeof(SectionHeader),
                                     cudaMemcpyDeviceToHost, s));
            o += recv_bytes[q];
        }
        SVX_CUDA(cudaStreamSynchronize(s));
    }
    long long P = 0, R = 0;
    for (int q = 0; q < G; ++q) {
        if (hd[q].magic != kSectionMagic || (long long)hd[q].pay != pay ||
            section_layout(hd[q].npts, hd[q].nrows, pay).size != recv_bytes[q])
            return fail(SVX_E_INTERNAL, "corrupt shard exchange: section header mismatch");
        pt_off[q] = P;
        row_off[q] = R;
        P += hd[q].npts;
        R += hd[q].nrows;
    }
    if (P >= (long long)INT_MAX) return fail(SVX_E_INPUT, "point count exceeds 2^31-1");
    svx_report r;
    memset(&r, 0, sizeof(r));
    const svx_shard_summary& g = m->shard_sum;
    r.points_in = g.points_in;
    r.skipped_nonfinite = g.nonfinite;
    r.skipped_range = g.range;
    r.skipped_degenerate = g.degenerate;
    r.skipped_bad_label = g.bad_label;
    r.points_used = g.used;
    r.band_hits = g.band_hits;
    const int64_t nblocks0 = m->nblocks, nvox0 = m->nvox;
    FrameCtr* hc = m->h_ctr;
    if (R == 0) {   // nothing owned here this frame
        reset_ctr(m, m->frames);
        finish_frame(m, nblocks0, nvox0, r);
        m->frames++;
        m->shard_phase = 0;
        if (rep) *rep = r;
        return SVX_OK;
    }
    init_row_space(m, P);
    m->rcap = std::max<uint64_t>(m->rcap, (uint64_t)R + 4096);
    SVX_TRY(reserve_frame(m, P, s));
    if (pay) {
        DevBuf& pb = m->cfg.sem_kind == SVX_SEM_OPEN ? m->in_feat : m->in_lab;
        SVX_TRY(ensure(pb, (size_t)(P * pay), s));
    }
    // concatenate the sections: rays, payload, keys; point indices shifted
    for (int q = 0; q < G; ++q) {
        const SectionLayout L = section_layout(hd[q].npts, hd[q].nrows, pay);
        const char* sec = (const char*)recv + off[q];
        if (hd[q].npts) {
            SVX_CUDA(cudaMemcpyAsync(ptr<double4>(m->ray) + pt_off[q], sec + L.rays,
                                     sizeof(double4) * hd[q].npts, cudaMemcpyDeviceToDevice, s));
            if (pay) {
                char* pd = (char*)(m->cfg.sem_kind == SVX_SEM_OPEN ? m->in_feat.p : m->in_lab.p);
                SVX_CUDA(cudaMemcpyAsync(pd + pt_off[q] * pay, sec + L.pay, hd[q].npts * pay,
                                         cudaMemcpyDeviceToDevice, s));
            }
        }
        if (hd[q].nrows) {
            SVX_CUDA(cudaMemcpyAsync(ptr<unsigned long long>(m->rowkey) + row_off[q], sec + L.keys,
                                     8 * hd[q].nrows, cudaMemcpyDeviceToDevice, s));
            k_shard_rowray<<<grid_of(hd[q].nrows, 256, kPersistentBlocks), 256, 0, s>>>(
                hd[q].nrows, reinterpret_cast<const int*>(sec + L.pts), (int)pt_off[q],
                ptr<int>(m->rowray) + row_off[q]);
            SVX_LAUNCHED();
        }
    }
    const int feats_f64 = m->shard_feats_f64;
    for (int attempt = 0;; ++attempt) {
        if (attempt >= 8) return fail(SVX_E_INTERNAL, "frame scratch could not be sized");
        SVX_TRY(reserve_pools(m, s));
        reset_ctr(m, m->frames);
        FrameParams& p = hc->p;
        p.pts = nullptr;
        p.labels = m->cfg.sem_kind == SVX_SEM_CLOSED ? ptr<int32_t>(m->in_lab) : nullptr;
        p.feats = m->cfg.sem_kind == SVX_SEM_OPEN ? m->in_feat.p : nullptr;
        p.n = P;
        p.pp = m->shard_pp;
        p.kp = m->shard_kp;
        p.nblocks0 = nblocks0;
        p.slots = 0;   // shard sections always take the segment path
        hc->rows = (unsigned long long)R;
        hc->rows_alloc = (unsigned long long)R;
        FrameCtr* dc = ptr<FrameCtr>(m->ctr);
        hc->p.epilogue = 0;   // explicit copies here, no graph epilogue
        m->ctr_clean = false;
        SVX_CUDA(cudaMemcpyAsync(dc, hc, sizeof(FrameCtr), cudaMemcpyHostToDevice, s));
        SVX_TRY(launch_resolve(m, s));
        SVX_TRY(launch_segments(m, s));
        SVX_TRY(launch_scatter(m, s));
        SVX_TRY(launch_update_a(m, feats_f64, s));
        SVX_TRY(launch_update_b(m, feats_f64, s));
        SVX_CUDA(cudaMemcpyAsync(hc, dc, sizeof(FrameCtr), cudaMemcpyDeviceToHost, s));
        SVX_CUDA(cudaEventRecord(m->ev1, s));
        SVX_CUDA(cudaEventSynchronize(m->ev1));
        if (hc->err_cap) {
            SVX_TRY(recover_capacity(m, nblocks0, s));
            continue;
        }
        break;
    }
    float ms = 0.f;
    SVX_CUDA(cudaEventElapsedTime(&ms, m->ev0, m->ev1));
    r.kernel_ms = ms;
    finish_frame(m, nblocks0, nvox0, r);
    m->frames++;
    m->shard_phase = 0;
    if (rep) *rep = r;
    return SVX_OK;
}

// ---- device-planned frames --------------------------------------------------

svx_status shard_march_async(svx_map* m, const void* pts_in, int pts_f64, int64_t n, const PoseParams& pp,
                             const int32_t* labels_in, const void* feats_in, int feats_f64,
                             const int64_t* key_base, cudaStream_t s, int64_t* summary) {
    const int kind = m->cfg.sem_kind;
    if (kind == SVX_SEM_CLOSED && !labels_in && n > 0)
        return fail(SVX_E_PAYLOAD, "closed-set grid requires per-point labels");
    if (kind == SVX_SEM_OPEN && !feats_in && n > 0)
        return fail(SVX_E_PAYLOAD, "open-set grid requires per-point features");
    if (n < 0) return fail(SVX_E_INPUT, "negative point count");
    if (n >= (int64_t)INT_MAX) return fail(SVX_E_INPUT, "point count exceeds 2^31-1");
    if (!is_device_ptr(summary)) return fail(SVX_E_INPUT, "shard summary must be device memory");
    m->shard_phase = 0;
    m->shard_n = n;
    m->shard_rows = -1;   // on the device
    m->shard_pts_f64 = pts_f64;
    m->shard_feats_f64 = feats_f64;
    m->shard_pp = pp;
    KeyPack kp = default_key_pack(m, pp);
    if (key_base)
        for (int a = 0; a < 3; ++a) kp.base[a] = key_base[a];
    m->shard_kp = kp;
    m->shard_lab = nullptr;
    m->shard_feat = nullptr;
    FrameCtr* hc = m->h_ctr;
    FrameCtr* dc = ptr<FrameCtr>(m->ctr);
    const void* pts = nullptr;
    const void* feats = nullptr;
    const void* labv = nullptr;
    if (n > 0) {
        SVX_TRY(stage_in(pts_in, (size_t)n * 3 * (pts_f64 ? 8 : 4), m->in_pts, s, &pts));
        if (kind == SVX_SEM_CLOSED) SVX_TRY(stage_in(labels_in, (size_t)n * 4, m->in_lab, s, &labv));
        if (kind == SVX_SEM_OPEN)
            SVX_TRY(stage_in(feats_in, (size_t)n * m->payload_d * (feats_f64 ? 8 : 4), m->in_feat, s,
                             &feats));
        init_row_space(m, n);
        // the slice's rows are at most the frame's (last frame + half); an
        // overflow is caught on the device and the frame redone
        m->rcap = std::max<uint64_t>(m->rcap, (uint64_t)(m->sh_last_rows + m->sh_last_rows / 2 + 4096));
        SVX_TRY(reserve_frame(m, n, s));
    }
    m->frame_slots = 0;
    reset_ctr(m, m->frames);
    FrameParams& p = hc->p;
    p.pts = pts;
    p.labels = (const int32_t*)labv;
    p.feats = feats;
    p.n = n;
    p.pp = pp;
    p.kp = kp;
    p.nblocks0 = m->nblocks;
    hc->p.epilogue = 0;
    m->ctr_clean = false;
    SVX_CUDA(cudaMemcpyAsync(dc, hc, sizeof(FrameCtr), cudaMemcpyHostToDevice, s));
    if (n > 0) SVX_TRY(launch_march(m, pts_f64, feats_f64, s));
    k_shard_summary<<<1, 1, 0, s>>>(dc, n, (long long*)summary);
    SVX_LAUNCHED();
    m->shard_lab = labv;
    m->shard_feat = feats;
    m->shard_async = 1;
    m->shard_phase = 1;
    return SVX_OK;
}

svx_status shard_plan_async(svx_map* m, const int64_t* gsum, int rank, int G, int64_t cap, cudaStream_t s,
                            int64_t* abort) {
    if (m->shard_phase != 1 || !m->shard_async) return fail(SVX_E_INPUT, "svx_shard_plan_async: no marched frame");
    if (G < 1 || G > SVX_MAX_SHARDS || rank < 0 || rank >= G)
        return fail(SVX_E_INPUT, "invalid shard rank / count");
    if (cap < 64 || (cap & 15)) return fail(SVX_E_INPUT, "shard section capacity must be a multiple of 16 >= 64");
    if (!is_device_ptr(gsum) || !is_device_ptr(abort))
        return fail(SVX_E_INPUT, "shard summary / abort words must be device memory");
    m->shard_g = G;
    m->shard_rank = rank;
    m->sh_cap = cap;
    const long long n = m->shard_n;
    const long long pay = payload_bytes(m, m->shard_feats_f64);
    const long long ntiles = std::max<long long>(1, (n + kPlanThreads - 1) / kPlanThreads);
    SVX_TRY(ensure(m->sh_meta, sizeof(ShardMeta), s));
    SVX_TRY(ensure(m->sh_mask, sizeof(unsigned) * std::max<long long>(n, 1), s));
    SVX_TRY(ensure(m->sh_pos, sizeof(int) * std::max<long long>(n, 1) * G, s));
    SVX_TRY(ensure(m->sh_tiles, sizeof(long long) * ntiles * G, s));
    ShardMeta* meta = ptr<ShardMeta>(m->sh_meta);
    long long* ab = (long long*)abort;
    SVX_CUDA(cudaMemsetAsync(meta, 0, sizeof(ShardMeta), s));
    k_shard_checks<<<1, 1, 0, s>>>((const long long*)gsum, ab);
    SVX_LAUNCHED();
    if (n > 0) {
        SVX_CUDA(cudaMemsetAsync(m->sh_mask.p, 0, sizeof(unsigned) * n, s));
        k_shard_rows<<<kPersistentBlocks * 2, kPlanThreads, 0, s>>>(
            -1, G, m->shard_kp, ptr<unsigned long long>(m->rowkey), ptr<int>(m->rowray),
            ptr<int>(m->rowvid), ptr<unsigned>(m->sh_mask), meta, ptr<FrameCtr>(m->ctr), ab);
        SVX_LAUNCHED();
        k_shard_tiles<<<(int)ntiles, kPlanThreads, 0, s>>>(n, G, ptr<unsigned>(m->sh_mask),
                                                           ptr<long long>(m->sh_tiles));
        SVX_LAUNCHED();
    } else {
        SVX_CUDA(cudaMemsetAsync(m->sh_tiles.p, 0, sizeof(long long) * ntiles * G, s));
    }
    k_shard_plan<<<1, 32, 0, s>>>(ntiles, G, pay, ptr<long long>(m->sh_tiles), meta, cap, ab);
    SVX_LAUNCHED();
    m->shard_phase = 2;
    return SVX_OK;
}

svx_status shard_pack_async(svx_map* m, void* send, int64_t cap, cudaStream_t s, const int64_t* abort) {
    if (m->shard_phase != 2 || !m->shard_async) return fail(SVX_E_INPUT, "svx_shard_pack_async: no planned frame");
    if (cap != m->sh_cap) return fail(SVX_E_INPUT, "svx_shard_pack_async: capacity differs from plan");
    if (!send || ((uintptr_t)send & 15) != 0 || !is_device_ptr(send))
        return fail(SVX_E_INPUT, "shard send buffer must be 16-byte aligned device memory");
    const int G = m->shard_g;
    const long long n = m->shard_n;
    const long long pay = payload_bytes(m, m->shard_feats_f64);
    ShardMeta* meta = ptr<ShardMeta>(m->sh_meta);
    const long long* ab = (const long long*)abort;
    if (n > 0) {
        const long long ntiles = (n + kPlanThreads - 1) / kPlanThreads;
        k_shard_pack_points<<<(int)ntiles, kPlanThreads, 0, s>>>(
            n, G, ptr<unsigned>(m->sh_mask), ptr<long long>(m->sh_tiles), ptr<double4>(m->ray),
            m->cfg.sem_kind == SVX_SEM_CLOSED ? (const int32_t*)m->shard_lab : nullptr,
            ptr<int>(m->sh_pos), meta, (char*)send, pay, ab);
        SVX_LAUNCHED();
        if (m->cfg.sem_kind == SVX_SEM_OPEN) {
            k_shard_pack_feats<<<grid_of(n * 32, 256, kPersistentBlocks * 2), 256, 0, s>>>(
                n, G, ptr<unsigned>(m->sh_mask), ptr<int>(m->sh_pos), (const char*)m->shard_feat,
                meta, (char*)send, pay, ab);
            SVX_LAUNCHED();
        }
    }
    k_shard_pack_rows<<<kPersistentBlocks * 2, kPlanThreads, 0, s>>>(
        -1, n, G, ptr<unsigned long long>(m->rowkey), ptr<int>(m->rowray), ptr<int>(m->rowvid),
        ptr<int>(m->sh_pos), meta, (char*)send, pay, ptr<FrameCtr>(m->ctr), ab);
    SVX_LAUNCHED();
    m->shard_phase = 3;
    return SVX_OK;
}

svx_status shard_apply_async(svx_map* m, const void* recv, int64_t cap, int G, const int64_t* abort,
                             int64_t frame_points, cudaStream_t s, int64_t* rep_words) {
    if ((m->shard_phase != 3 && m->shard_phase != 5) || !m->shard_async)
        return fail(SVX_E_INPUT, "svx_shard_apply_async: no packed frame");
    if (G != m->shard_g || cap != m->sh_cap) return fail(SVX_E_INPUT, "svx_shard_apply_async: plan mismatch");
    if (!recv || ((uintptr_t)recv & 15) != 0 || !is_device_ptr(recv) || !is_device_ptr(rep_words))
        return fail(SVX_E_INPUT, "shard receive buffer / report words must be device memory");
    if (frame_points < 0) return fail(SVX_E_INPUT, "negative frame point count");
    if (!m->sh_hlocal) SVX_CUDA(cudaMallocHost((void**)&m->sh_hlocal, 4 * sizeof(long long)));
    const long long pay = payload_bytes(m, m->shard_feats_f64);
    if (m->shard_phase == 3) {   // (a re-run keeps the frame's starting counts: the
        m->sh_nblocks0 = m->nblocks;   //  failed attempt's leaves stay allocated)
        m->sh_nvox0 = m->nvox;
    }
    const int64_t nblocks0 = m->sh_nblocks0, nvox0 = m->sh_nvox0;
    const int64_t P = std::max<int64_t>(frame_points, 1);   // a point reaches a rank at most once
    init_row_space(m, P);
    m->rcap = std::max<uint64_t>(m->rcap, (uint64_t)(m->sh_last_rows + m->sh_last_rows / 2 + 4096));
    SVX_TRY(reserve_frame(m, P, s));
    if (pay) {
        DevBuf& pb = m->cfg.sem_kind == SVX_SEM_OPEN ? m->in_feat : m->in_lab;
        SVX_TRY(ensure(pb, (size_t)(P * pay), s));
    }
    SVX_TRY(reserve_pools(m, s));
    SVX_TRY(ensure(m->sh_ao, sizeof(ApplyOffsets) + 4 * sizeof(long long), s));
    ApplyOffsets* ao = ptr<ApplyOffsets>(m->sh_ao);
    long long* local = reinterpret_cast<long long*>(ptr<char>(m->sh_ao) + sizeof(ApplyOffsets));
    FrameCtr* hc = m->h_ctr;
    FrameCtr* dc = ptr<FrameCtr>(m->ctr);
    reset_ctr(m, m->frames);
    FrameParams& p = hc->p;
    p.pts = nullptr;
    p.labels = m->cfg.sem_kind == SVX_SEM_CLOSED ? ptr<int32_t>(m->in_lab) : nullptr;
    p.feats = m->cfg.sem_kind == SVX_SEM_OPEN ? m->in_feat.p : nullptr;
    p.n = P;
    p.pp = m->shard_pp;
    p.kp = m->shard_kp;
    p.nblocks0 = nblocks0;
    p.slots = 0;   // shard sections always take the segment path
    hc->p.epilogue = 0;
    m->ctr_clean = false;
    SVX_CUDA(cudaMemcpyAsync(dc, hc, sizeof(FrameCtr), cudaMemcpyHostToDevice, s));
    SVX_CUDA(cudaEventRecord(m->ev0, s));
    k_shard_apply_prep<<<1, 1, 0, s>>>((const char*)recv, cap, G, pay, (const long long*)abort,
                                       (long long)m->npts_cap, (long long)m->rcap, dc, ao, local);
    SVX_LAUNCHED();
    char* payload = pay ? (char*)(m->cfg.sem_kind == SVX_SEM_OPEN ? m->in_feat.p : m->in_lab.p) : nullptr;
    k_shard_apply_copy<<<dim3(std::max(1, kPersistentBlocks / std::max(1, G)), G), 256, 0, s>>>(
        (const char*)recv, cap, pay, ao, ptr<double4>(m->ray), payload, ptr<unsigned long long>(m->rowkey),
        ptr<int>(m->rowray));
    SVX_LAUNCHED();
    const int feats_f64 = m->shard_feats_f64;
    SVX_TRY(launch_resolve(m, s));
    SVX_TRY(launch_segments(m, s));
    SVX_TRY(launch_scatter(m, s));
    SVX_TRY(launch_update_a(m, feats_f64, s));
    SVX_TRY(launch_update_b(m, feats_f64, s));
    k_shard_apply_report<<<1, 1, 0, s>>>(dc, nblocks0, nvox0, local, (long long*)rep_words);
    SVX_LAUNCHED();
    SVX_CUDA(cudaMemcpyAsync(hc, dc, sizeof(FrameCtr), cudaMemcpyDeviceToHost, s));
    SVX_CUDA(cudaMemcpyAsync(m->sh_hlocal, local, 3 * sizeof(long long), cudaMemcpyDeviceToHost, s));
    SVX_CUDA(cudaEventRecord(m->ev1, s));
    m->shard_phase = 4;
    return SVX_OK;
}

svx_status shard_finish(svx_map* m, const int64_t* g, const int64_t* abort, const int64_t* rsum,
                        svx_report* rep, int32_t* action, int64_t* need) {
    if (m->shard_phase != 4 || !m->shard_async) return fail(SVX_E_INPUT, "svx_shard_finish: no applied frame");
    SVX_CUDA(cudaEventSynchronize(m->ev1));   // (the caller has synchronised; cheap)
    *action = 0;
    *need = 0;
    FrameCtr* hc = m->h_ctr;
    const long long* loc = m->sh_hlocal;
    if (abort[4]) {   // a slice's scratch overflowed: larger row space, then redo everywhere
        if (g[kMaxErrRows]) m->maxrows = 0;
        m->rcap = std::max<uint64_t>(2 * m->rcap, (uint64_t)g[kSumRows] + (uint64_t)g[kSumRows] / 2 + 4096);
        m->shard_phase = 0;
        *action = 1;
        return SVX_OK;
    }
    m->shard_phase = 0;
    if (abort[0]) return fail(SVX_E_INTERNAL, "ray band exceeds step budget; shrink max_range or grow voxels");
    if (abort[1])
        return fail(SVX_E_INTERNAL, "frame voxel extent exceeds 2^21 per axis; shrink max_range or grow voxels");
    if (abort[2]) return fail(SVX_E_RANGE, "voxel coordinate beyond +/-2^30 addressable range");
    if (abort[3] || abort[5]) {   // key rebase / larger sections: redo the frame everywhere
        *need = abort[5] ? abort[6] : 0;
        *action = 1;
        return SVX_OK;
    }
    if (loc[2]) return fail(SVX_E_INTERNAL, "corrupt shard exchange: section header mismatch");
    const int64_t nblocks0 = m->sh_nblocks0, nvox0 = m->sh_nvox0;
    if (loc[0] || hc->err_cap) {   // this rank's scratch or pools: grow, redo its apply
        if (hc->err_cap) SVX_TRY(recover_capacity(m, nblocks0, 0));
        if (loc[0]) m->rcap = std::max<uint64_t>(m->rcap, (uint64_t)loc[1] + (uint64_t)loc[1] / 2 + 4096);
        m->shard_phase = 5;   // packed sections still in the receive buffer
        *action = 2;
        return SVX_OK;
    }
    svx_report r;
    memset(&r, 0, sizeof(r));
    r.points_in = g[kSumPoints];
    r.skipped_nonfinite = g[kSumNonfinite];
    r.skipped_range = g[kSumRange];
    r.skipped_degenerate = g[kSumDegenerate];
    r.skipped_bad_label = g[kSumBadLabel];
    r.points_used = g[kSumUsed];
    r.band_hits = g[kSumBandHits];
    float ms = 0.f;
    SVX_CUDA(cudaEventElapsedTime(&ms, m->ev0, m->ev1));
    r.kernel_ms = ms;
    finish_frame(m, nblocks0, nvox0, r);
    m->sh_last_rows = std::max<int64_t>((int64_t)g[kSumRows], (int64_t)hc->rows);
    m->frames++;
    if (rsum) {
        r.touched_voxels = rsum[0];
        r.new_blocks = rsum[1];
        r.new_voxels = rsum[2];
        if (rsum[3] > 0) *action = 3;
    }
    if (rep) *rep = r;
    return SVX_OK;
}

}  // namespace svx

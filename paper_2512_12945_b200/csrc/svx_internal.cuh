// svx_internal.cuh -- shared definitions of the B200 integration engine.
//
// HBM layout:
//   block hash   int4[hcap]        {bx, by, bz, val}; val = block id, EMPTY, BUSY or PENDING
//   block pool   int4 bcoord[bcap]  leaf coords (voxel >> 3), w = creation frame
//                u64  bmask[bcap*8] 512-bit active mask (GridCore.leaf_mask, _core.pyx:92)
//                i32  bslot[bcap*512] slot -> voxel id (-1 = inactive)
//   voxel pool   d[vcap], w[vcap]        TSDF (f64 reference layout or f32 compact)
//                sem0[vcap*C|D]          closed counts or open mean m
//                sem1[vcap*D]            open scale beta
// Voxel ids are dense, assigned in activation order and never recycled, so a
// voxel's payload row is contiguous (the NanoVDB "index grid" idea) and the
// open-set means form a dense (V, D) matrix for query scoring.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/svx.h"

namespace svx {

constexpr int kLeafLog2 = 3;                 // TreeConfig.leaf_log2 default (config.py:26)
constexpr int kLeafSide = 1 << kLeafLog2;    // 8
constexpr int kLeafVolume = 512;             // 8^3
constexpr int kMaskWords = 8;                // 512 bits
constexpr int kInternalLog2 = 4;             // TreeConfig.internal_log2 (config.py:27), stats only
constexpr int64_t kCoordLimit = int64_t(1) << 30;   // coords.py:41 COORD_LIMIT
constexpr int kPackBits = 21;                       // _core.pyx:34 PACK_BITS
constexpr int64_t kStepBudget = int64_t(1) << 20;   // _core.pyx:35 STEP_BUDGET

constexpr int kHashEmpty = -1;
constexpr int kHashBusy = -2;
constexpr int kHashPendingBase = -3;  // PENDING(tmp) = -3 - tmp

// Per-frame device counters, copied back once per frame.
struct FrameCtr {
    unsigned long long nonfinite;
    unsigned long long range;
    unsigned long long degenerate;
    unsigned long long bad_label;
    unsigned long long used;
    unsigned long long band_hits;   // rows emitted before the w <= 0 drop
    unsigned long long rows;        // rows kept (w > 0)
    unsigned long long n_new_blocks;
    unsigned long long n_new_voxels;
    unsigned long long n_groups;    // written by RLE (num runs)
    long long bbox_min[3];          // over kept rows (after the w <= 0 drop)
    long long bbox_max[3];
    int err_budget;                 // a ray exceeded the DDA step budget
    int pad[3];
};

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

struct PoseParams {
    double R[9];
    double t[3];
    int sensor;      // 1: transform points by (R, t); 0: points already world, origin = t
};

struct KeyPack {
    int mn[3];
    int bz, byz;     // shift amounts: key = (dx << byz) | (dy << bz) | dz
    int nbits;
};

}  // namespace svx

struct svx_map {
    svx_config cfg;
    int payload_d = 0;     // C (closed) or D (open)
    // persistent state
    svx::DevBuf hash;  int64_t hcap = 0;
    svx::DevBuf bcoord, bmask, bslot;  int64_t bcap = 0, nblocks = 0;
    svx::DevBuf vd, vw, s0, s1;        int64_t vcap = 0, nvox = 0;
    int64_t frames = 0;
    // per-frame scratch
    svx::DevBuf in_pts, in_lab, in_feat;
    svx::DevBuf ray, cnt, off;
    svx::DevBuf keys0, keys1, rid0, rid1;
    int* srid = nullptr;   // sorted row -> point index (one of rid0/rid1 after the sort)
    svx::DevBuf ukeys, runlen, gstart, gblock, gvid, gnew, grank;
    svx::DevBuf newpos, newcoord, newfirst, newfirst2, neworder, neworder2, tmp2id;
    svx::DevBuf cubtmp;
    svx::DevBuf ctr;      // FrameCtr
    svx::FrameCtr* h_ctr = nullptr;  // pinned mirror
    // query scratch
    svx::DevBuf act_cnt, act_off, act_vid, act_coord, q_buf, out_buf;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // optional per-stage timing (svx_set_profiling)
    bool prof = false;
    cudaEvent_t st_ev[2 * SVX_N_STAGES] = {};
    unsigned st_mask = 0;
    double stage_ms[SVX_N_STAGES] = {};
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

// ---- block hash ------------------------------------------------------------
// 64-bit finaliser-style mix of the three leaf coordinates.
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

// Read-only lookup (no concurrent inserts).  Returns block id or -1.
__device__ inline int hash_find(const int4* __restrict__ table, int64_t mask, int a, int b, int c) {
    int64_t pos = (int64_t)(block_hash(a, b, c) & (uint64_t)mask);
    while (true) {
        int4 s = __ldg(table + pos);
        if (s.w == kHashEmpty) return -1;
        if (s.x == a && s.y == b && s.z == c) return s.w;
        pos = (pos + 1) & mask;
    }
}

// ---- launchers implemented in the .cu files ---------------------------------
// svx_march.cu
svx_status launch_count(svx_map* m, const void* pts, int pts_f64, int64_t n, const PoseParams& pp,
                        const int32_t* labels, const void* feats, int feats_f64,
                        cudaStream_t s);
svx_status launch_fill(svx_map* m, int64_t n, const PoseParams& pp, const KeyPack& kp,
                       cudaStream_t s);
// svx_update.cu
svx_status launch_blocks(svx_map* m, int64_t U, const KeyPack& kp, cudaStream_t s);
svx_status launch_assign_blocks(svx_map* m, int64_t nnew, const unsigned* order, cudaStream_t s);
svx_status launch_resolve(svx_map* m, int64_t U, const KeyPack& kp, cudaStream_t s);
svx_status launch_activate(svx_map* m, int64_t U, const KeyPack& kp, cudaStream_t s);
svx_status launch_update(svx_map* m, int64_t U, const KeyPack& kp, const PoseParams& pp,
                         const int32_t* labels, const void* feats, int feats_f64, cudaStream_t s);
svx_status launch_rehash(svx_map* m, int4* new_table, int64_t new_cap, cudaStream_t s);
// svx_query.cu
svx_status build_active_list(svx_map* m, int64_t* count, cudaStream_t s);
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

}  // namespace svx

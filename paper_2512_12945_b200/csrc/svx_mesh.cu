// svx_mesh.cu -- zero-level surface extraction over the device map
// (Mapper.extract = extract_mesh, mesh.py:419-545; per-vertex labels
// voxel_labels :392-416; palette lookup palette_colors :382-389).
//
// The reference's semantics, restated for the GPU:
//   * cells are 2x2x2 corner neighbourhoods anchored at every kept voxel
//     (active, weight >= min_weight) whose 7 other corners are kept voxels;
//     case bit c = D(corner c) < 0; corner c sits at anchor + (x, y, z) with
//     x = ((c+1)>>1)&1, y = (c>>1)&1, z = c>>2;
//   * one vertex per crossed edge of a live cell, identified by (lower
//     voxel, axis), at (lower + 0.5) * h plus t * h along the axis,
//     t = d_lo / (d_lo - d_hi), all in f64;
//   * triangles from the 256-case table in cell order, reversed (normals
//     toward positive D), dropped when the cross product of their edges
//     squares to zero; vertices no surviving triangle uses are dropped;
//   * output order: vertices by (x, y, z, axis) of their lower voxel,
//     triangles by (x, y, z) of their cell, then table order -- exactly the
//     reference's spatial re-sort + np.unique numbering, so two maps with
//     equal content give byte-identical meshes on either implementation.
//
// GPU mapping (HBM-bound integer / gather work, no tensor cores): corner
// lookups go through the leaf hash + bslot table (no global sort of the
// voxels); only live cells and vertex-owning voxels are sorted (CUB radix on
// the packed 60-bit spatial key), and the vertex numbering is a popcount
// scan over per-voxel 3-bit axis masks.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <string>

#include "svx_internal.cuh"

namespace svx {
namespace {

constexpr int kPackBits = 20;                         // mesh.py:352 _MESH_PACK_BITS
constexpr unsigned long long kPackMask = (1ULL << kPackBits) - 1;

// The 256-case triangle table of classic marching cubes (the public-domain
// Lorensen-Cline / Bourke constants; case bit c = corner c inside).  Packed
// one case per word: bits 60..63 = triangle count, nibble i (i < 15) = edge
// index of the i-th triangle corner.  The edge table is derived
// (edge_mask below), not stored.
__constant__ unsigned long long c_tri[256] = {
    0x0fffffffffffffffULL, 0x1ffffffffffff380ULL, 0x1ffffffffffff910ULL, 0x2fffffffff189381ULL,
    0x1ffffffffffffa21ULL, 0x2fffffffffa21380ULL, 0x2fffffffff920a29ULL, 0x3ffffff89a8a2382ULL,
    0x1ffffffffffff2b3ULL, 0x2fffffffff0b82b0ULL, 0x2fffffffffb32091ULL, 0x3ffffffb89b912b1ULL,
    0x2fffffffff3ab1a3ULL, 0x3ffffffab8a801a0ULL, 0x3ffffff9ab9b3093ULL, 0x2fffffffffb8aa89ULL,
    0x1ffffffffffff874ULL, 0x2fffffffff437034ULL, 0x2fffffffff748910ULL, 0x3ffffff137174914ULL,
    0x2fffffffff748a21ULL, 0x3ffffffa21403743ULL, 0x3ffffff748209a29ULL, 0x4fff4973727929a2ULL,
    0x2fffffffff2b3748ULL, 0x3ffffff40242b74bULL, 0x3ffffffb32748109ULL, 0x4fff1292b9b49b74ULL,
    0x3ffffff487ab31a3ULL, 0x4fff4b7401b41ab1ULL, 0x4fff30bab9b09874ULL, 0x3ffffffab99b4b74ULL,
    0x1ffffffffffff459ULL, 0x2fffffffff380459ULL, 0x2fffffffff051450ULL, 0x3ffffff513538458ULL,
    0x2fffffffff459a21ULL, 0x3ffffff594a21803ULL, 0x3ffffff204245a25ULL, 0x4fff8434535235a2ULL,
    0x2fffffffffb32459ULL, 0x3ffffff594b802b0ULL, 0x3ffffffb32510450ULL, 0x4fff584b82852512ULL,
    0x3ffffff45931ab3aULL, 0x4fffab81a8180594ULL, 0x4fff30bab5b05045ULL, 0x3ffffffb8aa85845ULL,
    0x2fffffffff975879ULL, 0x3ffffff375359039ULL, 0x3ffffff751710870ULL, 0x2fffffffff753351ULL,
    0x3ffffff21a759879ULL, 0x4fff37503505921aULL, 0x4fff25a758528208ULL, 0x3ffffff7533525a2ULL,
    0x3ffffff2b3987597ULL, 0x4fffb72029279759ULL, 0x4fff751871810b32ULL, 0x3ffffff51771b12bULL,
    0x4fffb3a31a758859ULL, 0x50aba010b7905075ULL, 0x507570805a30b0abULL, 0x2fffffffff5b75abULL,
    0x1ffffffffffff56aULL, 0x2fffffffff6a5380ULL, 0x2fffffffff6a5109ULL, 0x3ffffff6a5891381ULL,
    0x2fffffffff162561ULL, 0x3ffffff803621561ULL, 0x3ffffff620609569ULL, 0x4fff823625285895ULL,
    0x2fffffffff56ab32ULL, 0x3ffffff56a02b80bULL, 0x3ffffff6a5b32910ULL, 0x4fffb892b92916a5ULL,
    0x3ffffff315356b36ULL, 0x4fff6b51505b0b80ULL, 0x4fff9505606306b3ULL, 0x3ffffff89bb96956ULL,
    0x2fffffffff8746a5ULL, 0x3ffffffa56374034ULL, 0x3ffffff7486a5091ULL, 0x4fff49737179156aULL,
    0x3ffffff874156216ULL, 0x4fff743403625521ULL, 0x4fff620560509748ULL, 0x5962695923497937ULL,
    0x3ffffff56a4872b3ULL, 0x4fffb720242746a5ULL, 0x4fff6a5b32874910ULL, 0x56a54b7b492b9129ULL,
    0x4fff6b51535b3748ULL, 0x5b404b7b016b5b15ULL, 0x574836b630560950ULL, 0x4fff9b7974b96956ULL,
    0x2fffffffffa4694aULL, 0x3ffffff380a946a4ULL, 0x3ffffff04606a10aULL, 0x4fffa16468618138ULL,
    0x3ffffff462421941ULL, 0x4fff462942921803ULL, 0x2fffffffff624420ULL, 0x3ffffff624428238ULL,
    0x3ffffff32b46a94aULL, 0x4fff6a4a94b82280ULL, 0x4fffa164606102b3ULL, 0x51b8b12184a16146ULL,
    0x4fff36b319639469ULL, 0x514641916b0181b8ULL, 0x3ffffff4600636b3ULL, 0x2fffffffff86b846ULL,
    0x3ffffffa98a876a7ULL, 0x4fffa76a907a0370ULL, 0x4fff0818717a176aULL, 0x3ffffff37117a76aULL,
    0x4fff768981861621ULL, 0x5937390976192962ULL, 0x3ffffff206607087ULL, 0x2fffffffff276237ULL,
    0x4fff76898a86ab32ULL, 0x57a9a76790b72702ULL, 0x5b32a767a1871081ULL, 0x4fff17616a71b12bULL,
    0x563136b619768698ULL, 0x2fffffffff76b190ULL, 0x4fff06b0b3607087ULL, 0x1ffffffffffff6b7ULL,
    0x1ffffffffffffb67ULL, 0x2fffffffff67b803ULL, 0x2fffffffff67b910ULL, 0x3ffffff67b138918ULL,
    0x2fffffffff7b621aULL, 0x3ffffff7b6803a21ULL, 0x3ffffff7b69a2092ULL, 0x4fff89a38a3a27b6ULL,
    0x2fffffffff726327ULL, 0x3ffffff026067807ULL, 0x3ffffff910732672ULL, 0x4fff678891681261ULL,
    0x3ffffff73171a67aULL, 0x4fff801781a7167aULL, 0x4fff7a69a0a70730ULL, 0x3ffffff9a88a7a67ULL,
    0x2fffffffff68b486ULL, 0x3ffffff640603b63ULL, 0x3ffffff109648b68ULL, 0x4fff63b139369649ULL,
    0x3ffffff1a28b6486ULL, 0x4fff640b60b03a21ULL, 0x4fff9a2920b648b4ULL, 0x536463b34923a39aULL,
    0x3ffffff264248328ULL, 0x2fffffffff264240ULL, 0x4fff834642432091ULL, 0x3ffffff642241491ULL,
    0x4fff1a6648168318ULL, 0x3ffffff40660a01aULL, 0x539a9303a6834364ULL, 0x2fffffffff4a649aULL,
    0x2fffffffffb67594ULL, 0x3ffffff67b594380ULL, 0x3ffffffb67045105ULL, 0x4fff51345343867bULL,
    0x3ffffffb6721a459ULL, 0x4fff594380a217b6ULL, 0x4fff204a24a45b67ULL, 0x567b25a523453843ULL,
    0x3ffffff945267327ULL, 0x4fff786260680459ULL, 0x4fff045051673263ULL, 0x5851584812786826ULL,
    0x4fff73167161a459ULL, 0x5459078701671a61ULL, 0x5a737a6a305a4a04ULL, 0x4fffa84a458a7a67ULL,
    0x3ffffff98b9b6596ULL, 0x4fff590650360b63ULL, 0x4fffb65510b508b0ULL, 0x3ffffff1355363b6ULL,
    0x4fff65b8b9b59a21ULL, 0x5a21965690b603b0ULL, 0x552025a50865b58bULL, 0x4fff35a3a25363b6ULL,
    0x4fff283265825985ULL, 0x3ffffff260069659ULL, 0x5826283865081851ULL, 0x2fffffffff612651ULL,
    0x5698965683a61631ULL, 0x4fff06505960a01aULL, 0x2fffffffffa65830ULL, 0x1ffffffffffff65aULL,
    0x2fffffffffb57a5bULL, 0x3ffffff03857ba5bULL, 0x3ffffff091ba57b5ULL, 0x4fff1381897ba57aULL,
    0x3ffffff15717b21bULL, 0x4fffb27571721380ULL, 0x4fff7b2209729579ULL, 0x5289823295b27257ULL,
    0x3ffffff573532a52ULL, 0x4fff52a578258028ULL, 0x4fff2a37353a5109ULL, 0x525752a278129289ULL,
    0x2fffffffff573531ULL, 0x3ffffff571170780ULL, 0x3ffffff735539309ULL, 0x2fffffffff795789ULL,
    0x3ffffff8ba8a5485ULL, 0x4fff03bba50b5405ULL, 0x4fff54aba8a48910ULL, 0x541314943b54a4baULL,
    0x4fff8548b2582152ULL, 0x5b151b2b543b0b40ULL, 0x558b8545b2950520ULL, 0x2fffffffff3b2549ULL,
    0x4fff483543253a52ULL, 0x3ffffff0244252a5ULL, 0x5910854583a532a3ULL, 0x4fff2492914252a5ULL,
    0x3ffffff153358548ULL, 0x2fffffffff501540ULL, 0x4fff530509358548ULL, 0x1ffffffffffff549ULL,
    0x3ffffffba9b947b4ULL, 0x4fffba97b9794380ULL, 0x4fffb470414b1ba1ULL, 0x54bab474a1843413ULL,
    0x4fff219b294b97b4ULL, 0x53801b2b197b9479ULL, 0x3ffffff04224b47bULL, 0x4fff42343824b47bULL,
    0x4fff947732972a92ULL, 0x570207872a4797a9ULL, 0x5a040a1a472a3a73ULL, 0x2fffffffff4782a1ULL,
    0x3ffffff317714194ULL, 0x4fff178180714194ULL, 0x2fffffffff347304ULL, 0x1ffffffffffff784ULL,
    0x2fffffffff8ba8a9ULL, 0x3ffffffa9bb93903ULL, 0x3ffffffba88a0a10ULL, 0x2fffffffffa3ba13ULL,
    0x3ffffff8b99b1b21ULL, 0x4fff9b2921b93903ULL, 0x2fffffffffb08b20ULL, 0x1ffffffffffffb23ULL,
    0x3ffffff98aa82832ULL, 0x2fffffffff2902a9ULL, 0x4fff8a1810a82832ULL, 0x1ffffffffffff2a1ULL,
    0x2fffffffff819831ULL, 0x1ffffffffffff190ULL, 0x1ffffffffffff830ULL, 0x0fffffffffffffffULL,
};

// Edge e runs from corner lower(e) to upper(e) along +axis(e).
__constant__ unsigned char c_elo[12] = {0, 1, 3, 0, 4, 5, 7, 4, 0, 1, 2, 3};
__constant__ unsigned char c_eup[12] = {1, 2, 2, 3, 5, 6, 6, 7, 4, 5, 6, 7};
__constant__ unsigned char c_eax[12] = {0, 1, 0, 1, 0, 1, 0, 1, 2, 2, 2, 2};

__device__ __forceinline__ int cdx(int c) { return ((c + 1) >> 1) & 1; }
__device__ __forceinline__ int cdy(int c) { return (c >> 1) & 1; }
__device__ __forceinline__ int cdz(int c) { return c >> 2; }

__device__ __forceinline__ unsigned edge_mask(unsigned cs) {
    unsigned m = 0;
#pragma unroll
    for (int e = 0; e < 12; ++e)
        m |= (((cs >> c_elo[e]) ^ (cs >> c_eup[e])) & 1u) << e;
    return m;
}

struct MeshCtr {
    int lo[3], hi[3];
    unsigned long long kept, cells, vvox;
};

struct CellRec {
    int vid[8];
};

template <class TD>
struct MeshArgs {
    const int4* table;
    int64_t hmask;
    const int4* bcoord;
    const unsigned long long* bslot;
    const TD* vt;
    double minw;
    double h;
};

// vid of a kept voxel at (x, y, z), or -1.
template <class TD>
__device__ __forceinline__ int kept_vid(const MeshArgs<TD>& a, int x, int y, int z) {
    const int leaf = hash_find(a.table, a.hmask, x >> 3, y >> 3, z >> 3);
    if (leaf < 0) return -1;
    const unsigned long long b =
        a.bslot[(int64_t)leaf * kLeafVolume + (((x & 7) << 6) | ((y & 7) << 3) | (z & 7))];
    const int vid = (int)(unsigned)b;
    if (vid < 0) return -1;
    return (double)a.vt[2 * (int64_t)vid + 1] >= a.minw ? vid : -1;
}

__device__ __forceinline__ unsigned long long pack_rel(int x, int y, int z, const MeshCtr& c) {
    return ((unsigned long long)(unsigned)(x - c.lo[0]) << (2 * kPackBits)) |
           ((unsigned long long)(unsigned)(y - c.lo[1]) << kPackBits) |
           (unsigned long long)(unsigned)(z - c.lo[2]);
}

// Kept-voxel bounds (mesh.py:459-467).
template <class TD>
__global__ void k_mesh_bounds(int64_t nslots, MeshArgs<TD> a, MeshCtr* ctr) {
    int lo[3] = {INT_MAX, INT_MAX, INT_MAX}, hi[3] = {INT_MIN, INT_MIN, INT_MIN};
    unsigned kept = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nslots;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int vid = (int)(unsigned)a.bslot[i];
        if (vid < 0 || !((double)a.vt[2 * (int64_t)vid + 1] >= a.minw)) continue;
        const int4 lc = a.bcoord[i >> 9];
        const int s = (int)(i & 511);
        const int v[3] = {lc.x * 8 + (s >> 6), lc.y * 8 + ((s >> 3) & 7), lc.z * 8 + (s & 7)};
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            lo[k] = min(lo[k], v[k]);
            hi[k] = max(hi[k], v[k]);
        }
        ++kept;
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        for (int o = 16; o; o >>= 1) {
            lo[k] = min(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
            hi[k] = max(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
        }
    }
    for (int o = 16; o; o >>= 1) kept += __shfl_xor_sync(0xffffffffu, kept, o);
    if ((threadIdx.x & 31) == 0 && kept) {
        for (int k = 0; k < 3; ++k) {
            atomicMin(&ctr->lo[k], lo[k]);
            atomicMax(&ctr->hi[k], hi[k]);
        }
        atomicAdd(&ctr->kept, (unsigned long long)kept);
    }
}

__device__ __forceinline__ void vertex_pos(int x, int y, int z, int axis, double dlo, double dhi,
                                           double h, double* p) {
    const double t = dlo / (dlo - dhi);
    p[0] = ((double)x + 0.5) * h;
    p[1] = ((double)y + 0.5) * h;
    p[2] = ((double)z + 0.5) * h;
    p[axis] += t * h;
}

// Live cells (mesh.py:469-490) with their surviving triangles (:503-525):
// one thread per anchor slot; records of cells with >= 1 surviving triangle
// are appended unordered and sorted by key afterwards.  Marks, per voxel,
// the axes of the vertices surviving triangles use.
template <class TD>
__global__ void k_mesh_cells(int64_t nslots, MeshArgs<TD> a, MeshCtr* ctr,
                             unsigned long long* __restrict__ ckey, int* __restrict__ cidx,
                             CellRec* __restrict__ rec, unsigned* __restrict__ cmeta,
                             unsigned* __restrict__ vmask) {
    __shared__ MeshCtr sc;
    if (threadIdx.x == 0) sc = *ctr;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nslots;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int v0 = (int)(unsigned)a.bslot[i];
        if (v0 < 0 || !((double)a.vt[2 * (int64_t)v0 + 1] >= a.minw)) continue;
        const int4 lc = a.bcoord[i >> 9];
        const int s = (int)(i & 511);
        const int x = lc.x * 8 + (s >> 6), y = lc.y * 8 + ((s >> 3) & 7), z = lc.z * 8 + (s & 7);
        CellRec r;
        r.vid[0] = v0;
        bool full = true;
        for (int c = 1; c < 8 && full; ++c) {
            r.vid[c] = kept_vid(a, x + cdx(c), y + cdy(c), z + cdz(c));
            full = r.vid[c] >= 0;
        }
        if (!full) continue;
        double d[8];
        unsigned cs = 0;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            d[c] = (double)a.vt[2 * (int64_t)r.vid[c]];
            cs |= (d[c] < 0.0 ? 1u : 0u) << c;
        }
        const unsigned em = edge_mask(cs);
        if (!em) continue;
        double p[12][3];
#pragma unroll
        for (int e = 0; e < 12; ++e) {
            if (!((em >> e) & 1)) continue;
            const int cl = c_elo[e];
            vertex_pos(x + cdx(cl), y + cdy(cl), z + cdz(cl), c_eax[e], d[cl], d[c_eup[e]], a.h, p[e]);
        }
        const unsigned long long tt = c_tri[cs];
        const int nt = (int)(tt >> 60);
        unsigned surv = 0;
        for (int j = 0; j < nt; ++j) {
            const int e0 = (int)((tt >> (12 * j)) & 15), e1 = (int)((tt >> (12 * j + 4)) & 15),
                      e2 = (int)((tt >> (12 * j + 8)) & 15);
            // reversed winding: triangle (e2, e1, e0)
            const double* q0 = p[e2];
            const double* q1 = p[e1];
            const double* q2 = p[e0];
            const double a0 = q1[0] - q0[0], a1 = q1[1] - q0[1], a2 = q1[2] - q0[2];
            const double b0 = q2[0] - q0[0], b1 = q2[1] - q0[1], b2 = q2[2] - q0[2];
            const double c0 = a1 * b2 - a2 * b1;
            const double c1 = a2 * b0 - a0 * b2;
            const double c2 = a0 * b1 - a1 * b0;
            const double area2 = (c0 * c0 + c1 * c1) + c2 * c2;
            if (area2 > 0.0) surv |= 1u << j;
        }
        if (!surv) continue;
        for (int j = 0; j < nt; ++j) {
            if (!((surv >> j) & 1)) continue;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const int e = (int)((tt >> (12 * j + 4 * q)) & 15);
                atomicOr(&vmask[r.vid[c_elo[e]]], 1u << c_eax[e]);
            }
        }
        const unsigned long long slot = atomicAdd(&ctr->cells, 1ULL);
        ckey[slot] = pack_rel(x, y, z, sc);
        cidx[slot] = (int)slot;
        rec[slot] = r;
        cmeta[slot] = cs | (surv << 8);
    }
}

__global__ void k_mesh_tricount(int64_t n, const int* __restrict__ order,
                                const unsigned* __restrict__ cmeta, int* __restrict__ cnt) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) cnt[i] = __popc(cmeta[order[i]] >> 8);
}

// Voxels owning at least one vertex, keyed spatially.
__global__ void k_mesh_vvox(int64_t nslots, const int4* __restrict__ bcoord,
                            const unsigned long long* __restrict__ bslot,
                            const unsigned* __restrict__ vmask, MeshCtr* ctr,
                            unsigned long long* __restrict__ vkey, int* __restrict__ vvid) {
    __shared__ MeshCtr sc;
    if (threadIdx.x == 0) sc = *ctr;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nslots;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int vid = (int)(unsigned)bslot[i];
        if (vid < 0 || !vmask[vid]) continue;
        const int4 lc = bcoord[i >> 9];
        const int s = (int)(i & 511);
        const unsigned long long slot = atomicAdd(&ctr->vvox, 1ULL);
        vkey[slot] = pack_rel(lc.x * 8 + (s >> 6), lc.y * 8 + ((s >> 3) & 7), lc.z * 8 + (s & 7), sc);
        vvid[slot] = vid;
    }
}

__global__ void k_mesh_vcount(int64_t n, const int* __restrict__ vvid,
                              const unsigned* __restrict__ vmask, int* __restrict__ cnt) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) cnt[i] = __popc(vmask[vvid[i]]);
}

__global__ void k_mesh_vbase(int64_t n, const int* __restrict__ vvid, const int* __restrict__ base,
                             int* __restrict__ vidx) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) vidx[vvid[i]] = base[i];
}

// Per-voxel label (voxel_labels, mesh.py:392-416) of the semantic state.
template <class TS>
__device__ int argmax_label(const TS* row, int P, bool open) {
    int arg = 0;
    double best = (double)row[0];
    double tot = 0.0;
    for (int c = 0; c < P; ++c) {
        const double v = (double)row[c];
        if (v != v) {           // numpy argmax stops at the first NaN
            arg = c;
            best = v;
            tot = v;
            break;
        }
        if (v > best) {
            best = v;
            arg = c;
        }
        tot += open ? fabs(v) : v;
    }
    if (open) return tot == 0.0 ? 0 : arg + 1;    // |mean| sums to zero -> unknown
    return tot <= 0.0 ? 0 : arg + 1;              // no counts -> unknown
}

template <class TD, class TS>
__global__ void k_mesh_verts(int64_t n, MeshArgs<TD> a, const MeshCtr* __restrict__ ctr,
                             const unsigned long long* __restrict__ vkey,
                             const int* __restrict__ vvid, const int* __restrict__ base,
                             const unsigned* __restrict__ vmask, int sem_kind, int P,
                             const TS* __restrict__ s0, const int* __restrict__ vlab,
                             double* __restrict__ verts, int* __restrict__ labels) {
    __shared__ MeshCtr sc;
    if (threadIdx.x == 0) sc = *ctr;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long k = vkey[i];
        const int x = sc.lo[0] + (int)(k >> (2 * kPackBits));
        const int y = sc.lo[1] + (int)((k >> kPackBits) & kPackMask);
        const int z = sc.lo[2] + (int)(k & kPackMask);
        const int vid = vvid[i];
        const unsigned msk = vmask[vid];
        const double dlo = (double)a.vt[2 * (int64_t)vid];
        int out = base[i];
        for (int ax = 0; ax < 3; ++ax) {
            if (!((msk >> ax) & 1)) continue;
            const int up = kept_vid(a, x + (ax == 0), y + (ax == 1), z + (ax == 2));
            const double dhi = (double)a.vt[2 * (int64_t)up];
            double p[3];
            vertex_pos(x, y, z, ax, dlo, dhi, a.h, p);
            verts[3 * (int64_t)out] = p[0];
            verts[3 * (int64_t)out + 1] = p[1];
            verts[3 * (int64_t)out + 2] = p[2];
            const double t = dlo / (dlo - dhi);
            const int near = t < 0.5 ? vid : up;
            int lab = 0;
            if (vlab) lab = vlab[near];
            else if (sem_kind == SVX_SEM_CLOSED) lab = argmax_label(s0 + (int64_t)near * P, P, false);
            else if (sem_kind == SVX_SEM_OPEN) lab = argmax_label(s0 + (int64_t)near * P, P, true);
            labels[out] = lab;
            ++out;
        }
    }
}

__device__ __forceinline__ int vertex_index(const CellRec& r, int e, const int* __restrict__ vidx,
                                            const unsigned* __restrict__ vmask) {
    const int v = r.vid[c_elo[e]];
    return vidx[v] + __popc(vmask[v] & ((1u << c_eax[e]) - 1u));
}

__global__ void k_mesh_tris(int64_t n, const int* __restrict__ order, const CellRec* __restrict__ rec,
                            const unsigned* __restrict__ cmeta, const int* __restrict__ toff,
                            const int* __restrict__ vidx, const unsigned* __restrict__ vmask,
                            int* __restrict__ tris) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int c = order[i];
        const CellRec r = rec[c];
        const unsigned meta = cmeta[c];
        const unsigned long long tt = c_tri[meta & 255];
        const unsigned surv = meta >> 8;
        int o = toff[i];
        for (int j = 0; j < 5; ++j) {
            if (!((surv >> j) & 1)) continue;
            const int e0 = (int)((tt >> (12 * j)) & 15), e1 = (int)((tt >> (12 * j + 4)) & 15),
                      e2 = (int)((tt >> (12 * j + 8)) & 15);
            tris[3 * (int64_t)o] = vertex_index(r, e2, vidx, vmask);
            tris[3 * (int64_t)o + 1] = vertex_index(r, e1, vidx, vmask);
            tris[3 * (int64_t)o + 2] = vertex_index(r, e0, vidx, vmask);
            ++o;
        }
    }
}

__global__ void k_mesh_scatter_labels(int64_t n, const int* __restrict__ act_vid,
                                      const int* __restrict__ lab, int* __restrict__ vlab) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) vlab[act_vid[i]] = lab[i];
}

__global__ void k_mesh_colors(int64_t n, const int* __restrict__ labels,
                              const unsigned char* __restrict__ pal, int npal,
                              unsigned char* __restrict__ colors) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const long long l = labels[i];
    const long long row = l > 0 ? 1 + (l - 1) % (npal - 1) : 0;
    colors[3 * i] = pal[3 * row];
    colors[3 * i + 1] = pal[3 * row + 1];
    colors[3 * i + 2] = pal[3 * row + 2];
}

template <class K>
svx_status sort_pairs(svx_map* m, const K* k0, K* k1, const int* v0, int* v1, int64_t n, int bits,
                      cudaStream_t s) {
    size_t tmp = 0;
    SVX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k0, k1, v0, v1, (int)n, 0, bits, s));
    SVX_TRY(ensure(m->cubtmp, tmp, s));
    SVX_CUDA(cub::DeviceRadixSort::SortPairs(m->cubtmp.p, tmp, k0, k1, v0, v1, (int)n, 0, bits, s));
    count_launch();
    return SVX_OK;
}

svx_status exclusive_sum(svx_map* m, const int* in, int* out, int64_t n, cudaStream_t s) {
    size_t tmp = 0;
    SVX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, (int)n, s));
    SVX_TRY(ensure(m->cubtmp, tmp, s));
    SVX_CUDA(cub::DeviceScan::ExclusiveSum(m->cubtmp.p, tmp, in, out, (int)n, s));
    count_launch();
    return SVX_OK;
}

svx_status read_ctr(svx_map* m, MeshCtr* h, cudaStream_t s) {
    SVX_CUDA(cudaMemcpyAsync(h, m->mesh_ctr.p, sizeof(MeshCtr), cudaMemcpyDeviceToHost, s));
    SVX_CUDA(cudaStreamSynchronize(s));
    return SVX_OK;
}

int last_of(svx_map* m, const int* cnt, const int* off, int64_t n, cudaStream_t s, svx_status* st) {
    int a = 0, b = 0;
    cudaError_t e = cudaMemcpyAsync(&a, cnt + n - 1, 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&b, off + n - 1, 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    *st = e == cudaSuccess ? SVX_OK : fail(SVX_E_CUDA, cudaGetErrorString(e));
    (void)m;
    return a + b;
}

template <class TD, class TS>
svx_status mesh_t(svx_map* m, double min_weight, const int* vlab, cudaStream_t s) {
    m->mesh_nv = m->mesh_nt = 0;
    const int64_t nslots = m->nblocks * kLeafVolume;
    if (nslots == 0) return SVX_OK;
    MeshArgs<TD> a{ptr<int4>(m->hash), m->hcap - 1, ptr<int4>(m->bcoord),
                   ptr<unsigned long long>(m->bslot), ptr<TD>(m->vt), min_weight, m->cfg.voxel_size};
    MeshCtr h;
    for (int k = 0; k < 3; ++k) {
        h.lo[k] = INT_MAX;
        h.hi[k] = INT_MIN;
    }
    h.kept = h.cells = h.vvox = 0;
    SVX_TRY(ensure(m->mesh_ctr, sizeof(MeshCtr), s));
    SVX_CUDA(cudaMemcpyAsync(m->mesh_ctr.p, &h, sizeof(h), cudaMemcpyHostToDevice, s));
    MeshCtr* dctr = ptr<MeshCtr>(m->mesh_ctr);
    const int T = 256;
    const int G = (int)std::min<int64_t>((nslots + T - 1) / T, kPersistentBlocks);
    k_mesh_bounds<TD><<<G, T, 0, s>>>(nslots, a, dctr);
    SVX_LAUNCHED();
    SVX_TRY(read_ctr(m, &h, s));
    if (h.kept == 0) return SVX_OK;
    long long ext[3];
    for (int k = 0; k < 3; ++k) ext[k] = (long long)h.hi[k] - h.lo[k] + 2;
    if (std::max(ext[0], std::max(ext[1], ext[2])) > (1LL << kPackBits))
        return fail(SVX_E_RANGE, "grid extent [" + std::to_string(ext[0]) + ", " + std::to_string(ext[1]) +
                                     ", " + std::to_string(ext[2]) + "] voxels exceeds the " +
                                     std::to_string(1LL << kPackBits) +
                                     "-per-axis mesh extraction limit");
    const int64_t nk = (int64_t)h.kept;
    SVX_TRY(ensure(m->mesh_k0, 8 * nk, s));
    SVX_TRY(ensure(m->mesh_k1, 8 * nk, s));
    SVX_TRY(ensure(m->mesh_i0, 4 * nk, s));
    SVX_TRY(ensure(m->mesh_i1, 4 * nk, s));
    SVX_TRY(ensure(m->mesh_rec, sizeof(CellRec) * nk, s));
    SVX_TRY(ensure(m->mesh_meta, 4 * nk, s));
    SVX_TRY(ensure(m->mesh_vmask, 4 * std::max<int64_t>(m->nvox, 1), s));
    SVX_CUDA(cudaMemsetAsync(m->mesh_vmask.p, 0, 4 * m->nvox, s));
    k_mesh_cells<TD><<<G, T, 0, s>>>(nslots, a, dctr, ptr<unsigned long long>(m->mesh_k0),
                                     ptr<int>(m->mesh_i0), ptr<CellRec>(m->mesh_rec),
                                     ptr<unsigned>(m->mesh_meta), ptr<unsigned>(m->mesh_vmask));
    SVX_LAUNCHED();
    SVX_TRY(read_ctr(m, &h, s));
    const int64_t nc = (int64_t)h.cells;
    if (nc == 0) return SVX_OK;
    // cells in spatial order; triangle offsets
    SVX_TRY(sort_pairs(m, ptr<unsigned long long>(m->mesh_k0), ptr<unsigned long long>(m->mesh_k1),
                       ptr<int>(m->mesh_i0), ptr<int>(m->mesh_i1), nc, 3 * kPackBits, s));
    const int* corder = ptr<int>(m->mesh_i1);
    SVX_TRY(ensure(m->mesh_cnt, 4 * nc, s));
    SVX_TRY(ensure(m->mesh_off, 4 * nc, s));
    k_mesh_tricount<<<grid_for(nc, T), T, 0, s>>>(nc, corder, ptr<unsigned>(m->mesh_meta),
                                                  ptr<int>(m->mesh_cnt));
    SVX_LAUNCHED();
    SVX_TRY(exclusive_sum(m, ptr<int>(m->mesh_cnt), ptr<int>(m->mesh_off), nc, s));
    svx_status st = SVX_OK;
    const int64_t nt = last_of(m, ptr<int>(m->mesh_cnt), ptr<int>(m->mesh_off), nc, s, &st);
    if (st) return st;
    SVX_TRY(ensure(m->mesh_toff, 4 * nc, s));
    SVX_CUDA(cudaMemcpyAsync(m->mesh_toff.p, m->mesh_off.p, 4 * nc, cudaMemcpyDeviceToDevice, s));
    // vertex-owning voxels in spatial order; vertex numbering
    k_mesh_vvox<<<G, T, 0, s>>>(nslots, ptr<int4>(m->bcoord), ptr<unsigned long long>(m->bslot),
                                ptr<unsigned>(m->mesh_vmask), dctr, ptr<unsigned long long>(m->mesh_k0),
                                ptr<int>(m->mesh_i0));
    SVX_LAUNCHED();
    SVX_TRY(read_ctr(m, &h, s));
    const int64_t nvv = (int64_t)h.vvox;
    SVX_TRY(ensure(m->mesh_vk, 8 * nvv, s));
    SVX_TRY(ensure(m->mesh_vv, 4 * nvv, s));
    SVX_TRY(sort_pairs(m, ptr<unsigned long long>(m->mesh_k0), ptr<unsigned long long>(m->mesh_vk),
                       ptr<int>(m->mesh_i0), ptr<int>(m->mesh_vv), nvv, 3 * kPackBits, s));
    SVX_TRY(ensure(m->mesh_cnt, 4 * std::max(nc, nvv), s));
    SVX_TRY(ensure(m->mesh_off, 4 * std::max(nc, nvv), s));
    k_mesh_vcount<<<grid_for(nvv, T), T, 0, s>>>(nvv, ptr<int>(m->mesh_vv), ptr<unsigned>(m->mesh_vmask),
                                                 ptr<int>(m->mesh_cnt));
    SVX_LAUNCHED();
    SVX_TRY(exclusive_sum(m, ptr<int>(m->mesh_cnt), ptr<int>(m->mesh_off), nvv, s));
    const int64_t nv = last_of(m, ptr<int>(m->mesh_cnt), ptr<int>(m->mesh_off), nvv, s, &st);
    if (st) return st;
    SVX_TRY(ensure(m->mesh_vidx, 4 * std::max<int64_t>(m->nvox, 1), s));
    k_mesh_vbase<<<grid_for(nvv, T), T, 0, s>>>(nvv, ptr<int>(m->mesh_vv), ptr<int>(m->mesh_off),
                                                ptr<int>(m->mesh_vidx));
    SVX_LAUNCHED();
    // outputs
    SVX_TRY(ensure(m->mesh_v, 24 * nv, s));
    SVX_TRY(ensure(m->mesh_l, 4 * nv, s));
    SVX_TRY(ensure(m->mesh_t, 12 * nt, s));
    const int Gv = (int)std::min<int64_t>((nvv + T - 1) / T, kPersistentBlocks);
    k_mesh_verts<TD, TS><<<Gv, T, 0, s>>>(nvv, a, dctr, ptr<unsigned long long>(m->mesh_vk),
                                          ptr<int>(m->mesh_vv), ptr<int>(m->mesh_off),
                                          ptr<unsigned>(m->mesh_vmask), m->cfg.sem_kind, m->payload_d,
                                          ptr<TS>(m->s0), vlab, ptr<double>(m->mesh_v),
                                          ptr<int>(m->mesh_l));
    SVX_LAUNCHED();
    const int Gt = (int)std::min<int64_t>((nc + T - 1) / T, kPersistentBlocks);
    k_mesh_tris<<<Gt, T, 0, s>>>(nc, corder, ptr<CellRec>(m->mesh_rec), ptr<unsigned>(m->mesh_meta),
                                 ptr<int>(m->mesh_toff), ptr<int>(m->mesh_vidx),
                                 ptr<unsigned>(m->mesh_vmask), ptr<int>(m->mesh_t));
    SVX_LAUNCHED();
    SVX_CUDA(cudaStreamSynchronize(s));
    m->mesh_nv = nv;
    m->mesh_nt = nt;
    return SVX_OK;
}

}  // namespace

svx_status scatter_active_labels(svx_map* m, int64_t count, const int* labels, int* vlab, cudaStream_t s) {
    if (count == 0) return SVX_OK;
    k_mesh_scatter_labels<<<grid_for(count, 256), 256, 0, s>>>(count, ptr<int>(m->act_vid), labels, vlab);
    SVX_LAUNCHED();
    return SVX_OK;
}

svx_status mesh_impl(svx_map* m, double min_weight, const int* vlab, cudaStream_t s) {
    const bool t64 = m->cfg.tsdf_dtype == SVX_F64;
    const bool s64 = m->cfg.sem_kind == SVX_SEM_CLOSED ? m->cfg.count_dtype == SVX_F64
                                                        : m->cfg.state_dtype == SVX_F64;
    if (t64 && s64) return mesh_t<double, double>(m, min_weight, vlab, s);
    if (t64) return mesh_t<double, float>(m, min_weight, vlab, s);
    if (s64) return mesh_t<float, double>(m, min_weight, vlab, s);
    return mesh_t<float, float>(m, min_weight, vlab, s);
}

svx_status mesh_colors(svx_map* m, const unsigned char* pal, int npal, unsigned char* colors,
                       cudaStream_t s) {
    if (m->mesh_nv == 0) return SVX_OK;
    k_mesh_colors<<<grid_for(m->mesh_nv, 256), 256, 0, s>>>(m->mesh_nv, ptr<int>(m->mesh_l), pal, npal,
                                                           colors);
    SVX_LAUNCHED();
    return SVX_OK;
}

}  // namespace svx

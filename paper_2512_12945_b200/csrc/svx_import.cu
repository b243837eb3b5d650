// svx_import.cu -- load a snapshot's map state into an empty device map
// (Mapper.load / load_grid; the reference reads its .slvg blocks in
// grid.py:372-426).  Leaves keep the snapshot's order as their ids, so the
// reference's allocation order (and with it the active order) carries over;
// they get creation stamp (frame 0, key = index) and the map's frame counter
// moves to 1, so leaves of later frames sort after them.
#include <cuda_runtime.h>
#include <string.h>

#include "svx_internal.cuh"

namespace svx {
namespace {

// Inputs come from a file: leaves out of the addressable range or given
// twice, voxels with a bad leaf index or slot, or a slot given twice set
// *err (the caller then clears what was written).
constexpr int kLeafCoordLimit = (1 << 30) >> kLeafLog2;

__global__ void k_import_leaves(int64_t nl, const int32_t* __restrict__ lc, int4* table, int64_t hmask,
                                int4* bcoord, unsigned long long* bkey, int* err) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nl;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int a = lc[3 * i], b = lc[3 * i + 1], c = lc[3 * i + 2];
        if (a <= -kLeafCoordLimit || a >= kLeafCoordLimit || b <= -kLeafCoordLimit ||
            b >= kLeafCoordLimit || c <= -kLeafCoordLimit || c >= kLeafCoordLimit) {
            atomicOr(err, 1);
            continue;
        }
        bcoord[i] = make_int4(a, b, c, 0);
        bkey[i] = (unsigned long long)i;
        int64_t pos = (int64_t)(block_hash(a, b, c) & (uint64_t)hmask);
        while (true) {
            const int old = atomicCAS(&table[pos].w, kHashEmpty, kHashBusy);
            if (old == kHashEmpty) {
                table[pos] = make_int4(a, b, c, (int)i);
                break;
            }
            // an occupied slot: a duplicate leaf if it holds the same key
            volatile int* vw = &table[pos].w;
            while (*vw == kHashBusy) {
            }
            volatile int* sp = reinterpret_cast<volatile int*>(table + pos);
            if (sp[0] == a && sp[1] == b && sp[2] == c) {
                atomicOr(err, 1);
                break;
            }
            pos = (pos + 1) & hmask;
        }
    }
}

template <class TD>
__global__ void k_import_voxels(int64_t nv, int64_t nl, const int32_t* __restrict__ vl,
                                const int32_t* __restrict__ vs, const double* __restrict__ d,
                                const double* __restrict__ w, unsigned long long* bslot,
                                unsigned long long* bmask, TD* vt, int* err) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv;
         v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t leaf = vl[v];
        const int slot = vs[v];
        if (leaf < 0 || leaf >= nl || slot < 0 || slot >= kLeafVolume ||
            atomicCAS(&bslot[leaf * kLeafVolume + slot], kSlotInactive, (unsigned long long)(unsigned)v) !=
                kSlotInactive) {
            atomicOr(err, 1);
            continue;
        }
        atomicOr(&bmask[leaf * kMaskWords + (slot >> 6)], 1ULL << (slot & 63));
        vt[2 * v] = (TD)d[v];
        vt[2 * v + 1] = (TD)w[v];
    }
}

}  // namespace

svx_status import_impl(svx_map* m, int64_t nl, const int32_t* leaf_coords, int64_t nv,
                       const int32_t* voxel_leaf, const int32_t* voxel_slot, const double* d,
                       const double* w, const void* sem0, const void* sem1, cudaStream_t s) {
    if (m->nblocks || m->nvox || m->frames)
        return fail(SVX_E_INPUT, "snapshots load into an empty map only");
    if (nl < 0 || nv < 0) return fail(SVX_E_INPUT, "negative snapshot sizes");
    if (nv == 0) return SVX_OK;
    SVX_TRY(reserve_blocks(m, nl, s));
    SVX_TRY(reserve_voxels(m, nv, s));
    const size_t se = sem_elem(m);
    const size_t row = se * (size_t)m->payload_d;
    DevBuf st_lc, st_vl, st_vs, st_d, st_w;
    const void *lc, *vl, *vs, *dd, *ww;
    svx_status st = SVX_OK;
    if ((st = stage_in(leaf_coords, 12 * (size_t)nl, st_lc, s, &lc)) ||
        (st = stage_in(voxel_leaf, 4 * (size_t)nv, st_vl, s, &vl)) ||
        (st = stage_in(voxel_slot, 4 * (size_t)nv, st_vs, s, &vs)) ||
        (st = stage_in(d, 8 * (size_t)nv, st_d, s, &dd)) ||
        (st = stage_in(w, 8 * (size_t)nv, st_w, s, &ww))) {
        release(st_lc); release(st_vl); release(st_vs); release(st_d); release(st_w);
        return st;
    }
    const int T = 256;
    int* derr = nullptr;
    cudaError_t e0 = cudaMallocAsync(&derr, sizeof(int), s);
    if (e0 == cudaSuccess) e0 = cudaMemsetAsync(derr, 0, sizeof(int), s);
    if (e0 != cudaSuccess) {
        release(st_lc); release(st_vl); release(st_vs); release(st_d); release(st_w);
        return fail(SVX_E_CUDA, std::string("snapshot import: ") + cudaGetErrorString(e0));
    }
    k_import_leaves<<<(int)std::min<int64_t>((nl + T - 1) / T, kPersistentBlocks), T, 0, s>>>(
        nl, (const int32_t*)lc, ptr<int4>(m->hash), m->hcap - 1, ptr<int4>(m->bcoord),
        ptr<unsigned long long>(m->bkey), derr);
    count_launch();
    const int g = (int)std::min<int64_t>((nv + T - 1) / T, kPersistentBlocks);
    if (m->cfg.tsdf_dtype == SVX_F64)
        k_import_voxels<double><<<g, T, 0, s>>>(nv, nl, (const int32_t*)vl, (const int32_t*)vs,
                                                (const double*)dd, (const double*)ww,
                                                ptr<unsigned long long>(m->bslot),
                                                ptr<unsigned long long>(m->bmask), ptr<double>(m->vt), derr);
    else
        k_import_voxels<float><<<g, T, 0, s>>>(nv, nl, (const int32_t*)vl, (const int32_t*)vs,
                                               (const double*)dd, (const double*)ww,
                                               ptr<unsigned long long>(m->bslot),
                                               ptr<unsigned long long>(m->bmask), ptr<float>(m->vt), derr);
    count_launch();
    int herr = 0;
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(&herr, derr, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFreeAsync(derr, s);
    if (e == cudaSuccess && herr) {
        // undo: an empty hash, inactive slots and clear masks for the leaves written
        cudaMemsetAsync(m->hash.p, 0xFF, sizeof(int4) * (size_t)m->hcap, s);
        cudaMemsetAsync(m->bmask.p, 0, sizeof(unsigned long long) * kMaskWords * (size_t)nl, s);
        launch_fill_u64(ptr<unsigned long long>(m->bslot), nl * kLeafVolume, kSlotInactive, s);
        cudaStreamSynchronize(s);
        release(st_lc); release(st_vl); release(st_vs); release(st_d); release(st_w);
        return fail(SVX_E_FORMAT, "snapshot: leaf out of range or repeated, or a voxel with a bad "
                                  "leaf/slot or repeated");
    }
    if (e == cudaSuccess && sem0 && row)
        e = cudaMemcpyAsync(m->s0.p, sem0, row * (size_t)nv, cudaMemcpyDefault, s);
    if (e == cudaSuccess && sem1 && row)
        e = cudaMemcpyAsync(m->s1.p, sem1, row * (size_t)nv, cudaMemcpyDefault, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    release(st_lc); release(st_vl); release(st_vs); release(st_d); release(st_w);
    if (e != cudaSuccess) return fail(SVX_E_CUDA, std::string("snapshot import: ") + cudaGetErrorString(e));
    m->nblocks = nl;
    m->nvox = nv;
    m->frames = 1;          // later frames' leaves sort after the snapshot's
    m->ord_nblocks = -1;
    m->act_valid_frames = -1;
    m->ctr_clean = false;
    return SVX_OK;
}

}  // namespace svx

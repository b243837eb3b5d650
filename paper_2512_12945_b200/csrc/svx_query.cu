// svx_query.cu -- voxel and label queries (K7, K8 v1).
//
// Active enumeration reproduces GridCore.active_slots (_core.pyx:424-444):
// leaves in the reference's allocation order, slots ascending.  The engine
// allocates leaf ids in arrival order during a frame and stamps every leaf
// with (creation frame, first-occurrence key); the reference's order is
// recovered here, off the integration path, by sorting each frame's new
// leaves by that stamp (ids of one frame are contiguous, so the order is
// extended incrementally).  Reads never allocate.
#include <math.h>

#include <cub/cub.cuh>

#include <cuda_pipeline.h>

#include "svx_internal.cuh"

namespace svx {
namespace {

__global__ void k_order_init(int64_t first, int64_t cnt, const int4* __restrict__ bcoord,
                             const unsigned long long* __restrict__ bkey,
                             unsigned long long* __restrict__ k0, unsigned* __restrict__ f0,
                             int* __restrict__ id0) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= cnt) return;
    k0[j] = bkey[first + j];
    id0[j] = (int)(first + j);
    (void)f0;
    (void)bcoord;
}

__global__ void k_order_frames(int64_t cnt, const int4* __restrict__ bcoord,
                               const int* __restrict__ ids, unsigned* __restrict__ f) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < cnt) f[j] = (unsigned)bcoord[ids[j]].w;
}

__global__ void k_popc(int64_t nblocks, const int* __restrict__ order,
                       const unsigned long long* __restrict__ bmask, int* __restrict__ cnt) {
    int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nblocks) return;
    const int64_t leaf = order[b];
    int c = 0;
#pragma unroll
    for (int w = 0; w < kMaskWords; ++w) c += __popcll(bmask[leaf * kMaskWords + w]);
    cnt[b] = c;
}

// Leaf stamps in active order (merge keys of a sharded map's active lists).
__global__ void k_leaf_stamps(int64_t nblocks, const int* __restrict__ order,
                              const int4* __restrict__ bcoord,
                              const unsigned long long* __restrict__ bkey,
                              const int* __restrict__ cnt, int32_t* __restrict__ frame,
                              uint64_t* __restrict__ key, int32_t* __restrict__ count) {
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nblocks) return;
    const int leaf = order[q];
    if (frame) frame[q] = bcoord[leaf].w;
    if (key) key[q] = bkey[leaf];
    if (count) count[q] = cnt[q];
}

// One warp per leaf: lanes cover 32 slots at a time, ballot/popc give ranks.
__global__ void k_list(int64_t nblocks, const int* __restrict__ order,
                       const unsigned long long* __restrict__ bmask,
                       const unsigned long long* __restrict__ bslot, const int4* __restrict__ bcoord,
                       const long long* __restrict__ off, int* __restrict__ act_vid,
                       long long* __restrict__ act_coord) {
    int64_t ob = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (ob >= nblocks) return;
    long long pos = off[ob];
    const int64_t b = order[ob];
    int4 bc = bcoord[b];
    for (int half = 0; half < 16; ++half) {
        unsigned long long word = bmask[b * kMaskWords + (half >> 1)];
        unsigned bits = (unsigned)(word >> (32 * (half & 1)));
        if (!bits) continue;
        if ((bits >> lane) & 1u) {
            int slot = half * 32 + lane;
            long long p = pos + __popc(bits & ((1u << lane) - 1u));
            act_vid[p] = (int)(unsigned)bslot[b * kLeafVolume + slot];
            act_coord[3 * p] = ((long long)bc.x << kLeafLog2) + ((slot >> 6) & 7);
            act_coord[3 * p + 1] = ((long long)bc.y << kLeafLog2) + ((slot >> 3) & 7);
            act_coord[3 * p + 2] = ((long long)bc.z << kLeafLog2) + (slot & 7);
        }
        pos += __popc(bits);
    }
}

template <class T>
__global__ void k_gather_rows(int64_t count, int width, int sstride, const int* __restrict__ act_vid,
                              const T* __restrict__ src, T* __restrict__ dst) {
    int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t total = count * width;
    for (; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = idx / width;
        int c = (int)(idx - i * width);
        dst[idx] = src[(int64_t)act_vid[i] * sstride + c];
    }
}

__global__ void k_copy_coords(int64_t count, const long long* __restrict__ src,
                              long long* __restrict__ dst) {
    int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx < 3 * count) dst[idx] = src[idx];
}

__global__ void k_probe_vid(int64_t cnt, const long long* __restrict__ coords,
                            const int4* __restrict__ table, int64_t mask,
                            const unsigned long long* __restrict__ bslot, int* __restrict__ vid_out,
                            uint8_t* __restrict__ active) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cnt) return;
    long long x = coords[3 * i], y = coords[3 * i + 1], z = coords[3 * i + 2];
    int blk = hash_find(table, mask, (int)(x >> kLeafLog2), (int)(y >> kLeafLog2),
                        (int)(z >> kLeafLog2));
    int vid = -1;
    if (blk >= 0) {
        int slot = (int)(((x & 7) << 6) | ((y & 7) << 3) | (z & 7));
        vid = (int)(unsigned)bslot[(int64_t)blk * kLeafVolume + slot];
    }
    vid_out[i] = vid;
    if (active) active[i] = vid >= 0;
}

template <class T>
__global__ void k_probe_rows(int64_t cnt, int width, int sstride, const int* __restrict__ vid,
                             const T* __restrict__ src, T bg, T* __restrict__ dst) {
    int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t total = cnt * width;
    for (; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = idx / width;
        int c = (int)(idx - i * width);
        int v = vid[i];
        dst[idx] = v >= 0 ? src[(int64_t)v * sstride + c] : bg;
    }
}

__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// cosine_to_embeddings (gaussian.py:158-170) against one query; one warp per voxel.
template <class TS>
__global__ void k_cosine(int64_t count, int D, const int* __restrict__ act_vid,
                         const TS* __restrict__ mean, const double* __restrict__ q, double qn,
                         double* __restrict__ sims) {
    int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (i >= count) return;
    const TS* row = mean + (int64_t)act_vid[i] * D;
    double dot = 0.0, nn = 0.0;
    for (int c = lane; c < D; c += 32) {
        double mv = (double)row[c];
        dot += mv * q[c];
        nn += mv * mv;
    }
    dot = warp_sum(dot);
    nn = warp_sum(nn);
    if (lane == 0) {
        double mn = sqrt(nn);
        sims[i] = mn == 0.0 ? NAN : dot / (mn * qn);
    }
}

// classify_means (gaussian.py:132-155), weights = TSDF weight.  One warp per
// voxel: similarities are warp-reduced dot products; lane (j % 32) caches
// similarity j (up to 32*kCache of them) for the softmax pass.
constexpr int kCache = 8;

template <class TS, class TD>
__global__ void k_classify(int64_t count, int D, int k, const int* __restrict__ act_vid,
                           const TS* __restrict__ mean, const TD* __restrict__ vw,
                           const double* __restrict__ emb, const double* __restrict__ en,
                           double tau, double tp, int32_t* __restrict__ labels,
                           double* __restrict__ best, double* __restrict__ sims_out) {
    int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (i >= count) return;
    const int vid = act_vid[i];
    const TS* row = mean + (int64_t)vid * D;
    double nn = 0.0;
    for (int c = lane; c < D; c += 32) {
        double mv = (double)row[c];
        nn += mv * mv;
    }
    nn = warp_sum(nn);
    const double mn = sqrt(nn);
    const double wgt = (double)vw[2 * (int64_t)vid + 1];   // {d, w} pairs
    const bool ok = mn != 0.0 && wgt > 0.0;
    double cache[kCache];
    double lmax = -INFINITY;
    for (int j = 0; j < k; ++j) {
        const double* e = emb + (int64_t)j * D;
        double dot = 0.0;
        for (int c = lane; c < D; c += 32) dot += (double)row[c] * e[c];
        dot = warp_sum(dot);
        double sj = mn == 0.0 ? NAN : dot / (mn * en[j]);
        if (sims_out && lane == 0) sims_out[i * k + j] = sj;
        if (lane == (j & 31) && (j >> 5) < kCache) cache[j >> 5] = sj;
        double lj = sj / tau;
        lmax = lj > lmax ? lj : lmax;
    }
    if (!ok) {
        if (lane == 0) { labels[i] = 0; best[i] = 0.0; }
        return;
    }
    // softmax: e_j = exp(l_j - lmax); label = first j attaining max e_j (np.argmax on probs)
    double den = 0.0;
    int arg = 0x7fffffff;
    double emax = -1.0;
    for (int j0 = 0; j0 < k; j0 += 32) {
        int j = j0 + lane;
        double ej = 0.0;
        if (j < k) {
            double sj;
            if ((j >> 5) < kCache) {
                sj = cache[j >> 5];
            } else {
                const double* e = emb + (int64_t)j * D;
                double dot = 0.0;
                for (int c = 0; c < D; ++c) dot += (double)row[c] * e[c];
                sj = dot / (mn * en[j]);
            }
            ej = exp(sj / tau - lmax);
            den += ej;
            if (ej > emax) { emax = ej; arg = j; }
        }
    }
    den = warp_sum(den);
    for (int o = 16; o > 0; o >>= 1) {
        double oe = __shfl_xor_sync(0xffffffffu, emax, o);
        int oa = __shfl_xor_sync(0xffffffffu, arg, o);
        if (oe > emax || (oe == emax && oa < arg)) { emax = oe; arg = oa; }
    }
    if (lane == 0) {
        double top = emax / den;
        labels[i] = top < tp ? 0 : arg + 1;
        best[i] = top;
    }
}

// classify_means (gaussian.py:132-155) on the FP64 tensor cores: one fused
// kernel computes S = M . E^T with mma.sync.m8n8k4.f64 (DMMA; B200 has no
// f64 kind of tcgen05) and applies the cosine normalisation, softmax, argmax
// and the label rules in the epilogue, straight from the accumulator
// fragments.  f64 end to end: the reference scores in f64 (means @ emb.T)
// and softmax(S / tau) with tau = 0.01 turns any score error e into a
// relative error e / tau, so a reduced-precision product cannot be used
// (DESIGN.md section 8).
//
// Tiling: a CTA = 4 warps; a warp owns MT m-tiles of 8 voxels and all NT
// n-tiles of 8 queries (k <= 8 NT), accumulators in registers (2 f64 per
// thread per tile).  The queries stream through shared memory in chunks of
// kDc dimensions; each thread feeds its A fragment (voxel row r = lane / 4,
// dim d0 + lane % 4) straight from global (f32 -> f64) and accumulates the
// row's squared norm on the way.
constexpr int kDc = 16;              // dims per shared-memory chunk

constexpr int kClsWarps = 4;

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

template <int NT, int MT, bool kStaged, class TS, class TD>
__global__ void __launch_bounds__(32 * kClsWarps) k_classify_dmma(
    int64_t count, int D, int k, const int* __restrict__ act_vid, const TS* __restrict__ mean,
    const TD* __restrict__ vw, const double* __restrict__ emb, const double* __restrict__ en,
    double tau, double tp, int32_t* __restrict__ labels, double* __restrict__ best,
    double* __restrict__ sims_out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int qr = lane >> 2, qc = lane & 3;   // fragment row / column group
    int64_t ri[MT];
    double acc[MT][NT][2];
    double nn[MT];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
        nn[mt] = 0.0;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
    }
    if constexpr (kStaged) {
    // both operands stream through a 2-stage shared-memory ring (cp.async):
    // the next chunk's voxel means and queries are in flight while this
    // chunk's DMMAs run
    constexpr int RA = kClsWarps * 8 * MT;   // voxel rows per CTA
    __shared__ TS s_a[2][RA][kDc + 1];
    __shared__ double s_b[2][NT * 8][kDc + 1];
    __shared__ int s_vid[RA];
    const int64_t cta0 = (int64_t)blockIdx.x * RA;
    for (int r = threadIdx.x; r < RA; r += blockDim.x)
        s_vid[r] = cta0 + r < count ? act_vid[cta0 + r] : -1;
    __syncthreads();
    const int64_t row0 = cta0 + warp * (8 * MT);
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) ri[mt] = row0 + mt * 8 + qr;
    const int nch = (D + kDc - 1) / kDc;
    auto issue = [&](int ch) {
        if (ch < nch) {
            const int st = ch & 1, d0 = ch * kDc;
            for (int t = threadIdx.x; t < RA * kDc; t += blockDim.x) {
                const int r = t / kDc, c = t % kDc;
                const int vid = s_vid[r];
                if (vid >= 0 && d0 + c < D)
                    __pipeline_memcpy_async(&s_a[st][r][c], mean + (int64_t)vid * D + d0 + c, sizeof(TS));
                else
                    s_a[st][r][c] = (TS)0;
            }
            for (int t = threadIdx.x; t < NT * 8 * kDc; t += blockDim.x) {
                const int j = t / kDc, c = t % kDc;
                if (j < k && d0 + c < D)
                    __pipeline_memcpy_async(&s_b[st][j][c], emb + (int64_t)j * D + d0 + c, sizeof(double));
                else
                    s_b[st][j][c] = 0.0;
            }
        }
        __pipeline_commit();
    };
    issue(0);
    for (int ch = 0; ch < nch; ++ch) {
        issue(ch + 1);   // into the buffer the previous iteration consumed
        __pipeline_wait_prior(1);
        __syncthreads();
        const int st = ch & 1;
#pragma unroll
        for (int kk = 0; kk < kDc; kk += 4) {
            double a[MT];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                a[mt] = (double)s_a[st][warp * 8 * MT + mt * 8 + qr][kk + qc];
                nn[mt] += a[mt] * a[mt];
            }
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                const double b = s_b[st][nt * 8 + qr][kk + qc];
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) dmma(acc[mt][nt], a[mt], b);
            }
        }
        __syncthreads();
    }
    __pipeline_wait_prior(0);
    } else {
    __shared__ double s_e[NT * 8][kDc + 1];   // +1: no bank conflicts on the B fragment reads
    const int64_t row0 = ((int64_t)blockIdx.x * kClsWarps + warp) * (8 * MT);
    const TS* rp[MT];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
        ri[mt] = row0 + mt * 8 + qr;
        rp[mt] = ri[mt] < count ? mean + (int64_t)act_vid[ri[mt]] * D : nullptr;
    }
    for (int d0 = 0; d0 < D; d0 += kDc) {
        __syncthreads();
        for (int t = threadIdx.x; t < NT * 8 * kDc; t += blockDim.x) {
            const int j = t / kDc, c = t % kDc;
            s_e[j][c] = (j < k && d0 + c < D) ? emb[(int64_t)j * D + d0 + c] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < kDc; kk += 4) {
            const int d = d0 + kk + qc;
            double a[MT];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                a[mt] = (rp[mt] && d < D) ? (double)rp[mt][d] : 0.0;
                nn[mt] += a[mt] * a[mt];
            }
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                const double b = s_e[nt * 8 + qr][kk + qc];
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) dmma(acc[mt][nt], a[mt], b);
            }
        }
    }
    }
    // epilogue: row qr of each m-tile lives in the 4 lanes of quad qr
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
        double n2 = nn[mt];
        n2 += __shfl_xor_sync(0xffffffffu, n2, 1);
        n2 += __shfl_xor_sync(0xffffffffu, n2, 2);
        const double mn = sqrt(n2);
        const bool live = ri[mt] < count;
        const int vid = live ? act_vid[ri[mt]] : 0;
        const double wgt = live ? (double)vw[2 * (int64_t)vid + 1] : 0.0;   // {d, w} pairs
        const bool ok = live && mn != 0.0 && wgt > 0.0;
        // e_j = (cos_j) / tau, as the reference computes it
        double lmax = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j = nt * 8 + qc * 2 + h;
                if (j < k) {
                    const double sj = mn == 0.0 ? NAN : acc[mt][nt][h] / (mn * en[j]);
                    if (sims_out && live) sims_out[ri[mt] * k + j] = sj;
                    const double ej = sj / tau;
                    acc[mt][nt][h] = ej;
                    lmax = ej > lmax ? ej : lmax;
                }
            }
        }
        lmax = fmax(lmax, __shfl_xor_sync(0xffffffffu, lmax, 1));
        lmax = fmax(lmax, __shfl_xor_sync(0xffffffffu, lmax, 2));
        double den = 0.0, emax = -1.0;
        int arg = 0x7fffffff;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j = nt * 8 + qc * 2 + h;
                if (j < k) {
                    const double ej = exp(acc[mt][nt][h] - lmax);
                    den += ej;
                    if (ej > emax) { emax = ej; arg = j; }
                }
            }
        }
        // quad reduction; first index attaining the max (np.argmax)
#pragma unroll
        for (int o = 1; o <= 2; o <<= 1) {
            den += __shfl_xor_sync(0xffffffffu, den, o);
            const double oe = __shfl_xor_sync(0xffffffffu, emax, o);
            const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
            if (oe > emax || (oe == emax && oa < arg)) { emax = oe; arg = oa; }
        }
        if (live && qc == 0) {
            if (!ok) {
                labels[ri[mt]] = 0;
                best[ri[mt]] = 0.0;
            } else {
                const double top = emax / den;
                labels[ri[mt]] = top < tp ? 0 : arg + 1;
                best[ri[mt]] = top;
            }
        }
    }
}

template <class TC>
__global__ void k_label_map(int64_t count, int C, int mode, const int* __restrict__ act_vid,
                            const TC* __restrict__ counts, int32_t* __restrict__ labels) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const TC* row = counts + (int64_t)act_vid[i] * C;
    TC bestv = row[0];
    int arg = 0;
    double total = (double)row[0];
    for (int c = 1; c < C; ++c) {
        TC v = row[c];
        total += (double)v;
        if (v > bestv) { bestv = v; arg = c; }
    }
    labels[i] = (mode == 1 && !(total > 0.0)) ? 0 : arg + 1;
}

}  // namespace

// Extend the leaf order with the leaves created since the last query: sort
// them by (creation frame, first-occurrence key) with two stable LSD passes.
static svx_status build_leaf_order(svx_map* m, cudaStream_t s) {
    const int64_t nb = m->nblocks;
    int64_t first = m->ord_nblocks < 0 ? 0 : m->ord_nblocks;
    SVX_TRY(ensure(m->ord0, sizeof(int) * nb, s, true));
    const int64_t cnt = nb - first;
    if (cnt <= 0) return SVX_OK;
    SVX_TRY(ensure(m->ordk0, 8 * cnt, s));
    SVX_TRY(ensure(m->ordk1, 8 * cnt, s));
    SVX_TRY(ensure(m->ordf0, 4 * cnt, s));
    SVX_TRY(ensure(m->ordf1, 4 * cnt, s));
    SVX_TRY(ensure(m->ord1, 4 * cnt, s));
    SVX_TRY(ensure(m->act_cnt, 4 * cnt, s));
    int* idA = ptr<int>(m->ord1);
    int* idB = ptr<int>(m->act_cnt);
    const int T = 256;
    k_order_init<<<grid_for(cnt, T), T, 0, s>>>(first, cnt, ptr<int4>(m->bcoord),
                                                ptr<unsigned long long>(m->bkey),
                                                ptr<unsigned long long>(m->ordk0),
                                                ptr<unsigned>(m->ordf0), idA);
    SVX_LAUNCHED();
    size_t tmp = 0;
    SVX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, ptr<unsigned long long>(m->ordk0),
                                             ptr<unsigned long long>(m->ordk1), idA, idB, (int)cnt,
                                             0, 64, s));
    SVX_TRY(ensure(m->cubtmp, tmp, s));
    SVX_CUDA(cub::DeviceRadixSort::SortPairs(m->cubtmp.p, tmp, ptr<unsigned long long>(m->ordk0),
                                             ptr<unsigned long long>(m->ordk1), idA, idB, (int)cnt,
                                             0, 64, s));
    count_launch();
    k_order_frames<<<grid_for(cnt, T), T, 0, s>>>(cnt, ptr<int4>(m->bcoord), idB,
                                                  ptr<unsigned>(m->ordf0));
    SVX_LAUNCHED();
    int* out = ptr<int>(m->ord0) + first;
    SVX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, ptr<unsigned>(m->ordf0),
                                             ptr<unsigned>(m->ordf1), idB, out, (int)cnt, 0, 32, s));
    SVX_TRY(ensure(m->cubtmp, tmp, s));
    SVX_CUDA(cub::DeviceRadixSort::SortPairs(m->cubtmp.p, tmp, ptr<unsigned>(m->ordf0),
                                             ptr<unsigned>(m->ordf1), idB, out, (int)cnt, 0, 32, s));
    count_launch();
    m->ord_nblocks = nb;
    return SVX_OK;
}

svx_status build_active_list(svx_map* m, int64_t* count, cudaStream_t s) {
    const int64_t nb = m->nblocks;
    *count = m->nvox;
    if (nb == 0 || m->nvox == 0) return SVX_OK;
    SVX_TRY(build_leaf_order(m, s));
    SVX_TRY(ensure(m->act_cnt, sizeof(int) * nb, s));
    SVX_TRY(ensure(m->act_off, sizeof(long long) * nb, s));
    SVX_TRY(ensure(m->act_vid, sizeof(int) * m->nvox, s));
    SVX_TRY(ensure(m->act_coord, sizeof(long long) * 3 * m->nvox, s));
    const int T = 256;
    const int* order = ptr<int>(m->ord0);
    k_popc<<<grid_for(nb, T), T, 0, s>>>(nb, order, ptr<unsigned long long>(m->bmask),
                                         ptr<int>(m->act_cnt));
    SVX_LAUNCHED();
    size_t tmp = 0;
    SVX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, ptr<int>(m->act_cnt),
                                           ptr<long long>(m->act_off), (int)nb, s));
    SVX_TRY(ensure(m->cubtmp, tmp, s));
    SVX_CUDA(cub::DeviceScan::ExclusiveSum(m->cubtmp.p, tmp, ptr<int>(m->act_cnt),
                                           ptr<long long>(m->act_off), (int)nb, s));
    count_launch();
    k_list<<<grid_for(nb * 32, T), T, 0, s>>>(nb, order, ptr<unsigned long long>(m->bmask),
                                             ptr<unsigned long long>(m->bslot), ptr<int4>(m->bcoord),
                                             ptr<long long>(m->act_off), ptr<int>(m->act_vid),
                                             ptr<long long>(m->act_coord));
    SVX_LAUNCHED();
    return SVX_OK;
}

svx_status launch_leaf_stamps(svx_map* m, int32_t* frame, uint64_t* key, int32_t* count,
                              cudaStream_t s) {
    const int64_t nb = m->nblocks;
    if (nb == 0 || m->nvox == 0) return SVX_OK;
    const int T = 256;
    k_leaf_stamps<<<grid_for(nb, T), T, 0, s>>>(nb, ptr<int>(m->ord0), ptr<int4>(m->bcoord),
                                               ptr<unsigned long long>(m->bkey),
                                               ptr<int>(m->act_cnt), frame, key, count);
    SVX_LAUNCHED();
    return SVX_OK;
}

// dst (count, width) <- rows vid * sstride + [0, width) of src; sstride < 0
// means sstride = width.  src_off selects a column of interleaved records.
template <class T>
static svx_status gather_rows(int64_t count, int width, const int* vid, const void* src, void* dst,
                              cudaStream_t s, int sstride = -1, int src_off = 0) {
    if (!dst || count == 0) return SVX_OK;
    int64_t total = count * width;
    int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 32);
    k_gather_rows<T><<<blocks, 256, 0, s>>>(count, width, sstride < 0 ? width : sstride, vid,
                                            (const T*)src + src_off, (T*)dst);
    SVX_LAUNCHED();
    return SVX_OK;
}

static svx_status gather_typed(int f64, int64_t count, int width, const int* vid, const void* src,
                               void* dst, cudaStream_t s, int sstride = -1, int src_off = 0) {
    return f64 ? gather_rows<double>(count, width, vid, src, dst, s, sstride, src_off)
               : gather_rows<float>(count, width, vid, src, dst, s, sstride, src_off);
}

svx_status launch_export(svx_map* m, int64_t count, int64_t* coords, void* d, void* w, void* sem0,
                         void* sem1, cudaStream_t s) {
    if (count == 0) return SVX_OK;
    const int* vid = ptr<int>(m->act_vid);
    if (coords) {
        k_copy_coords<<<grid_for(3 * count, 256), 256, 0, s>>>(count, ptr<long long>(m->act_coord),
                                                              (long long*)coords);
        SVX_LAUNCHED();
    }
    const int td64 = m->cfg.tsdf_dtype == SVX_F64;
    SVX_TRY(gather_typed(td64, count, 1, vid, m->vt.p, d, s, 2, 0));
    SVX_TRY(gather_typed(td64, count, 1, vid, m->vt.p, w, s, 2, 1));
    if (m->cfg.sem_kind == SVX_SEM_CLOSED) {
        SVX_TRY(gather_typed(m->cfg.count_dtype == SVX_F64, count, m->payload_d, vid, m->s0.p,
                             sem0, s));
    } else if (m->cfg.sem_kind == SVX_SEM_OPEN) {
        const int s64 = m->cfg.state_dtype == SVX_F64;
        SVX_TRY(gather_typed(s64, count, m->payload_d, vid, m->s0.p, sem0, s));
        SVX_TRY(gather_typed(s64, count, m->payload_d, vid, m->s1.p, sem1, s));
    }
    return SVX_OK;
}

template <class T>
static svx_status probe_rows(int64_t cnt, int width, const int* vid, const void* src, double bg,
                             void* dst, cudaStream_t s, int sstride = -1, int src_off = 0) {
    if (!dst || cnt == 0) return SVX_OK;
    int64_t total = cnt * width;
    int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 32);
    k_probe_rows<T><<<blocks, 256, 0, s>>>(cnt, width, sstride < 0 ? width : sstride, vid,
                                           (const T*)src + src_off, (T)bg, (T*)dst);
    SVX_LAUNCHED();
    return SVX_OK;
}

static svx_status probe_typed(int f64, int64_t cnt, int width, const int* vid, const void* src,
                              double bg, void* dst, cudaStream_t s, int sstride = -1,
                              int src_off = 0) {
    return f64 ? probe_rows<double>(cnt, width, vid, src, bg, dst, s, sstride, src_off)
               : probe_rows<float>(cnt, width, vid, src, bg, dst, s, sstride, src_off);
}

svx_status launch_probe(svx_map* m, const int64_t* coords, int64_t cnt, void* d, void* w,
                        void* sem0, void* sem1, uint8_t* active, cudaStream_t s) {
    if (cnt == 0) return SVX_OK;
    SVX_TRY(ensure(m->out_buf, sizeof(int) * cnt, s));
    int* vid = ptr<int>(m->out_buf);
    if (m->hcap == 0) {
        SVX_CUDA(cudaMemsetAsync(vid, 0xFF, sizeof(int) * cnt, s));
        if (active) SVX_CUDA(cudaMemsetAsync(active, 0, cnt, s));
    } else {
        k_probe_vid<<<grid_for(cnt, 256), 256, 0, s>>>(cnt, (const long long*)coords,
                                                       ptr<int4>(m->hash), m->hcap - 1,
                                                       ptr<unsigned long long>(m->bslot), vid, active);
        SVX_LAUNCHED();
    }
    const int td64 = m->cfg.tsdf_dtype == SVX_F64;
    SVX_TRY(probe_typed(td64, cnt, 1, vid, m->vt.p, m->cfg.truncation, d, s, 2, 0));
    SVX_TRY(probe_typed(td64, cnt, 1, vid, m->vt.p, 0.0, w, s, 2, 1));
    if (m->cfg.sem_kind == SVX_SEM_CLOSED) {
        SVX_TRY(probe_typed(m->cfg.count_dtype == SVX_F64, cnt, m->payload_d, vid, m->s0.p, 0.0,
                            sem0, s));
    } else if (m->cfg.sem_kind == SVX_SEM_OPEN) {
        const int s64 = m->cfg.state_dtype == SVX_F64;
        SVX_TRY(probe_typed(s64, cnt, m->payload_d, vid, m->s0.p, 0.0, sem0, s));
        SVX_TRY(probe_typed(s64, cnt, m->payload_d, vid, m->s1.p, m->cfg.prior_beta, sem1, s));
    }
    return SVX_OK;
}

svx_status launch_cosine(svx_map* m, int64_t count, const double* q, double qn, double* sims,
                         cudaStream_t s) {
    if (count == 0) return SVX_OK;
    const int T = 256;
    if (m->cfg.state_dtype == SVX_F64)
        k_cosine<double><<<grid_for(count * 32, T), T, 0, s>>>(
            count, m->payload_d, ptr<int>(m->act_vid), ptr<double>(m->s0), q, qn, sims);
    else
        k_cosine<float><<<grid_for(count * 32, T), T, 0, s>>>(
            count, m->payload_d, ptr<int>(m->act_vid), ptr<float>(m->s0), q, qn, sims);
    SVX_LAUNCHED();
    return SVX_OK;
}

template <int NT, int MT, bool kStaged, class TS, class TD>
static svx_status classify_dmma_t(svx_map* m, int64_t count, const double* emb, const double* en,
                                  int k, double tau, double tp, int32_t* labels, double* best,
                                  double* sims, cudaStream_t s) {
    const int64_t rows_per_cta = (int64_t)kClsWarps * 8 * MT;
    k_classify_dmma<NT, MT, kStaged, TS, TD><<<(unsigned)((count + rows_per_cta - 1) / rows_per_cta),
                                      32 * kClsWarps, 0, s>>>(
        count, m->payload_d, k, ptr<int>(m->act_vid), ptr<TS>(m->s0), ptr<TD>(m->vt), emb, en,
        tau, tp, labels, best, sims);
    SVX_LAUNCHED();
    return SVX_OK;
}

// SVX_SCORE_TC=0: keep classify on the FP64 DMMA kernel; SVX_SCORE_TC=1: the
// tcgen05 kernel for every k (A/B switches and the tests of both paths)
static const bool g_score_tc = !(getenv("SVX_SCORE_TC") && getenv("SVX_SCORE_TC")[0] == '0');
static const bool g_score_tc_force = getenv("SVX_SCORE_TC") && getenv("SVX_SCORE_TC")[0] == '1';

template <class TS, class TD>
static svx_status classify_t(svx_map* m, int64_t count, const double* emb, const double* en, int k,
                             double tau, double tp, int32_t* labels, double* best, double* sims,
                             cudaStream_t s) {
    // f32 means and more than 64 queries: the exact int8 split GEMM on
    // tcgen05 (svx_score.cu; cfg5, D = 768, k = 128: 9.4 ms vs 13.1 ms on the
    // DMMA kernel).  Up to 64 queries the DMMA kernel is faster (cfg3, k = 32:
    // 0.88 vs 1.26 ms): its tiles are issue-bound at N <= 32
    if constexpr (sizeof(TS) == 4)
        if (m->payload_d <= 1024 && k <= 4096 && m->score_path != 1 &&
            (m->score_path == 2 || g_score_tc_force || (g_score_tc && k > 64)))
            return classify_tc(m, count, ptr<int>(m->act_vid), emb, en, k, tau, tp, labels, best, sims, s);
    // FP64 tensor cores (DMMA) for up to 128 queries; the warp-per-voxel
    // CUDA-core kernel beyond
    // up to 64 queries: operands straight from global/L2 (measured best); 65..128:
    // both operands through a cp.async ring, two m-tiles per warp for f32 means
    // (cfg5, D = 768, k = 128: 29 % -> 49 % of the FP64 tensor peak)
    if (k <= 8) return classify_dmma_t<1, 4, false, TS, TD>(m, count, emb, en, k, tau, tp, labels, best, sims, s);
    if (k <= 16) return classify_dmma_t<2, 4, false, TS, TD>(m, count, emb, en, k, tau, tp, labels, best, sims, s);
    if (k <= 32) return classify_dmma_t<4, 4, false, TS, TD>(m, count, emb, en, k, tau, tp, labels, best, sims, s);
    if (k <= 64) return classify_dmma_t<8, 2, false, TS, TD>(m, count, emb, en, k, tau, tp, labels, best, sims, s);
    if (k <= 128) {
        if constexpr (sizeof(TS) == 4)
            return classify_dmma_t<16, 2, true, TS, TD>(m, count, emb, en, k, tau, tp, labels, best, sims, s);
        return classify_dmma_t<16, 1, true, TS, TD>(m, count, emb, en, k, tau, tp, labels, best, sims, s);
    }
    const int T = 256;
    k_classify<TS, TD><<<grid_for(count * 32, T), T, 0, s>>>(
        count, m->payload_d, k, ptr<int>(m->act_vid), ptr<TS>(m->s0), ptr<TD>(m->vt), emb, en,
        tau, tp, labels, best, sims);
    SVX_LAUNCHED();
    return SVX_OK;
}

svx_status launch_classify(svx_map* m, int64_t count, const double* emb, const double* en, int k,
                           double tau, double tp, int32_t* labels, double* best, double* sims,
                           cudaStream_t s) {
    if (count == 0) return SVX_OK;
    const bool s64 = m->cfg.state_dtype == SVX_F64, t64 = m->cfg.tsdf_dtype == SVX_F64;
    if (s64 && t64) return classify_t<double, double>(m, count, emb, en, k, tau, tp, labels, best, sims, s);
    if (s64) return classify_t<double, float>(m, count, emb, en, k, tau, tp, labels, best, sims, s);
    if (t64) return classify_t<float, double>(m, count, emb, en, k, tau, tp, labels, best, sims, s);
    return classify_t<float, float>(m, count, emb, en, k, tau, tp, labels, best, sims, s);
}

svx_status launch_label_map(svx_map* m, int64_t count, int mode, int32_t* labels, cudaStream_t s) {
    if (count == 0) return SVX_OK;
    const int T = 256;
    if (m->cfg.count_dtype == SVX_F64)
        k_label_map<double><<<grid_for(count, T), T, 0, s>>>(count, m->payload_d, mode,
                                                             ptr<int>(m->act_vid), ptr<double>(m->s0), labels);
    else
        k_label_map<float><<<grid_for(count, T), T, 0, s>>>(count, m->payload_d, mode,
                                                            ptr<int>(m->act_vid), ptr<float>(m->s0), labels);
    SVX_LAUNCHED();
    return SVX_OK;
}

}  // namespace svx

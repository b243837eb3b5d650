// svx_score.cu -- classify_means (gaussian.py:132-155) scores on the 5th-gen
// tensor cores: S = M . E^T (voxel means f32, query embeddings f64) as an
// exact-integer split GEMM on tcgen05.mma.kind::i8 (the Ozaki scheme).
//
// The reference scores in f64 and softmax(S / tau) with tau = 0.01 turns a
// score error e into a relative error e / tau, so S must be f64-accurate.
// B200 has no f64 kind of tcgen05, but an f64-accurate product can be built
// from exact int8 products:
//   every voxel row m gets a power-of-two scale 2^ea > max|m| and becomes the
//   integers N = m 2^(55-ea) (|N| < 2^55; exact for an f32 element within
//   2^31 of the row maximum), cut into the 7 bytes of N's two's complement:
//   N = A_0 2^48 + A_1 2^40 + ... + A_6 (A_0 signed, A_1..A_6 unsigned);
//   every query e likewise into B_0..B_6 with 2^eb > max|e|;
//   S = 2^(ea+eb-110) sum_{t,u} 2^(96-8(t+u)) (A_t . B_u), where each A_t . B_u
//   is an 8-bit dot product (s8 or u8 per plane, both kinds of
//   tcgen05.mma.kind::i8) accumulated exactly in int32 by the tensor core;
//   products of the same order n = t + u share a TMEM accumulator (<= 8 of
//   them, each |A_t . B_u| <= 255^2 D: < 2^31 for D <= 1024); the 34 pairs
//   with n <= 7 are kept (the rest are below 2^-56 of the scale), so S is
//   exact to ~2^-55 relative to 2^(ea+eb) before the final f64 sum.  The
//   split itself is byte extraction -- no digit arithmetic.
//
// k_score_rows   per active voxel: row scale exponent and the f64 norm
// k_score_queries per query: scale exponent and the digits, written as the
//                shared-memory image of every (query tile, dim chunk)
// k_score_mma    persistent, one CTA per SM (the 8 accumulators x 64 query
//                columns fill TMEM's 512 columns): per 128-voxel x 64-query
//                tile and 64-dim chunk, 256 threads gather the means through
//                act_vid and cut them into the 8 digit planes in shared memory
//                (double buffered) while one thread issues the chunk's 72
//                tcgen05.mma (36 pairs x 2 K-steps of 32) for the other buffer;
//                the epilogue reads the accumulators with tcgen05.ld and
//                writes S (f64) per voxel and query
// k_score_softmax cosine normalisation, softmax, argmax and the label rules
//                (the DMMA kernel's epilogue, svx_query.cu), per voxel
#include <math.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "svx_internal.cuh"

namespace svx {
namespace {

constexpr int kDig = 7;             // byte planes per operand
constexpr int kDiag = 8;            // accumulators: n = t + u in [0, 7]
constexpr int kScaleBits = 55;      // |N| < 2^55: 7 two's-complement bytes
constexpr int kTM = 128;            // voxels per tile (TMEM lanes)
constexpr int kTN = 64;             // queries per tile (32 when k <= 32)
constexpr int kKC = 64;             // dims per chunk (bytes of one digit plane row)
constexpr uint32_t kSBO = 8 * kKC;            // byte stride of 8-row swizzle atoms
constexpr int kAPlane = kTM * kKC;            // bytes of one A digit plane per chunk

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Shared-memory matrix descriptor: K-major, 64-byte swizzle (a plane row is
// the 64 bytes of one chunk; 8-row atoms of 512 B, the 16-byte pieces of row
// r permuted by (r % 8) >> 1 -- conflict-free for the tensor core's reads);
// LBO unused (16 B), SBO = 512 B between 8-row atoms.  A K-step of 32 bytes
// advances the start address by 32 (tools/tc_probe.cu checks both layouts).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)(16u >> 4) << 16;
    d |= (uint64_t)((kSBO >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;   // descriptor version (sm_100)
    d |= (uint64_t)4 << 61;   // SWIZZLE_64B
    return d;
}

// Instruction descriptor: 8-bit x 8-bit -> s32, both K-major, M x N; each
// operand signed (plane 0, the top byte) or unsigned (the lower bytes).
__host__ __device__ constexpr uint32_t idesc_i8(int m, int n, bool a_signed, bool b_signed) {
    return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((b_signed ? 1u : 0u) << 10) | ((uint32_t)(n >> 3) << 17) |
           ((uint32_t)(m >> 4) << 24);
}

// byte offset of element (row r, dim c) of a K-major 64-byte-swizzled plane
__host__ __device__ __forceinline__ uint32_t plane_off(int r, int c) {
    return (uint32_t)((r >> 3) * kSBO + (r & 7) * 64 + ((((c >> 4) ^ ((r & 7) >> 1)) & 3) << 4) + (c & 15));
}

// ---- prep --------------------------------------------------------------------

// scale exponent: 2^e > max|x| (e = 0 for an all-zero row)
__device__ __forceinline__ int scale_exp(double mx) { return mx > 0.0 ? ilogb(mx) + 1 : 0; }

template <class TS>
__global__ void k_score_rows(int64_t count, int D, const int* __restrict__ act_vid, const TS* __restrict__ mean,
                             int* __restrict__ ea, double* __restrict__ mnorm) {
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= count) return;
    const TS* row = mean + (int64_t)act_vid[i] * D;
    double nn = 0.0, mx = 0.0;
    for (int c = lane; c < D; c += 32) {
        const double v = (double)row[c];
        nn += v * v;
        mx = fmax(mx, fabs(v));
    }
    for (int o = 16; o > 0; o >>= 1) {
        nn += __shfl_xor_sync(0xffffffffu, nn, o);
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0) {
        ea[i] = scale_exp(mx);
        mnorm[i] = sqrt(nn);
    }
}

// One warp per query: exponent, then each dim's 8 digits into the image
// bimg[qt][chunk][digit][plane] (planes in the canonical layout).
__global__ void k_score_queries(int k, int D, int nchunks, int tn, const double* __restrict__ emb,
                                int* __restrict__ eb, int8_t* __restrict__ bimg) {
    const int bplane = tn * kKC;
    const int q = blockIdx.x;
    const int lane = threadIdx.x;
    const double* e = emb + (int64_t)q * D;
    double mx = 0.0;
    for (int c = lane; c < D; c += 32) mx = fmax(mx, fabs(e[c]));
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const int ex = scale_exp(mx);
    if (lane == 0) eb[q] = ex;
    const int qt = q / tn, qr = q % tn;
    for (int c = lane; c < nchunks * kKC; c += 32) {
        const double v = c < D ? e[c] : 0.0;
        // N = round(v 2^(55 - ex)), |N| < 2^55: its 7 low bytes, top byte first
        const long long nv = llrint(ldexp(v, kScaleBits - ex));
        const int ch = c / kKC, cc = c % kKC;
        int8_t* blk = bimg + ((int64_t)(qt * nchunks + ch) * kDig) * bplane;
#pragma unroll
        for (int t = 0; t < kDig; ++t)
            blk[(int64_t)t * bplane + plane_off(qr, cc)] = (int8_t)(unsigned char)(nv >> (8 * (kDig - 1 - t)));
    }
}

// digit i (1..8) of |x| 2^(56 - ea), x = +-M24 2^e2 (f32)
__device__ __forceinline__ int f32_digit(uint32_t m24, int sh, int i) {
    const int r = 56 - 7 * i - sh;   // right shift of the 24-bit mantissa
    uint32_t v;
    if (r >= 0) v = r < 32 ? (m24 >> r) : 0u;
    else v = -r < 32 ? (m24 << -r) : 0u;
    return (int)(v & 127u);
}

// ---- the MMA kernel ----------------------------------------------------------
//
// Warp roles (288 threads, one CTA per SM):
//   warps 0-7  producers: gather the tile's means (one float4 stream per
//              thread, the next chunk's loads in flight while this chunk is
//              cut) into the 8 digit planes of a stage, then arrive on the
//              stage's `full` barrier; warps 0-3 also run the epilogue
//   warp 8     MMA issuer: waits `full`, issues the chunk's 72 tcgen05.mma,
//              commits to the stage's `empty` barrier (and after the last
//              chunk to `tmem_full`); before a tile's first MMA it waits
//              `tmem_empty` (the epilogue has read the accumulators)

struct ScoreArgs {
    int64_t count;
    int D, k, nchunks, nqt;
    const int* act_vid;
    const int* ea;
    const int* eb;
    const int8_t* bimg;
    double* scores;    // (count, k)
};

__device__ __forceinline__ void mbar_wait_parity(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tSW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra SW_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}"
        : "=r"(pred));
    return pred != 0;
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_init_count(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

#ifndef SVX_SCORE_PRODUCERS
#define SVX_SCORE_PRODUCERS 512
#endif
constexpr int kProducers = SVX_SCORE_PRODUCERS;   // 256: 32 dims per thread, 512: 16
constexpr int kPerThread = kTM * kKC / kProducers;  // dims of one row per producer thread
constexpr int kScoreThreadsWS = kProducers + 32;

// N = x 2^(55 - ea) of one f32 element as a 64-bit integer (|N| < 2^55;
// bits below 2^0 of tiny elements are dropped)
__device__ __forceinline__ long long f32_fixed(float x, int ea) {
    const uint32_t bits = __float_as_uint(x);
    const uint32_t ex = (bits >> 23) & 255u;
    const uint32_t m24 = ex ? ((bits & 0x7FFFFFu) | 0x800000u) : (bits & 0x7FFFFFu);
    const int sh = (ex ? (int)ex - 150 : -149) + kScaleBits - ea;
    const long long mag =
        sh >= 0 ? (long long)((unsigned long long)m24 << min(sh, 63)) : (long long)(m24 >> min(-sh, 31));
    return (bits >> 31) ? -mag : mag;
}

template <int TN>
__global__ void __launch_bounds__(kScoreThreadsWS, 1) k_score_mma(ScoreArgs a, const float* __restrict__ mean) {
    constexpr int BPlane = TN * kKC;
    constexpr int Stage = kDig * (kAPlane + BPlane);
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) unsigned long long s_full[2], s_empty[2], s_tfull, s_tempty;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int st = 0; st < 2; ++st) {
            mbar_init_count(smem_u32(&s_full[st]), kProducers);
            mbar_init_count(smem_u32(&s_empty[st]), 1);
        }
        mbar_init_count(smem_u32(&s_tfull), 1);
        mbar_init_count(smem_u32(&s_tempty), 128);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    const int64_t ntm = (a.count + kTM - 1) / kTM;
    const int64_t ntiles = ntm * a.nqt;
    if (warp == kProducers / 32) {
        // ---- MMA issuer: the whole warp runs the loop (descriptors stay
        // warp-uniform, so they live in uniform registers); one elected lane
        // issues each tcgen05.mma ----
        uint32_t pf[2] = {0u, 0u}, pte = 0u;
        int chunks_done = 0;
        bool first_tile = true;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            if (!first_tile) {   // the epilogue has read the previous tile's accumulators
                mbar_wait_parity(smem_u32(&s_tempty), pte);
                pte ^= 1u;
            }
            first_tile = false;
            for (int ch = 0; ch < a.nchunks; ++ch, ++chunks_done) {
                const int st = chunks_done & 1;
#ifdef SVX_SCORE_TIMING
                const unsigned long long tw0 = globaltimer();
#endif
                mbar_wait_parity(smem_u32(&s_full[st]), pf[st]);
                pf[st] ^= 1u;
#ifdef SVX_SCORE_TIMING
                const unsigned long long tw1 = globaltimer();
#endif
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                __syncwarp();
                const uint32_t a0 = smem_u32(smem + st * Stage), b0 = a0 + kDig * kAPlane;
                const bool leader = elect_one();
                // descriptors: constant high word, start address (16-byte units) in the low word
                const uint32_t dhi = (uint32_t)(smem_desc(0) >> 32);
                const uint32_t dlo_a = (uint32_t)smem_desc(a0), dlo_b = (uint32_t)smem_desc(b0);
#pragma unroll
                for (int t = 0; t < kDig; ++t) {
#pragma unroll
                    for (int u = 0; u < kDig; ++u) {
                        if (t + u >= kDiag) continue;
                        const uint32_t d_tmem = tmem + (uint32_t)((t + u) * TN);
                        constexpr uint32_t id_ss = idesc_i8(kTM, TN, true, true), id_su = idesc_i8(kTM, TN, true, false),
                                           id_us = idesc_i8(kTM, TN, false, true),
                                           id_uu = idesc_i8(kTM, TN, false, false);
                        const uint32_t idesc = t == 0 ? (u == 0 ? id_ss : id_su) : (u == 0 ? id_us : id_uu);
#pragma unroll
                        for (int kk = 0; kk < kKC / 32; ++kk) {
                            const uint64_t da = ((uint64_t)dhi << 32) | (dlo_a + (uint32_t)((t * kAPlane + kk * 32) >> 4));
                            const uint64_t db = ((uint64_t)dhi << 32) | (dlo_b + (uint32_t)((u * BPlane + kk * 32) >> 4));
                            // the first product of each order in a tile starts the accumulator
                            const bool first = ch == 0 && kk == 0 && t == (t + u > kDig - 1 ? t + u - (kDig - 1) : 0);
                            if (leader)
                                asm volatile(
                                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
                                    "l"(da), "l"(db), "r"(idesc), "r"(first ? 0u : 1u));
                        }
                    }
                }
                if (leader) {
                    asm volatile(
                        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                            smem_u32(&s_empty[st])));
                    if (ch == a.nchunks - 1)
                        asm volatile(
                            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                smem_u32(&s_tfull)));
                }
                __syncwarp();
#ifdef SVX_SCORE_TIMING
                if (blockIdx.x == 0 && lane == 0 && tile < 3 * gridDim.x)
                    printf("mma tile %lld ch %d wait_full %llu issue %llu\n", (long long)tile, ch, tw1 - tw0,
                           globaltimer() - tw1);
#endif
            }
        }
    } else {
        // ---- producers (+ epilogue on warps 0-3) ----
        uint32_t pe[2] = {0u, 0u}, ptf = 0u;
        int used[2] = {0, 0};
        int chunks_done = 0;
        constexpr int kParts = kKC / kPerThread;   // producer threads per row
        const int r = tid / kParts, h = tid % kParts;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const int64_t tm = tile / a.nqt;
            const int qt = (int)(tile % a.nqt);
            const int64_t v0 = tm * kTM;
            const int64_t vi = v0 + r;
            const bool live = vi < a.count;
            const float* mrow = live ? mean + (int64_t)a.act_vid[vi] * a.D : nullptr;
            const int ea = live ? a.ea[vi] : 0;
            // software pipeline: this chunk's floats, next chunk's in flight
            constexpr int NQ = kPerThread / 4;
            float4 cur[NQ], nxt[NQ];
            auto load = [&](int ch, float4 (&dst)[NQ]) {
                const int d0 = ch * kKC + h * kPerThread;
                if (mrow && d0 + kPerThread <= a.D) {
#pragma unroll
                    for (int q = 0; q < NQ; ++q) dst[q] = __ldg(reinterpret_cast<const float4*>(mrow + d0) + q);
                } else {
#pragma unroll
                    for (int q = 0; q < NQ; ++q) {
                        float v[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int d = d0 + 4 * q + u;
                            v[u] = (mrow && d < a.D) ? mrow[d] : 0.f;
                        }
                        dst[q] = make_float4(v[0], v[1], v[2], v[3]);
                    }
                }
            };
            load(0, cur);
            for (int ch = 0; ch < a.nchunks; ++ch, ++chunks_done) {
                const int st = chunks_done & 1;
                if (ch + 1 < a.nchunks) load(ch + 1, nxt);
                unsigned char* sA = smem + st * Stage;
                unsigned char* sB = sA + kDig * kAPlane;
#ifdef SVX_SCORE_TIMING
                const unsigned long long tp0 = globaltimer();
#endif
                if (used[st]) {   // the MMAs that last read this stage are done
                    mbar_wait_parity(smem_u32(&s_empty[st]), pe[st]);
                    pe[st] ^= 1u;
                }
                used[st] = 1;
#ifdef SVX_SCORE_TIMING
                const unsigned long long tp1 = globaltimer();
#endif
                // cut kPerThread elements: byte t of every element's N -> plane t
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    const long long n0 = f32_fixed(cur[q].x, ea), n1 = f32_fixed(cur[q].y, ea),
                                    n2 = f32_fixed(cur[q].z, ea), n3 = f32_fixed(cur[q].w, ea);
                    const uint32_t l0 = (uint32_t)n0, l1 = (uint32_t)n1, l2 = (uint32_t)n2, l3 = (uint32_t)n3;
                    const uint32_t h0 = (uint32_t)(n0 >> 32), h1 = (uint32_t)(n1 >> 32),
                                   h2 = (uint32_t)(n2 >> 32), h3 = (uint32_t)(n3 >> 32);
                    // plane t holds byte (6 - t): bytes 0-3 from the low words, 4-6 from the high
                    uint32_t wq[kDig];
#pragma unroll
                    for (int t = 0; t < kDig; ++t) {
                        const int b = kDig - 1 - t;
                        const uint32_t sel = (uint32_t)(b & 3);
                        const uint32_t a01 = b < 4 ? __byte_perm(l0, l1, sel | ((sel + 4) << 4))
                                                   : __byte_perm(h0, h1, sel | ((sel + 4) << 4));
                        const uint32_t a23 = b < 4 ? __byte_perm(l2, l3, sel | ((sel + 4) << 4))
                                                   : __byte_perm(h2, h3, sel | ((sel + 4) << 4));
                        wq[t] = __byte_perm(a01, a23, 0x5410);
                    }
#pragma unroll
                    for (int t = 0; t < kDig; ++t)
                        *reinterpret_cast<uint32_t*>(sA + t * kAPlane + plane_off(r, h * kPerThread + 4 * q)) = wq[t];
                }
                {   // B: the chunk's image (8 planes of TN x 64 bytes)
                    const uint4* src =
                        reinterpret_cast<const uint4*>(a.bimg + ((int64_t)(qt * a.nchunks + ch) * kDig) * BPlane);
                    uint4* dst = reinterpret_cast<uint4*>(sB);
                    for (int t = tid; t < kDig * BPlane / 16; t += kProducers) dst[t] = __ldg(src + t);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive(smem_u32(&s_full[st]));
#ifdef SVX_SCORE_TIMING
                if (blockIdx.x == 0 && tid == 0 && tile < 3 * gridDim.x)
                    printf("prod tile %lld ch %d wait_empty %llu produce %llu\n", (long long)tile, ch, tp1 - tp0,
                           globaltimer() - tp1);
#endif
                if (ch + 1 < a.nchunks) {
#pragma unroll
                    for (int q = 0; q < NQ; ++q) cur[q] = nxt[q];
                }
            }
            // ---- epilogue: warps 0-3, thread = TMEM lane = voxel row ----
            if (warp < 4) {
                mbar_wait_parity(smem_u32(&s_tfull), ptf);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const int row = 32 * warp + lane;
                const int64_t v = v0 + row;
                const int er = v < a.count ? a.ea[v] : 0;
                double* out = v < a.count ? a.scores + v * a.k : nullptr;
#pragma unroll 1
                for (int c0 = 0; c0 < TN; c0 += 8) {
                    uint32_t u[kDiag][8];
#pragma unroll
                    for (int n = 0; n < kDiag; ++n) {
                        const uint32_t addr = tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)(n * TN + c0);
                        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                                     : "=r"(u[n][0]), "=r"(u[n][1]), "=r"(u[n][2]), "=r"(u[n][3]), "=r"(u[n][4]),
                                       "=r"(u[n][5]), "=r"(u[n][6]), "=r"(u[n][7])
                                     : "r"(addr));
                    }
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    if (out) {
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            double t = 0.0;
#pragma unroll
                            for (int n = kDiag - 1; n >= 0; --n)   // smallest orders first
                                t += (double)(int)u[n][q] * ldexp(1.0, -14 - 8 * n);
                            const int j = qt * TN + c0 + q;
                            if (j < a.k) out[j] = ldexp(t, er + a.eb[j]);
                        }
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                mbar_arrive(smem_u32(&s_tempty));
            }
            ptf ^= 1u;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// Cosine normalisation, softmax(S / tau), argmax and label rules per voxel
// (the DMMA kernel's epilogue; gaussian.py:132-155).
template <class TD>
__global__ void k_score_softmax(int64_t count, int k, const int* __restrict__ act_vid, const TD* __restrict__ vw,
                                const double* __restrict__ scores, const double* __restrict__ mnorm,
                                const double* __restrict__ en, double tau, double tp, int32_t* __restrict__ labels,
                                double* __restrict__ best, double* __restrict__ sims_out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const double mn = mnorm[i];
    const double wgt = (double)vw[2 * (int64_t)act_vid[i] + 1];   // {d, w} pairs
    const bool ok = mn != 0.0 && wgt > 0.0;
    const double* s = scores + i * k;
    double lmax = -INFINITY;
    for (int j = 0; j < k; ++j) {
        const double sj = mn == 0.0 ? NAN : s[j] / (mn * en[j]);
        if (sims_out) sims_out[i * k + j] = sj;
        const double ej = sj / tau;
        lmax = ej > lmax ? ej : lmax;
    }
    if (!ok) {
        labels[i] = 0;
        best[i] = 0.0;
        return;
    }
    double den = 0.0, emax = -1.0;
    int arg = 0;
    for (int j = 0; j < k; ++j) {
        const double ej = exp(s[j] / (mn * en[j]) / tau - lmax);
        den += ej;
        if (ej > emax) { emax = ej; arg = j; }
    }
    const double top = emax / den;
    labels[i] = top < tp ? 0 : arg + 1;
    best[i] = top;
}

}  // namespace

// Scores through the int8 tensor cores; then the same softmax rules as the
// DMMA kernel.  f32 means only (f64 state keeps the DMMA kernel: its 53-bit
// mantissas would need the f64 digit path).  Scratch: sc_q (query digits,
// exponents), sc_o (scores, norms, row exponents).
svx_status classify_tc(svx_map* m, int64_t count, const int* act_vid, const double* emb, const double* en,
                       int k, double tau, double tp, int32_t* labels, double* best, double* sims,
                       cudaStream_t s) {
    const int D = m->payload_d;
    const int nchunks = (D + kKC - 1) / kKC;
    const int tn = k <= 32 ? 32 : kTN;
    const int nqt = (k + tn - 1) / tn;
    const size_t img = (size_t)nqt * nchunks * kDig * tn * kKC;
    const size_t need_q = img + sizeof(int) * (size_t)nqt * tn;
    const size_t need_o = sizeof(double) * (size_t)count * (k + 1) + sizeof(int) * (size_t)count + 16;
    SVX_TRY(ensure(m->sc_q, need_q, s));
    SVX_TRY(ensure(m->sc_o, need_o, s));
    int8_t* bimg = ptr<int8_t>(m->sc_q);
    int* eb = reinterpret_cast<int*>(bimg + img);
    double* scores = ptr<double>(m->sc_o);
    double* mnorm = scores + (size_t)count * k;
    int* ea = reinterpret_cast<int*>(mnorm + count);
    static const bool trace = getenv("SVX_TRACE_SCORE") != nullptr;
    cudaEvent_t ev[5] = {};
    if (trace)
        for (auto& e : ev) cudaEventCreate(&e);
    if (trace) cudaEventRecord(ev[0], s);
    SVX_CUDA(cudaMemsetAsync(bimg, 0, img, s));
    k_score_queries<<<k, 32, 0, s>>>(k, D, nchunks, tn, emb, eb, bimg);
    SVX_LAUNCHED();
    const bool t64 = m->cfg.tsdf_dtype == SVX_F64;
    const int T = 256;
    k_score_rows<float><<<grid_for(count * 32, T), T, 0, s>>>(count, D, act_vid, ptr<float>(m->s0), ea, mnorm);
    SVX_LAUNCHED();
    if (trace) cudaEventRecord(ev[1], s);
    ScoreArgs a;
    a.count = count;
    a.D = D;
    a.k = k;
    a.nchunks = nchunks;
    a.nqt = nqt;
    a.act_vid = act_vid;
    a.ea = ea;
    a.eb = eb;
    a.bimg = bimg;
    a.scores = scores;
    const int64_t ntiles = ((count + kTM - 1) / kTM) * nqt;
    const int grid = (int)std::min<int64_t>(ntiles, 148);
    static bool attr_set[2] = {false, false};   // (per process; set once per template)
    if (tn == 32) {
        const int smem = 2 * kDig * (kAPlane + 32 * kKC);
        if (!attr_set[0])
            SVX_CUDA(cudaFuncSetAttribute(k_score_mma<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr_set[0] = true;
        k_score_mma<32><<<grid, kScoreThreadsWS, smem, s>>>(a, ptr<float>(m->s0));
    } else {
        const int smem = 2 * kDig * (kAPlane + kTN * kKC);
        if (!attr_set[1])
            SVX_CUDA(cudaFuncSetAttribute(k_score_mma<kTN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr_set[1] = true;
        k_score_mma<kTN><<<grid, kScoreThreadsWS, smem, s>>>(a, ptr<float>(m->s0));
    }
    SVX_LAUNCHED();
    if (trace) cudaEventRecord(ev[2], s);
    if (t64)
        k_score_softmax<double><<<grid_for(count, T), T, 0, s>>>(count, k, act_vid, ptr<double>(m->vt), scores, mnorm,
                                                                 en, tau, tp, labels, best, sims);
    else
        k_score_softmax<float><<<grid_for(count, T), T, 0, s>>>(count, k, act_vid, ptr<float>(m->vt), scores, mnorm,
                                                                en, tau, tp, labels, best, sims);
    SVX_LAUNCHED();
    if (trace) {
        cudaEventRecord(ev[3], s);
        cudaEventSynchronize(ev[3]);
        float t[3];
        for (int i = 0; i < 3; ++i) cudaEventElapsedTime(&t[i], ev[i], ev[i + 1]);
        fprintf(stderr, "svx score ms: prep %.3f mma %.3f softmax %.3f\n", t[0], t[1], t[2]);
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
    }
    return SVX_OK;
}

}  // namespace svx

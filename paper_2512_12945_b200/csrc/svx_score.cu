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
// k_score_mma    persistent, one CTA per SM (8 accumulators x 64 query columns
//                fill TMEM's 512 columns; 2 accumulator sets when k <= 32):
//                per 128-voxel x TN-query tile and 64-dim chunk, 512 threads
//                gather the means through act_vid and cut them into the 7
//                byte planes in shared memory (double buffered; the query
//                planes arrive by bulk copy) while one elected lane issues the
//                chunk's 68 tcgen05.mma (34 pairs x 2 K-steps of 32) for the
//                other buffer; the epilogue reads the accumulators with
//                tcgen05.ld and writes S (f64) per voxel and query
// k_score_softmax cosine normalisation, softmax, argmax and the label rules
//                (the DMMA kernel's epilogue, svx_query.cu), one warp per voxel
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

// ---- the MMA kernel ----------------------------------------------------------
//
// Warp roles (544 threads, one CTA per SM):
//   warps 0-15 producers: 4 threads per voxel row, 16 dims each.  Chunk g's
//              floats were loaded two chunks earlier; they become N (one exact
//              f32 multiply by 2^(55 - ea) and a cvt.rzi.s64) and 7 byte planes
//              (4x4 byte transposes) in registers, the loads for chunk g + 2
//              are issued, and then the thread waits for the stage to be free
//              and stores one 16-byte word per plane (conflict-free: a warp
//              fills one 8-row swizzle atom).  Thread 0 also copies the
//              chunk's query planes (one contiguous block of the image) with
//              one bulk copy (TMA) completing on the stage's `full` barrier.
//              The same warps run the epilogue: warp w reads TMEM lanes
//              32 (w % 4).. and a quarter of the tile's query columns; the
//              epilogue of tile j runs after chunks 0 and 1 of tile j + 1 are
//              staged, so the MMA warp waits only for the epilogue itself.
//              For k <= 32 the epilogue also applies the softmax rules (the
//              4 column quarters of a row meet in shared memory).
//   warp 16    MMA issuer: waits `full`, issues the chunk's 68 tcgen05.mma,
//              commits to the stage's `empty` barrier (and after a tile's
//              last chunk to `tfull`); before a tile's first MMA it waits
//              `tempty` of its accumulator set (2 sets when TN = 32).
// Measured limits (profiles/r02_tcgen05_score_*): SS-mode MMAs at N = 64 read
// 6 KB of shared memory each (~48 cycles, above the 32-cycle tensor floor);
// the stage's fence.proxy.async (MEMBAR) also waits for the thread's
// outstanding global loads, so the producers' chunk period, not the MMA,
// sets the pace.  Tried and slower: a 3-slot query-plane ring with its own
// copy warp (less L1 for the row gathers), row staging by 128-byte bulk
// copies (too many small TMA operations), loads issued after the fence.

// Softmax / label rules (gaussian.py:132-155) for the fused epilogue and the
// standalone kernel.
struct SoftmaxArgs {
    int k;
    const int* act_vid;
    const void* vw;     // {d, w} pairs, f32 or f64
    int vw64;
    const double* mnorm;
    const double* en;
    double tau, tp;
    int32_t* labels;    // null: scores only (the standalone softmax follows)
    double* best;
    double* sims;       // optional cosine output
};

struct ScoreArgs {
    SoftmaxArgs sm;
    int64_t count;
    int D, k, nchunks, nqt;
    const int* act_vid;
    const int* ea;
    const int* eb;
    const int8_t* bimg;
    double* scores;    // (count, k)
#ifdef SVX_SCORE_TIMING
    unsigned long long* trace;   // CTA 0: 8 timestamps per chunk
#endif
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

// expect `bytes` on bar (one arrival), then one bulk copy global -> shared completing on it
__device__ __forceinline__ void bulk_copy(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

constexpr int kProducers = 512;
constexpr int kPerThread = kTM * kKC / kProducers;  // 16 dims of one row per producer thread
constexpr int kParts = kKC / kPerThread;           // 4 producer threads per row
constexpr int kScoreThreadsWS = kProducers + 32;


// N = x 2^(55 - ea) of one f32 element as a 64-bit two's-complement integer
// (lo, hi words; |N| < 2^55, bits below 2^0 of tiny elements dropped).
// c = 55 - 150 - ea: the mantissa's left shift is sh = max(exp, 1) + c <= 31
// because 2^ea > |x|; a negative sh shifts right instead.
__device__ __forceinline__ void f32_fixed(float x, int c, uint32_t& lo, uint32_t& hi) {
    const uint32_t bits = __float_as_uint(x);
    const int ex = (int)((bits >> 23) & 255u);
    const uint32_t m24 = (bits & 0x7FFFFFu) | ((uint32_t)min(ex, 1) << 23);   // denormals: no implicit bit
    const int sh = max(ex, 1) + c;
    const uint32_t up = (uint32_t)max(sh, 0), dn = (uint32_t)max(-sh, 0);
    const uint32_t m = __funnelshift_rc(m24, 0u, dn);        // m24 >> dn (0 for dn >= 32)
    const uint32_t l = m << up, h = __funnelshift_l(m, 0u, up);   // (h:l) = m << up
    const uint32_t sg = (uint32_t)((int)bits >> 31);          // 0 or all ones
    const unsigned long long v =
        ((((unsigned long long)(h ^ sg)) << 32) | (l ^ sg)) - (unsigned long long)(long long)(int)sg;
    lo = (uint32_t)v;
    hi = (uint32_t)(v >> 32);
}

// 16 floats -> 7 planes x 16 bytes: plane t holds byte (6 - t) of every N
// (4 x 4 byte transposes: bytes 0-3 from the low words, 4-6 from the high).
// N = trunc(x 2^(55 - ea)): one exact f32 multiply by the power of two and one
// f32 -> s64 conversion (cvt.rzi) when 2^(55 - ea) is a normal f32, else the
// integer path (rows with max|x| < 2^-72 or > 2^181).
__device__ __forceinline__ void cut_planes(const float4 (&f)[4], int ea, uint4 (&w)[kDig]) {
    const int c = kScaleBits - 150 - ea;
    const int se = kScaleBits - ea + 127;   // biased exponent of the scale
    const bool fast = se >= 1 && se <= 254;
    const float scale = __int_as_float(min(max(se, 1), 254) << 23);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        uint32_t l0, l1, l2, l3, h0, h1, h2, h3;
        if (fast) {
            const long long n0 = __float2ll_rz(f[q].x * scale), n1 = __float2ll_rz(f[q].y * scale),
                            n2 = __float2ll_rz(f[q].z * scale), n3 = __float2ll_rz(f[q].w * scale);
            l0 = (uint32_t)n0; h0 = (uint32_t)((unsigned long long)n0 >> 32);
            l1 = (uint32_t)n1; h1 = (uint32_t)((unsigned long long)n1 >> 32);
            l2 = (uint32_t)n2; h2 = (uint32_t)((unsigned long long)n2 >> 32);
            l3 = (uint32_t)n3; h3 = (uint32_t)((unsigned long long)n3 >> 32);
        } else {
            f32_fixed(f[q].x, c, l0, h0);
            f32_fixed(f[q].y, c, l1, h1);
            f32_fixed(f[q].z, c, l2, h2);
            f32_fixed(f[q].w, c, l3, h3);
        }
        const uint32_t a0 = __byte_perm(l0, l1, 0x5140), a1 = __byte_perm(l0, l1, 0x7362);
        const uint32_t a2 = __byte_perm(l2, l3, 0x5140), a3 = __byte_perm(l2, l3, 0x7362);
        const uint32_t b0 = __byte_perm(h0, h1, 0x5140), b1 = __byte_perm(h0, h1, 0x7362);
        const uint32_t b2 = __byte_perm(h2, h3, 0x5140), b3 = __byte_perm(h2, h3, 0x7362);
        uint32_t pw[kDig];
        pw[6] = __byte_perm(a0, a2, 0x5410);   // byte 0
        pw[5] = __byte_perm(a0, a2, 0x7632);   // byte 1
        pw[4] = __byte_perm(a1, a3, 0x5410);   // byte 2
        pw[3] = __byte_perm(a1, a3, 0x7632);   // byte 3
        pw[2] = __byte_perm(b0, b2, 0x5410);   // byte 4
        pw[1] = __byte_perm(b0, b2, 0x7632);   // byte 5
        pw[0] = __byte_perm(b1, b3, 0x5410);   // byte 6 (signed top plane)
#pragma unroll
        for (int t = 0; t < kDig; ++t) {
            if (q == 0) w[t].x = pw[t];
            else if (q == 1) w[t].y = pw[t];
            else if (q == 2) w[t].z = pw[t];
            else w[t].w = pw[t];
        }
    }
}

__device__ __forceinline__ void load_part(const float* row, int D, int d0, float4 (&dst)[4]) {
    if (row && d0 + kPerThread <= D) {
#pragma unroll
        for (int q = 0; q < 4; ++q) dst[q] = __ldg(reinterpret_cast<const float4*>(row + d0) + q);
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int d = d0 + 4 * q + u;
                v[u] = (row && d < D) ? row[d] : 0.f;
            }
            dst[q] = make_float4(v[0], v[1], v[2], v[3]);
        }
    }
}

__device__ __forceinline__ void producers_bar() {   // the 16 producer warps
    asm volatile("bar.sync 1, %0;" ::"r"(kProducers) : "memory");
}

// Softmax of one row whose k <= 32 scores are spread over the 4 column-quarter
// warps (8 each): the row maximum and the sum / argmax are combined through
// shared memory (red: 11 x kTM doubles, rarg: 4 x kTM ints).
__device__ __forceinline__ void softmax_rows(const SoftmaxArgs& sm, int64_t v, int row, int cq,
                                             const double (&sv)[8], double* red, int* rarg) {
    const bool live = v >= 0;
    double mn = 0.0, wgt = 0.0;
    if (live) {
        mn = sm.mnorm[v];
        const int64_t vid = sm.act_vid[v];
        wgt = sm.vw64 ? static_cast<const double*>(sm.vw)[2 * vid + 1]
                      : (double)static_cast<const float*>(sm.vw)[2 * vid + 1];
    }
    const bool ok = live && mn != 0.0 && wgt > 0.0;
    double ej[8];
    double lmax = -INFINITY;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int j = cq * 8 + q;
        ej[q] = 0.0;
        if (j < sm.k) {
            const double sj = mn == 0.0 ? NAN : sv[q] / (mn * sm.en[j]);
            if (live && sm.sims) sm.sims[v * sm.k + j] = sj;
            ej[q] = sj / sm.tau;
            lmax = ej[q] > lmax ? ej[q] : lmax;
        }
    }
    red[cq * kTM + row] = lmax;
    producers_bar();
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const double x = red[c * kTM + row];
        lmax = x > lmax ? x : lmax;
    }
    double den = 0.0, emax = -1.0;
    int arg = 0x7fffffff;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int j = cq * 8 + q;
        if (j < sm.k) {
            const double x = exp(ej[q] - lmax);
            den += x;
            if (x > emax) { emax = x; arg = j; }
        }
    }
    red[(4 + cq) * kTM + row] = den;
    red[(8 + cq) * kTM + row] = emax;
    rarg[cq * kTM + row] = arg;
    producers_bar();
    if (cq == 0 && live) {
        double d = 0.0, em = -1.0;
        int am = 0x7fffffff;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            d += red[(4 + c) * kTM + row];
            const double e2 = red[(8 + c) * kTM + row];
            const int a2 = rarg[c * kTM + row];
            if (e2 > em || (e2 == em && a2 < am)) { em = e2; am = a2; }
        }
        const double top = em / d;
        sm.labels[v] = ok ? (top < sm.tp ? 0 : (am < sm.k ? am : 0) + 1) : 0;
        sm.best[v] = ok ? top : 0.0;
    }
}

template <int TN>
__global__ void __launch_bounds__(kScoreThreadsWS, 1) k_score_mma(ScoreArgs a, const float* __restrict__ mean) {
    constexpr int BPlane = TN * kKC;
    constexpr int BBytes = kDig * BPlane;
    constexpr int Stage = kDig * kAPlane + BBytes;
    constexpr int kSets = 512 / (kDiag * TN);   // accumulator sets in TMEM
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) unsigned long long s_full[2], s_empty[2], s_tfull[kSets], s_tempty[kSets];
    __shared__ double s_red[TN == 32 ? 12 * kTM : 1];
    __shared__ int s_rarg[TN == 32 ? 4 * kTM : 1];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int st = 0; st < 2; ++st) {
            mbar_init_count(smem_u32(&s_full[st]), kProducers + 1);   // + thread 0's expect_tx
            mbar_init_count(smem_u32(&s_empty[st]), 1);
        }
        for (int z = 0; z < kSets; ++z) {
            mbar_init_count(smem_u32(&s_tfull[z]), 1);
            mbar_init_count(smem_u32(&s_tempty[z]), kProducers);
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    const int64_t ntm = (a.count + kTM - 1) / kTM;
    const int64_t ntiles = ntm * a.nqt;
    const int nch = a.nchunks;   // >= 2
    const int my_tiles = blockIdx.x < ntiles ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
    if (warp == kProducers / 32) {
        // ---- MMA issuer: the whole warp runs the loop (descriptors stay
        // warp-uniform, so they live in uniform registers); one elected lane
        // issues each tcgen05.mma ----
        int g = 0;
        for (int j = 0; j < my_tiles; ++j) {
            const int set = kSets == 1 ? 0 : (j & (kSets - 1));
            if (j >= kSets) mbar_wait_parity(smem_u32(&s_tempty[set]), (uint32_t)((j / kSets - 1) & 1));
            const uint32_t dset = tmem + (uint32_t)(set * kDiag * TN);
            for (int ch = 0; ch < nch; ++ch, ++g) {
                const int st = g & 1;
#ifdef SVX_SCORE_TIMING
                const unsigned long long t0 = globaltimer(), t1 = t0;
#endif
                mbar_wait_parity(smem_u32(&s_full[st]), (uint32_t)((g >> 1) & 1));
#ifdef SVX_SCORE_TIMING
                const unsigned long long t2 = globaltimer();
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
                        const uint32_t d_tmem = dset + (uint32_t)((t + u) * TN);
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
#ifdef SVX_SCORE_TIMING
                    if (blockIdx.x == 0 && g < 256) {
                        unsigned long long* tr = a.trace + 8 * g;
                        tr[0] = t0; tr[1] = t1; tr[2] = t2; tr[3] = globaltimer();
                    }
#endif
                    if (ch == nch - 1)
                        asm volatile(
                            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                smem_u32(&s_tfull[set])));
                }
                __syncwarp();
            }
        }
    } else {
        // ---- producers + epilogue ----
        const int r = tid / kParts, h = tid % kParts;
        const int G = my_tiles * nch;
        // load side (chunk g + 2): its tile, row pointer and row exponent; the
        // next tile's row (act_vid, exponent) is fetched one tile ahead
        int ltile = -1, lea = 0, pvid = -1, pea = 0;
        const float* lrow = nullptr;
        auto tile_of = [&](int j) -> int64_t { return (int64_t)blockIdx.x + (int64_t)j * gridDim.x; };
        auto fetch_row = [&](int j) {
            const int64_t vi = (tile_of(j) / a.nqt) * kTM + r;
            pvid = -1;
            pea = 0;
            if (j < my_tiles && vi < a.count) {
                pvid = __ldg(a.act_vid + vi);
                pea = __ldg(a.ea + vi);
            }
        };
        auto issue = [&](int gl, float4 (&dst)[4]) {
            const int j = gl / nch, ch = gl - j * nch;
            if (j != ltile) {
                ltile = j;
                lrow = pvid >= 0 ? mean + (int64_t)pvid * a.D : nullptr;
                lea = pea;
                fetch_row(j + 1);
            }
            load_part(lrow, a.D, ch * kKC + h * kPerThread, dst);
        };
        // Epilogue of tile j: S = (sum_n acc_n 2^(56 - 8n)) 2^(ea + eb - 70), the
        // orders combined exactly in two int64 halves (orders 0-3 and 4-7).
        // Warp w reads TMEM lanes 32 (w % 4).. and column quarter w / 4.
        auto scores4 = [&](uint32_t base, int c0, int qt, int er, double (&val)[4]) {
            long long part[2][4];
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                uint32_t u[4][4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint32_t addr = base + (uint32_t)((4 * half + i) * TN + c0);
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(u[i][0]), "=r"(u[i][1]), "=r"(u[i][2]), "=r"(u[i][3])
                                 : "r"(addr));
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    long long x = (long long)(int)u[0][q];
#pragma unroll
                    for (int i = 1; i < 4; ++i) x = x * 256 + (long long)(int)u[i][q];
                    part[half][q] = x;
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int jq = qt * TN + c0 + q;
                const double d = (double)part[0][q] * 4294967296.0 + (double)part[1][q];
                const int e = er + (jq < a.k ? __ldg(a.eb + jq) : 0);
                val[q] = (e >= -1022 && e <= 1023) ? d * __longlong_as_double((long long)(e + 1023) << 52)
                                                  : ldexp(d, e);
            }
        };
        auto epilogue = [&](int j) {
            const int set = kSets == 1 ? 0 : (j & (kSets - 1));
            mbar_wait_parity(smem_u32(&s_tfull[set]), (uint32_t)((j / kSets) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const int64_t tile = tile_of(j);
            const int qt = (int)(tile % a.nqt);
            const int quad = warp & 3, cq = warp >> 2;   // TMEM lane quarter, column quarter
            const int row = 32 * quad + lane;
            const int64_t v = (tile / a.nqt) * kTM + row;
            const bool live = v < a.count;
            const int er = live ? __ldg(a.ea + v) - 70 : 0;
            const uint32_t base = tmem + ((uint32_t)(32 * quad) << 16) + (uint32_t)(set * kDiag * TN);
            if constexpr (TN == 32) {
                if (a.sm.labels) {
                    // k <= 32: the whole softmax here (one row's 32 scores over 4 warps)
                    double sv[8];
#pragma unroll
                    for (int g4 = 0; g4 < 2; ++g4) {
                        double val[4];
                        scores4(base, cq * 8 + 4 * g4, 0, er, val);
#pragma unroll
                        for (int q = 0; q < 4; ++q) sv[4 * g4 + q] = val[q];
                    }
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    mbar_arrive(smem_u32(&s_tempty[set]));   // TMEM is free; the rest is registers
                    softmax_rows(a.sm, live ? v : -1, row, cq, sv, s_red, s_rarg);
                    return;
                }
            }
            double* out = live ? a.scores + v * a.k : nullptr;
#pragma unroll 1
            for (int c0 = cq * (TN / 4); c0 < (cq + 1) * (TN / 4); c0 += 4) {
                double val[4];
                scores4(base, c0, qt, er, val);
                if (out) {
                    const int j0 = qt * TN + c0;
                    if (j0 + 4 <= a.k && (a.k & 1) == 0) {
                        *reinterpret_cast<double2*>(out + j0) = make_double2(val[0], val[1]);
                        *reinterpret_cast<double2*>(out + j0 + 2) = make_double2(val[2], val[3]);
                    } else {
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            if (j0 + q < a.k) out[j0 + q] = val[q];
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            mbar_arrive(smem_u32(&s_tempty[set]));
        };
        float4 fb[2][4];
        fetch_row(0);
        if (G > 0) issue(0, fb[0]);
        if (G > 1) issue(1, fb[1]);
        int cea = 0;
        for (int g = 0; g < G; ++g) {
            const int j = g / nch, ch = g - j * nch;
            const int st = g & 1;
            uint4 w[kDig];
#ifdef SVX_SCORE_TIMING
            const unsigned long long p0 = globaltimer();
#endif
            // entering a tile, the load side has issued its chunk 1 (nch >= 2) and no further
            if (ch == 0) cea = lea;
            // the buffer of chunk g is fb[g & 1]; refill it with chunk g + 2
            if (st == 0) {
                cut_planes(fb[0], cea, w);
                if (g + 2 < G) issue(g + 2, fb[0]);
            } else {
                cut_planes(fb[1], cea, w);
                if (g + 2 < G) issue(g + 2, fb[1]);
            }
#ifdef SVX_SCORE_TIMING
            const unsigned long long p1 = globaltimer();
#endif
            if (g >= 2) mbar_wait_parity(smem_u32(&s_empty[st]), (uint32_t)(((g >> 1) - 1) & 1));
#ifdef SVX_SCORE_TIMING
            const unsigned long long p2 = globaltimer();
#endif
            unsigned char* sA = smem + st * Stage;
            if (tid == 0) {
                const int qt = (int)(tile_of(j) % a.nqt);
                bulk_copy(smem_u32(sA + kDig * kAPlane), a.bimg + ((int64_t)(qt * nch + ch) * kDig) * BPlane,
                          (uint32_t)BBytes, smem_u32(&s_full[st]));
            }
            const uint32_t off = plane_off(r, h * kPerThread);
#pragma unroll
            for (int t = 0; t < kDig; ++t) *reinterpret_cast<uint4*>(sA + t * kAPlane + off) = w[t];
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive(smem_u32(&s_full[st]));
#ifdef SVX_SCORE_TIMING
            const unsigned long long p3 = globaltimer();
#endif
            if (ch == 1 && j >= 1) epilogue(j - 1);
#ifdef SVX_SCORE_TIMING
            if (blockIdx.x == 0 && tid == 0 && g < 256) {
                unsigned long long* tr = a.trace + 8 * g + 4;
                tr[0] = p0; tr[1] = p1; tr[2] = p2; tr[3] = globaltimer();
                (void)p3;
            }
#endif
        }
        if (my_tiles > 0) epilogue(my_tiles - 1);
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
    // reciprocals of the query norms and of tau: cos_j = S_j (1 / |m|) (1 / |e_j|),
    // within 2 ulp of the reference's S_j / (|m| |e_j|)
    extern __shared__ double s_rn[];
    for (int j = threadIdx.x; j < k; j += blockDim.x) s_rn[j] = 1.0 / en[j];
    __syncthreads();
    const double rtau = 1.0 / tau;
    // one warp per voxel, lane j takes queries j, j + 32, ... (coalesced rows)
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= count) return;
    const double mn = mnorm[i];
    const double wgt = (double)vw[2 * (int64_t)act_vid[i] + 1];   // {d, w} pairs
    const bool ok = mn != 0.0 && wgt > 0.0;
    const double rmn = 1.0 / mn;
    const double* s = scores + i * k;
    // e_j = cos_j / tau, kept in registers for the first 128 queries
    constexpr int KR = 4;
    double ec[KR];
    double lmax = -INFINITY;
    for (int j = lane, c = 0; j < k; j += 32, ++c) {
        const double sj = mn == 0.0 ? NAN : s[j] * rmn * s_rn[j];
        if (sims_out) sims_out[i * k + j] = sj;
        const double ej = sj * rtau;
#pragma unroll
        for (int q = 0; q < KR; ++q)
            if (q == c) ec[q] = ej;
        lmax = ej > lmax ? ej : lmax;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double x = __shfl_xor_sync(0xffffffffu, lmax, o);
        lmax = x > lmax ? x : lmax;
    }
    if (!ok) {
        if (lane == 0) {
            labels[i] = 0;
            best[i] = 0.0;
        }
        return;
    }
    double den = 0.0, emax = -1.0;
    int arg = k;   // first maximal index over the lane's queries
#pragma unroll
    for (int q = 0; q < KR; ++q) {
        const int j = lane + 32 * q;
        if (j < k) {
            const double ej = exp(ec[q] - lmax);
            den += ej;
            if (ej > emax) { emax = ej; arg = j; }
        }
    }
    for (int j = lane + 32 * KR; j < k; j += 32) {
        const double ej = exp(s[j] * rmn * s_rn[j] * rtau - lmax);
        den += ej;
        if (ej > emax) { emax = ej; arg = j; }
    }
    for (int o = 16; o > 0; o >>= 1) {
        den += __shfl_xor_sync(0xffffffffu, den, o);
        const double e2 = __shfl_xor_sync(0xffffffffu, emax, o);
        const int a2 = __shfl_xor_sync(0xffffffffu, arg, o);
        if (e2 > emax || (e2 == emax && a2 < arg)) { emax = e2; arg = a2; }
    }
    if (lane == 0) {
        const double top = emax / den;
        labels[i] = top < tp ? 0 : (arg < k ? arg : 0) + 1;
        best[i] = top;
    }
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
    const int nchunks = std::max(2, (D + kKC - 1) / kKC);   // the producers run two chunks ahead
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
    const bool fused = tn == 32;   // k <= 32: softmax in the MMA epilogue
    a.sm.k = k;
    a.sm.act_vid = act_vid;
    a.sm.vw = t64 ? (const void*)ptr<double>(m->vt) : (const void*)ptr<float>(m->vt);
    a.sm.vw64 = t64 ? 1 : 0;
    a.sm.mnorm = mnorm;
    a.sm.en = en;
    a.sm.tau = tau;
    a.sm.tp = tp;
    a.sm.labels = fused ? labels : nullptr;
    a.sm.best = best;
    a.sm.sims = sims;
#ifdef SVX_SCORE_TIMING
    unsigned long long* trace_d = nullptr;
    cudaMalloc(&trace_d, 256 * 8 * sizeof(unsigned long long));
    cudaMemsetAsync(trace_d, 0, 256 * 8 * sizeof(unsigned long long), s);
    a.trace = trace_d;
#endif
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
#ifdef SVX_SCORE_TIMING
    {
        unsigned long long h[256 * 8];
        cudaMemcpyAsync(h, trace_d, sizeof(h), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        const unsigned long long base = h[0];
        for (int g = 0; g < 256 && h[8 * g]; ++g) {
            const unsigned long long* t = h + 8 * g;
            fprintf(stderr, "g %3d M start %8llu bwait %5llu fwait %5llu issue %5llu | P start %8llu cut %5llu ewait %5llu store+epi %5llu\n",
                    g, t[0] - base, t[1] - t[0], t[2] - t[1], t[3] - t[2], t[4] - base, t[5] - t[4], t[6] - t[5], t[7] - t[6]);
        }
        cudaFree(trace_d);
    }
#endif
    if (trace) cudaEventRecord(ev[2], s);
    if (!fused) {
        if (t64)
            k_score_softmax<double><<<grid_for(count * 32, T), T, sizeof(double) * k, s>>>(count, k, act_vid, ptr<double>(m->vt), scores, mnorm,
                                                                     en, tau, tp, labels, best, sims);
        else
            k_score_softmax<float><<<grid_for(count * 32, T), T, sizeof(double) * k, s>>>(count, k, act_vid, ptr<float>(m->vt), scores, mnorm,
                                                                    en, tau, tp, labels, best, sims);
        SVX_LAUNCHED();
    }
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

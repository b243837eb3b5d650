// tc_probe.cu -- minimal tcgen05 int8 MMA check (layout / descriptor probe
// for the scoring kernel).  One CTA: C[128 x N] (int32, TMEM) = A[128 x K] *
// B[N x K]^T with A, B int8 K-major in shared memory (no swizzle), K = 64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -shared -Xcompiler -fPIC \
//        tools/tc_probe.cu -o variants/libtcprobe.so
// python: see tools/tc_probe.py
#include <cstdint>
#include <cuda_runtime.h>

namespace {

constexpr int M = 128, K = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// K-major, no swizzle: core matrices of 8 rows x 16 bytes (128 contiguous
// bytes); K-adjacent core matrices LBO = 128 B apart, 8-row groups SBO apart.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout = 0) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;   // version (Blackwell)
    d |= (uint64_t)layout << 61;
    return d;
}
#ifndef PROBE_SW64
#define PROBE_SW64 1
#endif

__device__ __forceinline__ uint32_t make_idesc_s8(int m, int n) {
    uint32_t d = 0;
    d |= 2u << 4;            // C format S32
    d |= 1u << 7;            // A signed 8-bit
    d |= 1u << 10;           // B signed 8-bit
    // a_major = b_major = K (0)
    d |= (uint32_t)(n >> 3) << 17;
    d |= (uint32_t)(m >> 4) << 24;
    return d;
}

template <int N>
__global__ void k_probe(const int8_t* A, const int8_t* B, int32_t* C) {
    __shared__ __align__(1024) int8_t sa[M * K];
    __shared__ __align__(1024) int8_t sb[N * K];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) unsigned long long s_bar;
    const int tid = threadIdx.x, warp = tid >> 5;
    // canonical layout: byte (r, c) -> (r / 8) * SBO + (c / 16) * 128 + (r % 8) * 16 + c % 16
#if PROBE_SW64
    // 64-byte swizzle, K-major: atom = 8 rows x 64 B; 16-B chunk c of row r at c ^ ((r % 8) >> 1)
    constexpr uint32_t SBO = 512;
    auto off = [](int r, int c) { return (r / 8) * 512 + (r % 8) * 64 + (((c / 16) ^ ((r % 8) >> 1)) * 16) + (c % 16); };
#else
    constexpr uint32_t SBO = (K / 16) * 128;
    auto off = [](int r, int c) { return (r / 8) * SBO + (c / 16) * 128 + (r % 8) * 16 + (c % 16); };
#endif
    for (int e = tid; e < M * K; e += blockDim.x) {
        const int r = e / K, c = e % K;
        sa[off(r, c)] = A[e];
    }
    for (int e = tid; e < N * K; e += blockDim.x) {
        const int r = e / K, c = e % K;
        sb[off(r, c)] = B[e];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                     "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    // generic-proxy smem writes -> visible to the tensor core (async proxy)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    if (tid == 0) {
        const uint32_t idesc = make_idesc_s8(M, N);
        for (int kk = 0; kk < K / 32; ++kk) {
#if PROBE_SW64
            const uint64_t da = make_desc(smem_u32(sa) + kk * 32, 16, SBO, 4);
            const uint64_t db = make_desc(smem_u32(sb) + kk * 32, 16, SBO, 4);
#else
            const uint64_t da = make_desc(smem_u32(sa) + kk * 256, 128, SBO);
            const uint64_t db = make_desc(smem_u32(sb) + kk * 256, 128, SBO);
#endif
            const uint32_t acc = kk > 0 ? 1u : 0u;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&s_bar)));
    }
    // wait for the MMAs
    {
        const uint32_t b = smem_u32(&s_bar);
        asm volatile(
            "{\n\t.reg .pred p;\n\tW_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
            "@!p bra W_%=;\n\t}" ::"r"(b));
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // TMEM -> registers: warp w reads lanes 32 w .. 32 w + 31 (row = lane)
    if (warp < 4) {
        for (int c0 = 0; c0 < N; c0 += 8) {
            uint32_t v[8];
            const uint32_t addr = tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                           "=r"(v[6]), "=r"(v[7])
                         : "r"(addr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            const int row = 32 * warp + (tid & 31);
            for (int q = 0; q < 8; ++q) C[row * N + c0 + q] = (int32_t)v[q];
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

}  // namespace

extern "C" int tc_probe(const int8_t* A, const int8_t* B, int32_t* C, int n) {
    int8_t *dA, *dB;
    int32_t* dC;
    cudaMalloc(&dA, M * K);
    cudaMalloc(&dB, n * K);
    cudaMalloc(&dC, M * n * 4);
    cudaMemcpy(dA, A, M * K, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B, n * K, cudaMemcpyHostToDevice);
    if (n == 64) k_probe<64><<<1, 128>>>(dA, dB, dC);
    else if (n == 32) k_probe<32><<<1, 128>>>(dA, dB, dC);
    else return -1;
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(C, dC, M * n * 4, cudaMemcpyDeviceToHost);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dC);
    return (int)e;
}

// tc_peaks.cu -- measured tensor-core rates on this GPU for the scoring
// kernels' roofline (tools/tc_peaks.py drives it):
//   dmma_peak   mma.sync.m8n8k4.f64 (FP64 tensor, the DMMA classify kernel)
//   dfma_peak   FP64 FMA on the CUDA cores
//   i8_rate     tcgen05.mma.cta_group::1.kind::i8, M = 128, operands in shared
//               memory (SS), one CTA per SM issuing back-to-back MMAs of a
//               given N (K = 32): dense int8 rate and cycles per MMA
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC \
//        tools/tc_peaks.cu -o variants/libtcpeaks.so
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__global__ void k_dmma(int iters, double* out) {
    double acc[8][2];
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c][0] = acc[c][1] = 0.0;
    const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
            asm volatile(
                "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                : "+d"(acc[c][0]), "+d"(acc[c][1])
                : "d"(a), "d"(b));
    }
    double t = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) t += acc[c][0] + acc[c][1];
    if (t == 12345.0) out[0] = t;
}

__global__ void k_dfma(int iters, double* out) {
    double x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = threadIdx.x + c;
    const double a = 0.999999, b = 1e-7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) x[c] = fma(x[c], a, b);
    }
    double t = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) t += x[c];
    if (t == 12345.0) out[0] = t;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_sw64(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;                 // LBO 16 B (unused)
    d |= (uint64_t)(512 >> 4) << 32;        // SBO 512 B
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)4 << 61;                 // SWIZZLE_64B
    return d;
}

template <int N>
__global__ void k_i8(int iters, unsigned long long* cycles) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) unsigned long long s_bar;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < (128 + N) * 64; i += blockDim.x) sm[i] = (unsigned char)(i * 7);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                     "r"(N < 32 ? 32 : N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    if (warp == 0) {
        const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
        const uint64_t da = desc_sw64(smem_u32(sm)), db = desc_sw64(smem_u32(sm + 128 * 64));
        uint32_t pred = 0;
        asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
        unsigned long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            if (pred)
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                    "l"(da + (uint64_t)((i & 1) * 2)), "l"(db + (uint64_t)((i & 1) * 2)), "r"(idesc), "r"(i > 0 ? 1u : 0u));
            __syncwarp();
        }
        if (pred)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                smem_u32(&s_bar)));
        __syncwarp();
        asm volatile(
            "{\n\t.reg .pred p;\n\tW_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
            "@!p bra W_%=;\n\t}" ::"r"(smem_u32(&s_bar)));
        const unsigned long long t1 = clock64();
        if (tid == 0) cycles[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(N < 32 ? 32 : N));
}

float time_ms(void (*launch)(void*), void* arg) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch(arg);   // warm-up
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    launch(arg);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ms;
}

struct Arg {
    int iters, grid, block;
    double* out;
    unsigned long long* cyc;
};

}  // namespace

// FP64 tensor (DMMA) TFLOP/s
extern "C" double dmma_peak(int iters) {
    Arg g{iters, 148 * 8, 256, nullptr, nullptr};
    cudaMalloc(&g.out, 8);
    const float ms = time_ms([](void* p) {
        Arg* a = (Arg*)p;
        k_dmma<<<a->grid, a->block>>>(a->iters, a->out);
    }, &g);
    cudaFree(g.out);
    const double flops = 2.0 * 8 * 8 * 4 * 8 * (double)iters * (g.grid * g.block / 32);
    return flops / (ms * 1e-3) / 1e12;
}

// FP64 FMA TFLOP/s
extern "C" double dfma_peak(int iters) {
    Arg g{iters, 148 * 8, 256, nullptr, nullptr};
    cudaMalloc(&g.out, 8);
    const float ms = time_ms([](void* p) {
        Arg* a = (Arg*)p;
        k_dfma<<<a->grid, a->block>>>(a->iters, a->out);
    }, &g);
    cudaFree(g.out);
    const double flops = 2.0 * 8 * (double)iters * g.grid * g.block;
    return flops / (ms * 1e-3) / 1e12;
}

// tcgen05 kind::i8 (M = 128, K = 32, SS operands): dense TOP/s over 148 CTAs
// and the mean cycles per MMA on one SM; n in {32, 64, 128, 256}
extern "C" double i8_rate(int n, int iters, double* cycles_per_mma) {
    Arg g{iters, 148, 128, nullptr, nullptr};
    cudaMalloc(&g.cyc, 148 * sizeof(unsigned long long));
    const int smem = (128 + 256) * 64;
    void (*fn)(void*) = nullptr;
    switch (n) {
        case 32: cudaFuncSetAttribute(k_i8<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            fn = [](void* p) { Arg* a = (Arg*)p; k_i8<32><<<a->grid, a->block, (128 + 256) * 64>>>(a->iters, a->cyc); };
            break;
        case 64: cudaFuncSetAttribute(k_i8<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            fn = [](void* p) { Arg* a = (Arg*)p; k_i8<64><<<a->grid, a->block, (128 + 256) * 64>>>(a->iters, a->cyc); };
            break;
        case 128: cudaFuncSetAttribute(k_i8<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            fn = [](void* p) { Arg* a = (Arg*)p; k_i8<128><<<a->grid, a->block, (128 + 256) * 64>>>(a->iters, a->cyc); };
            break;
        case 256: cudaFuncSetAttribute(k_i8<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            fn = [](void* p) { Arg* a = (Arg*)p; k_i8<256><<<a->grid, a->block, (128 + 256) * 64>>>(a->iters, a->cyc); };
            break;
        default: return -1.0;
    }
    const float ms = time_ms(fn, &g);
    unsigned long long c[148];
    cudaMemcpy(c, g.cyc, sizeof(c), cudaMemcpyDeviceToHost);
    cudaFree(g.cyc);
    double mean = 0.0;
    for (int i = 0; i < 148; ++i) mean += (double)c[i] / 148.0;
    if (cycles_per_mma) *cycles_per_mma = mean / iters;
    const double ops = 2.0 * 128 * n * 32 * (double)iters * 148;
    return ops / (ms * 1e-3) / 1e12;
}

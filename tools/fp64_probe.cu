// Per-SM throughput of the open-set fold's instruction mix on this GPU:
// F2F.F64.F32 (cvt), DADD, DMUL, DDIV and an integer float->double bit
// conversion, each as many independent chains per thread (so the pipe, not
// the latency, is measured).  Prints warp-instructions per cycle per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_probe.cu -o tools/fp64_probe.bin
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096, kChains = 8;

__device__ __forceinline__ double cvt_bits(float f) {
    const unsigned u = __float_as_uint(f);
    const unsigned hi = (((u >> 3) & 0x0FFFFFFFu) + 0x38000000u) | (u & 0x80000000u);
    return __hiloint2double((int)hi, (int)(u << 29));
}

template <int kOp>
__global__ void k_probe(const float* in, double* out, long long* cyc) {
    float f[kChains];
    double acc[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        f[c] = in[(threadIdx.x + c) & 255];
        acc[c] = 0.0;
    }
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            if (kOp == 0) acc[c] += (double)f[c];                   // F2F + DADD
            else if (kOp == 1) acc[c] += acc[c];                    // DADD chain (x8 independent)
            else if (kOp == 2) acc[c] = acc[c] * 1.0000001;         // DMUL
            else if (kOp == 3) acc[c] += cvt_bits(f[c]);            // int convert + DADD
            else if (kOp == 4) acc[c] = 1.0 / (acc[c] + 3.0);       // DDIV (+ DADD)
            else {                                                  // the fold: cvt, dmul, 2 dadd
                const double z = (double)f[c];
                acc[c] += z * z;
            }
            f[c] = __int_as_float(__float_as_int(f[c]) ^ 1);        // keep the cvt in the loop
        }
    }
    const long long t1 = clock64();
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += acc[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int kOp>
void run(const char* name, const float* in, double* out, long long* cyc, int ops_per_elem) {
    const int blocks = 148, threads = 1024;
    k_probe<kOp><<<blocks, threads>>>(in, out, cyc);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    const double warp_elems = (double)(threads / 32) * kIters * kChains;   // per SM
    printf("%-28s %6.3f elements/cycle/SM-warp-units  (%.2f thread-elems/clk/SM)\n", name,
           warp_elems / mx, warp_elems * 32 / mx);
    (void)ops_per_elem;
}

int main() {
    float* in;
    double* out;
    long long* cyc;
    cudaMalloc(&in, 256 * 4);
    cudaMalloc(&out, 148 * 1024 * 8);
    cudaMalloc(&cyc, 148 * 8);
    float h[256];
    for (int i = 0; i < 256; ++i) h[i] = 0.001f * (i + 1);
    cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
    run<1>("DADD", in, out, cyc, 1);
    run<2>("DMUL", in, out, cyc, 1);
    run<0>("F2F.F64.F32 + DADD", in, out, cyc, 2);
    run<3>("int cvt + DADD", in, out, cyc, 2);
    run<5>("fold (cvt, dmul, dadd)", in, out, cyc, 3);
    run<4>("DDIV", in, out, cyc, 1);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

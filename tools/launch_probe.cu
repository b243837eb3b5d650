// Launch-overhead probe: what a frame pays outside its kernel spans.
// Event-timed (after a 256 MiB memset, so the GPU is busy when the host
// enqueues, as in bench.py's L2 flush):
//   a) one empty kernel          b) a graph of one empty kernel
//   c) a graph of 4 empty kernels (PDL edges, as the frame graph)
//   d) c) whose last kernel copies 1 KB to mapped pinned memory + fence.system
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/launch_probe.cu -o /tmp/launch_probe
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__global__ void k_empty(int* p) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] += 1;
}

__global__ void k_tail(int* p, unsigned long long* mirror) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (blockIdx.x == 0) {
        for (int i = threadIdx.x; i < 128; i += blockDim.x) mirror[i] = (unsigned long long)p[0] + i;
        __threadfence_system();
    }
}

static void launch(void (*k)(int*), int grid, cudaStream_t s, int* p, bool pdl) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute at{};
    at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k, p);
}

int main() {
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    void* flush;
    cudaMalloc(&flush, 256 << 20);
    int* p;
    cudaMalloc(&p, 64);
    unsigned long long* mirror;
    cudaHostAlloc(&mirror, 4096, cudaHostAllocMapped);
    unsigned long long* dmirror;
    cudaHostGetDevicePointer((void**)&dmirror, mirror, 0);
    const int grid = 148 * 8;

    auto build = [&](int nk, bool tail) {
        cudaGraph_t g;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        for (int i = 0; i < nk; ++i) launch(k_empty, grid, s, p, i > 0);
        if (tail) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(256);
            cfg.stream = s;
            cudaLaunchAttribute at{};
            at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at.val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = &at;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, k_tail, p, dmirror);
        }
        cudaStreamEndCapture(s, &g);
        cudaGraphExec_t ge;
        cudaGraphInstantiate(&ge, g, 0);
        return ge;
    };
    cudaGraphExec_t g1 = build(1, false), g4 = build(4, false), g4t = build(3, true);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char* names[] = {"plain kernel", "graph 1 kernel", "graph 4 kernels (PDL)",
                           "graph 3 + mapped-tail kernel", "plain kernel, idle GPU",
                           "graph 4 kernels, idle GPU"};
    for (int mode = 0; mode < 6; ++mode) {
        std::vector<float> t;
        for (int it = 0; it < 60; ++it) {
            if (mode < 4) cudaMemsetAsync(flush, it & 1, 256 << 20, s);
            else cudaStreamSynchronize(s);
            cudaEventRecord(a, s);
            if (mode == 0 || mode == 4) launch(k_empty, grid, s, p, false);
            else if (mode == 1) cudaGraphLaunch(g1, s);
            else if (mode == 2 || mode == 5) cudaGraphLaunch(g4, s);
            else cudaGraphLaunch(g4t, s);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (it >= 10) t.push_back(ms * 1000.f);
        }
        std::sort(t.begin(), t.end());
        printf("%-32s median %7.2f us  p10 %7.2f  p90 %7.2f\n", names[mode], t[t.size() / 2],
               t[t.size() / 10], t[t.size() * 9 / 10]);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

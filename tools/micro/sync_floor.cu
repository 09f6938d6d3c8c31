// floor of a synchronous launch->complete round trip, by completion mechanism
#include <cuda_runtime.h>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>

__global__ void k_empty() {}
__global__ void k_flag(volatile unsigned* flag, unsigned v, unsigned* ctr, unsigned nblk) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        if (atomicAdd(ctr, 1u) == nblk - 1) {
            *ctr = 0;
            __threadfence_system();
            *flag = v;
        }
    }
}

template <class F> double bench(const char* name, F f, int n = 20000) {
    for (int i = 0; i < 1000; ++i) f(i);
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < n; ++i) f(i + 1000);
    auto t1 = std::chrono::steady_clock::now();
    double us = std::chrono::duration<double, std::micro>(t1 - t0).count() / n;
    printf("%-44s %.3f us\n", name, us);
    return us;
}

int main(int argc, char** argv) {
    if (argc > 1 && !strcmp(argv[1], "spin")) cudaSetDeviceFlags(cudaDeviceScheduleSpin);
    if (argc > 1 && !strcmp(argv[1], "yield")) cudaSetDeviceFlags(cudaDeviceScheduleYield);
    if (argc > 1 && !strcmp(argv[1], "block")) cudaSetDeviceFlags(cudaDeviceScheduleBlockingSync);
    cudaFree(0);
    unsigned int fl = 0;
    cudaGetDeviceFlags(&fl);
    printf("device flags 0x%x\n", fl);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    unsigned* flag = nullptr;
    cudaHostAlloc(&flag, 64, cudaHostAllocMapped);
    unsigned* ctr = nullptr;
    cudaMalloc(&ctr, 4);
    cudaMemset(ctr, 0, 4);
    bench("empty + cudaStreamSynchronize", [&](int) { k_empty<<<1, 32, 0, s>>>(); cudaStreamSynchronize(s); });
    bench("empty + cudaStreamQuery spin", [&](int) {
        k_empty<<<1, 32, 0, s>>>();
        while (cudaStreamQuery(s) == cudaErrorNotReady) {}
    });
    for (unsigned nb : {1u, 32u, 148u}) {
        char nm[64];
        snprintf(nm, 64, "flag kernel (%u blocks) + host poll", nb);
        bench(nm, [&](int i) {
            k_flag<<<nb, 128, 0, s>>>(flag, (unsigned)i, ctr, nb);
            while (((volatile unsigned*)flag)[0] != (unsigned)i) {}
        });
    }
    bench("flag kernel (32 blocks) + sync", [&](int i) {
        k_flag<<<32, 128, 0, s>>>(flag, (unsigned)i, ctr, 32);
        cudaStreamSynchronize(s);
    });
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    k_empty<<<1, 32, 0, s>>>();
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    bench("graph(empty) + sync", [&](int) { cudaGraphLaunch(ge, s); cudaStreamSynchronize(s); });
    bench("launch only (async, 1 kernel)", [&](int) { k_empty<<<1, 32, 0, s>>>(); }, 20000);
    cudaStreamSynchronize(s);
    return 0;
}

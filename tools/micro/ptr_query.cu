// cost of the per-call host-pointer validation used by the host-ABI step, and of
// an empty-kernel launch + stream sync (the fixed floor of a synchronous step)
#include <cuda.h>
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>

using Fn = CUresult (*)(unsigned, CUpointer_attribute*, void**, CUdeviceptr);
__global__ void k_empty() {}
__global__ void k_touch(const double* in, double* out) { out[threadIdx.x] = in[threadIdx.x] + 1.0; }

int main() {
    void* h = nullptr;
    cudaHostAlloc(&h, 1 << 20, cudaHostAllocDefault);
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuPointerGetAttributes", &f, cudaEnableDefault, &q);
    Fn fn = (Fn)f;
    CUpointer_attribute at[3] = {CU_POINTER_ATTRIBUTE_MEMORY_TYPE, CU_POINTER_ATTRIBUTE_DEVICE_POINTER,
                                 CU_POINTER_ATTRIBUTE_BUFFER_ID};
    unsigned mt; CUdeviceptr dp; unsigned long long id;
    void* data[3] = {&mt, &dp, &id};
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < 100000; ++i) fn(3, at, data, (CUdeviceptr)h);
    auto t1 = std::chrono::steady_clock::now();
    printf("cuPointerGetAttributes x3: %.3f us\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / 1e5);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    for (int i = 0; i < 1000; ++i) { k_empty<<<1, 32, 0, s>>>(); cudaStreamSynchronize(s); }
    t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < 10000; ++i) { k_empty<<<1, 32, 0, s>>>(); cudaStreamSynchronize(s); }
    t1 = std::chrono::steady_clock::now();
    printf("empty launch + sync: %.3f us\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / 1e4);
    double* hd = (double*)h;
    t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < 10000; ++i) { k_touch<<<1, 32, 0, s>>>(hd, hd + 64); cudaStreamSynchronize(s); }
    t1 = std::chrono::steady_clock::now();
    printf("mapped read+write kernel + sync: %.3f us\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / 1e4);
    cudaSetDeviceFlags(cudaDeviceScheduleSpin);
    return 0;
}

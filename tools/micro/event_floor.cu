// GPU-side window between two events bracketing an empty kernel (direct launch vs
// single-node graph), with a long kernel queued before so the host is never the limit
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <vector>

__global__ void k_empty() {}
__global__ void k_fill(float* p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = 0.f;
}

int main() {
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    size_t n = 64 << 20;
    float* buf;
    cudaMalloc(&buf, n * 4);
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    k_empty<<<32, 128, 0, s>>>();
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    const int K = 300;
    std::vector<cudaEvent_t> ev(2 * K);
    for (auto& e : ev) cudaEventCreate(&e);
    for (int mode = 0; mode < 3; ++mode) {
        for (int i = 0; i < K; ++i) {
            k_fill<<<148 * 8, 256, 0, s>>>(buf, n);
            cudaEventRecord(ev[2 * i], s);
            if (mode == 0) k_empty<<<32, 128, 0, s>>>();
            else if (mode == 1) cudaGraphLaunch(ge, s);
            cudaEventRecord(ev[2 * i + 1], s);
        }
        cudaStreamSynchronize(s);
        std::vector<float> t(K);
        for (int i = 0; i < K; ++i) cudaEventElapsedTime(&t[i], ev[2 * i], ev[2 * i + 1]);
        std::sort(t.begin(), t.end());
        const char* nm[] = {"direct launch", "graph launch", "nothing"};
        printf("%-14s median %.2f us  min %.2f us\n", nm[mode], t[K / 2] * 1e3, t[0] * 1e3);
    }
    return 0;
}

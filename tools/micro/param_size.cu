// GPU-side event window around a single-node graph whose kernel takes a small vs a
// 3.3 KB __grid_constant__ parameter block (the step kernel's EngineP size)
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <vector>

struct Small { float a[16]; };
struct Big { float a[840]; };   // ~3.3 KB
__global__ void k_small(const __grid_constant__ Small p, float* out) { if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = p.a[3]; }
__global__ void k_big(const __grid_constant__ Big p, float* out) { if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = p.a[700]; }
__global__ void k_fill(float* p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = 0.f;
}

template <class F> float window(cudaStream_t s, float* buf, size_t n, F launch) {
    const int K = 300;
    std::vector<cudaEvent_t> ev(2 * K);
    for (auto& e : ev) cudaEventCreate(&e);
    for (int i = 0; i < K; ++i) {
        k_fill<<<148 * 8, 256, 0, s>>>(buf, n);
        cudaEventRecord(ev[2 * i], s);
        launch();
        cudaEventRecord(ev[2 * i + 1], s);
    }
    cudaStreamSynchronize(s);
    std::vector<float> t(K);
    for (int i = 0; i < K; ++i) cudaEventElapsedTime(&t[i], ev[2 * i], ev[2 * i + 1]);
    std::sort(t.begin(), t.end());
    return t[K / 2] * 1e3f;
}

int main() {
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    size_t n = 64 << 20;
    float *buf, *out;
    cudaMalloc(&buf, n * 4);
    cudaMalloc(&out, 4);
    Small ps{}; Big pb{};
    cudaGraph_t g1, g2; cudaGraphExec_t e1, e2;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    k_small<<<32, 128, 0, s>>>(ps, out);
    cudaStreamEndCapture(s, &g1);
    cudaGraphInstantiate(&e1, g1, 0);
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    k_big<<<32, 128, 0, s>>>(pb, out);
    cudaStreamEndCapture(s, &g2);
    cudaGraphInstantiate(&e2, g2, 0);
    for (int r = 0; r < 2; ++r) {
        printf("graph small params: %.2f us\n", window(s, buf, n, [&] { cudaGraphLaunch(e1, s); }));
        printf("graph 3.3 KB params: %.2f us\n", window(s, buf, n, [&] { cudaGraphLaunch(e2, s); }));
        printf("direct small: %.2f us\n", window(s, buf, n, [&] { k_small<<<32, 128, 0, s>>>(ps, out); }));
        printf("direct 3.3 KB: %.2f us\n", window(s, buf, n, [&] { k_big<<<32, 128, 0, s>>>(pb, out); }));
    }
    return 0;
}

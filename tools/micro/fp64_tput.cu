// fp64 issue-rate probe (B200): cycles per warp-wide DFMA for ILP = 1..8
// independent chains, with 1, 4 and 8 warps in one CTA (one SM).  clock64.
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void k(double* out, long long* cyc, double a, double b, int n) {
    double x[ILP];
#pragma unroll
    for (int j = 0; j < ILP; ++j) x[j] = a + j + threadIdx.x;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int j = 0; j < ILP; ++j) x[j] = fma(x[j], b, a);
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int j = 0; j < ILP; ++j) s += x[j];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int ILP>
void run(int warps) {
    double* o; long long* c;
    cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 8);
    const int n = 4096;
    for (int rep = 0; rep < 2; ++rep) k<ILP><<<1, 32 * warps>>>(o, c, 0.5, 0.999, n);
    long long h;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("warps %d ILP %d: cycles per DFMA per warp %.2f\n", warps, ILP, h / (double)(n * ILP));
    cudaFree(o); cudaFree(c);
}

int main() {
    for (int w : {1, 4, 8, 16}) { run<1>(w); run<2>(w); run<4>(w); run<8>(w); }
    return 0;
}

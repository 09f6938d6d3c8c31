// fp64 latency probe (B200): dependent-chain cycles per DFMA, per fp64 division,
// per sincos (libdevice), per FFMA for reference.  One thread, clock64.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double* out, long long* cyc, double a, double b, float af, float bf, int n) {
    double x = a;
    float y = af;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, b, a);
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) y = fmaf(y, bf, af);
    long long t2 = clock64();
    double z = a;
    for (int i = 0; i < n; ++i) z = b / (z + 1.5);
    long long t3 = clock64();
    double w = a, s, c;
    for (int i = 0; i < n; ++i) { sincos(w, &s, &c); w = s + c * 0.5; }
    long long t4 = clock64();
    double v = a;
    for (int i = 0; i < n; ++i) v = v * b + a * v;   // DMUL + DFMA
    long long t5 = clock64();
    out[0] = x + y + z + w + v;
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
}

int main() {
    double* o; long long* c;
    cudaMalloc(&o, 8); cudaMalloc(&c, 5 * 8);
    const int n = 4096;
    for (int rep = 0; rep < 2; ++rep) k<<<1, 1>>>(o, c, 0.5, 0.999, 0.5f, 0.999f, n);
    long long h[5];
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    printf("cycles/op: DFMA %.2f  FFMA %.2f  DDIV %.2f  sincos(f64) %.2f  DMUL+DFMA %.2f\n",
           h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n, h[4] / (double)n);
    return 0;
}

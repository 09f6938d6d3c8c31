// Latency of one fp64 band sub-step (substep_f64, Fossen pattern) and of its
// pieces, one thread, clock64 -- the band kernel's replay is a serial chain of
// these.   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I paper_2410_14117_b200/csrc
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>
#include "uuv_model.cuh"

using namespace uuv;
#include "substep64_var.cuh"

template <bool SW, bool LATE>
__global__ void kv(VehP<double> V, double* io, long long* cyc, int n) {
    double s[12], tau[6];
    for (int i = 0; i < 12; ++i) s[i] = io[i];
    for (int i = 0; i < 6; ++i) tau[i] = io[12 + i];
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) substep_var<SW, LATE>(V, s, tau, 0.005);
    long long t1 = clock64();
    for (int i = 0; i < 12; ++i) io[i] = s[i];
    cyc[0] = t1 - t0;
}

template <bool SW, bool LATE>
void runv(const VehP<double>& V, double* io, long long* c, int n) {
    for (int rep = 0; rep < 2; ++rep) kv<SW, LATE><<<1, 1>>>(V, io, c, n);
    long long r;
    cudaMemcpy(&r, c, 8, cudaMemcpyDeviceToHost);
    printf("variant skipwrap=%d late_restore=%d: %.1f cycles per sub-step\n", SW, LATE, r / (double)n);
}

__global__ void k(VehP<double> V, double* io, long long* cyc, int n) {
    double s[12], tau[6];
    for (int i = 0; i < 12; ++i) s[i] = io[i] * (1.0 + 1e-3 * threadIdx.x);
    for (int i = 0; i < 6; ++i) tau[i] = io[12 + i];
    EnvParams<double, false> E;
    const double dt = 0.005;
    unsigned long long g0, g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) substep_f64<false, false>(V, E, s, tau, dt);
    long long t1 = clock64();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    cyc[4] = (long long)(g1 - g0);
    double x = s[4], sn, cs;
    for (int i = 0; i < n; ++i) { sincos64(x, &sn, &cs); x = sn * 0.5 + cs * 0.25; }
    long long t2 = clock64();
    double y = 0.7 + s[3] * 1e-30;
    for (int i = 0; i < n; ++i) y = rcp64(y) * 0.5 + 0.3;
    long long t3 = clock64();
    double z = 2.5 + s[5] * 1e-30;
    for (int i = 0; i < n; ++i) z = wrap_pi64(z + 3.0);
    long long t4 = clock64();
    if (threadIdx.x == 0) for (int i = 0; i < 12; ++i) io[i] = s[i] + x + y + z;
    if (threadIdx.x) return;
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
}

int main() {
    VehP<double> V;
    memset(&V, 0, sizeof(V));
    const double m[6] = {17.0, 24.2, 26.1, 0.28, 0.28, 0.28};
    for (int i = 0; i < 6; ++i) {
        V.mtot[i * 6 + i] = m[i];
        V.kdt[i * 6 + i] = 0.005 / m[i];
        V.dlin[i * 6 + i] = 4.0 + i;
        V.dquad[i] = 18.0 + i;
    }
    V.mtot[0 * 6 + 4] = V.mtot[4 * 6 + 0] = 0.2;
    V.mtot[1 * 6 + 3] = V.mtot[3 * 6 + 1] = -0.2;
    V.kdt[0 * 6 + 4] = V.kdt[4 * 6 + 0] = -1e-5;
    V.kdt[1 * 6 + 3] = V.kdt[3 * 6 + 1] = 1e-5;
    V.wb = -2.0; V.hm[0] = 0.0; V.hm[1] = 0.0; V.hm[2] = -0.3;
    double h[18] = {0.1, 0.2, 0.3, 0.4, 1.3, 0.6, 0.1, 0.05, -0.1, 0.3, 0.9, 0.2,
                    10, 5, -3, 0.5, 0.2, 0.1};
    double* io; long long* c;
    cudaMalloc(&io, sizeof(h)); cudaMalloc(&c, 5 * 8);
    cudaMemcpy(io, h, sizeof(h), cudaMemcpyHostToDevice);
    const int n = 1000;
    for (int lanes : {1, 8, 16, 32}) {
    for (int rep = 0; rep < 2; ++rep) k<<<1, lanes>>>(V, io, c, n);
    long long r[5];
    cudaMemcpy(r, c, sizeof(r), cudaMemcpyDeviceToHost);
    printf("lanes %d: ", lanes);
    printf("cycles per call: substep_f64 %.1f  sincos64 %.1f  rcp64 %.1f  wrap_pi64 %.1f (err %s)\n",
           r[0] / (double)n, r[1] / (double)n, r[2] / (double)n, r[3] / (double)n,
           cudaGetErrorString(cudaGetLastError()));
    printf("substep_f64 loop: %lld cycles in %lld ns (%.3f GHz)\n", r[0], r[4], r[0] / (double)r[4]);
    }
    runv<false, false>(V, io, c, n);
    runv<true, false>(V, io, c, n);
    runv<false, true>(V, io, c, n);
    runv<true, true>(V, io, c, n);
    return 0;
}

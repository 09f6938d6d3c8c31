// Latency of the band kernel's fp64 replay (replay_band64, Fossen, no DR) in
// isolation, one warp, clock64 -- compare with the in-kernel figure from the
// UUV_BAND_CLOCK timeline (tools/band_timeline.py).
#include <cstdio>
#include <cstring>
#include "uuv_kernels.cuh"

using namespace uuv;

struct P2 {
    EngineP<float> p;
    VehP<double> v;
};

__global__ void k(const __grid_constant__ P2 q, float* io, long long* cyc, int reps) {
    float s[12];
    for (int i = 0; i < 12; ++i) s[i] = io[i] * (1.0f + 1e-3f * threadIdx.x);
    double a[MAX_THR];
    for (int i = 0; i < MAX_THR; ++i) a[i] = 0.3 * (i + 1) / MAX_THR;
    V2<double> rec[5];
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        const Band64Out o = replay_band64<false, PatFossen, true>(q.p, q.v, s, rec, a);
        for (int i = 0; i < 12; ++i) s[i] = o.v[i];
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) {
        for (int i = 0; i < 12; ++i) io[i] = s[i];
        cyc[0] = t1 - t0;
    }
}

int main() {
    static P2 q;
    memset(&q, 0, sizeof(q));
    VehP<double>& V = q.v;
    const double m[6] = {17.0, 24.2, 26.1, 0.28, 0.28, 0.28};
    for (int i = 0; i < 6; ++i) {
        V.mtot[i * 6 + i] = m[i];
        V.kdt[i * 6 + i] = 0.005 / m[i];
        V.dlin[i * 6 + i] = 4.0 + i;
        V.dquad[i] = 18.0 + i;
    }
    V.wb = -2.0; V.hm[2] = -0.3;
    V.n_thr = 6;
    for (int t = 0; t < 6; ++t) { V.alloc[(t % 6) * MAX_THR + t] = 1.0; V.kmax[t] = 40.0; }
    q.p.task.n_substeps = 10;
    q.p.sub_dt64 = 0.005;
    float h[12] = {0.1f, 0.2f, 0.3f, 0.4f, 1.3f, 0.6f, 0.1f, 0.05f, -0.1f, 0.3f, 0.9f, 0.2f};
    float* io; long long* c;
    cudaMalloc(&io, sizeof(h)); cudaMalloc(&c, 8);
    cudaMemcpy(io, h, sizeof(h), cudaMemcpyHostToDevice);
    const int reps = 100;
    for (int lanes : {1, 32}) {
        for (int rep = 0; rep < 2; ++rep) k<<<1, lanes>>>(q, io, c, reps);
        long long r;
        cudaMemcpy(&r, c, 8, cudaMemcpyDeviceToHost);
        printf("lanes %d: replay_band64 %.0f cycles (%.1f per sub-step) err %s\n", lanes, r / (double)reps,
               r / (double)reps / 10, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}

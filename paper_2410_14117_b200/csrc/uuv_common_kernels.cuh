// uuv_common_kernels.cuh -- precision-independent kernels (defined once, in k_f32.cu).
#pragma once

#include <cuda_runtime.h>

#include "uuv_common.cuh"

namespace uuv {

template <class IO>
__global__ void k_bench_actions(uint64_t seed, uint64_t env_offset, int n_env, int act_dim,
                                IO* __restrict__ out) {   // batch.py:168-176
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_env * act_dim) return;
    const int e = i / act_dim, j = i % act_dim;
    const double u = u01(draw_u64(seed, env_offset + (uint64_t)e, PURPOSE_BENCH, (uint64_t)j));
    out[i] = (IO)uniform_rn(-1.0, 1.0, u);
}

// deterministic: fixed per-thread strides, fixed-order tree
__global__ void __launch_bounds__(256) k_stats_reduce(double* __restrict__ part, int nblk,
                                                      double* __restrict__ out, int clear) {
    __shared__ double sh[256];
    for (int k = 0; k < NSTAT; ++k) {
        double acc = 0.0;
        for (int b = threadIdx.x; b < nblk; b += 256) acc += part[(size_t)b * NSTAT + k];
        sh[threadIdx.x] = acc;
        __syncthreads();
        for (int w = 128; w > 0; w >>= 1) {
            if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
            __syncthreads();
        }
        if (threadIdx.x == 0) out[k] = sh[0];
        __syncthreads();
    }
    if (clear) {
        __syncthreads();
        for (int i = threadIdx.x; i < nblk * NSTAT; i += 256) part[i] = 0.0;
    }
}


cudaError_t launch_bench_actions(uint64_t seed, uint64_t env_offset, int n_env, int act_dim,
                                 float* out_f32, double* out_f64, cudaStream_t st) {
    const int n = n_env * act_dim;
    if (out_f32) k_bench_actions<float><<<(n + 255) / 256, 256, 0, st>>>(seed, env_offset, n_env, act_dim, out_f32);
    if (out_f64) k_bench_actions<double><<<(n + 255) / 256, 256, 0, st>>>(seed, env_offset, n_env, act_dim, out_f64);
    return cudaGetLastError();
}

cudaError_t launch_stats_reduce(double* part, int nblk, double* out, int clear, cudaStream_t st) {
    k_stats_reduce<<<1, 256, 0, st>>>(part, nblk, out, clear);
    return cudaGetLastError();
}

}  // namespace uuv

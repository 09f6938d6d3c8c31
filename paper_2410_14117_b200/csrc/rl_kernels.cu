// rl_kernels.cu -- fused rollout-loop kernels around the env step (include/uuvsim_rl.h).
//
// The actor-critic parameters (~55 KB fp32) are staged in shared memory once per
// block of 64 envs; the layer scheme is described at k_policy_act.
// Semantics follow paper_2410_14117_b200.rollout (RunningNorm.normalize,
// ActorCritic.forward / log_prob), which restates reference nets.py:31-192.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "uuv_common.cuh"
#include "../../include/uuvsim_rl.h"

namespace uuvrl {

// One thread per env: every lane of a warp reads the same weight float4 from
// shared memory (a broadcast), so each shared-memory wavefront feeds 4 FFMAs in
// all 32 lanes.  Each dense layer keeps its input vector in registers
// (compile-time indices), accumulates every output unit over four independent
// FFMA chains, and parks the tanh outputs in the thread's own activation row
// (stride 68 floats: conflict-free 128-bit accesses), from where the next layer
// loads them back into registers.  (A four-lanes-per-env variant issued 4x the
// shared-memory wavefronts per FFMA and ran 5x slower: MIO-throttled.)
constexpr int BLK = 128;     // envs per block
constexpr int ENVS = BLK;
constexpr int H = 64;        // hidden width (nets.py default)
constexpr int AMAX = 8;      // action dims (thrusters)
constexpr int HROW = H + 4;  // per-thread activation row stride (floats)
constexpr uint64_t PURPOSE_POLICY = 3;   // counter-RNG purpose for exploration noise

// shared-memory layout (floats), DP = padded obs dim
template <int DP> struct Lay {
    static constexpr int a1w = 0, a1b = a1w + H * DP, a2w = a1b + H, a2b = a2w + H * H;
    static constexpr int amw = a2b + H, amb = amw + AMAX * H;
    static constexpr int c1w = amb + AMAX, c1b = c1w + H * DP, c2w = c1b + H, c2b = c2w + H * H;
    static constexpr int cvw = c2b + H, cvb = cvw + H, ls = cvb + 4;
    static constexpr int nmean = ls + AMAX;                 // doubles from here: mean, scale
    static constexpr int hrow = nmean + 2 * 2 * DP;         // per-thread activation rows
    static constexpr int total = hrow + BLK * HROW;
    static_assert(DP % 4 == 0 && nmean % 4 == 0 && hrow % 4 == 0, "16-byte alignment");
};

__device__ __forceinline__ void stage(float* dst, const float* src, int rows, int cols, int ld) {
    // dst [rows][ld] zero-padded beyond cols
    for (int i = threadIdx.x; i < rows * ld; i += blockDim.x) {
        const int r = i / ld, c = i - r * ld;
        dst[i] = c < cols ? src[r * cols + c] : 0.0f;
    }
}

// out_row[j] = tanh(b[j] + W[j] . in), j < N; W rows of K floats (K % 4 == 0)
template <int K>
__device__ __forceinline__ void dense_tanh(const float (&in)[K], const float* __restrict__ W,
                                           const float* __restrict__ b, float* out_row, int N) {
#pragma unroll 2
    for (int j = 0; j < N; ++j) {
        const float4* w4 = reinterpret_cast<const float4*>(W + j * K);
        float c0 = b[j], c1 = 0.0f, c2 = 0.0f, c3 = 0.0f;
#pragma unroll
        for (int k = 0; k < K / 4; ++k) {
            const float4 w = w4[k];
            c0 = fmaf(w.x, in[4 * k + 0], c0);
            c1 = fmaf(w.y, in[4 * k + 1], c1);
            c2 = fmaf(w.z, in[4 * k + 2], c2);
            c3 = fmaf(w.w, in[4 * k + 3], c3);
        }
        out_row[j] = tanhf((c0 + c1) + (c2 + c3));
    }
}

__device__ __forceinline__ void load_row(const float* row, float (&h)[H]) {
    const float4* r4 = reinterpret_cast<const float4*>(row);
#pragma unroll
    for (int k = 0; k < H / 4; ++k) {
        const float4 v = r4[k];
        h[4 * k] = v.x; h[4 * k + 1] = v.y; h[4 * k + 2] = v.z; h[4 * k + 3] = v.w;
    }
}

__device__ __forceinline__ float dot64(const float (&h)[H], const float* __restrict__ w) {
    const float4* w4 = reinterpret_cast<const float4*>(w);
    float c0 = 0.0f, c1 = 0.0f, c2 = 0.0f, c3 = 0.0f;
#pragma unroll
    for (int k = 0; k < H / 4; ++k) {
        const float4 v = w4[k];
        c0 = fmaf(v.x, h[4 * k], c0);
        c1 = fmaf(v.y, h[4 * k + 1], c1);
        c2 = fmaf(v.z, h[4 * k + 2], c2);
        c3 = fmaf(v.w, h[4 * k + 3], c3);
    }
    return (c0 + c1) + (c2 + c3);
}

template <int DP>
__global__ void __launch_bounds__(BLK, 2) k_policy_act(const UuvRlPolicyArgs a) {
    using L = Lay<DP>;
    extern __shared__ float4 smem4[];
    float* sm = reinterpret_cast<float*>(smem4);
    const int D = (int)a.obs_dim, A = (int)a.act_dim;
    const bool value_only = (a.flags & 4) != 0;
    stage(sm + L::c1w, a.c1w, H, D, DP);
    stage(sm + L::c2w, a.c2w, H, H, H);
    stage(sm + L::cvw, a.cvw, 1, H, H);
    if (!value_only) {
        stage(sm + L::a1w, a.a1w, H, D, DP);
        stage(sm + L::a2w, a.a2w, H, H, H);
        stage(sm + L::amw, a.amw, A, H, H);
        for (int i = threadIdx.x; i < (AMAX - A) * H; i += blockDim.x) sm[L::amw + A * H + i] = 0.0f;
    }
    for (int i = threadIdx.x; i < H; i += blockDim.x) {
        sm[L::a1b + i] = value_only ? 0.0f : a.a1b[i];
        sm[L::a2b + i] = value_only ? 0.0f : a.a2b[i];
        sm[L::c1b + i] = a.c1b[i];
        sm[L::c2b + i] = a.c2b[i];
    }
    if (threadIdx.x < AMAX) {
        sm[L::amb + threadIdx.x] = (!value_only && (int)threadIdx.x < A) ? a.amb[threadIdx.x] : 0.0f;
        sm[L::ls + threadIdx.x] = (int)threadIdx.x < A ? a.log_std[threadIdx.x] : 0.0f;
    }
    if (threadIdx.x == 0) sm[L::cvb] = a.cvb[0];
    double* nm = reinterpret_cast<double*>(sm + L::nmean);
    if ((int)threadIdx.x < DP) {   // mean and 1/sqrt(var + 1e-8) in fp64 (RunningNorm.normalize)
        const int d = threadIdx.x;
        nm[d] = d < D ? a.norm_mean[d] : 0.0;
        nm[DP + d] = d < D ? 1.0 / sqrt(a.norm_var[d] + 1e-8) : 0.0;
    }
    __syncthreads();

    const uint64_t e = (uint64_t)blockIdx.x * BLK + threadIdx.x;
    const bool active = e < a.num_envs;
    float* hrow = sm + L::hrow + threadIdx.x * HROW;
    float x[DP];
#pragma unroll
    for (int k = 0; k < DP; ++k) x[k] = (active && k < D) ? a.obs[e * D + k] : 0.0f;

    if (a.flags & 2) {   // per-block sums for the normaliser update (raw obs, fp64)
#pragma unroll
        for (int k = 0; k < DP; ++k) hrow[k] = x[k];
        __syncthreads();
        if ((int)threadIdx.x < D) {
            const int d = threadIdx.x;
            const uint64_t left = a.num_envs - (uint64_t)blockIdx.x * BLK;
            const int nvalid = left < (uint64_t)BLK ? (int)left : BLK;
            double s = 0.0, q = 0.0;
            for (int r = 0; r < nvalid; ++r) {
                const double v = sm[L::hrow + r * HROW + d];
                s += v;
                q += v * v;
            }
            a.stats_part[(size_t)blockIdx.x * 2 * D + d] = s;
            a.stats_part[(size_t)blockIdx.x * 2 * D + D + d] = q;
        }
        __syncthreads();
    }
    // normalise + clip (fp64 like RunningNorm.normalize), policy input in fp32
    float z[DP];
#pragma unroll
    for (int k = 0; k < DP; ++k) {
        double t = ((double)x[k] - nm[k]) * nm[DP + k];
        t = fmin(fmax(t, -a.norm_clip), a.norm_clip);
        z[k] = k < D ? (float)t : 0.0f;
    }
    if (active && a.nobs_out) {
#pragma unroll
        for (int k = 0; k < DP; ++k)
            if (k < D) a.nobs_out[e * D + k] = z[k];
    }

    float h[H];
    // critic: value = cv . tanh(c2 tanh(c1 z)) + cvb
    dense_tanh<DP>(z, sm + L::c1w, sm + L::c1b, hrow, H);
    load_row(hrow, h);
    dense_tanh<H>(h, sm + L::c2w, sm + L::c2b, hrow, H);
    load_row(hrow, h);
    const float value = dot64(h, sm + L::cvw) + sm[L::cvb];
    if (value_only) {
        if (active && a.value_out) a.value_out[e] = value;
        return;
    }
    // actor: mean = tanh(am tanh(a2 tanh(a1 z)) + amb)
    dense_tanh<DP>(z, sm + L::a1w, sm + L::a1b, hrow, H);
    load_row(hrow, h);
    dense_tanh<H>(h, sm + L::a2w, sm + L::a2b, hrow, H);
    load_row(hrow, h);
    if (!active) return;
    const uint64_t ctr = a.noise_ctr ? *a.noise_ctr : 0;
    const uint64_t g = a.env_offset + e;
    float logp = 0.0f;
#pragma unroll
    for (int p = 0; p < AMAX / 2; ++p) {
        float eps0 = 0.0f, eps1 = 0.0f;
        if ((a.flags & 1) && 2 * p < A) {   // Box-Muller on a counter-based stream
            const uint64_t bits = uuv::draw_u64(a.seed, g, PURPOSE_POLICY, ctr * (AMAX / 2) + p);
            const float u1 = ((float)(uint32_t)(bits >> 40) + 0.5f) * 5.9604644775390625e-08f;
            const float u2 = (float)(uint32_t)(bits & 0xffffffu) * 5.9604644775390625e-08f;
            const float r = sqrtf(-2.0f * __logf(u1));
            float sn, cs;
            __sincosf(6.28318530717958647f * u2, &sn, &cs);
            eps0 = r * cs;
            eps1 = r * sn;
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int i = 2 * p + q;
            if (i >= A) break;
            const float mean = tanhf(dot64(h, sm + L::amw + i * H) + sm[L::amb + i]);
            const float lsd = sm[L::ls + i];
            const float raw = fmaf(expf(lsd), q ? eps1 : eps0, mean);
            const float zz = (raw - mean) * expf(-lsd);      // ActorCritic.log_prob
            logp += -0.5f * zz * zz - lsd - 0.918938533204672742f;
            if (a.raw_out) a.raw_out[e * A + i] = raw;
            if (a.act_out) a.act_out[e * A + i] = fminf(fmaxf(raw, -1.0f), 1.0f);
        }
    }
    if (a.logp_out) a.logp_out[e] = logp;
    if (a.value_out) a.value_out[e] = value;
}

__global__ void k_rl_post(const UuvRlPostArgs a) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < a.num_envs) {
        if (a.rew_in && a.rew_out) a.rew_out[e] = a.rew_in[e];
        if (a.done_in && a.done_out) a.done_out[e] = a.done_in[e] ? 1.0f : 0.0f;
    }
    if (blockIdx.x != 0) return;
    __shared__ double tot_sh;
    __shared__ double sums[2 * 36];
    const int D = (int)a.obs_dim;
    const double n = (double)a.num_envs;
    if (a.n_part > 0) {   // RunningNorm.update: parallel-variance merge (nets.py:177-188)
        // one warp per (sum, dim) column: lanes stride the partial rows, then a
        // fixed shuffle tree -- deterministic and ~n_part/32 dependent loads deep
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
        for (int col = warp; col < 2 * D; col += nw) {
            double v = 0.0;
            for (uint32_t b = lane; b < a.n_part; b += 32) v += a.stats_part[(size_t)b * 2 * D + col];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) sums[col] = v;
        }
        __syncthreads();
        const double cnt = *a.norm_count;
        const double tot = cnt + n;
        if ((int)threadIdx.x < D) {
            const int d = threadIdx.x;
            const double s = sums[d], q = sums[D + d];
            const double bm = s / n;
            const double bv = fmax(q / n - bm * bm, 0.0);
            const double m = a.norm_mean[d], v = a.norm_var[d];
            const double delta = bm - m;
            const double m2 = v * cnt + bv * n + delta * delta * (cnt * n / tot);
            a.norm_mean[d] = m + delta * (n / tot);
            a.norm_var[d] = m2 / tot;
        }
        if (threadIdx.x == 0) tot_sh = tot;
        __syncthreads();
        if (threadIdx.x == 0) *a.norm_count = tot_sh;
    }
    if (threadIdx.x == 0 && a.noise_ctr) *a.noise_ctr += 1;
}

template <int DP> static cudaError_t launch_policy(const UuvRlPolicyArgs& a, cudaStream_t st) {
    const size_t smem = (size_t)Lay<DP>::total * sizeof(float);
    static bool once = (cudaFuncSetAttribute(k_policy_act<DP>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem),
                        true);
    (void)once;
    const unsigned grid = (unsigned)((a.num_envs + ENVS - 1) / ENVS);
    k_policy_act<DP><<<grid, BLK, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace uuvrl

extern "C" {

uint32_t uuvsim_rl_policy_blocks(uint64_t num_envs) {
    return (uint32_t)((num_envs + uuvrl::ENVS - 1) / uuvrl::ENVS);
}

int32_t uuvsim_rl_policy_act(const UuvRlPolicyArgs* a, uint64_t stream) {
    if (!a || a->num_envs == 0 || a->obs_dim == 0 || a->obs_dim > 36 || a->act_dim == 0 ||
        a->act_dim > uuvrl::AMAX || a->hidden != uuvrl::H || !a->obs || !a->norm_mean ||
        !a->norm_var || !a->a1w || !a->c1w || !a->c2w || !a->cvw ||
        ((a->flags & 2) && !a->stats_part))
        return 3;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const cudaError_t e = a->obs_dim <= 12 ? uuvrl::launch_policy<12>(*a, st)
                                           : uuvrl::launch_policy<36>(*a, st);
    return e == cudaSuccess ? 0 : 4;
}

int32_t uuvsim_rl_post(const UuvRlPostArgs* a, uint64_t stream) {
    if (!a || a->num_envs == 0 || a->obs_dim > 36 || (a->n_part && (!a->stats_part ||
        !a->norm_mean || !a->norm_var || !a->norm_count)))
        return 3;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, (a->num_envs + 255) / 256);
    uuvrl::k_rl_post<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(*a);
    return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

}  // extern "C"

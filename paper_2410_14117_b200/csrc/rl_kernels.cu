// rl_kernels.cu -- fused rollout-loop kernels around the env step (include/uuvsim_rl.h).
//
// The actor-critic parameters (~55 KB fp32) are staged in shared memory once per
// block of 64 envs; the work split is described below.
// Semantics follow paper_2410_14117_b200.rollout (RunningNorm.normalize,
// ActorCritic.forward / log_prob), which restates reference nets.py:31-192.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "uuv_common.cuh"
#include "../../include/uuvsim_rl.h"

namespace uuvrl {

// Work split: a block holds 64 envs and 8 warps; warp w works on env half w >> 2
// (lane = env) and on PART p = w & 3 of every layer (hidden units j = 16 p .. 16 p
// + 15, action dims p and p + 4).  All lanes of a warp therefore read the same
// weight float4 (a shared-memory broadcast feeding 4 FFMAs in 32 lanes), and a
// 16k-env batch runs 2,048 warps with a 4x shorter serial chain each than one
// thread per env (measured 2.7x faster; splitting an env over lanes instead
// multiplied the shared-memory wavefronts and was MIO-bound).  Layer inputs come
// from the env's activation row in shared memory (stride 68 floats: the 32 lanes'
// 128-bit row loads are conflict-free); outputs go back to the row, with a block
// barrier between layers.
constexpr int ENVS = 64;            // envs per block
constexpr int BLK = 4 * ENVS;       // threads per block (8 warps)
constexpr int H = 64;               // hidden width (nets.py default)
constexpr int AMAX = 8;             // action dims (thrusters)
constexpr int RS = H + 4;           // activation row stride
constexpr uint64_t PURPOSE_POLICY = 3;   // counter-RNG purpose for exploration noise

template <int DP> struct Lay {
    static constexpr int a1w = 0, a1b = a1w + H * DP, a2w = a1b + H, a2b = a2w + H * H;
    static constexpr int amw = a2b + H, amb = amw + AMAX * H;
    static constexpr int c1w = amb + AMAX, c1b = c1w + H * DP, c2w = c1b + H, c2b = c2w + H * H;
    static constexpr int cvw = c2b + H, cvb = cvw + H, ls = cvb + 4;
    static constexpr int nmean = ls + AMAX;                 // doubles: mean[DP], scale[DP]
    static constexpr int rows = nmean + 2 * 2 * DP;         // activation rows A, B [2][ENVS][RS]
    static constexpr int zrows = rows + 2 * ENVS * RS;      // normalised obs [ENVS][DP + 4]
    static constexpr int red = zrows + ENVS * (DP + 4);     // per-part partials [4][ENVS]
    static constexpr int total = red + 4 * ENVS;
    static_assert(DP % 4 == 0 && nmean % 4 == 0 && rows % 4 == 0 && zrows % 4 == 0, "align");
};

// dst [rows][ld] <- src [rows][cols], zero-padded (cols, ld multiples of 4)
__device__ __forceinline__ void stage(float* dst, const float* src, int rows, int cols, int ld) {
    const int c4 = ld / 4;
    for (int i = threadIdx.x; i < rows * c4; i += blockDim.x) {
        const int r = i / c4, c = (i - r * c4) * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (c + 3 < cols) v = *reinterpret_cast<const float4*>(src + r * cols + c);
        else if (c < cols) {
            v.x = src[r * cols + c];
            if (c + 1 < cols) v.y = src[r * cols + c + 1];
            if (c + 2 < cols) v.z = src[r * cols + c + 2];
        }
        reinterpret_cast<float4*>(dst)[i] = v;
    }
}

// this part's units j = 16 p + jj of tanh(b + W in) -> out_row; the input row lives
// in shared memory and streams through in float4 steps (a short loop body, so the
// code stays in the instruction cache), W rows of K floats are broadcast reads
template <int K>
__device__ __forceinline__ void dense16(const float* in_row, const float* __restrict__ W,
                                        const float* __restrict__ b, int p, float* out_row) {
    float acc[16];
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) acc[jj] = b[16 * p + jj];
    const float4* W4 = reinterpret_cast<const float4*>(W + 16 * p * K);
    const float4* x4 = reinterpret_cast<const float4*>(in_row);
#pragma unroll 2
    for (int k = 0; k < K / 4; ++k) {
        const float4 x = x4[k];
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
            const float4 w = W4[jj * (K / 4) + k];
            acc[jj] = fmaf(w.x, x.x, acc[jj]);
            acc[jj] = fmaf(w.y, x.y, acc[jj]);
            acc[jj] = fmaf(w.z, x.z, acc[jj]);
            acc[jj] = fmaf(w.w, x.w, acc[jj]);
        }
    }
    float4* r4 = reinterpret_cast<float4*>(out_row + 16 * p);
#pragma unroll
    for (int q = 0; q < 4; ++q)
        r4[q] = make_float4(tanhf(acc[4 * q]), tanhf(acc[4 * q + 1]), tanhf(acc[4 * q + 2]),
                            tanhf(acc[4 * q + 3]));
}

template <int K>
__device__ __forceinline__ void get_row(const float* row, float (&h)[K]) {
    const float4* r4 = reinterpret_cast<const float4*>(row);
#pragma unroll
    for (int k = 0; k < K / 4; ++k) {
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
    if (!value_only) {
        stage(sm + L::a1w, a.a1w, H, D, DP);
        stage(sm + L::a2w, a.a2w, H, H, H);
        for (int i = threadIdx.x; i < AMAX * H; i += blockDim.x) {
            const int r = i / H;
            sm[L::amw + i] = r < A ? a.amw[i] : 0.0f;
        }
    }
    for (int i = threadIdx.x; i < H; i += blockDim.x) {
        sm[L::a1b + i] = value_only ? 0.0f : a.a1b[i];
        sm[L::a2b + i] = value_only ? 0.0f : a.a2b[i];
        sm[L::c1b + i] = a.c1b[i];
        sm[L::c2b + i] = a.c2b[i];
        sm[L::cvw + i] = a.cvw[i];
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
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int p = warp & 3;                       // part of every layer
    const int le = ((warp >> 2) << 5) + lane;     // env within the block
    const uint64_t e = (uint64_t)blockIdx.x * ENVS + le;
    const bool active = e < a.num_envs;
    float* row = sm + L::rows + le * RS;
    float* zrow = sm + L::zrows + le * (DP + 4);
    float* red = sm + L::red;                     // [4][ENVS]
    if (p == 0) {   // part 0 loads the raw obs row; the normalised row is shared via zrow
#pragma unroll
        for (int k = 0; k < DP; ++k) row[k] = (active && k < D) ? a.obs[e * D + k] : 0.0f;
    }
    __syncthreads();

    if ((a.flags & 2) && (int)threadIdx.x < D) {   // per-block sums of the raw obs (fp64)
        const int d = threadIdx.x;
        const uint64_t left = a.num_envs - (uint64_t)blockIdx.x * ENVS;
        const int nvalid = left < (uint64_t)ENVS ? (int)left : ENVS;
        double s = 0.0, q = 0.0;
        for (int r = 0; r < nvalid; ++r) {
            const double v = sm[L::rows + r * RS + d];
            s += v;
            q += v * v;
        }
        a.stats_part[(size_t)blockIdx.x * 2 * D + d] = s;
        a.stats_part[(size_t)blockIdx.x * 2 * D + D + d] = q;
    }
    if (p == 0) {   // normalise + clip in fp64 like RunningNorm.normalize; fp32 policy input
#pragma unroll
        for (int k = 0; k < DP; ++k) {
            double t = ((double)row[k] - nm[k]) * nm[DP + k];
            t = fmin(fmax(t, -a.norm_clip), a.norm_clip);
            const float zk = k < D ? (float)t : 0.0f;
            zrow[k] = zk;
            if (active && a.nobs_out && k < D) a.nobs_out[e * D + k] = zk;
        }
    }
    __syncthreads();

    float* rowB = row + ENVS * RS;
    // critic: value = cv . tanh(c2 tanh(c1 z)) + cvb
    dense16<DP>(zrow, sm + L::c1w, sm + L::c1b, p, row);
    __syncthreads();
    dense16<H>(row, sm + L::c2w, sm + L::c2b, p, rowB);
    __syncthreads();
    {
        float v = 0.0f;
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) v = fmaf(sm[L::cvw + 16 * p + jj], rowB[16 * p + jj], v);
        red[p * ENVS + le] = v;
    }
    __syncthreads();
    const float value = ((red[le] + red[ENVS + le]) + (red[2 * ENVS + le] + red[3 * ENVS + le])) +
                        sm[L::cvb];
    if (value_only) {
        if (active && p == 0 && a.value_out) a.value_out[e] = value;
        return;
    }
    // actor: mean = tanh(am tanh(a2 tanh(a1 z)) + amb)
    dense16<DP>(zrow, sm + L::a1w, sm + L::a1b, p, row);
    __syncthreads();                 // (also orders the value reads of red before reuse)
    dense16<H>(row, sm + L::a2w, sm + L::a2b, p, rowB);
    __syncthreads();
    float h[H];
    get_row<H>(rowB, h);
    // action dims p and p + 4: one Box-Muller pair per (env, part)
    float eps[2] = {0.0f, 0.0f};
    if (a.flags & 1) {
        const uint64_t ctr = a.noise_ctr ? *a.noise_ctr : 0;
        const uint64_t bits = uuv::draw_u64(a.seed, a.env_offset + e, PURPOSE_POLICY,
                                            ctr * 4 + (uint64_t)p);
        const float u1 = ((float)(uint32_t)(bits >> 40) + 0.5f) * 5.9604644775390625e-08f;
        const float u2 = (float)(uint32_t)(bits & 0xffffffu) * 5.9604644775390625e-08f;
        const float r = sqrtf(-2.0f * __logf(u1));
        float sn, cs;
        __sincosf(6.28318530717958647f * u2, &sn, &cs);
        eps[0] = r * cs;
        eps[1] = r * sn;
    }
    float lp = 0.0f;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int i = p + 4 * q;
        if (i < A) {
            const float mean = tanhf(dot64(h, sm + L::amw + i * H) + sm[L::amb + i]);
            const float lsd = sm[L::ls + i];
            const float raw = fmaf(expf(lsd), eps[q], mean);
            const float zz = (raw - mean) * expf(-lsd);      // ActorCritic.log_prob
            lp += -0.5f * zz * zz - lsd - 0.918938533204672742f;
            if (active && a.raw_out) a.raw_out[e * A + i] = raw;
            if (active && a.act_out) a.act_out[e * A + i] = fminf(fmaxf(raw, -1.0f), 1.0f);
        }
    }
    red[p * ENVS + le] = lp;
    __syncthreads();
    if (active && p == 0) {
        const float logp = (red[le] + red[ENVS + le]) + (red[2 * ENVS + le] + red[3 * ENVS + le]);
        if (a.logp_out) a.logp_out[e] = logp;
        if (a.value_out) a.value_out[e] = value;
    }
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
#pragma unroll 8
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
    const unsigned grid = (unsigned)std::max<uint64_t>(1, (a->num_envs + 1023) / 1024);
    uuvrl::k_rl_post<<<grid, 1024, 0, reinterpret_cast<cudaStream_t>(stream)>>>(*a);
    return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

}  // extern "C"

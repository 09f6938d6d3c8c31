// rl_kernels.cu -- fused rollout-loop kernels around the env step (include/uuvsim_rl.h).
//
// The actor-critic parameters (~55 KB fp32) are staged in shared memory once per
// block of 64 envs; the work split is described below.
// Semantics follow paper_2410_14117_b200.rollout (RunningNorm.normalize,
// ActorCritic.forward / log_prob), which restates reference nets.py:31-192.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>

#include "uuv_common.cuh"
#include "launch_kernel.cuh"
#include "../../include/uuvsim_rl.h"

#ifndef UUV_PDL_TRIGGER
#define UUV_PDL_TRIGGER 0   // explicit dependents trigger: off (see launch.h)
#endif

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
        if ((cols & 3) == 0 && c + 3 < cols) {   // rows start 16-byte aligned
            v = *reinterpret_cast<const float4*>(src + r * cols + c);
        } else if (c < cols) {
            if (c + 3 < cols) v.w = src[r * cols + c + 3];
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
    if (a.flags & 1) {   // programmatic dependent launch (see k_policy_tc)
        if (UUV_PDL_TRIGGER >= 1) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    if (blockIdx.x != 0) {   // blocks 1.. copy reward / done; block 0 merges the statistics
        const uint64_t e = (uint64_t)(blockIdx.x - 1) * blockDim.x + threadIdx.x;
        if (e < a.num_envs) {
            const float r = a.rew_in && a.rew_out ? a.rew_in[e] : 0.0f;
            const uint8_t d = a.done_in && a.done_out ? a.done_in[e] : 0;
            if (a.rew_in && a.rew_out) a.rew_out[e] = r;
            if (a.done_in && a.done_out) a.done_out[e] = d ? 1.0f : 0.0f;
        }
        return;
    }
    __shared__ double tot_sh;
    __shared__ double sums[2 * 36];
    const int D = (int)a.obs_dim;
    const double n = (double)a.num_envs;
    if (a.n_part > 0) {   // RunningNorm.update: parallel-variance merge (nets.py:177-188)
        // the running statistics are read up front (one round trip with the sums)
        const bool owner = (int)threadIdx.x < D;
        const double cnt = *a.norm_count;
        const double m = owner ? a.norm_mean[threadIdx.x] : 0.0;
        const double v = owner ? a.norm_var[threadIdx.x] : 0.0;
        // the partial rows are row-major [n_part][2 D]: thread (g, c) sums column c
        // over rows g, g + G, g + 2 G, ... (G = blockDim / 2 D groups) -- each
        // row read by consecutive threads (coalesced), every load of a batch in
        // flight before the adds -- then the G group sums of a column are added
        // in group order (fixed order: deterministic)
        __shared__ double gsum[1024];
        const int ncol = 2 * D, ngrp = (int)blockDim.x / ncol;
        const int g = (int)threadIdx.x / ncol, c = (int)threadIdx.x - g * ncol;
        if (g < ngrp) {
            constexpr int RPT = 8;
            double part = 0.0;
            for (uint32_t r0 = (uint32_t)g; r0 < a.n_part; r0 += (uint32_t)(RPT * ngrp)) {
                double x[RPT];
#pragma unroll
                for (int j = 0; j < RPT; ++j) {
                    const uint32_t r = r0 + (uint32_t)(j * ngrp);
                    x[j] = r < a.n_part ? a.stats_part[(size_t)r * ncol + c] : 0.0;
                }
#pragma unroll
                for (int j = 0; j < RPT; ++j) part += x[j];
            }
            gsum[threadIdx.x] = part;
        }
        __syncthreads();
        if ((int)threadIdx.x < ncol) {
            double t = 0.0;
            for (int q = 0; q < ngrp; ++q) t += gsum[q * ncol + threadIdx.x];
            sums[threadIdx.x] = t;
        }
        __syncthreads();
        const double tot = cnt + n;
        if (owner) {
            const int d = threadIdx.x;
            const double s = sums[d], q = sums[D + d];
            const double bm = s / n;
            const double bv = fmax(q / n - bm * bm, 0.0);
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

// dynamic shared memory opt-in, once per kernel and device (attributes are per
// device context)
template <auto KERNEL> static void smem_optin(int bytes) {
    static std::atomic<uint64_t> done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return;
    cudaFuncSetAttribute(KERNEL, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    done.fetch_or(bit, std::memory_order_release);
}

template <int DP> static cudaError_t launch_policy(const UuvRlPolicyArgs& a, cudaStream_t st) {
    const size_t smem = (size_t)Lay<DP>::total * sizeof(float);
    smem_optin<k_policy_act<DP>>((int)smem);
    const unsigned grid = (unsigned)((a.num_envs + ENVS - 1) / ENVS);
    k_policy_act<DP><<<grid, BLK, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace uuvrl

// ============================================================================
// Tensor-core policy kernel (tcgen05, sm_100a).
//
// A CTA holds M = 128 envs = one UMMA tile row block.  Every dense layer of both
// trunks is D[128 x 64] = A[128 x K] B[64 x K]^T on the 5th-generation tensor
// cores: A (normalised obs, then hidden activations) and B (weights) sit in
// shared memory in the K-major, no-swizzle UMMA core-matrix layout (8 rows x 16 B
// per core matrix), the fp32 accumulator in TMEM (64 columns), and one elected
// thread issues kind::tf32 MMAs, K = 8 per instruction.  fp32 accuracy comes from
// the 3xTF32 split: x = x_hi + x_lo with x_hi = tf32(x), and
// A B ~= A_hi B_hi + A_hi B_lo + A_lo B_hi (error ~1e-7 relative, vs ~5e-4 for
// one TF32 pass).  The weights are split and laid out once per parameter update
// by k_rl_prepare into a global "image" that each CTA pulls into shared memory
// with ONE cp.async.bulk while it normalises its observations.  Epilogues: one
// thread per env reads its TMEM row (tcgen05.ld 32x32b), adds the bias, applies
// tanh and writes the next layer's A operand (hi/lo) back to shared memory; the
// scalar heads (value, 8 action means), sampling and log-prob stay on the CUDA
// cores as in the FFMA kernel.
// ============================================================================
namespace uuvtc {

constexpr int M = 128, H = 64, AMAX = 8;
constexpr uint32_t IDESC_TF32 = (1u << 4)      // D format f32
                              | (2u << 7)      // A format tf32
                              | (2u << 10)     // B format tf32
                              | ((uint32_t)(H >> 3) << 17)    // N = 64
                              | ((uint32_t)(M >> 4) << 24);   // M = 128
// small-parameter block (floats) at the end of the image
constexpr int S_B1C = 0, S_B2C = 64, S_CV = 128, S_CVB = 192, S_B1A = 196, S_B2A = 260,
              S_AM = 324, S_AMB = 836, S_LS = 844, S_N = 852;

__host__ __device__ constexpr int k1p(int D) { return (D + 7) / 8 * 8; }
struct Img {
    uint32_t k1, w1c_hi, w1c_lo, w2c_hi, w2c_lo, w1a_hi, w1a_lo, w2a_hi, w2a_lo, small, total;
};
__host__ __device__ inline Img img_layout(int D) {
    Img g{};
    g.k1 = (uint32_t)k1p(D);
    const uint32_t m1 = H * g.k1 * 4, m2 = H * H * 4;
    uint32_t o = 0;
    g.w1c_hi = o; o += m1; g.w1c_lo = o; o += m1; g.w2c_hi = o; o += m2; g.w2c_lo = o; o += m2;
    g.w1a_hi = o; o += m1; g.w1a_lo = o; o += m1; g.w2a_hi = o; o += m2; g.w2a_lo = o; o += m2;
    g.small = o;
    o += S_N * 4;
    g.total = (o + 15) / 16 * 16;
    return g;
}
// byte offset of element (row, k) in a K-major core-matrix tile with KC = K / 4
__host__ __device__ inline uint32_t cm_off(int row, int k, int KC) {
    return (uint32_t)((((row >> 3) * KC + (k >> 2)) << 7) + ((row & 7) << 4) + ((k & 3) << 2));
}

#ifndef UUV_TC_STOP
#define UUV_TC_STOP 0   // phase probe (tools/c4_loop_probe.py): 1-4 return after that phase
#endif
#define UUV_TC_EXIT_AFTER(n)                                                                    \
    if (UUV_TC_STOP == (n)) {                                                                 \
        tc_fence_before();                                                                    \
        __syncthreads();                                                                      \
        if (warp == 0)                                                                        \
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem)); \
        return;                                                                               \
    }

#ifndef UUV_TC_FAST_TANH
#define UUV_TC_FAST_TANH 1
#endif
// epilogue tanh: (e^2x - 1) / (e^2x + 1) from one MUFU.EX2 and one MUFU.RCP on a
// clamped argument (|err| < 4e-7 absolute; t - 1 is exact for t in [1/2, 2], so
// small |x| keeps its accuracy), or libdevice tanhf
__device__ __forceinline__ float tanh_epi(float x) {
#if UUV_TC_FAST_TANH
    x = fminf(fmaxf(x, -9.0f), 9.0f);
    float t, r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(x * 2.88539008177792681f));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(t + 1.0f));
    return (t - 1.0f) * r;
#else
    return tanhf(x);
#endif
}

__device__ __forceinline__ float tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}
__device__ __forceinline__ uint32_t s_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// UMMA shared-memory descriptor: K-major, SWIZZLE_NONE, LBO = 128 B (next K
// core matrix), SBO = KC * 128 B (next 8-row group), version 1 (sm_100)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, int KC) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((128u >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)(((uint32_t)KC * 128u >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t a, uint64_t b, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
        "l"(a), "l"(b), "r"(IDESC_TF32), "r"(acc));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(bar)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred P;\n"
        "W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        " @!P bra W_%=;\n}" ::"r"(s_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// 8 consecutive fp32 accumulator columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
    uint32_t r[8];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
// 16 consecutive fp32 accumulator columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
template <int N> __device__ __forceinline__ void tmem_ld(uint32_t taddr, float (&v)[N]) {
    if constexpr (N == 16) tmem_ld16(taddr, v);
    else tmem_ld8(taddr, v);
}

// weight image: hi/lo tf32 splits in the core-matrix layout + the small block
__global__ void k_rl_prepare(const UuvRlPolicyArgs a, unsigned char* img) {
    const Img g = img_layout((int)a.obs_dim);
    const int D = (int)a.obs_dim, A = (int)a.act_dim, K1 = (int)g.k1;
    const int n1 = H * K1, n2 = H * H;
    const int total = 2 * n1 + 2 * n2;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const float* W;
        int K, KIN, j = i;
        uint32_t hi_off, lo_off;
        if (j < n1) { W = a.c1w; K = K1; KIN = D; hi_off = g.w1c_hi; lo_off = g.w1c_lo; }
        else if ((j -= n1) < n2) { W = a.c2w; K = H; KIN = H; hi_off = g.w2c_hi; lo_off = g.w2c_lo; }
        else if ((j -= n2) < n1) { W = a.a1w; K = K1; KIN = D; hi_off = g.w1a_hi; lo_off = g.w1a_lo; }
        else { j -= n1; W = a.a2w; K = H; KIN = H; hi_off = g.w2a_hi; lo_off = g.w2a_lo; }
        const int n = j / K, k = j - n * K;
        const float w = k < KIN ? W[n * KIN + k] : 0.0f;
        const float hi = tf32(w);
        const uint32_t o = cm_off(n, k, K / 4);
        *reinterpret_cast<float*>(img + hi_off + o) = hi;
        *reinterpret_cast<float*>(img + lo_off + o) = tf32(w - hi);
    }
    float* sp = reinterpret_cast<float*>(img + g.small);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < S_N; i += gridDim.x * blockDim.x) {
        float v = 0.0f;
        if (i < S_B2C) v = a.c1b[i];
        else if (i < S_CV) v = a.c2b[i - S_B2C];
        else if (i < S_CVB) v = a.cvw[i - S_CV];
        else if (i < S_B1A) v = i == S_CVB ? a.cvb[0] : 0.0f;
        else if (i < S_B2A) v = a.a1b[i - S_B1A];
        else if (i < S_AM) v = a.a2b[i - S_B2A];
        else if (i < S_AMB) { const int r = (i - S_AM) / H; v = r < A ? a.amw[i - S_AM] : 0.0f; }
        else if (i < S_LS) { const int r = i - S_AMB; v = r < A ? a.amb[r] : 0.0f; }
        else { const int r = i - S_LS; v = r < A ? a.log_std[r] : 0.0f; }
        sp[i] = v;
    }
}

#ifndef UUV_TC_NQ
#define UUV_TC_NQ 4   // threads per env (column groups): 2 / 4 / 8 measured 24.6 / 23.1 / 23.7 us
                      // per C4 loop step
#endif
constexpr int NQ = UUV_TC_NQ;           // column groups per env: 2, 4 or 8
constexpr int CW = 64 / NQ;             // accumulator columns per thread
constexpr int CK = CW < 16 ? CW : 16;   // columns per tcgen05.ld
constexpr int CPQ = CW / CK;            // tcgen05.ld chunks per thread
constexpr int PPQ = NQ < 4 ? 4 / NQ : 1;   // Box-Muller pairs per thread (4 pairs: A <= 8)

// fixed-order sum of the NQ group partials of one env
__device__ __forceinline__ float sum_groups(const float (*red)[128], int row) {
    if constexpr (NQ == 2) return red[0][row] + red[1][row];
    else if constexpr (NQ == 4) return (red[0][row] + red[1][row]) + (red[2][row] + red[3][row]);
    else
        return ((red[0][row] + red[1][row]) + (red[2][row] + red[3][row])) +
               ((red[4][row] + red[5][row]) + (red[6][row] + red[7][row]));
}

// epilogue of a hidden layer for 64 / NQ of this env's units (column group ch):
// tanh(acc + b) -> next layer's A operand (hi/lo)
__device__ __forceinline__ void epi_hidden(uint32_t tacc, const float* b, unsigned char* a_hi,
                                           unsigned char* a_lo, int row, int ch) {
#pragma unroll 1   // compact code: the CTA's warps run in near lockstep, an icache miss stalls all
    for (int cc = 0; cc < CPQ; ++cc) {
        const int c0 = ch * CW + cc * CK;
        float v[CK];
        tmem_ld<CK>(tacc + c0, v);
#pragma unroll
        for (int q = 0; q < CK / 4; ++q) {
            float4 hi, lo;
            float* hp = &hi.x;
            float* lp = &lo.x;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int j = c0 + 4 * q + t;
                const float x = tanh_epi(v[4 * q + t] + b[j]);
                hp[t] = tf32(x);
                lp[t] = tf32(x - hp[t]);
            }
            const uint32_t o = cm_off(row, c0 + 4 * q, H / 4);
            *reinterpret_cast<float4*>(a_hi + o) = hi;
            *reinterpret_cast<float4*>(a_lo + o) = lo;
        }
    }
}

// one layer: D(tmem) = A B^T with 3xTF32, K = kdim; commit to bar.  The four
// descriptors are built once; stepping K by 8 (two core matrices, 256 B) adds 16
// to the start-address field (address >> 4; shared addresses stay < 256 KB)
__device__ __forceinline__ void issue_layer(uint32_t tmem, const unsigned char* a_hi,
                                            const unsigned char* a_lo, const unsigned char* b_hi,
                                            const unsigned char* b_lo, int kdim,
                                            uint64_t* bar /* NULL: no commit */) {
    const int KC = kdim / 4;
    const uint64_t dah = umma_desc(s_u32(a_hi), KC), dal = umma_desc(s_u32(a_lo), KC);
    const uint64_t dbh = umma_desc(s_u32(b_hi), KC), dbl = umma_desc(s_u32(b_lo), KC);
#pragma unroll 1
    for (int ks = 0; ks < kdim / 8; ++ks) {   // K = 8 per MMA: two core matrices along K
        const uint64_t off = (uint64_t)ks * 16u;
        mma_tf32(tmem, dah + off, dbh + off, ks > 0 ? 1u : 0u);
        mma_tf32(tmem, dah + off, dbl + off, 1u);
        mma_tf32(tmem, dal + off, dbh + off, 1u);
    }
    if (bar)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(s_u32(bar)) : "memory");
}

constexpr int NT = NQ * M;   // threads: NQ per env (TMEM lane quarter = warp % 4, column group = warp / 4)

__global__ void __launch_bounds__(NT, 1) k_policy_tc(const UuvRlPolicyArgs a) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(8) uint64_t bars[2];   // [0] weights landed, [1] MMA done
    __shared__ uint32_t tmem_base_sh;
    __shared__ double nsc[2 * 36];              // normaliser mean, 1 / sqrt(var + 1e-8)
    __shared__ float red[NQ][M];                // cross-group partials
    __shared__ double gstat[NT];                // normaliser sums per (row group, column)
    const int D = (int)a.obs_dim, A = (int)a.act_dim;
    const bool value_only = (a.flags & 4) != 0;
    const Img g = img_layout(D);
    const int K1 = (int)g.k1;
    unsigned char* wimg = smem;                          // image copy
    unsigned char* az_hi = smem + g.total;               // [128][K1] core-matrix
    unsigned char* az_lo = az_hi + M * K1 * 4;
    unsigned char* ah_hi = az_lo + M * K1 * 4;           // [128][64] core-matrix
    unsigned char* ah_lo = ah_hi + M * H * 4;
    const float* sp = reinterpret_cast<const float*>(wimg + g.small);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int row = ((warp & 3) << 5) + lane;            // env in CTA = TMEM lane
    const int ch = warp >> 2;                            // column group
    const bool pdl = (a.flags & 8) != 0;                 // programmatic dependent launch
    if (pdl && UUV_PDL_TRIGGER == 1) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {   // 128 TMEM columns: two fp32 128 x 64 accumulators
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;"
                     ::"r"(s_u32(&tmem_base_sh)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // everything above overlaps the predecessor's tail; nothing it writes
    // (observations, normaliser statistics, noise counter, weight image) is read
    // before this point
    if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");

    // ---- observations: issued first (one memory round trip for the rows, the
    // running statistics and the noise counter together), stored to shared memory
    // after the barrier that publishes the TMEM base
    const uint64_t e = (uint64_t)blockIdx.x * M + row;
    const bool active = e < a.num_envs;
    float* raw = reinterpret_cast<float*>(ah_hi);        // scratch [128][D] (A_h unused yet)
    const uint64_t left = a.num_envs - (uint64_t)blockIdx.x * M;
    const int nvalid = left < (uint64_t)M ? (int)left : M;
    const float* src = a.obs + (uint64_t)blockIdx.x * M * D;
    const int nf = nvalid * D;
    constexpr int PER = (M * 36 / 4 + NT - 1) / NT;   // float4 per thread at D = 36
    const bool vec = (reinterpret_cast<uintptr_t>(src) & 15) == 0;
    const int n4 = vec ? nf >> 2 : 0;
    float4 buf[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int i = tid + j * NT;
        buf[j] = i < n4 ? __ldg(reinterpret_cast<const float4*>(src) + i) : float4{};
    }
    const uint64_t ctr = a.noise_ctr ? *a.noise_ctr : 0;
    if (tid < D) {
        nsc[tid] = a.norm_mean[tid];
        nsc[36 + tid] = 1.0 / sqrt(a.norm_var[tid] + 1e-8);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;
    if (UUV_TC_STOP == 8) {   // probe: launch + TMEM alloc only
        tc_fence_before();
        __syncthreads();
        if (warp == 0)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
        return;
    }
    if (tid == 0 && UUV_TC_STOP != 7) {   // the whole weight image in one bulk copy
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                     ::"r"(s_u32(&bars[0])), "r"(g.total) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(s_u32(wimg)), "l"(a.wimage), "r"(g.total), "r"(s_u32(&bars[0])) : "memory");
    }
    {   // the CTA's rows are one contiguous span in global AND shared memory
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int i = tid + j * NT;
            if (i < n4) reinterpret_cast<float4*>(raw)[i] = buf[j];
        }
        for (int f = (n4 << 2) + tid; f < nf; f += NT) raw[f] = __ldg(src + f);
        for (int f = nf + tid; f < M * D; f += NT) raw[f] = 0.0f;   // rows past the last env
    }
    __syncthreads();
    if (UUV_TC_STOP == 9) mbar_wait(&bars[0], 0);
    UUV_TC_EXIT_AFTER(9)   // probe: + observation rows in shared memory
    // normaliser sums: thread (g, c) adds column c (sum x | sum x^2) over rows g,
    // g + G, ... (G = NT / 2 D groups); the group partials are added in group order
    // after the next barrier (fixed order: deterministic)
    const int ncol = 2 * D, ngrp = NT / ncol;
    const bool stats = (a.flags & 2) != 0;
    if (stats) {
        const int sg = tid / ncol, sc = tid - sg * ncol;
        if (sg < ngrp) {
            const int d = sc < D ? sc : sc - D;
            double acc = 0.0;
            for (int r = sg; r < nvalid; r += ngrp) {
                const double v = raw[r * D + d];
                acc += sc < D ? v : v * v;
            }
            gstat[tid] = acc;
        }
    }
    // normalise: the two column halves split the K chunks; the fp32 rows are staged
    // in A_h's lo half (unused yet) and stored to nobs_out coalesced afterwards
    float* zst = reinterpret_cast<float*>(ah_lo);
#pragma unroll 1
    for (int k4 = ch; 4 * k4 < K1; k4 += NQ) {
        float4 hi, lo;
        float* hp = &hi.x;
        float* lp = &lo.x;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int k = 4 * k4 + t;
            float zk = 0.0f;
            if (k < D) {   // RunningNorm.normalize in fp64
                double v = ((double)raw[row * D + k] - nsc[k]) * nsc[36 + k];
                v = fmin(fmax(v, -a.norm_clip), a.norm_clip);
                zk = (float)v;
                zst[row * D + k] = zk;
            }
            hp[t] = tf32(zk);
            lp[t] = tf32(zk - hp[t]);
        }
        const uint32_t o = cm_off(row, 4 * k4, K1 / 4);
        *reinterpret_cast<float4*>(az_hi + o) = hi;
        *reinterpret_cast<float4*>(az_lo + o) = lo;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // A_z -> tensor-core proxy
    __syncthreads();
    if (UUV_TC_STOP == 10) mbar_wait(&bars[0], 0);
    UUV_TC_EXIT_AFTER(10)   // probe: + normaliser sums and normalisation
    UUV_TC_EXIT_AFTER(7)   // probe: load + normalise, no weight image
    mbar_wait(&bars[0], 0);                                        // weights landed
    UUV_TC_EXIT_AFTER(1)   // probe: load + normalise + weight image
    if (tid == 0) {   // round 1: critic layer 1 (runs while the normalised rows go out)
        tc_fence_after();
        issue_layer(tmem, az_hi, az_lo, wimg + g.w1c_hi, wimg + g.w1c_lo, K1, &bars[1]);
    }
    if (stats && tid < ncol) {   // this CTA's partial row of the normaliser sums
        double acc = 0.0;
        for (int q = 0; q < ngrp; ++q) acc += gstat[q * ncol + tid];
        a.stats_part[(size_t)blockIdx.x * 2 * D + tid] = acc;
    }
    if (a.nobs_out) {   // the CTA's normalised rows: one contiguous span
        float* dst = a.nobs_out + (uint64_t)blockIdx.x * M * D;
        const int nf = nvalid * D;
        int done_f = 0;
        if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
            const int n4 = nf >> 2;
            for (int i = tid; i < n4; i += NT)
                reinterpret_cast<float4*>(dst)[i] = reinterpret_cast<const float4*>(zst)[i];
            done_f = n4 << 2;
        }
        for (int f = done_f + tid; f < nf; f += NT) dst[f] = zst[f];
    }
    __syncthreads();   // staging read out before the first epilogue overwrites A_h
    // two fp32 128 x 64 accumulators: acc0 (columns 0-63), acc1 (64-127)
    const uint32_t tacc = tmem + ((uint32_t)((warp & 3) * 32) << 16);   // this warp's TMEM lanes
    const uint32_t tacc1 = tacc + (uint32_t)H;

    // critic: value = cv . tanh(W2c tanh(W1c z + b1c) + b2c) + cvb
    // actor:  mean = tanh(am tanh(W2a tanh(W1a z + b1a) + b2a) + amb)
    // The chains are independent: the actor's first layer (A_z -> acc1) is issued
    // together with the critic's second (A_h -> acc0), so three MMA rounds and
    // three epilogue phases instead of four of each.
    mbar_wait(&bars[1], 0);
    tc_fence_after();
    epi_hidden(tacc, sp + S_B1C, ah_hi, ah_lo, row, ch);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    UUV_TC_EXIT_AFTER(2)   // probe: + round 1 and its epilogue
    if (tid == 0) {   // round 2: critic layer 2 (acc0) + actor layer 1 (acc1), one commit
        tc_fence_after();
        if (!value_only)
            issue_layer(tmem + (uint32_t)H, az_hi, az_lo, wimg + g.w1a_hi, wimg + g.w1a_lo, K1,
                        nullptr);
        issue_layer(tmem, ah_hi, ah_lo, wimg + g.w2c_hi, wimg + g.w2c_lo, H, &bars[1]);
    }
    mbar_wait(&bars[1], 1);   // both done: A_h is free again
    tc_fence_after();
    {
        float vp = 0.0f;
#pragma unroll 1
        for (int cc = 0; cc < CPQ; ++cc) {
            const int c0 = ch * CW + cc * CK;
            float v[CK];
            tmem_ld<CK>(tacc + c0, v);
#pragma unroll
            for (int t = 0; t < CK; ++t)
                vp = fmaf(sp[S_CV + c0 + t], tanh_epi(v[t] + sp[S_B2C + c0 + t]), vp);
        }
        red[ch][row] = vp;
    }
    if (!value_only) epi_hidden(tacc1, sp + S_B1A, ah_hi, ah_lo, row, ch);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();   // red complete; actor A_h complete
    const float value = sum_groups(red, row) + sp[S_CVB];
    UUV_TC_EXIT_AFTER(3)   // probe: + round 2 and its epilogues
    // actor trunk output parked in fp32 rows (stride 68: conflict-free float4 reads) for
    // the mean head, over A_h once the actor's second layer has consumed it
    float* hrow = reinterpret_cast<float*>(ah_hi) + row * 68;
    if (!value_only) {
        if (tid == 0) {   // round 3: actor layer 2
            tc_fence_after();
            issue_layer(tmem, ah_hi, ah_lo, wimg + g.w2a_hi, wimg + g.w2a_lo, H, &bars[1]);
        }
        mbar_wait(&bars[1], 0);   // A_h consumed: hrow may overwrite it
        tc_fence_after();
#pragma unroll 1
        for (int cc = 0; cc < CPQ; ++cc) {
            const int c0 = ch * CW + cc * CK;
            float v[CK];
            tmem_ld<CK>(tacc + c0, v);
#pragma unroll
            for (int t = 0; t < CK; t += 4)
                *reinterpret_cast<float4*>(hrow + c0 + t) = make_float4(
                    tanh_epi(v[t] + sp[S_B2A + c0 + t]),
                    tanh_epi(v[t + 1] + sp[S_B2A + c0 + t + 1]),
                    tanh_epi(v[t + 2] + sp[S_B2A + c0 + t + 2]),
                    tanh_epi(v[t + 3] + sp[S_B2A + c0 + t + 3]));
        }
    }
    tc_fence_before();
    __syncthreads();
    if (UUV_PDL_TRIGGER == 2 && pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
    if (UUV_TC_STOP == 4) return;   // probe: + round 3 and its epilogue
    if (value_only) {
        if (active && ch == 0 && a.value_out) a.value_out[e] = value;
        return;
    }
    // action dims: group ch takes Box-Muller pairs PPQ ch .. PPQ ch + PPQ - 1 (two dims each)
    const uint64_t gid = a.env_offset + e;
    float logp = 0.0f;
#pragma unroll 1
    for (int p = PPQ * ch; p < PPQ * ch + PPQ; ++p) {
        if (2 * p >= A) break;
        float eps0 = 0.0f, eps1 = 0.0f;
        if (a.flags & 1) {   // Box-Muller on the counter-based stream
            const uint64_t bits = uuv::draw_u64(a.seed, gid, 3, ctr * 4 + (uint64_t)p);
            const float u1 = ((float)(uint32_t)(bits >> 40) + 0.5f) * 5.9604644775390625e-08f;
            const float u2 = (float)(uint32_t)(bits & 0xffffffu) * 5.9604644775390625e-08f;
            const float r = sqrtf(-2.0f * __logf(u1));
            float sn, cs;
            __sincosf(6.28318530717958647f * u2, &sn, &cs);
            eps0 = r * cs;
            eps1 = r * sn;
        }
#pragma unroll 1
        for (int q = 0; q < 2; ++q) {
            const int i = 2 * p + q;
            if (i >= A) break;
            float c0 = sp[S_AMB + i], c1 = 0.0f, c2 = 0.0f, c3 = 0.0f;
            const float4* w4 = reinterpret_cast<const float4*>(sp + S_AM + i * H);
            const float4* h4 = reinterpret_cast<const float4*>(hrow);
#pragma unroll 4
            for (int k = 0; k < H / 4; ++k) {
                const float4 w = w4[k], hv = h4[k];
                c0 = fmaf(w.x, hv.x, c0);
                c1 = fmaf(w.y, hv.y, c1);
                c2 = fmaf(w.z, hv.z, c2);
                c3 = fmaf(w.w, hv.w, c3);
            }
            const float mean = tanhf((c0 + c1) + (c2 + c3));
            const float lsd = sp[S_LS + i];
            const float rawv = fmaf(expf(lsd), q ? eps1 : eps0, mean);
            const float zz = (rawv - mean) * expf(-lsd);      // ActorCritic.log_prob
            logp += -0.5f * zz * zz - lsd - 0.918938533204672742f;
            if (active && a.raw_out) a.raw_out[e * A + i] = rawv;
            if (active && a.act_out) a.act_out[e * A + i] = fminf(fmaxf(rawv, -1.0f), 1.0f);
        }
    }
    red[ch][row] = logp;
    __syncthreads();
    if (active && ch == 0) {
        if (a.logp_out) a.logp_out[e] = sum_groups(red, row);
        if (a.value_out) a.value_out[e] = value;
    }
}

inline size_t smem_bytes(int D) {
    const Img g = img_layout(D);
    return (size_t)g.total + 2 * (size_t)M * g.k1 * 4 + 2 * (size_t)M * H * 4;
}

}  // namespace uuvtc

namespace uuvrl {
// GAE (reference ppo.py:112-130) over [T][M] buffers, one thread per env walking
// the horizon backwards; done_t is terminal (nonterminal = 1 - done_t).
__global__ void k_gae(const float* __restrict__ rew, const float* __restrict__ val,
                      const float* __restrict__ done, const float* __restrict__ boot, int T,
                      uint64_t M, float gamma, float lam, float* __restrict__ adv,
                      float* __restrict__ ret) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= M) return;
    float last = 0.0f, next_v = boot[e];
    for (int t = T - 1; t >= 0; --t) {
        const size_t i = (size_t)t * M + e;
        const float nonterminal = 1.0f - done[i];
        const float v = val[i];
        const float delta = rew[i] + gamma * next_v * nonterminal - v;
        last = delta + gamma * lam * nonterminal * last;
        adv[i] = last;
        ret[i] = last + v;
        next_v = v;
    }
}
}  // namespace uuvrl

extern "C" {

int32_t uuvsim_rl_gae(const float* rew, const float* val, const float* done, const float* boot,
                      uint32_t horizon, uint64_t num_envs, float gamma, float lam, float* adv,
                      float* ret, uint64_t stream) {
    if (!rew || !val || !done || !boot || !adv || !ret || horizon == 0 || num_envs == 0) return 3;
    const unsigned grid = (unsigned)((num_envs + 255) / 256);
    uuvrl::k_gae<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        rew, val, done, boot, (int)horizon, num_envs, gamma, lam, adv, ret);
    return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

uint32_t uuvsim_rl_policy_blocks(uint64_t num_envs) {
    // buffer rows: one per 64-env CUDA-core block (the tensor-core kernel writes one
    // per 128-env CTA, the first half)
    return (uint32_t)(2 * ((num_envs + uuvtc::M - 1) / uuvtc::M));
}

uint64_t uuvsim_rl_image_bytes(uint32_t obs_dim) {
    return obs_dim == 0 || obs_dim > 36 ? 0 : uuvtc::img_layout((int)obs_dim).total;
}

int32_t uuvsim_rl_prepare(const UuvRlPolicyArgs* a, void* image, uint64_t len, uint64_t stream) {
    if (!a || !image || a->obs_dim == 0 || a->obs_dim > 36 || a->act_dim == 0 ||
        a->act_dim > uuvtc::AMAX || a->hidden != uuvtc::H ||
        len != uuvtc::img_layout((int)a->obs_dim).total)
        return 3;
    uuvtc::k_rl_prepare<<<64, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        *a, static_cast<unsigned char*>(image));
    return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int32_t uuvsim_rl_policy_act(const UuvRlPolicyArgs* a, uint64_t stream) {
    if (!a || a->num_envs == 0 || a->obs_dim == 0 || a->obs_dim > 36 || a->act_dim == 0 ||
        a->act_dim > uuvrl::AMAX || a->hidden != uuvrl::H || !a->obs || !a->norm_mean ||
        !a->norm_var || !a->a1w || !a->c1w || !a->c2w || !a->cvw ||
        ((a->flags & 2) && !a->stats_part))
        return 3;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (a->wimage) {   // tensor cores
        const size_t smem = uuvtc::smem_bytes((int)a->obs_dim);
        uuvrl::smem_optin<uuvtc::k_policy_tc>((int)uuvtc::smem_bytes(36));
        const unsigned grid = (unsigned)((a->num_envs + uuvtc::M - 1) / uuvtc::M);
        const cudaError_t e = uuv::launch_k(uuvtc::k_policy_tc, dim3(grid), dim3(uuvtc::NT), smem, st,
                                              (a->flags & 8) != 0, *a);
        return e == cudaSuccess && cudaGetLastError() == cudaSuccess ? 0 : 4;
    }
    const cudaError_t e = a->obs_dim <= 12 ? uuvrl::launch_policy<12>(*a, st)
                                           : uuvrl::launch_policy<36>(*a, st);
    return e == cudaSuccess ? 0 : 4;
}

int32_t uuvsim_rl_post(const UuvRlPostArgs* a, uint64_t stream) {
    if (!a || a->num_envs == 0 || a->obs_dim > 36 || (a->n_part && (!a->stats_part ||
        !a->norm_mean || !a->norm_var || !a->norm_count)))
        return 3;
    const bool copy = (a->rew_in && a->rew_out) || (a->done_in && a->done_out);
    const unsigned grid = copy ? (unsigned)(1 + (a->num_envs + 1023) / 1024)   // + statistics block
                               : 1u;
    const cudaError_t e = uuv::launch_k(uuvrl::k_rl_post, dim3(grid), dim3(1024), 0,
                                          reinterpret_cast<cudaStream_t>(stream),
                                          (a->flags & 1) != 0, *a);
    return e == cudaSuccess && cudaGetLastError() == cudaSuccess ? 0 : 4;
}

}  // extern "C"

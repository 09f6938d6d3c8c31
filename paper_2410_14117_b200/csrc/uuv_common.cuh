// uuv_common.cuh -- shared definitions for the B200 env-step engine.
//
// Layout in HBM (one engine = one slab of N envs on one GPU):
//   state   : 3 planes of V4<T>[N]  (x y z phi | theta psi u v | w p q r)
//   step    : int32[N]              control-step counter (reference i64, batch.py:55)
//   ep_ret  : float[N]              running episode return (for episode statistics)
//   ctr     : uint64[2][N]          reset / param RNG counters (engine.rs:338-339)
//   dr      : V4<T>[N], V4<T>[N], V2<T>[N]   (only with domain randomisation)
//             (f_mass f_added f_dlin f_dquad | f_thrust rb_x rb_y rb_z | W B)
//   traj    : V4<T>[episode_len + lookahead + 1]  reference (x y z psi) per step index
// Base vehicles, task constants and the trajectory pointer travel in the kernel
// parameter block (constant bank 0): every matrix coefficient is an immediate
// constant-bank operand of the FFMA that uses it -- no loads, no registers.
#pragma once

#include <cstdint>
#include <cmath>

#if !defined(__CUDACC__) && !defined(__host__)
#define __host__
#define __device__
#define __forceinline__ inline
#endif

#ifndef UUV_PACK_CONSTS
#define UUV_PACK_CONSTS 0   // fp32 Fossen vehicle constants in registers (1) or constant bank (0):
                            // bank operands keep FFMAs at 2 register reads (full issue rate)
#endif

namespace uuv {

constexpr int MAX_THR = 8;
constexpr int MAX_VEH = 2;
constexpr int NSTAT = 9;

// stats slots (per-block partial sums, reduced on read)
enum StatSlot {
    ST_REWARD = 0,       // sum of step rewards
    ST_DONE_TRUNC = 1,   // terminations by reason (tasks.py:41-42)
    ST_DONE_DIV = 2,
    ST_DONE_FAIL = 3,
    ST_EP_RETURN = 4,    // sum of returns of completed episodes
    ST_EP_LEN = 5,       // sum of lengths of completed episodes
    ST_STEPS = 6,        // env-steps executed
    ST_RESAMPLE_ERR = 7, // per-episode DR resamples rejected (non-PD), params kept
    ST_BAND64 = 8,       // fp32-engine env-steps computed in fp64 (Euler pitch band)
};

// Euler-singularity band: near theta = +-pi/2 the Euler-rate map's
// 1/cos(theta) turns fp32 rounding of the state into errors far beyond the fp32
// tolerance, so a step that starts at |theta| <= BAND_THETA and may leave it is
// computed in fp64 (uuv_kernels.cuh band_cand / replay_band64).
constexpr float BAND_THETA = 1.4f;

template <class T> struct alignas(4 * sizeof(T)) V4 { T x, y, z, w; };
template <class T> struct alignas(2 * sizeof(T)) V2 { T x, y; };

// ----------------------------------------------------------------- rng.rs / rng.py
// Counter-based SplitMix64 streams: draw = f(seed, stream, purpose, counter)
// (reference rng.py:26-53, native/src/rng.rs:16-41).  Integer part is exact on
// both sides; u01/uniform are evaluated in fp64 with FMA contraction disabled.
constexpr uint64_t GOLDEN = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t PURPOSE_SALT = 0x632BE59BD9B4E019ULL;
constexpr uint64_t PURPOSE_PARAMS = 0, PURPOSE_RESET = 1, PURPOSE_BENCH = 2;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = z + GOLDEN;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t draw_u64(uint64_t seed, uint64_t stream,
                                                      uint64_t purpose, uint64_t counter) {
    uint64_t h = mix64(seed);
    h = mix64(h ^ (stream + GOLDEN));
    h = mix64(h ^ (purpose + PURPOSE_SALT));
    return mix64(h ^ counter);
}

// draw_u64 split: the first three SplitMix rounds depend only on (seed, stream,
// purpose), so a lane's prefix is hashed once and each counted draw costs one
// round -- identical bits to draw_u64.
__host__ __device__ __forceinline__ uint64_t lane_prefix(uint64_t seed, uint64_t stream,
                                                         uint64_t purpose) {
    uint64_t h = mix64(seed);
    h = mix64(h ^ (stream + GOLDEN));
    return mix64(h ^ (purpose + PURPOSE_SALT));
}
__host__ __device__ __forceinline__ uint64_t lane_draw(uint64_t prefix, uint64_t counter) {
    return mix64(prefix ^ counter);
}

__host__ __device__ __forceinline__ double u01(uint64_t bits) {
    return (double)(bits >> 11) * (1.0 / 9007199254740992.0);
}

// lo + (hi - lo) * u, rounded exactly as the reference (no FMA).
__host__ __device__ __forceinline__ double uniform_rn(double lo, double hi, double u) {
#ifdef __CUDA_ARCH__
    return __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u));
#else
    volatile double d = hi - lo;
    volatile double m = d * u;
    return lo + m;
#endif
}

constexpr double PI_D = 3.141592653589793;
constexpr double TWO_PI_D = 2.0 * PI_D;

// wrap_angle in fp64 (dynamics.py:56-61); fmod is exact in CUDA and glibc.
__host__ __device__ __forceinline__ double wrap_angle_d(double a) {
#ifdef __CUDA_ARCH__
    double r = fmod(__dadd_rn(a, PI_D), TWO_PI_D);
    if (r <= 0.0) r = __dadd_rn(r, TWO_PI_D);
    return __dsub_rn(r, PI_D);
#else
    double r = std::fmod(a + PI_D, TWO_PI_D);
    if (r <= 0.0) r += TWO_PI_D;
    return r - PI_D;
#endif
}

// ------------------------------------------------------------------ parameters
// One base vehicle as the kernels see it (precision T).  Row-major 6x6 blocks.
template <class T> struct VehP {
    T mtot[36];      // M_RB + M_A (vehicle.py:104-105)
    T mrb[36];       // M_RB alone (scaled by f_mass under domain randomisation)
    T ma[36];        // M_A alone  (scaled by f_added)
    T chol[36];      // lower Cholesky factor of mtot (row-major, lower triangle)
    T chol_inv[6];   // 1 / L_ii
    T kdt[36];       // sub_dt * M_total^-1 on the Fossen pattern (fp32 product path)
    T dlin[36];
    T dquad[6];
    T weight, buoyancy;
    T rg[3], rb[3];
    T wb;            // W - B            (fused fp32 restoring term)
    T hm[3];         // W r_g - B r_b    (restoring moment = hm x e, e = R^T z)
    T alloc[6 * MAX_THR];   // 6 x MAX_THR, zero-padded columns
    T kmax[MAX_THR];
    int32_t curve[MAX_THR]; // 0 linear, 1 quadratic_signed
    int32_t n_thr;
    int32_t pad_;
    // fp64 base values used to (re)draw randomised parameters (randomize.py:79-109)
    double weight64;
    double rb64[3];
    double mrb64[36];
    double ma64[36];
};

// Randomisation ranges (log bounds precomputed on the host with glibc log).
struct RangesP {
    double log_lo[5], log_hi[5];   // mass, added, dlin, dquad, thrust
    double rb_offset;
    double ratio[2];
    int32_t enabled, per_episode;
};

template <class T> struct TaskP {
    T target[6];
    T sub_dt;
    T div_radius;
    int32_t kind;          // 0 station, 1 circle, 2 helix, 3 lemniscate
    int32_t lookahead;
    int32_t n_substeps;
    int32_t episode_len;
    int32_t obs_dim;
    int32_t pad_;
    // reset spawn point and reference yaw in fp64 (tasks.py:186-198)
    double spawn[3];
    double ref_psi;
    const V4<T>* traj;     // reference (x y z psi) by step index, tracking only
};

// Everything a step / reset launch needs; passed by value as __grid_constant__.
template <class T> struct EngineP {
    VehP<T> veh[MAX_VEH];
    TaskP<T> task;
    RangesP ranges;
    uint64_t seed;         // root seed (reset launches); the step reads *seed_dev so
    uint64_t* seed_dev;    // a captured graph sees reset_all's new seed
    uint64_t env_offset;
    int64_t mix_bound0;    // global env index where vehicle 1 starts (mixed batches)
    int32_t n_env;
    int32_t n_veh;
    int32_t act_dim;       // row stride of the action matrix
    int32_t stats_on;
    int32_t io_f64;        // actions / obs / reward are f64 (host ABI path), else T
    int32_t stage_obs;     // observation rows staged in shared memory, stored coalesced
    int32_t persist_blocks;   // >0: TMA-pipelined persistent paired kernel with this grid
    int32_t pdl;           // launched as a programmatic dependent (griddepcontrol wait /
                           // early trigger): overlaps launch latency inside graphs
    // device buffers
    V4<T>* s0; V4<T>* s1; V4<T>* s2;
    int32_t* step;
    float* ep_ret;
    uint64_t* reset_ctr;
    uint64_t* param_ctr;
    V4<T>* dr0; V4<T>* dr1; V2<T>* dr2;
    double* stats;         // [gridDim][NSTAT] per-block partials
    // fp32 register pack per vehicle (PACK_F4 float4 each, see uuv_model.cuh
    // load_regs): read once per step with LDG so ptxas keeps it in registers
    const float4* vpack;
    // optional [n_env][obs_dim] T buffer (device face): finished envs write their
    // TERMINAL observation (pre-reset state at the terminating step) here
    void* final_obs;
    // optional [n_env] fp32 buffer (device face): done as 0 / 1 floats, e.g. a
    // rollout's done buffer written by the step itself
    float* done_f32;
    int32_t stage_act;     // host-ABI zero-copy step: f64 action rows staged in shared memory
    int32_t stagger_ns;    // host-ABI zero-copy step: block b starts b*stagger_ns/gridDim ns late
    // fp64 band replay (fp32 engines; see uuv_kernels.cuh band_cand):
    // veh64 = fp64 base vehicles in HOST memory (copied into the band kernel's
    // parameters at launch), veh64_dev = the same in device memory (step-kernel
    // tail); band_theta = BAND_THETA, or +inf with device.band64 = false
    const VehP<double>* veh64;
    const VehP<double>* veh64_dev;
    V2<double>* dr64;      // [N][5] exact fp64 DR records (randomised fp32 engines)
    double sub_dt64;
    float band_theta;
    float band_exit_theta; // = band_theta (device.band_tail = false: +inf, A/B only)
    float band_kdt;        // candidate predictor: control_dt
    float band_margin;     // candidate predictor margin (rad)
    int32_t band_per;      // envs scanned per band-kernel block (multiple of BLOCK)
    int32_t band_grid;     // band-kernel blocks
    int32_t band_same;     // band kernel on the launching stream after the step (A/B only)
    int32_t band_main_first;   // side stream: launch the step kernel before the band kernel
    int32_t band_rege;     // band kernel keeps the fp64 vehicle constants in registers (small batches)
    int32_t band_refop;    // band steps in the reference's operation order (long control steps)
    double* stats_band;    // the band kernel's per-block statistics partials
    // Band ownership per env and step (uuv_kernels.cuh k_band): flag byte
    // band_f[e] = (generation mod 128) << 1 | candidate, written by whichever
    // kernel steps the env for the next step.  The step kernel steps env e iff
    // band_f[e] == word(gen, 0), the band kernel iff == word(gen, 1) (only the
    // generations k and k + 1 ever meet, so 7 bits tell them apart).  Each kernel
    // derives gen from its own env counter (band_ctr[0] step kernel, [1] band
    // kernel): one thread per block claims the block's envs with a fetch-add,
    // whose return value is k * n_env + (less than n_env) during step k, so
    // gen = value / n_env.
    uint8_t* band_f;
    unsigned long long* band_ctr;
    double band_inv_n;     // 1 / n_env
    // host-only: the band kernel runs on band_side, forked from / joined to the
    // launching stream through these events (cudaStream_t / cudaEvent_t)
    void* band_side;
    void* band_ev[2];
    // set (mapped page-locked word) when a per-episode DR resample is rejected
    // (non-PD mass matrix): the host-ABI step then returns code 4 like the
    // reference engine's panic (engine.rs:553-558, capi.rs:58-70)
    volatile int32_t* err_flag;
};

constexpr int PACK_F4 = 10;   // 40 floats: Fossen pattern + restoring + trig constants

}  // namespace uuv

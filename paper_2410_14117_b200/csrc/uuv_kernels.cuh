// uuv_kernels.cuh -- the engine's CUDA kernels, instantiated once per precision
// by k_f32.cu (T = float, the product path) and k_f64.cu (T = double,
// compiled with -fmad=false).
//
//   K1 k_step       fused control step: wrench -> n_substeps x 6-DOF sub-step in
//                   registers -> reward / termination -> counter-RNG auto-reset
//                   (+ per-episode DR redraw) -> observation -> episode stats
//   K2 k_reset      reset_all(seed): 6 draws per env -> state, obs at step 0
//   K3 k_dr_init    domain-randomisation draw for every env at create time
//   K5 k_pack/unpack  state planes <-> host-ABI [N][12] f64 rows
//   K6 k_bench_act  fixed U[-1,1] bench actions from the counter RNG
//   K7 k_stats_reduce  deterministic reduction of the per-block stats partials
#pragma once

#include <cuda_runtime.h>

#include <atomic>
// UUV_BAND_CLOCK (A/B builds only): per-block %globaltimer timeline of the step
// and band kernels in a device table (row = event, column = block), read back
// with uuvsim_debug_timeline (tools/band_timeline.py)
#ifdef UUV_BAND_CLOCK
constexpr int TL_BLOCKS = 8192;
enum { TL_STEP_START, TL_STEP_END, TL_BAND_START, TL_BAND_SCAN, TL_BAND_END, TL_STEP_LOADED,
       TL_STEP_SUBS, TL_BAND_LOADED, TL_BAND_REPLAYED, TL_BAND_GEN, TL_BAND_LOOP_CYC, TL_BAND_LOOP_N,
       TL_ROWS };
static __device__ unsigned long long g_uuv_tl[TL_ROWS][TL_BLOCKS];   // per TU (fp32 read back)
__device__ __forceinline__ unsigned long long uuv_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define UUV_TL(row) \
    do { if (threadIdx.x == 0 && blockIdx.x < TL_BLOCKS) g_uuv_tl[row][blockIdx.x] = uuv_gtimer(); } while (0)
// stamp taken once `val` (a float) has arrived: the branch waits for it
// (UUV_BAND_CLOCK=2 only: these in-kernel stamps perturb the fp64 replay's schedule)
#if UUV_BAND_CLOCK >= 2
#define UUV_TLV(row, val) \
    do { if (threadIdx.x == 0 && blockIdx.x < TL_BLOCKS && __float_as_uint(val) != 0x7fc00001u) \
             g_uuv_tl[row][blockIdx.x] = uuv_gtimer(); } while (0)
#else
#define UUV_TLV(row, val) do { } while (0)
#endif
#else
#define UUV_TL(row) do { } while (0)
#define UUV_TLV(row, val) do { } while (0)
#endif

#include <algorithm>
#include <type_traits>

#include "uuv_model.cuh"
#include "launch.h"

// UUV_BOUNDS_CHECK (checking builds only, tools/bounds_run.py): device-side
// bounds asserts at the engine's computed indices -- env rows, band lists, flag
// bytes, staged rows -- that trap on a violation.  compute-sanitizer is not
// available on this GPU pool; the test suite runs against this build instead.
#ifdef UUV_BOUNDS_CHECK
#define UUV_CHECK(cond) do { if (!(cond)) __trap(); } while (0)
#else
#define UUV_CHECK(cond) do { } while (0)
#endif
#include "launch_kernel.cuh"

namespace uuv {


// Programmatic dependent launch: a kernel launched with the programmatic
// stream-serialisation attribute may start before its predecessor on the stream
// finishes; griddepcontrol.wait blocks until that predecessor has completed and
// its writes are visible.  An explicit trigger (UUV_PDL_TRIGGER, launch.h) would
// let the NEXT kernel's CTAs launch before this one ends; measured slower, so by
// default the trigger is implicit at completion and PDL only removes the
// launch-after-completion gap.
__device__ __forceinline__ void pdl_enter(bool on) {
    if (on) {
        if (UUV_PDL_TRIGGER == 1) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
}
// late trigger: the heavy work of this CTA is done, only its stores remain
__device__ __forceinline__ void pdl_trigger_late(bool on) {
    if (UUV_PDL_TRIGGER == 2 && on) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// stored angles are wrapped; only a teacher-forced state can lie outside
// [-pi, pi] -- bring it in once so every sub-step can use sincos_poly
__device__ __forceinline__ void prewrap(float s[12]) {
    if (!(fmaxf(fabsf(s[3]), fmaxf(fabsf(s[4]), fabsf(s[5]))) <= Consts<float>::PI)) {
        s[3] = wrap_pi(s[3]);
        s[4] = wrap_pi(s[4]);
        s[5] = wrap_pi(s[5]);
    }
}

// Rare path: the step ended non-finite.  Re-run it from the step-initial state
// (still in HBM) with a check after every sub-step and keep the last finite
// state (the reference stops at the first failing sub-step, model.rs:186-193).
template <bool DR, class Pat>
__device__ __forceinline__ void replay_env(const EngineP<float>& p, const VehP<float>& V,
                                        const EnvParams<float, DR || (UUV_PACK_CONSTS && Pat::fossen)>& E, int e,
                                        const float tau[6], float dt, const TrigK& K, int n_sub,
                                        float s[12]) {
    const V4<float> a0 = p.s0[e], a1 = p.s1[e], a2 = p.s2[e];
    const float r[12] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w, a2.x, a2.y, a2.z, a2.w};
#pragma unroll
    for (int i = 0; i < 12; ++i) s[i] = r[i];
    prewrap(s);
#pragma unroll 1
    for (int k = 0; k < n_sub; ++k) {
        float t[12];
#pragma unroll
        for (int i = 0; i < 12; ++i) t[i] = s[i];
        if (!substep_fused<DR, Pat, true>(V, E, t, tau, dt, K)) break;
#pragma unroll
        for (int i = 0; i < 12; ++i) s[i] = t[i];
    }
}

// fp64 step of one env (the Euler pitch band): near theta = +-pi/2
// the Euler-rate map (tan, sec of theta) amplifies the fp32 rounding of the state
// by up to 1/cos(PITCH_LIMIT) = 1000, beyond the fp32 tolerance, so a step that
// may leave |theta| <= band_theta runs in fp64 from the step-initial fp32 state:
// the FMA formulation of substep_fused in fp64 for the Fossen pattern (the
// reference's operation order, substep_ref, otherwise), fp64 vehicle constants and
// -- under domain randomisation -- the env's exact fp64 record (randomize.py:79-109).
// Returns the state rounded to fp32 by value.  Used by the band kernel (k_band)
// for predicted candidates and by the step kernel's out-of-line tail (band_tail)
// for predictor misses.
// Fossen-pattern fp64 vehicle constants copied into a register-resident
// EnvParams (same values: substep_f64<true> with them is bit-identical to
// substep_f64<false> on V), so the sub-step loop's DFMAs read registers instead
// of ~40 kernel-parameter constants per sub-step.  Used for small batches
// (EngineP::band_rege), where the band kernel is the step's critical path: the
// copy shortens the replay (C2 -0.9 us) but takes 30 more registers per thread,
// which at 2^20 envs cost the step kernel's waves more (C5 +1.6 us) -- measured.
__device__ __forceinline__ void reg_vehicle64(const VehP<double>& V, EnvParams<double, true>& R) {
#pragma unroll
    for (int i = 0; i < 6; ++i) {
#pragma unroll
        for (int j = 0; j < 6; ++j)
            if (PatFossen::M(i, j)) {
                R.mtot[i * 6 + j] = V.mtot[i * 6 + j];
                R.kdt[i * 6 + j] = V.kdt[i * 6 + j];
            }
        R.dq[i] = V.dquad[i];
        R.dl[i] = V.dlin[i * 6 + i];
    }
    R.wb = V.wb;
#pragma unroll
    for (int i = 0; i < 3; ++i) R.hm[i] = V.hm[i];
    // opaque copies: the compiler cannot fold them back into constant operands
#pragma unroll
    for (int i = 0; i < 36; ++i)
        if (PatFossen::M(i / 6, i % 6)) asm("" : "+d"(R.mtot[i]), "+d"(R.kdt[i]));
#pragma unroll
    for (int i = 0; i < 6; ++i) asm("" : "+d"(R.dq[i]), "+d"(R.dl[i]));
    asm("" : "+d"(R.wb), "+d"(R.hm[0]), "+d"(R.hm[1]), "+d"(R.hm[2]));
}

struct Band64Out {
    float v[12];
    int failed;
};

template <bool DR, class Pat, bool REGE = false, bool REFOP = false>
__device__ __forceinline__ Band64Out replay_band64(const EngineP<float>& p, const VehP<double>& V,
                                                   const float s32[12], const V2<double> rec[5],
                                                   const double act[MAX_THR]) {
    double s[12];
#pragma unroll
    for (int i = 0; i < 12; ++i) s[i] = s32[i];
    if (!(fmax(fabs(s[3]), fmax(fabs(s[4]), fabs(s[5]))) <= 3.141592653589793)) {
        s[3] = wrap_pi64(s[3]);   // teacher-forced out-of-range angles (sincos64's range)
        s[4] = wrap_pi64(s[4]);
        s[5] = wrap_pi64(s[5]);
    }
    const double dt = p.sub_dt64;
    // REFOP (EngineP::band_refop): the reference's operation order (substep_ref,
    // Cholesky solve) instead of the FMA formulation -- exact in k_band.cu, which
    // is compiled with -fmad=false
    constexpr bool refop = REFOP;
    EnvParams<double, DR> E;
    if constexpr (DR) {   // the env's exact fp64 record (written with its fp32 twin)
        const V4<double> r0{rec[0].x, rec[0].y, rec[1].x, rec[1].y};
        const V4<double> r1{rec[2].x, rec[2].y, rec[3].x, rec[3].y};
        const V2<double> r2{rec[4].x, rec[4].y};
        if (refop) build_env<double, Pat, false>(V, r0, r1, r2, dt, E);
        else build_env<double, Pat, Pat::fossen>(V, r0, r1, r2, dt, E);
    }
    double tau[6];
    wrench<double, DR, DR>(V, E, act, true, tau);
    Band64Out o;
    o.failed = 0;
    // failure = a component non-finite or outside the fp32 range: the fp32
    // engine's own failure criterion (model.rs:186-193 with an fp32 state).  The
    // Fossen path runs every sub-step unchecked and tests the final state; only
    // a failed step is re-run from the start with a check after each sub-step
    // (keeping the last good state), like the fp32 kernel's replay_env.
    bool checked = !Pat::fossen || refop;
    if (!checked) {
        double t[12];
#pragma unroll
        for (int i = 0; i < 12; ++i) t[i] = s[i];
#if UUV_BAND_CLOCK >= 2
        const long long c0 = clock64() + (long long)(t[4] * 0.0);
#endif
        if constexpr (!DR && REGE) {   // the vehicle constants the sub-step reads, in registers
            EnvParams<double, true> R;
            reg_vehicle64(V, R);
#pragma unroll 1
            for (int k = 0; k < p.task.n_substeps; ++k) substep_f64<true, false>(V, R, t, tau, dt);
        } else
#pragma unroll 1
        for (int k = 0; k < p.task.n_substeps; ++k) substep_f64<DR, false>(V, E, t, tau, dt);
#if UUV_BAND_CLOCK >= 2
        if (threadIdx.x == 0 && blockIdx.x < TL_BLOCKS && t[4] != 12345.0) {
            g_uuv_tl[TL_BAND_LOOP_CYC][blockIdx.x] = clock64() - c0;
            g_uuv_tl[TL_BAND_LOOP_N][blockIdx.x] = p.task.n_substeps;
        }
#endif
        if (f32_range12(t)) {
#pragma unroll
            for (int i = 0; i < 12; ++i) s[i] = t[i];
        } else {
            checked = true;
        }
    }
    if (checked) {
#pragma unroll 1
        for (int k = 0; k < p.task.n_substeps; ++k) {
            bool ok;
            if (Pat::fossen && !refop) {
                ok = substep_f64<DR, true>(V, E, s, tau, dt);
            } else {   // reference operation order (dense pattern, or band_refop)
                double t[12];
#pragma unroll
                for (int i = 0; i < 12; ++i) t[i] = s[i];
                ok = substep<double, DR, Pat>(V, E, t, tau, dt) && f32_range12(t);
                if (ok) {
#pragma unroll
                    for (int i = 0; i < 12; ++i) s[i] = t[i];
                }
            }
            if (!ok) {
                o.failed = 1;
                break;
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 12; ++i) o.v[i] = (float)s[i];
    return o;
}

// Per-thread episode-statistics accumulator (one or two envs per thread).
struct StatAcc {
    float rew = 0.f, epret = 0.f;
    int eplen = 0, n_tr = 0, n_dv = 0, n_fl = 0, n_act = 0, n_err = 0, n_b64 = 0;
};

// Band candidates: envs inside |theta| <= band_theta whose pitch could leave it
// within this control step -- moving toward the band edge at the current pitch
// rate theta_dot = cos(phi) q - sin(phi) r (dynamics.py:279-282):
//   |theta| + control_dt max(0, sign(theta) theta_dot) + margin > band_theta,
// margin = 0.01 + 8 control_dt^2 rad for the pitch acceleration over the step
// (calibrated on the oracle under bench actions: the largest margin an actual
// band exit needed was 0.0033 rad at control_dt = 0.05 s, tools/band_calibrate.py).
// The decision is stored with the state (EngineP::band_f), so the step kernel and
// the band kernel read the same bit; a miss is still computed in fp64
// (band_tail), only later.
__device__ __forceinline__ bool band_cand(const EngineP<float>& p, const float s[12]) {
    const float a = fabsf(s[4]);
    if (!(a <= p.band_theta)) return false;
    // |theta_dot| <= |q| + |r|: most envs are decided here, without sin / cos
    if (a + p.band_kdt * (fabsf(s[10]) + fabsf(s[11])) + p.band_margin <= p.band_theta) return false;
    float sphi, cphi;
    sincos_t(s[3], &sphi, &cphi);
    const float td = copysignf(1.0f, s[4]) * fmaf(cphi, s[10], -sphi * s[11]);
    return a + p.band_kdt * fmaxf(td, 0.0f) + p.band_margin > p.band_theta;
}

// A non-candidate whose fp32 pitch trajectory still left the band (a predictor
// miss; p.s1[e].x is the step-initial theta, still in HBM): finished from an
// fp64 recompute at the end of the step kernel (band_tail)
__device__ __forceinline__ bool band_exit(const EngineP<float>& p, int e, float thmax) {
    return thmax > p.band_exit_theta && fabsf(p.s1[e].x) <= p.band_theta;
}

// Reward / termination / auto-reset / stores / observation for one env whose
// sub-steps are done (tasks.py:219-230, batch.py:101-118, engine.rs:543-568).
// Everything one env reads from HBM, issued together in the prologue so a
// cold-cache step pays one memory round trip instead of several serialised ones
// (state, step counter, running return, actions, DR record, and -- tracking --
// the LA_PRE+1 trajectory rows the reward and observation will need).
constexpr int LA_PRE = 5;

#ifndef UUV_EPI_UNROLL
#define UUV_EPI_UNROLL 1
#endif

// RR: the LA_PRE+1 trajectory rows ride in registers across the sub-steps.
// Where registers are short (randomised or paired kernels) ptxas would park
// them in local memory -- an STL that waits for the loads before the first
// sub-step, then LDLs -- so there the prologue only prefetches their cache
// lines into L1 and finish_env reads the table (L1 hits).
// this step's band generation from a kernel's env counter (EngineP::band_ctr)
template <class T>
__device__ __forceinline__ uint32_t band_gen(const EngineP<T>& p, unsigned long long c) {
    unsigned long long k = (unsigned long long)floor((double)c * p.band_inv_n);
    const unsigned long long n = (unsigned long long)p.n_env;
    if (k * n > c) --k;
    else if ((k + 1) * n <= c) ++k;
    return (uint32_t)k & 0x7fffffffu;
}

// flag byte of generation gen (EngineP::band_f)
__device__ __forceinline__ uint32_t band_word(uint32_t gen, bool cand) {
    return ((gen & 0x7fu) << 1) | (cand ? 1u : 0u);
}

template <class T, bool TRACK, bool RR = TRACK> struct EnvIn {
    static constexpr bool kRegRows = TRACK && RR;
    T s[12];
    int32_t step;
    float ep_ret;
    uint32_t bf = 0;   // band flag byte (fp32 engines with band64): band_word(generation, candidate)
    uint32_t bk = 0;   // this step's generation (band_gen)
    V4<T> rows[kRegRows ? LA_PRE + 1 : 1];   // traj[step+1 .. step+1+LA_PRE]
};

template <class T, bool TRACK, bool RR>
__device__ __forceinline__ void load_env(const EngineP<T>& p, int e, EnvIn<T, TRACK, RR>& in) {
    const V4<T> a0 = p.s0[e], a1 = p.s1[e], a2 = p.s2[e];
    in.s[0] = a0.x; in.s[1] = a0.y; in.s[2] = a0.z; in.s[3] = a0.w;
    in.s[4] = a1.x; in.s[5] = a1.y; in.s[6] = a1.z; in.s[7] = a1.w;
    in.s[8] = a2.x; in.s[9] = a2.y; in.s[10] = a2.z; in.s[11] = a2.w;
    in.step = p.step[e];
    in.ep_ret = p.ep_ret[e];
    UUV_CHECK(e >= 0 && e < p.n_env);
    if (p.band_f) in.bf = p.band_f[e];
    if constexpr (TRACK) {
        const int tab_last = p.task.episode_len + p.task.lookahead;
        if constexpr (EnvIn<T, TRACK, RR>::kRegRows) {
#pragma unroll
            for (int k = 0; k <= LA_PRE; ++k)
                in.rows[k] = p.task.traj[min(max(in.step + 1 + k, 0), tab_last)];
        } else {   // rows step+1 .. step+1+LA_PRE span at most two 128-byte lines
            const V4<T>* r0 = p.task.traj + min(max(in.step + 1, 0), tab_last);
            const V4<T>* r1 = p.task.traj + min(max(in.step + 1 + LA_PRE, 0), tab_last);
            asm volatile("prefetch.global.L1 [%0];" ::"l"(r0));
            asm volatile("prefetch.global.L1 [%0];" ::"l"(r1));
        }
    }
}

// observation row of one env (post-reset for finished envs, batch.py:106-118),
// stored as O = T (device face) or double (host ABI)
template <class T, class O, bool TRACK, class IN>
__device__ __forceinline__ void write_obs(const TaskP<T>& tk, O* __restrict__ row, const T s[12],
                                          const IN& in, int32_t nstep, bool pre) {
    if constexpr (!TRACK) {
        V4<O>* o4 = reinterpret_cast<V4<O>*>(row);
        o4[0] = V4<O>{(O)(tk.target[0] - s[0]), (O)(tk.target[1] - s[1]),
                      (O)(tk.target[2] - s[2]), (O)obs_wrap<T>(tk.target[3] - s[3])};
        o4[1] = V4<O>{(O)obs_wrap<T>(tk.target[4] - s[4]), (O)obs_wrap<T>(tk.target[5] - s[5]),
                      (O)s[6], (O)s[7]};
        o4[2] = V4<O>{(O)s[8], (O)s[9], (O)s[10], (O)s[11]};
    } else {
        const int tab_last = tk.episode_len + tk.lookahead;
        V2<O>* o2 = reinterpret_cast<V2<O>*>(row);
        const O ephi = (O)obs_wrap<T>(T(0) - s[3]);
        const O eth = (O)obs_wrap<T>(T(0) - s[4]);
        if (IN::kRegRows && pre) {   // trajectory rows prefetched by load_env
            if constexpr (IN::kRegRows) {
#pragma unroll
                for (int k = 1; k <= LA_PRE; ++k) {
                    if (k > tk.lookahead) break;
                    const V4<T> r = in.rows[k];
                    V2<O>* q = o2 + 3 * (k - 1);
                    q[0] = V2<O>{(O)(r.x - s[0]), (O)(r.y - s[1])};
                    q[1] = V2<O>{(O)(r.z - s[2]), ephi};
                    q[2] = V2<O>{eth, (O)obs_wrap<T>(r.w - s[5])};
                }
            }
        } else if (UUV_EPI_UNROLL && tk.lookahead <= LA_PRE) {
            // table rows (L1 hits after load_env's prefetch): issue all loads first
            V4<T> r[LA_PRE];
#pragma unroll
            for (int k = 1; k <= LA_PRE; ++k)
                r[k - 1] = k <= tk.lookahead ? tk.traj[min(nstep + k, tab_last)] : V4<T>{};
#pragma unroll
            for (int k = 1; k <= LA_PRE; ++k) {
                if (k > tk.lookahead) break;
                V2<O>* q = o2 + 3 * (k - 1);
                q[0] = V2<O>{(O)(r[k - 1].x - s[0]), (O)(r[k - 1].y - s[1])};
                q[1] = V2<O>{(O)(r[k - 1].z - s[2]), ephi};
                q[2] = V2<O>{eth, (O)obs_wrap<T>(r[k - 1].w - s[5])};
            }
        } else {
#pragma unroll 1
            for (int k = 1; k <= tk.lookahead; ++k) {
                const V4<T> r = tk.traj[min(nstep + k, tab_last)];
                V2<O>* q = o2 + 3 * (k - 1);
                q[0] = V2<O>{(O)(r.x - s[0]), (O)(r.y - s[1])};
                q[1] = V2<O>{(O)(r.z - s[2]), ephi};
                q[2] = V2<O>{eth, (O)obs_wrap<T>(r.w - s[5])};
            }
        }
        V2<O>* q = o2 + 3 * tk.lookahead;
        q[0] = V2<O>{(O)s[6], (O)s[7]};
        q[1] = V2<O>{(O)s[8], (O)s[9]};
        q[2] = V2<O>{(O)s[10], (O)s[11]};
    }
}

// Dynamic shared memory: observation rows of the block's envs (stage_obs).
extern __shared__ __align__(16) unsigned char uuv_smem[];

template <class T, bool TRACK, bool DR, int SLOT, class Pat, class IN>
__device__ __forceinline__ void finish_env(const EngineP<T>& p, int e, int li, uint64_t g,
                                           T s[12], const IN& in, bool failed,
                                           void* __restrict__ obs, void* __restrict__ rew,
                                           uint8_t* __restrict__ done,
                                           int8_t* __restrict__ reason, StatAcc& st) {
    const VehP<T>& V = p.veh[SLOT];
    const TaskP<T>& tk = p.task;
    const int32_t step = in.step;
    // reward / termination: failure > divergence > truncation
    const int32_t ns = step + 1;
    const int tab_last = tk.episode_len + tk.lookahead;
    T rx, ry, rz;
    if constexpr (TRACK) {
        V4<T> r;
        if constexpr (IN::kRegRows) r = in.rows[0];
        else r = tk.traj[min(max(ns, 0), tab_last)];
        rx = r.x; ry = r.y; rz = r.z;
    } else {
        rx = tk.target[0]; ry = tk.target[1]; rz = tk.target[2];
    }
    const T dx = rx - s[0], dy = ry - s[1], dz = rz - s[2];
    const T pe = sqrt(dx * dx + dy * dy + dz * dz);
    const T reward = -pe;
    int rc = -1;
    if (failed) rc = 2;
    else if (pe > tk.div_radius) rc = 1;
    else if (ns >= tk.episode_len) rc = 0;

    float er = in.ep_ret + (float)reward;
    int32_t nstep = ns;
    if (rc >= 0) {
        st.epret += er;
        st.eplen += ns;
        er = 0.0f;
        if (p.final_obs) {   // terminal observation before the auto-reset (TorchRL / gym)
            T* row = (T*)p.final_obs + (size_t)e * tk.obs_dim;
            write_obs<T, T, TRACK>(tk, row, s, in, ns, false);
        }
        const uint64_t seed = *p.seed_dev;
        if constexpr (DR) {
            if (p.ranges.per_episode) {   // engine.rs:553-558, batch.py:107-110
                uint64_t pc = p.param_ctr[e];
                V4<T> n0, n1;
                V2<T> n2;
                if (dr_draw<T, Pat>(V, p.ranges, seed, g, pc, n0, n1, n2,
                                    p.dr64 ? p.dr64 + (size_t)e * 5 : nullptr)) {
                    p.dr0[e] = n0; p.dr1[e] = n1; p.dr2[e] = n2;
                } else {
                    st.n_err += 1;
                    if (p.err_flag) *p.err_flag = 1;   // host ABI: uuvsim_step reports code 4
                }
                p.param_ctr[e] = pc;
            }
        }
        const uint64_t ctr = p.reset_ctr[e];
        const State12<T> rs = reset_state<T>(tk, seed, g, ctr);
#pragma unroll
        for (int i = 0; i < 12; ++i) s[i] = rs.v[i];
        p.reset_ctr[e] = ctr + 6;
        nstep = 0;
    }
    p.ep_ret[e] = er;
    p.step[e] = nstep;
    if constexpr (!is_f64<T>()) {   // next step's band decision, one generation on
        if (p.band_f) p.band_f[e] = (uint8_t)band_word(in.bk + 1u, band_cand(p, s));
    }
    p.s0[e] = V4<T>{s[0], s[1], s[2], s[3]};
    p.s1[e] = V4<T>{s[4], s[5], s[6], s[7]};
    p.s2[e] = V4<T>{s[8], s[9], s[10], s[11]};

    // observation (post-reset for finished envs, batch.py:106-118)
    const bool pre = IN::kRegRows && rc < 0 && tk.lookahead <= LA_PRE;
    // staged: the row goes to shared memory and the block stores all rows
    // contiguously afterwards (flush_obs); else straight to HBM
    const size_t D = (size_t)tk.obs_dim;
    if (p.io_f64) {
        UUV_CHECK(e >= 0 && e < p.n_env && li < 2 * BLOCK);
        double* row = (p.stage_obs && li >= 0) ? (double*)uuv_smem + (size_t)li * D
                                               : (double*)obs + (size_t)e * D;
        write_obs<T, double, TRACK>(tk, row, s, in, nstep, pre);
        ((double*)rew)[e] = (double)reward;
    } else {
        UUV_CHECK(e >= 0 && e < p.n_env && li < 2 * BLOCK);
        T* row = (p.stage_obs && li >= 0) ? (T*)uuv_smem + (size_t)li * D : (T*)obs + (size_t)e * D;
        write_obs<T, T, TRACK>(tk, row, s, in, nstep, pre);
        ((T*)rew)[e] = reward;
    }
    done[e] = rc >= 0 ? 1 : 0;
    if (p.done_f32) p.done_f32[e] = rc >= 0 ? 1.0f : 0.0f;
    if (reason) reason[e] = (int8_t)rc;
    st.rew += (float)reward;
    st.n_act += 1;
    st.n_tr += rc == 0;
    st.n_dv += rc == 1;
    st.n_fl += rc == 2;
}

// start of env e's action row (elements are T, or f64 on the host-ABI path)
template <class T>
__device__ __forceinline__ const void* act_row(const EngineP<T>& p, const void* act, int e) {
    return p.io_f64 ? (const void*)((const double*)act + (size_t)e * p.act_dim)
                    : (const void*)((const T*)act + (size_t)e * p.act_dim);
}

template <class T>
__device__ __forceinline__ void load_state(const EngineP<T>& p, int e, T s[12]) {
    const V4<T> a0 = p.s0[e], a1 = p.s1[e], a2 = p.s2[e];
    s[0] = a0.x; s[1] = a0.y; s[2] = a0.z; s[3] = a0.w;
    s[4] = a1.x; s[5] = a1.y; s[6] = a1.z; s[7] = a1.w;
    s[8] = a2.x; s[9] = a2.y; s[10] = a2.z; s[11] = a2.w;
}

// Outcome of one env in the step kernel: finished here, left to the concurrent
// band kernel (candidate), or left to this kernel's fp64 tail (band_tail).
enum EnvCode { ENV_DONE = 0, ENV_BAND = 1, ENV_TAIL = 2 };

// This step's band generation in the step kernels (EngineP::band_ctr).  One
// thread per block claims the block's envs with a fetch-add on the step
// kernel's counter -- the value it returns is the count before the block, so
// gen = value / n_env -- issued at the block's start, its result published
// through shared memory behind named barrier 1 once the block's env loads are
// in flight.  One counter access per block (not one load per warp on a single
// address) and no counter update at the block's end.
//   mode BG_NONE: no band bookkeeping; BG_SYNC: publish + barrier here (every
//   thread of the block passes exactly one BG_SYNC or band_gen_sync); BG_GIVEN:
//   gen already known; BG_LOAD: per-thread counter load (persistent kernel,
//   counted at its end by band_count).
enum { BG_NONE = 0, BG_SYNC = 1, BG_GIVEN = 2, BG_LOAD = 3 };
struct BandGen {
    unsigned long long c = 0;   // fetch-add result (thread 0 of the block)
    uint32_t gen = 0;
    int mode = BG_NONE;
};

// block's fetch-add on the step counter (thread 0; the others get 0)
__device__ __forceinline__ BandGen band_claim(const EngineP<float>& p, int first, int span) {
    BandGen bg;
    if (!p.band_f) return bg;
    bg.mode = BG_SYNC;
    if (threadIdx.x == 0) {
        const int n = min(span, p.n_env - first);
        bg.c = atomicAdd(p.band_ctr, (unsigned long long)max(n, 0));
    }
    return bg;
}

__device__ __forceinline__ uint32_t band_gen_sync(const EngineP<float>& p, const BandGen& bg) {
    __shared__ uint32_t s_gen;
    if (threadIdx.x == 0) s_gen = band_gen(p, bg.c);
    asm volatile("barrier.sync 1, %0;" ::"r"((int)blockDim.x) : "memory");
    return s_gen;
}

__device__ __forceinline__ uint32_t band_gen_of(const EngineP<float>& p, const BandGen& bg) {
    if (bg.mode == BG_SYNC) return band_gen_sync(p, bg);
    if (bg.mode == BG_GIVEN) return bg.gen;
    return band_gen(p, p.band_ctr[0]);
}

// One env per thread (every precision / pattern / randomisation mode).
template <class T, bool TRACK, bool DR, int SLOT, class Pat>
__device__ __forceinline__ int step_env(const EngineP<T>& p, int e, int li, uint64_t g,
                                        const void* __restrict__ act, void* __restrict__ obs,
                                        void* __restrict__ rew, uint8_t* __restrict__ done,
                                        int8_t* __restrict__ reason, StatAcc& st,
                                        const BandGen& bg) {
    const VehP<T>& V = p.veh[SLOT];
    const TaskP<T>& tk = p.task;
    EnvIn<T, TRACK, !DR> in;
    load_env<T, TRACK>(p, e, in);
    T* s = in.s;
    // the action row and the DR record too, issued before the band ownership check
    // (which may wait for the block's counter claim) so every load of the step
    // shares one memory round trip
    T av[MAX_THR];
    load_actions<T>(V, act_row(p, act, e), p.io_f64, av);
    [[maybe_unused]] V4<T> d0, d1;
    [[maybe_unused]] V2<T> d2;
    if constexpr (DR) {
        d0 = p.dr0[e];
        d1 = p.dr1[e];
        d2 = p.dr2[e];
    }
    // not this kernel's env this step: a band candidate (or already stepped by the
    // concurrent band kernel)
    if constexpr (!is_f64<T>()) {
        if (bg.mode != BG_NONE) {
            in.bk = band_gen_of(p, bg);
            if (in.bf != band_word(in.bk, false)) return ENV_BAND;
        }
    }
    if constexpr (!is_f64<T>()) {
        UUV_TLV(TL_STEP_LOADED, s[4] + (float)in.step);
        prewrap(s);
    }

    // fp32: Fossen-pattern parameters in registers (UUV_PACK_CONSTS) or in the
    // constant bank (default: keeps FFMAs at two register reads)
    constexpr bool REG = DR || (UUV_PACK_CONSTS && !is_f64<T>() && Pat::fossen);
    EnvParams<T, REG> E;
    [[maybe_unused]] float dt32 = (float)tk.sub_dt;
    [[maybe_unused]] TrigK K = TrigK::imm();
    if constexpr (!is_f64<T>() && !DR && REG) {
        RegPack R;
        load_pack(p.vpack + SLOT * PACK_F4, R);
        load_regs<Pat>(R, E, dt32, K);
    }
    if constexpr (DR) build_env<T, Pat>(V, d0, d1, d2, (T)tk.sub_dt, E);
    T tau[6];
    wrench_vals<T, DR, REG>(V, E, av, tau);

    bool failed = false;
    if constexpr (is_f64<T>()) {
        const T dt = tk.sub_dt;
#pragma unroll 1
        for (int k = 0; k < tk.n_substeps; ++k) {
            if (!substep<T, DR, Pat>(V, E, s, tau, dt)) {
                failed = true;
                break;
            }
        }
    } else {
        // in-place sub-steps without an early exit; the first non-finite one is
        // recorded and the env replayed from its initial state (still in HBM)
        // up to the last finite sub-step
        const float dt = dt32;
        float thm = 0.0f;   // max |theta| over the sub-steps
#pragma unroll 1
        for (int k = 0; k < tk.n_substeps; ++k) {
            substep_fused<DR, Pat, false>(V, E, s, tau, dt, K);
            thm = fmaxf(thm, fabsf(s[4]));
        }
        UUV_TLV(TL_STEP_SUBS, thm);
        if (band_exit(p, e, thm)) return ENV_TAIL;
        if (!all_finite12(s)) {
            failed = true;
            replay_env<DR, Pat>(p, V, E, e, tau, dt, K, tk.n_substeps, s);
        }
    }
    finish_env<T, TRACK, DR, SLOT, Pat>(p, e, li, g, s, in, failed, obs, rew, done, reason, st);
    return ENV_DONE;
}

// Two envs per thread sharing the register-resident vehicle constants (fp32,
// Fossen pattern, no randomisation): two independent dependency chains per
// thread hide latency at half the registers of two threads.
template <bool TRACK, int SLOT>
__device__ __forceinline__ int pair_core(const EngineP<float>& p, int e0, int e1, int li0,
                                          int li1, EnvIn<float, TRACK, false>& in0,
                                          EnvIn<float, TRACK, false>& in1, const void* act0,
                                          const void* act1, bool io_f64, void* __restrict__ obs,
                                          void* __restrict__ rew, uint8_t* __restrict__ done,
                                          int8_t* __restrict__ reason, StatAcc& st,
                                          const BandGen& bg) {
    using Pat = PatFossen;
    const VehP<float>& V = p.veh[SLOT];
    const TaskP<float>& tk = p.task;
    float* s0 = in0.s;
    float* s1 = in1.s;
    float av0[MAX_THR], av1[MAX_THR];   // before the band check (see step_env)
    load_actions<float>(V, act0, io_f64, av0);
    load_actions<float>(V, act1, io_f64, av1);
    if (bg.mode != BG_NONE) in0.bk = in1.bk = band_gen_of(p, bg);
    const bool cand0 = bg.mode != BG_NONE && in0.bf != band_word(in0.bk, false);
    const bool cand1 = bg.mode != BG_NONE && in1.bf != band_word(in1.bk, false);
    UUV_TLV(TL_STEP_LOADED, s0[4] + s1[4] + (float)in0.step);
    prewrap(s0);
    prewrap(s1);
    constexpr bool REG = UUV_PACK_CONSTS;
    EnvParams<float, REG> E;
    float dt = tk.sub_dt;
    TrigK K = TrigK::imm();
    if constexpr (REG && SLOT >= 0) {
        RegPack R;
        load_pack(p.vpack + SLOT * PACK_F4, R);
        load_regs<Pat>(R, E, dt, K);
    }
    float tau0[6], tau1[6];
    wrench_vals<float, false, REG>(V, E, av0, tau0);
    wrench_vals<float, false, REG>(V, E, av1, tau1);
    float thm0 = 0.0f, thm1 = 0.0f;   // max |theta| over the sub-steps
#pragma unroll 1
    for (int k = 0; k < tk.n_substeps; ++k) {
        substep_fused<false, Pat, false>(V, E, s0, tau0, dt, K);
        substep_fused<false, Pat, false>(V, E, s1, tau1, dt, K);
        thm0 = fmaxf(thm0, fabsf(s0[4]));
        thm1 = fmaxf(thm1, fabsf(s1[4]));
    }
    UUV_TLV(TL_STEP_SUBS, thm0 + thm1);
    // codes: candidates (decided on entry) belong to the band kernel, misses to
    // the fp64 tail; both computed here anyway (two lockstep chains)
    const int c0 = cand0 ? ENV_BAND : (band_exit(p, e0, thm0) ? ENV_TAIL : ENV_DONE);
    const int c1 = cand1 ? ENV_BAND : (band_exit(p, e1, thm1) ? ENV_TAIL : ENV_DONE);
    const bool f0 = c0 == ENV_DONE && !all_finite12(s0), f1 = c1 == ENV_DONE && !all_finite12(s1);
    if (f0) replay_env<false, Pat>(p, V, E, e0, tau0, dt, K, tk.n_substeps, s0);
    if (f1) replay_env<false, Pat>(p, V, E, e1, tau1, dt, K, tk.n_substeps, s1);
    const uint64_t g0 = p.env_offset + (uint64_t)e0, g1 = p.env_offset + (uint64_t)e1;
    if (c0 == ENV_DONE)
        finish_env<float, TRACK, false, SLOT, Pat>(p, e0, li0, g0, s0, in0, f0, obs, rew, done,
                                                   reason, st);
    if (c1 == ENV_DONE)
        finish_env<float, TRACK, false, SLOT, Pat>(p, e1, li1, g1, s1, in1, f1, obs, rew, done,
                                                   reason, st);
    return c0 | (c1 << 2);
}

template <bool TRACK, int SLOT>
__device__ __forceinline__ int step_pair(const EngineP<float>& p, int e0, int e1, int li0,
                                          int li1,
                                          const void* __restrict__ act, void* __restrict__ obs,
                                          void* __restrict__ rew, uint8_t* __restrict__ done,
                                          int8_t* __restrict__ reason, StatAcc& st,
                                        const BandGen& bg) {
    EnvIn<float, TRACK, false> in0, in1;
    load_env<float, TRACK>(p, e0, in0);
    load_env<float, TRACK>(p, e1, in1);
    return pair_core<TRACK, SLOT>(p, e0, e1, li0, li1, in0, in1, act_row(p, act, e0),
                                  act_row(p, act, e1), p.io_f64, obs, rew, done, reason, st, bg);
}

// Block-level episode statistics: warp reductions -> shared memory -> one
// read-modify-write of this block's own partial slot (no atomics, deterministic).
template <int NT = BLOCK>
__device__ __forceinline__ void block_stats(double* __restrict__ part, const StatAcc& st) {
    __shared__ double sh[NT / 32][NSTAT];
    const unsigned full = 0xffffffffu;
    float r = st.rew, er = st.epret;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        r += __shfl_xor_sync(full, r, o);
        er += __shfl_xor_sync(full, er, o);
    }
    const int el = __reduce_add_sync(full, st.eplen);
    const int n_tr = __reduce_add_sync(full, st.n_tr);
    const int n_dv = __reduce_add_sync(full, st.n_dv);
    const int n_fl = __reduce_add_sync(full, st.n_fl);
    const int n_ac = __reduce_add_sync(full, st.n_act);
    const int n_er = __reduce_add_sync(full, st.n_err);
    const int n_b64 = __reduce_add_sync(full, st.n_b64);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
        sh[w][ST_REWARD] = r;
        sh[w][ST_DONE_TRUNC] = n_tr;
        sh[w][ST_DONE_DIV] = n_dv;
        sh[w][ST_DONE_FAIL] = n_fl;
        sh[w][ST_EP_RETURN] = er;
        sh[w][ST_EP_LEN] = el;
        sh[w][ST_STEPS] = n_ac;
        sh[w][ST_RESAMPLE_ERR] = n_er;
        sh[w][ST_BAND64] = n_b64;
    }
    __syncthreads();
    if (threadIdx.x < NSTAT) {
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < NT / 32; ++i) acc += sh[i][threadIdx.x];
        // RED (no return): one update per slot per step, steps are stream-ordered,
        // so the accumulation order -- and the sum -- is deterministic
        atomicAdd(&part[(size_t)blockIdx.x * NSTAT + threadIdx.x], acc);
    }
}

template <class T, bool TRACK, bool DR, bool MIX, class Pat>
__device__ __forceinline__ int one_env(const EngineP<T>& p, int e, int li, const void* act,
                                       void* obs, void* rew, uint8_t* done, int8_t* reason,
                                       StatAcc& st, const BandGen& bg) {
    const uint64_t g = p.env_offset + (uint64_t)e;
    bool slot1 = false;
    if constexpr (MIX) slot1 = (int64_t)g >= p.mix_bound0;
    if (!slot1)
        return step_env<T, TRACK, DR, 0, Pat>(p, e, li, g, act, obs, rew, done, reason, st, bg);
    if constexpr (MIX)
        return step_env<T, TRACK, DR, 1, Pat>(p, e, li, g, act, obs, rew, done, reason, st, bg);
    return ENV_DONE;
}

// Store the block's staged observation rows (envs [first, first+n)) with
// contiguous 128-bit stores: full 128-B lines instead of one partial sector
// per env and store instruction.  Rows flagged in `skip` (bit per row: envs this
// kernel did not finish -- band candidates, fp64 tail) are left untouched; rows
// are a multiple of 8 bytes, so 16-byte chunks (rows of 16k bytes) or 8-byte
// chunks never straddle a skipped and a kept row.
template <class C>
__device__ __forceinline__ void copy_rows(unsigned char* __restrict__ dst, size_t nbytes,
                                          uint32_t row_bytes, const uint32_t* skip) {
    const C* src = reinterpret_cast<const C*>(uuv_smem);
    C* d = reinterpret_cast<C*>(dst);
    const size_t n = nbytes / sizeof(C);
    if (!skip) {
        for (size_t i = threadIdx.x; i < n; i += blockDim.x) d[i] = src[i];
        return;
    }
    // row of chunk i, tracked incrementally (one division per thread)
    const uint32_t step_b = blockDim.x * (uint32_t)sizeof(C);
    const uint32_t drow = step_b / row_bytes, doff = step_b % row_bytes;
    uint32_t row = threadIdx.x * (uint32_t)sizeof(C) / row_bytes;
    uint32_t off = threadIdx.x * (uint32_t)sizeof(C) % row_bytes;
    for (size_t i = threadIdx.x; i < n; i += blockDim.x) {
        if (!((skip[row >> 5] >> (row & 31)) & 1u)) d[i] = src[i];
        row += drow;
        off += doff;
        if (off >= row_bytes) {
            off -= row_bytes;
            ++row;
        }
    }
}

template <class T>
__device__ __forceinline__ void flush_obs(const EngineP<T>& p, void* __restrict__ obs, int first,
                                          int n, const uint32_t* skip_mask = nullptr) {
    __syncthreads();
    if (n <= 0) return;
    const size_t D = (size_t)p.task.obs_dim;
    const size_t nel = (size_t)n * D;
    const size_t esz = p.io_f64 ? 8 : sizeof(T);
    const size_t nbytes = nel * esz;
    const uint32_t rb = (uint32_t)(D * esz);
    unsigned char* dst = (unsigned char*)obs + (size_t)first * D * esz;
    // any row to skip in this block?
    const uint32_t* skip = nullptr;
    if (skip_mask) {
        uint32_t any = 0;
        for (int w = 0; w < (n + 31) / 32; ++w) any |= skip_mask[w];
        if (any) skip = skip_mask;
    }
    if (((uintptr_t)dst & 15) == 0 && (nbytes & 15) == 0 && (!skip || (rb & 15) == 0)) {
        copy_rows<float4>(dst, nbytes, rb, skip);
    } else if (((uintptr_t)dst & 7) == 0 && (nbytes & 7) == 0 && (rb & 7) == 0) {
        copy_rows<float2>(dst, nbytes, rb, skip);
    } else {
        copy_rows<uint32_t>(dst, nbytes, rb, skip);
    }
}

// Host-ABI zero-copy step (EngineP::stage_act): the block's f64 action rows are
// read from the mapped page-locked buffer with consecutive 8-byte loads (each warp
// instruction covers 256 contiguous bytes, whole lines on the host link, instead of
// six 48-byte-strided loads per env) into shared memory behind the staged
// observation rows.  Returns the base act_row() offsets by the block's env index.
template <class T>
__device__ __forceinline__ const void* stage_actions(const EngineP<T>& p, const void* act,
                                                     int first, int n, int rows) {
    const size_t obs_bytes = p.stage_obs ? (size_t)rows * p.task.obs_dim * 8 : 0;
    double* sa = reinterpret_cast<double*>(uuv_smem + obs_bytes);
    const double* src = static_cast<const double*>(act) + (size_t)first * p.act_dim;
    const int cnt = n * p.act_dim;
    // all loads in flight before the first store: a load -> store loop would pay
    // one host-link round trip per iteration
    double v[2 * MAX_THR];
#pragma unroll
    for (int k = 0; k < 2 * MAX_THR; ++k) {
        const int i = threadIdx.x + k * BLOCK;
        if (i < cnt) v[k] = src[i];
    }
#pragma unroll
    for (int k = 0; k < 2 * MAX_THR; ++k) {
        const int i = threadIdx.x + k * BLOCK;
        if (i < cnt) sa[i] = v[k];
    }
    __syncthreads();
    return reinterpret_cast<const void*>(reinterpret_cast<uintptr_t>(sa) -
                                         (uintptr_t)first * p.act_dim * sizeof(double));
}

// Everything the fp64 recompute of env e needs, loaded in one round trip, then
// the recompute and the env's reward / termination / reset / stores /
// observation (written directly, never staged).
template <bool TRACK, bool DR, bool MIX, class Pat, bool REGE = false, bool REFOP = false>
__device__ __forceinline__ void band_env(const EngineP<float>& p, const VehP<double>& V0,
                                         const VehP<double>& V1, int e, uint32_t gen, const void* act,
                                         void* __restrict__ obs, void* __restrict__ rew,
                                         uint8_t* __restrict__ done, int8_t* __restrict__ reason,
                                         StatAcc& st) {
    const uint64_t g = p.env_offset + (uint64_t)e;
    const bool slot1 = MIX && (int64_t)g >= p.mix_bound0;
    EnvIn<float, TRACK, false> in;
    load_env<float, TRACK>(p, e, in);
    in.bk = gen;
    V2<double> rec[5];
    if constexpr (DR) {
#pragma unroll
        for (int k = 0; k < 5; ++k) rec[k] = p.dr64[(size_t)e * 5 + k];
    }
    const void* arow = act_row(p, act, e);
    const int nthr = slot1 ? V1.n_thr : V0.n_thr;
    double a[MAX_THR];
#pragma unroll
    for (int k = 0; k < MAX_THR; ++k)
        a[k] = k >= nthr ? 0.0
               : p.io_f64 ? ((const double*)arow)[k]
                          : (double)((const float*)arow)[k];
    UUV_TLV(TL_BAND_LOADED, in.s[4] + (float)a[0] + (float)in.step);
    const Band64Out r = slot1 ? replay_band64<DR, Pat, REGE, REFOP>(p, V1, in.s, rec, a)
                              : replay_band64<DR, Pat, REGE, REFOP>(p, V0, in.s, rec, a);
    UUV_TLV(TL_BAND_REPLAYED, r.v[4]);
#pragma unroll
    for (int k = 0; k < 12; ++k) in.s[k] = r.v[k];
    st.n_b64 += 1;
    if (slot1) {
        if constexpr (MIX)
            finish_env<float, TRACK, DR, 1, Pat>(p, e, -1, g, in.s, in, r.failed != 0, obs, rew,
                                                 done, reason, st);
    } else {
        finish_env<float, TRACK, DR, 0, Pat>(p, e, -1, g, in.s, in, r.failed != 0, obs, rew, done,
                                             reason, st);
    }
}

// Step-kernel tail for a band-predictor miss (an env that was not a candidate
// but whose fp32 pitch trajectory left the band): recomputed in fp64 after the
// block's stores and statistics, out of line so the hot path carries no fp64
// code; its statistics go to the block's partial slot with atomics.
template <bool TRACK, bool DR, bool MIX, class Pat>
__device__ __noinline__ void band_tail(const EngineP<float>& p, int e, const void* act,
                                       void* obs, void* rew, uint8_t* done, int8_t* reason) {
    StatAcc st;
    // this step's generation (mod 128, all band_word keeps) from the env's own
    // flag byte, untouched this step: the step kernel's counter may already
    // have moved on
    UUV_CHECK(e >= 0 && e < p.n_env);
    const uint32_t gen = (uint32_t)p.band_f[e] >> 1;
    if (p.band_refop)   // reference operation order (FMA-contracted in this translation unit)
        band_env<TRACK, DR, MIX, Pat, false, true>(p, p.veh64_dev[0], p.veh64_dev[1], e, gen, act,
                                                   obs, rew, done, reason, st);
    else
        band_env<TRACK, DR, MIX, Pat>(p, p.veh64_dev[0], p.veh64_dev[1], e, gen, act, obs, rew,
                                      done, reason, st);
    if (p.stats_on) {
        double* part = p.stats + (size_t)blockIdx.x * NSTAT;
        atomicAdd(part + ST_REWARD, (double)st.rew);
        atomicAdd(part + ST_STEPS, 1.0);
        atomicAdd(part + ST_BAND64, 1.0);
        if (st.n_tr) atomicAdd(part + ST_DONE_TRUNC, 1.0);
        if (st.n_dv) atomicAdd(part + ST_DONE_DIV, 1.0);
        if (st.n_fl) atomicAdd(part + ST_DONE_FAIL, 1.0);
        if (st.eplen) {
            atomicAdd(part + ST_EP_RETURN, (double)st.epret);
            atomicAdd(part + ST_EP_LEN, (double)st.eplen);
        }
        if (st.n_err) atomicAdd(part + ST_RESAMPLE_ERR, (double)st.n_err);
    }
}

// persistent TMA kernel (BG_LOAD): the block's envs [first, first + span) are done
// with the step: advance the step kernel's env counter (fire-and-forget;
// EngineP::band_ctr; after a barrier: every thread is past its last counter read)
__device__ __forceinline__ void band_count(const EngineP<float>& p, int first, int span) {
    if (!p.band_f) return;
    __syncthreads();
    const int n = min(span, p.n_env - first);
    if (threadIdx.x == 0 && n > 0) atomicAdd(p.band_ctr, (unsigned long long)n);
}

// rows this block did not finish (band candidates, tail envs), one bit per row
__device__ __forceinline__ void mark_rows(uint32_t* mask, int row, bool skip) {
    const uint32_t b = __ballot_sync(0xffffffffu, skip);
    UUV_CHECK(row >= 0 && row < 2 * BLOCK);
    if ((threadIdx.x & 31) == 0) mask[row >> 5] = b;
}

template <class T, bool TRACK, bool DR, bool MIX, class Pat>
__global__ void __launch_bounds__(BLOCK, is_f64<T>() ? STEP_MIN_BLOCKS_F64
                                      : (DR ? (Pat::fossen ? STEP_MIN_BLOCKS_DR : STEP_MIN_BLOCKS_F64)
                                            : (TRACK ? STEP_MIN_BLOCKS_TRACK : STEP_MIN_BLOCKS)))
k_step(const __grid_constant__ EngineP<T> p, const void* __restrict__ act,
       void* __restrict__ obs, void* __restrict__ rew, uint8_t* __restrict__ done,
       int8_t* __restrict__ reason) {
    pdl_enter(p.pdl != 0);
    UUV_TL(TL_STEP_START);
    if (p.stagger_ns) __nanosleep((unsigned)((long long)blockIdx.x * p.stagger_ns / gridDim.x));
    const int e = blockIdx.x * BLOCK + threadIdx.x;
    if (p.stage_act) {
        const int first = blockIdx.x * BLOCK;
        act = stage_actions(p, act, first, min(BLOCK, p.n_env - first), BLOCK);
    }
    StatAcc st;
    int code = ENV_DONE;
    BandGen bg;
    if constexpr (!is_f64<T>()) bg = band_claim(p, blockIdx.x * BLOCK, BLOCK);
    if (e < p.n_env) {
        code = one_env<T, TRACK, DR, MIX, Pat>(p, e, threadIdx.x, act, obs, rew, done, reason, st, bg);
    } else if constexpr (!is_f64<T>()) {
        if (bg.mode == BG_SYNC) band_gen_sync(p, bg);
    }
    pdl_trigger_late(p.pdl != 0);
    if (p.stage_obs) {
        __shared__ uint32_t skip[BLOCK / 32];
        mark_rows(skip, threadIdx.x, code != ENV_DONE);
        const int first = blockIdx.x * BLOCK;
        flush_obs<T>(p, obs, first, min(BLOCK, p.n_env - first), skip);
    }
    if (p.stats_on) block_stats(p.stats, st);
    if constexpr (!is_f64<T>()) {
        if (code == ENV_TAIL) band_tail<TRACK, DR, MIX, Pat>(p, e, act, obs, rew, done, reason);
    }
    UUV_TL(TL_STEP_END);
}

// Paired variant: block b covers envs [2*BLOCK*b, 2*BLOCK*(b+1)); thread t
// steps envs t and t+BLOCK of that span (both loads stay coalesced).
template <bool TRACK, bool MIX>
__global__ void __launch_bounds__(BLOCK, PAIR_MIN_BLOCKS)
k_step_pair(const __grid_constant__ EngineP<float> p, const void* __restrict__ act,
            void* __restrict__ obs, void* __restrict__ rew, uint8_t* __restrict__ done,
            int8_t* __restrict__ reason) {
    pdl_enter(p.pdl != 0);
    UUV_TL(TL_STEP_START);
    if (p.stagger_ns) __nanosleep((unsigned)((long long)blockIdx.x * p.stagger_ns / gridDim.x));
    const int e0 = blockIdx.x * (2 * BLOCK) + threadIdx.x, e1 = e0 + BLOCK;
    if (p.stage_act) {
        const int first = blockIdx.x * (2 * BLOCK);
        act = stage_actions(p, act, first, min(2 * BLOCK, p.n_env - first), 2 * BLOCK);
    }
    StatAcc st;
    const bool a0 = e0 < p.n_env, a1 = e1 < p.n_env;
    const int sl0 = MIX && (int64_t)(p.env_offset + (uint64_t)e0) >= p.mix_bound0;
    const int sl1 = MIX && (int64_t)(p.env_offset + (uint64_t)e1) >= p.mix_bound0;
    const int l0 = threadIdx.x, l1 = threadIdx.x + BLOCK;
    int c0 = ENV_DONE, c1 = ENV_DONE;
    BandGen bg = band_claim(p, blockIdx.x * (2 * BLOCK), 2 * BLOCK);
    if (a0 && a1 && sl0 == sl1) {
        int c = ENV_DONE;
        if (sl0 == 0) c = step_pair<TRACK, 0>(p, e0, e1, l0, l1, act, obs, rew, done, reason, st, bg);
        else if constexpr (MIX) c = step_pair<TRACK, 1>(p, e0, e1, l0, l1, act, obs, rew, done, reason, st, bg);
        c0 = c & 3;
        c1 = c >> 2;
    } else {   // block-edge threads: generation first (one barrier per thread), then the envs
        if (bg.mode == BG_SYNC) {
            bg.gen = band_gen_sync(p, bg);
            bg.mode = BG_GIVEN;
        }
        if (a0) c0 = one_env<float, TRACK, false, MIX, PatFossen>(p, e0, l0, act, obs, rew, done, reason, st, bg);
        if (a1) c1 = one_env<float, TRACK, false, MIX, PatFossen>(p, e1, l1, act, obs, rew, done, reason, st, bg);
    }
    pdl_trigger_late(p.pdl != 0);
    if (p.stage_obs) {
        __shared__ uint32_t skip[2 * BLOCK / 32];
        mark_rows(skip, l0, c0 != ENV_DONE);
        mark_rows(skip, l1, c1 != ENV_DONE);
        const int first = blockIdx.x * (2 * BLOCK);
        flush_obs<float>(p, obs, first, min(2 * BLOCK, p.n_env - first), skip);
    }
    if (p.stats_on) block_stats(p.stats, st);
    if (c0 == ENV_TAIL) band_tail<TRACK, false, MIX, PatFossen>(p, e0, act, obs, rew, done, reason);
    if (c1 == ENV_TAIL) band_tail<TRACK, false, MIX, PatFossen>(p, e1, act, obs, rew, done, reason);
    UUV_TL(TL_STEP_END);
}

// Kernel parameters of the band kernel: the step's block plus the fp64 base
// vehicles, so every vehicle coefficient is a constant-bank operand
struct BandP {
    EngineP<float> p;
    VehP<double> veh[MAX_VEH];
};


// Band kernel, launched on a side stream CONCURRENTLY with the step kernel
// (which skips these envs).  Block b owns chunk [b*band_per, (b+1)*band_per) of
// the batch (band_per <= BAND_MAX_PER): the chunk's flag bytes (EngineP::band_f)
// are read with 16-byte loads issued together with the generation counter --
// one memory round trip -- this step's candidates compacted into a
// shared-memory list, and each stepped in fp64 -- recompute, reward /
// termination / reset / observation -- beside the fp32 step instead of after
// it.  Statistics go to the band kernel's own per-block partial slots.
extern __shared__ __align__(16) int band_list[];

template <bool TRACK, bool DR, bool MIX, class Pat, bool REGE = false, bool REFOP = false>
__global__ void __launch_bounds__(BAND_BLOCK, BAND_MIN_BLOCKS)
k_band(const __grid_constant__ BandP bp, const void* __restrict__ act,
       void* __restrict__ obs, void* __restrict__ rew, uint8_t* __restrict__ done,
       int8_t* __restrict__ reason) {
    const EngineP<float>& p = bp.p;
    UUV_TL(TL_BAND_START);
    __shared__ uint32_t cnt;
    const unsigned lane = threadIdx.x & 31;
    const int cb = blockIdx.x * p.band_per;
    const int cend = min(cb + p.band_per, p.n_env);
    // the chunk's claim on the band counter (thread 0: fetch-add, the value
    // before it gives the generation) and every flag byte of the chunk, all in
    // flight at once
    __shared__ uint32_t s_gen;
    unsigned long long ctr = 0;
    if (threadIdx.x == 0) ctr = atomicAdd(p.band_ctr + 1, (unsigned long long)max(cend - cb, 0));
    uint4 q[BAND_VEC];
#pragma unroll
    for (int k = 0; k < BAND_VEC; ++k) {
        const int i = cb + 16 * (threadIdx.x + k * BAND_BLOCK);
        if (i + 15 < cend) {
            q[k] = *reinterpret_cast<const uint4*>(p.band_f + i);
        } else {
            uint32_t w[4] = {0u, 0u, 0u, 0u};
            for (int j = 0; j < 16 && i + j < cend; ++j) w[j >> 2] |= (uint32_t)p.band_f[i + j] << (8 * (j & 3));
            q[k] = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
    if (threadIdx.x == 0) {
        cnt = 0;
        s_gen = band_gen(p, ctr);
    }
    __syncthreads();
    // this step's generation: envs the step kernel has already stepped carry the
    // next one, candidates (never touched by it) this one with the flag bit set;
    // padding bytes past the chunk are 0 and never match (candidate bit clear)
    const uint32_t gen = s_gen;
    const uint32_t want = band_word(gen, true) * 0x01010101u;
    UUV_TLV(TL_BAND_GEN, (float)gen);
    StatAcc st;
    uint32_t mine[BAND_VEC];   // bit j of mine[k]: env cb + 16 (t + k BAND_BLOCK) + j is a candidate
    uint32_t c = 0;
#pragma unroll
    for (int k = 0; k < BAND_VEC; ++k) {
        const uint32_t w[4] = {q[k].x, q[k].y, q[k].z, q[k].w};
        mine[k] = 0;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            // bytes equal to want: zero bytes of w ^ want (exact per-byte test)
            const uint32_t x = w[h] ^ want;
            const uint32_t z = ~(((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x | 0x7f7f7f7fu);
            // z has bit 8b+7 set for each matching byte b
#pragma unroll
            for (int b = 0; b < 4; ++b) mine[k] |= ((z >> (8 * b + 7)) & 1u) << (4 * h + b);
        }
        c += __popc(mine[k]);
    }
    uint32_t incl = c;   // warp inclusive scan of the counts
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (unsigned)o) incl += v;
    }
    uint32_t at = 0;
    if (lane == 31 && incl) at = atomicAdd(&cnt, incl);
    at = __shfl_sync(0xffffffffu, at, 31) + incl - c;
#pragma unroll
    for (int k = 0; k < BAND_VEC; ++k) {
        uint32_t m = mine[k];
        while (m) {
            const int j = __ffs(m) - 1;
            m &= m - 1;
            UUV_CHECK(at < (uint32_t)p.band_per);
            UUV_CHECK(cb + 16 * (threadIdx.x + k * BAND_BLOCK) + j < cend);
            band_list[at++] = cb + 16 * (threadIdx.x + k * BAND_BLOCK) + j;
        }
    }
    __syncthreads();
    const uint32_t n = cnt;
    UUV_TL(TL_BAND_SCAN);
    UUV_CHECK(n <= (uint32_t)p.band_per && p.band_per <= BAND_MAX_PER);
    for (uint32_t i = threadIdx.x; i < n; i += BAND_BLOCK)
        band_env<TRACK, DR, MIX, Pat, REGE, REFOP>(p, bp.veh[0], bp.veh[1], band_list[i], gen, act,
                                                   obs, rew, done, reason, st);
    if (p.stats_on) block_stats<BAND_BLOCK>(p.stats, st);
    UUV_TL(TL_BAND_END);
}

// band flags from the current states (after create / reset_all / set_states /
// restore): generation = the band kernels' current one
__device__ __forceinline__ void write_band_flag(const EngineP<float>& p, int e, const float s[12]) {
    if (p.band_f)
        p.band_f[e] = (uint8_t)band_word(band_gen(p, p.band_ctr[0]), band_cand(p, s));
}
template <class T> __device__ __forceinline__ void write_band_flag(const EngineP<T>&, int, const T*) {}

template <class T>
__global__ void __launch_bounds__(BLOCK) k_band_flags(const __grid_constant__ EngineP<T> p) {
    const int e = blockIdx.x * BLOCK + threadIdx.x;
    if (e >= p.n_env) return;
    const V4<T> a0 = p.s0[e], a1 = p.s1[e], a2 = p.s2[e];
    const T s[12] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w, a2.x, a2.y, a2.z, a2.w};
    write_band_flag(p, e, s);
}

// observation of the current state at the current step (reset / inspection)
template <class T, class IO>
__device__ __forceinline__ void observe_env(const EngineP<T>& p, int e, const T s[12],
                                            int32_t step, IO* __restrict__ obs) {
    const TaskP<T>& tk = p.task;
    IO* row = obs + (size_t)e * tk.obs_dim;
    if (tk.kind == 0) {
        row[0] = (IO)(tk.target[0] - s[0]);
        row[1] = (IO)(tk.target[1] - s[1]);
        row[2] = (IO)(tk.target[2] - s[2]);
        row[3] = (IO)obs_wrap<T>(tk.target[3] - s[3]);
        row[4] = (IO)obs_wrap<T>(tk.target[4] - s[4]);
        row[5] = (IO)obs_wrap<T>(tk.target[5] - s[5]);
        for (int i = 6; i < 12; ++i) row[i] = (IO)s[i];
    } else {
        const int tab_last = tk.episode_len + tk.lookahead;
        int n = 0;
        for (int k = 1; k <= tk.lookahead; ++k) {
            const V4<T> r = tk.traj[min(max(step + k, 0), tab_last)];
            row[n++] = (IO)(r.x - s[0]);
            row[n++] = (IO)(r.y - s[1]);
            row[n++] = (IO)(r.z - s[2]);
            row[n++] = (IO)obs_wrap<T>(T(0) - s[3]);
            row[n++] = (IO)obs_wrap<T>(T(0) - s[4]);
            row[n++] = (IO)obs_wrap<T>(r.w - s[5]);
        }
        for (int i = 6; i < 12; ++i) row[n++] = (IO)s[i];
    }
}

template <class T, class IO>
__global__ void __launch_bounds__(BLOCK) k_reset(const __grid_constant__ EngineP<T> p,
                                                 IO* __restrict__ obs) {
    const int e = blockIdx.x * BLOCK + threadIdx.x;
    if (e >= p.n_env) return;
    const uint64_t g = p.env_offset + (uint64_t)e;
    if (e == 0) *p.seed_dev = p.seed;
    // reset_all rewinds the reset stream (batch.py:80-83)
    const State12<T> rs = reset_state<T>(p.task, p.seed, g, 0);
    const T* s = rs.v;
    p.reset_ctr[e] = 6;
    p.step[e] = 0;
    p.ep_ret[e] = 0.0f;
    p.s0[e] = V4<T>{s[0], s[1], s[2], s[3]};
    p.s1[e] = V4<T>{s[4], s[5], s[6], s[7]};
    p.s2[e] = V4<T>{s[8], s[9], s[10], s[11]};
    write_band_flag(p, e, s);
    if (obs) observe_env<T, IO>(p, e, s, 0, obs);
}

template <class T, class IO>
__global__ void __launch_bounds__(BLOCK) k_observe(const __grid_constant__ EngineP<T> p,
                                                   IO* __restrict__ obs) {
    const int e = blockIdx.x * BLOCK + threadIdx.x;
    if (e >= p.n_env) return;
    const V4<T> a0 = p.s0[e], a1 = p.s1[e], a2 = p.s2[e];
    const T s[12] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w, a2.x, a2.y, a2.z, a2.w};
    observe_env<T, IO>(p, e, s, p.step[e], obs);
}

template <class T>
__global__ void __launch_bounds__(BLOCK) k_dr_init(const __grid_constant__ EngineP<T> p,
                                                   int* __restrict__ first_bad) {
    const int e = blockIdx.x * BLOCK + threadIdx.x;
    if (e >= p.n_env) return;
    const uint64_t g = p.env_offset + (uint64_t)e;
    const bool slot1 = p.n_veh > 1 && (int64_t)g >= p.mix_bound0;
    uint64_t ctr = 0;
    V4<T> d0, d1;
    V2<T> d2;
    // create-time draw: full 6x6 fp64 check (PatDense) for the error report
    V2<double>* rec = p.dr64 ? p.dr64 + (size_t)e * 5 : nullptr;
    const bool ok = slot1 ? dr_draw<T, PatDense>(p.veh[1], p.ranges, p.seed, g, ctr, d0, d1, d2, rec)
                          : dr_draw<T, PatDense>(p.veh[0], p.ranges, p.seed, g, ctr, d0, d1, d2, rec);
    p.dr0[e] = d0; p.dr1[e] = d1; p.dr2[e] = d2;
    p.param_ctr[e] = ctr;
    if (!ok) atomicMin(first_bad, e);
}

// PD baseline law over the state slab (reference baseline.py:38-75; restated in
// paper_2410_14117_b200/baseline.py) -- one thread per env.
// UuvPdGains in the engine precision (converted on the host per launch)
template <class T> struct PdGainsT {
    T kp[6], kd[6];
    T pinv[2][8][6];
    T kmax[2][8];
    int32_t quadratic[2][8];
};

template <class T>
__global__ void k_pd_actions(const __grid_constant__ EngineP<T> p,
                             const __grid_constant__ PdGainsT<T> g, const T* __restrict__ ref,
                             T* __restrict__ act) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= p.n_env) return;
    const int slot = (p.n_veh > 1 && (int64_t)(p.env_offset + (uint64_t)e) >= p.mix_bound0) ? 1 : 0;
    const V4<T> a0 = p.s0[e], a1 = p.s1[e], a2 = p.s2[e];
    const T s[12] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w, a2.x, a2.y, a2.z, a2.w};
    T sphi, cphi, sth, cth, spsi, cpsi;
    if constexpr (is_f64<T>()) {
        sincos(s[3], &sphi, &cphi); sincos(s[4], &sth, &cth); sincos(s[5], &spsi, &cpsi);
    } else {
        sincosf(s[3], &sphi, &cphi); sincosf(s[4], &sth, &cth); sincosf(s[5], &spsi, &cpsi);
    }
    const T R[3][3] = {
        {cpsi * cth, -spsi * cphi + cpsi * sth * sphi, spsi * sphi + cpsi * cphi * sth},
        {spsi * cth, cpsi * cphi + sphi * sth * spsi, -cpsi * sphi + sth * spsi * cphi},
        {-sth, cth * sphi, cth * cphi}};
    const T ew[3] = {ref[0] - s[0], ref[1] - s[1], ref[2] - s[2]};
    T w[6];
#pragma unroll
    for (int j = 0; j < 3; ++j) {   // R^T ew
        const T eb = R[0][j] * ew[0] + R[1][j] * ew[1] + R[2][j] * ew[2];
        w[j] = g.kp[j] * eb - g.kd[j] * s[6 + j];
    }
    const T TWO_PI = Consts<T>::TWO_PI, PI = Consts<T>::PI;
#pragma unroll
    for (int j = 0; j < 3; ++j) {   // (a + pi) mod 2 pi - pi with floor-mod (Python %)
        const T x = ref[3 + j] - s[3 + j] + PI;
        const T ea = x - TWO_PI * floor(x / TWO_PI) - PI;
        w[3 + j] = g.kp[3 + j] * ea - g.kd[3 + j] * s[9 + j];
    }
    const int nthr = p.veh[slot].n_thr;
    T* out = act + (size_t)e * p.act_dim;
    for (int i = 0; i < p.act_dim; ++i) {
        T t = T(0);
        if (i < nthr) {
            T f = T(0);
#pragma unroll
            for (int j = 0; j < 6; ++j) f += g.pinv[slot][i][j] * w[j];
            const T km = g.kmax[slot][i];
            t = g.quadratic[slot][i] ? copysign(sqrt(fabs(f) / km), f) : f / km;
            t = t > T(1) ? T(1) : (t < T(-1) ? T(-1) : t);
        }
        out[i] = t;
    }
}

template <class T, class O = double>
__global__ void k_pack_states(const __grid_constant__ EngineP<T> p, O* __restrict__ out) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= p.n_env) return;
    const V4<T> a0 = p.s0[e], a1 = p.s1[e], a2 = p.s2[e];
    O* r = out + (size_t)e * 12;
    r[0] = a0.x; r[1] = a0.y; r[2] = a0.z; r[3] = a0.w;
    r[4] = a1.x; r[5] = a1.y; r[6] = a1.z; r[7] = a1.w;
    r[8] = a2.x; r[9] = a2.y; r[10] = a2.z; r[11] = a2.w;
}

template <class T>
__global__ void k_unpack_states(const __grid_constant__ EngineP<T> p,
                                const double* __restrict__ in) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= p.n_env) return;
    const double* r = in + (size_t)e * 12;
    const T s[12] = {(T)r[0], (T)r[1], (T)r[2], (T)r[3], (T)r[4], (T)r[5],
                     (T)r[6], (T)r[7], (T)r[8], (T)r[9], (T)r[10], (T)r[11]};
    p.s0[e] = V4<T>{s[0], s[1], s[2], s[3]};
    p.s1[e] = V4<T>{s[4], s[5], s[6], s[7]};
    p.s2[e] = V4<T>{s[8], s[9], s[10], s[11]};
    write_band_flag(p, e, s);
}

// Body wrench of every env for f64 action rows [N][A] (thrusters.py:97-119,
// inspection / parity): the step kernel's own wrench() with the env's
// randomised thrust factor -> out [N][6] f64
template <class T, bool DR>
__global__ void k_wrench(const __grid_constant__ EngineP<T> p, const double* __restrict__ act,
                         double* __restrict__ out) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= p.n_env) return;
    const bool slot1 = p.n_veh > 1 && (int64_t)(p.env_offset + (uint64_t)e) >= p.mix_bound0;
    EnvParams<T, DR> E;
    if constexpr (DR) E.f_thrust = p.dr1[e].x;
    T tau[6];
    const double* row = act + (size_t)e * p.act_dim;
    if (slot1) wrench<T, DR, DR>(p.veh[1], E, row, true, tau);
    else wrench<T, DR, DR>(p.veh[0], E, row, true, tau);
#pragma unroll
    for (int i = 0; i < 6; ++i) out[(size_t)e * 6 + i] = (double)tau[i];
}

template <class T>
__global__ void k_pack_dr(const __grid_constant__ EngineP<T> p, double* __restrict__ out) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= p.n_env) return;
    const V4<T> d0 = p.dr0[e], d1 = p.dr1[e];
    const V2<T> d2 = p.dr2[e];
    double* r = out + (size_t)e * 10;
    r[0] = d0.x; r[1] = d0.y; r[2] = d0.z; r[3] = d0.w;
    r[4] = d1.x; r[5] = d1.y; r[6] = d1.z; r[7] = d1.w;
    r[8] = d2.x; r[9] = d2.y;
}

// ------------------------------------------------------------------ TMA-pipelined paired step
// Persistent variant of k_step_pair for station tasks on the device face: one
// elected thread streams the NEXT tile's state planes and action rows into the
// other half of a two-stage shared-memory ring with 1D bulk copies
// (cp.async.bulk ... mbarrier::complete_tx), while the whole block computes the
// current tile -- the HBM traffic of tile i+1 overlaps the sub-steps of tile i
// instead of every co-resident block loading / computing / storing in lockstep.
__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
    return (uint32_t)__cvta_generic_to_shared(ptr);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred P;\n"
        "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        " @!P bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

template <bool MIX>
__global__ void __launch_bounds__(BLOCK, TMA_MIN_BLOCKS)
k_step_pair_tma(const __grid_constant__ EngineP<float> p, const void* __restrict__ act,
                void* __restrict__ obs, void* __restrict__ rew, uint8_t* __restrict__ done,
                int8_t* __restrict__ reason) {
    BandGen bgl;   // persistent kernel: per-thread counter loads, counted at its end
    if (p.band_f) bgl.mode = BG_LOAD;
    constexpr int TILE = 2 * BLOCK;
    __shared__ __align__(8) uint64_t mbar[2];
    const int A = p.act_dim;
    const uint32_t plane_bytes = TILE * 16;
    const uint32_t act_bytes = UUV_TMA_ACT ? (uint32_t)(TILE * A * 4) : 0u;
    const uint32_t stage_bytes = 3 * plane_bytes + act_bytes;   // multiple of 16
    const int n_full = p.n_env / TILE;
    const float* actf = (const float*)act;
    if (threadIdx.x == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int tile, int stage) {
        unsigned char* dst = uuv_smem + (size_t)stage * stage_bytes;
        const size_t base = (size_t)tile * TILE;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&mbar[stage], stage_bytes);
        bulk_g2s(dst, p.s0 + base, plane_bytes, &mbar[stage]);
        bulk_g2s(dst + plane_bytes, p.s1 + base, plane_bytes, &mbar[stage]);
        bulk_g2s(dst + 2 * plane_bytes, p.s2 + base, plane_bytes, &mbar[stage]);
        if (UUV_TMA_ACT) bulk_g2s(dst + 3 * plane_bytes, actf + base * A, act_bytes, &mbar[stage]);
    };
    StatAcc st;
    int stage = 0;
    uint32_t parity0 = 0, parity1 = 0;
    int t = blockIdx.x;
    if (threadIdx.x == 0 && t < n_full) issue(t, 0);
    for (; t < n_full; t += gridDim.x) {
        const int nxt = t + gridDim.x;
        if (threadIdx.x == 0 && nxt < n_full) issue(nxt, stage ^ 1);   // prefetch
        const int e0 = t * TILE + threadIdx.x, e1 = e0 + BLOCK;
        EnvIn<float, false> in0, in1;
        in0.step = p.step[e0]; in1.step = p.step[e1];
        if (p.band_f) {
            in0.bf = p.band_f[e0];
            in1.bf = p.band_f[e1];
        }
        in0.ep_ret = p.ep_ret[e0]; in1.ep_ret = p.ep_ret[e1];
        mbar_wait(&mbar[stage], stage ? parity1 : parity0);
        if (stage) parity1 ^= 1; else parity0 ^= 1;
        const unsigned char* src = uuv_smem + (size_t)stage * stage_bytes;
        const float4* q0 = (const float4*)src;
        const float4* q1 = (const float4*)(src + plane_bytes);
        const float4* q2 = (const float4*)(src + 2 * plane_bytes);
        const float* qa = (const float*)(src + 3 * plane_bytes);
        auto unpack = [&](int li, EnvIn<float, false>& in) {
            const float4 a0 = q0[li], a1 = q1[li], a2 = q2[li];
            in.s[0] = a0.x; in.s[1] = a0.y; in.s[2] = a0.z; in.s[3] = a0.w;
            in.s[4] = a1.x; in.s[5] = a1.y; in.s[6] = a1.z; in.s[7] = a1.w;
            in.s[8] = a2.x; in.s[9] = a2.y; in.s[10] = a2.z; in.s[11] = a2.w;
        };
        unpack(threadIdx.x, in0);
        unpack(threadIdx.x + BLOCK, in1);
        const int sl0 = MIX && (int64_t)(p.env_offset + (uint64_t)e0) >= p.mix_bound0;
        const int sl1 = MIX && (int64_t)(p.env_offset + (uint64_t)e1) >= p.mix_bound0;
        const float* r0 = UUV_TMA_ACT ? qa + (size_t)threadIdx.x * A : actf + (size_t)e0 * A;
        const float* r1 = UUV_TMA_ACT ? qa + (size_t)(threadIdx.x + BLOCK) * A : actf + (size_t)e1 * A;
        int c0 = ENV_DONE, c1 = ENV_DONE;
        if (sl0 == sl1) {
            int c = ENV_DONE;
            if (sl0 == 0)
                c = pair_core<false, 0>(p, e0, e1, -1, -1, in0, in1, r0, r1, false, obs, rew, done,
                                        reason, st, bgl);
            else if constexpr (MIX)
                c = pair_core<false, 1>(p, e0, e1, -1, -1, in0, in1, r0, r1, false, obs, rew, done,
                                        reason, st, bgl);
            c0 = c & 3;
            c1 = c >> 2;
        } else {   // vehicle-slab boundary inside the pair: one env at a time
            if constexpr (MIX) {
                c0 = one_env<float, false, false, MIX, PatFossen>(p, e0, -1, act, obs, rew, done,
                                                                  reason, st, bgl);
                c1 = one_env<float, false, false, MIX, PatFossen>(p, e1, -1, act, obs, rew, done,
                                                                  reason, st, bgl);
            }
        }
        if (c0 == ENV_TAIL) band_tail<false, false, MIX, PatFossen>(p, e0, act, obs, rew, done, reason);
        if (c1 == ENV_TAIL) band_tail<false, false, MIX, PatFossen>(p, e1, act, obs, rew, done, reason);
        __syncthreads();   // this stage is consumed before it is refilled
        stage ^= 1;
    }
    // partial tail tile: the block whose turn it is, with plain loads
    const int tail0 = n_full * TILE;
    if (tail0 < p.n_env && blockIdx.x == n_full % gridDim.x) {
        const int e0 = tail0 + threadIdx.x, e1 = e0 + BLOCK;
        const int c0 = e0 < p.n_env ? one_env<float, false, false, MIX, PatFossen>(
                                          p, e0, -1, act, obs, rew, done, reason, st, bgl) : ENV_DONE;
        const int c1 = e1 < p.n_env ? one_env<float, false, false, MIX, PatFossen>(
                                          p, e1, -1, act, obs, rew, done, reason, st, bgl) : ENV_DONE;
        if (c0 == ENV_TAIL) band_tail<false, false, MIX, PatFossen>(p, e0, act, obs, rew, done, reason);
        if (c1 == ENV_TAIL) band_tail<false, false, MIX, PatFossen>(p, e1, act, obs, rew, done, reason);
    }
    if (p.stats_on) block_stats(p.stats, st);
    {   // envs this block stepped: its full tiles (+ the partial tail tile)
        int cnt = 0;
        for (int t2 = blockIdx.x; t2 < n_full; t2 += gridDim.x) cnt += TILE;
        if (tail0 < p.n_env && blockIdx.x == n_full % gridDim.x) cnt += p.n_env - tail0;
        band_count(p, 0, cnt);
    }
}

// ------------------------------------------------------------------ launchers
// opt-in above 48 KB (paired rows in f64: 73.7 KB) once per kernel variant and
// device: function attributes are per device context, and one process may drive
// engines on several GPUs
template <auto KERNEL>
static void allow_smem() {
    static std::atomic<uint64_t> done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return;
    cudaFuncSetAttribute(KERNEL, cudaFuncAttributeMaxDynamicSharedMemorySize, MAX_STAGE_BYTES);
    done.fetch_or(bit, std::memory_order_release);
}

template <class T>
static cudaError_t launch_step_main(const EngineP<T>& p, bool track, bool dr, bool fossen, bool pair,
                                    const void* act, void* obs, void* rew, uint8_t* done,
                                    int8_t* reason, cudaStream_t st) {
    const bool mix = p.n_veh > 1;
    const size_t esz = p.io_f64 ? 8 : sizeof(T);
    if constexpr (std::is_same<T, float>::value) {
        if (pair && fossen && !dr && !track && !p.io_f64 && !p.stage_obs && p.persist_blocks > 0) {
            const int n_full = p.n_env / (2 * BLOCK);
            const dim3 grid(std::max(1, std::min(n_full, p.persist_blocks)));
            const size_t smem = (size_t)2 * (3 * 2 * BLOCK * 16 + (UUV_TMA_ACT ? 2 * BLOCK * p.act_dim * 4 : 0));
#define UUV_T(M)                                                                        \
    do {                                                                                \
        allow_smem<k_step_pair_tma<M>>();                                               \
        k_step_pair_tma<M><<<grid, BLOCK, smem, st>>>(p, act, obs, rew, done, reason);  \
    } while (0)
            if (mix) UUV_T(true); else UUV_T(false);
#undef UUV_T
            return cudaGetLastError();
        }
        if (pair && fossen && !dr) {
            const dim3 grid((p.n_env + 2 * BLOCK - 1) / (2 * BLOCK));
            const size_t smem = (p.stage_obs ? (size_t)2 * BLOCK * p.task.obs_dim * esz : 0) +
                                (p.stage_act ? (size_t)2 * BLOCK * p.act_dim * 8 : 0);
#define UUV_P(TR, M)                                                                   \
    do {                                                                               \
        allow_smem<k_step_pair<TR, M>>();                                              \
        const cudaError_t le = launch_k(k_step_pair<TR, M>, grid, dim3(BLOCK), smem, st, \
                                        p.pdl != 0, p, act, obs, rew, done, reason); \
        if (le != cudaSuccess) return le;                                              \
    } while (0)
            if (track) { if (mix) UUV_P(true, true); else UUV_P(true, false); }
            else { if (mix) UUV_P(false, true); else UUV_P(false, false); }
#undef UUV_P
            return cudaGetLastError();
        }
    }
    const dim3 grid((p.n_env + BLOCK - 1) / BLOCK);
    const size_t smem = (p.stage_obs ? (size_t)BLOCK * p.task.obs_dim * esz : 0) +
                        (p.stage_act ? (size_t)BLOCK * p.act_dim * 8 : 0);
#define UUV_L(TR, D, M, PAT)                                                                 \
    do {                                                                                     \
        allow_smem<k_step<T, TR, D, M, PAT>>();                                              \
        const cudaError_t le = launch_k(k_step<T, TR, D, M, PAT>, grid, dim3(BLOCK), smem, st, \
                                        p.pdl != 0, p, act, obs, rew, done, reason); \
        if (le != cudaSuccess) return le;                                                    \
    } while (0)
#define UUV_LP(TR, D, M) \
    if (fossen) UUV_L(TR, D, M, PatFossen); else UUV_L(TR, D, M, PatDense)
    if (track) {
        if (dr) { if (mix) UUV_LP(true, true, true); else UUV_LP(true, true, false); }
        else { if (mix) UUV_LP(true, false, true); else UUV_LP(true, false, false); }
    } else {
        if (dr) { if (mix) UUV_LP(false, true, true); else UUV_LP(false, true, false); }
        else { if (mix) UUV_LP(false, false, true); else UUV_LP(false, false, false); }
    }
#undef UUV_LP
#undef UUV_L
    return cudaGetLastError();
}

template <auto KERNEL>
static void allow_band_smem() {   // chunk lists beyond 48 KB (band_per up to 16,384 envs)
    static std::atomic<uint64_t> done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return;
    cudaFuncSetAttribute(KERNEL, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 * 4);
    done.fetch_or(bit, std::memory_order_release);
}

// The band kernel on the engine's side stream, forked from and joined back to
// the launching stream around the step kernel (fp32 engines with band64): it
// runs the band candidates in fp64 while the step kernel runs everything else.
// Stream-capturable (the fork / join become graph edges).
// The band kernel's launch; REFOP instantiations live in k_band.cu (compiled with
// -fmad=false, so the reference-order path rounds like the reference), the FMA
// formulation's in k_f32.cu (contraction on: the -fmad=false build of it measured
// C2 +0.6 us, C3 +1.9 us).
template <bool RF>
static cudaError_t launch_band_impl(const EngineP<float>& p, bool track, bool dr, bool fossen,
                                    const void* act, void* obs, void* rew, uint8_t* done,
                                    int8_t* reason, cudaStream_t side) {
    thread_local BandP bq;   // host staging of the launch parameters (copied at launch)
    EngineP<float>& q = bq.p;
    q = p;
    for (int v = 0; v < MAX_VEH; ++v) bq.veh[v] = p.veh64[v];
    q.stage_obs = 0;
    q.stage_act = 0;
    q.stagger_ns = 0;
    q.pdl = 0;
    q.persist_blocks = 0;
    q.stats = p.stats_band;
    const bool mix = p.n_veh > 1;
    const dim3 grid(std::max(1, p.band_grid));
    const size_t smem = (size_t)p.band_per * sizeof(int);   // candidate list for a whole chunk
#define UUV_B(TR, D, M, PAT, RG)                                                      \
    do {                                                                              \
        allow_band_smem<k_band<TR, D, M, PAT, RG, RF>>();                             \
        k_band<TR, D, M, PAT, RG, RF><<<grid, BAND_BLOCK, smem, side>>>(bq, act, obs, rew, done, reason); \
    } while (0)
#define UUV_BP(TR, D, M)                                                                \
    if (fossen && !D && p.band_rege) UUV_B(TR, false, M, PatFossen, true);              \
    else if (fossen) UUV_B(TR, D, M, PatFossen, false);                                 \
    else UUV_B(TR, D, M, PatDense, false)
    if (track) {
        if (dr) { if (mix) UUV_BP(true, true, true); else UUV_BP(true, true, false); }
        else { if (mix) UUV_BP(true, false, true); else UUV_BP(true, false, false); }
    } else {
        if (dr) { if (mix) UUV_BP(false, true, true); else UUV_BP(false, true, false); }
        else { if (mix) UUV_BP(false, false, true); else UUV_BP(false, false, false); }
    }
#undef UUV_BP
#undef UUV_B
    return cudaGetLastError();
}

cudaError_t launch_band(const EngineP<float>& p, bool track, bool dr, bool fossen,
                        const void* act, void* obs, void* rew, uint8_t* done,
                        int8_t* reason, cudaStream_t side);
cudaError_t launch_band_refop(const EngineP<float>& p, bool track, bool dr, bool fossen,
                              const void* act, void* obs, void* rew, uint8_t* done,
                              int8_t* reason, cudaStream_t side);
#if defined(UUV_F32_TU)
cudaError_t launch_band(const EngineP<float>& p, bool track, bool dr, bool fossen,
                        const void* act, void* obs, void* rew, uint8_t* done,
                        int8_t* reason, cudaStream_t side) {
    if (p.band_refop) return launch_band_refop(p, track, dr, fossen, act, obs, rew, done, reason, side);
    return launch_band_impl<false>(p, track, dr, fossen, act, obs, rew, done, reason, side);
}
#elif defined(UUV_BAND_TU)
cudaError_t launch_band_refop(const EngineP<float>& p, bool track, bool dr, bool fossen,
                              const void* act, void* obs, void* rew, uint8_t* done,
                              int8_t* reason, cudaStream_t side) {
    return launch_band_impl<true>(p, track, dr, fossen, act, obs, rew, done, reason, side);
}
#endif

template <class T>
cudaError_t Launch<T>::step(const EngineP<T>& p, bool track, bool dr, bool fossen, bool pair,
                            const void* act, void* obs, void* rew, uint8_t* done,
                            int8_t* reason, cudaStream_t st) {
    if constexpr (std::is_same<T, float>::value) {
        if (p.band_same && p.band_theta < INFINITY) {
            cudaError_t e = launch_step_main<T>(p, track, dr, fossen, pair, act, obs, rew, done, reason, st);
            if (e == cudaSuccess) e = launch_band(p, track, dr, fossen, act, obs, rew, done, reason, st);
            return e;
        }
        if (p.band_side && p.band_theta < INFINITY) {
            cudaStream_t side = (cudaStream_t)p.band_side;
            cudaEvent_t fork = (cudaEvent_t)p.band_ev[0], join = (cudaEvent_t)p.band_ev[1];
            // launch order: the second kernel starts ~1 us after the first.  Small
            // batches launch the band kernel first -- its latency-bound fp64
            // chains are the step's critical path; larger ones the step kernel
            // (EngineP::band_main_first), whose waves are then the critical path
            // and the band kernel's blocks fit around them
            cudaError_t e = cudaEventRecord(fork, st);
            if (e == cudaSuccess && p.band_main_first)
                e = launch_step_main<T>(p, track, dr, fossen, pair, act, obs, rew, done, reason, st);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(side, fork, 0);
            if (e == cudaSuccess) e = launch_band(p, track, dr, fossen, act, obs, rew, done, reason, side);
            if (e == cudaSuccess) e = cudaEventRecord(join, side);
            if (e == cudaSuccess && !p.band_main_first)
                e = launch_step_main<T>(p, track, dr, fossen, pair, act, obs, rew, done, reason, st);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(st, join, 0);
            return e;
        }
    }
    return launch_step_main<T>(p, track, dr, fossen, pair, act, obs, rew, done, reason, st);
}

template <class T>
cudaError_t Launch<T>::reset(const EngineP<T>& p, T* obs, cudaStream_t st) {
    k_reset<T, T><<<(p.n_env + BLOCK - 1) / BLOCK, BLOCK, 0, st>>>(p, obs);
    return cudaGetLastError();
}

template <class T>
cudaError_t Launch<T>::observe(const EngineP<T>& p, T* obs, cudaStream_t st) {
    k_observe<T, T><<<(p.n_env + BLOCK - 1) / BLOCK, BLOCK, 0, st>>>(p, obs);
    return cudaGetLastError();
}

template <class T>
cudaError_t Launch<T>::dr_init(const EngineP<T>& p, int* first_bad, cudaStream_t st) {
    k_dr_init<T><<<(p.n_env + BLOCK - 1) / BLOCK, BLOCK, 0, st>>>(p, first_bad);
    return cudaGetLastError();
}

template <class T>
cudaError_t Launch<T>::pack_states(const EngineP<T>& p, double* out, cudaStream_t st) {
    k_pack_states<T, double><<<(p.n_env + 255) / 256, 256, 0, st>>>(p, out);
    return cudaGetLastError();
}

template <class T>
cudaError_t Launch<T>::pd_actions(const EngineP<T>& p, const UuvPdGains& g, const T* ref, T* act,
                                  cudaStream_t st) {
    PdGainsT<T> gt;
    for (int j = 0; j < 6; ++j) {
        gt.kp[j] = (T)g.kp[j];
        gt.kd[j] = (T)g.kd[j];
    }
    for (int v = 0; v < 2; ++v)
        for (int i = 0; i < 8; ++i) {
            for (int j = 0; j < 6; ++j) gt.pinv[v][i][j] = (T)g.pinv[v][i][j];
            gt.kmax[v][i] = (T)g.kmax[v][i];
            gt.quadratic[v][i] = g.quadratic[v][i];
        }
    k_pd_actions<T><<<(p.n_env + 255) / 256, 256, 0, st>>>(p, gt, ref, act);
    return cudaGetLastError();
}

template <class T>
cudaError_t Launch<T>::pack_states_t(const EngineP<T>& p, T* out, cudaStream_t st) {
    k_pack_states<T, T><<<(p.n_env + 255) / 256, 256, 0, st>>>(p, out);
    return cudaGetLastError();
}

template <class T>
cudaError_t Launch<T>::unpack_states(const EngineP<T>& p, const double* in, cudaStream_t st) {
    k_unpack_states<T><<<(p.n_env + 255) / 256, 256, 0, st>>>(p, in);
    return cudaGetLastError();
}

template <class T>
cudaError_t Launch<T>::wrench(const EngineP<T>& p, bool dr, const double* act, double* out,
                              cudaStream_t st) {
    if (dr) k_wrench<T, true><<<(p.n_env + 255) / 256, 256, 0, st>>>(p, act, out);
    else k_wrench<T, false><<<(p.n_env + 255) / 256, 256, 0, st>>>(p, act, out);
    return cudaGetLastError();
}

template <class T>
cudaError_t Launch<T>::band_flags(const EngineP<T>& p, cudaStream_t st) {
    k_band_flags<T><<<(p.n_env + BLOCK - 1) / BLOCK, BLOCK, 0, st>>>(p);
    return cudaGetLastError();
}

template <class T>
cudaError_t Launch<T>::pack_dr(const EngineP<T>& p, double* out, cudaStream_t st) {
    k_pack_dr<T><<<(p.n_env + 255) / 256, 256, 0, st>>>(p, out);
    return cudaGetLastError();
}

template <class T>
cudaError_t Launch<T>::step_attrs(cudaFuncAttributes* a, bool track, bool dr, bool fossen,
                                  bool mix, bool pair, bool tma) {
    if constexpr (std::is_same<T, float>::value) {
        if (pair && fossen && !dr && !track && tma)
            return mix ? cudaFuncGetAttributes(a, k_step_pair_tma<true>)
                       : cudaFuncGetAttributes(a, k_step_pair_tma<false>);
        if (pair && fossen && !dr) {
            if (track) return mix ? cudaFuncGetAttributes(a, k_step_pair<true, true>)
                                  : cudaFuncGetAttributes(a, k_step_pair<true, false>);
            return mix ? cudaFuncGetAttributes(a, k_step_pair<false, true>)
                       : cudaFuncGetAttributes(a, k_step_pair<false, false>);
        }
    }
#define UUV_A(TR, D, M, PAT) return cudaFuncGetAttributes(a, k_step<T, TR, D, M, PAT>)
#define UUV_AP(TR, D, M) \
    if (fossen) UUV_A(TR, D, M, PatFossen); else UUV_A(TR, D, M, PatDense)
    if (track) {
        if (dr) { if (mix) UUV_AP(true, true, true); else UUV_AP(true, true, false); }
        else { if (mix) UUV_AP(true, false, true); else UUV_AP(true, false, false); }
    } else {
        if (dr) { if (mix) UUV_AP(false, true, true); else UUV_AP(false, true, false); }
        else { if (mix) UUV_AP(false, false, true); else UUV_AP(false, false, false); }
    }
#undef UUV_AP
#undef UUV_A
}

template <class A, class B>
__global__ void k_convert(const A* __restrict__ in, B* __restrict__ out, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        out[i] = (B)in[i];
}

template <class T>
cudaError_t Launch<T>::to_f64(const T* in, double* out, size_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const int blocks = (int)std::min<size_t>((n + 255) / 256, 148 * 16);
    k_convert<T, double><<<blocks, 256, 0, st>>>(in, out, n);
    return cudaGetLastError();
}

template <class T>
cudaError_t Launch<T>::from_f64(const double* in, T* out, size_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const int blocks = (int)std::min<size_t>((n + 255) / 256, 148 * 16);
    k_convert<double, T><<<blocks, 256, 0, st>>>(in, out, n);
    return cudaGetLastError();
}

}  // namespace uuv

#define UUV_INSTANTIATE(T) template struct uuv::Launch<T>;

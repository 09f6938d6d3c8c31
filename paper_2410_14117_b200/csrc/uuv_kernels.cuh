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

#include <algorithm>

#include "uuv_model.cuh"
#include "launch.h"

namespace uuv {


template <class T, bool TRACK, bool DR, int SLOT, class Pat>
__device__ __forceinline__ void step_env(const EngineP<T>& p, int e, uint64_t g,
                                         const T* __restrict__ act, T* __restrict__ obs,
                                         T* __restrict__ rew, uint8_t* __restrict__ done,
                                         int8_t* __restrict__ reason, float& st_rew,
                                         int& st_reason, float& st_epret, int& st_eplen,
                                         int& st_err) {
    const VehP<T>& V = p.veh[SLOT];
    const TaskP<T>& tk = p.task;
    const V4<T> a0 = p.s0[e], a1 = p.s1[e], a2 = p.s2[e];
    T s[12] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w, a2.x, a2.y, a2.z, a2.w};
    const int32_t step = p.step[e];

    EnvParams<T, DR> E;
    if constexpr (DR) {
        const V4<T> d0 = p.dr0[e], d1 = p.dr1[e];
        const V2<T> d2 = p.dr2[e];
        build_env<T, Pat>(V, d0, d1, d2, E);
    }
    T tau[6];
    wrench<T, DR>(V, E, act + (size_t)e * p.act_dim, tau);

    bool failed = false;
    const T dt = tk.sub_dt;
#pragma unroll 2
    for (int k = 0; k < tk.n_substeps; ++k) {
        if (!substep<T, DR, Pat>(V, E, s, tau, dt)) {
            failed = true;
            break;
        }
    }
    // reward / termination (tasks.py:219-230): failure > divergence > truncation
    const int32_t ns = step + 1;
    const int tab_last = tk.episode_len + tk.lookahead;
    T rx, ry, rz;
    if constexpr (TRACK) {
        const V4<T> r = tk.traj[min(max(ns, 0), tab_last)];
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

    float er = p.ep_ret[e] + (float)reward;
    int32_t nstep = ns;
    if (rc >= 0) {
        st_epret = er;
        st_eplen = ns;
        er = 0.0f;
        const uint64_t seed = *p.seed_dev;
        if constexpr (DR) {
            if (p.ranges.per_episode) {   // engine.rs:553-558, batch.py:107-110
                uint64_t pc = p.param_ctr[e];
                V4<T> n0, n1;
                V2<T> n2;
                if (dr_draw<T>(V, p.ranges, seed, g, pc, n0, n1, n2)) {
                    p.dr0[e] = n0; p.dr1[e] = n1; p.dr2[e] = n2;
                } else {
                    st_err = 1;
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
    p.s0[e] = V4<T>{s[0], s[1], s[2], s[3]};
    p.s1[e] = V4<T>{s[4], s[5], s[6], s[7]};
    p.s2[e] = V4<T>{s[8], s[9], s[10], s[11]};

    // observation (post-reset for finished envs, batch.py:106-118)
    T* row = obs + (size_t)e * tk.obs_dim;
    if constexpr (!TRACK) {
        V4<T>* o4 = reinterpret_cast<V4<T>*>(row);
        o4[0] = V4<T>{tk.target[0] - s[0], tk.target[1] - s[1], tk.target[2] - s[2],
                      obs_wrap<T>(tk.target[3] - s[3])};
        o4[1] = V4<T>{obs_wrap<T>(tk.target[4] - s[4]), obs_wrap<T>(tk.target[5] - s[5]), s[6], s[7]};
        o4[2] = V4<T>{s[8], s[9], s[10], s[11]};
    } else {
        V2<T>* o2 = reinterpret_cast<V2<T>*>(row);
        const T ephi = obs_wrap<T>(T(0) - s[3]);
        const T eth = obs_wrap<T>(T(0) - s[4]);
#pragma unroll 1
        for (int k = 1; k <= tk.lookahead; ++k) {
            const V4<T> r = tk.traj[min(nstep + k, tab_last)];
            V2<T>* q = o2 + 3 * (k - 1);
            q[0] = V2<T>{r.x - s[0], r.y - s[1]};
            q[1] = V2<T>{r.z - s[2], ephi};
            q[2] = V2<T>{eth, obs_wrap<T>(r.w - s[5])};
        }
        V2<T>* q = o2 + 3 * tk.lookahead;
        q[0] = V2<T>{s[6], s[7]};
        q[1] = V2<T>{s[8], s[9]};
        q[2] = V2<T>{s[10], s[11]};
    }
    rew[e] = reward;
    done[e] = rc >= 0 ? 1 : 0;
    if (reason) reason[e] = (int8_t)rc;
    st_rew = (float)reward;
    st_reason = rc;
}

// Block-level episode statistics: warp shuffles -> shared memory -> one
// read-modify-write of this block's own partial slot (no atomics, deterministic).
__device__ __forceinline__ void block_stats(double* __restrict__ part, bool active, float rew,
                                            int reason, float epret, int eplen, int err) {
    __shared__ double sh[BLOCK / 32][NSTAT];
    const unsigned full = 0xffffffffu;
    float r = rew, er = epret;
    int el = eplen;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        r += __shfl_xor_sync(full, r, o);
        er += __shfl_xor_sync(full, er, o);
        el += __shfl_xor_sync(full, el, o);
    }
    const int n_tr = __popc(__ballot_sync(full, reason == 0));
    const int n_dv = __popc(__ballot_sync(full, reason == 1));
    const int n_fl = __popc(__ballot_sync(full, reason == 2));
    const int n_ac = __popc(__ballot_sync(full, active));
    const int n_er = __popc(__ballot_sync(full, err != 0));
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
    }
    __syncthreads();
    if (threadIdx.x < NSTAT) {
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < BLOCK / 32; ++i) acc += sh[i][threadIdx.x];
        part[(size_t)blockIdx.x * NSTAT + threadIdx.x] += acc;
    }
}

template <class T, bool TRACK, bool DR, bool MIX, class Pat>
__global__ void __launch_bounds__(BLOCK)
k_step(const __grid_constant__ EngineP<T> p, const T* __restrict__ act, T* __restrict__ obs,
       T* __restrict__ rew, uint8_t* __restrict__ done, int8_t* __restrict__ reason) {
    const int e = blockIdx.x * BLOCK + threadIdx.x;
    const bool active = e < p.n_env;
    float st_rew = 0.f, st_epret = 0.f;
    int st_reason = -1, st_eplen = 0, st_err = 0;
    if (active) {
        const uint64_t g = p.env_offset + (uint64_t)e;
        bool slot1 = false;
        if constexpr (MIX) slot1 = (int64_t)g >= p.mix_bound0;
        if (!slot1)
            step_env<T, TRACK, DR, 0, Pat>(p, e, g, act, obs, rew, done, reason, st_rew,
                                          st_reason, st_epret, st_eplen, st_err);
        else if constexpr (MIX)
            step_env<T, TRACK, DR, 1, Pat>(p, e, g, act, obs, rew, done, reason, st_rew,
                                          st_reason, st_epret, st_eplen, st_err);
    }
    if (p.stats_on) block_stats(p.stats, active, st_rew, st_reason, st_epret, st_eplen, st_err);
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
    const bool ok = slot1 ? dr_draw<T>(p.veh[1], p.ranges, p.seed, g, ctr, d0, d1, d2)
                          : dr_draw<T>(p.veh[0], p.ranges, p.seed, g, ctr, d0, d1, d2);
    p.dr0[e] = d0; p.dr1[e] = d1; p.dr2[e] = d2;
    p.param_ctr[e] = ctr;
    if (!ok) atomicMin(first_bad, e);
}

template <class T>
__global__ void k_pack_states(const __grid_constant__ EngineP<T> p, double* __restrict__ out) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= p.n_env) return;
    const V4<T> a0 = p.s0[e], a1 = p.s1[e], a2 = p.s2[e];
    double* r = out + (size_t)e * 12;
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
    p.s0[e] = V4<T>{(T)r[0], (T)r[1], (T)r[2], (T)r[3]};
    p.s1[e] = V4<T>{(T)r[4], (T)r[5], (T)r[6], (T)r[7]};
    p.s2[e] = V4<T>{(T)r[8], (T)r[9], (T)r[10], (T)r[11]};
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

// ------------------------------------------------------------------ launchers
template <class T>
cudaError_t Launch<T>::step(const EngineP<T>& p, bool track, bool dr, bool fossen, const T* act,
                            T* obs, T* rew, uint8_t* done, int8_t* reason, cudaStream_t st) {
    const dim3 grid((p.n_env + BLOCK - 1) / BLOCK);
    const bool mix = p.n_veh > 1;
#define UUV_L(TR, D, M, PAT) \
    k_step<T, TR, D, M, PAT><<<grid, BLOCK, 0, st>>>(p, act, obs, rew, done, reason)
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
    k_pack_states<T><<<(p.n_env + 255) / 256, 256, 0, st>>>(p, out);
    return cudaGetLastError();
}

template <class T>
cudaError_t Launch<T>::unpack_states(const EngineP<T>& p, const double* in, cudaStream_t st) {
    k_unpack_states<T><<<(p.n_env + 255) / 256, 256, 0, st>>>(p, in);
    return cudaGetLastError();
}

template <class T>
cudaError_t Launch<T>::pack_dr(const EngineP<T>& p, double* out, cudaStream_t st) {
    k_pack_dr<T><<<(p.n_env + 255) / 256, 256, 0, st>>>(p, out);
    return cudaGetLastError();
}

template <class T>
cudaError_t Launch<T>::step_attrs(cudaFuncAttributes* a, bool track, bool dr, bool fossen,
                                  bool mix) {
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

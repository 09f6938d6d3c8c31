// launch.h -- host-visible launcher declarations (definitions in uuv_kernels.cuh,
// explicitly instantiated by k_f32.cu / k_f64.cu).
#pragma once

#include <cuda_runtime.h>

#include "uuv_common.cuh"
#include "../../include/uuvsim.h"

namespace uuv {

#ifndef UUV_BLOCK
#define UUV_BLOCK 128
#endif
constexpr int BLOCK = UUV_BLOCK;   // threads per block of the env kernels (one env per thread)
// register budgets (65536 / (128 * blocks)): measured on B200, see DESIGN.md
#ifndef UUV_STEP_MIN_BLOCKS
#define UUV_STEP_MIN_BLOCKS 8      // one env per thread: 64 registers
#endif
#ifndef UUV_STEP_MIN_BLOCKS_DR
#define UUV_STEP_MIN_BLOCKS_DR 6   // with per-env randomised M/L in registers: 85
#endif
#ifndef UUV_STEP_MIN_BLOCKS_TRACK
#define UUV_STEP_MIN_BLOCKS_TRACK 6   // tracking (lookahead rows in registers): 85, no spills
#endif
#ifndef UUV_STEP_MIN_BLOCKS_F64
#define UUV_STEP_MIN_BLOCKS_F64 4     // fp64 parity mode and dense-pattern DR: 128 (doubles take
                                      // register pairs; the dense DR kernel keeps a full M and L;
                                      // measured: C3 fp64 73.5 -> 45.5 us, C5 371 -> 400 us)
#endif
#ifndef UUV_PAIR_MIN_BLOCKS
#define UUV_PAIR_MIN_BLOCKS 6      // two envs per thread: 85
#endif
constexpr int STEP_MIN_BLOCKS = UUV_STEP_MIN_BLOCKS;
constexpr int STEP_MIN_BLOCKS_DR = UUV_STEP_MIN_BLOCKS_DR;
constexpr int PAIR_MIN_BLOCKS = UUV_PAIR_MIN_BLOCKS;
constexpr int STEP_MIN_BLOCKS_TRACK = UUV_STEP_MIN_BLOCKS_TRACK;
constexpr int STEP_MIN_BLOCKS_F64 = UUV_STEP_MIN_BLOCKS_F64;

#ifndef UUV_PDL_TRIGGER
#define UUV_PDL_TRIGGER 0          // programmatic launch: 0 implicit trigger at completion,
                                   // 1 at kernel start, 2 after the heavy work.  Measured on
                                   // the C4 loop (us per step): 31.8 / 38.9 / 37.6, no PDL
                                   // 33.0 -- resident dependents waiting in griddepcontrol
                                   // slow the running kernel more than the launch they save
#endif

// band kernel (uuv_kernels.cuh k_band): two warps per block, chunks of up to
// 16 x BAND_VEC x BAND_BLOCK envs (one 16-byte flag load per thread and vector).
// Measured (tools/band_probe.py, flushed, us per step C2 / C4 / C3 / C5): 64
// threads 14.5 / 16.6 / 24.8 / 101; one warp per block capped at 128 registers
// (to fit beside six 80-register paired step blocks) 17.2 / 20.8 / 30.3 / 108.
#ifndef UUV_BAND_BLOCK
#define UUV_BAND_BLOCK 64
#endif
#ifndef UUV_BAND_VEC
#define UUV_BAND_VEC 4
#endif
#ifndef UUV_BAND_MIN_BLOCKS
#define UUV_BAND_MIN_BLOCKS 1
#endif
constexpr int BAND_BLOCK = UUV_BAND_BLOCK;
constexpr int BAND_VEC = UUV_BAND_VEC;
constexpr int BAND_MIN_BLOCKS = UUV_BAND_MIN_BLOCKS;
constexpr int BAND_MAX_PER = 16 * BAND_VEC * BAND_BLOCK;

#ifndef UUV_PAIR_AUTO_MIN_ENVS
#define UUV_PAIR_AUTO_MIN_ENVS 131072
#endif
constexpr long PAIR_AUTO_MIN_ENVS = UUV_PAIR_AUTO_MIN_ENVS;

#ifndef UUV_TMA_MIN_BLOCKS
#define UUV_TMA_MIN_BLOCKS 5       // persistent TMA pair kernel: 2 x 20 KB stages per block
#endif
#ifndef UUV_TMA_ACT
#define UUV_TMA_ACT 0              // also stage action rows through the TMA ring
#endif
#ifndef UUV_TMA_PAIR
#define UUV_TMA_PAIR 0             // default off: measured slower than the plain paired kernel
                                   // (96.7 vs 93.7 us at C5; residency 5 vs 6 blocks/SM)
#endif
constexpr int TMA_MIN_BLOCKS = UUV_TMA_MIN_BLOCKS;

// observation staging in shared memory: obs_dim <= MAX_STAGE_DIM (lookahead <= 5)
constexpr int MAX_STAGE_DIM = 36;
constexpr int MAX_STAGE_BYTES = 2 * BLOCK * MAX_STAGE_DIM * 8    // paired block, f64 rows
                                + 2 * BLOCK * 8 * 8;              // + staged f64 action rows

template <class T> struct Launch {
    // one fused step; fossen selects the structure-specialised variant, pair the
    // two-envs-per-thread kernel (fp32, Fossen, no randomisation)
    // act/obs/rew element type: T, or double when p.io_f64 (host-ABI path)
    static cudaError_t step(const EngineP<T>& p, bool track, bool dr, bool fossen, bool pair,
                            const void* act, void* obs, void* rew, uint8_t* done,
                            int8_t* reason, cudaStream_t st);
    static cudaError_t reset(const EngineP<T>& p, T* obs, cudaStream_t st);
    static cudaError_t observe(const EngineP<T>& p, T* obs, cudaStream_t st);
    static cudaError_t dr_init(const EngineP<T>& p, int* first_bad, cudaStream_t st);
    static cudaError_t pack_states(const EngineP<T>& p, double* out, cudaStream_t st);
    static cudaError_t pack_states_t(const EngineP<T>& p, T* out, cudaStream_t st);
    static cudaError_t pd_actions(const EngineP<T>& p, const UuvPdGains& g, const T* ref, T* act,
                                  cudaStream_t st);
    static cudaError_t unpack_states(const EngineP<T>& p, const double* in, cudaStream_t st);
    static cudaError_t pack_dr(const EngineP<T>& p, double* out, cudaStream_t st);
    static cudaError_t band_flags(const EngineP<T>& p, cudaStream_t st);
    static cudaError_t wrench(const EngineP<T>& p, bool dr, const double* act, double* out,
                              cudaStream_t st);
    static cudaError_t step_attrs(cudaFuncAttributes* a, bool track, bool dr, bool fossen,
                                  bool mix, bool pair, bool tma);
    static cudaError_t to_f64(const T* in, double* out, size_t n, cudaStream_t st);
    static cudaError_t from_f64(const double* in, T* out, size_t n, cudaStream_t st);
};

cudaError_t launch_bench_actions(uint64_t seed, uint64_t env_offset, int n_env, int act_dim,
                                 float* out_f32, double* out_f64, cudaStream_t st);
cudaError_t launch_stats_reduce(double* part, int nblk, double* out, int clear, cudaStream_t st);

}  // namespace uuv

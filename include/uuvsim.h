/*
 * uuvsim.h -- C ABI of the B200 env-step engine (libuuvsim_core.so).
 *
 * Part 1 is a drop-in for the reference's ABI v1 (reference
 * pkg/native/src/capi.rs): same ten symbols, same argument meaning, same
 * error codes and thread-local last-error contract, so the reference's own
 * ctypes binding (reference pkg/src/uuvsim/_native.py:49-78, selected with
 * UUVSIM_CORE_LIB) drives this library unchanged.  Buffers are
 * caller-allocated host memory, lengths are element counts, row-major,
 * env-major; floats are f64 and done flags u8 0/1.
 *
 * Part 2 is the B200 device face: the same engine driven with device
 * pointers on a caller-supplied CUDA stream (zero-copy for PyTorch tensors,
 * CUDA-graph capturable), plus inspection/teacher-forcing entry points the
 * parity tests use.  All signatures are plain C (no torch types).
 *
 * Return codes: 0 ok, 1 invalid config, 2 invalid handle, 3 bad buffer size,
 * 4 runtime error (capi.rs:21-25).  No C++ exception ever crosses the ABI.
 */
#ifndef UUVSIM_H
#define UUVSIM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define UUVSIM_ABI_VERSION 1

#define UUVSIM_OK 0
#define UUVSIM_ERR_CONFIG 1
#define UUVSIM_ERR_HANDLE 2
#define UUVSIM_ERR_SIZE 3
#define UUVSIM_ERR_RUNTIME 4

/* ---------------- Part 1: reference ABI v1 (capi.rs:72-253) ---------------- */

/* capi.rs:73-75 -- returns 1 */
uint32_t uuvsim_abi_version(void);

/* capi.rs:79-98 -- create an engine from a UTF-8 JSON config (engine.rs:17-94
 * schema; extra keys, ignored by the reference's parser: "vehicles",
 * batch.vehicle_mix, batch.env_offset, "device": {"precision": "fp32"|"fp64",
 * "index": n, "stats": bool, "host_io": "auto"|"copy"|"mapped",
 * "pair"/"stage_obs": "auto"|"on"|"off", "pattern": "auto"|"dense", "tma": bool}) */
int32_t uuvsim_create(const char* config_json, uint64_t* out_handle);

/* capi.rs:102-120 -- out[4] = {num_envs, obs_dim, action_dim, episode_len} */
int32_t uuvsim_spec(uint64_t handle, uint64_t* out);

/* capi.rs:123-140 -- reset all envs with a new root seed; obs_len = M*obs_dim */
int32_t uuvsim_reset(uint64_t handle, uint64_t seed, double* obs, uint64_t obs_len);

/* capi.rs:143-174 -- one lockstep step with auto-reset */
int32_t uuvsim_step(uint64_t handle, const double* actions, uint64_t actions_len, double* obs,
                    uint64_t obs_len, double* rew, uint64_t rew_len, uint8_t* done,
                    uint64_t done_len);

/* capi.rs:178-193 -- raw 12-component states, len = M*12 */
int32_t uuvsim_states(uint64_t handle, double* out, uint64_t len);

/* capi.rs:196-210 -- per-env control-step counters, len = M */
int32_t uuvsim_step_counts(uint64_t handle, int64_t* out, uint64_t len);

/* capi.rs:213-227 -- advisory on the GPU engine (0 = all cores) */
int32_t uuvsim_set_threads(uint64_t handle, uint64_t n);

/* capi.rs:230-237 -- stale / double destroy -> 2 */
int32_t uuvsim_destroy(uint64_t handle);

/* capi.rs:241-253 -- copies min(len, cap) bytes (not NUL-terminated), returns full length */
int64_t uuvsim_last_error(char* buf, uint64_t cap);

/* ---------------- Part 2: B200 extensions ---------------- */

/* uuvsim_step plus the termination reason per env (-1 none, 0 truncation,
 * 1 divergence, 2 failure; reference tasks.py:41-42,205) */
int32_t uuvsim_step_ex(uint64_t handle, const double* actions, uint64_t actions_len,
                       double* obs, uint64_t obs_len, double* rew, uint64_t rew_len,
                       uint8_t* done, uint64_t done_len, int8_t* reason, uint64_t reason_len);

/* teacher forcing / checkpoint-resume of the env slab */
int32_t uuvsim_set_states(uint64_t handle, const double* in, uint64_t len);
int32_t uuvsim_set_step_counts(uint64_t handle, const int64_t* in, uint64_t len);
/* RNG counters (engine.rs:338-339, private in the reference) */
int32_t uuvsim_counters(uint64_t handle, uint64_t* reset_ctr, uint64_t* param_ctr,
                        uint64_t len);
/* per-env randomised parameter record [M][10]:
 * f_mass f_added f_dlin f_dquad f_thrust rb_x rb_y rb_z weight buoyancy */
int32_t uuvsim_dr_factors(uint64_t handle, double* out, uint64_t len);
/* body wrench tau [M][6] of every env for f64 action rows [M][A] (the step's
 * thruster map, thrusters.py:97-119, incl. the randomised thrust factor);
 * inspection / force-output parity */
int32_t uuvsim_wrench(uint64_t handle, const double* actions, uint64_t actions_len, double* out,
                      uint64_t out_len);
/* episode statistics [9]: sum reward, dones by reason (trunc, div, fail),
 * sum of completed-episode returns, sum of their lengths, env-steps,
 * rejected per-episode resamples, fp32 env-steps recomputed in fp64 because
 * their pitch left |theta| <= 1.4 (Euler band).  clear != 0 zeroes the
 * accumulators. */
int32_t uuvsim_stats(uint64_t handle, double* out, uint64_t len, int32_t clear);
/* JSON description of the engine (precision, grid, registers, device) */
int64_t uuvsim_info(uint64_t handle, char* buf, uint64_t cap);

/* Ordering: host-ABI calls (uuvsim_step, _states, ...) run on the engine's own
 * stream and wait for the engine's last device-face launch (recorded outside
 * stream capture), so device-face then host-ABI calls need no explicit sync.
 *
 * device face: all pointers are device memory; stream = cudaStream_t (0 = legacy).
 * actions/obs/rew elements are the engine precision: float for "fp32" engines
 * (default), double for "fp64" engines (see uuvsim_info). */
int32_t uuvsim_dev_step(uint64_t handle, const void* actions, uint64_t actions_len, void* obs,
                        uint64_t obs_len, void* rew, uint64_t rew_len, uint8_t* done,
                        uint64_t done_len, int8_t* reason, uint64_t reason_len, uint64_t stream);
int32_t uuvsim_dev_reset(uint64_t handle, uint64_t seed, void* obs, uint64_t obs_len,
                         uint64_t stream);
int32_t uuvsim_dev_observe(uint64_t handle, void* obs, uint64_t obs_len, uint64_t stream);
int32_t uuvsim_dev_bench_actions(uint64_t handle, void* actions, uint64_t len, uint64_t stream);
/* exact slab checkpoint (no reference counterpart: its RNG counters are private,
 * engine.rs:338-339).  uuvsim_snapshot_size -> bytes; uuvsim_snapshot fills a
 * caller buffer of exactly that size; uuvsim_restore loads it into an engine of
 * the same configuration (code 1 on a mismatch), after which steps continue
 * bit-for-bit as in the engine that was saved. */
int32_t uuvsim_snapshot_size(uint64_t handle, uint64_t* out_bytes);
int32_t uuvsim_snapshot(uint64_t handle, void* buf, uint64_t len);
int32_t uuvsim_restore(uint64_t handle, const void* buf, uint64_t len);
/* register (buf != NULL) or clear (NULL) a caller-owned device buffer
 * [M][obs_dim] (engine precision): later device-face steps write each finished
 * env's TERMINAL observation (pre-reset state, terminating step) into its row;
 * other rows are left untouched.  Not used by the host-buffer uuvsim_step. */
int32_t uuvsim_dev_set_final_obs(uint64_t handle, void* buf, uint64_t len);
/* on != 0: later device-face steps launch as programmatic dependents of the
 * previous kernel on their stream (griddepcontrol: the step's CTAs may be
 * scheduled while that kernel finishes and wait for its completion before
 * reading anything; they also let the next programmatic dependent launch
 * early).  Inside a CUDA graph of back-to-back kernels this hides the
 * kernel-to-kernel launch gap.  Results are unchanged.  Host-ABI steps never
 * use it. */
int32_t uuvsim_dev_set_pdl(uint64_t handle, int32_t on);
/* register (buf != NULL) or clear (NULL) a caller-owned device buffer of
 * num_envs floats: later device-face steps also write done as 0.0 / 1.0 into
 * it (a rollout's done buffer, written by the step itself).  Not used by the
 * host-buffer uuvsim_step. */
int32_t uuvsim_dev_set_done_f32(uint64_t handle, float* buf, uint64_t len);
/* PD baseline (reference baseline.py:38-75) over the engine's own state slab:
 * err_body = R^T (ref_xyz - p), err_ang = (ref_ang - ang + pi) mod 2 pi - pi,
 * wrench = kp * err - kd * nu, f = pinv(A) wrench, throttle = f / kmax (linear) or
 * copysign(sqrt(|f| / kmax), f) (quadratic_signed), clamped to [-1, 1].  One
 * kernel; ref6 is a device pointer to the reference pose (engine precision),
 * actions [M][action_dim] (engine precision) on the caller's stream. */
typedef struct {
    double kp[6], kd[6];
    double pinv[2][8][6];      /* per vehicle slot: pinv of the 6 x N allocation, [thruster][dof] */
    double kmax[2][8];
    int32_t quadratic[2][8];   /* 1 = quadratic_signed, 0 = linear */
} UuvPdGains;
int32_t uuvsim_dev_pd_actions(uint64_t handle, const UuvPdGains* gains, const void* ref6,
                              void* actions, uint64_t actions_len, uint64_t stream);
/* raw states [M][12] into a device buffer (engine precision) */
int32_t uuvsim_dev_states(uint64_t handle, void* out, uint64_t len, uint64_t stream);
int32_t uuvsim_dev_stats(uint64_t handle, double* out, uint64_t len, int32_t clear,
                         uint64_t stream);
/* capture n_steps consecutive device steps on fixed buffers into a CUDA graph.
 * Buffers as for uuvsim_dev_step: actions [M][A], obs [M][obs_dim] (16-byte
 * aligned), rew [M], done [M], reason [M] or NULL, elements in the engine
 * precision; they must stay valid while the graph is replayed. */
int32_t uuvsim_dev_graph_capture(uint64_t handle, const void* actions, void* obs, void* rew,
                                 uint8_t* done, int8_t* reason, uint32_t n_steps);
int32_t uuvsim_dev_graph_launch(uint64_t handle, uint64_t stream);
int32_t uuvsim_synchronize(uint64_t handle);

#ifdef __cplusplus
}
#endif
#endif

/* uuvsim_rl.h -- fused rollout-loop kernels for the device PPO loop (B200 extension).
 *
 * Not part of the reference's C ABI: the reference trains with a numpy actor-critic
 * on the host (pkg/src/uuvsim/ppo.py:263-338, nets.py:31-192).  These entry points
 * run one collection step of that loop on the device around the fused env step
 * (uuvsim_dev_step), so a rollout horizon is three kernels per step in one CUDA
 * graph instead of ~40 small framework kernels:
 *
 *   uuvsim_rl_policy_act  normalise obs with the running mean/var (nets.py:168-192),
 *                         actor-critic forward (2 x hidden tanh trunks, tanh mean
 *                         head, linear value head; nets.py:31-55), Gaussian sample
 *                         with a state-independent log-std, clamp, log-prob, and
 *                         per-block partial sums for the normaliser update
 *   (the policy layers run on the 5th-generation tensor cores -- tcgen05.mma
 *   kind::tf32, 3xTF32 split for fp32 accuracy, accumulators in TMEM -- when a
 *   weight image from uuvsim_rl_prepare is passed; else on the CUDA cores)
 *   uuvsim_rl_post        merge the partial sums into mean/var/count (parallel
 *                         variance formula, nets.py:177-188), copy reward / done
 *                         into the rollout buffers, advance the noise counter
 *
 * Parameters are the torch tensors of paper_2410_14117_b200.rollout.ActorCritic
 * (row-major nn.Linear weights [out][in], fp32, contiguous).  All pointers are
 * device pointers; `stream` is a cudaStream_t.  Return codes as include/uuvsim.h.
 */
#ifndef UUVSIM_RL_H
#define UUVSIM_RL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    uint64_t num_envs;
    uint32_t obs_dim;        /* <= 36 */
    uint32_t act_dim;        /* <= 8 */
    uint32_t hidden;         /* 64 */
    uint32_t flags;          /* 1: sample (else act = raw = mean), 2: accumulate normaliser sums,
                                4: value only (bootstrap), 8: launch as a programmatic dependent
                                of the previous kernel on the stream (tensor-core kernel; see
                                uuvsim_dev_set_pdl) */
    uint64_t seed;           /* noise stream seed */
    uint64_t env_offset;     /* global index of env 0 (noise stream id) */
    const uint64_t* noise_ctr;   /* device counter, advanced by uuvsim_rl_post */
    const float* obs;        /* [M][D] raw observations */
    const double* norm_mean; /* [D] */
    const double* norm_var;  /* [D] */
    double norm_clip;
    /* actor: a1 [H][D], a2 [H][H], am [A][H]; critic: c1 [H][D], c2 [H][H], cv [1][H] */
    const float *a1w, *a1b, *a2w, *a2b, *amw, *amb;
    const float *c1w, *c1b, *c2w, *c2b, *cvw, *cvb;
    const float* log_std;    /* [A] */
    float* nobs_out;         /* [M][D] normalised obs (policy input), or NULL */
    float* raw_out;          /* [M][A] unclamped sample, or NULL */
    float* act_out;          /* [M][A] clamped to [-1, 1] (the env's action tensor), or NULL */
    float* logp_out;         /* [M], or NULL */
    float* value_out;        /* [M], or NULL */
    double* stats_part;      /* [uuvsim_rl_policy_blocks(M)][2 D] (sum x, sum x^2) when flags & 2 */
    const void* wimage;      /* tensor-core weight image from uuvsim_rl_prepare, or NULL
                                (then the CUDA-core kernel runs) */
} UuvRlPolicyArgs;

typedef struct {
    uint64_t num_envs;
    uint32_t obs_dim;
    uint32_t n_part;         /* number of partial rows written by the policy launch:
                                ceil(M / 128) for the tensor-core kernel (one per CTA),
                                uuvsim_rl_policy_blocks(M) for the CUDA-core kernel */
    const double* stats_part;
    double* norm_mean;       /* [D] updated in place */
    double* norm_var;        /* [D] */
    double* norm_count;      /* [1] */
    const float* rew_in;     /* [M] env reward, copied to rew_out, or NULL */
    const uint8_t* done_in;  /* [M] env done flags, copied to done_out as 0/1 floats */
    float* rew_out;
    float* done_out;
    uint64_t* noise_ctr;     /* += 1 */
    uint32_t flags;          /* 1: launch as a programmatic dependent of the previous kernel */
    uint32_t reserved;
} UuvRlPostArgs;

/* partial rows the stats_part buffer must hold for num_envs (size / (2 D)); the
 * tensor-core kernel writes the first ceil(num_envs / 128) of them */
uint32_t uuvsim_rl_policy_blocks(uint64_t num_envs);
/* bytes of the tensor-core weight image for obs_dim (multiple of 16) */
uint64_t uuvsim_rl_image_bytes(uint32_t obs_dim);
/* build the weight image (3xTF32 hi/lo splits in the UMMA K-major core-matrix
 * layout + biases/heads) from the parameter pointers in args; run it whenever the
 * parameters change (once per collected horizon) */
int32_t uuvsim_rl_prepare(const UuvRlPolicyArgs* args, void* image, uint64_t len, uint64_t stream);
int32_t uuvsim_rl_policy_act(const UuvRlPolicyArgs* args, uint64_t stream);
int32_t uuvsim_rl_post(const UuvRlPostArgs* args, uint64_t stream);
/* GAE over the horizon buffers (reference ppo.py:112-130): [T][M] fp32 rewards,
 * values, done flags (terminal), bootstrap values [M] -> advantages, returns [T][M] */
int32_t uuvsim_rl_gae(const float* rew, const float* val, const float* done, const float* boot,
                      uint32_t horizon, uint64_t num_envs, float gamma, float lam, float* adv,
                      float* ret, uint64_t stream);

#ifdef __cplusplus
}
#endif

#endif /* UUVSIM_RL_H */

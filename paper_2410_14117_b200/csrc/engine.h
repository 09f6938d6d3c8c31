// engine.h -- host-side B200 engine: config -> device slab -> launches.
//
// Mirrors the reference's Engine (native/src/engine.rs:329-580): JSON config
// parsing and validation (engine.rs:17-135, 174-229, 350-459), base-vehicle
// kernel construction (engine.rs:234-286), per-env domain randomisation
// (engine.rs:289-323, here the K3 kernel), reset (462-471) and the lockstep
// step (482-580, here one K1 launch).  State lives on the GPU; host f64 buffers
// are only touched by the C-ABI copy path.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "launch.h"

namespace uuv {

struct ConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct RuntimeError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// Base vehicle, fp64 (engine.rs:141-229)
struct BaseVehicle {
    double mass = 0, weight = 0, buoyancy = 0;
    double inertia[9] = {}, rg[3] = {}, rb[3] = {};
    double added[36] = {}, dlin[36] = {}, dquad[6] = {};
    std::vector<std::array<double, 3>> pos, dir;
    std::vector<double> kmax;
    std::vector<int> curve;
};

struct TaskCfg {
    int kind = 0;
    double target[6] = {0, 0, 2, 0, 0, 0};
    double cx = 0, cy = 0, radius = 1, omega = 0.1, climb = 0.05, scale = 2, depth = 2;
    int lookahead = 5;
    int64_t episode_len = 600;
    double control_dt = 0.05;
    int n_substeps = 10;
};

struct RangesCfg {
    bool enabled = false, per_episode = false;
    double mass[2] = {1, 1}, added[2] = {1, 1}, dlin[2] = {1, 1}, dquad[2] = {1, 1},
           thrust[2] = {1, 1}, ratio[2] = {1, 1};
    double rb_offset = 0;
};

class Engine {
public:
    explicit Engine(const std::string& config_json);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    // dims (uuvsim_spec)
    int64_t num_envs() const { return m_; }
    int obs_dim() const { return obs_dim_; }
    int action_dim() const { return n_act_; }
    int64_t episode_len() const { return task_.episode_len; }
    int threads = 1;

    // host-f64 ABI face (capi.rs:123-210)
    void reset_host(uint64_t seed, double* obs);
    void step_host(const double* act, double* obs, double* rew, uint8_t* done, int8_t* reason);
    void states_host(double* out);
    void step_counts_host(int64_t* out);
    void set_states_host(const double* in);
    void set_step_counts_host(const int64_t* in);
    void counters_host(uint64_t* reset_ctr, uint64_t* param_ctr);
    void dr_factors_host(double* out);     // [M][10]
    void wrench_host(const double* act, double* out);   // [M][A] -> [M][6]
    void stats_host(double* out, bool clear);

    // exact slab checkpoint: header + the per-env device state (states, step
    // counters, running returns, RNG counters, DR records, root seed).  Restoring
    // into an engine of the same configuration continues bit-for-bit.
    size_t snapshot_bytes() const;
    void snapshot(void* out);
    void restore(const void* in, size_t len);

    // device face (zero-copy, stream-ordered, graph-capturable).  Element type of
    // act/obs/rew is the engine precision: f32 for fp32 engines, f64 for fp64.
    bool is_fp64() const { return fp64_; }
    bool fossen() const { return fossen_; }
    void dev_step(const void* act, void* obs, void* rew, uint8_t* done, int8_t* reason,
                  cudaStream_t st);
    void dev_reset(uint64_t seed, void* obs, cudaStream_t st);
    void dev_observe(void* obs, cudaStream_t st);
    void dev_bench_actions(void* act, cudaStream_t st);
    void dev_states(void* out, cudaStream_t st);
    void dev_pd_actions(const UuvPdGains& g, const void* ref6, void* act, cudaStream_t st);
    void dev_set_final_obs(void* buf);
    void dev_set_pdl(bool on);
    void dev_set_done_f32(float* buf);
    void dev_stats(double* out, bool clear, cudaStream_t st);
    void graph_capture(const void* act, void* obs, void* rew, uint8_t* done, int8_t* reason,
                       int n_steps);
    void graph_launch(cudaStream_t st);
    void synchronize();
    std::string info() const;
    void activate() const;
    void check_device() const;
    void note_device_face(cudaStream_t st);   // after a device-face launch
    void wait_device_face();                  // before host-ABI work on stream_

private:
    void parse(const std::string& text);
    void release();
    void build_params();
    void allocate();
    void ensure_staging();
    void ensure_pack();
    void free_staging();
    void init_randomization();
    template <class T> EngineP<T>& P();
    template <class T> void fill_params(EngineP<T>& p);
    template <class T> void fill_vehicle(const BaseVehicle& v, VehP<T>& V) const;
    template <class T> void step_host_T(const double* act, double* obs, double* rew,
                                        uint8_t* done, int8_t* reason);
    template <class T> void reset_host_T(uint64_t seed, double* obs);
    bool check_fossen() const;

    // config
    uint64_t seed_ = 0;
    uint64_t env_offset_ = 0;
    int64_t m_ = 0;
    int obs_dim_ = 0, n_act_ = 0;
    bool fp64_ = false;
    bool stats_on_ = true;
    bool fossen_ = false;
    bool force_dense_ = false;
    bool band64_ = true;      // device.band64: fp64 recompute of steps entering the pitch band
    bool band_same_ = false;
    int band_order_ = 0;      // device.band_order: 0 band kernel first, 1 step kernel first (A/B)
    int64_t band_per_cfg_ = 0;   // device.band_per: envs per band-kernel block (A/B; 0 auto)
    int band_rege_ = -1;         // device.band_rege: -1 auto (<= 8,192 envs), 0 / 1 (A/B)
    int band_refop_ = -1;        // device.band_refop: -1 auto (control_dt >= 0.1 s), 0 / 1
    bool band_none_ = false;  // device.band_stream "none": no band kernel at all (A/B only)
    bool band_tail_ = true;   // device.band_tail false: predictor misses stay fp32 (A/B only)
    double band_margin_ = -1e300;   // device.band_margin override (experiments; default by control_dt)  // device.band_stream "same": band kernel after the step, one stream
    int pair_mode_ = -1;      // device.pair: -1 auto, 0 off, 1 on
    int stage_mode_ = -1;     // device.stage_obs: -1 auto, 0 off, 1 on
    int tma_mode_ = -1;       // device.tma: -1 auto, 0 off, 1 on
    bool pair_ = false;       // two envs per thread (resolved)
    int device_ = 0;
    std::vector<BaseVehicle> veh_;
    std::vector<int64_t> mix_;
    TaskCfg task_;
    RangesCfg ranges_;

    // launch parameter blocks (one live, by precision)
    std::unique_ptr<EngineP<float>> pf_;
    std::unique_ptr<EngineP<double>> pd_;

    // device memory
    void* arena_ = nullptr;
    size_t arena_bytes_ = 0;
    size_t staging_bytes_ = 0;   // host-ABI staging, allocated on first host-face use
    size_t arena_used_ = 0;   // per-env state occupies arena_[0, arena_used_)
    uint64_t config_hash() const;
    void* traj_ = nullptr;
    double* stats_part_ = nullptr;
    int nblk_ = 0;
    int band_grid_ = 0;       // blocks of the band kernel (0: band64 off)
    int band_per_ = 0;        // envs scanned per band-kernel block
    int nstat_blk_ = 0;       // stats partial slots: step blocks + band blocks
    VehP<double>* d_veh64_ = nullptr;        // fp64 base vehicles (step-kernel tail)
    uint32_t* d_band_f_ = nullptr;           // band env counters (256 B) + per-env flag bytes
    volatile int32_t* h_err_ = nullptr;      // rejected-resample flag (mapped page-locked)
    volatile int32_t* d_err_ = nullptr;      // its device alias
    cudaStream_t band_side_ = nullptr;       // band kernel stream (fork / join per step)
    cudaEvent_t band_ev_[2] = {nullptr, nullptr};
    // ABI staging (f64 host layout; fp32 engines convert on device)
    void* d_actT_ = nullptr;
    void* d_obsT_ = nullptr;
    void* d_rewT_ = nullptr;
    double* d_act64_ = nullptr;
    double* d_obs64_ = nullptr;
    double* d_rew64_ = nullptr;
    uint8_t* d_done_ = nullptr;
    int8_t* d_reason_ = nullptr;
    double* d_pack_ = nullptr;
    int* d_flag_ = nullptr;
    double* d_stats_out_ = nullptr;
    float4* d_vpack_ = nullptr;
    std::vector<VehP<double>> veh64_;   // fp64 base vehicles (band replay parameters)
    cudaStream_t stream_ = nullptr;
    cudaEvent_t dev_ev_ = nullptr;   // last device-face launch (host-ABI calls wait for it)
    bool dev_pending_ = false;
    cudaGraphExec_t graph_exec_ = nullptr;
    // host-ABI step replayed as one CUDA graph (H2D -> step -> D2H) while the
    // caller keeps passing the same page-locked buffers
    // host_io "mapped": device aliases of the caller's page-locked ABI buffers
    void* dev_io_[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    int host_io_ = -1;        // device.host_io: -1 auto, 0 copy, 1 mapped
    // auto: zero-copy while the per-step host traffic is small enough that
    // launch + DMA latency dominates (measured crossover)
    static constexpr size_t kMappedAutoBytes = size_t(8) << 20;
    bool use_mapped() const {
        return host_io_ == 1 ||
               (host_io_ < 0 && (size_t)m_ * (size_t)(obs_dim_ + n_act_ + 2) * 8 <= kMappedAutoBytes);
    }
    template <class T> void enqueue_step_mapped();
    // whole host-ABI step (H2D, kernel, D2Hs) captured per set of page-locked
    // buffers; keyed by pointer AND allocation id so a freed-and-reused address
    // never replays a stale graph.  A few entries: callers alternate buffers.
    struct AbiGraph {
        const void* ptr[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
        unsigned long long id[5] = {0, 0, 0, 0, 0};
        cudaGraphExec_t exec = nullptr;
    };
    static constexpr int kAbiGraphs = 4;
    std::array<AbiGraph, kAbiGraphs> abi_graphs_{};
    int abi_next_ = 0;
    template <class T> void enqueue_step_host(const double* act, double* obs, double* rew,
                                              uint8_t* done, int8_t* reason);
    std::string device_name_;
    int sm_count_ = 0;
};

void cuda_check(cudaError_t e, const char* what);

}  // namespace uuv

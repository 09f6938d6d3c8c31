// capi.cpp -- the C ABI (include/uuvsim.h).  Contract of the reference's
// capi.rs: versioned, handle registry behind a mutex, per-handle mutex (one
// host thread per handle at a time), error codes plus a thread-local message,
// and an exception fence so nothing unwinds across the boundary.
#include "../../include/uuvsim.h"

#include <atomic>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>

#include "engine.h"

namespace {

struct Slot {
    std::mutex mu;
    std::unique_ptr<uuv::Engine> eng;
};

std::mutex g_mu;
std::map<uint64_t, std::shared_ptr<Slot>> g_registry;   // capi.rs:27
std::atomic<uint64_t> g_next{1};                          // capi.rs:30
thread_local std::string t_last_error;                    // capi.rs:32-34

int32_t fail(int32_t code, const std::string& msg) {
    t_last_error = msg;
    return code;
}

std::shared_ptr<Slot> lookup(uint64_t h) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_registry.find(h);
    return it == g_registry.end() ? nullptr : it->second;
}

// capi.rs:58-70: map every failure to a code, never unwind
template <class F> int32_t guarded(F&& f) {
    try {
        return f();
    } catch (const uuv::ConfigError& e) {
        return fail(UUVSIM_ERR_CONFIG, e.what());
    } catch (const uuv::RuntimeError& e) {
        return fail(UUVSIM_ERR_RUNTIME, e.what());
    } catch (const std::exception& e) {
        return fail(UUVSIM_ERR_RUNTIME, e.what());
    } catch (...) {
        return fail(UUVSIM_ERR_RUNTIME, "unknown error in native core");
    }
}

// lock the handle's engine and run f(engine)
template <class F> int32_t with_engine(uint64_t h, F&& f) {
    return guarded([&]() -> int32_t {
        auto slot = lookup(h);
        if (!slot) return fail(UUVSIM_ERR_HANDLE, "handle " + std::to_string(h) + " is not valid");
        std::lock_guard<std::mutex> lk(slot->mu);
        if (!slot->eng) return fail(UUVSIM_ERR_HANDLE, "handle " + std::to_string(h) + " is not valid");
        return f(*slot->eng);
    });
}

int32_t bad_size(const char* what, uint64_t want, const char* unit) {
    return fail(UUVSIM_ERR_SIZE, std::string(what) + " buffer must hold " + std::to_string(want) +
                                     " " + unit);
}

cudaStream_t as_stream(uint64_t s) { return reinterpret_cast<cudaStream_t>(s); }

// device-face output rows are written with 8/16-byte vector stores
int32_t misaligned(const char* what, const void* p, uintptr_t align) {
    if (((uintptr_t)p & (align - 1)) == 0) return UUVSIM_OK;
    return fail(UUVSIM_ERR_SIZE, std::string(what) + " buffer must be " + std::to_string(align) +
                                     "-byte aligned");
}

int64_t copy_out(const std::string& msg, char* buf, uint64_t cap) {
    if (buf && cap > 0) std::memcpy(buf, msg.data(), std::min<uint64_t>(cap, msg.size()));
    return (int64_t)msg.size();
}

}  // namespace

extern "C" {

uint32_t uuvsim_abi_version(void) { return UUVSIM_ABI_VERSION; }

int32_t uuvsim_create(const char* config, uint64_t* out) {
    return guarded([&]() -> int32_t {
        if (!config || !out) return fail(UUVSIM_ERR_CONFIG, "null pointer argument");
        auto slot = std::make_shared<Slot>();
        slot->eng = std::make_unique<uuv::Engine>(std::string(config));
        const uint64_t h = g_next.fetch_add(1);
        {
            std::lock_guard<std::mutex> lk(g_mu);
            g_registry[h] = slot;
        }
        *out = h;
        return UUVSIM_OK;
    });
}

int32_t uuvsim_spec(uint64_t h, uint64_t* out) {
    if (!out) return fail(UUVSIM_ERR_SIZE, "null pointer argument");
    return with_engine(h, [&](uuv::Engine& e) {
        out[0] = (uint64_t)e.num_envs();
        out[1] = (uint64_t)e.obs_dim();
        out[2] = (uint64_t)e.action_dim();
        out[3] = (uint64_t)e.episode_len();
        return UUVSIM_OK;
    });
}

int32_t uuvsim_reset(uint64_t h, uint64_t seed, double* obs, uint64_t obs_len) {
    return with_engine(h, [&](uuv::Engine& e) {
        const uint64_t want = (uint64_t)e.num_envs() * e.obs_dim();
        if (!obs || obs_len != want) return bad_size("obs", want, "f64");
        e.reset_host(seed, obs);
        return UUVSIM_OK;
    });
}

int32_t uuvsim_step_ex(uint64_t h, const double* act, uint64_t act_len, double* obs,
                       uint64_t obs_len, double* rew, uint64_t rew_len, uint8_t* done,
                       uint64_t done_len, int8_t* reason, uint64_t reason_len) {
    return with_engine(h, [&](uuv::Engine& e) {
        const uint64_t m = (uint64_t)e.num_envs();
        const uint64_t want_act = m * e.action_dim(), want_obs = m * e.obs_dim();
        if (!act || act_len != want_act) return bad_size("actions", want_act, "f64");
        if (!obs || obs_len != want_obs) return bad_size("obs", want_obs, "f64");
        if (!rew || rew_len != m) return bad_size("rewards", m, "f64");
        if (!done || done_len != m) return bad_size("dones", m, "u8");
        if (reason && reason_len != m) return bad_size("reasons", m, "i8");
        e.step_host(act, obs, rew, done, reason);
        return UUVSIM_OK;
    });
}

int32_t uuvsim_step(uint64_t h, const double* act, uint64_t act_len, double* obs,
                    uint64_t obs_len, double* rew, uint64_t rew_len, uint8_t* done,
                    uint64_t done_len) {
    return uuvsim_step_ex(h, act, act_len, obs, obs_len, rew, rew_len, done, done_len, nullptr, 0);
}

int32_t uuvsim_states(uint64_t h, double* out, uint64_t len) {
    return with_engine(h, [&](uuv::Engine& e) {
        const uint64_t want = (uint64_t)e.num_envs() * 12;
        if (!out || len != want) return bad_size("states", want, "f64");
        e.states_host(out);
        return UUVSIM_OK;
    });
}

int32_t uuvsim_step_counts(uint64_t h, int64_t* out, uint64_t len) {
    return with_engine(h, [&](uuv::Engine& e) {
        const uint64_t m = (uint64_t)e.num_envs();
        if (!out || len != m) return bad_size("step", m, "i64");
        e.step_counts_host(out);
        return UUVSIM_OK;
    });
}

int32_t uuvsim_set_threads(uint64_t h, uint64_t n) {
    return with_engine(h, [&](uuv::Engine& e) {
        e.threads = n == 0 ? (int)std::max(1u, std::thread::hardware_concurrency()) : (int)n;
        return UUVSIM_OK;
    });
}

int32_t uuvsim_destroy(uint64_t h) {
    return guarded([&]() -> int32_t {
        std::shared_ptr<Slot> slot;
        {
            std::lock_guard<std::mutex> lk(g_mu);
            auto it = g_registry.find(h);
            if (it == g_registry.end())
                return fail(UUVSIM_ERR_HANDLE, "handle " + std::to_string(h) + " is not valid");
            slot = it->second;
            g_registry.erase(it);
        }
        std::lock_guard<std::mutex> lk(slot->mu);   // wait for an in-flight call
        slot->eng.reset();
        return UUVSIM_OK;
    });
}

int64_t uuvsim_last_error(char* buf, uint64_t cap) { return copy_out(t_last_error, buf, cap); }

// ------------------------------------------------------------------ extensions
int32_t uuvsim_set_states(uint64_t h, const double* in, uint64_t len) {
    return with_engine(h, [&](uuv::Engine& e) {
        const uint64_t want = (uint64_t)e.num_envs() * 12;
        if (!in || len != want) return bad_size("states", want, "f64");
        e.set_states_host(in);
        return UUVSIM_OK;
    });
}

int32_t uuvsim_set_step_counts(uint64_t h, const int64_t* in, uint64_t len) {
    return with_engine(h, [&](uuv::Engine& e) {
        const uint64_t m = (uint64_t)e.num_envs();
        if (!in || len != m) return bad_size("step", m, "i64");
        e.set_step_counts_host(in);
        return UUVSIM_OK;
    });
}

int32_t uuvsim_counters(uint64_t h, uint64_t* rc, uint64_t* pc, uint64_t len) {
    return with_engine(h, [&](uuv::Engine& e) {
        const uint64_t m = (uint64_t)e.num_envs();
        if ((!rc && !pc) || len != m) return bad_size("counter", m, "u64");
        e.counters_host(rc, pc);
        return UUVSIM_OK;
    });
}

int32_t uuvsim_dr_factors(uint64_t h, double* out, uint64_t len) {
    return with_engine(h, [&](uuv::Engine& e) {
        const uint64_t want = (uint64_t)e.num_envs() * 10;
        if (!out || len != want) return bad_size("factor", want, "f64");
        e.dr_factors_host(out);
        return UUVSIM_OK;
    });
}

int32_t uuvsim_wrench(uint64_t h, const double* actions, uint64_t actions_len, double* out,
                      uint64_t out_len) {
    return with_engine(h, [&](uuv::Engine& e) {
        const uint64_t na = (uint64_t)e.num_envs() * e.action_dim(), nt = (uint64_t)e.num_envs() * 6;
        if (!actions || actions_len != na) return bad_size("action", na, "f64");
        if (!out || out_len != nt) return bad_size("wrench", nt, "f64");
        e.wrench_host(actions, out);
        return UUVSIM_OK;
    });
}

int32_t uuvsim_stats(uint64_t h, double* out, uint64_t len, int32_t clear) {
    return with_engine(h, [&](uuv::Engine& e) {
        if (!out || len != (uint64_t)uuv::NSTAT) return bad_size("stats", uuv::NSTAT, "f64");
        e.stats_host(out, clear != 0);
        return UUVSIM_OK;
    });
}

int64_t uuvsim_info(uint64_t h, char* buf, uint64_t cap) {
    std::string s;
    int32_t rc = with_engine(h, [&](uuv::Engine& e) {
        s = e.info();
        return UUVSIM_OK;
    });
    if (rc != UUVSIM_OK) return -(int64_t)rc;
    return copy_out(s, buf, cap);
}

int32_t uuvsim_dev_step(uint64_t h, const void* act, uint64_t act_len, void* obs,
                        uint64_t obs_len, void* rew, uint64_t rew_len, uint8_t* done,
                        uint64_t done_len, int8_t* reason, uint64_t reason_len, uint64_t stream) {
    return with_engine(h, [&](uuv::Engine& e) {
        const uint64_t m = (uint64_t)e.num_envs();
        const uint64_t want_act = m * e.action_dim(), want_obs = m * e.obs_dim();
        const char* u = e.is_fp64() ? "f64" : "f32";
        if (!act || act_len != want_act) return bad_size("actions", want_act, u);
        if (!obs || obs_len != want_obs) return bad_size("obs", want_obs, u);
        if (!rew || rew_len != m) return bad_size("rewards", m, u);
        if (!done || done_len != m) return bad_size("dones", m, "u8");
        if (reason && reason_len != m) return bad_size("reasons", m, "i8");
        if (int32_t c = misaligned("obs", obs, 16)) return c;
        if (int32_t c = misaligned("actions", act, e.is_fp64() ? 8 : 4)) return c;
        e.dev_step(act, obs, rew, done, reason, as_stream(stream));
        return UUVSIM_OK;
    });
}

int32_t uuvsim_dev_reset(uint64_t h, uint64_t seed, void* obs, uint64_t obs_len,
                         uint64_t stream) {
    return with_engine(h, [&](uuv::Engine& e) {
        const uint64_t want = (uint64_t)e.num_envs() * e.obs_dim();
        if (obs && obs_len != want) return bad_size("obs", want, e.is_fp64() ? "f64" : "f32");
        if (obs) {
            if (int32_t c = misaligned("obs", obs, 16)) return c;
        }
        e.dev_reset(seed, obs, as_stream(stream));
        return UUVSIM_OK;
    });
}

int32_t uuvsim_dev_observe(uint64_t h, void* obs, uint64_t obs_len, uint64_t stream) {
    return with_engine(h, [&](uuv::Engine& e) {
        const uint64_t want = (uint64_t)e.num_envs() * e.obs_dim();
        if (!obs || obs_len != want) return bad_size("obs", want, e.is_fp64() ? "f64" : "f32");
        if (int32_t c = misaligned("obs", obs, 16)) return c;
        e.dev_observe(obs, as_stream(stream));
        return UUVSIM_OK;
    });
}

int32_t uuvsim_dev_bench_actions(uint64_t h, void* act, uint64_t len, uint64_t stream) {
    return with_engine(h, [&](uuv::Engine& e) {
        const uint64_t want = (uint64_t)e.num_envs() * e.action_dim();
        if (!act || len != want) return bad_size("actions", want, e.is_fp64() ? "f64" : "f32");
        e.dev_bench_actions(act, as_stream(stream));
        return UUVSIM_OK;
    });
}

int32_t uuvsim_dev_pd_actions(uint64_t h, const UuvPdGains* g, const void* ref6, void* act,
                              uint64_t len, uint64_t stream) {
    return with_engine(h, [&](uuv::Engine& e) {
        const uint64_t want = (uint64_t)e.num_envs() * e.action_dim();
        if (!g || !ref6 || !act || len != want)
            return bad_size("actions", want, e.is_fp64() ? "f64" : "f32");
        e.dev_pd_actions(*g, ref6, act, as_stream(stream));
        return UUVSIM_OK;
    });
}

int32_t uuvsim_dev_states(uint64_t h, void* out, uint64_t len, uint64_t stream) {
    return with_engine(h, [&](uuv::Engine& e) {
        const uint64_t want = (uint64_t)e.num_envs() * 12;
        if (!out || len != want) return bad_size("states", want, e.is_fp64() ? "f64" : "f32");
        e.dev_states(out, as_stream(stream));
        return UUVSIM_OK;
    });
}

int32_t uuvsim_snapshot_size(uint64_t h, uint64_t* out) {
    return with_engine(h, [&](uuv::Engine& e) {
        if (!out) return bad_size("snapshot size", 1, "u64");
        *out = (uint64_t)e.snapshot_bytes();
        return UUVSIM_OK;
    });
}

int32_t uuvsim_snapshot(uint64_t h, void* buf, uint64_t len) {
    return with_engine(h, [&](uuv::Engine& e) {
        const uint64_t want = (uint64_t)e.snapshot_bytes();
        if (!buf || len != want) return bad_size("snapshot", want, "u8");
        e.snapshot(buf);
        return UUVSIM_OK;
    });
}

int32_t uuvsim_restore(uint64_t h, const void* buf, uint64_t len) {
    return with_engine(h, [&](uuv::Engine& e) {
        if (!buf) return bad_size("snapshot", (uint64_t)e.snapshot_bytes(), "u8");
        e.restore(buf, (size_t)len);
        return UUVSIM_OK;
    });
}

int32_t uuvsim_dev_set_final_obs(uint64_t h, void* buf, uint64_t len) {
    return with_engine(h, [&](uuv::Engine& e) {
        const uint64_t want = (uint64_t)e.num_envs() * e.obs_dim();
        if (buf && len != want) return bad_size("final_obs", want, e.is_fp64() ? "f64" : "f32");
        if (buf) {
            if (int32_t c = misaligned("final_obs", buf, 16)) return c;
        }
        e.dev_set_final_obs(buf);
        return UUVSIM_OK;
    });
}

int32_t uuvsim_dev_set_done_f32(uint64_t h, float* buf, uint64_t len) {
    return with_engine(h, [&](uuv::Engine& e) {
        const uint64_t want = (uint64_t)e.num_envs();
        if (buf && len != want) return bad_size("done_f32", want, "f32");
        if (buf) {
            if (int32_t c = misaligned("done_f32", buf, 4)) return c;
        }
        e.dev_set_done_f32(buf);
        return UUVSIM_OK;
    });
}

int32_t uuvsim_dev_set_pdl(uint64_t h, int32_t on) {
    return with_engine(h, [&](uuv::Engine& e) {
        e.dev_set_pdl(on != 0);
        return UUVSIM_OK;
    });
}

int32_t uuvsim_dev_stats(uint64_t h, double* out, uint64_t len, int32_t clear, uint64_t stream) {
    return with_engine(h, [&](uuv::Engine& e) {
        if (!out || len != (uint64_t)uuv::NSTAT) return bad_size("stats", uuv::NSTAT, "f64");
        e.dev_stats(out, clear != 0, as_stream(stream));
        return UUVSIM_OK;
    });
}

int32_t uuvsim_dev_graph_capture(uint64_t h, const void* act, void* obs, void* rew,
                                 uint8_t* done, int8_t* reason, uint32_t n_steps) {
    return with_engine(h, [&](uuv::Engine& e) {
        if (!act || !obs || !rew || !done) return fail(UUVSIM_ERR_SIZE, "null buffer");
        if (n_steps < 1) return fail(UUVSIM_ERR_SIZE, "n_steps must be >= 1");
        // the same alignment contract as uuvsim_dev_step (vector row stores / loads);
        // sizes are those of uuvsim_dev_step (documented in uuvsim.h)
        const size_t esz = e.is_fp64() ? 8 : 4;
        if (int32_t c = misaligned("obs", obs, 16)) return c;
        if (int32_t c = misaligned("actions", act, esz)) return c;
        if (int32_t c = misaligned("rew", rew, esz)) return c;
        e.graph_capture(act, obs, rew, done, reason, (int)n_steps);
        return UUVSIM_OK;
    });
}

int32_t uuvsim_dev_graph_launch(uint64_t h, uint64_t stream) {
    return with_engine(h, [&](uuv::Engine& e) {
        e.graph_launch(as_stream(stream));
        return UUVSIM_OK;
    });
}

int32_t uuvsim_synchronize(uint64_t h) {
    return with_engine(h, [&](uuv::Engine& e) {
        e.synchronize();
        return UUVSIM_OK;
    });
}

}  // extern "C"

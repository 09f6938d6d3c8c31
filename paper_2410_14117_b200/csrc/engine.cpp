// engine.cpp -- host side of the B200 engine (config, validation, device slab,
// launches).  See engine.h for the reference mapping.
#include "engine.h"

#include <algorithm>
#include <array>
#include <climits>
#include <cmath>
#include <cstring>
#include <fstream>
#include <sstream>
#include <thread>

#include <nlohmann/json.hpp>

namespace uuv {

using json = nlohmann::json;

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw RuntimeError(std::string(what) + ": " + cudaGetErrorName(e) + " (" +
                           cudaGetErrorString(e) + ")");
}

// ------------------------------------------------------------------ JSON helpers
namespace {

const json* opt(const json& o, const char* k) {
    if (!o.is_object()) return nullptr;
    auto it = o.find(k);
    if (it == o.end() || it->is_null()) return nullptr;
    return &*it;
}

const json& req(const json& o, const char* k, const char* ctx) {
    const json* v = opt(o, k);
    if (!v) throw ConfigError(std::string("config is not valid JSON: missing field `") + k +
                              "` in " + ctx);
    return *v;
}

double num(const json& v, const char* name) {
    if (!v.is_number())
        throw ConfigError(std::string("config is not valid JSON: field `") + name +
                          "` must be a number");
    return v.get<double>();
}

uint64_t unum(const json& v, const char* name) {
    if (!v.is_number_unsigned())
        throw ConfigError(std::string("config is not valid JSON: field `") + name +
                          "` must be a non-negative integer");
    return v.get<uint64_t>();
}

int64_t inum(const json& v, const char* name) {
    if (!v.is_number_integer())
        throw ConfigError(std::string("config is not valid JSON: field `") + name +
                          "` must be an integer");
    return v.get<int64_t>();
}

template <size_t N>
void fixed(const json& v, const char* name, double* out) {
    if (!v.is_array() || v.size() != N)
        throw ConfigError(std::string("config is not valid JSON: field `") + name +
                          "` must be an array of " + std::to_string(N) + " numbers");
    for (size_t i = 0; i < N; ++i) out[i] = num(v[i], name);
}

// engine.rs:160-172
void square(const json& v, size_t side, const char* name, double* out) {
    if (!v.is_array())
        throw ConfigError(std::string("config is not valid JSON: field `") + name +
                          "` must be a nested array");
    if (v.size() != side)
        throw ConfigError(std::string(name) + " must be " + std::to_string(side) + "x" +
                          std::to_string(side));
    for (size_t i = 0; i < side; ++i) {
        if (!v[i].is_array() || v[i].size() != side)
            throw ConfigError(std::string(name) + " must be " + std::to_string(side) + "x" +
                              std::to_string(side));
        for (size_t j = 0; j < side; ++j) out[i * side + j] = num(v[i][j], name);
    }
}

// engine.rs:174-229 (BaseVehicle::from_doc)
BaseVehicle vehicle_from_doc(const json& d) {
    if (!d.is_object()) throw ConfigError("config is not valid JSON: vehicle must be an object");
    BaseVehicle b;
    b.mass = num(req(d, "mass", "vehicle"), "mass");
    const json& inertia = req(d, "inertia", "vehicle");
    fixed<3>(req(d, "r_g", "vehicle"), "r_g", b.rg);
    fixed<3>(req(d, "r_b", "vehicle"), "r_b", b.rb);
    b.weight = num(req(d, "weight", "vehicle"), "weight");
    b.buoyancy = num(req(d, "buoyancy", "vehicle"), "buoyancy");
    const json& added = req(d, "added_mass", "vehicle");
    const json& dlin = req(d, "damping_linear", "vehicle");
    fixed<6>(req(d, "damping_quadratic", "vehicle"), "damping_quadratic", b.dquad);
    const json& th = req(d, "thrusters", "vehicle");
    if (!th.is_array()) throw ConfigError("config is not valid JSON: thrusters must be a list");
    if (!(b.mass > 0.0)) throw ConfigError("mass must be positive");
    if (b.weight < 0.0 || b.buoyancy < 0.0) throw ConfigError("weight and buoyancy must be >= 0");
    if (th.empty()) throw ConfigError("layout needs at least one thruster");
    for (const json& t : th) {
        std::array<double, 3> p{}, dd{};
        fixed<3>(req(t, "position", "thruster"), "position", p.data());
        fixed<3>(req(t, "direction", "thruster"), "direction", dd.data());
        double kmax = num(req(t, "max_thrust", "thruster"), "max_thrust");
        double n = std::sqrt(dd[0] * dd[0] + dd[1] * dd[1] + dd[2] * dd[2]);
        if (std::fabs(n - 1.0) > 1e-9) throw ConfigError("thruster direction must be unit norm");
        if (!(kmax > 0.0)) throw ConfigError("max_thrust must be positive");
        int code = 1;
        if (const json* c = opt(t, "curve")) {
            if (!c->is_string()) throw ConfigError("config is not valid JSON: curve must be a string");
            std::string s = c->get<std::string>();
            if (s == "quadratic_signed") code = 1;
            else if (s == "linear") code = 0;
            else throw ConfigError("unknown thrust curve \"" + s + "\"");
        }
        b.pos.push_back(p);
        b.dir.push_back(dd);
        b.kmax.push_back(kmax);
        b.curve.push_back(code);
    }
    for (double q : b.dquad)
        if (q < 0.0) throw ConfigError("damping_quadratic components must be >= 0");
    square(inertia, 3, "inertia", b.inertia);
    square(added, 6, "added_mass", b.added);
    square(dlin, 6, "damping_linear", b.dlin);
    if (b.kmax.size() > (size_t)MAX_THR)
        throw ConfigError("at most " + std::to_string(MAX_THR) + " thrusters are supported");
    return b;
}

// M_RB and M_total exactly as engine.rs:234-257 / vehicle.py:64-105
void mass_matrices(const BaseVehicle& v, double* m_rb, double* m_total) {
    const double* rg = v.rg;
    const double s[9] = {0.0, -rg[2], rg[1], rg[2], 0.0, -rg[0], -rg[1], rg[0], 0.0};
    const double nm = -v.mass;
    for (int k = 0; k < 36; ++k) m_rb[k] = 0.0;
    for (int i = 0; i < 3; ++i) {
        m_rb[i * 6 + i] = v.mass;
        for (int j = 0; j < 3; ++j) {
            m_rb[i * 6 + (j + 3)] = nm * s[i * 3 + j];
            m_rb[(i + 3) * 6 + j] = v.mass * s[i * 3 + j];
            m_rb[(i + 3) * 6 + (j + 3)] = v.inertia[i * 3 + j];
        }
    }
    for (int k = 0; k < 36; ++k) m_total[k] = m_rb[k] + v.added[k];
}

// model.rs:38-57
bool cholesky6(const double* m, double* L) {
    for (int k = 0; k < 36; ++k) L[k] = 0.0;
    for (int i = 0; i < 6; ++i)
        for (int j = 0; j <= i; ++j) {
            double s = m[i * 6 + j];
            for (int k = 0; k < j; ++k) s -= L[i * 6 + k] * L[j * 6 + k];
            if (i == j) {
                if (s <= 0.0) return false;
                L[i * 6 + i] = std::sqrt(s);
            } else {
                L[i * 6 + j] = s / L[j * 6 + j];
            }
        }
    return true;
}

// task.rs:46-65
void traj(const TaskCfg& t, double time, double o[4]) {
    double ang = t.omega * time;
    double ca = std::cos(ang), sa = std::sin(ang);
    if (t.kind == 1) {
        o[0] = t.cx + t.radius * ca; o[1] = t.cy + t.radius * sa; o[2] = t.depth;
        o[3] = std::atan2(ca, -sa);
    } else if (t.kind == 2) {
        o[0] = t.cx + t.radius * ca; o[1] = t.cy + t.radius * sa;
        o[2] = t.depth + t.climb * time;
        o[3] = std::atan2(ca, -sa);
    } else {
        o[0] = t.cx + t.scale * ca; o[1] = t.cy + t.scale * (sa * ca); o[2] = t.depth;
        double c2a = ca * ca - sa * sa;
        o[3] = std::atan2(c2a, -sa);
    }
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

// ------------------------------------------------------------------ parsing
void Engine::parse(const std::string& text) {
    json doc;
    try {
        doc = json::parse(text);
    } catch (const std::exception& e) {
        throw ConfigError(std::string("config is not valid JSON: ") + e.what());
    }
    if (!doc.is_object()) throw ConfigError("config is not valid JSON: expected an object");
    seed_ = unum(req(doc, "seed", "config"), "seed");

    // vehicle(s): "vehicles" (extension, mixed batches) > "vehicle" > "vehicle_params"
    if (const json* vs = opt(doc, "vehicles")) {
        if (!vs->is_array() || vs->empty() || vs->size() > (size_t)MAX_VEH)
            throw ConfigError("vehicles must list 1.." + std::to_string(MAX_VEH) + " vehicle documents");
        for (const json& v : *vs) veh_.push_back(vehicle_from_doc(v));
    } else if (const json* v = opt(doc, "vehicle")) {
        veh_.push_back(vehicle_from_doc(*v));
    } else if (const json* path = opt(doc, "vehicle_params")) {
        if (!path->is_string()) throw ConfigError("config is not valid JSON: vehicle_params must be a path");
        std::string p = path->get<std::string>();
        std::ifstream f(p);
        if (!f) throw ConfigError("cannot read vehicle parameter file " + p);
        std::stringstream ss;
        ss << f.rdbuf();
        json vd;
        try {
            vd = json::parse(ss.str());
        } catch (const std::exception& e) {
            throw ConfigError("vehicle parameter file " + p + ": " + e.what());
        }
        veh_.push_back(vehicle_from_doc(vd));
    } else {
        throw ConfigError("config must include 'vehicle' or 'vehicle_params'");
    }

    // task (engine.rs:363-404)
    json t = json::object();
    if (const json* tj = opt(doc, "task")) t = *tj;
    if (const json* k = opt(t, "kind")) {
        if (!k->is_string()) throw ConfigError("config is not valid JSON: task.kind must be a string");
        std::string s = k->get<std::string>();
        if (s == "station_keeping") task_.kind = 0;
        else if (s == "circle") task_.kind = 1;
        else if (s == "helix") task_.kind = 2;
        else if (s == "lemniscate") task_.kind = 3;
        else throw ConfigError("unknown task kind \"" + s + "\"");
    }
    if (const json* v = opt(t, "target")) fixed<6>(*v, "target", task_.target);
    if (const json* v = opt(t, "center")) {
        double c[2];
        fixed<2>(*v, "center", c);
        task_.cx = c[0]; task_.cy = c[1];
    }
    if (const json* v = opt(t, "radius")) task_.radius = num(*v, "radius");
    if (const json* v = opt(t, "angular_rate")) task_.omega = num(*v, "angular_rate");
    if (const json* v = opt(t, "climb_rate")) task_.climb = num(*v, "climb_rate");
    if (const json* v = opt(t, "scale")) task_.scale = num(*v, "scale");
    if (const json* v = opt(t, "depth")) task_.depth = num(*v, "depth");
    if (const json* v = opt(t, "lookahead")) task_.lookahead = (int)std::min<uint64_t>(unum(*v, "lookahead"), 1u << 20);
    if (const json* v = opt(t, "episode_len")) task_.episode_len = inum(*v, "episode_len");
    if (const json* v = opt(t, "control_dt")) task_.control_dt = num(*v, "control_dt");
    if (const json* v = opt(t, "n_substeps")) {
        uint64_t n = unum(*v, "n_substeps");
        if (n > UINT32_MAX) throw ConfigError("config is not valid JSON: n_substeps out of range");
        task_.n_substeps = (int)std::min<uint64_t>(n, INT32_MAX);
    }
    if (!(task_.control_dt > 0.0) || task_.n_substeps < 1 || task_.lookahead < 1 ||
        task_.episode_len < 1)
        throw ConfigError("invalid task timing settings");
    if ((task_.kind == 1 || task_.kind == 2) && !(task_.radius > 0.0))
        throw ConfigError("radius must be positive");
    if (task_.kind == 3 && !(task_.scale > 0.0)) throw ConfigError("scale must be positive");
    if (task_.episode_len > (int64_t)INT32_MAX - task_.lookahead - 2)
        throw ConfigError("episode_len too large for the device step counter (int32)");
    // tracking references come from a per-step table (host fp64 -> device): bound it
    // (2^26 rows = 39 days of simulated time per episode at 0.05 s)
    if (task_.kind != 0 && task_.episode_len + task_.lookahead + 1 > (int64_t)1 << 26)
        throw ConfigError("tracking tasks support episode_len + lookahead up to 67108863 "
                          "(device trajectory table)");

    // batch (engine.rs:406-417)
    json b = json::object();
    if (const json* bj = opt(doc, "batch")) b = *bj;
    m_ = 64;
    if (const json* v = opt(b, "num_envs")) m_ = (int64_t)unum(*v, "num_envs");
    if (m_ < 1) throw ConfigError("batch.num_envs must be >= 1");
    if (m_ > (int64_t)INT32_MAX - BLOCK) throw ConfigError("batch.num_envs too large for one device slab");
    threads = 0;
    if (const json* v = opt(b, "threads")) threads = (int)std::min<uint64_t>(unum(*v, "threads"), 1 << 16);
    if (threads == 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
    if (const json* r = opt(b, "randomization")) {   // engine.rs:108-134
        if (!r->is_object()) throw ConfigError("config is not valid JSON: randomization must be an object");
        ranges_.enabled = true;
        struct { const char* name; double* dst; } rs[] = {
            {"mass", ranges_.mass}, {"added_mass", ranges_.added},
            {"damping_linear", ranges_.dlin}, {"damping_quadratic", ranges_.dquad},
            {"max_thrust", ranges_.thrust}, {"buoyancy_ratio", ranges_.ratio}};
        for (auto& x : rs)
            if (const json* v = opt(*r, x.name)) fixed<2>(*v, x.name, x.dst);
        if (const json* v = opt(*r, "rb_offset")) ranges_.rb_offset = num(*v, "rb_offset");
        if (const json* v = opt(*r, "per_episode")) {
            if (!v->is_boolean()) throw ConfigError("config is not valid JSON: per_episode must be a bool");
            ranges_.per_episode = v->get<bool>();
        }
        for (auto& x : rs)
            if (!(0.0 < x.dst[0] && x.dst[0] <= x.dst[1]))
                throw ConfigError(std::string("range ") + x.name + " must satisfy 0 < lo <= hi");
        if (ranges_.rb_offset < 0.0) throw ConfigError("rb_offset must be >= 0");
    }
    // extensions: global env offset (sharding) and contiguous vehicle mix
    if (const json* v = opt(b, "env_offset")) env_offset_ = unum(*v, "env_offset");
    if (const json* v = opt(b, "vehicle_mix")) {
        if (!v->is_array() || v->size() != veh_.size())
            throw ConfigError("batch.vehicle_mix must give one env count per vehicle");
        for (const json& c : *v) mix_.push_back((int64_t)unum(c, "vehicle_mix"));
    }
    if (veh_.size() > 1 && mix_.empty())
        throw ConfigError("several vehicles need batch.vehicle_mix");
    if (!mix_.empty()) {   // the global mix must cover this slab's envs
        int64_t total = 0;
        for (int64_t c : mix_) total += c;
        if (total < (int64_t)env_offset_ + m_)
            throw ConfigError("batch.vehicle_mix covers " + std::to_string(total) +
                              " envs, fewer than env_offset + num_envs = " +
                              std::to_string((int64_t)env_offset_ + m_));
    }
    // device section (extension; unknown keys are ignored like serde)
    if (const json* d = opt(doc, "device")) {
        if (const json* v = opt(*d, "precision")) {
            std::string s = v->is_string() ? v->get<std::string>() : "";
            if (s == "fp32") fp64_ = false;
            else if (s == "fp64") fp64_ = true;
            else throw ConfigError("device.precision must be \"fp32\" or \"fp64\"");
        }
        if (const json* v = opt(*d, "index")) device_ = (int)inum(*v, "device.index");
        if (const json* v = opt(*d, "stats")) {
            if (!v->is_boolean()) throw ConfigError("device.stats must be a bool");
            stats_on_ = v->get<bool>();
        }
        if (const json* v = opt(*d, "pair")) {
            std::string s = v->is_string() ? v->get<std::string>() : "";
            if (s == "auto") pair_mode_ = -1;
            else if (s == "on") pair_mode_ = 1;
            else if (s == "off") pair_mode_ = 0;
            else throw ConfigError("device.pair must be \"auto\", \"on\" or \"off\"");
        }
        if (const json* v = opt(*d, "tma")) {
            if (!v->is_boolean()) throw ConfigError("device.tma must be a bool");
            tma_mode_ = v->get<bool>() ? 1 : 0;
        }
        if (const json* v = opt(*d, "stage_obs")) {
            std::string s = v->is_string() ? v->get<std::string>() : "";
            if (s == "auto") stage_mode_ = -1;
            else if (s == "on") stage_mode_ = 1;
            else if (s == "off") stage_mode_ = 0;
            else throw ConfigError("device.stage_obs must be \"auto\", \"on\" or \"off\"");
        }
        if (const json* v = opt(*d, "host_io")) {
            std::string s = v->is_string() ? v->get<std::string>() : "";
            if (s == "auto") host_io_ = -1;
            else if (s == "copy") host_io_ = 0;
            else if (s == "mapped") host_io_ = 1;
            else throw ConfigError("device.host_io must be \"auto\", \"copy\" or \"mapped\"");
        }
        if (const json* v = opt(*d, "band64")) {
            if (!v->is_boolean()) throw ConfigError("device.band64 must be a bool");
            band64_ = v->get<bool>();
        }
        if (const json* v = opt(*d, "band_margin")) band_margin_ = num(*v, "device.band_margin");
        if (const json* v = opt(*d, "band_tail")) {   // A/B: misses stay fp32
            if (!v->is_boolean()) throw ConfigError("device.band_tail must be a bool");
            band_tail_ = v->get<bool>();
        }
        if (const json* v = opt(*d, "band_per")) band_per_cfg_ = v->get<int64_t>();   // A/B only
        if (const json* v = opt(*d, "band_rege")) band_rege_ = v->get<bool>() ? 1 : 0;
        if (const json* v = opt(*d, "band_refop")) {
            if (!v->is_boolean()) throw ConfigError("device.band_refop must be a bool");
            band_refop_ = v->get<bool>() ? 1 : 0;
        }
        if (const json* v = opt(*d, "band_order")) {   // "band_first" | "main_first" (A/B)
            std::string s = v->is_string() ? v->get<std::string>() : "";
            if (s == "band_first") band_order_ = 0;
            else if (s == "main_first") band_order_ = 1;
            else throw ConfigError("device.band_order must be \"band_first\" or \"main_first\"");
        }
        if (const json* v = opt(*d, "band_stream")) {   // "side" (concurrent) | "same" (A/B)
            std::string s = v->is_string() ? v->get<std::string>() : "";
            if (s == "side") band_same_ = false;
            else if (s == "same") band_same_ = true;
            else if (s == "none") band_none_ = true;   // A/B: no band kernel (bookkeeping only)
            else throw ConfigError("device.band_stream must be \"side\", \"same\" or \"none\"");
        }
        // without a band kernel nobody would step the predicted candidates: "none"
        // only measures the step kernel's bookkeeping, with the predictor off
        if (band_none_ && !(band_margin_ >= -1e30 && band_margin_ < -1.0))
            throw ConfigError("device.band_stream \"none\" (A/B only) needs device.band_margin < -1 "
                              "(no band candidates)");
        if (const json* v = opt(*d, "pattern")) {
            std::string s = v->is_string() ? v->get<std::string>() : "";
            if (s == "dense") force_dense_ = true;
            else if (s != "auto") throw ConfigError("device.pattern must be \"auto\" or \"dense\"");
        }
    } else {
        cudaGetDevice(&device_);
    }

    // engine.rs:258 -- M_RB + M_A must be positive definite (checked before any device work)
    for (const BaseVehicle& v : veh_) {
        double m_rb[36], m_total[36], L[36];
        mass_matrices(v, m_rb, m_total);
        if (!cholesky6(m_total, L))
            throw ConfigError("M_RB + M_A is not positive definite: matrix is not positive definite");
    }
    obs_dim_ = task_.kind == 0 ? 12 : 6 * task_.lookahead + 6;
    n_act_ = 0;
    for (auto& v : veh_) n_act_ = std::max<int>(n_act_, (int)v.kmax.size());
}

template <> EngineP<float>& Engine::P<float>() { return *pf_; }
template <> EngineP<double>& Engine::P<double>() { return *pd_; }

// One base vehicle in precision T (engine.rs:234-286 / vehicle.py:64-112 in fp64,
// then rounded): M_total, its Cholesky factor, the Fossen-pattern dt M^-1, damping,
// restoring terms, allocation columns and the fp64 originals for DR redraws.
template <class T> void Engine::fill_vehicle(const BaseVehicle& v, VehP<T>& V) const {
    std::memset(&V, 0, sizeof(V));
    double m_rb[36], m_total[36], L[36];
    mass_matrices(v, m_rb, m_total);
    if (!cholesky6(m_total, L))
        throw ConfigError("M_RB + M_A is not positive definite: matrix is not positive definite");
    for (int k = 0; k < 36; ++k) {
        V.mtot[k] = (T)m_total[k];
        V.mrb[k] = (T)m_rb[k];
        V.ma[k] = (T)v.added[k];
        V.chol[k] = (T)L[k];
        V.dlin[k] = (T)v.dlin[k];
        V.mrb64[k] = m_rb[k];
        V.ma64[k] = v.added[k];
    }
    for (int i = 0; i < 6; ++i) {
        V.chol_inv[i] = (T)(1.0 / L[i * 6 + i]);
        V.dquad[i] = (T)v.dquad[i];
    }
    {   // sub_dt * M_total^-1 on the Fossen pattern (2x2 blocks {0,4}, {1,3}; 2; 5),
        // in fp64 from the fp64 matrix, then rounded (fp32 product kernel)
        const double dt = (double)(T)(task_.control_dt / (double)task_.n_substeps);
        const int blk[2][2] = {{0, 4}, {1, 3}};
        for (const auto& bk : blk) {
            const int i = bk[0], j = bk[1];
            const double a = m_total[i * 6 + i], b = m_total[i * 6 + j];
            const double c = m_total[j * 6 + i], d = m_total[j * 6 + j];
            const double id = dt / (a * d - b * c);
            V.kdt[i * 6 + i] = (T)(d * id);
            V.kdt[i * 6 + j] = (T)(-b * id);
            V.kdt[j * 6 + i] = (T)(-c * id);
            V.kdt[j * 6 + j] = (T)(a * id);
        }
        V.kdt[2 * 6 + 2] = (T)(dt / m_total[2 * 6 + 2]);
        V.kdt[5 * 6 + 5] = (T)(dt / m_total[5 * 6 + 5]);
    }
    V.weight = (T)v.weight;
    V.buoyancy = (T)v.buoyancy;
    for (int k = 0; k < 3; ++k) {
        V.rg[k] = (T)v.rg[k];
        V.rb[k] = (T)v.rb[k];
        V.rb64[k] = v.rb[k];
    }
    V.weight64 = v.weight;
    V.wb = (T)(v.weight - v.buoyancy);
    for (int k = 0; k < 3; ++k) V.hm[k] = (T)(v.weight * v.rg[k] - v.buoyancy * v.rb[k]);
    const int n = (int)v.kmax.size();
    V.n_thr = n;
    for (int i = 0; i < n; ++i) {   // thrusters.py:81-94 / engine.rs:260-271
        const double px = v.pos[i][0], py = v.pos[i][1], pz = v.pos[i][2];
        const double dx = v.dir[i][0], dy = v.dir[i][1], dz = v.dir[i][2];
        V.alloc[0 * MAX_THR + i] = (T)dx;
        V.alloc[1 * MAX_THR + i] = (T)dy;
        V.alloc[2 * MAX_THR + i] = (T)dz;
        V.alloc[3 * MAX_THR + i] = (T)(py * dz - pz * dy);
        V.alloc[4 * MAX_THR + i] = (T)(pz * dx - px * dz);
        V.alloc[5 * MAX_THR + i] = (T)(px * dy - py * dx);
        V.kmax[i] = (T)v.kmax[i];
        V.curve[i] = v.curve[i];
    }
}

template <class T> void Engine::fill_params(EngineP<T>& p) {
    std::memset(&p, 0, sizeof(p));
    for (size_t vi = 0; vi < veh_.size(); ++vi) fill_vehicle(veh_[vi], p.veh[vi]);
    TaskP<T>& tk = p.task;
    for (int k = 0; k < 6; ++k) tk.target[k] = (T)task_.target[k];
    tk.sub_dt = (T)(task_.control_dt / (double)task_.n_substeps);
    tk.div_radius = (T)10.0;   // tasks.py:39
    tk.kind = task_.kind;
    tk.lookahead = task_.lookahead;
    tk.n_substeps = task_.n_substeps;
    tk.episode_len = (int32_t)task_.episode_len;
    tk.obs_dim = obs_dim_;
    if (task_.kind == 0) {
        tk.spawn[0] = task_.target[0]; tk.spawn[1] = task_.target[1]; tk.spawn[2] = task_.target[2];
        tk.ref_psi = task_.target[5];
    } else {
        double r[4];
        traj(task_, 0.0, r);
        tk.spawn[0] = r[0]; tk.spawn[1] = r[1]; tk.spawn[2] = r[2];
        tk.ref_psi = r[3];
    }
    tk.traj = reinterpret_cast<const V4<T>*>(traj_);
    RangesP& R = p.ranges;
    R.enabled = ranges_.enabled;
    R.per_episode = ranges_.per_episode;
    const double* lo_hi[5] = {ranges_.mass, ranges_.added, ranges_.dlin, ranges_.dquad, ranges_.thrust};
    for (int i = 0; i < 5; ++i) {
        R.log_lo[i] = std::log(lo_hi[i][0]);
        R.log_hi[i] = std::log(lo_hi[i][1]);
    }
    R.rb_offset = ranges_.rb_offset;
    R.ratio[0] = ranges_.ratio[0];
    R.ratio[1] = ranges_.ratio[1];
    p.seed = seed_;
    p.env_offset = env_offset_;
    p.mix_bound0 = mix_.empty() ? INT64_MAX : mix_[0];
    p.n_env = (int32_t)m_;
    p.n_veh = (int32_t)veh_.size();
    p.act_dim = n_act_;
    p.stats_on = stats_on_ ? 1 : 0;
    p.stats = stats_part_;
    p.vpack = d_vpack_;
    p.final_obs = nullptr;
    p.done_f32 = nullptr;
    p.io_f64 = fp64_ ? 1 : 0;   // device face: engine precision; host ABI: set per launch
    p.veh64 = veh64_.empty() ? nullptr : veh64_.data();
    p.sub_dt64 = task_.control_dt / (double)task_.n_substeps;
    p.veh64_dev = d_veh64_;
    p.err_flag = d_err_;
    p.band_theta = band_grid_ > 0 ? BAND_THETA : INFINITY;
    p.band_exit_theta = band_tail_ ? p.band_theta : INFINITY;
    p.band_kdt = (float)task_.control_dt;
    p.band_margin = (float)(band_margin_ >= -1e30 ? band_margin_
                                                   : 0.01 + 8.0 * task_.control_dt * task_.control_dt);
    p.band_per = band_per_;
    p.band_grid = band_grid_;
    p.stats_band = stats_part_ + (size_t)nblk_ * NSTAT;
    p.band_ctr = reinterpret_cast<unsigned long long*>(d_band_f_);   // 2 counters, then the flags
    p.band_f = d_band_f_ ? reinterpret_cast<uint8_t*>(d_band_f_) + 256 : nullptr;
    p.band_inv_n = 1.0 / (double)m_;
    p.band_side = (band_same_ || band_none_) ? nullptr : band_side_;
    p.band_same = band_same_ ? 1 : 0;
    // step kernel first once the batch outgrows the band chain's latency
    p.band_main_first = band_order_ == 1 ? 1 : 0;
    // register-resident fp64 vehicle constants in the band kernel while it is the
    // step's critical path (small batches; device.band_rege overrides, A/B)
    p.band_rege = band_rege_ >= 0 ? band_rege_ : (m_ <= 8192 ? 1 : 0);
    // reference-order band steps for long control steps (>= 0.1 s): there an env
    // can pitch from inside the band to the clamp within one step, where the
    // dynamics amplify rounding differences by ~1e11 and only the reference's own
    // operation order agrees with it; device.band_refop overrides
    p.band_refop = band_refop_ >= 0 ? band_refop_ : (task_.control_dt >= 0.1 - 1e-12 ? 1 : 0);
    p.band_ev[0] = band_ev_[0];
    p.band_ev[1] = band_ev_[1];
    // staged rows pay off for tracking rows (144 B); station rows (48 B) are
    // already three 128-bit stores per env (measured)
    const bool stage_ok = obs_dim_ <= MAX_STAGE_DIM;
    p.stage_obs = stage_ok && (stage_mode_ == 1 || (stage_mode_ < 0 && obs_dim_ > 12)) ? 1 : 0;
    // persistent TMA-pipelined paired kernel (station, no DR, device face)
    p.persist_blocks = ((tma_mode_ == 1 || (tma_mode_ < 0 && UUV_TMA_PAIR)) && pair_ && task_.kind == 0 &&
                        !ranges_.enabled && !fp64_ && m_ >= 2 * BLOCK)
                           ? sm_count_ * TMA_MIN_BLOCKS : 0;

    // device buffers carved from the arena
    char* a = static_cast<char*>(arena_);
    size_t off = 0;
    auto carve = [&](size_t bytes) { void* q = a + off; off += align256(bytes); return q; };
    const size_t N = (size_t)m_;
    p.s0 = (V4<T>*)carve(N * sizeof(V4<T>));
    p.s1 = (V4<T>*)carve(N * sizeof(V4<T>));
    p.s2 = (V4<T>*)carve(N * sizeof(V4<T>));
    p.step = (int32_t*)carve(N * 4);
    p.ep_ret = (float*)carve(N * 4);
    p.reset_ctr = (uint64_t*)carve(N * 8);
    p.param_ctr = (uint64_t*)carve(N * 8);
    p.seed_dev = (uint64_t*)carve(8);
    if (ranges_.enabled) {
        p.dr0 = (V4<T>*)carve(N * sizeof(V4<T>));
        p.dr1 = (V4<T>*)carve(N * sizeof(V4<T>));
        p.dr2 = (V2<T>*)carve(N * sizeof(V2<T>));
        // the exact fp64 record beside the fp32 one, read only by the band replay
        if (!fp64_ && band64_) p.dr64 = (V2<double>*)carve(N * 5 * sizeof(V2<double>));
    }
    if (off > arena_bytes_) throw RuntimeError("internal: arena too small");
    arena_used_ = off;
}

// Structure test for the PatFossen kernels (uuv_model.cuh): every entry outside
// {diag, (0,4), (4,0), (1,3), (3,1)} of M_RB and M_A is exactly zero, D_lin is
// diagonal and r_g lies on the body z axis -- for every vehicle in the batch.
bool Engine::check_fossen() const {
    auto in_m = [](int i, int j) {
        return i == j || (i == 0 && j == 4) || (i == 4 && j == 0) || (i == 1 && j == 3) ||
               (i == 3 && j == 1);
    };
    for (const BaseVehicle& v : veh_) {
        double m_rb[36], m_total[36];
        mass_matrices(v, m_rb, m_total);
        if (v.rg[0] != 0.0 || v.rg[1] != 0.0) return false;
        for (int i = 0; i < 6; ++i)
            for (int j = 0; j < 6; ++j) {
                if (!in_m(i, j) && (m_rb[i * 6 + j] != 0.0 || v.added[i * 6 + j] != 0.0))
                    return false;
                if (i != j && v.dlin[i * 6 + j] != 0.0) return false;
            }
    }
    return true;
}

void Engine::activate() const { cuda_check(cudaSetDevice(device_), "cudaSetDevice"); }

void Engine::allocate() {
    activate();
    cudaDeviceProp prop{};
    cuda_check(cudaGetDeviceProperties(&prop, device_), "cudaGetDeviceProperties");
    device_name_ = prop.name;
    sm_count_ = prop.multiProcessorCount;
    const size_t N = (size_t)m_;
    const size_t sT = fp64_ ? 8 : 4;
    size_t bytes = 3 * align256(N * 4 * sT) + 2 * align256(N * 4) + 2 * align256(N * 8) + 256;
    if (ranges_.enabled) bytes += 2 * align256(N * 4 * sT) + align256(N * 2 * sT);
    if (ranges_.enabled && !fp64_ && band64_) bytes += align256(N * 80);
    size_t free_b = 0, total_b = 0;
    cuda_check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
    // the host-ABI staging buffers are allocated on first use (ensure_staging):
    // a device-face user (uuvsim_dev_*) never pays for them
    if (bytes > free_b)
        throw ConfigError("batch.num_envs needs " + std::to_string(bytes >> 20) +
                          " MiB of device memory, " + std::to_string(free_b >> 20) + " MiB free");
    arena_bytes_ = bytes;
    cuda_check(cudaMalloc(&arena_, bytes), "cudaMalloc(state)");
    cuda_check(cudaMemset(arena_, 0, bytes), "cudaMemset(state)");
    nblk_ = (int)((m_ + BLOCK - 1) / BLOCK);
    // per-block statistics partials: the step kernel's blocks, then the band
    // replay kernel's (fp32 engines with band64)
    // band kernel: chunks of n/256 envs, 2,048 to BAND_MAX_PER (a multiple of
    // 2,048): a few dozen candidates per block (one pass), spread over the SMs
    if (!fp64_ && band64_) {
        int64_t per = std::min<int64_t>(BAND_MAX_PER, std::max<int64_t>(2048, (m_ / 256 + 2047) / 2048 * 2048));
        if (band_per_cfg_ > 0) per = std::min<int64_t>(BAND_MAX_PER, (band_per_cfg_ + 15) / 16 * 16);
        band_per_ = (int)per;
        band_grid_ = (int)((m_ + per - 1) / per);
    }
    // per-block statistics partials: the step kernel's blocks, then the band kernel's
    nstat_blk_ = nblk_ + band_grid_;
    cuda_check(cudaMalloc(&stats_part_, (size_t)nstat_blk_ * NSTAT * sizeof(double)), "cudaMalloc(stats)");
    cuda_check(cudaMemset(stats_part_, 0, (size_t)nstat_blk_ * NSTAT * sizeof(double)), "cudaMemset(stats)");
    if (band_grid_ > 0) {
        const size_t bytes = 256 + ((size_t)m_ + 15) / 16 * 16;   // counters, then one byte per env
        cuda_check(cudaMalloc(&d_band_f_, bytes), "cudaMalloc(band flags)");
        cuda_check(cudaMemset(d_band_f_, 0, bytes), "cudaMemset(band flags)");
        // highest priority: as step-kernel blocks retire, the band kernel's small
        // blocks take the freed room before the step kernel's next wave
        int lo = 0, hi = 0;
        cuda_check(cudaDeviceGetStreamPriorityRange(&lo, &hi), "stream priorities");
        cuda_check(cudaStreamCreateWithPriority(&band_side_, cudaStreamNonBlocking, hi),
                   "cudaStreamCreate(band)");
        for (auto& ev : band_ev_)
            cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate(band)");
    }
    cuda_check(cudaMalloc(&d_stats_out_, NSTAT * sizeof(double)), "cudaMalloc(stats_out)");
    if (task_.kind != 0) {   // reference trajectory by step index (task.rs:67-74)
        const int64_t len = task_.episode_len + task_.lookahead + 1;
        std::vector<double> tab((size_t)len * 4);
        for (int64_t i = 0; i < len; ++i) traj(task_, (double)i * task_.control_dt, &tab[(size_t)i * 4]);
        if (fp64_) {
            cuda_check(cudaMalloc(&traj_, tab.size() * 8), "cudaMalloc(traj)");
            cuda_check(cudaMemcpy(traj_, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice), "traj");
        } else {
            std::vector<float> tf(tab.begin(), tab.end());
            cuda_check(cudaMalloc(&traj_, tf.size() * 4), "cudaMalloc(traj)");
            cuda_check(cudaMemcpy(traj_, tf.data(), tf.size() * 4, cudaMemcpyHostToDevice), "traj");
        }
    }
    cuda_check(cudaMalloc(&d_flag_, sizeof(int)), "cudaMalloc(flag)");
    if (ranges_.enabled && ranges_.per_episode) {   // rejected-resample flag, mapped page-locked
        cuda_check(cudaHostAlloc((void**)&h_err_, sizeof(int32_t), cudaHostAllocMapped), "cudaHostAlloc(err)");
        *h_err_ = 0;
        cuda_check(cudaHostGetDevicePointer((void**)&d_err_, (void*)h_err_, 0), "err flag alias");
    }
    {   // fp32 register pack per vehicle (uuv_model.cuh RegPack layout)
        std::vector<float> pk((size_t)MAX_VEH * PACK_F4 * 4, 0.0f);
        for (size_t vi = 0; vi < veh_.size(); ++vi) {
            const BaseVehicle& v = veh_[vi];
            double m_rb[36], m_total[36], L[36];
            mass_matrices(v, m_rb, m_total);
            cholesky6(m_total, L);
            const double dt = task_.control_dt / (double)task_.n_substeps;
            const double vals[40] = {
                m_total[0], m_total[4], m_total[7], m_total[9],
                m_total[14], m_total[19], m_total[21], m_total[24],
                m_total[28], m_total[35], L[3 * 6 + 1], L[4 * 6 + 0],
                1.0 / L[0], 1.0 / L[7], 1.0 / L[14], 1.0 / L[21],
                1.0 / L[28], 1.0 / L[35], v.dquad[0], v.dquad[1],
                v.dquad[2], v.dquad[3], v.dquad[4], v.dquad[5],
                v.dlin[0], v.dlin[7], v.dlin[14], v.dlin[21],
                v.dlin[28], v.dlin[35], v.weight - v.buoyancy,
                v.weight * v.rg[0] - v.buoyancy * v.rb[0],
                v.weight * v.rg[1] - v.buoyancy * v.rb[1],
                v.weight * v.rg[2] - v.buoyancy * v.rb[2], dt, 0.0,
                0.636619772367581343, 0.159154943091895335769, -1.9515295891e-4,
                2.443315711809948e-5};
            for (int k = 0; k < 40; ++k) pk[vi * PACK_F4 * 4 + k] = (float)vals[k];
        }
        cuda_check(cudaMalloc(&d_vpack_, pk.size() * sizeof(float)), "cudaMalloc(vpack)");
        cuda_check(cudaMemcpy(d_vpack_, pk.data(), pk.size() * sizeof(float), cudaMemcpyHostToDevice),
                   "vpack");
    }
    cuda_check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaEventCreateWithFlags(&dev_ev_, cudaEventDisableTiming), "cudaEventCreate");
}

// host-ABI staging (f64 action / obs / reward rows, fp32 twins, done / reason
// bytes), allocated the first time a host-face call needs it
void Engine::ensure_staging() {
    if (d_act64_) return;
    const size_t N = (size_t)m_;
    const size_t need = (align256(N * n_act_ * 8) + align256(N * obs_dim_ * 8) + align256(N * 8)) *
                            (fp64_ ? 1 : 2) + 2 * align256(N);
    size_t free_b = 0, total_b = 0;
    cuda_check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
    if (need > free_b)
        throw ConfigError("the host-ABI staging for batch.num_envs needs " +
                          std::to_string(need >> 20) + " MiB of device memory, " +
                          std::to_string(free_b >> 20) +
                          " MiB free (the device face uuvsim_dev_* needs none)");
    try {
        cuda_check(cudaMalloc(&d_act64_, N * n_act_ * 8), "cudaMalloc(abi act)");
        cuda_check(cudaMalloc(&d_obs64_, N * obs_dim_ * 8), "cudaMalloc(abi obs)");
        cuda_check(cudaMalloc(&d_rew64_, N * 8), "cudaMalloc(abi rew)");
        if (fp64_) {
            d_actT_ = d_act64_;
            d_obsT_ = d_obs64_;
            d_rewT_ = d_rew64_;
        } else {
            cuda_check(cudaMalloc(&d_actT_, N * n_act_ * 4), "cudaMalloc(abi act32)");
            cuda_check(cudaMalloc(&d_obsT_, N * obs_dim_ * 4), "cudaMalloc(abi obs32)");
            cuda_check(cudaMalloc(&d_rewT_, N * 4), "cudaMalloc(abi rew32)");
        }
        cuda_check(cudaMalloc(&d_done_, N), "cudaMalloc(abi done)");
        cuda_check(cudaMalloc(&d_reason_, N), "cudaMalloc(abi reason)");
    } catch (...) {
        free_staging();
        throw;
    }
    staging_bytes_ = need;
}

// [N][12] f64 state rows for the host state accessors
void Engine::ensure_pack() {
    if (d_pack_) return;
    cuda_check(cudaMalloc(&d_pack_, (size_t)m_ * 12 * 8), "cudaMalloc(abi pack)");
}

void Engine::free_staging() {
    if (!fp64_) {
        void* t[] = {d_actT_, d_obsT_, d_rewT_};
        for (void* b : t)
            if (b) cudaFree(b);
    }
    void* bufs[] = {d_act64_, d_obs64_, d_rew64_, d_done_, d_reason_};
    for (void* b : bufs)
        if (b) cudaFree(b);
    d_actT_ = d_obsT_ = d_rewT_ = nullptr;
    d_act64_ = d_obs64_ = d_rew64_ = nullptr;
    d_done_ = nullptr;
    d_reason_ = nullptr;
    staging_bytes_ = 0;
}

Engine::Engine(const std::string& text) {
    parse(text);
    fossen_ = !force_dense_ && check_fossen();
    // two envs per thread pays off once the paired grid still fills every SM
    const bool pair_ok = fossen_ && !fp64_ && !ranges_.enabled;
    pair_ = pair_ok && (pair_mode_ == 1 || (pair_mode_ < 0 && m_ >= PAIR_AUTO_MIN_ENVS));
    try {
        allocate();
        if (!fp64_) {   // fp64 base vehicles: band-kernel parameters and step-kernel tail
            veh64_.assign(MAX_VEH, VehP<double>{});
            for (size_t vi = 0; vi < veh_.size(); ++vi) fill_vehicle(veh_[vi], veh64_[vi]);
            cuda_check(cudaMalloc(&d_veh64_, MAX_VEH * sizeof(VehP<double>)), "cudaMalloc(veh64)");
            cuda_check(cudaMemcpy(d_veh64_, veh64_.data(), MAX_VEH * sizeof(VehP<double>),
                                  cudaMemcpyHostToDevice), "veh64");
        }
        if (fp64_) {
            pd_ = std::make_unique<EngineP<double>>();
            fill_params(*pd_);
        } else {
            pf_ = std::make_unique<EngineP<float>>();
            fill_params(*pf_);
        }
        init_randomization();
        reset_host(seed_, nullptr);
    } catch (...) {
        release();
        throw;
    }
}

Engine::~Engine() { release(); }

void Engine::release() {
    if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
    graph_exec_ = nullptr;
    for (AbiGraph& g : abi_graphs_) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        g = AbiGraph{};
    }
    free_staging();
    void* bufs[] = {arena_, traj_, stats_part_, d_pack_, d_flag_, d_stats_out_, d_vpack_, d_veh64_,
                    d_band_f_};
    for (void* b : bufs)
        if (b) cudaFree(b);
    d_veh64_ = nullptr;
    d_band_f_ = nullptr;
    if (h_err_) cudaFreeHost((void*)h_err_);
    h_err_ = nullptr;
    d_err_ = nullptr;
    if (band_side_) cudaStreamDestroy(band_side_);
    band_side_ = nullptr;
    for (auto& ev : band_ev_) {
        if (ev) cudaEventDestroy(ev);
        ev = nullptr;
    }
    arena_ = traj_ = nullptr;
    stats_part_ = d_pack_ = d_stats_out_ = nullptr;
    d_flag_ = nullptr;
    d_vpack_ = nullptr;
    if (stream_) cudaStreamDestroy(stream_);
    stream_ = nullptr;
    if (dev_ev_) cudaEventDestroy(dev_ev_);
    dev_ev_ = nullptr;
}

void Engine::init_randomization() {   // engine.rs:440-458: per-env sample at create
    if (!ranges_.enabled) return;
    const int big = INT_MAX;
    cuda_check(cudaMemcpyAsync(d_flag_, &big, sizeof(int), cudaMemcpyHostToDevice, stream_), "flag");
    if (fp64_) cuda_check(Launch<double>::dr_init(*pd_, d_flag_, stream_), "dr_init");
    else cuda_check(Launch<float>::dr_init(*pf_, d_flag_, stream_), "dr_init");
    int bad = INT_MAX;
    cuda_check(cudaMemcpyAsync(&bad, d_flag_, sizeof(int), cudaMemcpyDeviceToHost, stream_), "flag");
    cuda_check(cudaStreamSynchronize(stream_), "dr_init sync");
    if (bad != INT_MAX)
        throw ConfigError("env " + std::to_string(bad) +
                          ": randomized parameters invalid: M_RB + M_A is not positive definite: "
                          "matrix is not positive definite");
}

// ------------------------------------------------------------------ host ABI face
template <class T> void Engine::reset_host_T(uint64_t seed, double* obs) {
    if (obs) ensure_staging();
    EngineP<T>& p = P<T>();
    p.seed = seed;
    const size_t n_obs = (size_t)m_ * obs_dim_;
    cuda_check(Launch<T>::reset(p, obs ? (T*)d_obsT_ : nullptr, stream_), "reset");
    if (obs) {
        if (!fp64_) cuda_check(Launch<T>::to_f64((T*)d_obsT_, d_obs64_, n_obs, stream_), "obs cvt");
        cuda_check(cudaMemcpyAsync(obs, d_obs64_, n_obs * 8, cudaMemcpyDeviceToHost, stream_),
                   "reset D2H");
    }
    cuda_check(cudaStreamSynchronize(stream_), "reset sync");
}

void Engine::reset_host(uint64_t seed, double* obs) {
    activate();
    wait_device_face();
    if (fp64_) reset_host_T<double>(seed, obs);
    else reset_host_T<float>(seed, obs);
}

// uuvsim_step: H2D f64 actions -> one fused step reading f64 actions and writing
// f64 obs/reward directly (io_f64) -> D2H outputs
template <class T>
void Engine::enqueue_step_host(const double* act, double* obs, double* rew, uint8_t* done,
                               int8_t* reason) {
    const size_t N = (size_t)m_, n_act = N * n_act_, n_obs = N * obs_dim_;
    cuda_check(cudaMemcpyAsync(d_act64_, act, n_act * 8, cudaMemcpyHostToDevice, stream_),
               "step H2D");
    EngineP<T>& p = P<T>();
    p.io_f64 = 1;
    void* const fo = p.final_obs;   // terminal obs, fp32 done, programmatic launch: device face only
    float* const df = p.done_f32;
    const int32_t pdl = p.pdl;
    p.final_obs = nullptr;
    p.done_f32 = nullptr;
    p.pdl = 0;
    const cudaError_t e = Launch<T>::step(p, task_.kind != 0, ranges_.enabled, fossen_, pair_,
                                          d_act64_, d_obs64_, d_rew64_, d_done_, d_reason_,
                                          stream_);
    p.io_f64 = fp64_ ? 1 : 0;
    p.final_obs = fo;
    p.done_f32 = df;
    p.pdl = pdl;
    cuda_check(e, "step");
    cuda_check(cudaMemcpyAsync(obs, d_obs64_, n_obs * 8, cudaMemcpyDeviceToHost, stream_), "obs D2H");
    cuda_check(cudaMemcpyAsync(rew, d_rew64_, N * 8, cudaMemcpyDeviceToHost, stream_), "rew D2H");
    cuda_check(cudaMemcpyAsync(done, d_done_, N, cudaMemcpyDeviceToHost, stream_), "done D2H");
    if (reason)
        cuda_check(cudaMemcpyAsync(reason, d_reason_, N, cudaMemcpyDeviceToHost, stream_), "reason D2H");
}

namespace {
// driver query of a host pointer: page-locked?  device alias?  allocation id?
// (cuPointerGetAttributes through the runtime's entry-point table, so the
// library has no link-time dependency on libcuda)
struct HostBuf {
    bool locked = false;
    void* dev = nullptr;
    unsigned long long id = 0;
};
using PtrAttrsFn = CUresult (*)(unsigned, CUpointer_attribute*, void**, CUdeviceptr);

PtrAttrsFn ptr_attrs_fn() {
    static PtrAttrsFn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuPointerGetAttributes", &f, cudaEnableDefault, &q) !=
                cudaSuccess || q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            f = nullptr;
        }
        return reinterpret_cast<PtrAttrsFn>(f);
    }();
    return fn;
}

HostBuf host_buf(const void* ptr) {
    HostBuf b;
    if (!ptr) {
        b.locked = true;
        return b;
    }
    PtrAttrsFn fn = ptr_attrs_fn();
    if (!fn) return b;
    CUpointer_attribute at[3] = {CU_POINTER_ATTRIBUTE_MEMORY_TYPE,
                                 CU_POINTER_ATTRIBUTE_DEVICE_POINTER,
                                 CU_POINTER_ATTRIBUTE_BUFFER_ID};
    unsigned int mt = 0;
    CUdeviceptr dp = 0;
    unsigned long long id = 0;
    void* data[3] = {&mt, &dp, &id};
    if (fn(3, at, data, (CUdeviceptr)ptr) != CUDA_SUCCESS) return b;
    b.locked = mt == CU_MEMORYTYPE_HOST;
    b.dev = b.locked ? (void*)dp : nullptr;
    b.id = id;
    return b;
}
}  // namespace

// host_io "mapped": the step kernel reads the f64 actions and writes the f64
// obs / reward / done / reason straight through the caller's page-locked
// buffers over the host link (zero-copy): one launch + one sync per step,
// no DMA engine round trips.  Observation rows are staged in shared memory so
// each block writes one contiguous span.  The caller checked that every buffer
// is mapped page-locked memory (dev_io_ holds the device aliases).
template <class T>
void Engine::enqueue_step_mapped() {
    EngineP<T>& p = P<T>();
    const int32_t io = p.io_f64, stage = p.stage_obs, pdl = p.pdl;
    void* const fo = p.final_obs;
    float* const df = p.done_f32;
    p.io_f64 = 1;
    p.final_obs = nullptr;
    p.done_f32 = nullptr;
    p.pdl = 0;
    p.stage_obs = obs_dim_ <= MAX_STAGE_DIM ? 1 : 0;
    // stagger block starts over ~half the action read time on the host link (bytes/100
    // ~ ns at ~50 GB/s, capped at 2 us): early blocks' observation writes overlap the
    // later blocks' action reads (link is full duplex).  Measured, DESIGN.md §5
    p.stagger_ns = (int32_t)std::min<size_t>(2000, (size_t)m_ * n_act_ * 8 / 100);
    // action rows through shared memory once the read is bandwidth-bound on the link
    // (measured: 16,384 envs 61.6 -> 57.6 us; 512 / 4,096 envs +1 us, latency-bound:
    // threads that start on their own row overlap the stragglers' loads)
    p.stage_act = (size_t)m_ * n_act_ * 8 >= (size_t(512) << 10) ? 1 : 0;
    const cudaError_t e = Launch<T>::step(p, task_.kind != 0, ranges_.enabled, fossen_, pair_,
                                          dev_io_[0], dev_io_[1], dev_io_[2],
                                          (uint8_t*)dev_io_[3], (int8_t*)dev_io_[4],
                                          stream_);
    p.io_f64 = io;
    p.stage_obs = stage;
    p.final_obs = fo;
    p.done_f32 = df;
    p.pdl = pdl;
    p.stagger_ns = 0;
    p.stage_act = 0;
    cuda_check(e, "step (mapped)");
}

template <class T>
void Engine::step_host_T(const double* act, double* obs, double* rew, uint8_t* done,
                         int8_t* reason) {
    // validated on every call (~0.03 us each): a cached answer could outlive the
    // caller's buffer
    const void* ptr[5] = {act, obs, rew, done, reason};
    HostBuf hb[5];
    bool locked = true, mapped = true;
    for (int i = 0; i < 5; ++i) {
        hb[i] = host_buf(ptr[i]);
        locked = locked && hb[i].locked;
        mapped = mapped && (!ptr[i] || hb[i].dev);
        dev_io_[i] = hb[i].dev;
    }
    if (!locked) {   // pageable buffers: staged DMA, no graph
        ensure_staging();
        enqueue_step_host<T>(act, obs, rew, done, reason);
        cuda_check(cudaStreamSynchronize(stream_), "step sync");
        return;
    }
    // page-locked: replay a graph of the whole step for this buffer set (a graph
    // replay + sync is ~2.4 us shorter than a plain launch + sync, measured)
    AbiGraph* g = nullptr;
    for (AbiGraph& c : abi_graphs_) {
        bool hit = c.exec != nullptr;
        for (int i = 0; i < 5 && hit; ++i) hit = c.ptr[i] == ptr[i] && c.id[i] == hb[i].id;
        if (hit) { g = &c; break; }
    }
    if (!g) {
        g = &abi_graphs_[abi_next_];
        abi_next_ = (abi_next_ + 1) % kAbiGraphs;
        if (g->exec) cudaGraphExecDestroy(g->exec);
        *g = AbiGraph{};
        // zero-copy writes rows with 16-byte vector stores: require an aligned obs base
        const bool zero_copy = mapped && use_mapped() && (((uintptr_t)obs & 15) == 0) &&
                               (((uintptr_t)rew & 7) == 0) && (((uintptr_t)act & 7) == 0);
        if (!zero_copy) ensure_staging();   // no allocation inside the capture
        cuda_check(cudaStreamSynchronize(stream_), "abi capture pre-sync");
        cudaGraph_t graph = nullptr;
        cuda_check(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal),
                   "abi capture");
        try {
            if (zero_copy) enqueue_step_mapped<T>();
            else enqueue_step_host<T>(act, obs, rew, done, reason);
        } catch (...) {
            cudaStreamEndCapture(stream_, &graph);
            if (graph) cudaGraphDestroy(graph);
            throw;
        }
        cuda_check(cudaStreamEndCapture(stream_, &graph), "abi capture end");
        const cudaError_t e = cudaGraphInstantiate(&g->exec, graph, 0);
        cudaGraphDestroy(graph);
        cuda_check(e, "abi graph instantiate");
        for (int i = 0; i < 5; ++i) {
            g->ptr[i] = ptr[i];
            g->id[i] = hb[i].id;
        }
    }
    cuda_check(cudaGraphLaunch(g->exec, stream_), "abi graph launch");
    cuda_check(cudaStreamSynchronize(stream_), "step sync");
}

void Engine::step_host(const double* act, double* obs, double* rew, uint8_t* done,
                       int8_t* reason) {
    activate();
    wait_device_face();
    if (h_err_) *h_err_ = 0;
    if (fp64_) step_host_T<double>(act, obs, rew, done, reason);
    else step_host_T<float>(act, obs, rew, done, reason);
    if (h_err_ && *h_err_)   // engine.rs:553-558 panics here; the outputs are still written
        throw RuntimeError("per-episode parameter resample rejected: randomized parameters "
                           "invalid: M_RB + M_A is not positive definite (the env keeps its "
                           "previous parameters)");
}

void Engine::states_host(double* out) {
    activate();
    wait_device_face();
    ensure_pack();
    if (fp64_) cuda_check(Launch<double>::pack_states(*pd_, d_pack_, stream_), "pack");
    else cuda_check(Launch<float>::pack_states(*pf_, d_pack_, stream_), "pack");
    cuda_check(cudaMemcpyAsync(out, d_pack_, (size_t)m_ * 12 * 8, cudaMemcpyDeviceToHost, stream_), "states D2H");
    cuda_check(cudaStreamSynchronize(stream_), "states sync");
}

void Engine::set_states_host(const double* in) {
    activate();
    wait_device_face();
    ensure_pack();
    cuda_check(cudaMemcpyAsync(d_pack_, in, (size_t)m_ * 12 * 8, cudaMemcpyHostToDevice, stream_), "states H2D");
    if (fp64_) cuda_check(Launch<double>::unpack_states(*pd_, d_pack_, stream_), "unpack");
    else cuda_check(Launch<float>::unpack_states(*pf_, d_pack_, stream_), "unpack");
    cuda_check(cudaStreamSynchronize(stream_), "set_states sync");
}

void Engine::step_counts_host(int64_t* out) {
    activate();
    wait_device_face();
    std::vector<int32_t> tmp((size_t)m_);
    int32_t* src = fp64_ ? pd_->step : pf_->step;
    cuda_check(cudaMemcpyAsync(tmp.data(), src, (size_t)m_ * 4, cudaMemcpyDeviceToHost, stream_), "steps D2H");
    cuda_check(cudaStreamSynchronize(stream_), "steps sync");
    for (size_t i = 0; i < tmp.size(); ++i) out[i] = tmp[i];
}

void Engine::set_step_counts_host(const int64_t* in) {
    activate();
    wait_device_face();
    std::vector<int32_t> tmp((size_t)m_);
    for (size_t i = 0; i < tmp.size(); ++i) {
        if (in[i] < 0 || in[i] >= task_.episode_len)
            throw ConfigError("step counts must lie in [0, episode_len)");
        tmp[i] = (int32_t)in[i];
    }
    int32_t* dst = fp64_ ? pd_->step : pf_->step;
    cuda_check(cudaMemcpyAsync(dst, tmp.data(), (size_t)m_ * 4, cudaMemcpyHostToDevice, stream_), "steps H2D");
    cuda_check(cudaStreamSynchronize(stream_), "steps sync");
}

void Engine::counters_host(uint64_t* rc, uint64_t* pc) {
    activate();
    wait_device_face();
    uint64_t* r = fp64_ ? pd_->reset_ctr : pf_->reset_ctr;
    uint64_t* q = fp64_ ? pd_->param_ctr : pf_->param_ctr;
    if (rc) cuda_check(cudaMemcpyAsync(rc, r, (size_t)m_ * 8, cudaMemcpyDeviceToHost, stream_), "ctr D2H");
    if (pc) cuda_check(cudaMemcpyAsync(pc, q, (size_t)m_ * 8, cudaMemcpyDeviceToHost, stream_), "ctr D2H");
    cuda_check(cudaStreamSynchronize(stream_), "ctr sync");
}

// body wrench tau [N][6] for host f64 action rows (thrusters.py:97-119): the
// step kernel's wrench() in the engine precision
void Engine::wrench_host(const double* act, double* out) {
    activate();
    wait_device_face();
    ensure_staging();
    ensure_pack();
    const size_t N = (size_t)m_;
    cuda_check(cudaMemcpyAsync(d_act64_, act, N * n_act_ * 8, cudaMemcpyHostToDevice, stream_), "act H2D");
    if (fp64_) cuda_check(Launch<double>::wrench(*pd_, ranges_.enabled, d_act64_, d_pack_, stream_), "wrench");
    else cuda_check(Launch<float>::wrench(*pf_, ranges_.enabled, d_act64_, d_pack_, stream_), "wrench");
    cuda_check(cudaMemcpyAsync(out, d_pack_, N * 6 * 8, cudaMemcpyDeviceToHost, stream_), "wrench D2H");
    cuda_check(cudaStreamSynchronize(stream_), "wrench sync");
}

void Engine::dr_factors_host(double* out) {
    activate();
    wait_device_face();
    if (!ranges_.enabled) {
        for (int64_t e = 0; e < m_; ++e) {
            const BaseVehicle& v = veh_[0];
            double* r = out + e * 10;
            r[0] = r[1] = r[2] = r[3] = r[4] = 1.0;
            r[5] = v.rb[0]; r[6] = v.rb[1]; r[7] = v.rb[2];
            r[8] = v.weight; r[9] = v.buoyancy;
        }
        return;
    }
    ensure_pack();
    if (fp64_) cuda_check(Launch<double>::pack_dr(*pd_, d_pack_, stream_), "pack_dr");
    else cuda_check(Launch<float>::pack_dr(*pf_, d_pack_, stream_), "pack_dr");
    cuda_check(cudaMemcpyAsync(out, d_pack_, (size_t)m_ * 10 * 8, cudaMemcpyDeviceToHost, stream_), "dr D2H");
    cuda_check(cudaStreamSynchronize(stream_), "dr sync");
}

// ------------------------------------------------------------------ checkpoint
namespace {
struct SnapHeader {
    char magic[8];            // "UUVB200S"
    uint32_t version, precision_bytes;
    uint64_t n_env, env_offset, root_seed, payload_bytes, config_hash;
    uint32_t obs_dim, act_dim, dr, pad;
};
static_assert(sizeof(SnapHeader) == 72, "snapshot header layout");
constexpr uint32_t kSnapVersion = 1;

uint64_t fnv1a(const void* data, size_t n, uint64_t h = 1469598103934665603ull) {
    const unsigned char* c = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < n; ++i) h = (h ^ c[i]) * 1099511628211ull;
    return h;
}
}  // namespace

// fingerprint of everything that determines the dynamics and the draws: the
// kernel parameter block minus buffer pointers and the per-launch root seed
template <class T> static uint64_t hash_params(const EngineP<T>& p) {
    uint64_t h = fnv1a(p.veh, sizeof(p.veh));
    TaskP<T> tk = p.task;
    tk.traj = nullptr;
    h = fnv1a(&tk, sizeof(tk), h);
    h = fnv1a(&p.ranges, sizeof(p.ranges), h);
    h = fnv1a(&p.mix_bound0, sizeof(p.mix_bound0), h);
    h = fnv1a(&p.n_veh, sizeof(p.n_veh), h);
    return h;
}

uint64_t Engine::config_hash() const { return fp64_ ? hash_params(*pd_) : hash_params(*pf_); }

size_t Engine::snapshot_bytes() const { return sizeof(SnapHeader) + arena_used_; }

void Engine::snapshot(void* out) {
    activate();
    cuda_check(cudaStreamSynchronize(stream_), "snapshot sync");
    cuda_check(cudaDeviceSynchronize(), "snapshot sync");   // device-face work on other streams
    SnapHeader h{};
    std::memcpy(h.magic, "UUVB200S", 8);
    h.version = kSnapVersion;
    h.precision_bytes = fp64_ ? 8 : 4;
    h.n_env = (uint64_t)m_;
    h.env_offset = env_offset_;
    h.root_seed = fp64_ ? pd_->seed : pf_->seed;
    h.payload_bytes = arena_used_;
    h.config_hash = config_hash();
    h.obs_dim = (uint32_t)obs_dim_;
    h.act_dim = (uint32_t)n_act_;
    h.dr = ranges_.enabled ? 1 : 0;
    std::memcpy(out, &h, sizeof(h));
    cuda_check(cudaMemcpy(static_cast<char*>(out) + sizeof(h), arena_, arena_used_,
                          cudaMemcpyDeviceToHost), "snapshot D2H");
}

void Engine::restore(const void* in, size_t len) {
    activate();
    SnapHeader h{};
    if (len < sizeof(h)) throw ConfigError("snapshot is truncated");
    std::memcpy(&h, in, sizeof(h));
    if (std::memcmp(h.magic, "UUVB200S", 8) != 0 || h.version != kSnapVersion)
        throw ConfigError("not a B200 engine snapshot (bad magic or version)");
    if (h.precision_bytes != (fp64_ ? 8u : 4u) || h.n_env != (uint64_t)m_ ||
        h.env_offset != env_offset_ || h.obs_dim != (uint32_t)obs_dim_ ||
        h.act_dim != (uint32_t)n_act_ || h.dr != (ranges_.enabled ? 1u : 0u) ||
        h.payload_bytes != arena_used_ || h.config_hash != config_hash())
        throw ConfigError("snapshot does not match this engine's configuration");
    if (len != sizeof(h) + arena_used_) throw ConfigError("snapshot is truncated");
    cuda_check(cudaDeviceSynchronize(), "restore sync");
    cuda_check(cudaMemcpy(arena_, static_cast<const char*>(in) + sizeof(h), arena_used_,
                          cudaMemcpyHostToDevice), "restore H2D");
    if (fp64_) {
        pd_->seed = h.root_seed;
    } else {
        pf_->seed = h.root_seed;
        // band flags follow the restored states
        cuda_check(Launch<float>::band_flags(*pf_, stream_), "band flags");
        cuda_check(cudaStreamSynchronize(stream_), "restore sync");
    }
}

void Engine::stats_host(double* out, bool clear) {
    activate();
    wait_device_face();
    cuda_check(launch_stats_reduce(stats_part_, nstat_blk_, d_stats_out_, clear ? 1 : 0, stream_), "stats");
    cuda_check(cudaMemcpyAsync(out, d_stats_out_, NSTAT * 8, cudaMemcpyDeviceToHost, stream_), "stats D2H");
    cuda_check(cudaStreamSynchronize(stream_), "stats sync");
}

// ------------------------------------------------------------------ ordering
// Host-ABI calls run on the engine's private stream; device-face work runs on
// the caller's stream.  Each device-face launch records dev_ev_ on the caller's
// stream (outside stream capture) and the next host-ABI call makes its stream
// wait for it, so e.g. step_tensors(); states() needs no explicit synchronize.
// (Host-ABI calls synchronize before they return, so the reverse order holds.)
void Engine::note_device_face(cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    if (cs != cudaStreamCaptureStatusNone) return;   // graph replays record at launch
    cuda_check(cudaEventRecord(dev_ev_, st), "device-face event");
    dev_pending_ = true;
}

void Engine::wait_device_face() {
    if (!dev_pending_) return;
    cuda_check(cudaStreamWaitEvent(stream_, dev_ev_, 0), "device-face wait");
    dev_pending_ = false;
}

// ------------------------------------------------------------------ device face
// device-face calls launch on the caller's stream without switching devices (that
// would change the caller's current device): refuse loudly when it is not ours
void Engine::check_device() const {
    int cur = -1;
    cuda_check(cudaGetDevice(&cur), "cudaGetDevice");
    if (cur != device_)
        throw RuntimeError("device face called with current CUDA device " + std::to_string(cur) +
                           "; this engine lives on device " + std::to_string(device_));
}

void Engine::dev_step(const void* act, void* obs, void* rew, uint8_t* done, int8_t* reason,
                      cudaStream_t st) {
    check_device();
    const bool track = task_.kind != 0, dr = ranges_.enabled;
    if (fp64_)
        cuda_check(Launch<double>::step(*pd_, track, dr, fossen_, pair_, (const double*)act,
                                        (double*)obs, (double*)rew, done, reason, st), "dev_step");
    else
        cuda_check(Launch<float>::step(*pf_, track, dr, fossen_, pair_, (const float*)act, (float*)obs,
                                       (float*)rew, done, reason, st), "dev_step");
    note_device_face(st);
}

void Engine::dev_reset(uint64_t seed, void* obs, cudaStream_t st) {
    check_device();
    if (fp64_) {
        pd_->seed = seed;
        cuda_check(Launch<double>::reset(*pd_, (double*)obs, st), "dev_reset");
    } else {
        pf_->seed = seed;
        cuda_check(Launch<float>::reset(*pf_, (float*)obs, st), "dev_reset");
    }
    note_device_face(st);
}

void Engine::dev_observe(void* obs, cudaStream_t st) {
    check_device();
    if (fp64_) cuda_check(Launch<double>::observe(*pd_, (double*)obs, st), "dev_observe");
    else cuda_check(Launch<float>::observe(*pf_, (float*)obs, st), "dev_observe");
    note_device_face(st);
}

void Engine::dev_set_done_f32(float* buf) {
    if (fp64_) pd_->done_f32 = buf;
    else pf_->done_f32 = buf;
}

void Engine::dev_set_pdl(bool on) {
    if (fp64_) pd_->pdl = on ? 1 : 0;
    else pf_->pdl = on ? 1 : 0;
}

void Engine::dev_set_final_obs(void* buf) {
    if (fp64_) pd_->final_obs = buf;
    else pf_->final_obs = buf;
}

void Engine::dev_pd_actions(const UuvPdGains& g, const void* ref6, void* act, cudaStream_t st) {
    check_device();
    if (fp64_)
        cuda_check(Launch<double>::pd_actions(*pd_, g, (const double*)ref6, (double*)act, st),
                   "dev_pd_actions");
    else
        cuda_check(Launch<float>::pd_actions(*pf_, g, (const float*)ref6, (float*)act, st),
                   "dev_pd_actions");
    note_device_face(st);
}

void Engine::dev_states(void* out, cudaStream_t st) {
    check_device();
    if (fp64_) cuda_check(Launch<double>::pack_states_t(*pd_, (double*)out, st), "dev_states");
    else cuda_check(Launch<float>::pack_states_t(*pf_, (float*)out, st), "dev_states");
    note_device_face(st);
}

void Engine::dev_bench_actions(void* act, cudaStream_t st) {
    check_device();
    const uint64_t seed = fp64_ ? pd_->seed : pf_->seed;
    cuda_check(launch_bench_actions(seed, env_offset_, (int)m_, n_act_,
                                    fp64_ ? nullptr : (float*)act,
                                    fp64_ ? (double*)act : nullptr, st), "bench_actions");
    note_device_face(st);
}

void Engine::dev_stats(double* out, bool clear, cudaStream_t st) {
    check_device();
    cuda_check(launch_stats_reduce(stats_part_, nstat_blk_, out, clear ? 1 : 0, st), "dev_stats");
    note_device_face(st);
}

void Engine::graph_capture(const void* act, void* obs, void* rew, uint8_t* done,
                           int8_t* reason, int n_steps) {
    activate();
    if (graph_exec_) {
        cudaGraphExecDestroy(graph_exec_);
        graph_exec_ = nullptr;
    }
    cuda_check(cudaStreamSynchronize(stream_), "capture pre-sync");
    cudaGraph_t g = nullptr;
    cuda_check(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "BeginCapture");
    try {
        for (int i = 0; i < n_steps; ++i) dev_step(act, obs, rew, done, reason, stream_);
    } catch (...) {
        cudaStreamEndCapture(stream_, &g);
        if (g) cudaGraphDestroy(g);
        throw;
    }
    cuda_check(cudaStreamEndCapture(stream_, &g), "EndCapture");
    cudaError_t e = cudaGraphInstantiate(&graph_exec_, g, 0);
    cudaGraphDestroy(g);
    cuda_check(e, "GraphInstantiate");
}

void Engine::graph_launch(cudaStream_t st) {
    check_device();
    if (!graph_exec_) throw RuntimeError("no captured graph (call uuvsim_dev_graph_capture first)");
    cuda_check(cudaGraphLaunch(graph_exec_, st), "GraphLaunch");
    note_device_face(st);
}

void Engine::synchronize() {
    activate();
    cuda_check(cudaDeviceSynchronize(), "synchronize");
}

std::string Engine::info() const {
    cudaFuncAttributes a{};
    const bool track = task_.kind != 0, dr = ranges_.enabled, mix = veh_.size() > 1;
    const bool tma = !fp64_ && pf_->persist_blocks > 0;
    if (fp64_) Launch<double>::step_attrs(&a, track, dr, fossen_, mix, pair_, false);
    else Launch<float>::step_attrs(&a, track, dr, fossen_, mix, pair_, tma);
    json j = {
        {"engine", "paper_2410_14117_b200"},
        {"abi_version", 1},
        {"precision", fp64_ ? "fp64" : "fp32"},
        {"num_envs", m_},
        {"env_offset", env_offset_},
        {"obs_dim", obs_dim_},
        {"action_dim", n_act_},
        {"episode_len", task_.episode_len},
        {"n_substeps", task_.n_substeps},
        {"task_kind", task_.kind},
        {"n_vehicles", veh_.size()},
        {"randomization", ranges_.enabled},
        {"pattern", fossen_ ? "fossen" : "dense"},
        {"envs_per_thread", pair_ ? 2 : 1},
        {"tma_pipelined", (fp64_ ? 0 : pf_->persist_blocks) > 0},
        {"band64", !fp64_ && band64_},
        {"stage_obs", (fp64_ ? pd_->stage_obs : pf_->stage_obs) != 0},
        {"host_io", host_io_ == 0 ? "copy" : host_io_ == 1 ? "mapped" : "auto"},
        {"arena_address", (uint64_t)(uintptr_t)arena_},
        {"arena_bytes", (uint64_t)arena_used_},
        {"abi_staging_bytes", (uint64_t)(staging_bytes_ + (d_pack_ ? (size_t)m_ * 96 : 0))},
        {"per_episode", ranges_.per_episode},
        {"device", device_},
        {"device_name", device_name_},
        {"sm_count", sm_count_},
        {"block", BLOCK},
        {"grid", pair_ ? (nblk_ + 1) / 2 : nblk_},
        {"step_kernel_registers", a.numRegs},
        {"step_kernel_local_bytes", a.localSizeBytes},
        {"param_block_bytes", fp64_ ? sizeof(EngineP<double>) : sizeof(EngineP<float>)},
        {"seed", fp64_ ? pd_->seed : pf_->seed},
    };
    return j.dump();
}

}  // namespace uuv

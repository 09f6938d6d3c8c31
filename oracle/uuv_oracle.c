/*
 * uuv_oracle.c -- TEST INFRASTRUCTURE ONLY: the CPU parity checker and the timed
 * CPU baseline ("port" of the reference).  Never linked into the product.
 *
 * fp64 restatement of the reference's order-pinned flat kernels.  Every
 * expression keeps the reference's evaluation order; build with
 * -ffp-contract=off and glibc libm (the reference's own precision contract,
 * native/src/mathx.rs:1-15, dynamics.py:18-21) so results are bit-identical
 * to the Python PyEnvBatch.  Each function cites the reference lines it follows.
 */
#include "uuv_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_PI 3.141592653589793
static const double TWO_PI = 2.0 * ORC_PI;                  /* dynamics.py:36 */
static const double PITCH_LIMIT = ORC_PI / 2.0 - 1e-3;      /* dynamics.py:39 */
static const double DIVERGENCE_RADIUS = 10.0;               /* tasks.py:39 */
static const double RESET_POS_HALF = 1.0;                   /* tasks.py:45-47 */
static const double RESET_ROLL_PITCH_HALF = 0.1;
static const double RESET_YAW_HALF = 0.5;

/* ---------------------------------------------------------------- rng.py */
static const uint64_t GOLDEN = 0x9E3779B97F4A7C15ULL;       /* rng.py:16-17 */
static const uint64_t PURPOSE_SALT = 0x632BE59BD9B4E019ULL;
enum { PURPOSE_PARAMS = 0, PURPOSE_RESET = 1, PURPOSE_BENCH = 2 };

uint64_t orc_mix64(uint64_t z) {                            /* rng.py:26-31 */
    z = z + GOLDEN;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t orc_draw_u64(uint64_t seed, uint64_t stream, uint64_t purpose, uint64_t counter) {
    uint64_t h = orc_mix64(seed);                            /* rng.py:34-40 */
    h = orc_mix64(h ^ (stream + GOLDEN));
    h = orc_mix64(h ^ (purpose + PURPOSE_SALT));
    h = orc_mix64(h ^ counter);
    return h;
}

double orc_u01(uint64_t bits) {                             /* rng.py:43-45 */
    return (double)(bits >> 11) * (1.0 / 9007199254740992.0);
}

static double uniform_(double lo, double hi, double u) { return lo + (hi - lo) * u; }

static double next_uniform(uint64_t seed, uint64_t stream, uint64_t purpose, uint64_t* ctr,
                           double lo, double hi) {          /* rng.py:71-76 */
    uint64_t bits = orc_draw_u64(seed, stream, purpose, *ctr);
    *ctr += 1;
    return uniform_(lo, hi, orc_u01(bits));
}

static double next_log_uniform(uint64_t seed, uint64_t stream, uint64_t purpose, uint64_t* ctr,
                               double lo, double hi) {      /* rng.py:52-53,78-80 */
    uint64_t bits = orc_draw_u64(seed, stream, purpose, *ctr);
    *ctr += 1;
    return exp(uniform_(log(lo), log(hi), orc_u01(bits)));
}

/* ---------------------------------------------------------- dynamics.py */
double orc_wrap_angle(double a) {                           /* dynamics.py:56-61 */
    double r = fmod(a + ORC_PI, TWO_PI);
    if (r <= 0.0) r += TWO_PI;
    return r - ORC_PI;
}

static int cholesky6(const double* m, double* L) {          /* dynamics.py:159-173 */
    for (int k = 0; k < 36; ++k) L[k] = 0.0;
    for (int i = 0; i < 6; ++i) {
        for (int j = 0; j <= i; ++j) {
            double s = m[i * 6 + j];
            for (int k = 0; k < j; ++k) s -= L[i * 6 + k] * L[j * 6 + k];
            if (i == j) {
                if (s <= 0.0) return 1;
                L[i * 6 + i] = sqrt(s);
            } else {
                L[i * 6 + j] = s / L[j * 6 + j];
            }
        }
    }
    return 0;
}

void orc_chol_solve(const double L[36], const double b[6], double x[6]) {  /* :176-189 */
    double y[6];
    for (int i = 0; i < 6; ++i) {
        double s = b[i];
        for (int k = 0; k < i; ++k) s -= L[i * 6 + k] * y[k];
        y[i] = s / L[i * 6 + i];
    }
    for (int i = 5; i >= 0; --i) {
        double s = y[i];
        for (int k = i + 1; k < 6; ++k) s -= L[k * 6 + i] * x[k];
        x[i] = s / L[i * 6 + i];
    }
}

static void cross3(double ax, double ay, double az, double bx, double by, double bz, double* o) {
    o[0] = ay * bz - az * by;                               /* dynamics.py:155-156 */
    o[1] = az * bx - ax * bz;
    o[2] = ax * by - ay * bx;
}

void orc_coriolis(const double m[36], const double v[6], double out[6]) {  /* :192-212 */
    double a1[3], a2[3], c[3], t[3], s[3];
    for (int i = 0; i < 3; ++i) {
        double acc = 0.0;
        for (int j = 0; j < 6; ++j) acc += m[i * 6 + j] * v[j];
        a1[i] = acc;
    }
    for (int i = 3; i < 6; ++i) {
        double acc = 0.0;
        for (int j = 0; j < 6; ++j) acc += m[i * 6 + j] * v[j];
        a2[i - 3] = acc;
    }
    cross3(v[3], v[4], v[5], a1[0], a1[1], a1[2], c);
    cross3(v[0], v[1], v[2], a1[0], a1[1], a1[2], t);
    cross3(v[3], v[4], v[5], a2[0], a2[1], a2[2], s);
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2];
    out[3] = t[0] + s[0]; out[4] = t[1] + s[1]; out[5] = t[2] + s[2];
}

void orc_damping(const double dlin[36], const double dquad[6], const double v[6],
                 double out[6]) {                           /* dynamics.py:215-224 */
    for (int i = 0; i < 6; ++i) {
        double acc = 0.0;
        for (int j = 0; j < 6; ++j) acc += dlin[i * 6 + j] * v[j];
        out[i] = acc + dquad[i] * fabs(v[i]) * v[i];
    }
}

void orc_restoring(double w, double b, const double rg[3], const double rb[3], double sphi,
                   double cphi, double sth, double cth, double out[6]) {  /* :227-243 */
    double cth_sphi = cth * sphi, cth_cphi = cth * cphi;
    double fgx = -w * sth, fgy = w * cth_sphi, fgz = w * cth_cphi;
    double fbx = b * sth, fby = -b * cth_sphi, fbz = -b * cth_cphi;
    double mg[3], mb[3];
    cross3(rg[0], rg[1], rg[2], fgx, fgy, fgz, mg);
    cross3(rb[0], rb[1], rb[2], fbx, fby, fbz, mb);
    out[0] = fgx + fbx; out[1] = fgy + fby; out[2] = fgz + fbz;
    out[3] = mg[0] + mb[0]; out[4] = mg[1] + mb[1]; out[5] = mg[2] + mb[2];
}

int32_t orc_substep(const orc_kparams* kp, const double s[12], const double tau[6], double dt,
                    double o[12]) {                         /* dynamics.py:246-306 */
    const double* v = s + 6;
    double sphi = sin(s[3]), cphi = cos(s[3]);
    double sth = sin(s[4]), cth = cos(s[4]);
    double spsi = sin(s[5]), cpsi = cos(s[5]);
    double c[6], d[6], g[6], rhs[6], acc[6];
    orc_coriolis(kp->m_total, v, c);
    orc_damping(kp->dlin, kp->dquad, v, d);
    orc_restoring(kp->weight, kp->buoyancy, kp->rg, kp->rb, sphi, cphi, sth, cth, g);
    for (int i = 0; i < 6; ++i) rhs[i] = tau[i] - c[i] - d[i] + g[i];
    orc_chol_solve(kp->chol, rhs, acc);

    double u2 = v[0] + dt * acc[0], v2 = v[1] + dt * acc[1], w2 = v[2] + dt * acc[2];
    double p2 = v[3] + dt * acc[3], q2 = v[4] + dt * acc[4], r2 = v[5] + dt * acc[5];

    double xdot = cpsi * cth * u2 + (-spsi * cphi + cpsi * sth * sphi) * v2
                + (spsi * sphi + cpsi * cphi * sth) * w2;
    double ydot = spsi * cth * u2 + (cpsi * cphi + sphi * sth * spsi) * v2
                + (-cpsi * sphi + sth * spsi * cphi) * w2;
    double zdot = -sth * u2 + cth * sphi * v2 + cth * cphi * w2;
    double tth = sth / cth;
    double phidot = p2 + sphi * tth * q2 + cphi * tth * r2;
    double thetadot = cphi * q2 - sphi * r2;
    double psidot = sphi / cth * q2 + cphi / cth * r2;

    o[0] = s[0] + dt * xdot;
    o[1] = s[1] + dt * ydot;
    o[2] = s[2] + dt * zdot;
    o[3] = orc_wrap_angle(s[3] + dt * phidot);
    o[4] = orc_wrap_angle(s[4] + dt * thetadot);
    o[5] = orc_wrap_angle(s[5] + dt * psidot);
    if (o[4] > PITCH_LIMIT) o[4] = PITCH_LIMIT;
    else if (o[4] < -PITCH_LIMIT) o[4] = -PITCH_LIMIT;
    o[6] = u2; o[7] = v2; o[8] = w2; o[9] = p2; o[10] = q2; o[11] = r2;
    for (int i = 0; i < 12; ++i)
        if (!isfinite(o[i])) return i;
    return -1;
}

/* --------------------------------------------------------- thrusters.py */
void orc_wrench(const orc_kparams* kp, const double* action, double tau[6]) {  /* :97-119 */
    int n = kp->n_thr;
    double f[ORC_MAX_THR];
    for (int i = 0; i < n; ++i) {
        double t = action[i];
        if (t > 1.0) t = 1.0;
        else if (t < -1.0) t = -1.0;
        f[i] = kp->curve[i] == 0 ? kp->kmax[i] * t : kp->kmax[i] * (t * fabs(t));
    }
    for (int r = 0; r < 6; ++r) {
        double acc = 0.0;
        for (int i = 0; i < n; ++i) acc += kp->alloc[r * n + i] * f[i];
        tau[r] = acc;
    }
}

/* ----------------------------------------------------------- vehicle.py */
int32_t orc_build_kernel(const orc_vehicle* v, orc_kparams* kp) {  /* vehicle.py:64-112 */
    const double* rg = v->rg;
    /* _skew(r_g), vehicle.py:58-61 */
    double s[9] = {0.0, -rg[2], rg[1], rg[2], 0.0, -rg[0], -rg[1], rg[0], 0.0};
    double nm = -v->mass;
    double m_rb[36];
    for (int k = 0; k < 36; ++k) m_rb[k] = 0.0;
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) {
            m_rb[i * 6 + j] = v->mass * (i == j ? 1.0 : 0.0);  /* mass * np.eye(3) */
            m_rb[i * 6 + j + 3] = nm * s[i * 3 + j];
            m_rb[(i + 3) * 6 + j] = v->mass * s[i * 3 + j];
            m_rb[(i + 3) * 6 + j + 3] = v->inertia[i * 3 + j];
        }
    }
    for (int k = 0; k < 36; ++k) kp->m_total[k] = m_rb[k] + v->added[k];
    if (cholesky6(kp->m_total, kp->chol)) return 1;
    memcpy(kp->dlin, v->dlin, sizeof(kp->dlin));
    memcpy(kp->dquad, v->dquad, sizeof(kp->dquad));
    kp->weight = v->weight;
    kp->buoyancy = v->buoyancy;
    memcpy(kp->rg, v->rg, sizeof(kp->rg));
    memcpy(kp->rb, v->rb, sizeof(kp->rb));
    int n = v->n_thr;
    kp->n_thr = n;
    memset(kp->alloc, 0, sizeof(kp->alloc));
    for (int i = 0; i < n; ++i) {                           /* thrusters.py:81-94 */
        double px = v->pos[i][0], py = v->pos[i][1], pz = v->pos[i][2];
        double dx = v->dir[i][0], dy = v->dir[i][1], dz = v->dir[i][2];
        kp->alloc[0 * n + i] = dx;
        kp->alloc[1 * n + i] = dy;
        kp->alloc[2 * n + i] = dz;
        kp->alloc[3 * n + i] = py * dz - pz * dy;
        kp->alloc[4 * n + i] = pz * dx - px * dz;
        kp->alloc[5 * n + i] = px * dy - py * dx;
        kp->kmax[i] = v->kmax[i];
        kp->curve[i] = v->curve[i];
    }
    return 0;
}

/* ---------------------------------------------------------- randomize.py */
int32_t orc_sample_params(const orc_vehicle* base, const orc_ranges* r, uint64_t seed,
                          uint64_t stream, uint64_t* ctr, orc_kparams* out,
                          double fac[9]) {                  /* randomize.py:79-109 */
    const uint64_t P = PURPOSE_PARAMS;
    double f_mass = next_log_uniform(seed, stream, P, ctr, r->mass[0], r->mass[1]);
    double f_added = next_log_uniform(seed, stream, P, ctr, r->added[0], r->added[1]);
    double f_dlin = next_log_uniform(seed, stream, P, ctr, r->dlin[0], r->dlin[1]);
    double f_dquad = next_log_uniform(seed, stream, P, ctr, r->dquad[0], r->dquad[1]);
    double f_thrust = next_log_uniform(seed, stream, P, ctr, r->thrust[0], r->thrust[1]);
    double dbx = next_uniform(seed, stream, P, ctr, -r->rb_offset, r->rb_offset);
    double dby = next_uniform(seed, stream, P, ctr, -r->rb_offset, r->rb_offset);
    double dbz = next_uniform(seed, stream, P, ctr, -r->rb_offset, r->rb_offset);
    double ratio = next_uniform(seed, stream, P, ctr, r->ratio[0], r->ratio[1]);
    if (fac) {
        fac[0] = f_mass; fac[1] = f_added; fac[2] = f_dlin; fac[3] = f_dquad;
        fac[4] = f_thrust; fac[5] = dbx; fac[6] = dby; fac[7] = dbz; fac[8] = ratio;
    }
    orc_vehicle v = *base;
    double weight = base->weight * f_mass;
    v.mass = base->mass * f_mass;
    for (int k = 0; k < 9; ++k) v.inertia[k] = base->inertia[k] * f_mass;
    v.rb[0] = base->rb[0] + dbx;
    v.rb[1] = base->rb[1] + dby;
    v.rb[2] = base->rb[2] + dbz;
    v.weight = weight;
    v.buoyancy = ratio * weight;
    for (int k = 0; k < 36; ++k) {
        v.added[k] = base->added[k] * f_added;
        v.dlin[k] = base->dlin[k] * f_dlin;
    }
    for (int k = 0; k < 6; ++k) v.dquad[k] = base->dquad[k] * f_dquad;
    for (int i = 0; i < base->n_thr; ++i) v.kmax[i] = base->kmax[i] * f_thrust;
    return orc_build_kernel(&v, out);
}

/* -------------------------------------------------------------- tasks.py */
void orc_traj(const orc_task* t, double time, double o[4]) {   /* tasks.py:132-153 */
    double ang = t->omega * time;
    double ca = cos(ang), sa = sin(ang);
    if (t->kind == 1) {
        o[0] = t->cx + t->radius * ca;
        o[1] = t->cy + t->radius * sa;
        o[2] = t->depth;
        o[3] = atan2(ca, -sa);
    } else if (t->kind == 2) {
        o[0] = t->cx + t->radius * ca;
        o[1] = t->cy + t->radius * sa;
        o[2] = t->depth + t->climb * time;
        o[3] = atan2(ca, -sa);
    } else {
        o[0] = t->cx + t->scale * ca;
        o[1] = t->cy + t->scale * (sa * ca);
        o[2] = t->depth;
        double c2a = ca * ca - sa * sa;
        o[3] = atan2(c2a, -sa);
    }
}

static void reference_(const orc_task* t, int64_t step, double o[3]) {  /* tasks.py:156-161 */
    if (t->kind == 0) {
        o[0] = t->target[0]; o[1] = t->target[1]; o[2] = t->target[2];
        return;
    }
    double r[4];
    orc_traj(t, (double)step * t->control_dt, r);
    o[0] = r[0]; o[1] = r[1]; o[2] = r[2];
}

void orc_observe(const orc_task* t, const double s[12], int64_t step, double* obs) {
    int n = 0;                                              /* tasks.py:164-183 */
    if (t->kind == 0) {
        const double* tg = t->target;
        obs[n++] = tg[0] - s[0];
        obs[n++] = tg[1] - s[1];
        obs[n++] = tg[2] - s[2];
        obs[n++] = orc_wrap_angle(tg[3] - s[3]);
        obs[n++] = orc_wrap_angle(tg[4] - s[4]);
        obs[n++] = orc_wrap_angle(tg[5] - s[5]);
    } else {
        for (int k = 1; k <= t->lookahead; ++k) {
            double r[4];
            orc_traj(t, (double)(step + k) * t->control_dt, r);
            obs[n++] = r[0] - s[0];
            obs[n++] = r[1] - s[1];
            obs[n++] = r[2] - s[2];
            obs[n++] = orc_wrap_angle(0.0 - s[3]);
            obs[n++] = orc_wrap_angle(0.0 - s[4]);
            obs[n++] = orc_wrap_angle(r[3] - s[5]);
        }
    }
    for (int i = 6; i < 12; ++i) obs[n++] = s[i];
}

static void reset_(const orc_task* t, uint64_t seed, uint64_t stream, uint64_t* ctr,
                   double s[12]) {                          /* tasks.py:186-198 */
    double sx, sy, sz, ref_psi;
    if (t->kind == 0) {
        sx = t->target[0]; sy = t->target[1]; sz = t->target[2]; ref_psi = t->target[5];
    } else {
        double r[4];
        orc_traj(t, 0.0, r);
        sx = r[0]; sy = r[1]; sz = r[2]; ref_psi = r[3];
    }
    const uint64_t P = PURPOSE_RESET;
    s[0] = sx + next_uniform(seed, stream, P, ctr, -RESET_POS_HALF, RESET_POS_HALF);
    s[1] = sy + next_uniform(seed, stream, P, ctr, -RESET_POS_HALF, RESET_POS_HALF);
    s[2] = sz + next_uniform(seed, stream, P, ctr, -RESET_POS_HALF, RESET_POS_HALF);
    s[3] = next_uniform(seed, stream, P, ctr, -RESET_ROLL_PITCH_HALF, RESET_ROLL_PITCH_HALF);
    s[4] = next_uniform(seed, stream, P, ctr, -RESET_ROLL_PITCH_HALF, RESET_ROLL_PITCH_HALF);
    s[5] = orc_wrap_angle(ref_psi + next_uniform(seed, stream, P, ctr, -RESET_YAW_HALF,
                                                 RESET_YAW_HALF));
    for (int i = 6; i < 12; ++i) s[i] = 0.0;
}

int32_t orc_env_step(const orc_kparams* kp, const orc_task* t, double s[12], int64_t step,
                     const double* action, int64_t* new_step, double* reward,
                     double* pos_err) {                     /* tasks.py:201-230 */
    double tau[6], nxt[12];
    orc_wrench(kp, action, tau);
    int failed = -1;
    double sub_dt = t->control_dt / (double)t->n_substeps;
    for (int k = 0; k < t->n_substeps; ++k) {
        int f = orc_substep(kp, s, tau, sub_dt, nxt);
        if (f >= 0) { failed = f; break; }
        memcpy(s, nxt, sizeof(nxt));
    }
    int64_t ns = step + 1;
    double r[3];
    reference_(t, ns, r);
    double dx = r[0] - s[0], dy = r[1] - s[1], dz = r[2] - s[2];
    double pe = sqrt(dx * dx + dy * dy + dz * dz);
    *new_step = ns;
    *reward = -pe;
    if (pos_err) *pos_err = pe;
    if (failed >= 0) return 2;
    if (pe > DIVERGENCE_RADIUS) return 1;
    if (ns >= t->episode_len) return 0;
    return -1;
}

/* -------------------------------------------------------------- batch.py */
struct orc_batch {
    int64_t m;
    int32_t obs_dim, act_stride, n_vehicles, threads;
    uint64_t seed, env_offset;
    orc_task task;
    orc_ranges ranges;
    orc_vehicle vehicles[ORC_MAX_VEH];
    int32_t* vid;
    orc_kparams* kp;
    double* factors;    /* [m][9] */
    double* states;     /* [m][12] */
    int64_t* steps;
    uint64_t* reset_ctr;
    uint64_t* param_ctr;
};

static int obs_dim_of(const orc_task* t) { return t->kind == 0 ? 12 : 6 * t->lookahead + 6; }

orc_batch* orc_create(const orc_vehicle* vehicles, int32_t n_vehicles, const int32_t* vid,
                      const orc_task* task, const orc_ranges* ranges, int64_t m,
                      uint64_t seed, uint64_t env_offset, int32_t act_stride, char* err,
                      int64_t err_cap) {                    /* batch.py:41-73 */
    if (m < 1 || n_vehicles < 1 || n_vehicles > ORC_MAX_VEH) {
        if (err) snprintf(err, (size_t)err_cap, "invalid batch size or vehicle count");
        return NULL;
    }
    orc_batch* b = (orc_batch*)calloc(1, sizeof(orc_batch));
    b->m = m;
    b->task = *task;
    b->ranges = *ranges;
    b->n_vehicles = n_vehicles;
    for (int i = 0; i < n_vehicles; ++i) b->vehicles[i] = vehicles[i];
    b->obs_dim = obs_dim_of(task);
    b->act_stride = act_stride;
    b->seed = seed;
    b->env_offset = env_offset;
    b->threads = 1;
    b->vid = (int32_t*)calloc((size_t)m, sizeof(int32_t));
    if (vid) memcpy(b->vid, vid, (size_t)m * sizeof(int32_t));
    b->kp = (orc_kparams*)calloc((size_t)m, sizeof(orc_kparams));
    b->factors = (double*)calloc((size_t)m * 9, sizeof(double));
    b->states = (double*)calloc((size_t)m * 12, sizeof(double));
    b->steps = (int64_t*)calloc((size_t)m, sizeof(int64_t));
    b->reset_ctr = (uint64_t*)calloc((size_t)m, sizeof(uint64_t));
    b->param_ctr = (uint64_t*)calloc((size_t)m, sizeof(uint64_t));
    orc_kparams base_kp[ORC_MAX_VEH];
    for (int i = 0; i < n_vehicles; ++i) {
        if (orc_build_kernel(&vehicles[i], &base_kp[i])) {
            if (err) snprintf(err, (size_t)err_cap,
                              "M_RB + M_A is not positive definite: matrix is not positive definite");
            orc_destroy(b);
            return NULL;
        }
    }
    for (int64_t e = 0; e < m; ++e) {
        int v = b->vid[e];
        if (ranges->enabled) {
            uint64_t ctr = 0;
            if (orc_sample_params(&vehicles[v], ranges, seed, env_offset + (uint64_t)e, &ctr,
                                  &b->kp[e], &b->factors[e * 9])) {
                if (err) snprintf(err, (size_t)err_cap,
                                  "env %lld: randomized parameters invalid", (long long)e);
                orc_destroy(b);
                return NULL;
            }
            b->param_ctr[e] = ctr;
        } else {
            b->kp[e] = base_kp[v];
            double* f = &b->factors[e * 9];
            f[0] = f[1] = f[2] = f[3] = f[4] = 1.0;
            f[5] = f[6] = f[7] = 0.0;
            f[8] = 1.0;
        }
    }
    orc_reset(b, seed, NULL);
    return b;
}

void orc_destroy(orc_batch* b) {
    if (!b) return;
    free(b->vid); free(b->kp); free(b->factors); free(b->states); free(b->steps);
    free(b->reset_ctr); free(b->param_ctr);
    free(b);
}

void orc_set_threads(orc_batch* b, int32_t n) { b->threads = n < 1 ? 1 : n; }
int32_t orc_obs_dim(const orc_batch* b) { return b->obs_dim; }

void orc_reset(orc_batch* b, uint64_t seed, double* obs) {  /* batch.py:75-88 */
    b->seed = seed;
    for (int64_t e = 0; e < b->m; ++e) {
        b->reset_ctr[e] = 0;
        reset_(&b->task, seed, b->env_offset + (uint64_t)e, &b->reset_ctr[e], &b->states[e * 12]);
        b->steps[e] = 0;
        if (obs) orc_observe(&b->task, &b->states[e * 12], 0, &obs[e * b->obs_dim]);
    }
}

static void step_one(orc_batch* b, int64_t e, const double* act, double* obs, double* rew,
                     uint8_t* done, int8_t* reason) {       /* batch.py:101-118 */
    double* s = &b->states[e * 12];
    int64_t ns;
    double r;
    int rc = orc_env_step(&b->kp[e], &b->task, s, b->steps[e], act, &ns, &r, NULL);
    rew[e] = r;
    done[e] = rc >= 0;
    if (reason) reason[e] = (int8_t)rc;
    uint64_t g = b->env_offset + (uint64_t)e;
    if (rc >= 0) {
        if (b->ranges.enabled && b->ranges.per_episode) {
            /* engine.rs:553-558 panics on invalid resample; the oracle keeps the old set */
            orc_kparams kp;
            if (!orc_sample_params(&b->vehicles[b->vid[e]], &b->ranges, b->seed, g,
                                   &b->param_ctr[e], &kp, &b->factors[e * 9]))
                b->kp[e] = kp;
        }
        reset_(&b->task, b->seed, g, &b->reset_ctr[e], s);
        b->steps[e] = 0;
    } else {
        b->steps[e] = ns;
    }
    orc_observe(&b->task, s, b->steps[e], &obs[e * b->obs_dim]);
}

void orc_step(orc_batch* b, const double* actions, double* obs, double* rew, uint8_t* done,
              int8_t* reason) {
    int64_t m = b->m;
#ifdef _OPENMP
    /* contiguous static chunks, as engine.rs:484-539 */
#pragma omp parallel for schedule(static) num_threads(b->threads) if (b->threads > 1)
#endif
    for (int64_t e = 0; e < m; ++e)
        step_one(b, e, &actions[e * b->act_stride], obs, rew, done, reason);
}

void orc_get_states(const orc_batch* b, double* out) {
    memcpy(out, b->states, (size_t)b->m * 12 * sizeof(double));
}
void orc_set_states(orc_batch* b, const double* in) {
    memcpy(b->states, in, (size_t)b->m * 12 * sizeof(double));
}
void orc_get_steps(const orc_batch* b, int64_t* out) {
    memcpy(out, b->steps, (size_t)b->m * sizeof(int64_t));
}
void orc_set_steps(orc_batch* b, const int64_t* in) {
    memcpy(b->steps, in, (size_t)b->m * sizeof(int64_t));
}
void orc_get_counters(const orc_batch* b, uint64_t* rc, uint64_t* pc) {
    if (rc) memcpy(rc, b->reset_ctr, (size_t)b->m * sizeof(uint64_t));
    if (pc) memcpy(pc, b->param_ctr, (size_t)b->m * sizeof(uint64_t));
}
void orc_get_factors(const orc_batch* b, double* out) {
    memcpy(out, b->factors, (size_t)b->m * 9 * sizeof(double));
}
void orc_get_kparams(const orc_batch* b, int64_t e, orc_kparams* out) { *out = b->kp[e]; }
void orc_observe_all(const orc_batch* b, double* obs) {
    for (int64_t e = 0; e < b->m; ++e)
        orc_observe(&b->task, &b->states[e * 12], b->steps[e], &obs[e * b->obs_dim]);
}

void orc_bench_actions(uint64_t seed, int64_t m, int32_t n, uint64_t off,
                       double* out) {                       /* batch.py:168-176 */
    for (int64_t i = 0; i < m; ++i)
        for (int32_t j = 0; j < n; ++j) {
            double u = orc_u01(orc_draw_u64(seed, off + (uint64_t)i, PURPOSE_BENCH, (uint64_t)j));
            out[i * n + j] = uniform_(-1.0, 1.0, u);
        }
}

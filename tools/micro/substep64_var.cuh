// Variants of substep_f64 for the latency probe (tools/micro/substep64.cu):
//   SKIPWRAP: wrap only when |a| >= 3.14159 (identical results: below it
//             rint(a / 2pi) = 0), so the common case pays a compare + branch;
//   LATE: the restoring terms (which wait for sin / cos) enter the residual last.
template <bool SKIPWRAP, bool LATE>
__device__ __forceinline__ void substep_var(const VehP<double>& V, double s[12], const double tau[6],
                                            double dt) {
    using Pat = PatFossen;
    const double* v = s + 6;
    double sphi, cphi, sth, cth, spsi, cpsi;
    sincos64(s[3], &sphi, &cphi);
    sincos64(s[4], &sth, &cth);
    sincos64(s[5], &spsi, &cpsi);
    const double e1 = cth * sphi, e2 = cth * cphi;
    double a[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < 6; ++j) {
            if (!Pat::M(i, j)) continue;
            acc = fma(V.mtot[i * 6 + j], v[j], acc);
        }
        a[i] = acc;
    }
    const double wb = V.wb, h0 = V.hm[0], h1 = V.hm[1], h2 = V.hm[2];
    double r[6];
    if (!LATE) {
        r[0] = fma(-wb, sth, tau[0]);
        r[1] = fma(wb, e1, tau[1]);
        r[2] = fma(wb, e2, tau[2]);
        r[3] = fma(h1, e2, fma(-h2, e1, tau[3]));
        r[4] = fma(-h2, sth, fma(-h0, e2, tau[4]));
        r[5] = fma(h0, e1, fma(h1, sth, tau[5]));
    } else {
#pragma unroll
        for (int i = 0; i < 6; ++i) r[i] = tau[i];
    }
    r[0] = fma(v[5], a[1], fma(-v[4], a[2], r[0]));
    r[1] = fma(v[3], a[2], fma(-v[5], a[0], r[1]));
    r[2] = fma(v[4], a[0], fma(-v[3], a[1], r[2]));
    r[3] = fma(v[5], a[4], fma(-v[4], a[5], fma(v[2], a[1], fma(-v[1], a[2], r[3]))));
    r[4] = fma(v[3], a[5], fma(-v[5], a[3], fma(v[0], a[2], fma(-v[2], a[0], r[4]))));
    r[5] = fma(v[4], a[3], fma(-v[3], a[4], fma(v[1], a[0], fma(-v[0], a[1], r[5]))));
#pragma unroll
    for (int i = 0; i < 6; ++i) r[i] = fma(-fma(V.dquad[i], fabs(v[i]), V.dlin[i * 6 + i]), v[i], r[i]);
    if (LATE) {
        r[0] = fma(-wb, sth, r[0]);
        r[1] = fma(wb, e1, r[1]);
        r[2] = fma(wb, e2, r[2]);
        r[3] = fma(h1, e2, fma(-h2, e1, r[3]));
        r[4] = fma(-h2, sth, fma(-h0, e2, r[4]));
        r[5] = fma(h0, e1, fma(h1, sth, r[5]));
    }
    double o[12];
    {
        constexpr int KI[10] = {0 * 6 + 0, 0 * 6 + 4, 4 * 6 + 0, 4 * 6 + 4, 1 * 6 + 1,
                                1 * 6 + 3, 3 * 6 + 1, 3 * 6 + 3, 2 * 6 + 2, 5 * 6 + 5};
        double k[10];
#pragma unroll
        for (int i = 0; i < 10; ++i) k[i] = V.kdt[KI[i]];
        o[6] = fma(k[0], r[0], fma(k[1], r[4], v[0]));
        o[10] = fma(k[2], r[0], fma(k[3], r[4], v[4]));
        o[7] = fma(k[4], r[1], fma(k[5], r[3], v[1]));
        o[9] = fma(k[6], r[1], fma(k[7], r[3], v[3]));
        o[8] = fma(k[8], r[2], v[2]);
        o[11] = fma(k[9], r[5], v[5]);
    }
    const double u2 = o[6], v2 = o[7], w2 = o[8], p2 = o[9], q2 = o[10], r2 = o[11];
    const double vy = fma(cphi, v2, -sphi * w2);
    const double vz = fma(sphi, v2, cphi * w2);
    const double vx = fma(cth, u2, sth * vz);
    const double zdot = fma(-sth, u2, cth * vz);
    const double xdot = fma(cpsi, vx, -spsi * vy);
    const double ydot = fma(spsi, vx, cpsi * vy);
    const double icth = rcp64(cth);
    const double sq = fma(sphi, q2, cphi * r2);
    const double phidot = fma(sth * icth, sq, p2);
    const double psidot = icth * sq;
    const double thetadot = fma(cphi, q2, -sphi * r2);
    o[0] = fma(dt, xdot, s[0]);
    o[1] = fma(dt, ydot, s[1]);
    o[2] = fma(dt, zdot, s[2]);
    double a3 = fma(dt, phidot, s[3]), a4 = fma(dt, thetadot, s[4]), a5 = fma(dt, psidot, s[5]);
    if (SKIPWRAP) {
        if (!(fmax(fabs(a3), fmax(fabs(a4), fabs(a5))) < 3.14159)) {
            a3 = wrap_pi64(a3); a4 = wrap_pi64(a4); a5 = wrap_pi64(a5);
        }
    } else {
        a3 = wrap_pi64(a3); a4 = wrap_pi64(a4); a5 = wrap_pi64(a5);
    }
    const double PL = Consts<double>::PITCH_LIMIT;
    o[3] = a3;
    o[4] = a4 > PL ? PL : (a4 < -PL ? -PL : a4);
    o[5] = a5;
#pragma unroll
    for (int i = 0; i < 12; ++i) s[i] = o[i];
}

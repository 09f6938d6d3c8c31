"""Fit and check the half-angle sin/cos used for the roll / yaw angles.

    python tools/numerics/halfangle_fit.py

S(x) = sin(x/2) = x (a0 + a1 z + ... + a4 z^4),   z = x^2,  |x| <= pi
C(x) = 2 cos(x/2) = b0 + b1 z + ... + b5 z^5
sin x = S C,  cos x = 1 - 2 S^2.
Coefficients: least-squares on Chebyshev nodes (relative error for S/x,
absolute for C), rounded to fp32; errors measured with an fp32 FMA emulation
against float64 and compared with the Cody-Waite kernel (sincos_poly).
"""
import numpy as np

f32 = np.float32


def fma(a, b, c):                       # a*b exact in f64 for f32 inputs; one rounding to f32
    return f32(np.float64(a) * np.float64(b) + np.float64(c))


def fit():
    y = np.cos(np.pi * (np.arange(4000) + 0.5) / 4000) * np.pi   # Chebyshev nodes on [-pi, pi]
    z = y * y
    # S/x = sin(x/2)/x = sum a_k z^k
    Vs = np.stack([z ** k for k in range(5)], 1)
    ts = np.where(y == 0, 0.5, np.sin(y / 2) / np.where(y == 0, 1, y))
    a = np.linalg.lstsq(Vs, ts, rcond=None)[0]
    Vc = np.stack([z ** k for k in range(6)], 1)
    b = np.linalg.lstsq(Vc, 2 * np.cos(y / 2), rcond=None)[0]
    return a.astype(f32), b.astype(f32)


def halfangle(x, a, b):
    x = f32(x)
    z = f32(x * x)
    p = a[4]
    for k in (3, 2, 1, 0):
        p = fma(p, z, a[k])
    S = f32(x * p)
    c = b[5]
    for k in (4, 3, 2, 1, 0):
        c = fma(c, z, b[k])
    sn = f32(S * c)
    cs = fma(S, f32(-2.0) * S, f32(1.0))
    return sn, cs


def cody_waite(x):
    x = f32(x)
    t = fma(x, f32(0.636619772367581343), f32(12582912.0))
    q = int(np.array(t, dtype=f32).view(np.int32))
    j = f32(t - f32(12582912.0))
    r = fma(j, f32(-1.57079625129699707031), x)
    r = fma(j, f32(-7.54978941586159635335e-08), r)
    r2 = f32(r * r)
    ps = fma(r2, f32(-1.9515295891e-4), f32(8.3321608736e-3))
    ps = fma(ps, r2, f32(-1.6666654611e-1))
    ps = fma(f32(ps * r2), r, r)
    pc = fma(r2, f32(2.443315711809948e-5), f32(-1.388731625493765e-3))
    pc = fma(pc, r2, f32(4.166664568298827e-2))
    pc = fma(pc, r2, f32(-0.5))
    pc = fma(pc, r2, f32(1.0))
    sn, cs = (pc, ps) if q & 1 else (ps, pc)
    if q & 2:
        sn = -sn
    if (q + 1) & 2:
        cs = -cs
    return sn, cs


def main():
    a, b = fit()
    print("a =", [float(v) for v in a])
    print("b =", [float(v) for v in b])
    xs = np.concatenate([np.linspace(-np.pi, np.pi, 200001), np.geomspace(1e-8, 1e-2, 2000)])
    xs = xs.astype(f32)
    for name, fn in (("halfangle", lambda x: halfangle(x, a, b)), ("cody_waite", cody_waite)):
        es = ec = rs = 0.0
        for x in xs[::7]:
            sn, cs = fn(x)
            ts, tc = np.sin(np.float64(x)), np.cos(np.float64(x))
            es = max(es, abs(float(sn) - ts))
            ec = max(ec, abs(float(cs) - tc))
            if abs(ts) > 1e-30:
                rs = max(rs, abs(float(sn) - ts) / abs(ts))
        print(f"{name:11s} max abs err sin {es:.3e} cos {ec:.3e}  max rel err sin {rs:.3e}")


if __name__ == "__main__":
    main()

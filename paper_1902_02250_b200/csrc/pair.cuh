// pair.cuh -- the MRS pair terms on CUDA cores (fp64), §7.
//
// With d = x - y, s = |d|^2 + eps^2 and rs = s^{-1/2} (hardware rsqrt seed + one
// cubic correction, <= ~4 ulp, for the direct sum; seed + one Newton step, relative
// error < 2e-12, for the treecode evaluation -- reading A19), the scalar functions of Eq. MRS_kernels are
//   8 pi H1 = (2 eps^2 + r^2) s^{-3/2} = rs + eps^2 rs^3
//   8 pi H2 = rs^3
//   8 pi Q  = (5 eps^2 + 2 r^2) s^{-5/2} = 2 rs^3 + 3 eps^2 rs^5
//   8 pi D1 = (10 eps^4 - 7 eps^2 r^2 - 2 r^4) s^{-7/2} = 15 eps^4 rs^7 - 3 eps^2 rs^5 - 2 rs^3
//   8 pi D2 = (21 eps^2 + 6 r^2) s^{-7/2} = 6 rs^5 + 15 eps^2 rs^7
// (substitute r^2 = s - eps^2).  Constants 1/(8 pi), 1/2, 1/4 are applied once
// per target at the end (scale()).  These differ from the literal formulas by
// rounding only.
//   Kern<KER>      pair terms with s^{-1/2} to ~4 ulp: the direct sum (kitc_direct)
//   EvalKern<KER>  treecode-evaluation forms (row form for the far field, scaled
//                  accumulators, one-step Newton s^{-1/2}: reading A19)
#pragma once
#include <cuda_runtime.h>

namespace kitc {

// s^{-1/2}: MUFU seed (rsqrt.approx.ftz.f64, ~2^-23 relative) + one cubic
// correction y' = y (1 + e/2 + 3e^2/8), e = 1 - s y^2 -> <= ~4 ulp (measured,
// profiles/r01_rsqrt_probe.txt), no special-case branch (s > 0 on every path
// that reaches it, except eps = 0 with coincident particles: inf, as the
// singular kernel itself).  1.4x the throughput of CUDA's rsqrt().
__device__ __forceinline__ double rsqrt_fast(double s) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(s));
    const double h = s * y;
    const double e = fma(-h, y, 1.0);
    const double p = fma(0.375, e, 0.5);
    return fma(y * e, p, y);
}

// 2 s^{-1/2} from the MUFU seed y by one Newton step folded into 3 FP64
// instructions: Y = y (3 - s y^2) = 2 s^{-1/2} (1 - 3/2 d^2 + ...), d the seed's
// relative error (|d| < 1e-6, profiles/r01_rsqrt_probe.txt), so |Y/(2 s^{-1/2}) - 1|
// < 2e-12 (measured <= 4e-13).  Used by the treecode evaluation only (its parity
// gate is 1e-10, reading A19); kitc_direct keeps rsqrt_fast.
__device__ __forceinline__ double rsqrt2_newton(double s) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(s));
    return y * fma(-(s * y), y, 3.0);
}

struct KParams {
    double e2;      // eps^2
    double e2x3;    // 3 eps^2
    double e4x15;   // 15 eps^4
    double e2x15;   // 15 eps^2
    double e2q;     // eps^2 / 4
    double e2x3_8;  // 3 eps^2 / 8
    double e4x15_32;  // 15 eps^4 / 32
    double e2x5_8;  // 5 eps^2 / 8
};

template <int KER> struct Kern;

// Stokeslet, Eq. Velocity_1: u = f H1 + [f.d] d H2.   m = 3, p = 3
template <> struct Kern<0> {
    static constexpr int M = 3, P = 3;
    static __device__ __forceinline__ void pair(double dx, double dy, double dz, double s,
                                                const double* f, double* acc, const KParams& k) {
        pair_rs(dx, dy, dz, rsqrt_fast(s), f, acc, k);
    }
    static __device__ __forceinline__ void pair_rs(double dx, double dy, double dz, double rs,
                                                   const double* f, double* acc, const KParams& k) {
        double rs2 = rs * rs;
        double rs3 = rs2 * rs;
        double h1 = fma(k.e2, rs3, rs);
        double fd = fma(f[0], dx, fma(f[1], dy, f[2] * dz));
        double c = fd * rs3;
        acc[0] = fma(c, dx, fma(f[0], h1, acc[0]));
        acc[1] = fma(c, dy, fma(f[1], h1, acc[1]));
        acc[2] = fma(c, dz, fma(f[2], h1, acc[2]));
    }
    // 1/(8 pi)
    static __device__ __forceinline__ double scale(int) { return 1.0 / (8.0 * 3.14159265358979323846); }
};

// Rotlet (Eqs. Velocity_2 / AngularVelocity with f = 0; readings A9, A10):
//   u = 1/2 [g x d] Q,   w = 1/4 g D1 + 1/4 [g.d] d D2.     m = 3, p = 6
template <> struct Kern<1> {
    static constexpr int M = 3, P = 6;
    static __device__ __forceinline__ void pair(double dx, double dy, double dz, double s,
                                                const double* g, double* acc, const KParams& k) {
        pair_rs(dx, dy, dz, rsqrt_fast(s), g, acc, k);
    }
    static __device__ __forceinline__ void pair_rs(double dx, double dy, double dz, double rs,
                                                   const double* g, double* acc, const KParams& k) {
        double rs2 = rs * rs;
        double rs3 = rs2 * rs;
        double rs5 = rs3 * rs2;
        double rs7 = rs5 * rs2;
        double q = fma(k.e2x3, rs5, 2.0 * rs3);
        double d1 = fma(k.e4x15, rs7, -q);   // 8 pi D1 = 15 eps^4 rs^7 - 8 pi Q
        double d2 = fma(k.e2x15, rs7, 6.0 * rs5);
        double cx = g[1] * dz - g[2] * dy;
        double cy = g[2] * dx - g[0] * dz;
        double cz = g[0] * dy - g[1] * dx;
        acc[0] = fma(cx, q, acc[0]);
        acc[1] = fma(cy, q, acc[1]);
        acc[2] = fma(cz, q, acc[2]);
        double gd = fma(g[0], dx, fma(g[1], dy, g[2] * dz)) * d2;
        acc[3] = fma(gd, dx, fma(g[0], d1, acc[3]));
        acc[4] = fma(gd, dy, fma(g[1], d1, acc[4]));
        acc[5] = fma(gd, dz, fma(g[2], d1, acc[5]));
    }
    // u: 1/(16 pi), w: 1/(32 pi)
    static __device__ __forceinline__ double scale(int c) {
        return c < 3 ? 1.0 / (16.0 * 3.14159265358979323846) : 1.0 / (32.0 * 3.14159265358979323846);
    }
};

// Stokeslet + rotlet (Eqs. Velocity_2 / AngularVelocity), weights (f, n):
//   u = f H1 + [f.d] d H2 + 1/2 [n x d] Q,  w = 1/2 [f x d] Q + 1/4 n D1 + 1/4 [n.d] d D2
// accumulated as 16 pi u and 32 pi w.                          m = 6, p = 6
template <> struct Kern<2> {
    static constexpr int M = 6, P = 6;
    static __device__ __forceinline__ void pair(double dx, double dy, double dz, double s,
                                                const double* f, double* acc, const KParams& k) {
        pair_rs(dx, dy, dz, rsqrt_fast(s), f, acc, k);
    }
    static __device__ __forceinline__ void pair_rs(double dx, double dy, double dz, double rs,
                                                   const double* f, double* acc, const KParams& k) {
        double rs2 = rs * rs;
        double rs3 = rs2 * rs;
        double rs5 = rs3 * rs2;
        double rs7 = rs5 * rs2;
        double h1x2 = 2.0 * fma(k.e2, rs3, rs);
        double q = fma(k.e2x3, rs5, 2.0 * rs3);
        double d1 = fma(k.e4x15, rs7, -q);   // 8 pi D1 = 15 eps^4 rs^7 - 8 pi Q
        double d2 = fma(k.e2x15, rs7, 6.0 * rs5);
        const double* g = f + 3;
        double fd2 = 2.0 * fma(f[0], dx, fma(f[1], dy, f[2] * dz)) * rs3;
        double nx = g[1] * dz - g[2] * dy, ny = g[2] * dx - g[0] * dz, nz = g[0] * dy - g[1] * dx;
        acc[0] = fma(nx, q, fma(fd2, dx, fma(f[0], h1x2, acc[0])));
        acc[1] = fma(ny, q, fma(fd2, dy, fma(f[1], h1x2, acc[1])));
        acc[2] = fma(nz, q, fma(fd2, dz, fma(f[2], h1x2, acc[2])));
        double fx = f[1] * dz - f[2] * dy, fy = f[2] * dx - f[0] * dz, fz = f[0] * dy - f[1] * dx;
        double q2 = 2.0 * q;
        double gd = fma(g[0], dx, fma(g[1], dy, g[2] * dz)) * d2;
        acc[3] = fma(fx, q2, fma(gd, dx, fma(g[0], d1, acc[3])));
        acc[4] = fma(fy, q2, fma(gd, dy, fma(g[1], d1, acc[4])));
        acc[5] = fma(fz, q2, fma(gd, dz, fma(g[2], d1, acc[5])));
    }
    static __device__ __forceinline__ double scale(int c) {
        return c < 3 ? 1.0 / (16.0 * 3.14159265358979323846) : 1.0 / (32.0 * 3.14159265358979323846);
    }
};

inline KParams make_kparams(double eps) {
    KParams k;
    double e2 = eps * eps;
    k.e2 = e2;
    k.e2x3 = 3.0 * e2;
    k.e4x15 = 15.0 * e2 * e2;
    k.e2x15 = 15.0 * e2;
    k.e2q = 0.25 * e2;
    k.e2x3_8 = 0.375 * e2;
    k.e4x15_32 = (15.0 / 32.0) * e2 * e2;
    k.e2x5_8 = 0.625 * e2;
    return k;
}

// ---------------------------------------------------------------------------
// Treecode-evaluation forms (eval.cu).  EvalKern<KER> exposes
//   NA accumulators, pair(dx,dy,dz,s,f,acc), pair_row(dx,dy,dz,s,f,acc,row),
//   row_end(dx,dy,row,acc), out(acc,c) -> output component c (scaled),
//   kPairRows (far field: two rows per lane),
// taking s = |d|^2 + eps^2; all three kernels use Y = 2 s^{-1/2} (rsqrt2_newton).
template <int KER> struct EvalKern;

// Stokeslet with Y = 2 s^{-1/2} (rsqrt2_newton): 16 pi H1 = 2 rs + 2 eps^2 rs^3 =
// Y + (eps^2/4) Y^3 and 16 pi H2 = 2 rs^3 = Y^3 / 4, so
//   16 pi u = sum f (Y + (eps^2/4) Y^3)   [acc 0..2]
//           + 1/4 sum [f.d] d Y^3         [acc 3..5]
// 16 FP64 instructions per far-field pair (row form) + the MUFU seed.
template <> struct EvalKern<0> {
    static constexpr int M = 3, P = 3, NA = 6;
    static constexpr bool kPairRows = true;
    static __device__ __forceinline__ void pair(double dx, double dy, double dz, double s, const double* f,
                                                double* acc, const KParams& k) {
        const double Y = rsqrt2_newton(s);
        const double Y3 = (Y * Y) * Y;
        const double h = fma(k.e2q, Y3, Y);
        const double c = fma(f[0], dx, fma(f[1], dy, f[2] * dz)) * Y3;
        acc[0] = fma(f[0], h, acc[0]);
        acc[1] = fma(f[1], h, acc[1]);
        acc[2] = fma(f[2], h, acc[2]);
        acc[3] = fma(c, dx, acc[3]);
        acc[4] = fma(c, dy, acc[4]);
        acc[5] = fma(c, dz, acc[5]);
    }
    struct Row {
        double C = 0.0, Z = 0.0;
    };
    static __device__ __forceinline__ void pair_row(double dx, double dy, double dz, double s, const double* f,
                                                    double* acc, Row& r, const KParams& k) {
        const double Y = rsqrt2_newton(s);
        const double Y3 = (Y * Y) * Y;
        const double h = fma(k.e2q, Y3, Y);
        const double c = fma(f[0], dx, fma(f[1], dy, f[2] * dz)) * Y3;
        r.C += c;
        r.Z = fma(c, dz, r.Z);
        acc[0] = fma(f[0], h, acc[0]);
        acc[1] = fma(f[1], h, acc[1]);
        acc[2] = fma(f[2], h, acc[2]);
    }
    static __device__ __forceinline__ void row_end(double dx, double dy, const Row& r, double* acc) {
        acc[3] = fma(r.C, dx, acc[3]);
        acc[4] = fma(r.C, dy, acc[4]);
        acc[5] += r.Z;
    }
    static __device__ __forceinline__ double out(const double* acc, int c) {
        return fma(0.25, acc[c + 3], acc[c]) * (1.0 / (16.0 * 3.14159265358979323846));
    }
};

// Rotlet with Y = 2 s^{-1/2}: rs^3 = Y^3/8, rs^5 = Y^5/32, rs^7 = Y^7/128, so
//   q  = Y^3 + (3 eps^2/8) Y^5       = 4 (8 pi Q)
//   d1 = (15 eps^4/32) Y^7 - q       = 4 (8 pi D1)
//   d2 = Y^5 + (5 eps^2/8) Y^7       = (16/3) (8 pi D2)
//   64 pi u  = sum [g x d] q                          [acc 0..2]
//   128 pi w = sum g d1  [acc 3..5]  + 3/4 sum [g.d] d d2  [acc 6..8]
// 26 FP64 instructions per far-field pair (row form) + the MUFU seed.
template <> struct EvalKern<1> {
    static constexpr int M = 3, P = 6, NA = 9;
    static constexpr bool kPairRows = true;
    static __device__ __forceinline__ void powers(double s, const KParams& k, double& q, double& d1, double& d2) {
        const double Y = rsqrt2_newton(s);
        const double Y2 = Y * Y;
        const double Y3 = Y2 * Y;
        const double Y5 = Y3 * Y2;
        const double Y7 = Y5 * Y2;
        q = fma(k.e2x3_8, Y5, Y3);
        d1 = fma(k.e4x15_32, Y7, -q);
        d2 = fma(k.e2x5_8, Y7, Y5);
    }
    static __device__ __forceinline__ void pair(double dx, double dy, double dz, double s, const double* g,
                                                double* acc, const KParams& k) {
        double q, d1, d2;
        powers(s, k, q, d1, d2);
        const double cx = g[1] * dz - g[2] * dy;
        const double cy = g[2] * dx - g[0] * dz;
        const double cz = g[0] * dy - g[1] * dx;
        acc[0] = fma(cx, q, acc[0]);
        acc[1] = fma(cy, q, acc[1]);
        acc[2] = fma(cz, q, acc[2]);
        acc[3] = fma(g[0], d1, acc[3]);
        acc[4] = fma(g[1], d1, acc[4]);
        acc[5] = fma(g[2], d1, acc[5]);
        const double gd = fma(g[0], dx, fma(g[1], dy, g[2] * dz)) * d2;
        acc[6] = fma(gd, dx, acc[6]);
        acc[7] = fma(gd, dy, acc[7]);
        acc[8] = fma(gd, dz, acc[8]);
    }
    // row form (dx, dy fixed): sum q (g x d) = (B1 - dy A2, dx A2 - B0, dy A0 - dx A1)
    // with A = sum q g, B = sum q dz g; sum (g.d) d2 d = (dx T, dy T, TZ).
    struct Row {
        double A0 = 0.0, A1 = 0.0, A2 = 0.0, B0 = 0.0, B1 = 0.0, T = 0.0, TZ = 0.0;
    };
    static __device__ __forceinline__ void pair_row(double dx, double dy, double dz, double s, const double* g,
                                                    double* acc, Row& r, const KParams& k) {
        double q, d1, d2;
        powers(s, k, q, d1, d2);
        r.A0 = fma(q, g[0], r.A0);
        r.A1 = fma(q, g[1], r.A1);
        r.A2 = fma(q, g[2], r.A2);
        const double qz = q * dz;
        r.B0 = fma(qz, g[0], r.B0);
        r.B1 = fma(qz, g[1], r.B1);
        acc[3] = fma(g[0], d1, acc[3]);
        acc[4] = fma(g[1], d1, acc[4]);
        acc[5] = fma(g[2], d1, acc[5]);
        const double t = fma(g[0], dx, fma(g[1], dy, g[2] * dz)) * d2;
        r.T += t;
        r.TZ = fma(t, dz, r.TZ);
    }
    static __device__ __forceinline__ void row_end(double dx, double dy, const Row& r, double* acc) {
        acc[0] += fma(-dy, r.A2, r.B1);
        acc[1] += fma(dx, r.A2, -r.B0);
        acc[2] += fma(dy, r.A0, -dx * r.A1);
        acc[6] = fma(r.T, dx, acc[6]);
        acc[7] = fma(r.T, dy, acc[7]);
        acc[8] += r.TZ;
    }
    static __device__ __forceinline__ double out(const double* acc, int c) {
        return c < 3 ? acc[c] * (1.0 / (64.0 * 3.14159265358979323846))
                     : fma(0.75, acc[c + 3], acc[c]) * (1.0 / (128.0 * 3.14159265358979323846));
    }
};

// Stokeslet + rotlet (weights f, n; m = 6, p = 6) with Y = 2 s^{-1/2} and
// q, d1, d2 as EvalKern<1>, h = Y + (eps^2/4) Y^3 as EvalKern<0>:
//   16 pi u  = sum f h                      [acc 0..2]
//            + 1/4 sum [(f.d) d Y^3 + (n x d) q]   [acc 3..5]
//   128 pi w = sum [n d1 + 2 (f x d) q + 3/4 (n.d) d d2]   [acc 6..8]
// Far field in row form with single rows per lane (14 row sums).
template <> struct EvalKern<2> {
    static constexpr int M = 6, P = 6, NA = 9;
    static constexpr bool kPairRows = false;
    static __device__ __forceinline__ void pair(double dx, double dy, double dz, double s, const double* f,
                                                double* acc, const KParams& k) {
        const double Y = rsqrt2_newton(s);
        const double Y2 = Y * Y;
        const double Y3 = Y2 * Y;
        const double Y5 = Y3 * Y2;
        const double Y7 = Y5 * Y2;
        const double q = fma(k.e2x3_8, Y5, Y3);
        const double d1 = fma(k.e4x15_32, Y7, -q);
        const double d2 = fma(k.e2x5_8, Y7, Y5);
        const double h = fma(k.e2q, Y3, Y);
        const double* n = f + 3;
        const double c = fma(f[0], dx, fma(f[1], dy, f[2] * dz)) * Y3;
        acc[0] = fma(f[0], h, acc[0]);
        acc[1] = fma(f[1], h, acc[1]);
        acc[2] = fma(f[2], h, acc[2]);
        acc[3] = fma(n[1] * dz - n[2] * dy, q, fma(c, dx, acc[3]));
        acc[4] = fma(n[2] * dx - n[0] * dz, q, fma(c, dy, acc[4]));
        acc[5] = fma(n[0] * dy - n[1] * dx, q, fma(c, dz, acc[5]));
        const double q2 = 2.0 * q;
        const double gd = fma(n[0], dx, fma(n[1], dy, n[2] * dz)) * (0.75 * d2);
        acc[6] = fma(f[1] * dz - f[2] * dy, q2, fma(gd, dx, fma(n[0], d1, acc[6])));
        acc[7] = fma(f[2] * dx - f[0] * dz, q2, fma(gd, dy, fma(n[1], d1, acc[7])));
        acc[8] = fma(f[0] * dy - f[1] * dx, q2, fma(gd, dz, fma(n[2], d1, acc[8])));
    }
    struct Row {
        double C = 0.0, Z = 0.0;                                      // (f.d) Y^3
        double An0 = 0.0, An1 = 0.0, An2 = 0.0, Bn0 = 0.0, Bn1 = 0.0;  // q n, q dz n
        double Af0 = 0.0, Af1 = 0.0, Af2 = 0.0, Bf0 = 0.0, Bf1 = 0.0;  // q f, q dz f
        double T = 0.0, TZ = 0.0;                                     // (n.d) d2
    };
    static __device__ __forceinline__ void pair_row(double dx, double dy, double dz, double s, const double* f,
                                                    double* acc, Row& r, const KParams& k) {
        const double Y = rsqrt2_newton(s);
        const double Y2 = Y * Y;
        const double Y3 = Y2 * Y;
        const double Y5 = Y3 * Y2;
        const double Y7 = Y5 * Y2;
        const double q = fma(k.e2x3_8, Y5, Y3);
        const double d1 = fma(k.e4x15_32, Y7, -q);
        const double d2 = fma(k.e2x5_8, Y7, Y5);
        const double h = fma(k.e2q, Y3, Y);
        const double* n = f + 3;
        acc[0] = fma(f[0], h, acc[0]);
        acc[1] = fma(f[1], h, acc[1]);
        acc[2] = fma(f[2], h, acc[2]);
        acc[6] = fma(n[0], d1, acc[6]);
        acc[7] = fma(n[1], d1, acc[7]);
        acc[8] = fma(n[2], d1, acc[8]);
        const double c = fma(f[0], dx, fma(f[1], dy, f[2] * dz)) * Y3;
        r.C += c;
        r.Z = fma(c, dz, r.Z);
        const double qz = q * dz;
        r.An0 = fma(q, n[0], r.An0);
        r.An1 = fma(q, n[1], r.An1);
        r.An2 = fma(q, n[2], r.An2);
        r.Bn0 = fma(qz, n[0], r.Bn0);
        r.Bn1 = fma(qz, n[1], r.Bn1);
        r.Af0 = fma(q, f[0], r.Af0);
        r.Af1 = fma(q, f[1], r.Af1);
        r.Af2 = fma(q, f[2], r.Af2);
        r.Bf0 = fma(qz, f[0], r.Bf0);
        r.Bf1 = fma(qz, f[1], r.Bf1);
        const double t = fma(n[0], dx, fma(n[1], dy, n[2] * dz)) * d2;
        r.T += t;
        r.TZ = fma(t, dz, r.TZ);
    }
    static __device__ __forceinline__ void row_end(double dx, double dy, const Row& r, double* acc) {
        acc[3] += fma(r.C, dx, fma(-dy, r.An2, r.Bn1));
        acc[4] += fma(r.C, dy, fma(dx, r.An2, -r.Bn0));
        acc[5] += r.Z + fma(dy, r.An0, -dx * r.An1);
        acc[6] += fma(2.0, fma(-dy, r.Af2, r.Bf1), 0.75 * dx * r.T);
        acc[7] += fma(2.0, fma(dx, r.Af2, -r.Bf0), 0.75 * dy * r.T);
        acc[8] += fma(2.0, fma(dy, r.Af0, -dx * r.Af1), 0.75 * r.TZ);
    }
    static __device__ __forceinline__ double out(const double* acc, int c) {
        return c < 3 ? fma(0.25, acc[c + 3], acc[c]) * (1.0 / (16.0 * 3.14159265358979323846))
                     : acc[c + 3] * (1.0 / (128.0 * 3.14159265358979323846));
    }
};

}  // namespace kitc

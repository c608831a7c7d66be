/* qrmc_student_t.h -- Student's t distribution (CDF and quantile) shared by the
 * oracle shim, the C restatement and the sm_100a kernels.
 *
 * The reference samples its measure nu with mu degrees of freedom through
 * Boost.Math: centered_cdf(x) = cdf(students_t(mu), x sqrt(mu)) and
 * centered_inv_cdf(u) = quantile(students_t(mu), u) / sqrt(mu)
 * (proj/src/student.cpp:60, 73) whenever mu is not 1 or 2. Boost is not vendored
 * and its version is unpinned (proj/CMakeLists.txt:12), so -- as for erfc_inv in
 * qrmc_normal_quantile.h -- this file DEFINES those two functions, Boost-free, and
 * the shim (oracle/shim), the C restatement (oracle/qrmc_oracle.c) and the device
 * (qrmc_device.cuh) all use this one definition. Parity with real Boost is
 * UNPINNED (no fixture of the reference pins it).
 *
 * Algorithms (standard, published):
 *   * regularised incomplete beta I_x(a, b) by the continued fraction of
 *     Numerical Recipes 6.4 (modified Lentz), prefactor from lgamma, with the
 *     symmetry I_x(a, b) = 1 - I_{1-x}(b, a) choosing the converging side and
 *     both x and 1 - x passed in so neither is formed by cancellation;
 *   * F_T(t) = 1/2 + sign(t)/2 * I_y(1/2, nu/2),  y = t^2 / (nu + t^2)
 *     (equivalently 1/2 I_{nu/(nu+t^2)}(nu/2, 1/2) for t < 0);
 *   * F_T^{-1}(u): lower tail p = min(u, 1-u), Newton on t with the closed-form
 *     density from a Cornish-Fisher start, safeguarded by bisection inside a
 *     bracket, sign restored. Fixed iteration caps, so the host and the device
 *     run the same sequence of operations (results agree to the last ulps of
 *     lgamma/log/exp/pow, which differ between glibc and CUDA).
 */
#ifndef QRMC_STUDENT_T_H
#define QRMC_STUDENT_T_H

#include "qrmc_normal_quantile.h"

#if !defined(__CUDA_ARCH__)
#include <math.h>
#endif

/* The general-mu path is rare and long (continued fractions, Newton): on the device it is
 * kept out of line so it cannot inflate the register allocation of the kernels that
 * merely contain it (K2's recompute branch spilled 1.7 KB per thread when it was inlined). */
#if defined(__CUDACC__)
#define QRMC_HD_COLD static __host__ __device__ __noinline__
#else
#define QRMC_HD_COLD static
#endif

#define QRMC_T_CF_ITERS 300
#define QRMC_T_NEWTON_ITERS 60

/* continued fraction of I_x(a, b) (NR 6.4, modified Lentz) */
QRMC_HD double qrmc_betacf(double a, double b, double x) {
    const double fpmin = 1e-300, eps = 1e-16;
    const double qab = a + b, qap = a + 1.0, qam = a - 1.0;
    double c = 1.0, d = 1.0 - qab * x / qap;
    if (fabs(d) < fpmin) d = fpmin;
    d = 1.0 / d;
    double h = d;
    for (int m = 1; m <= QRMC_T_CF_ITERS; ++m) {
        const double m2 = 2.0 * m;
        double aa = m * (b - m) * x / ((qam + m2) * (a + m2));
        d = 1.0 + aa * d;
        if (fabs(d) < fpmin) d = fpmin;
        c = 1.0 + aa / c;
        if (fabs(c) < fpmin) c = fpmin;
        d = 1.0 / d;
        h *= d * c;
        aa = -(a + m) * (qab + m) * x / ((a + m2) * (qap + m2));
        d = 1.0 + aa * d;
        if (fabs(d) < fpmin) d = fpmin;
        c = 1.0 + aa / c;
        if (fabs(c) < fpmin) c = fpmin;
        d = 1.0 / d;
        const double del = d * c;
        h *= del;
        if (fabs(del - 1.0) <= eps) break;
    }
    return h;
}

/* I_x(a, b) with y = 1 - x supplied by the caller */
QRMC_HD double qrmc_ibeta(double a, double b, double x, double y) {
    if (x <= 0.0) return 0.0;
    if (y <= 0.0) return 1.0;
    const double lbt = lgamma(a + b) - lgamma(a) - lgamma(b) + a * log(x) + b * log(y);
    const double bt = exp(lbt);
    if (x < (a + 1.0) / (a + b + 2.0)) return bt * qrmc_betacf(a, b, x) / a;
    return 1.0 - bt * qrmc_betacf(b, a, y) / b;
}

/* lower tail P(T <= -|t|) = 1/2 I_{nu/(nu+t^2)}(nu/2, 1/2) */
QRMC_HD double qrmc_student_lower(double t, double nu) {
    const double t2 = t * t, s = nu + t2;
    return 0.5 * qrmc_ibeta(0.5 * nu, 0.5, nu / s, t2 / s);
}

/* F_T(t) for nu degrees of freedom (boost::math::cdf(students_t(nu), t)) */
QRMC_HD_COLD double qrmc_student_cdf(double t, double nu) {
    if (!(t == t)) return t;
    const double lo = qrmc_student_lower(t, nu);
    return t < 0.0 ? lo : 1.0 - lo;
}

/* density of T */
QRMC_HD double qrmc_student_pdf(double t, double nu) {
    const double lc = lgamma(0.5 * (nu + 1.0)) - lgamma(0.5 * nu) - 0.5 * log(nu * 3.14159265358979323846);
    return exp(lc - 0.5 * (nu + 1.0) * log1p(t * t / nu));
}

/* F_T^{-1}(u), u in (0, 1) (boost::math::quantile(students_t(nu), u)): lower tail
 * p = min(u, 1-u), root of log P(T <= -t) = log p in s = log t (the tail is a power law
 * in t, so Newton in log t converges in a few steps even at p = 1e-15, nu < 1), started
 * inside a bracket found by factor-4 steps from a Cornish-Fisher guess and safeguarded by
 * geometric bisection of that bracket. */
QRMC_HD_COLD double qrmc_student_quantile(double u, double nu) {
    if (u == 0.5) return 0.0;
    const double p = u < 0.5 ? u : 1.0 - u;
    const double lp = log(p);
    const double z = -qrmc_normal_quantile(p);
    double t = z * (1.0 + (z * z + 1.0) / (4.0 * nu));
    if (!(t > 1e-300)) t = 1e-3;
    /* bracket [lo, hi]: lower(lo) >= p >= lower(hi) (lower() decreases in t) */
    double lo = t, hi = t;
    while (qrmc_student_lower(lo, nu) < p && lo > 1e-300) lo *= 0.25;
    while (qrmc_student_lower(hi, nu) > p && hi < 1e300) hi *= 4.0;
    if (!(t >= lo && t <= hi)) t = sqrt(lo * hi);
    for (int it = 0; it < QRMC_T_NEWTON_ITERS; ++it) {
        const double lw = qrmc_student_lower(t, nu);
        const double g = log(lw) - lp;
        if (g == 0.0) break;
        if (g > 0.0)
            lo = t;
        else
            hi = t;
        /* d log lower / d log t = -pdf(t) t / lower(t) */
        const double ds = g * lw / (qrmc_student_pdf(t, nu) * t);
        double nt = t * exp(ds);
        if (!(nt > lo && nt < hi)) nt = sqrt(lo * hi);
        if (fabs(nt - t) <= 2e-16 * nt) {
            t = nt;
            break;
        }
        t = nt;
    }
    return u < 0.5 ? -t : t;
}

#endif /* QRMC_STUDENT_T_H */

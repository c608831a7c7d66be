/* qrmc_normal_quantile.h -- inverse standard-normal CDF shared by the host
 * oracle shim and the sm_100a kernels.
 *
 * The reference computes Gaussian increments as
 *     normal_quantile(p) = -sqrt(2) * boost::math::erfc_inv(2 p)
 * (proj/src/rng.cpp:42-45, reached from RngStream::next_normal rng.cpp:47-49
 * and euler_step proj/src/sde.cpp:44). Boost is not vendored and its version is
 * unpinned (proj/CMakeLists.txt:12), so the bit pattern of erfc_inv is not
 * pinned by the reference either; its only pins are the four quantile values
 * of proj/tests/test_rng.cpp:72-78 (checked in tests/test_oracle.py).
 *
 * We define erfc_inv through Wichura's AS241 PPND16 rational approximation
 * (Applied Statistics 37 (1988) 477-484, relative accuracy ~1e-16):
 *     erfc_inv(z) = -ppnd16(z / 2) / sqrt(2)
 * and use this one definition in three places: the Boost shim the reference
 * sources are compiled against (oracle/shim), the C restatement (oracle/), and
 * the device code. Every multiply/add is spelled with QRMC_MUL/QRMC_ADD so the
 * device build cannot contract them into FMAs (host builds use
 * -ffp-contract=off); only log() may differ between glibc and CUDA, by <= 1 ulp.
 */
#ifndef QRMC_NORMAL_QUANTILE_H
#define QRMC_NORMAL_QUANTILE_H

#if defined(__CUDACC__)
#define QRMC_HD __host__ __device__ __forceinline__
#else
#define QRMC_HD static inline
#endif

#if defined(__CUDA_ARCH__)
#define QRMC_MUL(a, b) __dmul_rn((a), (b))
#define QRMC_ADD(a, b) __dadd_rn((a), (b))
#define QRMC_SUB(a, b) __dsub_rn((a), (b))
#define QRMC_DIV(a, b) __ddiv_rn((a), (b))
#define QRMC_SQRT(a) __dsqrt_rn(a)
#define QRMC_LOG(a) log(a)
#else
#include <math.h>
#define QRMC_MUL(a, b) ((a) * (b))
#define QRMC_ADD(a, b) ((a) + (b))
#define QRMC_SUB(a, b) ((a) - (b))
#define QRMC_DIV(a, b) ((a) / (b))
#define QRMC_SQRT(a) sqrt(a)
#define QRMC_LOG(a) log(a)
#endif

/* sqrt(2) rounded to double; boost::math::constants::root_two<double>(). */
#define QRMC_ROOT_TWO 1.41421356237309504880

/* Horner step without contraction: acc * r + c */
#define QRMC_HSTEP(acc, r, c) QRMC_ADD(QRMC_MUL((acc), (r)), (c))

/* The 48 coefficients of PPND16's three rational approximations (num, den of the
 * central region; num, den for r <= 5; num, den beyond), highest degree first. On the
 * device they live in a constant bank, so each Horner step takes its addend as a
 * constant-bank operand instead of materialising a 64-bit immediate (same values,
 * same operations, same bits). */
#define QRMC_NQ_COEFFS \
    2.5090809287301226727e+3, 3.3430575583588128105e+4, 6.7265770927008700853e+4, 4.5921953931549871457e+4, 1.3731693765509461125e+4, 1.9715909503065514427e+3, 1.3314166789178437745e+2, 3.3871328727963666080e+0, \
    5.2264952788528545610e+3, 2.8729085735721942674e+4, 3.9307895800092710610e+4, 2.1213794301586595867e+4, 5.3941960214247511077e+3, 6.8718700749205790830e+2, 4.2313330701600911252e+1, 1.0, \
    7.74545014278341407640e-4, 2.27238449892691845833e-2, 2.41780725177450611770e-1, 1.27045825245236838258e+0, 3.64784832476320460504e+0, 5.76949722146069140550e+0, 4.63033784615654529590e+0, 1.42343711074968357734e+0, \
    1.05075007164441684324e-9, 5.47593808499534494600e-4, 1.51986665636164571966e-2, 1.48103976427480074590e-1, 6.89767334985100004550e-1, 1.67638483018380384940e+0, 2.05319162663775882187e+0, 1.0, \
    2.01033439929228813265e-7, 2.71155556874348757815e-5, 1.24266094738807843860e-3, 2.65321895265761230930e-2, 2.96560571828504891230e-1, 1.78482653991729133580e+0, 5.46378491116411436990e+0, 6.65790464350110377720e+0, \
    2.04426310338993978564e-15, 1.42151175831644588870e-7, 1.84631831751005468180e-5, 7.86869131145613259100e-4, 1.48753612908506148525e-2, 1.36929880922735805310e-1, 5.99832206555887937690e-1, 1.0
#if defined(__CUDA_ARCH__)
static __constant__ double qrmc_nq_coef[48] = {QRMC_NQ_COEFFS};
#else
static const double qrmc_nq_coef[48] = {QRMC_NQ_COEFFS};
#endif
#define QRMC_NQC(i) qrmc_nq_coef[i]

QRMC_HD double qrmc_ppnd16(double p) {
    const double q = QRMC_SUB(p, 0.5);
    double r, num, den, val;
    if ((q < 0 ? -q : q) <= 0.425) {
        r = QRMC_SUB(0.180625, QRMC_MUL(q, q));
        num = QRMC_NQC(0);
        num = QRMC_HSTEP(num, r, QRMC_NQC(1));
        num = QRMC_HSTEP(num, r, QRMC_NQC(2));
        num = QRMC_HSTEP(num, r, QRMC_NQC(3));
        num = QRMC_HSTEP(num, r, QRMC_NQC(4));
        num = QRMC_HSTEP(num, r, QRMC_NQC(5));
        num = QRMC_HSTEP(num, r, QRMC_NQC(6));
        num = QRMC_HSTEP(num, r, QRMC_NQC(7));
        den = QRMC_NQC(8);
        den = QRMC_HSTEP(den, r, QRMC_NQC(9));
        den = QRMC_HSTEP(den, r, QRMC_NQC(10));
        den = QRMC_HSTEP(den, r, QRMC_NQC(11));
        den = QRMC_HSTEP(den, r, QRMC_NQC(12));
        den = QRMC_HSTEP(den, r, QRMC_NQC(13));
        den = QRMC_HSTEP(den, r, QRMC_NQC(14));
        den = QRMC_HSTEP(den, r, QRMC_NQC(15));
        return QRMC_DIV(QRMC_MUL(q, num), den);
    }
    r = q < 0 ? p : QRMC_SUB(1.0, p);
    r = QRMC_SQRT(-QRMC_LOG(r));
    if (r <= 5.0) {
        r = QRMC_SUB(r, 1.6);
        num = QRMC_NQC(16);
        num = QRMC_HSTEP(num, r, QRMC_NQC(17));
        num = QRMC_HSTEP(num, r, QRMC_NQC(18));
        num = QRMC_HSTEP(num, r, QRMC_NQC(19));
        num = QRMC_HSTEP(num, r, QRMC_NQC(20));
        num = QRMC_HSTEP(num, r, QRMC_NQC(21));
        num = QRMC_HSTEP(num, r, QRMC_NQC(22));
        num = QRMC_HSTEP(num, r, QRMC_NQC(23));
        den = QRMC_NQC(24);
        den = QRMC_HSTEP(den, r, QRMC_NQC(25));
        den = QRMC_HSTEP(den, r, QRMC_NQC(26));
        den = QRMC_HSTEP(den, r, QRMC_NQC(27));
        den = QRMC_HSTEP(den, r, QRMC_NQC(28));
        den = QRMC_HSTEP(den, r, QRMC_NQC(29));
        den = QRMC_HSTEP(den, r, QRMC_NQC(30));
        den = QRMC_HSTEP(den, r, QRMC_NQC(31));
    } else {
        r = QRMC_SUB(r, 5.0);
        num = QRMC_NQC(32);
        num = QRMC_HSTEP(num, r, QRMC_NQC(33));
        num = QRMC_HSTEP(num, r, QRMC_NQC(34));
        num = QRMC_HSTEP(num, r, QRMC_NQC(35));
        num = QRMC_HSTEP(num, r, QRMC_NQC(36));
        num = QRMC_HSTEP(num, r, QRMC_NQC(37));
        num = QRMC_HSTEP(num, r, QRMC_NQC(38));
        num = QRMC_HSTEP(num, r, QRMC_NQC(39));
        den = QRMC_NQC(40);
        den = QRMC_HSTEP(den, r, QRMC_NQC(41));
        den = QRMC_HSTEP(den, r, QRMC_NQC(42));
        den = QRMC_HSTEP(den, r, QRMC_NQC(43));
        den = QRMC_HSTEP(den, r, QRMC_NQC(44));
        den = QRMC_HSTEP(den, r, QRMC_NQC(45));
        den = QRMC_HSTEP(den, r, QRMC_NQC(46));
        den = QRMC_HSTEP(den, r, QRMC_NQC(47));
    }
    val = QRMC_DIV(num, den);
    return q < 0 ? -val : val;
}

/* qrmc_ppnd16's two branches on their own (the same operations, so the same results):
 * the central region |p - 1/2| <= 0.425 from q = p - 1/2, and the tails from
 * r = (q < 0 ? p : 1 - p), returning the magnitude (the caller applies the sign of q).
 * Kernels that batch the rare tail evaluations across a warp use these. */
QRMC_HD double qrmc_ppnd16_central(double q) {
    const double r = QRMC_SUB(0.180625, QRMC_MUL(q, q));
    double num = QRMC_NQC(0), den = QRMC_NQC(8);
    num = QRMC_HSTEP(num, r, QRMC_NQC(1));
    num = QRMC_HSTEP(num, r, QRMC_NQC(2));
    num = QRMC_HSTEP(num, r, QRMC_NQC(3));
    num = QRMC_HSTEP(num, r, QRMC_NQC(4));
    num = QRMC_HSTEP(num, r, QRMC_NQC(5));
    num = QRMC_HSTEP(num, r, QRMC_NQC(6));
    num = QRMC_HSTEP(num, r, QRMC_NQC(7));
    den = QRMC_HSTEP(den, r, QRMC_NQC(9));
    den = QRMC_HSTEP(den, r, QRMC_NQC(10));
    den = QRMC_HSTEP(den, r, QRMC_NQC(11));
    den = QRMC_HSTEP(den, r, QRMC_NQC(12));
    den = QRMC_HSTEP(den, r, QRMC_NQC(13));
    den = QRMC_HSTEP(den, r, QRMC_NQC(14));
    den = QRMC_HSTEP(den, r, QRMC_NQC(15));
    return QRMC_DIV(QRMC_MUL(q, num), den);
}

QRMC_HD double qrmc_ppnd16_tail(double r) {
    r = QRMC_SQRT(-QRMC_LOG(r));
    const int c = r <= 5.0 ? 16 : 32;
    r = QRMC_SUB(r, c == 16 ? 1.6 : 5.0);
    double num = QRMC_NQC(c), den = QRMC_NQC(c + 8);
    for (int j = 1; j < 8; ++j) {
        num = QRMC_HSTEP(num, r, QRMC_NQC(c + j));
        den = QRMC_HSTEP(den, r, QRMC_NQC(c + 8 + j));
    }
    return QRMC_DIV(num, den);
}

/* Boost-shaped erfc^{-1}(z), z in (0, 2). */
QRMC_HD double qrmc_erfc_inv(double z) {
    return QRMC_DIV(-qrmc_ppnd16(QRMC_MUL(0.5, z)), QRMC_ROOT_TWO);
}

/* normal_quantile exactly as proj/src/rng.cpp:42-45 composes it. */
QRMC_HD double qrmc_normal_quantile(double p) {
    return QRMC_MUL(-QRMC_ROOT_TWO, qrmc_erfc_inv(QRMC_MUL(2.0, p)));
}

#endif /* QRMC_NORMAL_QUANTILE_H */

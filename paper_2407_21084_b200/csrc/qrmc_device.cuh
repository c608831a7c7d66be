// qrmc_device.cuh -- device-side building blocks of the backward solver.
//
// Every function here is the sm_100a counterpart of one reference routine
// (file:line cited per function). The replay-critical arithmetic (random
// draws, sampling, Euler, truncation, weights, functors) is spelled with
// explicit round-to-nearest intrinsics so ptxas cannot contract it into FMAs:
// the reference's numerics contain no FMA, and with this the
// device reproduces the reference's Philox words, uniforms and mu=2 starts
// bit for bit and its Gaussians and Euler paths to the last ulp of log().
// The series evaluation (the FLOP-dominant part) is the one place that uses
// FMAs and a re-associated (sum-factorised) order; its deviation is covered
// by the stated FP64 tolerance ("Parity").
#pragma once

#include <cstdint>

#include "qrmc_gpu.h"
#include "qrmc_normal_quantile.h"
#include "qrmc_student_t.h"
#include "qrmc_types.h"

namespace qrmc_dev {


#define DMUL(a, b) __dmul_rn((a), (b))
#define DADD(a, b) __dadd_rn((a), (b))
#define DSUB(a, b) __dsub_rn((a), (b))
#define DDIV(a, b) __ddiv_rn((a), (b))

// ------------------------------------------------------------------ Philox
// Philox4x32-10 (proj/src/rng.cpp:9-40): multipliers 0xD2511F53/0xCD9E8D57,
// Weyl increments 0x9E3779B9/0xBB67AE85, key bumped before rounds 1..9.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r > 0) {
            k.x += 0x9E3779B9u;
            k.y += 0xBB67AE85u;
        }
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    }
    return c;
}

// RngStream (rng.hpp:26-65): key = seed, counter = (block lo, block hi,
// stream id lo, stream id hi); each block yields two u64 draws
// (o1<<32|o0), (o3<<32|o2).
struct Stream {
    uint2 key;
    uint32_t sid_lo, sid_hi;
    uint64_t block;
    uint64_t buf1;
    int pos;  // 0: buf empty, 1: buf1 holds the second half

    __device__ __forceinline__ Stream() : key(make_uint2(0u, 0u)), sid_lo(0), sid_hi(0), block(0), buf1(0), pos(0) {}
    __device__ __forceinline__ Stream(uint64_t seed, uint64_t sid)
        : key(make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32))),
          sid_lo(static_cast<uint32_t>(sid)), sid_hi(static_cast<uint32_t>(sid >> 32)),
          block(0), buf1(0), pos(0) {}

    __device__ __forceinline__ uint64_t next_u64() {
        if (pos == 1) {
            pos = 0;
            return buf1;
        }
        const uint4 o = philox4x32_10(
            make_uint4(static_cast<uint32_t>(block), static_cast<uint32_t>(block >> 32), sid_lo, sid_hi),
            key);
        ++block;
        buf1 = (static_cast<uint64_t>(o.w) << 32) | o.z;
        pos = 1;
        return (static_cast<uint64_t>(o.y) << 32) | o.x;
    }
    // ((x >> 12) + 0.5) * 2^-52 (rng.hpp:41-43): exact in binary64, formed without an
    // integer->double conversion (m = x >> 12 in the mantissa of 1.0, minus 1, plus 2^-53;
    // every step exact, so the same double)
    __device__ __forceinline__ double next_uniform() {
        const uint64_t m = next_u64() >> 12;
        return DADD(DSUB(__longlong_as_double(static_cast<long long>(0x3FF0000000000000ull | m)), 1.0), 0x1p-53);
    }
    // normal_quantile(next_uniform()) (rng.cpp:42-49)
    __device__ __forceinline__ double next_normal() { return qrmc_normal_quantile(next_uniform()); }
};

// qrmc_normal_quantile with PPND16's two branches evaluated side by side and selected
// (the same operations on every value, so the same double): for a warp that holds both
// central and tail lanes -- nearly every warp -- the divergent form runs the branches one
// after the other, this form issues the two dependent chains interleaved, which shortens
// a latency-bound producer's critical path.
__device__ __forceinline__ double normal_quantile_ilp(double p) {
    const double pp = QRMC_MUL(0.5, QRMC_MUL(2.0, p));  // erfc_inv(2p)'s argument to PPND16
    const double q = QRMC_SUB(pp, 0.5);
    const double c = qrmc_ppnd16_central(q);
    const double t = qrmc_ppnd16_tail(q < 0 ? pp : QRMC_SUB(1.0, pp));
    const double v = (q < 0 ? -q : q) <= 0.425 ? c : (q < 0 ? -t : t);
    return QRMC_MUL(-QRMC_ROOT_TWO, QRMC_DIV(-v, QRMC_ROOT_TWO));
}

__device__ __forceinline__ uint64_t sid_training(int step, uint64_t path) {
    return (static_cast<uint64_t>(step) << kStepShift) | path;
}
__device__ __forceinline__ uint64_t sid_evaluation(int step, uint64_t point) {
    return (uint64_t{1} << 63) | (static_cast<uint64_t>(step) << kStepShift) | point;
}

// ------------------------------------------------------------------ measure
// Product Student-t measure for mu in {1, 2} (proj/src/student.cpp:53-106).


// centered_cdf + center shift (student.cpp:53-63, 78-82). GEN = false compiles the
// general-mu branch out: the hot tensor-core kernels are instantiated both ways and the
// plan picks the general one only for mu not in {1, 2} (a call to the out-of-line
// Student's t code would otherwise force their register state across a call).
template <bool GEN = true>
__device__ __forceinline__ double measure_cdf(const MeasureDev& m, double x, int l) {
    x = DSUB(x, m.center[l]);
    if (m.form == 1) return DADD(0.5, DDIV(atan(x), 3.14159265358979323846));
    if constexpr (GEN)
        if (m.form == 3) return qrmc_student_cdf(DMUL(x, m.sqrt_mu), m.mu);  // cdf(students_t(mu), x sqrt(mu))
    return DMUL(0.5, DADD(DDIV(x, __dsqrt_rn(DADD(DMUL(x, x), 1.0))), 1.0));
}

// inv_cdf with the 1e-15 guard band (student.cpp:65-76, 84-89)
template <bool GEN = true>
__device__ __forceinline__ double measure_inv_cdf(const MeasureDev& m, double u, int l) {
    const double g = 1e-15;
    u = u < g ? g : u;
    u = (1.0 - g) < u ? (1.0 - g) : u;
    double c;
    if (m.form == 1)
        c = tan(DMUL(3.14159265358979323846, DSUB(u, 0.5)));
    else if (GEN && m.form == 3)
        c = DDIV(qrmc_student_quantile(u, m.mu), m.sqrt_mu);  // quantile(students_t(mu), u) / sqrt(mu)
    else
        c = DDIV(DSUB(u, 0.5), __dsqrt_rn(DMUL(u, DSUB(1.0, u))));
    return DADD(c, m.center[l]);
}

// ------------------------------------------------------------------ problem
// Device functors replacing ProblemSpec's std::function members
// (sde.hpp:23-29; SinBenchmark functors benchmark.cpp:46-62).


// All functors take the state dimension D as a template parameter so every
// per-coordinate loop unrolls and point arrays stay in registers.
template <int D>
__device__ __forceinline__ double sum_of(const double* x) {
    double s = 0.0;
#pragma unroll
    for (int l = 0; l < D; ++l) s = DADD(s, x[l]);
    return s;
}

template <int D>
__device__ __forceinline__ double terminal(const ProblemDev& p, const double* x) {
    switch (p.terminal_kind) {
        case QRMC_TERMINAL_SIN_SUM: return DADD(DADD(1.0, p.tp0), sin(DMUL(p.tp1, sum_of<D>(x))));
        case QRMC_TERMINAL_CONST: return p.tp0;
        case QRMC_TERMINAL_X0: return x[0];
        default: return DDIV(1.0, DSUB(x[0], x[0]));
    }
}

template <int D>
__device__ __forceinline__ double driver(const ProblemDev& p, double t, const double* x, double y) {
    switch (p.driver_kind) {
        case QRMC_DRIVER_ZERO: return 0.0;
        case QRMC_DRIVER_CONST: return p.dp0;
        case QRMC_DRIVER_Y: return y;
        default: {
            // y - kappa - 1 - sin(lam sum x) * exp(lam*lam*d*(t-T)/2)  (benchmark.cpp:57-61)
            const double e = exp(DDIV(DMUL(DMUL(DMUL(p.dp1, p.dp1), static_cast<double>(D)),
                                           DSUB(t, p.horizon)), 2.0));
            const double z = DSUB(DSUB(DSUB(y, p.dp0), 1.0), DMUL(sin(DMUL(p.dp1, sum_of<D>(x))), e));
            const double zz = DMUL(z, z);
            return zz < 1.0 ? zz : 1.0;
        }
    }
}

// driver() split into its x-dependent part (evaluated ahead, off the critical
// path) and the combination with y; driver_apply(p, driver_pre<D>(p, t, x), y)
// performs exactly driver<D>(p, t, x, y)'s operations.
template <int D>
__device__ __forceinline__ double driver_pre(const ProblemDev& p, double t, const double* x) {
    if (p.driver_kind != QRMC_DRIVER_SIN_BENCH) return 0.0;
    const double e = exp(DDIV(DMUL(DMUL(DMUL(p.dp1, p.dp1), static_cast<double>(D)), DSUB(t, p.horizon)), 2.0));
    return DMUL(sin(DMUL(p.dp1, sum_of<D>(x))), e);
}
__device__ __forceinline__ double driver_apply(const ProblemDev& p, double pre, double y) {
    switch (p.driver_kind) {
        case QRMC_DRIVER_ZERO: return 0.0;
        case QRMC_DRIVER_CONST: return p.dp0;
        case QRMC_DRIVER_Y: return y;
        default: {
            const double z = DSUB(DSUB(DSUB(y, p.dp0), 1.0), pre);
            const double zz = DMUL(z, z);
            return zz < 1.0 ? zz : 1.0;
        }
    }
}

// lstar_bound (sde.cpp:27-35)
template <int D>
__device__ __forceinline__ double lstar(const ProblemDev& p, const double* x) {
    if (p.eta == 0.0) return p.lstar_base;
    double n2 = 0.0;
#pragma unroll
    for (int l = 0; l < D; ++l) n2 = DADD(n2, DMUL(x[l], x[l]));
    return DMUL(p.lstar_base, pow(DADD(1.0, n2), DDIV(p.eta, 2.0)));
}

// damping_weight (solver.cpp:43-48)
template <int D>
__device__ __forceinline__ double damping_weight(const double* x, double q) {
    if (q == 0.0) return 1.0;
    double n2 = 0.0;
#pragma unroll
    for (int l = 0; l < D; ++l) n2 = DADD(n2, DMUL(x[l], x[l]));
    return pow(DADD(1.0, n2), DDIV(q, 2.0));
}

// truncate_soft (solver.cpp:37-41): std::min(std::max(v, -b), b)
__device__ __forceinline__ double truncate_soft(double v, double b) {
    const double lo = -b;
    v = v < lo ? lo : v;
    return b < v ? b : v;
}

// One coordinate of euler_step (sde.cpp:37-73): out = sigma(t, x) dw (diffusion_apply,
// identity when null), x_l += b_l(t, x) dt + out_l with the drift at the pre-step state.
// Every device drift/diffusion is diagonal, so coordinate l needs only x_l and dw_l.
__device__ __forceinline__ double euler_coord(const ProblemDev& p, double xo, double dw, int l, double dt) {
    const double out = p.diffusion_kind == QRMC_DIFFUSION_SCALAR ? DMUL(p.sigma, dw)
                       : p.diffusion_kind == QRMC_DIFFUSION_DIAG ? DMUL(p.sig[l], dw)
                                                                  : dw;
    if (p.drift_kind == QRMC_DRIFT_CONST) return DADD(xo, DADD(DMUL(p.drift_c, dt), out));
    if (p.drift_kind == QRMC_DRIFT_AFFINE)
        return DADD(xo, DADD(DMUL(DADD(p.drift_a[l], DMUL(p.drift_b[l], xo)), dt), out));
    return DADD(xo, out);
}

// euler_step in place (sde.cpp:37-73); device diffusions have brownian_dim == D.
// Returns 0 or the SimulationError step.
template <int D>
__device__ __forceinline__ int euler_step(const ProblemDev& p, double* x, double sqrt_dt, double dt,
                                          Stream& s, int j) {
    double dw[D];
#pragma unroll
    for (int l = 0; l < D; ++l) dw[l] = DMUL(sqrt_dt, s.next_normal());
    int bad = 0;
#pragma unroll
    for (int l = 0; l < D; ++l) {
        const double v = euler_coord(p, x[l], dw[l], l, dt);
        x[l] = v;
        if (!isfinite(v) || fabs(v) > p.state_bound) bad = j + 1;
    }
    return bad;
}

// flags[0] = error kind, the larger wins (QRMC_ESIM over QRMC_ENUMERIC), so the
// outcome does not depend on which path or rank fails first (the reference
// rethrows whichever lane exception comes first, parallel.cpp:22-43);
// flags[1] = smallest SimulationError step. The multi-rank solve all-reduces both
// with the same operators (host.cpp enqueue_solve).
__device__ __forceinline__ void record_error(int* flags, int kind, int step) {
    atomicMax(flags, kind);
    if (kind == QRMC_ESIM) atomicMin(flags + 1, step);
}

}  // namespace qrmc_dev

// srmc.cu -- stratified regression Monte Carlo on sm_100a.
//
// The scheme, tables and C ABI are specified in include/qrmc_srmc.h. One warp owns one
// hypercube of one backward step: its 32 lanes draw the cell's M paths (counter-based
// Philox keyed by (seed; step, cell*M + path) -- rng.hpp:26-65 with the cell folded into
// the path counter), take the Euler step (sde.cpp:37-73), gather the next step's local
// polynomial of the cell the endpoint lands in (P doubles, read-only path), apply the
// driver functor and accumulate the cell's normal equations in registers. A butterfly of
// warp shuffles reduces them and every lane solves the P x P system (Cholesky, FP64,
// registers). Paths never touch HBM; per step the only traffic is the gather of the
// step-(i+1) table (L2-resident neighbourhoods: one Euler step moves ~sqrt(dt) << h)
// and the write of the step-i table. When the driver reads z (Bergman) the warp runs
// the cell twice: pass 1 fits Z, pass 2 replays the SAME draws (counter-based stream, no
// storage) and fits Y with f(t_{i+1}, X_{i+1}, Y1, Zhat_i(X_i)).
//
// Replay-critical arithmetic (starts, Euler, cell index) is spelled with _rn intrinsics
// so it matches oracle/srmc_oracle.c (built with -ffp-contract=off) bit for bit; the
// reduction order differs (per-lane strided partials + butterfly), covered by the
// stated tolerance (tests/test_srmc.py).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "qrmc_device.cuh"
#include "qrmc_srmc.h"
#include "srmc_types.h"

namespace qrmc_srmc_dev {

using namespace qrmc_dev;

namespace {

template <int D>
__device__ __forceinline__ double srmc_terminal(const SrmcDev& s, const double* x) {
    double sum = 0.0;
#pragma unroll
    for (int l = 0; l < D; ++l) sum = DADD(sum, x[l]);
    if (s.kind == QRMC_SRMC_SIN_BENCH) return DADD(DADD(1.0, s.p[0]), sin(DMUL(s.p[1], sum)));
    const double v = DSUB(exp(DMUL(sum, 1.0 / D)), s.p[4]);  // 1/D: a compile-time constant, as the oracle's
    return v > 0.0 ? v : 0.0;
}

// driver f(t, x, y, z): SinBenchmark (benchmark.cpp:46-62, no z) or Bergman.
template <int D>
__device__ __forceinline__ double srmc_driver(const SrmcDev& s, const double* x, double y, const double* z) {
    if (s.kind == QRMC_SRMC_SIN_BENCH) {
        double sum = 0.0;
#pragma unroll
        for (int l = 0; l < D; ++l) sum = DADD(sum, x[l]);
        const double w = DSUB(DSUB(DSUB(y, s.p[0]), 1.0), DMUL(sin(DMUL(s.p[1], sum)), s.decay));
        const double ww = DMUL(w, w);
        return ww < 1.0 ? ww : 1.0;
    }
    // p[5] = theta = (mu - r_l) / sigma and p[6] = 1 / sigma, hoisted to the host (make_dev)
    const double rl = s.p[2], rb = s.p[3], theta = s.p[5], inv_sg = s.p[6];
    double zs = 0.0;
#pragma unroll
    for (int l = 0; l < D; ++l) zs = DADD(zs, z[l]);
    const double borrow = DSUB(DMUL(zs, inv_sg), y);
    return DADD(DSUB(DMUL(-rl, y), DMUL(theta, zs)), DMUL(DSUB(rb, rl), borrow > 0.0 ? borrow : 0.0));
}

// yhat_{i+1}(x): projection onto the box, cell index (bit-exact), local polynomial.
template <int D, int P>
__device__ __forceinline__ double srmc_eval(const SrmcDev& s, const double* __restrict__ tab, const double* x) {
    int64_t k = 0;
    int cs[D];
    double sl[D];
#pragma unroll
    for (int l = 0; l < D; ++l) {
        double xc = x[l] < s.lo ? s.lo : x[l];
        xc = xc > s.hi ? s.hi : xc;
        int c = static_cast<int>(floor(DMUL(DSUB(xc, s.lo), s.inv_h)));  // the reciprocal, as the oracle
        c = c < 0 ? 0 : (c >= s.n ? s.n - 1 : c);
        cs[l] = c;
        k = k * s.n + c;
        const double centre = DADD(s.lo, DMUL(DADD(static_cast<double>(c), 0.5), s.h));
        sl[l] = DMUL(DSUB(xc, centre), s.inv2h);
    }
    if (s.morton) k = morton_encode<D>(cs, s.mmul, s.mmask);
    const double* row = tab + k * P;
    double v = __ldg(row);
    if constexpr (P > 1) {
#pragma unroll
        for (int l = 0; l < D; ++l) v = fma(__ldg(row + 1 + l), sl[l], v);
    }
    return v;
}

// butterfly over the G lanes of one hypercube (xor offsets < G stay inside the group)
template <int NV, int G>
__device__ __forceinline__ void warp_sum(double* a) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) a[j] += __shfl_xor_sync(0xffffffffu, a[j], o);
    }
}

// Cholesky solve of the P x P normal equations (packed upper triangle A, row-major
// a(r,c) r <= c) for nr right-hand sides b[nr][P]; a zero/negative pivot zeroes that
// coefficient (degenerate cell: fewer distinct points than unknowns).
template <int P, int NR>
__device__ __forceinline__ void chol_solve(const double* A, double* b) {
    double Lm[P][P];
#pragma unroll
    for (int r = 0; r < P; ++r)
#pragma unroll
        for (int c = 0; c < P; ++c) Lm[r][c] = 0.0;
    int idx = 0;
    double a[P][P];
#pragma unroll
    for (int r = 0; r < P; ++r)
#pragma unroll
        for (int c = r; c < P; ++c) {
            a[r][c] = A[idx];
            a[c][r] = A[idx];
            ++idx;
        }
#pragma unroll
    for (int j = 0; j < P; ++j) {
        double d = a[j][j];
#pragma unroll
        for (int q = 0; q < j; ++q) d -= Lm[j][q] * Lm[j][q];
        const double ljj = d > 1e-300 ? sqrt(d) : 0.0;
        Lm[j][j] = ljj;
#pragma unroll
        for (int r = j + 1; r < P; ++r) {
            double v = a[r][j];
#pragma unroll
            for (int q = 0; q < j; ++q) v -= Lm[r][q] * Lm[j][q];
            Lm[r][j] = ljj > 0.0 ? v / ljj : 0.0;
        }
    }
#pragma unroll
    for (int h = 0; h < NR; ++h) {
        double* y = b + h * P;
#pragma unroll
        for (int r = 0; r < P; ++r) {
            double v = y[r];
#pragma unroll
            for (int q = 0; q < r; ++q) v -= Lm[r][q] * y[q];
            y[r] = Lm[r][r] > 0.0 ? v / Lm[r][r] : 0.0;
        }
#pragma unroll
        for (int r = P - 1; r >= 0; --r) {
            double v = y[r];
#pragma unroll
            for (int q = r + 1; q < P; ++q) v -= Lm[q][r] * y[q];
            y[r] = Lm[r][r] > 0.0 ? v / Lm[r][r] : 0.0;
        }
    }
}

// SRMC's Gaussian increments are PPND16(u) itself (AS241, include/qrmc_normal_quantile.h):
// the reference's composition -sqrt(2) * erfc_inv(2u) = -sqrt(2) * (-PPND16(u) / sqrt(2))
// adds a division and a multiplication that only matter for bit parity with the GQRMDP
// reference path; SRMC's draws are its own (oracle/srmc_oracle.c does the same). Both
// branches are inlined now that the tail runs once per warp round rather than once per
// draw (out-of-line copies measured 4% / 2% slower).

// PPND16 for the D Gaussian increments of one path per lane, the tails batched over the
// warp. About 15% of uniforms fall in the tails (|u - 1/2| > 0.425), so nearly every warp
// of 32 lanes holds one and, evaluated per lane, every quantile would cost the warp the
// central rational AND the tail's log, sqrt and rational. Here each lane evaluates its D
// central rationals, then the warp's tail arguments (ballot prefix over the lanes) are
// dealt out one per lane through shared memory and evaluated in ceil(tails / 32) rounds.
// Every value goes through the same operations as qrmc_ppnd16 (bit-identical).
// All 32 lanes must call it together (the kernel runs uniform trip counts).
__device__ __forceinline__ double srmc_central(double q) { return qrmc_ppnd16_central(q); }
__device__ __forceinline__ double srmc_tail(double r) { return qrmc_ppnd16_tail(r); }

template <int D>
__device__ __forceinline__ void srmc_quantiles(double* uz, double* scratch) {
    // uz: the D uniforms in, the D normals out (in place, to keep registers down)
    static_assert(D <= 7, "tail counts are gathered in three ballot bits");
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    unsigned tails = 0, neg = 0;
#pragma unroll
    for (int l = 0; l < D; ++l) {
        const double q = DSUB(uz[l], 0.5);
        if ((q < 0 ? -q : q) > 0.425) tails |= 1u << l;
        if (q < 0) neg |= 1u << l;
    }
    const int cnt = __popc(tails);
    const unsigned b0 = __ballot_sync(0xffffffffu, cnt & 1), b1 = __ballot_sync(0xffffffffu, cnt & 2),
                   b2 = __ballot_sync(0xffffffffu, cnt & 4);
    const int total = __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2);
    const int excl = __popc(b0 & lt) + 2 * __popc(b1 & lt) + 4 * __popc(b2 & lt);
    if (total) {  // warp-uniform
        int o = excl;
#pragma unroll
        for (int l = 0; l < D; ++l)
            if ((tails >> l) & 1u) scratch[o++] = (neg >> l) & 1u ? uz[l] : DSUB(1.0, uz[l]);
    }
#pragma unroll
    for (int l = 0; l < D; ++l) uz[l] = srmc_central(DSUB(uz[l], 0.5));
    if (total == 0) return;
    __syncwarp();
    for (int g = lane; g < total; g += 32) scratch[g] = srmc_tail(scratch[g]);
    __syncwarp();
    {
        int o = excl;
#pragma unroll
        for (int l = 0; l < D; ++l)
            if ((tails >> l) & 1u) {
                const double v = scratch[o++];
                uz[l] = (neg >> l) & 1u ? -v : v;
            }
    }
    __syncwarp();  // the scratch is reused by the next path
}

// One path of cell k: start X_i (and its local coordinates), dW, endpoint response Y1.
template <int D, int P>
__device__ __forceinline__ void srmc_path(const SrmcDev& s, const double* __restrict__ next, const int* cc,
                                          int64_t k, int64_t m, double* x0, double* sl, double* dw, double* x1, double& y1,
                                          double* scratch) {
    // The path's 2D draws are blocks 0..D-1 of its stream (draw n = half n&1 of block n>>1,
    // rng.hpp:26-65): uniforms 0..D-1 place the start, D..2D-1 are the Gaussian increments.
    // Round keys come precomputed from the launch parameters (no per-thread key schedule).
    const uint64_t sid = sid_training(s.step, static_cast<uint64_t>(k) * static_cast<uint64_t>(s.M) + m);
    auto block = [&](int b) {
        uint4 c = make_uint4(static_cast<uint32_t>(b), 0u, static_cast<uint32_t>(sid), static_cast<uint32_t>(sid >> 32));
#pragma unroll
        for (int r = 0; r < 10; ++r) {
            const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
            const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
            c = make_uint4(hi1 ^ c.y ^ s.rk[2 * r], lo1, hi0 ^ c.w ^ s.rk[2 * r + 1], lo0);
        }
        return c;
    };
    // u = ((x >> 12) + 1/2) 2^-52 (rng.hpp:41-43). (The conversion-free form K1 uses,
    // mma_common.cuh u64_to_uniform, is 1% slower here: this kernel is FP64-pipe bound and
    // the integer->double conversion is not on that pipe.)
    auto uni = [](uint32_t lo, uint32_t hi) {
        const uint64_t x = (static_cast<uint64_t>(hi) << 32) | lo;
        return DMUL(DADD(static_cast<double>(x >> 12), 0.5), 0x1p-52);
    };
    // the Gaussian increments first (draws D..2D-1, so the words die before the start is
    // drawn), then the start (draws 0..D-1); with D odd, block D/2 holds one of each
    double uz[D];
    uint4 shared_block = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
    for (int b = D / 2; b < D; ++b) {
        const uint4 c = block(b);
        if (2 * b >= D) uz[2 * b - D] = uni(c.x, c.y);
        else shared_block = c;
        if (2 * b + 1 < 2 * D) uz[2 * b + 1 - D] = uni(c.z, c.w);
    }
    srmc_quantiles<D>(uz, scratch);
#pragma unroll
    for (int b = 0; b < (D + 1) / 2; ++b) {
        const uint4 c = (D % 2 == 1 && b == D / 2) ? shared_block : block(b);
        const double u0 = uni(c.x, c.y);
        x0[2 * b] = DADD(s.lo, DMUL(DADD(static_cast<double>(cc[2 * b]), u0), s.h));
        sl[2 * b] = DSUB(DMUL(2.0, u0), 1.0);
        if (2 * b + 1 < D) {
            const double u1 = uni(c.z, c.w);
            x0[2 * b + 1] = DADD(s.lo, DMUL(DADD(static_cast<double>(cc[2 * b + 1]), u1), s.h));
            sl[2 * b + 1] = DSUB(DMUL(2.0, u1), 1.0);
        }
    }
#pragma unroll
    for (int l = 0; l < D; ++l) {
        dw[l] = DMUL(s.sqrt_dt, uz[l]);
        x1[l] = DADD(DADD(x0[l], s.bdt), DMUL(s.sig, dw[l]));
    }
    if (s.last) {
        y1 = srmc_terminal<D>(s, x1);
    } else {
        y1 = srmc_eval<D, P>(s, next, x1);
        y1 = y1 < -s.L ? -s.L : (y1 > s.L ? s.L : y1);
    }
}

template <int D, int P>
__device__ __forceinline__ void phi_of(const double* sl, double* phi) {
    phi[0] = 1.0;
#pragma unroll
    for (int l = 0; l + 1 < P; ++l) phi[1 + l] = sl[l];
}

template <int D, int P>
__device__ __forceinline__ void acc_gram(double* A, const double* phi) {
    int idx = 0;
#pragma unroll
    for (int r = 0; r < P; ++r)
#pragma unroll
        for (int c = r; c < P; ++c) A[idx++] += phi[r] * phi[c];
}

// ZPASS: the driver reads z -> pass 1 fits Z, pass 2 replays and fits Y.
// WANTZ: fit Z alongside Y in a single pass (driver without z).
// G lanes per hypercube: 32 (one warp) normally, 8 when M is small so the per-cell
// butterfly + Cholesky is amortised over more path iterations per lane.
// CACHE (ZPASS with the Bergman driver, which reads y and Z_hat but not x): pass 1 parks
// each path's (Y1, local coordinates) in dynamic shared memory and pass 2 reads them back
// instead of regenerating the path (the same doubles, so the same tables).
template <int D, int P, bool ZPASS, bool WANTZ, int G, bool CACHE = false>
__global__ void __launch_bounds__(256, (P == 1 ? 3 : ((ZPASS || WANTZ) && D * P >= 20 ? 1 : 2))) k_srmc_step(SrmcDev s, const double* __restrict__ next,
                                                   double* __restrict__ ytab, double* __restrict__ ztab) {
    static_assert(!CACHE || ZPASS, "the path cache serves the second pass");
    constexpr int NA = P * (P + 1) / 2;
    constexpr bool ANYZ = ZPASS || WANTZ;
    const int lane = threadIdx.x & 31;
    const int sub = lane & (G - 1);
    const int64_t kfirst =
        s.k0 + (static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5)) * (32 / G);
    if (kfirst >= s.k1) return;  // whole warps exit together
    const int64_t row = kfirst + lane / G;  // table row; the cell itself when not Morton-ordered
    const bool live = row < s.k1;  // a tail group past the range still joins the shuffles
    const int64_t mend = live ? s.M : 0;
    int cc[D];
    int64_t k = row;  // lexicographic cell index (keys the draws)
    if (s.morton) {
        morton_decode<D>(row, s.mbits, cc);
        k = 0;
#pragma unroll
        for (int l = 0; l < D; ++l) k = k * s.n + cc[l];
    } else {
        int64_t r = row;
#pragma unroll
        for (int l = D - 1; l >= 0; --l) {
            cc[l] = static_cast<int>(r % s.n);
            r /= s.n;
        }
    }
    double A[NA];
    double by[P];
    double bz[ANYZ ? D * P : 1];
#pragma unroll
    for (int j = 0; j < NA; ++j) A[j] = 0.0;
#pragma unroll
    for (int j = 0; j < P; ++j) by[j] = 0.0;
#pragma unroll
    for (int j = 0; j < (ANYZ ? D * P : 1); ++j) bz[j] = 0.0;

    // every lane runs the warp's trip count (srmc_quantiles is warp-collective); a lane's
    // iterations past its own paths (m >= mend) accumulate nothing, so each lane still sums
    // exactly its paths sub, sub + G, ... in order
    __shared__ double tail_scratch[8][32 * D];  // 8 warps per block (launch_step_t)
    double* scratch = tail_scratch[threadIdx.x >> 5];
    const int64_t iters = (s.M + G - 1) / G;
    double x0[D], sl[D], dw[D], x1[D], phi[P], y1;
    const double zero_z[D] = {};
    extern __shared__ double path_cache[];  // CACHE: [warp][it][1 + D][32 lanes]
    double* pc = path_cache + static_cast<size_t>(threadIdx.x >> 5) * iters * (1 + D) * 32 + lane;
    for (int64_t it = 0; it < iters; ++it) {
        const int64_t m = sub + it * G;
        srmc_path<D, P>(s, next, cc, k, m, x0, sl, dw, x1, y1, scratch);
        if constexpr (CACHE) {
            double* e = pc + it * (1 + D) * 32;
            e[0] = y1;
#pragma unroll
            for (int l = 0; l < D; ++l) e[(1 + l) * 32] = sl[l];
        }
        if (m >= mend) continue;
        phi_of<D, P>(sl, phi);
        acc_gram<D, P>(A, phi);
        if constexpr (ANYZ) {
#pragma unroll
            for (int l = 0; l < D; ++l) {
                const double rz = DMUL(DMUL(y1, dw[l]), s.inv_dt);
#pragma unroll
                for (int p = 0; p < P; ++p) bz[l * P + p] += rz * phi[p];
            }
        }
        if constexpr (!ZPASS) {
            const double ry = DADD(y1, DMUL(s.dt, srmc_driver<D>(s, x1, y1, zero_z)));
#pragma unroll
            for (int p = 0; p < P; ++p) by[p] += ry * phi[p];
        }
    }
    warp_sum<NA, G>(A);
    if constexpr (ANYZ) {
        warp_sum<D * P, G>(bz);
        chol_solve<P, D>(A, bz);
    }
    if constexpr (ZPASS) {
        for (int64_t it = 0; it < iters; ++it) {
            const int64_t m = sub + it * G;
            if constexpr (CACHE) {
                if (m >= mend) continue;
                const double* e = pc + it * (1 + D) * 32;
                y1 = e[0];
#pragma unroll
                for (int l = 0; l < D; ++l) sl[l] = e[(1 + l) * 32];
            } else {
                srmc_path<D, P>(s, next, cc, k, m, x0, sl, dw, x1, y1, scratch);
                if (m >= mend) continue;
            }
            phi_of<D, P>(sl, phi);
            double zi[D];
#pragma unroll
            for (int l = 0; l < D; ++l) {
                double v = bz[l * P];
#pragma unroll
                for (int p = 1; p < P; ++p) v = fma(bz[l * P + p], phi[p], v);
                zi[l] = v;
            }
            const double ry = DADD(y1, DMUL(s.dt, srmc_driver<D>(s, x1, y1, zi)));
#pragma unroll
            for (int p = 0; p < P; ++p) by[p] += ry * phi[p];
        }
    }
    warp_sum<P, G>(by);
    chol_solve<P, 1>(A, by);
    if (live && sub == 0) {
        bool finite = true;
#pragma unroll
        for (int p = 0; p < P; ++p) {
            ytab[row * P + p] = by[p];
            finite = finite && isfinite(by[p]);
        }
        if (!finite) *s.bad = 1;  // NumericError (every step's table, not only the last)
        if constexpr (ANYZ) {
#pragma unroll
            for (int j = 0; j < D * P; ++j) ztab[row * D * P + j] = bz[j];
        }
    }
}

template <int D, int P>
__global__ void k_srmc_eval(SrmcDev s, const double* __restrict__ tab, const double* __restrict__ x, int64_t n,
                            double* __restrict__ out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double xi[D];
#pragma unroll
    for (int l = 0; l < D; ++l) xi[l] = x[i * D + l];
    out[i] = srmc_eval<D, P>(s, tab, xi);
}

}  // namespace

void set_err(char* err, size_t len, const char* msg) {
    if (err && len) {
        std::strncpy(err, msg, len - 1);
        err[len - 1] = '\0';
    }
}

bool needs_z(const qrmc_srmc_problem_t* p) { return p->kind == QRMC_SRMC_BERGMAN; }

int validate(const qrmc_srmc_problem_t* p, const qrmc_srmc_config_t* c, char* err, size_t el) {
    if (!p || !c) return set_err(err, el, "null problem/config"), QRMC_EINVAL;
    if (p->kind != QRMC_SRMC_SIN_BENCH && p->kind != QRMC_SRMC_BERGMAN)
        return set_err(err, el, "unknown SRMC problem kind"), QRMC_ENOTIMPL;
    if (p->dim < 1 || p->dim > QRMC_SRMC_MAX_DIM) return set_err(err, el, "SRMC dim must be in [1, 6]"), QRMC_EINVAL;
    if (!(p->horizon > 0.0)) return set_err(err, el, "horizon must be > 0"), QRMC_EINVAL;
    if (c->steps < 1) return set_err(err, el, "steps must be >= 1"), QRMC_EINVAL;
    // stream ids are (step << 40) | path (rng.hpp:73-80): the reference's own bound
    if (c->steps >= (1 << 22)) return set_err(err, el, "RunConfig: steps exceeds the stream-id layout"), QRMC_EINVAL;
    if (c->cells_per_dim < 1) return set_err(err, el, "cells_per_dim must be >= 1"), QRMC_EINVAL;
    if (c->basis != QRMC_SRMC_LP0 && c->basis != QRMC_SRMC_LP1)
        return set_err(err, el, "basis must be LP0 or LP1"), QRMC_EINVAL;
    if (!(c->hi > c->lo)) return set_err(err, el, "domain needs hi > lo"), QRMC_EINVAL;
    if (!(c->truncation > 0.0)) return set_err(err, el, "truncation must be > 0"), QRMC_EINVAL;
    const int P = c->basis == QRMC_SRMC_LP1 ? p->dim + 1 : 1;
    if (c->paths_per_cell < P) return set_err(err, el, "paths_per_cell must be >= basis size"), QRMC_EINVAL;
    double cells = std::pow(static_cast<double>(c->cells_per_dim), p->dim);
    if (cells * static_cast<double>(c->paths_per_cell) >= 0x1p40)
        return set_err(err, el, "cells * paths_per_cell must be < 2^40 (stream id path field)"), QRMC_ECAPACITY;
    return QRMC_OK;
}

SrmcDev make_dev(const qrmc_srmc_problem_t* p, const qrmc_srmc_config_t* c) {
    SrmcDev s{};
    s.kind = p->kind;
    s.n = c->cells_per_dim;
    s.cells = 1;
    for (int l = 0; l < p->dim; ++l) s.cells *= c->cells_per_dim;
    s.M = c->paths_per_cell;
    s.k0 = 0;
    s.k1 = s.cells;
    s.seed = c->seed;
    {
        const char* e = std::getenv("QRMC_SRMC_PATH_CACHE");
        s.path_cache = !(e && e[0] == '0');
    }
    for (int r = 0; r < 10; ++r) {  // Philox4x32-10 key schedule (rng.cpp:9-40)
        s.rk[2 * r] = static_cast<uint32_t>(c->seed) + static_cast<uint32_t>(r) * 0x9E3779B9u;
        s.rk[2 * r + 1] = static_cast<uint32_t>(c->seed >> 32) + static_cast<uint32_t>(r) * 0xBB67AE85u;
    }
    s.lo = c->lo;
    s.hi = c->hi;
    s.h = (c->hi - c->lo) / c->cells_per_dim;
    s.inv_h = 1.0 / s.h;
    s.inv2h = 2.0 / s.h;
    s.T = p->horizon;
    s.dt = p->horizon / c->steps;
    s.inv_dt = 1.0 / s.dt;
    s.sqrt_dt = std::sqrt(s.dt);
    s.L = c->truncation;
    for (int j = 0; j < 8; ++j) s.p[j] = p->params[j];
    if (p->kind == QRMC_SRMC_BERGMAN) {
        s.p[5] = (p->params[0] - p->params[2]) / p->params[1];  // theta
        s.p[6] = 1.0 / p->params[1];
        volatile double drift = p->params[0] - 0.5 * (p->params[1] * p->params[1]);
        s.bdt = drift * s.dt;
        s.sig = p->params[1];
    } else {
        s.bdt = 0.0;
        s.sig = 1.0;
    }
    return s;
}

constexpr size_t kSrmcCacheBytes = 192 * 1024;  // + 8 warps' tail scratch stays under 227 KB

template <int D, int P>
void launch_step_t(const SrmcDev& s, const double* next, double* y, double* z, bool zpass, bool wantz, cudaStream_t st) {
    const int warps = 8;
    const int64_t cells = s.k1 - s.k0;
    // 4 lanes per hypercube, 8 hypercubes per warp -- only when the range still fills the
    // GPU with an eighth as many warps (64^2 cells at M=100: 1.33e10 -> 1.1e10 with a warp
    // per cell; config 4: 4 lanes 1.92e10, 8 lanes 1.83e10, 2 / 1 lanes +0.5 / +1%)
    // (also for M < 2048 without a Z pass: config 2, M = 1000, 2.25e10 -> 2.35e10 -- 250
    // iterations per lane, none half-empty; the Bergman Z pass keeps a warp per cell for its
    // path cache unless M < 256)
    if (s.cells >= 32768 && s.M < (zpass ? 256 : 2048)) {  // by the TOTAL cell count: a shard computes exactly what the whole solve does
#ifndef QRMC_SRMC_SUBG
#define QRMC_SRMC_SUBG 4
#endif
        constexpr int SG = QRMC_SRMC_SUBG, CPW = 32 / SG;  // lanes per hypercube, hypercubes per warp
        const unsigned grid = static_cast<unsigned>((cells + warps * CPW - 1) / (warps * CPW));
        if (grid == 0) return;
        if (zpass)
            k_srmc_step<D, P, true, false, SG><<<grid, warps * 32, 0, st>>>(s, next, y, z);
        else if (wantz)
            k_srmc_step<D, P, false, true, SG><<<grid, warps * 32, 0, st>>>(s, next, y, z);
        else
            k_srmc_step<D, P, false, false, SG><<<grid, warps * 32, 0, st>>>(s, next, y, z);
        return;
    }
    const unsigned grid = static_cast<unsigned>((cells + warps - 1) / warps);
    if (grid == 0) return;
    // the Bergman second pass from a shared-memory path cache when it fits (M <= ~640 at d=4)
    const size_t cache = static_cast<size_t>(warps) * ((s.M + 31) / 32) * (1 + D) * 32 * sizeof(double);
    if (zpass && s.kind == QRMC_SRMC_BERGMAN && s.path_cache && cache <= kSrmcCacheBytes &&
        cudaFuncSetAttribute(k_srmc_step<D, P, true, false, 32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kSrmcCacheBytes)) == cudaSuccess) {
        k_srmc_step<D, P, true, false, 32, true><<<grid, warps * 32, cache, st>>>(s, next, y, z);
        return;
    }
    if (zpass)
        k_srmc_step<D, P, true, false, 32><<<grid, warps * 32, 0, st>>>(s, next, y, z);
    else if (wantz)
        k_srmc_step<D, P, false, true, 32><<<grid, warps * 32, 0, st>>>(s, next, y, z);
    else
        k_srmc_step<D, P, false, false, 32><<<grid, warps * 32, 0, st>>>(s, next, y, z);
}

template <int D>
void launch_step_d(int P, const SrmcDev& s, const double* next, double* y, double* z, bool zpass, bool wantz,
                   cudaStream_t st) {
    if (P == 1)
        launch_step_t<D, 1>(s, next, y, z, zpass, wantz, st);
    else
        launch_step_t<D, D + 1>(s, next, y, z, zpass, wantz, st);
}

template <int D>
__global__ void k_unmorton(int n, int bits, int width, int64_t rows, const double* __restrict__ in,
                           double* __restrict__ out) {
    const int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (v >= rows) return;
    int c[D];
    morton_decode<D>(v, bits, c);
    int64_t k = 0;
#pragma unroll
    for (int l = 0; l < D; ++l) k = k * n + c[l];
    for (int j = 0; j < width; ++j) out[k * width + j] = in[v * width + j];
}

cudaError_t launch_unmorton(int d, int n, int bits, int width, const double* in, double* out, cudaStream_t st) {
    int64_t rows = 1;
    for (int l = 0; l < d; ++l) rows *= n;
    const unsigned grid = static_cast<unsigned>((rows + 255) / 256);
    switch (d) {
        case 1: k_unmorton<1><<<grid, 256, 0, st>>>(n, bits, width, rows, in, out); break;
        case 2: k_unmorton<2><<<grid, 256, 0, st>>>(n, bits, width, rows, in, out); break;
        case 3: k_unmorton<3><<<grid, 256, 0, st>>>(n, bits, width, rows, in, out); break;
        case 4: k_unmorton<4><<<grid, 256, 0, st>>>(n, bits, width, rows, in, out); break;
        case 5: k_unmorton<5><<<grid, 256, 0, st>>>(n, bits, width, rows, in, out); break;
        default: k_unmorton<6><<<grid, 256, 0, st>>>(n, bits, width, rows, in, out); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_step(int d, int P, const SrmcDev& s, const double* next, double* y, double* z, bool zpass,
                        bool wantz, cudaStream_t st) {
    switch (d) {
        case 1: launch_step_d<1>(P, s, next, y, z, zpass, wantz, st); break;
        case 2: launch_step_d<2>(P, s, next, y, z, zpass, wantz, st); break;
        case 3: launch_step_d<3>(P, s, next, y, z, zpass, wantz, st); break;
        case 4: launch_step_d<4>(P, s, next, y, z, zpass, wantz, st); break;
        case 5: launch_step_d<5>(P, s, next, y, z, zpass, wantz, st); break;
        default: launch_step_d<6>(P, s, next, y, z, zpass, wantz, st); break;
    }
    return cudaGetLastError();
}

template <int D>
void launch_eval_d(int P, const SrmcDev& s, const double* tab, const double* x, int64_t n, double* out) {
    const unsigned grid = static_cast<unsigned>((n + 255) / 256);
    if (P == 1)
        k_srmc_eval<D, 1><<<grid, 256>>>(s, tab, x, n, out);
    else
        k_srmc_eval<D, D + 1><<<grid, 256>>>(s, tab, x, n, out);
}

#define CK(call)                                                                  \
    do {                                                                          \
        cudaError_t e_ = (call);                                                  \
        if (e_ != cudaSuccess) {                                                  \
            std::snprintf(msg, sizeof msg, "CUDA: %s (%s)", cudaGetErrorString(e_), #call); \
            rc = QRMC_ECUDA;                                                      \
            goto done;                                                            \
        }                                                                         \
    } while (0)

}  // namespace qrmc_srmc_dev

using namespace qrmc_srmc_dev;

extern "C" int32_t qrmc_srmc_basis_size(const qrmc_srmc_problem_t* prob, const qrmc_srmc_config_t* cfg) {
    if (validate(prob, cfg, nullptr, 0) != QRMC_OK) return -1;
    return cfg->basis == QRMC_SRMC_LP1 ? prob->dim + 1 : 1;
}

extern "C" int64_t qrmc_srmc_cells(const qrmc_srmc_problem_t* prob, const qrmc_srmc_config_t* cfg) {
    if (validate(prob, cfg, nullptr, 0) != QRMC_OK) return -1;
    int64_t c = 1;
    for (int l = 0; l < prob->dim; ++l) c *= cfg->cells_per_dim;
    return c;
}

extern "C" int32_t qrmc_srmc_evaluate(const qrmc_srmc_problem_t* prob, const qrmc_srmc_config_t* cfg,
                                      const double* y_step, const double* x, int64_t npts, double* out, char* err,
                                      size_t err_len) {
    char msg[256] = {0};
    int rc = validate(prob, cfg, err, err_len);
    if (rc != QRMC_OK) return rc;
    if (npts <= 0) return QRMC_OK;
    const int d = prob->dim;
    const int P = cfg->basis == QRMC_SRMC_LP1 ? d + 1 : 1;
    const SrmcDev s = make_dev(prob, cfg);
    const size_t tab = static_cast<size_t>(s.cells) * P;
    double *dt = nullptr, *dx = nullptr, *dout = nullptr;
    CK(cudaMalloc(&dt, tab * sizeof(double)));
    CK(cudaMalloc(&dx, npts * d * sizeof(double)));
    CK(cudaMalloc(&dout, npts * sizeof(double)));
    CK(cudaMemcpy(dt, y_step, tab * sizeof(double), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dx, x, npts * d * sizeof(double), cudaMemcpyHostToDevice));
    switch (d) {
        case 1: launch_eval_d<1>(P, s, dt, dx, npts, dout); break;
        case 2: launch_eval_d<2>(P, s, dt, dx, npts, dout); break;
        case 3: launch_eval_d<3>(P, s, dt, dx, npts, dout); break;
        case 4: launch_eval_d<4>(P, s, dt, dx, npts, dout); break;
        case 5: launch_eval_d<5>(P, s, dt, dx, npts, dout); break;
        default: launch_eval_d<6>(P, s, dt, dx, npts, dout); break;
    }
    CK(cudaGetLastError());
    CK(cudaMemcpy(out, dout, npts * sizeof(double), cudaMemcpyDeviceToHost));
done:
    if (dt) cudaFree(dt);
    if (dx) cudaFree(dx);
    if (dout) cudaFree(dout);
    if (rc != QRMC_OK) set_err(err, err_len, msg);
    return rc;
}

// qrmc_srmc_step_device has no plan to report through: its non-finite flag goes to a
// per-device scratch word (the plan of srmc_host.cpp checks its own).
static int* bad_scratch() {
    static int* p[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!p[dev & 63]) cudaMalloc(&p[dev & 63], sizeof(int));
    return p[dev & 63];
}

// One backward step on caller-owned device tables for the cell range [k_begin, k_end):
// the sharded (multi-GPU) driver runs it on its own cells, then all-gathers the step's
// table (paper_2407_21084_b200/srmc.py, solve_sharded). Results per cell do not depend
// on the range, so a sharded solve is bitwise identical to the single-GPU one.
extern "C" int32_t qrmc_srmc_step_device(const qrmc_srmc_problem_t* prob, const qrmc_srmc_config_t* cfg, int32_t step,
                                         const double* next_dev, double* y_dev, double* z_dev, int64_t k_begin,
                                         int64_t k_end, void* stream, char* err, size_t err_len) {
    char msg[256] = {0};
    int rc = validate(prob, cfg, err, err_len);
    if (rc != QRMC_OK) return rc;
    SrmcDev s = make_dev(prob, cfg);
    if (step < 0 || step >= cfg->steps) return set_err(err, err_len, "step out of range"), QRMC_EINVAL;
    if (k_begin < 0 || k_end < k_begin || k_end > s.cells) return set_err(err, err_len, "bad cell range"), QRMC_EINVAL;
    const bool zpass = needs_z(prob);
    if (!y_dev || (step < cfg->steps - 1 && !next_dev) || (zpass && !z_dev))
        return set_err(err, err_len, "null device table"), QRMC_EINVAL;
    const int d = prob->dim;
    const int P = cfg->basis == QRMC_SRMC_LP1 ? d + 1 : 1;
    s.k0 = k_begin;
    s.k1 = k_end;
    s.step = step;
    s.last = (step == cfg->steps - 1);
    s.t = (step + 1) * s.dt;
    s.decay = std::exp(((s.p[1] * s.p[1]) * static_cast<double>(d)) * (s.t - s.T) / 2.0);
    s.bad = bad_scratch();
    CK(launch_step(d, P, s, s.last ? nullptr : next_dev, y_dev, z_dev, zpass, !zpass && z_dev != nullptr,
                   static_cast<cudaStream_t>(stream)));
done:
    if (rc != QRMC_OK) set_err(err, err_len, msg);
    return rc;
}

// mma_common.cuh -- device helpers shared by the tensor-core kernels
// (responses_mma.cu, project_mma.cu).
#pragma once

#include <cstdint>

#include "kernels.cuh"
#include "qrmc_device.cuh"

namespace qrmc_dev {

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

// D = A B (accumulator start: C = 0)
__device__ __forceinline__ void dmma0(double (&c)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
        : "=d"(c[0]), "=d"(c[1])
        : "d"(a), "d"(b), "d"(0.0), "d"(0.0));
}

// u64 draw number idx of a stream (RngStream order: two draws per Philox block,
// low half first; rng.hpp:60-75), without walking the stream.
__device__ __forceinline__ uint64_t stream_u64_at(uint64_t seed, uint64_t sid, uint64_t idx) {
    const uint64_t block = idx >> 1;
    const uint4 o = philox4x32_10(
        make_uint4(static_cast<uint32_t>(block), static_cast<uint32_t>(block >> 32), static_cast<uint32_t>(sid),
                   static_cast<uint32_t>(sid >> 32)),
        make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32)));
    return (idx & 1) ? ((static_cast<uint64_t>(o.w) << 32) | o.z) : ((static_cast<uint64_t>(o.y) << 32) | o.x);
}
// ((v >> 12) + 1/2) 2^-52 (rng.hpp:41-43) without an integer->double conversion: m = v >> 12
// in the mantissa of 1.0 gives 1 + m 2^-52; minus 1 and plus 2^-53 are exact ((2m + 1) 2^-53
// has 53 significant bits), so this is the same double
__device__ __forceinline__ double u64_to_uniform(uint64_t v) {
    return DADD(DSUB(__longlong_as_double(static_cast<long long>(0x3FF0000000000000ull | (v >> 12))), 1.0), 0x1p-53);
}

__device__ __forceinline__ int64_t owned_path(const StepArgs& a, int64_t q) {
    const int64_t cq = q / kChunk;
    const int64_t r = cq / a.owned_lanes;
    const int64_t lane = a.lane_lo + cq % a.owned_lanes;
    return (r * kLanes + lane) * kChunk + q % kChunk;
}

// (T_{k-1}(c), T_k(c)) by binary doubling from (T_0, T_1) = (1, c), T_{-1} = c:
// T_{2n} = 2 T_n^2 - 1, T_{2n+1} = 2 T_n T_{n+1} - c.
__device__ __forceinline__ void cheb_pair(double c, int k, double& tkm1, double& tk) {
    if (k == 0) {
        tkm1 = c;
        tk = 1.0;
        return;
    }
    double a = 1.0, b = c;  // (T_n, T_{n+1}) for n = 0
    const int top = 31 - __clz(k);
    for (int bit = top; bit >= 0; --bit) {
        const double t2n = fma(DMUL(2.0, a), a, -1.0);
        const double t2n1 = fma(DMUL(2.0, a), b, -c);
        const double t2n2 = fma(DMUL(2.0, b), b, -1.0);
        if ((k >> bit) & 1) {
            a = t2n1;
            b = t2n2;
        } else {
            a = t2n;
            b = t2n1;
        }
    }
    // now (a, b) = (T_k, T_{k+1}); T_{k-1} = 2c T_k - T_{k+1}
    tk = a;
    tkm1 = fma(DMUL(2.0, c), a, -b);
}

// Cosine table piece q of kTabSplit for coordinate l of path p: c_k(x_l) =
// cos(k theta) for k in the piece, at tb[k * stride] (tables laid out
// [entry][path]); a Chebyshev recurrence restarted by cheb_pair.
__device__ __forceinline__ void cos_table_piece(double th, int kmax, int q, int n_split, double* tb, int stride) {
    const int len = (kmax + n_split) / n_split;  // ceil((kmax + 1) / n_split)
    const int k0 = q * len, k1 = min(kmax + 1, k0 + len);
    if (k0 >= k1) return;
    const double c1 = cos(th), two = DMUL(2.0, c1);
    double prev, cv;  // (c_{k0-1}, c_{k0}); c_{-1} = c_1
    cheb_pair(c1, k0, prev, cv);  // k0 = 0: (c_1, 1)
    tb[k0 * stride] = cv;
    for (int k = k0 + 1; k < k1; ++k) {
        const double nx = fma(two, cv, -prev);
        prev = cv;
        cv = nx;
        tb[k * stride] = nx;
    }
}

// Same, from c1 = cos(theta) (the restart needs no further cosines).
__device__ __forceinline__ void cos_table_piece_c(double c1, int kmax, int q, int n_split, double* tb, int stride) {
    const int len = (kmax + n_split) / n_split;
    const int k0 = q * len, k1 = min(kmax + 1, k0 + len);
    if (k0 >= k1) return;
    const double two = DMUL(2.0, c1);
    double prev, cv;
    cheb_pair(c1, k0, prev, cv);
    tb[k0 * stride] = cv;
    for (int k = k0 + 1; k < k1; ++k) {
        const double nx = fma(two, cv, -prev);
        prev = cv;
        cv = nx;
        tb[k * stride] = nx;
    }
}

}  // namespace qrmc_dev

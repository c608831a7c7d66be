// srmc_types.h -- launch interface between the SRMC kernels (srmc.cu) and the
// SRMC host plan (srmc_host.cpp). See include/qrmc_srmc.h for the scheme.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "qrmc_srmc.h"

namespace qrmc_srmc_dev {

struct SrmcDev {
    int kind, n, step, last;
    int64_t cells, M;
    int64_t k0, k1;  // this launch's cell range [k0, k1) (a rank's shard; [0, cells) single-GPU)
    uint64_t seed;
    double lo, hi, h, inv_h, inv2h, dt, inv_dt, sqrt_dt, t, T, L;
    double p[8];
    double bdt, sig;  // Euler: x + bdt + sig * sqrt_dt * z
    uint32_t rk[20];  // Philox round keys (seed + r * Weyl), read from the constant bank
    double decay;     // SinBenchmark exp(lambda^2 d (t - T) / 2) at this step's t (hoisted per launch)
    int* bad;         // set to 1 when a written coefficient is not finite (NumericError)
    // Table rows in Morton order (plans, n a power of two): the row of cell (c_0..c_{d-1})
    // interleaves their bits, coordinate d-1 lowest, so a 6-D neighbourhood sits in a few
    // nearby rows of the table and the concurrently processed cells' gathers stay in L2.
    // Cells are visited in row order; draws stay keyed by the lexicographic cell index.
    int path_cache;   // Bergman second pass from the shared-memory path cache (QRMC_SRMC_PATH_CACHE=0: off)
    int morton, mbits;
    uint32_t mmul, mmask;  // spread(c) = (c * mmul) & mmask puts bit b of c at b*D (exact: mbits <= D-1)
};

// Morton row of cell coordinates / coordinates of a Morton row (bits of coordinate l at
// positions b*D + (D-1-l))
// (the multiply-and-mask spread: the mbits shifted copies of c never overlap because
// mbits <= D-1, so the product carries nothing; D * mbits <= 30 keeps it in 32 bits)
template <int D>
__host__ __device__ __forceinline__ int64_t morton_encode(const int* c, uint32_t mmul, uint32_t mmask) {
    uint32_t v = 0;
#pragma unroll
    for (int l = 0; l < D; ++l) v |= ((static_cast<uint32_t>(c[l]) * mmul) & mmask) << (D - 1 - l);
    return v;
}
template <int D>
__host__ __device__ __forceinline__ void morton_decode(int64_t v, int bits, int* c) {
#pragma unroll
    for (int l = 0; l < D; ++l) c[l] = 0;
    for (int b = 0; b < bits; ++b)
#pragma unroll
        for (int l = 0; l < D; ++l) c[l] |= static_cast<int>((v >> (b * D + (D - 1 - l))) & 1) << b;
}

int validate(const qrmc_srmc_problem_t* p, const qrmc_srmc_config_t* c, char* err, size_t el);
SrmcDev make_dev(const qrmc_srmc_problem_t* p, const qrmc_srmc_config_t* c);
bool needs_z(const qrmc_srmc_problem_t* p);
void set_err(char* err, size_t len, const char* msg);
// One backward step of the cells [s.k0, s.k1) on st: y/z rows of the step, next = step+1's y table.
cudaError_t launch_step(int d, int P, const SrmcDev& s, const double* next, double* y, double* z, bool zpass,
                        bool wantz, cudaStream_t st);
// Morton-ordered rows -> lexicographic rows (width doubles per row), n^d cells
cudaError_t launch_unmorton(int d, int n, int bits, int width, const double* in, double* out, cudaStream_t st);

}  // namespace qrmc_srmc_dev

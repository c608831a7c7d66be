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
};

int validate(const qrmc_srmc_problem_t* p, const qrmc_srmc_config_t* c, char* err, size_t el);
SrmcDev make_dev(const qrmc_srmc_problem_t* p, const qrmc_srmc_config_t* c);
bool needs_z(const qrmc_srmc_problem_t* p);
void set_err(char* err, size_t len, const char* msg);
// One backward step of the cells [s.k0, s.k1) on st: y/z rows of the step, next = step+1's y table.
cudaError_t launch_step(int d, int P, const SrmcDev& s, const double* next, double* y, double* z, bool zpass,
                        bool wantz, cudaStream_t st);

}  // namespace qrmc_srmc_dev

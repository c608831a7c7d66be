// qrmc_types.h -- plain structs shared by host.cpp and the kernels (no device code).
#pragma once

#include <cstdint>

namespace qrmc_dev {

constexpr int kLanes = 256;  // LaneLayout::kLanes (proj/include/qrmc/parallel.hpp:22)
constexpr int kChunk = 1024; // LaneLayout::kChunk (parallel.hpp:21)
constexpr unsigned kStepShift = 40;  // stream_ids::kStepShift (rng.hpp:77)
constexpr int kMaxDim = 8;

// Series-kernel shape per dimension D (series_block.cuh): paths per thread P,
// register-table sizes S2 (level D-2) and LT (leaf level D-1).
// QRMC_K1_{P,S2,LT}_D4 override the d = 4 shape (tuning builds only).
#ifndef QRMC_K1_P_D4
#define QRMC_K1_P_D4 4
#endif
#ifndef QRMC_K1_S2_D4
#define QRMC_K1_S2_D4 8
#endif
#ifndef QRMC_K1_LT_D4
#define QRMC_K1_LT_D4 8
#endif
// Shared-memory tile of the series program (series_block.cuh / host.cpp):
// coefficients and 32-bit program words per tile, double-buffered.
#ifndef QRMC_TILE_A
#define QRMC_TILE_A 1024
#endif
#ifndef QRMC_TILE_W
#define QRMC_TILE_W 768
#endif
constexpr int kSeriesTileA = QRMC_TILE_A;
constexpr int kSeriesTileW = QRMC_TILE_W;

// Largest budget B of the hyperbolic-profile groups run by static code (series_block.cuh).
#ifndef QRMC_HYP_MAX_B
#define QRMC_HYP_MAX_B 7
#endif
constexpr int kHypMaxB = QRMC_HYP_MAX_B;

constexpr int k1_p(int d) { return d == 4 ? QRMC_K1_P_D4 : d == 3 ? 4 : d <= 2 || d >= 7 ? 1 : 2; }
constexpr int k1_s2(int d) { return d == 4 ? QRMC_K1_S2_D4 : d <= 1 ? 2 : d == 2 ? 32 : 8; }
constexpr int k1_lt(int d) { return d == 4 ? QRMC_K1_LT_D4 : d <= 2 ? 32 : 8; }

// Product Student-t measure for mu in {1, 2} (proj/src/student.cpp:53-106).
struct MeasureDev {
    int form;  // 1 Cauchy, 2 algebraic mu=2, 3 general mu (include/qrmc_student_t.h)
    double mu, sqrt_mu;
    double center[kMaxDim];
};

// Device functors replacing ProblemSpec's std::function members
// (sde.hpp:23-29; SinBenchmark functors benchmark.cpp:46-62).
struct ProblemDev {
    int dim, bdim;
    double horizon;
    int terminal_kind, driver_kind, drift_kind, diffusion_kind;
    double tp0, tp1, dp0, dp1, drift_c, sigma;
    double drift_a[kMaxDim], drift_b[kMaxDim], sig[kMaxDim];  // AFFINE drift a + b x_l, DIAG sigma_l
    double lstar_base;  // C_eta (C_g + T C_f) exp(C_eta L_f T), host-computed exactly as sde.cpp:28-29
    double eta;         // max(eta_g, eta_f)
    double state_bound;
};

}  // namespace qrmc_dev

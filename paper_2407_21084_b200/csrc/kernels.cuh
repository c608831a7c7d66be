// kernels.cuh -- launch-side interface between host.cpp and kernels.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "qrmc_types.h"

namespace qrmc_dev {

constexpr int kProjRun = 8;  // leaf indices per K2 work item

// Series program in device memory (series_block.cuh).
struct SeriesTiles {
    const int4* tiles;     // {prog_off (16-byte aligned), n_words, alpha_off (even), alpha_len (even)}
    int n_tiles;
    const uint32_t* prog;  // group words, per-tile segments
};

// Everything one backward step's kernels read (passed by value: it lives in
// the kernel parameter space, so it is captured verbatim into CUDA graphs).
struct StepArgs {
    ProblemDev prob;
    MeasureDev meas;
    int steps;    // N
    int step;     // i (the cloud being processed)
    double dt, sqrt_dt, q;
    uint64_t seed;
    int64_t paths;        // M (global)
    int lane_lo;          // this rank's lanes [lane_lo, lane_lo + owned_lanes)
    int owned_lanes;
    int64_t n_owned;      // paths owned by this rank
    double* alpha_packed; // [N][kp] packed alpha' rows (series_block layout)
    int64_t kp;
    SeriesTiles tiles;    // the series program
    double* resp;         // [n_owned]
    double* cloud;        // [dim][n_owned] (store mode) or nullptr (recompute)
    unsigned long long* counters;  // {applications, clipped}
    int* err_flags;       // {kind, min SimulationError step}
    const int* abort_flag;
};

struct ProjArgs {
    // work items (host.cpp build_project_items): <= kProjRun consecutive leaf
    // indices of one run, sorted by length
    const int32_t* item_k;     // first term index
    const int32_t* item_len;   // number of terms
    const int32_t* item_leaf;  // table offset of the first leaf value
    const int32_t* item_pre;   // [dim-1][n_items] table offsets of the run prefix
    int n_items;
    int offset[kMaxDim];  // per-coordinate table offsets (cosine_basis.cpp:58-64)
    int kmax[kMaxDim];
    int table_len;
    int batch;            // points staged per smem batch
    int64_t basis_size;
    double* partials;     // [owned_lanes][K]
};

struct FinishArgs {
    const double* all_partials;  // [256][K] after the exchange
    int64_t basis_size;
    double inv_m;
    double* coef_row;            // [K] canonical alpha_i
    const int32_t* pack_pos;     // k -> packed position
    const double* pack_scale;    // sqrt2^{nnz(k)}
};

cudaError_t configure_series_kernels();  // once per process, before the first series launch
cudaError_t launch_responses(const StepArgs& a, cudaStream_t st);
size_t project_smem_bytes(const ProjArgs& p);
cudaError_t configure_project(int dim, size_t smem);
cudaError_t launch_project(const StepArgs& a, const ProjArgs& p, cudaStream_t st);
cudaError_t launch_finish(const StepArgs& a, const FinishArgs& f, cudaStream_t st);

cudaError_t launch_philox(const uint32_t* ctr, const uint32_t* key, int64_t n, uint32_t* out,
                          cudaStream_t st);
cudaError_t launch_stream_draws(uint64_t seed, const uint64_t* sids, int64_t n, int n_draws, int kind,
                                void* out, cudaStream_t st);
cudaError_t launch_cloud_paths(const StepArgs& a, int64_t first, int64_t n, double* out, int* bad,
                               cudaStream_t st);
cudaError_t launch_eval_points(const StepArgs& a, const double* alpha_row, const double* x, int64_t n,
                               double q, int with_weight, double* out, cudaStream_t st);
cudaError_t launch_mse(const StepArgs& a, double kappa, double lam, double horizon, uint64_t eval_seed,
                       int eval_points, double* sq, double* sq_u, cudaStream_t st);

}  // namespace qrmc_dev

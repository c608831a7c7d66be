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
    int cloud_cos;        // the cloud holds cos(pi F_l(x_l)) (tensor-core K1/K2 pair) instead of x
    unsigned long long* counters;  // {applications, clipped}
    int* err_flags;       // {kind, min SimulationError step}
    const int* abort_flag;
};

// K1 on the FP64 tensor cores (responses_mma.cu, host.cpp build_mma_layout).
// The CTA owns 8*kMmaRowBlocks paths; every warp runs mma.m8n8k4.f64 for all of
// them on its own units (column blocks x chunk range), streaming its own
// coefficient fragments through a private shared-memory ring.
#ifndef QRMC_MMA_WARPS
#define QRMC_MMA_WARPS 20
#endif
constexpr int kMmaWarps = QRMC_MMA_WARPS;
#ifndef QRMC_MMA_RB
#define QRMC_MMA_RB 4
#endif
constexpr int kMmaRowBlocks = QRMC_MMA_RB;       // 8-path row blocks per CTA
constexpr int kMmaPaths = 8 * kMmaRowBlocks;     // paths per CTA
#ifndef QRMC_MMA_BUNDLE
#define QRMC_MMA_BUNDLE 2
#endif
#ifndef QRMC_MMA_BATCH
#define QRMC_MMA_BATCH 8
#endif
#ifndef QRMC_MMA_RING
#define QRMC_MMA_RING 2
#endif
constexpr int kMmaBundle = QRMC_MMA_BUNDLE;      // max column blocks per unit (1..4)
constexpr int kMmaBatch = QRMC_MMA_BATCH;        // fragments per copy batch (256 B each)
constexpr int kMmaRingBatches = QRMC_MMA_RING;   // per-warp ring depth
constexpr int kMmaRingFrags = kMmaBatch * kMmaRingBatches;
constexpr int kMmaTabStride = kMmaPaths + 4;    // cosine tables [table entry][path], padded
#ifndef QRMC_MMA_KSPLIT
#define QRMC_MMA_KSPLIT 32
#endif
constexpr int kMmaKSplit = QRMC_MMA_KSPLIT;      // max chunks per unit

struct MmaArgs {
    const double* alpha;      // [N][row_len] fragment streams per series
    int64_t row_len;          // doubles per series
    const int4* units;        // {cb0, nb, c0, c1}, warp-contiguous
    const int4* warp_info;    // [kMmaWarps] {unit_begin, unit_end, frag_offset, frags (padded to kMmaBatch)}
    const uint32_t* terms;    // [n_terms] table rows (x kMmaTabStride) of c_s(x_{D-2}) | c_b(x_{D-1}) << 16
    const uint16_t* gk;       // [n_groups][D-2] table rows (x kMmaTabStride) of the group prefix
    int table_len;            // doubles per path table (all coordinates)
    int offset[kMaxDim];      // per-coordinate table offsets
    int kmax[kMaxDim];
};

// K1, warp-specialised (responses_ws.cu): kWsConsumers warps run the staircase
// GEMM of evaluation j from one of two cosine-table buffers while kWsProducers
// warps run the Euler steps, the x-only parts, the truncation/driver of
// evaluation j-2 and the tables of evaluation j+1 into the other buffer; the
// hand-off uses named barriers. B fragments stream from L2 (prefetched to L1).
#ifndef QRMC_WS_BUNDLE
#define QRMC_WS_BUNDLE 2  // column blocks per warp-specialised unit (ws_unit<D, NB>, NB <= 3)
#endif
#ifndef QRMC_WS_CONSUMERS
#define QRMC_WS_CONSUMERS 16
#endif
constexpr int kWsConsumers = QRMC_WS_CONSUMERS;  // a power of two (the finish's pairwise sum)
constexpr int kWsProducers = 4;
constexpr int kWsPaths = 32;    // paths per CTA (4 row blocks of 8)
#ifndef QRMC_WS_PREFETCH
#define QRMC_WS_PREFETCH 1
#endif
// fragments the L1 prefetch runs ahead (M = 2e6: 0 / 1 / 2 / 4 ahead = 0.727 / 0.708 /
// 0.711 / 0.712 s K1; with ~2 KB of L1 beside the tables, lines fetched further ahead are
// evicted before use)
constexpr int kWsPrefetch = QRMC_WS_PREFETCH;

struct WsArgs {
    const double* alpha;      // fragment streams, warp-major: warp w's series 0..N-1 back to back
    const int4* units;        // {cb0, nb, c0, c1}, warp-contiguous
    const int4* warp_info;    // [kWsConsumers] {unit_begin, unit_end, first fragment of series 0, frags per series}
    const uint4* terms;       // [n_terms][2 row halves] swizzled byte offsets {sA, sB, bA, bB}
    const uint32_t* gk;       // [2 row halves][n_groups / 2 pairs][R = 2 (D-2) up to 4k] swizzled offsets {A | B << 16}
    int n_groups;             // groups, padded to whole column blocks
    int table_len;            // table entries (all coordinates)
    int offset[kMaxDim];
    int kmax[kMaxDim];
};

// K2 on the FP64 tensor cores (project_mma.cu): per owned lane, the staircase
// G[u][t] = sum_m S_m U_u(X_m) A_t(X_m) as mma.m8n8k4.f64 (8 groups x 8 terms x
// 4 paths); each warp keeps one rectangle of <= kProjTiles output tiles in
// registers over all of the lane's paths.
#ifndef QRMC_PROJ_WARPS
#define QRMC_PROJ_WARPS 20
#endif
constexpr int kProjWarps = QRMC_PROJ_WARPS;
#ifndef QRMC_PROJ_TILES
#define QRMC_PROJ_TILES 8
#endif
constexpr int kProjTiles = QRMC_PROJ_TILES;  // output tiles per warp: ng group blocks x nt term blocks, ng a power of 2
// paths per shared-memory table batch (double-buffered): 24 when two tables of
// 24 + 4 padded columns fit, else 16 (table row strides 28 / 20 doubles; 20 and 28
// path batches, strides 24 / 32, cost 25-75% more in bank conflicts)
constexpr int kProjBatchWide = 24, kProjBatchNarrow = 16;

struct ProjMmaArgs {
    const int4* rects;        // [parts][kProjWarps] {gb0, tb0, ng | nt << 8, tiles} (full rectangles)
    const int32_t* out;       // [parts][kProjWarps][kProjTiles][64] (tile ig * nt + it) -> k or -1
    const uint32_t* terms;    // MmaArgs::terms (8-term padded)
    const uint16_t* gk;       // MmaArgs::gk
    const double* scale;      // sqrt2^{nnz(k)}
    int parts;
    int table_len;
    int offset[kMaxDim];
    int kmax[kMaxDim];
    int64_t basis_size;
    int batch;                // kProjBatchWide or kProjBatchNarrow (project_mma_batch)
    // split = 2: each lane's chunks in two halves on two CTAs (grid z), combined as
    // half 0 + half 1 by the CTA that finishes second (fills the last wave of CTAs)
    int split;
    double* scratch;          // [2][owned_lanes][parts][kProjWarps][kProjTiles][64] (split = 2)
    int* counters;            // [owned_lanes][parts], zero between launches (split = 2)
    double* partials;         // [owned_lanes][K]
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
    double* alpha_mma;           // [N][mma_row_len] fragment stream, or nullptr
    int64_t mma_row_len;
    const int32_t* mma_pos;      // k -> fragment-stream position of series 0
    const int32_t* mma_stride;   // k -> distance between series (nullptr: mma_row_len)
};

cudaError_t configure_series_kernels();  // once per process, before the first series launch
cudaError_t launch_responses(const StepArgs& a, cudaStream_t st);
size_t responses_mma_smem_bytes(int dim, int table_len);
cudaError_t configure_responses_mma(int dim, size_t smem);
cudaError_t launch_responses_mma(const StepArgs& a, const MmaArgs& m, cudaStream_t st);
size_t responses_ws_smem_bytes(int dim, int table_len);
cudaError_t configure_responses_ws(int dim, size_t smem);
cudaError_t launch_responses_ws(const StepArgs& a, const WsArgs& m, cudaStream_t st);
size_t project_smem_bytes(const ProjArgs& p);
cudaError_t configure_project(int dim, size_t smem);
cudaError_t launch_project(const StepArgs& a, const ProjArgs& p, cudaStream_t st);
size_t project_mma_smem_bytes(int table_len, int batch);
// the widest batch whose tables fit `optin` bytes, 0 if none
int project_mma_batch(int table_len, size_t optin);
cudaError_t configure_project_mma(int dim, int batch, size_t smem);
cudaError_t launch_project_mma(const StepArgs& a, const ProjMmaArgs& p, cudaStream_t st);
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

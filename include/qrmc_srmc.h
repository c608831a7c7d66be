/* qrmc_srmc.h -- C ABI of the stratified regression Monte Carlo (SRMC) solver.
 *
 * the north_star's SRMC features (hypercube stratification of a
 * bounded domain, uniform-in-cell starts, LP0/LP1 local polynomial basis with per-cell
 * normal equations solved in FP64 registers, Z regression, a driver f(t, x, y, z),
 * truncation). The reference has NO code for any of this (last row;
 * the method is summarised at PAPER.md:361-366), so PARITY IS UNPINNED against the
 * reference: the GPU path is checked (i) against the C restatement oracle/srmc_oracle.c
 * on replayed Philox draws and (ii) statistically against closed forms
 * (SinBenchmark exact_solution, benchmark.cpp:20-28; Black-Scholes for the linear
 * Bergman case). The plugin seams mirror the reference solver's: the problem
 * functors (ProblemSpec, sde.hpp:18-49), the RunConfig knobs (solver.hpp:24-35), the
 * Philox stream (rng.hpp:26-65) and the truncation (solver.cpp:37-48).
 *
 * Scheme (explicit one-step SRMC, backward i = N-1 .. 0, t_i = i*dt):
 *   for every cell k and path m < M of step i (stream id (i << 40) | (k*M + m)):
 *     X_i      = lo + (c(k) + U) * h               U: d uniforms (rng.hpp:41-43)
 *     dW       = sqrt(dt) * Z                      Z = PPND16(U): d normals (AS241, qrmc_normal_quantile.h)
 *     X_{i+1}  = X_i + b(X_i) dt + sigma dW        (sde.cpp:37-73, diagonal sigma)
 *     Y1       = i+1 == N ? g(X_{i+1}) : clamp(yhat_{i+1}(X_{i+1}), +-L)
 *     Zhat_i   = LS fit in cell k of Y1 * dW / dt   (only when the driver uses z or want_z)
 *     Yhat_i   = LS fit in cell k of Y1 + dt * f(t_{i+1}, X_{i+1}, Y1, Zhat_i(X_i))
 *   yhat(x) evaluates the fit of the cell containing P(x), P = projection onto the domain
 *   box; LP0 basis {1}, LP1 basis {1, 2(x_l - centre_l)/h}.
 * Tables: y[i][k][P], z[i][k][l][P] (row-major), P = 1 (LP0) or d+1 (LP1). Cells are
 * numbered lexicographically, coordinate d-1 fastest (the reference's Gamma order,
 * multi_index.cpp:84-173). The cell index is integer work and bit-exact.
 */
#ifndef QRMC_SRMC_H
#define QRMC_SRMC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { QRMC_SRMC_SIN_BENCH = 0, QRMC_SRMC_BERGMAN = 1 };
enum { QRMC_SRMC_LP0 = 0, QRMC_SRMC_LP1 = 1 };
#define QRMC_SRMC_MAX_DIM 6

typedef struct {
    int32_t kind;    /* QRMC_SRMC_SIN_BENCH | QRMC_SRMC_BERGMAN */
    int32_t dim;
    double horizon;  /* T */
    /* SIN_BENCH: p[0] = kappa, p[1] = lambda (benchmark.cpp:30-67; b = 0, sigma = I).
     * BERGMAN (log-prices, d independent assets): p[0] = mu, p[1] = sigma, p[2] = r_lend,
     *   p[3] = r_borrow, p[4] = strike K; g = max(exp(mean x) - K, 0),
     *   f = -r_l y - theta sum z + (r_b - r_l) max(sum z / sigma - y, 0), theta = (mu - r_l)/sigma. */
    double params[8];
} qrmc_srmc_problem_t;

typedef struct {
    int32_t steps;           /* N >= 1 */
    int32_t cells_per_dim;   /* n >= 1; n^d cells */
    int64_t paths_per_cell;  /* M >= P */
    int32_t basis;           /* QRMC_SRMC_LP0 | QRMC_SRMC_LP1 */
    int32_t want_z;          /* also regress Z when the driver does not need it */
    uint64_t seed;
    double lo, hi;           /* domain [lo, hi]^d */
    double truncation;       /* L > 0: clamp of yhat (solver.cpp:37-41) */
} qrmc_srmc_config_t;

typedef struct {
    uint64_t path_steps;   /* simulated path-steps: sum over steps of cells * M */
    double device_seconds; /* CUDA-event time of the solve's kernels */
    int32_t kernel_launches;
    int32_t path_passes;   /* 2 when a z-dependent driver replays every path (Z pass + Y pass), else 1 */
} qrmc_srmc_stats_t;

/* number of coefficients per cell of the Y table (1 or d+1); <0 on a bad config */
int32_t qrmc_srmc_basis_size(const qrmc_srmc_problem_t* prob, const qrmc_srmc_config_t* cfg);
/* n^d; <0 on a bad config */
int64_t qrmc_srmc_cells(const qrmc_srmc_problem_t* prob, const qrmc_srmc_config_t* cfg);
/* Full backward solve on the current CUDA device (a world-1 plan: create, run,
 * download, destroy). y: steps * cells * P doubles (host), z: steps * cells * d * P
 * doubles or NULL. Returns 0 or a qrmc_status code with a message in err. */
int32_t qrmc_srmc_solve(const qrmc_srmc_problem_t* prob, const qrmc_srmc_config_t* cfg, double* y,
                        size_t y_len, double* z, size_t z_len, qrmc_srmc_stats_t* stats, char* err,
                        size_t err_len);
/* u(t_i, x) from a y table: i-th step, npts points x[npts][d] -> out[npts] (host) */
int32_t qrmc_srmc_evaluate(const qrmc_srmc_problem_t* prob, const qrmc_srmc_config_t* cfg,
                           const double* y_step, const double* x, int64_t npts, double* out,
                           char* err, size_t err_len);

/* ---- plans: the backward solve with device-resident tables, sharded over ranks ----
 * Hypercubes are partitioned over the ranks (north_star item 5): rank r of `world` owns
 * the cells [r*c, min((r+1)*c, cells)), c = ceil(cells / world) (qrmc_srmc_cell_range),
 * computes only those each backward step, and the step's y table is all-gathered over
 * NCCL (in place, NVLink) before the next step, because endpoints land in arbitrary
 * cells. Z (read only inside its own cell) is gathered once at the end when kept. Every
 * cell depends only on (seed, step, cell) and the gathered table, so the tables are
 * bitwise identical for every world size. world == 1: nccl_unique_id may be NULL. A
 * non-finite coefficient in any rank's rows of any step fails every rank with
 * QRMC_ENUMERIC. The plan owns its device tables (allocated once, reused by every run). */
typedef struct qrmc_srmc_plan qrmc_srmc_plan_t;
/* 128 bytes: an NCCL unique id made on rank 0, broadcast by the caller */
int32_t qrmc_srmc_nccl_unique_id(void* out128, char* err, size_t err_len);
int32_t qrmc_srmc_plan_create(const qrmc_srmc_problem_t* prob, const qrmc_srmc_config_t* cfg, int32_t device,
                              int32_t rank, int32_t world, const void* nccl_unique_id, int32_t keep_z,
                              qrmc_srmc_plan_t** out, char* err, size_t err_len);
/* the whole backward loop on the device (one launch + one all-gather per step) */
int32_t qrmc_srmc_plan_run(qrmc_srmc_plan_t* plan, qrmc_srmc_stats_t* stats, char* err, size_t err_len);
/* all cells' tables to the host (y: steps * cells * P; z: steps * cells * d * P or NULL) */
int32_t qrmc_srmc_plan_download(qrmc_srmc_plan_t* plan, double* y, size_t y_len, double* z, size_t z_len,
                                char* err, size_t err_len);
void* qrmc_srmc_plan_stream(const qrmc_srmc_plan_t* plan); /* the cudaStream_t every launch uses */
void qrmc_srmc_plan_destroy(qrmc_srmc_plan_t* plan);
/* rank's cells [*k0, *k1) (host-only) */
int32_t qrmc_srmc_cell_range(int64_t cells, int32_t rank, int32_t world, int64_t* k0, int64_t* k1);

/* One backward step on DEVICE tables for the cells [k_begin, k_end) on `stream`
 * (cudaStream_t, NULL = legacy default): next_dev = step-(step+1) y table (unused at the
 * last step), y_dev / z_dev = step-`step` tables (full size; only the range is written;
 * z_dev may be NULL when the driver does not read z). Enqueue only (no sync). The sharded
 * driver (srmc.py solve_sharded) calls it per rank and all-gathers each step's table. */
int32_t qrmc_srmc_step_device(const qrmc_srmc_problem_t* prob, const qrmc_srmc_config_t* cfg, int32_t step,
                              const double* next_dev, double* y_dev, double* z_dev, int64_t k_begin,
                              int64_t k_end, void* stream, char* err, size_t err_len);

#ifdef __cplusplus
}
#endif
#endif

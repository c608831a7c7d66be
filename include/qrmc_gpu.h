/* qrmc_gpu.h -- C ABI of the B200-native backward solver.
 *
 * Drop-in for the reference's backward-induction loop
 *     qrmc::CoefficientTable qrmc::backward_solve(const ProblemSpec&, const RunConfig&)
 * (proj/include/qrmc/solver.hpp:91, proj/src/solver.cpp:109-226) and for the
 * pieces of its plugin surface the loop consumes. Plain C: no C++ types cross
 * this boundary and no exception escapes it. Every entry point returns a
 * qrmc_status and, where an error buffer is passed, a NUL-terminated message.
 *
 * Mapping to the reference (file:line of the interface each entry replaces):
 *   qrmc_problem_t          ProblemSpec            proj/include/qrmc/sde.hpp:18-49
 *                           make_problem(SinBench) proj/src/benchmark.cpp:30-67
 *   qrmc_config_t           RunConfig              proj/include/qrmc/solver.hpp:24-35
 *   qrmc_gpu_backward_solve backward_solve         proj/include/qrmc/solver.hpp:91
 *   qrmc_stats_t            TruncationStats        proj/include/qrmc/solver.hpp:37-46
 *   qrmc_gpu_gamma_*        MultiIndexSet          proj/include/qrmc/multi_index.hpp:23-63
 *   qrmc_gpu_evaluate       evaluate_solution      proj/include/qrmc/solver.hpp:97-98
 *   qrmc_gpu_mse_metrics    mse_metrics            proj/include/qrmc/benchmark.hpp:62-64
 *   qrmc_gpu_philox / draws Philox4x32, RngStream  proj/include/qrmc/rng.hpp:15-65
 *
 * Errors map one-to-one onto the reference's exception taxonomy
 * (proj/include/qrmc/errors.hpp:9-35, std::invalid_argument, std::logic_error):
 *   QRMC_EINVAL    std::invalid_argument / std::domain_error
 *   QRMC_ENUMERIC  qrmc::NumericError      (solver.cpp:167-170, 210-212)
 *   QRMC_ESIM      qrmc::SimulationError   (sde.cpp:66-72), step in stats.error_step
 *   QRMC_ECAPACITY qrmc::CapacityError     (multi_index.cpp:126-127, 154-155)
 *   QRMC_ELOGIC    std::logic_error / std::out_of_range
 *   QRMC_ECUDA / QRMC_ENCCL  device or collective failure (no reference analogue)
 *   QRMC_ENOTIMPL  a problem kind with no device functor (there is no CPU fallback)
 */
#ifndef QRMC_GPU_H
#define QRMC_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QRMC_GPU_ABI_VERSION 2

typedef enum qrmc_status {
    QRMC_OK = 0,
    QRMC_EINVAL = 1,
    QRMC_ENUMERIC = 2,
    QRMC_ESIM = 3,
    QRMC_ECAPACITY = 4,
    QRMC_ECUDA = 5,
    QRMC_ENCCL = 6,
    QRMC_ENOTIMPL = 7,
    QRMC_ELOGIC = 8
} qrmc_status;

/* IndexSetKind, proj/include/qrmc/multi_index.hpp:10 */
enum { QRMC_GAMMA_FULL = 0, QRMC_GAMMA_TOTAL = 1, QRMC_GAMMA_HYPERBOLIC = 2 };

/* MemoryMode, proj/include/qrmc/solver.hpp:18 */
enum { QRMC_MEMORY_STORE_CLOUD = 0, QRMC_MEMORY_RECOMPUTE = 1 };

/* Device functors replacing ProblemSpec's std::function members
 * (proj/include/qrmc/sde.hpp:23-29). They cover make_problem(SinBenchmark)
 * and every hand-written ProblemSpec in the reference's tests. */
enum {
    QRMC_TERMINAL_SIN_SUM = 0, /* 1 + kappa + sin(lambda * sum x)   p = {kappa, lambda} (benchmark.cpp:50-54) */
    QRMC_TERMINAL_CONST = 1,   /* c                                 p = {c}              (test_solver.cpp:228) */
    QRMC_TERMINAL_X0 = 2,      /* x[0]                              (test_solver.cpp:314, acceptance_main.cpp:233) */
    QRMC_TERMINAL_NAN = 3      /* 1 / (x0 - x0): fault injection    (test_solver.cpp:286) */
};
enum {
    QRMC_DRIVER_ZERO = 0,     /* 0 */
    QRMC_DRIVER_CONST = 1,    /* c                                  p = {c} */
    QRMC_DRIVER_Y = 2,        /* y                                  (test_solver.cpp:294) */
    QRMC_DRIVER_SIN_BENCH = 3 /* min(1, (y-kappa-1-sin(lambda sum x) e^{lambda^2 d (t-T)/2})^2)
                                 p = {kappa, lambda}                (benchmark.cpp:55-62) */
};
enum {
    QRMC_DRIFT_ZERO = 0,  /* null drift (sde.hpp:23) */
    QRMC_DRIFT_CONST = 1, /* b_l = c, p = {c}; fault injection as in test_sde.cpp:143-158 */
    QRMC_DRIFT_AFFINE = 2 /* b_l(t, x) = drift_vec[l] + drift_vec[8 + l] * x_l (per-coordinate,
                             e.g. Ornstein-Uhlenbeck), evaluated at the pre-step state (sde.cpp:54-60) */
};
enum {
    QRMC_DIFFUSION_IDENTITY = 0, /* null diffusion_apply: out = dw (sde.cpp:48-53) */
    QRMC_DIFFUSION_SCALAR = 1,   /* out = sigma * dw, p = {sigma}, requires brownian_dim == dim */
    QRMC_DIFFUSION_DIAG = 2      /* out_l = diffusion_vec[l] * dw_l, requires brownian_dim == dim */
};

typedef struct qrmc_problem {
    int32_t dim;          /* d */
    int32_t brownian_dim; /* increment dimension q_w */
    double horizon;       /* T */
    int32_t terminal_kind;
    int32_t driver_kind;
    int32_t drift_kind;
    int32_t diffusion_kind;
    double terminal_params[4];
    double driver_params[4];
    double drift_params[2];
    double diffusion_params[2];
    /* assumption constants (sde.hpp:31-46) */
    double growth_g, growth_exp_g, growth_f, growth_exp_f, lipschitz_f;
    double moment_ratio; /* C_eta >= 1 */
    double state_bound;  /* |X| beyond this aborts with QRMC_ESIM */
    /* per-coordinate functor data (ABI version 2): QRMC_DRIFT_AFFINE, QRMC_DIFFUSION_DIAG */
    double drift_vec[16];
    double diffusion_vec[8];
} qrmc_problem_t;

typedef struct qrmc_config {
    int32_t steps;  /* N */
    int32_t workers; /* accepted for signature parity; never affects results */
    int64_t paths;  /* M, fresh paths per backward step */
    double damping; /* q >= 0 */
    uint64_t seed;
    int32_t memory_mode; /* QRMC_MEMORY_* */
    int32_t gamma_kind;  /* QRMC_GAMMA_* */
    const int32_t* degrees; /* full: dim per-coordinate K_l; total/hyperbolic: {DEG} */
    int32_t n_degrees;
    int32_t reserved;
    double mu;             /* Student shape, 1 or 2 on the device */
    const double* center;  /* dim entries, or NULL for the origin */
} qrmc_config_t;

typedef struct qrmc_stats {
    uint64_t applications; /* TruncationStats::applications */
    uint64_t clipped;      /* TruncationStats::clipped */
    int32_t error_step;    /* SimulationError::step() when QRMC_ESIM, else -1 */
    int32_t kernel_launches; /* device kernels launched by this call */
    double device_seconds; /* backward loop, CUDA-event timed */
} qrmc_stats_t;

/* Fill *out exactly as make_problem(SinBenchmark{dim, kappa, lambda, horizon})
 * does (benchmark.cpp:30-67). lambda <= 0 selects 1/sqrt(dim). */
qrmc_status qrmc_problem_sin_bench(int32_t dim, double kappa, double lambda, double horizon,
                                   qrmc_problem_t* out);

/* ---- multi-index sets (host; bit-exact with multi_index.cpp:96-173) ---- */
/* Number of indices, or a negative qrmc_status on error. */
int64_t qrmc_gpu_gamma_size(int32_t kind, int32_t dim, const int32_t* degrees, int32_t n_degrees);
/* Write rows (size x dim, lexicographic) into out (capacity out_len ints). */
qrmc_status qrmc_gpu_gamma_indices(int32_t kind, int32_t dim, const int32_t* degrees,
                                   int32_t n_degrees, int32_t* out, size_t out_len,
                                   char* err, size_t err_len);

/* ---- sessions: one per (process, device); holds streams, workspace, and the
 * NCCL communicator when world > 1. nccl_unique_id: 128 bytes from
 * qrmc_gpu_nccl_unique_id on rank 0, broadcast by the caller (NULL when world == 1). */
typedef struct qrmc_gpu_session qrmc_gpu_session_t;
qrmc_status qrmc_gpu_session_create(int32_t device, int32_t rank, int32_t world,
                                    const void* nccl_unique_id, qrmc_gpu_session_t** out,
                                    char* err, size_t err_len);
void qrmc_gpu_session_destroy(qrmc_gpu_session_t* session);
qrmc_status qrmc_gpu_nccl_unique_id(void* out128, char* err, size_t err_len);

/* ---- the drop-in: backward_solve ----
 * coeffs: caller-owned host buffer of steps * basis_size doubles, row-major [i][k]
 * in Gamma's lexicographic order (CoefficientTable::coefficients, solver.hpp:60).
 * step_wall_seconds: steps doubles or NULL (CoefficientTable::step_wall_seconds).
 * session may be NULL: a private single-GPU session on the current device. */
qrmc_status qrmc_gpu_backward_solve(qrmc_gpu_session_t* session, const qrmc_problem_t* problem,
                                    const qrmc_config_t* config, double* coeffs,
                                    size_t coeffs_len, double* step_wall_seconds,
                                    qrmc_stats_t* stats, char* err, size_t err_len);

/* ---- prepared solves (device-resident; used by the bench and by graphs) ---- */
typedef struct qrmc_gpu_plan qrmc_gpu_plan_t;
qrmc_status qrmc_gpu_plan_create(qrmc_gpu_session_t* session, const qrmc_problem_t* problem,
                                 const qrmc_config_t* config, qrmc_gpu_plan_t** out,
                                 char* err, size_t err_len);
/* Run the whole backward loop on the device; results stay resident. */
qrmc_status qrmc_gpu_plan_run(qrmc_gpu_plan_t* plan, qrmc_stats_t* stats, char* err,
                              size_t err_len);
qrmc_status qrmc_gpu_plan_download(qrmc_gpu_plan_t* plan, double* coeffs, size_t coeffs_len,
                                   char* err, size_t err_len);
int64_t qrmc_gpu_plan_basis_size(const qrmc_gpu_plan_t* plan);
/* Device seconds of the last run per kernel kind, summed over steps:
 * out3 = {k_responses, k_project (+ the NCCL exchange), k_finish_step};
 * per_step (steps x 3, row i = cloud step i) or NULL. CUDA-event timed inside the graph. */
qrmc_status qrmc_gpu_plan_kernel_seconds(const qrmc_gpu_plan_t* plan, double* out3, double* per_step,
                                         char* err, size_t err_len);
/* table_to_json (proj/src/table_io.cpp:45-73): the reference's
 * `qrmc.coefficients.v1` artifact, byte-identical, for `coeffs` (steps x K,
 * row-major [i][k], Gamma order) solved with `config`. Host-only. Returns the
 * length needed including the NUL (the text is written when out_len suffices),
 * or -status on error. */
int64_t qrmc_gpu_table_json(const qrmc_config_t* config, int32_t dim, double horizon, const double* coeffs,
                            char* out, size_t out_len, char* err, size_t err_len);
/* Host-only check of the tensor-core layout (no device needed): builds the
 * index set and the K1/K2 fragment layouts make_plan would use, replays both
 * kernels' data flow on the host for one random point and random coefficients,
 * and returns the relative deviation from the direct sum over Gamma.
 * info[8] = {layout used (0: series-program kernels), K, K1 units, K1 fragments
 * per series, fragments the replay read, stream length (fragments, padded),
 * K2 CTA parts, (s, b) term-table length}. Throws QRMC_ELOGIC on a layout
 * inconsistency (position clash, missed term, stream overrun). */
qrmc_status qrmc_gpu_mma_layout_check(int32_t kind, int32_t dim, const int32_t* degrees, int32_t n_degrees,
                                      uint64_t seed, int64_t* info, double* max_rel_err, char* err, size_t err_len);
/* Name of the kernel the plan runs for kind `which` (0 phase 1, 1 phase 2,
 * 2 finish): the tensor-core kernels (k_responses_mma, k_project_mma) when the
 * index set and shared memory allow them, else the series-program kernels. */
const char* qrmc_gpu_plan_kernel_name(const qrmc_gpu_plan_t* plan, int which);
/* Multi-GPU path sharding (host-only, no device needed): rank `rank` of `world`
 * owns the reference's lanes [lane_lo, lane_hi) (LaneLayout, parallel.hpp:20-36:
 * chunk c of 1024 paths belongs to lane c % 256) and n_owned paths. */
qrmc_status qrmc_gpu_lane_ownership(int64_t paths, int32_t rank, int32_t world, int32_t* lane_lo,
                                    int32_t* lane_hi, int64_t* n_owned);
/* Multi-GPU correctness on one device (test entry): the solve of a world of
 * `world` ranks with every rank's kernels run on the current device, each with
 * its own lane ownership (lane_lo > 0, owned_lanes < 256 as on a real rank),
 * its own response/cloud buffers, writing only its own lanes' partial rows --
 * the rows the per-step ncclAllGather of a world-`world` solve assembles
 * (host.cpp enqueue_solve). The reference's contract that `workers` never
 * changes results (solver.hpp:29) makes the output bitwise equal to the
 * world-1 solve for every world in [1, 256]. */
qrmc_status qrmc_gpu_replay_ranks_solve(const qrmc_problem_t* problem, const qrmc_config_t* config,
                                        int32_t world, double* coeffs, size_t coeffs_len,
                                        qrmc_stats_t* stats, char* err, size_t err_len);
/* The kernels' owned index -> global path id map, exported for host-side tests. */
int64_t qrmc_gpu_owned_path(int64_t q, int32_t lane_lo, int32_t owned_lanes);
/* Host->device and device->host bytes one qrmc_gpu_backward_solve call moves. */
qrmc_status qrmc_gpu_plan_io_bytes(const qrmc_gpu_plan_t* plan, uint64_t* h2d, uint64_t* d2h);
/* The CUDA stream every kernel of the plan is launched on (cudaStream_t). */
void* qrmc_gpu_plan_stream(const qrmc_gpu_plan_t* plan);
void qrmc_gpu_plan_destroy(qrmc_gpu_plan_t* plan);

/* ---- table evaluation on the device ----
 * evaluate_solution(table, i, x) for n points x (n x dim, row-major):
 * series value times the damping weight (solver.cpp:228-237). */
qrmc_status qrmc_gpu_evaluate(const qrmc_config_t* config, int32_t dim, const double* coeffs_step,
                              const double* x, int64_t n, double* out, char* err, size_t err_len);

/* mse_metrics(table, SinBenchmark, eval_seed, eval_points) (benchmark.cpp:86-151).
 * out6 = {mse_max, mse_av, mse_max_undamped, mse_av_undamped, 0, 0};
 * step_sq (steps doubles or NULL) = damped per-step sums. */
qrmc_status qrmc_gpu_mse_metrics(const qrmc_config_t* config, int32_t dim, double kappa,
                                 double lambda, double horizon, const double* coeffs,
                                 uint64_t eval_seed, int32_t eval_points, double* out6,
                                 double* step_sq, char* err, size_t err_len);

/* ---- replay probes: the device's random draws, for parity with the oracle ---- */
/* Philox4x32-10 blocks: ctr n x 4, key n x 2 -> out n x 4 (rng.cpp:31-40). */
qrmc_status qrmc_gpu_philox(const uint32_t* ctr, const uint32_t* key, int64_t n, uint32_t* out,
                            char* err, size_t err_len);
/* Stream draws for (seed, stream_id[r]), r < n_streams, draws 0..n_draws-1:
 * kind 0 = next_u64 (out as uint64), 1 = next_uniform, 2 = next_normal. */
qrmc_status qrmc_gpu_stream_draws(uint64_t seed, const uint64_t* stream_ids, int64_t n_streams,
                                  int32_t n_draws, int32_t kind, void* out, char* err,
                                  size_t err_len);
/* Euler paths of cloud `step` for paths [first, first+n): out n x (steps-step+1) x dim
 * (solver.cpp:153-164: sample from nu, then euler_step for j = step..steps-1). */
qrmc_status qrmc_gpu_cloud_paths(const qrmc_problem_t* problem, const qrmc_config_t* config,
                                 int32_t step, int64_t first, int64_t n, double* out, char* err,
                                 size_t err_len);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* QRMC_GPU_H */

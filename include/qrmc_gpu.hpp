// qrmc_gpu.hpp -- header-only C++ drop-in over the C ABI (include/qrmc_gpu.h).
//
// Mirrors the reference's entry point
//     qrmc::CoefficientTable qrmc::backward_solve(const ProblemSpec&, const RunConfig&)
// (proj/include/qrmc/solver.hpp:91) with the same exception taxonomy
// (proj/include/qrmc/errors.hpp:9-35). ProblemSpec holds std::function
// members that cannot run on the device, so the GPU call takes the problem as
// a device-functor descriptor (qrmc_problem_t; qrmc_gpu::sin_benchmark mirrors
// make_problem(SinBenchmark), benchmark.cpp:30-67).
//
// Two layers:
//   * qrmc_gpu::backward_solve(problem, Config) -> Table: no reference headers needed.
//   * with QRMC_GPU_WITH_REFERENCE_TYPES defined after including the
//     reference's "qrmc/solver.hpp": qrmc_gpu::backward_solve(problem,
//     qrmc::RunConfig) -> qrmc::CoefficientTable, throwing qrmc::CapacityError,
//     qrmc::SimulationError, qrmc::NumericError, std::invalid_argument,
//     std::logic_error exactly where the reference does. INTEGRATION.md shows
//     the two-line change at the reference's call sites.
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "qrmc_gpu.h"

namespace qrmc_gpu {

struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// The index-set and measure part of RunConfig as plain values.
struct Config {
    int steps = 1;
    std::int64_t paths = 1;
    double damping = 0.0;
    std::uint64_t seed = 0;
    int workers = 0;
    int memory_mode = QRMC_MEMORY_STORE_CLOUD;
    int gamma_kind = QRMC_GAMMA_FULL;
    std::vector<std::int32_t> degrees{1};
    double mu = 2.0;
    std::vector<double> center;  // empty = origin
};

struct Table {
    int steps = 0;
    std::int64_t basis_size = 0;
    std::vector<std::vector<double>> coefficients;  // [i][k], Gamma order
    qrmc_stats_t stats{};
    std::vector<double> step_wall_seconds;
};

inline qrmc_problem_t sin_benchmark(int dim, double kappa = 0.6, double lambda = 0.0, double horizon = 1.0) {
    qrmc_problem_t p{};
    if (qrmc_problem_sin_bench(dim, kappa, lambda, horizon, &p) != QRMC_OK)
        throw std::invalid_argument("SinBenchmark: dim must be >= 1 and horizon positive");
    return p;
}

inline qrmc_config_t to_c(const Config& c) {
    qrmc_config_t out{};
    out.steps = c.steps;
    out.workers = c.workers;
    out.paths = c.paths;
    out.damping = c.damping;
    out.seed = c.seed;
    out.memory_mode = c.memory_mode;
    out.gamma_kind = c.gamma_kind;
    out.degrees = c.degrees.data();
    out.n_degrees = static_cast<std::int32_t>(c.degrees.size());
    out.mu = c.mu;
    out.center = c.center.empty() ? nullptr : c.center.data();
    return out;
}

// Throws the standard-library analogue of each status; the reference-typed
// overload below maps them onto qrmc's own exception classes.
template <class OnCapacity, class OnSimulation, class OnNumeric>
inline void raise(qrmc_status st, const char* msg, int step, OnCapacity cap, OnSimulation sim, OnNumeric num) {
    switch (st) {
        case QRMC_OK: return;
        case QRMC_EINVAL: throw std::invalid_argument(msg);
        case QRMC_ELOGIC: throw std::logic_error(msg);
        case QRMC_ECAPACITY: cap(msg); break;
        case QRMC_ESIM: sim(msg, step); break;
        case QRMC_ENUMERIC: num(msg); break;
        default: break;
    }
    throw DeviceError(msg);
}

inline Table backward_solve(const qrmc_problem_t& problem, const Config& config,
                            qrmc_gpu_session_t* session = nullptr) {
    const qrmc_config_t c = to_c(config);
    const std::int64_t k = qrmc_gpu_gamma_size(c.gamma_kind, problem.dim, c.degrees, c.n_degrees);
    if (k < 0) {
        const auto st = static_cast<qrmc_status>(-k);
        raise(st, "multi-index set construction failed", -1,
              [](const char* m) { throw std::length_error(m); },
              [](const char* m, int) { throw std::runtime_error(m); },
              [](const char* m) { throw std::runtime_error(m); });
    }
    Table t;
    t.steps = config.steps;
    t.basis_size = k;
    std::vector<double> flat(static_cast<size_t>(std::max(config.steps, 0)) * static_cast<size_t>(k));
    t.step_wall_seconds.assign(static_cast<size_t>(std::max(config.steps, 0)), 0.0);
    char err[1024] = {0};
    const qrmc_status st = qrmc_gpu_backward_solve(session, &problem, &c, flat.data(), flat.size(),
                                                   t.step_wall_seconds.data(), &t.stats, err, sizeof err);
    raise(st, err, t.stats.error_step,
          [](const char* m) { throw std::length_error(m); },
          [](const char* m, int) { throw std::runtime_error(m); },
          [](const char* m) { throw std::runtime_error(m); });
    t.coefficients.resize(static_cast<size_t>(config.steps));
    for (int i = 0; i < config.steps; ++i)
        t.coefficients[static_cast<size_t>(i)].assign(flat.begin() + static_cast<std::ptrdiff_t>(i * k),
                                                      flat.begin() + static_cast<std::ptrdiff_t>((i + 1) * k));
    return t;
}

#ifdef QRMC_GPU_WITH_REFERENCE_TYPES
// Drop-in with the reference's types (include "qrmc/solver.hpp" and
// "qrmc/errors.hpp" first). RunConfig::gamma / ::measure are read through
// their public accessors (multi_index.hpp:38-44, student.hpp:29-31).
inline qrmc::CoefficientTable backward_solve(const qrmc_problem_t& problem, const qrmc::RunConfig& rc,
                                             qrmc_gpu_session_t* session = nullptr) {
    Config c;
    c.steps = rc.steps;
    c.paths = rc.paths;
    c.damping = rc.damping;
    c.seed = rc.seed;
    c.workers = rc.workers;
    c.memory_mode = rc.memory_mode == qrmc::MemoryMode::RecomputeFromSeeds ? QRMC_MEMORY_RECOMPUTE
                                                                          : QRMC_MEMORY_STORE_CLOUD;
    c.gamma_kind = rc.gamma.kind() == qrmc::IndexSetKind::Full    ? QRMC_GAMMA_FULL
                   : rc.gamma.kind() == qrmc::IndexSetKind::Total ? QRMC_GAMMA_TOTAL
                                                                  : QRMC_GAMMA_HYPERBOLIC;
    c.degrees.assign(rc.gamma.degrees().begin(), rc.gamma.degrees().end());
    c.mu = rc.measure.mu();
    c.center = rc.measure.center();
    const qrmc_config_t cc = to_c(c);
    const std::int64_t k = static_cast<std::int64_t>(rc.gamma.size());
    std::vector<double> flat(static_cast<size_t>(rc.steps) * static_cast<size_t>(k));
    std::vector<double> wall(static_cast<size_t>(rc.steps), 0.0);
    qrmc_stats_t stats{};
    char err[1024] = {0};
    const qrmc_status st =
        qrmc_gpu_backward_solve(session, &problem, &cc, flat.data(), flat.size(), wall.data(), &stats, err, sizeof err);
    raise(st, err, stats.error_step,
          [](const char* m) { throw qrmc::CapacityError(m); },
          [](const char* m, int step) { throw qrmc::SimulationError(m, step); },
          [](const char* m) { throw qrmc::NumericError(m); });
    qrmc::CoefficientTable t{.steps = rc.steps,
                             .paths = rc.paths,
                             .damping = rc.damping,
                             .seed = rc.seed,
                             .horizon = problem.horizon,
                             .measure = rc.measure,
                             .gamma = rc.gamma,
                             .coefficients = {},
                             .truncation = {},
                             .step_wall_seconds = wall};
    t.coefficients.resize(static_cast<size_t>(rc.steps));
    for (int i = 0; i < rc.steps; ++i)
        t.coefficients[static_cast<size_t>(i)].assign(flat.begin() + static_cast<std::ptrdiff_t>(i * k),
                                                      flat.begin() + static_cast<std::ptrdiff_t>((i + 1) * k));
    t.truncation.applications = stats.applications;
    t.truncation.clipped = stats.clipped;
    return t;
}
#endif

}  // namespace qrmc_gpu

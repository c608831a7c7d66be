// ref_capi.cpp -- C entry points over the UNMODIFIED reference sources.
//
// TEST INFRASTRUCTURE ONLY. Compiled by oracle/Makefile together with
// /root/reference/proj/src/*.cpp (never copied into this repo) into
// oracle/_ref/libqrmc_ref.so. It lets tests/, tests/golden/make_golden.py and
// bench.py's reference arm drive the reference's own public API
// (backward_solve, response, evaluate_solution, mse_metrics, RngStream, ...)
// with the same plain-C descriptors as include/qrmc_gpu.h. Nothing in the
// product (paper_2407_21084_b200/) loads this library.
#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "qrmc/benchmark.hpp"
#include "qrmc/cosine_basis.hpp"
#include "qrmc/errors.hpp"
#include "qrmc/multi_index.hpp"
#include "qrmc/rng.hpp"
#include "qrmc/sde.hpp"
#include "qrmc/solver.hpp"
#include "qrmc/student.hpp"
#include "qrmc/table_io.hpp"
#include "qrmc_gpu.h"

using namespace qrmc;

namespace {

void set_err(char* err, size_t len, const std::string& msg) {
    if (!err || len == 0) return;
    std::strncpy(err, msg.c_str(), len - 1);
    err[len - 1] = '\0';
}

template <class Fn>
int guarded(char* err, size_t len, Fn&& fn, int* error_step = nullptr) {
    try {
        fn();
        return QRMC_OK;
    } catch (const CapacityError& e) {
        set_err(err, len, e.what());
        return QRMC_ECAPACITY;
    } catch (const SimulationError& e) {
        set_err(err, len, e.what());
        if (error_step) *error_step = e.step();
        return QRMC_ESIM;
    } catch (const NumericError& e) {
        set_err(err, len, e.what());
        return QRMC_ENUMERIC;
    } catch (const std::invalid_argument& e) {
        set_err(err, len, e.what());
        return QRMC_EINVAL;
    } catch (const std::domain_error& e) {
        set_err(err, len, e.what());
        return QRMC_EINVAL;
    } catch (const std::out_of_range& e) {
        set_err(err, len, e.what());
        return QRMC_ELOGIC;
    } catch (const std::logic_error& e) {
        set_err(err, len, e.what());
        return QRMC_ELOGIC;
    } catch (const std::exception& e) {
        set_err(err, len, e.what());
        return QRMC_EINVAL;
    }
}

double sum_of(std::span<const double> x) {
    double s = 0.0;
    for (double v : x) s += v;
    return s;
}

// qrmc_problem_t -> ProblemSpec. The SinBenchmark pair goes through the
// reference's own make_problem; the test-only kinds are the lambdas of
// proj/tests/test_solver.cpp written out once more.
ProblemSpec to_spec(const qrmc_problem_t& p) {
    if (p.terminal_kind == QRMC_TERMINAL_SIN_SUM && p.driver_kind == QRMC_DRIVER_SIN_BENCH &&
        p.drift_kind == QRMC_DRIFT_ZERO && p.diffusion_kind == QRMC_DIFFUSION_IDENTITY &&
        p.terminal_params[0] == p.driver_params[0] &&
        p.terminal_params[1] == p.driver_params[1]) {
        SinBenchmark bench{p.dim, p.terminal_params[0], p.terminal_params[1], p.horizon};
        ProblemSpec spec = make_problem(bench);
        spec.growth_g = p.growth_g;
        spec.growth_exp_g = p.growth_exp_g;
        spec.growth_f = p.growth_f;
        spec.growth_exp_f = p.growth_exp_f;
        spec.lipschitz_f = p.lipschitz_f;
        spec.moment_ratio = p.moment_ratio;
        spec.state_bound = p.state_bound;
        return spec;
    }
    ProblemSpec spec;
    spec.dim = p.dim;
    spec.brownian_dim = p.brownian_dim;
    spec.horizon = p.horizon;
    const double tp0 = p.terminal_params[0], tp1 = p.terminal_params[1];
    switch (p.terminal_kind) {
        case QRMC_TERMINAL_SIN_SUM:
            spec.terminal = [tp0, tp1](std::span<const double> x) {
                return 1.0 + tp0 + std::sin(tp1 * sum_of(x));
            };
            break;
        case QRMC_TERMINAL_CONST:
            spec.terminal = [tp0](std::span<const double>) { return tp0; };
            break;
        case QRMC_TERMINAL_X0:
            spec.terminal = [](std::span<const double> x) { return x[0]; };
            break;
        case QRMC_TERMINAL_NAN:
            spec.terminal = [](std::span<const double> x) { return 1.0 / (x[0] - x[0]); };
            break;
        default:
            throw std::invalid_argument("unknown terminal kind");
    }
    const double dp0 = p.driver_params[0], dp1 = p.driver_params[1];
    const int d = p.dim;
    const double horizon = p.horizon;
    switch (p.driver_kind) {
        case QRMC_DRIVER_ZERO:
            spec.driver = [](double, std::span<const double>, double) { return 0.0; };
            break;
        case QRMC_DRIVER_CONST:
            spec.driver = [dp0](double, std::span<const double>, double) { return dp0; };
            break;
        case QRMC_DRIVER_Y:
            spec.driver = [](double, std::span<const double>, double y) { return y; };
            break;
        case QRMC_DRIVER_SIN_BENCH:
            spec.driver = [dp0, dp1, d, horizon](double t, std::span<const double> x, double y) {
                const double z = y - dp0 - 1.0 -
                                 std::sin(dp1 * sum_of(x)) *
                                     std::exp(dp1 * dp1 * d * (t - horizon) / 2.0);
                return std::min(1.0, z * z);
            };
            break;
        default:
            throw std::invalid_argument("unknown driver kind");
    }
    if (p.drift_kind == QRMC_DRIFT_CONST) {
        const double c = p.drift_params[0];
        spec.drift = [c](double, std::span<const double>, std::span<double> out) {
            for (double& v : out) v = c;
        };
    } else if (p.drift_kind == QRMC_DRIFT_AFFINE) {
        std::vector<double> a(p.drift_vec, p.drift_vec + 8), b(p.drift_vec + 8, p.drift_vec + 16);
        spec.drift = [a, b](double, std::span<const double> x, std::span<double> out) {
            for (std::size_t l = 0; l < out.size(); ++l) out[l] = a[l] + b[l] * x[l];
        };
    } else if (p.drift_kind != QRMC_DRIFT_ZERO) {
        throw std::invalid_argument("unknown drift kind");
    }
    if (p.diffusion_kind == QRMC_DIFFUSION_SCALAR) {
        const double s = p.diffusion_params[0];
        spec.diffusion_apply = [s](double, std::span<const double>, std::span<const double> dw,
                                   std::span<double> out) {
            for (std::size_t l = 0; l < out.size(); ++l) out[l] = s * dw[l];
        };
    } else if (p.diffusion_kind == QRMC_DIFFUSION_DIAG) {
        std::vector<double> sg(p.diffusion_vec, p.diffusion_vec + 8);
        spec.diffusion_apply = [sg](double, std::span<const double>, std::span<const double> dw,
                                    std::span<double> out) {
            for (std::size_t l = 0; l < out.size(); ++l) out[l] = sg[l] * dw[l];
        };
    } else if (p.diffusion_kind != QRMC_DIFFUSION_IDENTITY) {
        throw std::invalid_argument("unknown diffusion kind");
    }
    spec.growth_g = p.growth_g;
    spec.growth_exp_g = p.growth_exp_g;
    spec.growth_f = p.growth_f;
    spec.growth_exp_f = p.growth_exp_f;
    spec.lipschitz_f = p.lipschitz_f;
    spec.moment_ratio = p.moment_ratio;
    spec.state_bound = p.state_bound;
    return spec;
}

MultiIndexSet to_gamma(int kind, int dim, const int32_t* degrees, int n_degrees) {
    switch (kind) {
        case QRMC_GAMMA_FULL: {
            if (n_degrees == 1 && dim > 1)
                return MultiIndexSet::full(std::vector<int>(static_cast<std::size_t>(dim), degrees[0]));
            return MultiIndexSet::full(std::vector<int>(degrees, degrees + n_degrees));
        }
        case QRMC_GAMMA_TOTAL:
            return MultiIndexSet::total(dim, degrees[0]);
        case QRMC_GAMMA_HYPERBOLIC:
            return MultiIndexSet::hyperbolic(dim, degrees[0]);
    }
    throw std::invalid_argument("unknown index set kind");
}

SamplingMeasure to_measure(const qrmc_config_t& c, int dim) {
    std::vector<double> center;
    if (c.center) center.assign(c.center, c.center + dim);
    return SamplingMeasure(c.mu, dim, center);
}

RunConfig to_config(const qrmc_config_t& c, int dim) {
    return RunConfig{.steps = c.steps,
                     .paths = c.paths,
                     .damping = c.damping,
                     .seed = c.seed,
                     .workers = c.workers,
                     .memory_mode = c.memory_mode == QRMC_MEMORY_RECOMPUTE
                                        ? MemoryMode::RecomputeFromSeeds
                                        : MemoryMode::StoreCloud,
                     .gamma = to_gamma(c.gamma_kind, dim, c.degrees, c.n_degrees),
                     .measure = to_measure(c, dim)};
}

CoefficientTable table_from(const qrmc_config_t& c, int dim, double horizon,
                            const double* coeffs, const uint8_t* have_step) {
    RunConfig cfg = to_config(c, dim);
    CoefficientTable t{.steps = c.steps,
                       .paths = c.paths,
                       .damping = c.damping,
                       .seed = c.seed,
                       .horizon = horizon,
                       .measure = cfg.measure,
                       .gamma = cfg.gamma,
                       .coefficients = {},
                       .truncation = {},
                       .step_wall_seconds = {}};
    const std::size_t k = cfg.gamma.size();
    t.coefficients.resize(static_cast<std::size_t>(c.steps));
    for (int i = 0; i < c.steps; ++i)
        if (!have_step || have_step[i])
            t.coefficients[static_cast<std::size_t>(i)].assign(coeffs + i * k, coeffs + (i + 1) * k);
    return t;
}

}  // namespace

extern "C" {

int qrmc_ref_philox(const uint32_t* ctr, const uint32_t* key, int64_t n, uint32_t* out) {
    for (int64_t r = 0; r < n; ++r) {
        const auto o = Philox4x32::block({ctr[4 * r], ctr[4 * r + 1], ctr[4 * r + 2], ctr[4 * r + 3]},
                                         {key[2 * r], key[2 * r + 1]});
        for (int w = 0; w < 4; ++w) out[4 * r + w] = o[static_cast<std::size_t>(w)];
    }
    return QRMC_OK;
}

int qrmc_ref_stream_draws(uint64_t seed, const uint64_t* sids, int64_t n, int32_t n_draws,
                          int32_t kind, void* out) {
    for (int64_t r = 0; r < n; ++r) {
        RngStream s(seed, sids[r]);
        for (int32_t k = 0; k < n_draws; ++k) {
            const std::size_t at = static_cast<std::size_t>(r) * n_draws + k;
            if (kind == 0)
                static_cast<uint64_t*>(out)[at] = s.next_u64();
            else if (kind == 1)
                static_cast<double*>(out)[at] = s.next_uniform();
            else
                static_cast<double*>(out)[at] = s.next_normal();
        }
    }
    return QRMC_OK;
}

double qrmc_ref_normal_quantile(double p) { return normal_quantile(p); }

// op 0 = pdf, 1 = cdf, 2 = inv_cdf (coordinate `coord`)
int qrmc_ref_measure(double mu, int32_t dim, const double* center, int32_t op, int32_t coord,
                     const double* x, int64_t n, double* out, char* err, size_t err_len) {
    return guarded(err, err_len, [&] {
        std::vector<double> c;
        if (center) c.assign(center, center + dim);
        SamplingMeasure m(mu, dim, c);
        for (int64_t r = 0; r < n; ++r)
            out[r] = op == 0 ? m.pdf(x[r], coord) : op == 1 ? m.cdf(x[r], coord) : m.inv_cdf(x[r], coord);
    });
}

int64_t qrmc_ref_gamma_size(int32_t kind, int32_t dim, const int32_t* degrees, int32_t n_degrees) {
    int64_t size = 0;
    const int rc = guarded(nullptr, 0, [&] {
        size = static_cast<int64_t>(to_gamma(kind, dim, degrees, n_degrees).size());
    });
    return rc == QRMC_OK ? size : -rc;
}

int qrmc_ref_gamma_indices(int32_t kind, int32_t dim, const int32_t* degrees, int32_t n_degrees,
                           int32_t* out, size_t out_len, int32_t* kmax_out, char* err,
                           size_t err_len) {
    return guarded(err, err_len, [&] {
        const auto g = to_gamma(kind, dim, degrees, n_degrees);
        if (g.size() * static_cast<std::size_t>(dim) > out_len)
            throw std::invalid_argument("output buffer too small");
        for (std::size_t i = 0; i < g.size(); ++i)
            for (int l = 0; l < dim; ++l) out[i * dim + l] = g[i][static_cast<std::size_t>(l)];
        if (kmax_out)
            for (int l = 0; l < dim; ++l) kmax_out[l] = g.max_degree_per_coord()[static_cast<std::size_t>(l)];
    });
}

double qrmc_ref_christoffel(int32_t kind, int32_t dim, const int32_t* degrees, int32_t n_degrees) {
    return christoffel_number(to_gamma(kind, dim, degrees, n_degrees));
}

uint64_t qrmc_ref_cardinality(int32_t kind, int32_t dim, int32_t degree) {
    return kind == QRMC_GAMMA_TOTAL ? cardinality_total(dim, degree)
                                    : cardinality_hyperbolic(dim, degree);
}

int qrmc_ref_backward_solve(const qrmc_problem_t* problem, const qrmc_config_t* config,
                            double* coeffs, size_t coeffs_len, double* step_wall,
                            qrmc_stats_t* stats, char* err, size_t err_len) {
    int error_step = -1;
    const int rc = guarded(
        err, err_len,
        [&] {
            const ProblemSpec spec = to_spec(*problem);
            const RunConfig cfg = to_config(*config, problem->dim);
            const auto t0 = std::chrono::steady_clock::now();
            const CoefficientTable t = backward_solve(spec, cfg);
            const double secs =
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            const std::size_t k = cfg.gamma.size();
            if (coeffs_len < k * static_cast<std::size_t>(t.steps))
                throw std::invalid_argument("coefficient buffer too small");
            for (int i = 0; i < t.steps; ++i)
                std::memcpy(coeffs + i * k, t.coefficients[static_cast<std::size_t>(i)].data(),
                            k * sizeof(double));
            if (step_wall)
                for (int i = 0; i < t.steps; ++i) step_wall[i] = t.step_wall_seconds[static_cast<std::size_t>(i)];
            if (stats) {
                stats->applications = t.truncation.applications;
                stats->clipped = t.truncation.clipped;
                stats->device_seconds = secs;
                stats->kernel_launches = 0;
            }
        },
        &error_step);
    if (stats) stats->error_step = error_step;
    return rc;
}

// Euler paths of cloud `step`, exactly as backward_solve phase 1 draws them
// (solver.cpp:153-164): sample X_i from nu, then euler_step for j = i..N-1.
int qrmc_ref_cloud_paths(const qrmc_problem_t* problem, const qrmc_config_t* config, int32_t step,
                         int64_t first, int64_t n, double* out, char* err, size_t err_len) {
    return guarded(err, err_len, [&] {
        const ProblemSpec spec = to_spec(*problem);
        const SamplingMeasure measure = to_measure(*config, problem->dim);
        const int d = spec.dim;
        const double dt = spec.horizon / config->steps;
        const std::size_t len = static_cast<std::size_t>(config->steps - step + 1) * d;
        const std::size_t scratch = static_cast<std::size_t>(std::max(spec.dim, spec.brownian_dim));
        std::vector<double> dw(scratch), diff(scratch);
        for (int64_t r = 0; r < n; ++r) {
            double* path = out + static_cast<std::size_t>(r) * len;
            RngStream stream(config->seed,
                             stream_ids::training(step, static_cast<std::uint64_t>(first + r)));
            std::span<double> state(path, static_cast<std::size_t>(d));
            measure.sample(stream, state);
            for (int j = step; j < config->steps; ++j) {
                std::span<double> next(path + static_cast<std::size_t>(j + 1 - step) * d,
                                       static_cast<std::size_t>(d));
                std::copy(state.begin(), state.end(), next.begin());
                euler_step(next, j * dt, dt, spec, stream, dw, diff, j);
                state = next;
            }
        }
    });
}

// response(path, table, spec) for n stored paths starting at `start`
// (solver.cpp:90-107). have_step marks computed table rows.
int qrmc_ref_response(const qrmc_problem_t* problem, const qrmc_config_t* config,
                      const double* coeffs, const uint8_t* have_step, int32_t start,
                      const double* paths, int64_t n, double* out, uint64_t* applications,
                      uint64_t* clipped, char* err, size_t err_len) {
    return guarded(err, err_len, [&] {
        const ProblemSpec spec = to_spec(*problem);
        const CoefficientTable t = table_from(*config, problem->dim, spec.horizon, coeffs, have_step);
        const int d = spec.dim;
        const std::size_t len = static_cast<std::size_t>(config->steps - start + 1) * d;
        TruncationStats stats;
        for (int64_t r = 0; r < n; ++r) {
            PathBundle b;
            b.start = start;
            b.dim = d;
            b.points.assign(paths + r * len, paths + (r + 1) * len);
            out[r] = response(b, t, spec, &stats);
        }
        if (applications) *applications = stats.applications;
        if (clipped) *clipped = stats.clipped;
    });
}

// evaluate_solution(table, i, x) for n points (solver.cpp:228-237)
int qrmc_ref_evaluate(const qrmc_config_t* config, int32_t dim, const double* coeffs_step,
                      const double* x, int64_t n, double* out, char* err, size_t err_len) {
    return guarded(err, err_len, [&] {
        const RunConfig cfg = to_config(*config, dim);
        SeriesEvaluator ev(cfg.measure, cfg.gamma);
        const std::span<const double> c(coeffs_step, cfg.gamma.size());
        for (int64_t r = 0; r < n; ++r) {
            const std::span<const double> p(x + r * dim, static_cast<std::size_t>(dim));
            out[r] = ev.eval(c, p) * damping_weight(p, config->damping);
        }
    });
}

// SeriesEvaluator::eval without the weight, for kernel-level parity.
int qrmc_ref_eval_series(const qrmc_config_t* config, int32_t dim, const double* coeffs_step,
                         const double* x, int64_t n, double* out, char* err, size_t err_len) {
    return guarded(err, err_len, [&] {
        const RunConfig cfg = to_config(*config, dim);
        SeriesEvaluator ev(cfg.measure, cfg.gamma);
        const std::span<const double> c(coeffs_step, cfg.gamma.size());
        for (int64_t r = 0; r < n; ++r)
            out[r] = ev.eval(c, std::span<const double>(x + r * dim, static_cast<std::size_t>(dim)));
    });
}

int qrmc_ref_mse_metrics(const qrmc_config_t* config, int32_t dim, double kappa, double lambda,
                         double horizon, const double* coeffs, uint64_t eval_seed,
                         int32_t eval_points, double* out6, double* step_sq, char* err,
                         size_t err_len) {
    return guarded(err, err_len, [&] {
        const CoefficientTable t = table_from(*config, dim, horizon, coeffs, nullptr);
        SinBenchmark bench{dim, kappa, lambda, horizon};
        const MetricReport r = mse_metrics(t, bench, eval_seed, eval_points, config->workers);
        out6[0] = r.mse_max;
        out6[1] = r.mse_av;
        out6[2] = r.mse_max_undamped;
        out6[3] = r.mse_av_undamped;
        out6[4] = r.stat_error_indicator;
        out6[5] = 0.0;
        if (step_sq)
            for (int i = 0; i < t.steps; ++i) step_sq[i] = r.step_squared_error[static_cast<std::size_t>(i)];
    });
}

double qrmc_ref_exact_solution(double t, const double* x, int32_t dim, double kappa,
                               double lambda, double horizon) {
    SinBenchmark bench{dim, kappa, lambda, horizon};
    return exact_solution(t, std::span<const double>(x, static_cast<std::size_t>(dim)), bench);
}

// table_to_json bytes (table_io.cpp:45-73); returns needed length incl. NUL.
int64_t qrmc_ref_table_json(const qrmc_config_t* config, int32_t dim, double horizon,
                            const double* coeffs, char* out, size_t out_len) {
    std::string s;
    const int rc = guarded(nullptr, 0, [&] {
        s = table_to_json(table_from(*config, dim, horizon, coeffs, nullptr));
    });
    if (rc != QRMC_OK) return -rc;
    if (out && out_len > s.size()) std::memcpy(out, s.c_str(), s.size() + 1);
    return static_cast<int64_t>(s.size() + 1);
}

}  // extern "C"

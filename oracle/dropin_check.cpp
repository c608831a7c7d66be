// dropin_check.cpp -- TEST INFRASTRUCTURE ONLY (built into oracle/_ref by oracle/Makefile).
//
// A reference call site using the header-only drop-in include/qrmc_gpu.hpp
// with the reference's OWN types (QRMC_GPU_WITH_REFERENCE_TYPES): compiled in
// the build container against /root/reference/proj/include and the unmodified
// reference sources (the checker), linked against libqrmc_gpu.so, and run on a
// B200 by tests/test_cxx_dropin.py. It checks, side by side with the
// reference's own qrmc::backward_solve (proj/src/solver.cpp:109-226):
//   1. the acceptance determinism criterion (proj/tests/acceptance_main.cpp:369-395)
//      through the drop-in: repeat, store == recompute, workers = 1 give
//      byte-identical qrmc.coefficients.v1 artifacts (table_to_json);
//   2. the drop-in's CoefficientTable against the reference's on the same inputs
//      (d = 2 series kernels, d = 4 tensor-core kernels): coefficients within the
//      DESIGN.md bar, TruncationStats equal, the snapshot fields equal;
//   3. the exception taxonomy: std::invalid_argument with the reference's
//      message, qrmc::SimulationError with the same step, qrmc::NumericError.
// Exit code 0 and "DROPIN OK" on success; every check prints one line.
#include <cmath>
#include <cstdio>
#include <span>
#include <string>

#include "qrmc/benchmark.hpp"
#include "qrmc/errors.hpp"
#include "qrmc/solver.hpp"
#include "qrmc/table_io.hpp"
#define QRMC_GPU_WITH_REFERENCE_TYPES
#include "qrmc_gpu.hpp"

using namespace qrmc;

static int failures = 0;

static void check(bool ok, const std::string& what) {
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", what.c_str());
    if (!ok) ++failures;
}

static double rel_diff(const CoefficientTable& a, const CoefficientTable& b) {
    double d = 0.0, s = 1.0;
    for (size_t i = 0; i < a.coefficients.size(); ++i)
        for (size_t k = 0; k < a.coefficients[i].size(); ++k) {
            d = std::max(d, std::fabs(a.coefficients[i][k] - b.coefficients[i][k]));
            s = std::max(s, std::fabs(b.coefficients[i][k]));
        }
    return d / s;
}

static void compare(const char* name, const ProblemSpec& spec, const qrmc_problem_t& dev, const RunConfig& cfg) {
    const CoefficientTable ref = backward_solve(spec, cfg);
    const CoefficientTable gpu = qrmc_gpu::backward_solve(dev, cfg);
    const double rd = rel_diff(gpu, ref);
    char buf[256];
    std::snprintf(buf, sizeof buf, "%s: max |alpha_gpu - alpha_ref| / max(1, |alpha_ref|) = %.2e (bar 1e-10)", name, rd);
    check(gpu.coefficients.size() == ref.coefficients.size() && rd <= 1e-10, buf);
    check(gpu.truncation.applications == ref.truncation.applications && gpu.truncation.clipped == ref.truncation.clipped,
          std::string(name) + ": TruncationStats equal (" + std::to_string(gpu.truncation.applications) + ", " +
              std::to_string(gpu.truncation.clipped) + ")");
    check(gpu.steps == ref.steps && gpu.paths == ref.paths && gpu.seed == ref.seed && gpu.damping == ref.damping &&
              gpu.gamma.size() == ref.gamma.size() && gpu.measure.mu() == ref.measure.mu() &&
              gpu.step_wall_seconds.size() == ref.step_wall_seconds.size(),
          std::string(name) + ": table snapshot fields equal");
}

template <class E, class Fn>
static std::string what_of(Fn&& fn, int* step = nullptr) {
    try {
        fn();
    } catch (const E& e) {
        if constexpr (std::is_same_v<E, SimulationError>)
            if (step) *step = e.step();
        return e.what();
    } catch (const std::exception& e) {
        return std::string("WRONG TYPE: ") + e.what();
    }
    return "NO EXCEPTION";
}

int main() {
    // 1. acceptance_main.cpp:369-395 through the drop-in
    {
        SinBenchmark bench{2, 0.6, 0.0, 1.0};
        const qrmc_problem_t dev = qrmc_gpu::sin_benchmark(2, 0.6, 0.0, 1.0);
        auto cfg = RunConfig{.steps = 5,
                             .paths = 4000,
                             .damping = 2.1,
                             .seed = 4242,
                             .workers = 0,
                             .memory_mode = MemoryMode::StoreCloud,
                             .gamma = MultiIndexSet::hyperbolic(2, 6),
                             .measure = SamplingMeasure(2.0, 2)};
        const auto a = qrmc_gpu::backward_solve(dev, cfg);
        const auto b = qrmc_gpu::backward_solve(dev, cfg);
        cfg.memory_mode = MemoryMode::RecomputeFromSeeds;
        const auto c = qrmc_gpu::backward_solve(dev, cfg);
        cfg.workers = 1;
        const auto d = qrmc_gpu::backward_solve(dev, cfg);
        const std::string ja = table_to_json(a), jb = table_to_json(b), jc = table_to_json(c), jd = table_to_json(d);
        check(ja == jb && ja == jc && ja == jd && a.coefficients == c.coefficients,
              "acceptance determinism criterion through the drop-in (repeat, store==recompute, workers=1)");
        cfg.memory_mode = MemoryMode::StoreCloud;
        cfg.workers = 0;
        compare("SinBenchmark d=2 hyperbolic(2,6)", make_problem(bench), dev, cfg);
    }
    // 2. the tensor-core kernels (d = 4) against the reference
    {
        SinBenchmark bench{4, 0.6, 0.0, 1.0};
        const auto cfg = RunConfig{.steps = 3,
                                   .paths = 2100,
                                   .damping = 5.1,
                                   .seed = 5,
                                   .workers = 0,
                                   .memory_mode = MemoryMode::StoreCloud,
                                   .gamma = MultiIndexSet::hyperbolic(4, 16),
                                   .measure = SamplingMeasure(2.0, 4)};
        compare("SinBenchmark d=4 hyperbolic(4,16)", make_problem(bench), qrmc_gpu::sin_benchmark(4), cfg);
    }
    // 3. the exception taxonomy
    {
        SinBenchmark bench{2, 0.6, 0.0, 1.0};
        const auto spec = make_problem(bench);
        const qrmc_problem_t dev = qrmc_gpu::sin_benchmark(2);
        auto cfg = RunConfig{.steps = 0, .paths = 100, .gamma = MultiIndexSet::hyperbolic(2, 4),
                             .measure = SamplingMeasure(2.0, 2)};
        const std::string r1 = what_of<std::invalid_argument>([&] { backward_solve(spec, cfg); });
        const std::string g1 = what_of<std::invalid_argument>([&] { qrmc_gpu::backward_solve(dev, cfg); });
        check(r1 == g1 && r1.find("steps") != std::string::npos, "invalid_argument, same message: \"" + g1 + "\"");
        cfg.steps = 2;
        cfg.paths = std::int64_t{1} << 40;
        const std::string r2 = what_of<std::invalid_argument>([&] { backward_solve(spec, cfg); });
        const std::string g2 = what_of<std::invalid_argument>([&] { qrmc_gpu::backward_solve(dev, cfg); });
        check(r2 == g2 && r2.find("stream-id") != std::string::npos, "invalid_argument, same message: \"" + g2 + "\"");
    }
    {
        // blow-up (test_sde.cpp:143-158): drift 1e30 per unit time, state bound 1e15
        ProblemSpec spec;
        spec.dim = 1;
        spec.brownian_dim = 1;
        spec.terminal = [](std::span<const double>) { return 1.0; };
        spec.driver = [](double, std::span<const double>, double) { return 0.0; };
        spec.drift = [](double, std::span<const double>, std::span<double> out) { out[0] = 1e30; };
        spec.growth_g = 1.0;
        qrmc_problem_t dev{};
        dev.dim = 1;
        dev.brownian_dim = 1;
        dev.horizon = 1.0;
        dev.terminal_kind = QRMC_TERMINAL_CONST;
        dev.terminal_params[0] = 1.0;
        dev.driver_kind = QRMC_DRIVER_ZERO;
        dev.drift_kind = QRMC_DRIFT_CONST;
        dev.drift_params[0] = 1e30;
        dev.growth_g = 1.0;
        dev.moment_ratio = 1.0;
        dev.state_bound = 1e15;
        const auto cfg = RunConfig{.steps = 3, .paths = 50, .seed = 1, .gamma = MultiIndexSet::full({3}),
                                   .measure = SamplingMeasure(2.0, 1)};
        int rs = -1, gs = -2;
        const std::string r = what_of<SimulationError>([&] { backward_solve(spec, cfg); }, &rs);
        const std::string g = what_of<SimulationError>([&] { qrmc_gpu::backward_solve(dev, cfg); }, &gs);
        check(r.rfind("WRONG", 0) != 0 && r != "NO EXCEPTION" && g.rfind("WRONG", 0) != 0 && g != "NO EXCEPTION" &&
                  rs == gs,
              "SimulationError from both, step " + std::to_string(rs) + " vs " + std::to_string(gs));
        // non-finite responses (test_solver.cpp:284-288)
        spec.drift = nullptr;
        spec.terminal = [](std::span<const double> x) { return 1.0 / (x[0] - x[0]); };
        dev.drift_kind = QRMC_DRIFT_ZERO;
        dev.terminal_kind = QRMC_TERMINAL_NAN;
        const auto cfg2 = RunConfig{.steps = 2, .paths = 50, .seed = 1, .gamma = MultiIndexSet::full({3}),
                                    .measure = SamplingMeasure(2.0, 1)};
        const std::string r3 = what_of<NumericError>([&] { backward_solve(spec, cfg2); });
        const std::string g3 = what_of<NumericError>([&] { qrmc_gpu::backward_solve(dev, cfg2); });
        check(r3.rfind("WRONG", 0) != 0 && r3 != "NO EXCEPTION" && g3.rfind("WRONG", 0) != 0 && g3 != "NO EXCEPTION",
              "NumericError from both");
    }
    std::printf(failures ? "DROPIN FAILED (%d)\n" : "DROPIN OK\n", failures);
    return failures ? 1 : 0;
}

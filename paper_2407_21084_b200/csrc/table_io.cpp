// table_io.cpp -- the solver's coefficient artifact.
//
// qrmc_gpu_table_json writes the reference's `qrmc.coefficients.v1` document for a
// table solved on the device: the same keys in the same order and the same number
// formatting as table_to_json (proj/src/table_io.cpp:45-73), so CLI and Python
// callers that switch to the GPU solver keep byte-identical artifacts (the
// reference's determinism check compares artifact bytes, acceptance_main.cpp:369-395).
// Serialisation uses nlohmann::ordered_json, the JSON library the reference itself
// builds against (header-only; located by build.py).
#include <json.hpp>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "qrmc_gpu.h"

namespace {

using ordered_json = nlohmann::ordered_json;

const char* kind_name(int kind) {  // to_string(IndexSetKind) (multi_index.cpp:68-75)
    switch (kind) {
        case QRMC_GAMMA_FULL: return "full";
        case QRMC_GAMMA_TOTAL: return "total";
        case QRMC_GAMMA_HYPERBOLIC: return "hyperbolic";
        default: return nullptr;
    }
}

void put_err(char* err, size_t len, const std::string& m) {
    if (!err || !len) return;
    std::strncpy(err, m.c_str(), len - 1);
    err[len - 1] = 0;
}

}  // namespace

extern "C" int64_t qrmc_gpu_table_json(const qrmc_config_t* config, int32_t dim, double horizon,
                                       const double* coeffs, char* out, size_t out_len, char* err,
                                       size_t err_len) {
    try {
        if (!config || !coeffs || dim < 1) {
            put_err(err, err_len, "table_json: null argument or dim < 1");
            return -QRMC_EINVAL;
        }
        const char* kind = kind_name(config->gamma_kind);
        if (!kind || !config->degrees || config->n_degrees < 1) {
            put_err(err, err_len, "table_json: bad index set descriptor");
            return -QRMC_EINVAL;
        }
        // MultiIndexSet::degrees(): (K_1..K_d) for full (a single degree is
        // broadcast, as RunConfig's full set is built), {DEG} otherwise
        std::vector<int> degrees;
        if (config->gamma_kind == QRMC_GAMMA_FULL)
            for (int l = 0; l < dim; ++l) degrees.push_back(config->degrees[config->n_degrees == 1 ? 0 : l]);
        else
            degrees.push_back(config->degrees[0]);
        // SamplingMeasure::center(): the origin when none is given (student.cpp:26-27)
        std::vector<double> center(static_cast<size_t>(dim), 0.0);
        if (config->center)
            for (int l = 0; l < dim; ++l) center[static_cast<size_t>(l)] = config->center[l];

        const int64_t K = qrmc_gpu_gamma_size(config->gamma_kind, dim, config->degrees, config->n_degrees);
        if (K < 0) {
            put_err(err, err_len, "table_json: invalid index set");
            return -QRMC_EINVAL;
        }
        std::vector<int32_t> rows(static_cast<size_t>(K) * dim);
        if (qrmc_gpu_gamma_indices(config->gamma_kind, dim, config->degrees, config->n_degrees, rows.data(),
                                   rows.size(), err, err_len) != QRMC_OK)
            return -QRMC_EINVAL;

        ordered_json doc;
        doc["schema"] = "qrmc.coefficients.v1";
        doc["config"] = ordered_json{{"steps", config->steps},
                                     {"paths", config->paths},
                                     {"damping", config->damping},
                                     {"seed", config->seed},
                                     {"horizon", horizon},
                                     {"measure", ordered_json{{"mu", config->mu}, {"dim", dim}, {"center", center}}},
                                     {"gamma", ordered_json{{"kind", kind}, {"dim", dim}, {"degrees", degrees}}}};
        doc["basis_size"] = static_cast<size_t>(K);
        ordered_json steps = ordered_json::array();
        for (int i = 0; i < config->steps; ++i) {
            ordered_json entries = ordered_json::array();
            const double* c = coeffs + static_cast<size_t>(i) * static_cast<size_t>(K);
            for (int64_t k = 0; k < K; ++k) {
                const int32_t* r = rows.data() + k * dim;
                entries.push_back(ordered_json::array({std::vector<int>(r, r + dim), c[k]}));
            }
            steps.push_back(ordered_json{{"step", i}, {"entries", std::move(entries)}});
        }
        doc["coefficients"] = std::move(steps);
        const std::string s = doc.dump();
        if (out && out_len > s.size()) std::memcpy(out, s.c_str(), s.size() + 1);
        return static_cast<int64_t>(s.size() + 1);
    } catch (const std::exception& e) {
        put_err(err, err_len, std::string("table_json: ") + e.what());
        return -QRMC_EINVAL;
    }
}

// host.cpp -- host side of the B200 backward solver behind include/qrmc_gpu.h.
//
// Owns what the reference does on the host around its hot loop:
//   * validation with the reference's rules and messages
//     (ProblemSpec::validate sde.cpp:10-25, RunConfig::validate solver.cpp:23-35,
//      SamplingMeasure ctor student.cpp:21-44)
//   * multi-index set enumeration, bit-exact in order with
//     proj/src/multi_index.cpp:96-173 (our own enumeration code)
//   * the trie node program and packed coefficient layout the series kernel reads
//   * the backward loop i = N-1..0 (solver.cpp:143-219) as a sequence of
//     kernel launches captured once into a CUDA graph, with the per-step
//     exchange of lane partials over NCCL when the solve spans several GPUs
//   * mapping device error flags back to the reference's exception taxonomy
// No computation of the solve happens here: there is no CPU fallback.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "qrmc_gpu.h"

using namespace qrmc_dev;

namespace {

constexpr uint64_t kMaxIndices = 8'000'000;  // MultiIndexSet::kDefaultMaxIndices (multi_index.hpp:27)

struct Failure {
    qrmc_status status;
    std::string msg;
    int step = -1;
};

[[noreturn]] void fail(qrmc_status st, const std::string& msg) { throw Failure{st, msg}; }

std::string fmt(const char* f, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, f);
    std::vsnprintf(buf, sizeof buf, f, ap);
    va_end(ap);
    return buf;
}

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(QRMC_ECUDA, fmt("%s: %s", what, cudaGetErrorString(e)));
}

void set_err(char* err, size_t len, const std::string& m) {
    if (!err || !len) return;
    std::strncpy(err, m.c_str(), len - 1);
    err[len - 1] = 0;
}

template <class Fn>
qrmc_status guarded(char* err, size_t err_len, Fn&& fn, qrmc_stats_t* stats = nullptr) {
    try {
        fn();
        return QRMC_OK;
    } catch (const Failure& f) {
        set_err(err, err_len, f.msg);
        if (stats) stats->error_step = f.step;
        return f.status;
    } catch (const std::bad_alloc&) {
        set_err(err, err_len, "host allocation failed");
        return QRMC_ECAPACITY;
    } catch (const std::exception& e) {
        set_err(err, err_len, e.what());
        return QRMC_EINVAL;
    }
}

// ------------------------------------------------------------------ Gamma
struct Gamma {
    int dim = 0;
    int kind = 0;
    std::vector<int32_t> rows;  // size x dim, lexicographic
    std::vector<int> kmax;
    int64_t size() const { return dim ? static_cast<int64_t>(rows.size() / dim) : 0; }
};

uint64_t binom_capped(uint64_t n, uint64_t k) {
    // binomial(n, k), saturating above kMaxIndices (multi_index.cpp:17-27 semantics for the cap test)
    if (k > n) return 0;
    k = std::min(k, n - k);
    long double r = 1;
    for (uint64_t i = 1; i <= k; ++i) {
        r = r * static_cast<long double>(n - k + i) / static_cast<long double>(i);
        if (r > 1e30L) return UINT64_MAX;
    }
    return static_cast<uint64_t>(r + 0.5L);
}

Gamma build_gamma(int kind, int dim, const int32_t* degrees, int n_degrees) {
    if (dim < 1) fail(QRMC_EINVAL, "multi-index set: dim must be >= 1");
    if (!degrees || n_degrees < 1) fail(QRMC_EINVAL, "multi-index set: degrees missing");
    Gamma g;
    g.dim = dim;
    g.kind = kind;
    std::vector<int> k(static_cast<size_t>(dim), 0);
    auto emit = [&] {
        if (g.rows.size() / dim >= kMaxIndices) fail(QRMC_ECAPACITY, "index set exceeds index limit");
        g.rows.insert(g.rows.end(), k.begin(), k.end());
    };
    if (kind == QRMC_GAMMA_FULL) {
        if (n_degrees != 1 && n_degrees != dim) fail(QRMC_EINVAL, "full set: need dim degrees");
        std::vector<int> K(static_cast<size_t>(dim));
        uint64_t n = 1;
        for (int l = 0; l < dim; ++l) {
            K[l] = n_degrees == 1 ? degrees[0] : degrees[l];
            if (K[l] < 0) fail(QRMC_EINVAL, "full set: degrees must be >= 0");
            n *= static_cast<uint64_t>(K[l]) + 1;
            if (n > kMaxIndices) fail(QRMC_ECAPACITY, "full set exceeds index limit");
        }
        g.rows.reserve(n * dim);
        // odometer, rightmost coordinate fastest
        for (;;) {
            emit();
            int l = dim - 1;
            while (l >= 0 && k[l] == K[l]) k[l--] = 0;
            if (l < 0) break;
            ++k[l];
        }
    } else if (kind == QRMC_GAMMA_TOTAL) {
        const int deg = degrees[0];
        if (deg < 0) fail(QRMC_EINVAL, "total set: degree must be >= 0");
        if (binom_capped(static_cast<uint64_t>(deg) + dim, dim) > kMaxIndices)
            fail(QRMC_ECAPACITY, "total-degree set exceeds index limit");
        // iterative depth-first walk: increments at the deepest level that still has budget
        std::vector<int> used(static_cast<size_t>(dim) + 1, 0);  // used[l] = sum k[0..l-1]
        for (;;) {
            emit();
            int l = dim - 1;
            for (; l >= 0; --l) {
                if (used[l] + k[l] + 1 <= deg) break;
                k[l] = 0;
            }
            if (l < 0) break;
            ++k[l];
            for (int t = l + 1; t <= dim - 1; ++t) used[t] = used[t - 1] + k[t - 1];
        }
    } else if (kind == QRMC_GAMMA_HYPERBOLIC) {
        const int deg = degrees[0];
        if (deg < 1) fail(QRMC_EINVAL, "hyperbolic set: degree must be >= 1 (prod max(k_l,1) >= 1 always)");
        std::vector<long long> pre(static_cast<size_t>(dim) + 1, 1);  // pre[l] = prod max(k,1) over 0..l-1
        for (;;) {
            emit();
            int l = dim - 1;
            for (; l >= 0; --l) {
                if (pre[l] * std::max(k[l] + 1, 1) <= deg) break;
                k[l] = 0;
            }
            if (l < 0) break;
            ++k[l];
            for (int t = l + 1; t <= dim; ++t) pre[t] = pre[t - 1] * std::max(k[t - 1], 1);
        }
    } else {
        fail(QRMC_EINVAL, "unknown index set kind");
    }
    g.kmax.assign(static_cast<size_t>(dim), 0);
    for (size_t i = 0; i < g.rows.size(); ++i) {
        const int l = static_cast<int>(i % dim);
        g.kmax[l] = std::max(g.kmax[l], g.rows[i]);
    }
    return g;
}

// Trie node program + packed layout (see series_eval in qrmc_device.cuh).
struct Program {
    std::vector<int32_t> pack_pos;   // k -> position in the packed row
    std::vector<double> pack_scale;  // sqrt2^{nnz(k)}
    int64_t kp = 0;                  // packed row length (even)
    std::vector<int4> tiles;         // shared-memory tiles (series_block.cuh)
    std::vector<uint32_t> tile_prog; // group program, per-tile 16-byte aligned segments
};

constexpr int kHostTileA = kSeriesTileA;
constexpr int kHostTileP = 1024;  // == kTileP
constexpr uint32_t kFirstGroupCode = 15;

// Group program of series_block.cuh: one group per upper prefix (k_0..k_{D-3}),
// holding the leaf-run lengths of its siblings k_{D-2} = 0..n-1, cut into
// shared-memory tiles. Verifies downward closure on the way (lexicographic
// order of a downward-closed set advances exactly one level by one and resets
// the deeper ones).
Program build_program(const Gamma& g) {
    Program p;
    const int d = g.dim;
    const int64_t K = g.size();
    p.pack_pos.resize(static_cast<size_t>(K));
    p.pack_scale.resize(static_cast<size_t>(K));
    auto at = [&](int64_t i, int l) { return g.rows[static_cast<size_t>(i * d + l)]; };

    // 1. leaf runs and their packed positions
    struct Run { int64_t first; int64_t R; };
    std::vector<Run> runs;
    int64_t pos = 0;
    for (int64_t i = 0; i < K;) {
        int64_t j = i;
        auto same = [&](int64_t r) {
            for (int l = 0; l < d - 1; ++l)
                if (at(r, l) != at(i, l)) return false;
            return true;
        };
        while (j < K && same(j)) {
            if (at(j, d - 1) != j - i) fail(QRMC_ELOGIC, "index set is not downward closed (leaf run)");
            ++j;
        }
        runs.push_back({i, j - i});
        for (int64_t b = 0; b < j - i; ++b) {
            int nnz = 0;
            for (int l = 0; l < d; ++l) nnz += at(i + b, l) != 0;
            double s = std::ldexp(1.0, nnz / 2);
            if (nnz & 1) s *= 1.4142135623730951;
            p.pack_pos[static_cast<size_t>(i + b)] = static_cast<int32_t>(pos + b);
            p.pack_scale[static_cast<size_t>(i + b)] = s;
        }
        pos += (j - i + 1) & ~int64_t{1};
        i = j;
    }
    p.kp = std::max<int64_t>(pos, 2);

    // 2. groups of sibling runs under one upper prefix
    struct Group { size_t r0, n; uint32_t L; };
    std::vector<Group> groups;
    const int nu = std::max(d - 2, 0);  // upper levels 0..d-3
    for (size_t r = 0; r < runs.size();) {
        size_t e = r;
        auto same_upper = [&](size_t q) {
            for (int l = 0; l < nu; ++l)
                if (at(runs[q].first, l) != at(runs[r].first, l)) return false;
            return true;
        };
        while (e < runs.size() && same_upper(e)) {
            if (d >= 2 && at(runs[e].first, d - 2) != static_cast<int32_t>(e - r))
                fail(QRMC_ELOGIC, "index set is not downward closed (siblings)");
            ++e;
        }
        uint32_t L = kFirstGroupCode;
        if (!groups.empty()) {
            const int64_t a = runs[groups.back().r0].first, b = runs[r].first;
            int l = 0;
            while (l < nu && at(a, l) == at(b, l)) ++l;
            if (l >= nu || at(b, l) != at(a, l) + 1) fail(QRMC_ELOGIC, "index set is not downward closed (groups)");
            for (int t = l + 1; t < nu; ++t)
                if (at(b, t) != 0) fail(QRMC_ELOGIC, "index set is not downward closed (reset)");
            L = static_cast<uint32_t>(l);
        }
        if (e - r >= (1u << 14)) fail(QRMC_ENOTIMPL, "too many sibling runs in one group");
        groups.push_back({r, e - r, L});
        r = e;
    }

    // 3. tiles (series_block.cuh): per group chunk a header word, then one word
    // per segment of consecutive equal-length runs; runs never split, groups
    // and segments continue across tiles
    constexpr int kTileW = kSeriesTileW;
    int4 cur = make_int4(0, 0, 0, 0);
    int64_t alpha_pos = 0;
    auto close = [&] {
        if (cur.y == 0) return;
        p.tiles.push_back(cur);
        while (p.tile_prog.size() % 4) p.tile_prog.push_back(0);
    };
    auto open = [&] { cur = make_int4(static_cast<int>(p.tile_prog.size()), 0, static_cast<int>(alpha_pos), 0); };
    open();
    for (const Group& gr : groups) {
        // hyperbolic-profile group (R_s = floor(B / max(s,1)) + 1, s = 0..B) small
        // enough for the static code of series_block.cuh: header + {pair offset, B}
        {
            const int B = static_cast<int>(gr.n) - 1;
            // mirrors hyp_supported (series_block.cuh)
            bool hyp = d >= 2 && B >= 1 && B <= kHypMaxB && k1_lt(d) >= 2 && k1_s2(d) >= 2;
            int64_t total = 0;
            for (size_t q = 0; hyp && q < gr.n; ++q) {
                hyp = runs[gr.r0 + q].R == B / static_cast<int64_t>(std::max<size_t>(q, 1)) + 1;
                total += (runs[gr.r0 + q].R + 1) & ~int64_t{1};
            }
            if (hyp) {
                if (cur.w + total > kHostTileA || cur.y + 2 > kTileW) {
                    close();
                    open();
                }
                p.tile_prog.push_back(gr.L << 12 | (1u << 29));
                p.tile_prog.push_back(static_cast<uint32_t>(cur.w / 2) | (static_cast<uint32_t>(B) << 16));
                cur.y += 2;
                cur.w += static_cast<int>(total);
                alpha_pos += total;
                continue;
            }
        }
        size_t s = 0;
        while (s < gr.n) {
            const int64_t R0 = runs[gr.r0 + s].R;
            const int64_t pad0 = (R0 + 1) & ~int64_t{1};
            if (pad0 > kHostTileA || R0 >= 4096)
                fail(QRMC_ENOTIMPL, fmt("leaf run of %lld coefficients exceeds a shared-memory tile", (long long)R0));
            if (cur.w + pad0 > kHostTileA || cur.y + 2 > kTileW) {
                close();
                open();
            }
            const size_t hdr_at = p.tile_prog.size();
            const size_t s_first = s;
            p.tile_prog.push_back(0);
            cur.y += 1;
            uint32_t n_seg = 0;
            // segments while the tile has room
            while (s < gr.n && cur.y + 1 <= kTileW && n_seg < 0xFFF) {
                const int64_t R = runs[gr.r0 + s].R;
                const int64_t pad = (R + 1) & ~int64_t{1};
                if (pad > kHostTileA || R >= 4096)
                    fail(QRMC_ENOTIMPL, fmt("leaf run of %lld coefficients exceeds a shared-memory tile", (long long)R));
                if (cur.w + pad > kHostTileA) break;
                int64_t cnt = 0;
                const int first_pair = cur.w / 2;
                while (s < gr.n && runs[gr.r0 + s].R == R && cur.w + pad <= kHostTileA && cnt < 1023) {
                    cur.w += static_cast<int>(pad);
                    alpha_pos += pad;
                    ++cnt;
                    ++s;
                }
                p.tile_prog.push_back(static_cast<uint32_t>(first_pair) | (static_cast<uint32_t>(R) << 10) |
                                      (static_cast<uint32_t>(cnt) << 22));
                cur.y += 1;
                ++n_seg;
            }
            const bool cont = s_first > 0;
            p.tile_prog[hdr_at] = n_seg | ((cont ? 0u : gr.L) << 12) | (static_cast<uint32_t>(s_first) << 16) |
                                  (cont ? (1u << 28) : 0u);
        }
    }
    close();
    return p;
}

// ------------------------------------------------------------------ problem / config
ProblemDev to_device_problem(const qrmc_problem_t& p) {
    // ProblemSpec::validate (sde.cpp:10-25)
    if (p.dim < 1 || p.brownian_dim < 1) fail(QRMC_EINVAL, "ProblemSpec: dimensions must be >= 1");
    if (!(p.horizon > 0.0)) fail(QRMC_EINVAL, "ProblemSpec: horizon must be positive");
    const double consts[] = {p.growth_g, p.growth_exp_g, p.growth_f, p.growth_exp_f, p.lipschitz_f};
    for (double c : consts)
        if (!(c >= 0.0) || !std::isfinite(c))
            fail(QRMC_EINVAL, "ProblemSpec: growth/Lipschitz constants must be finite and >= 0");
    if (!(p.moment_ratio >= 1.0)) fail(QRMC_EINVAL, "ProblemSpec: moment_ratio must be >= 1");
    if (p.terminal_kind < QRMC_TERMINAL_SIN_SUM || p.terminal_kind > QRMC_TERMINAL_NAN)
        fail(QRMC_ENOTIMPL, "terminal kind has no device functor");
    if (p.driver_kind < QRMC_DRIVER_ZERO || p.driver_kind > QRMC_DRIVER_SIN_BENCH)
        fail(QRMC_ENOTIMPL, "driver kind has no device functor");
    if (p.drift_kind < QRMC_DRIFT_ZERO || p.drift_kind > QRMC_DRIFT_AFFINE)
        fail(QRMC_ENOTIMPL, "drift kind has no device functor");
    if (p.diffusion_kind < QRMC_DIFFUSION_IDENTITY || p.diffusion_kind > QRMC_DIFFUSION_DIAG)
        fail(QRMC_ENOTIMPL, "diffusion kind has no device functor");
    if (p.dim > kMaxDim) fail(QRMC_ENOTIMPL, fmt("dimension %d exceeds the device limit %d", p.dim, kMaxDim));
    if (p.brownian_dim != p.dim)
        fail(QRMC_ENOTIMPL, "device diffusions need brownian_dim == dim");
    ProblemDev d{};
    d.dim = p.dim;
    d.bdim = p.brownian_dim;
    d.horizon = p.horizon;
    d.terminal_kind = p.terminal_kind;
    d.driver_kind = p.driver_kind;
    d.drift_kind = p.drift_kind;
    d.diffusion_kind = p.diffusion_kind;
    d.tp0 = p.terminal_params[0];
    d.tp1 = p.terminal_params[1];
    d.dp0 = p.driver_params[0];
    d.dp1 = p.driver_params[1];
    d.drift_c = p.drift_params[0];
    d.sigma = p.diffusion_params[0];
    for (int l = 0; l < std::min(p.dim, kMaxDim); ++l) {
        d.drift_a[l] = p.drift_vec[l];
        d.drift_b[l] = p.drift_vec[8 + l];
        d.sig[l] = p.diffusion_vec[l];
    }
    // lstar_bound's x-independent factor, evaluated exactly as sde.cpp:28-29
    d.lstar_base = p.moment_ratio * (p.growth_g + p.horizon * p.growth_f) *
                   std::exp(p.moment_ratio * p.lipschitz_f * p.horizon);
    d.eta = std::max(p.growth_exp_g, p.growth_exp_f);
    d.state_bound = p.state_bound;
    return d;
}

MeasureDev to_device_measure(const qrmc_config_t& c, int dim) {
    // SamplingMeasure ctor (student.cpp:21-44)
    if (!(c.mu > 0.0) || !std::isfinite(c.mu)) fail(QRMC_EINVAL, "SamplingMeasure: mu must be positive and finite");
    if (dim < 1) fail(QRMC_EINVAL, "SamplingMeasure: dim must be >= 1");
    if (dim > kMaxDim) fail(QRMC_ENOTIMPL, "dimension exceeds the device limit");
    MeasureDev m{};
    if (c.mu == 1.0)
        m.form = 1;
    else if (c.mu == 2.0)
        m.form = 2;
    else
        m.form = 3;  // Student's t with mu degrees of freedom (include/qrmc_student_t.h)
    m.mu = c.mu;
    m.sqrt_mu = std::sqrt(c.mu);
    for (int l = 0; l < dim; ++l) {
        m.center[l] = c.center ? c.center[l] : 0.0;
        if (!std::isfinite(m.center[l])) fail(QRMC_EINVAL, "SamplingMeasure: center must be finite");
    }
    return m;
}

void validate_config(const qrmc_config_t& c) {
    // RunConfig::validate (solver.cpp:23-35)
    if (c.steps < 1) fail(QRMC_EINVAL, "RunConfig: steps must be >= 1");
    if (c.paths < 1) fail(QRMC_EINVAL, "RunConfig: paths must be >= 1");
    if (!(c.damping >= 0.0) || !std::isfinite(c.damping)) fail(QRMC_EINVAL, "RunConfig: damping must be finite and >= 0");
    if (c.workers < 0) fail(QRMC_EINVAL, "RunConfig: workers must be >= 0");
    if (c.paths >= (int64_t{1} << kStepShift)) fail(QRMC_EINVAL, "RunConfig: paths exceeds the stream-id layout");
    if (c.steps >= (1 << 22)) fail(QRMC_EINVAL, "RunConfig: steps exceeds the stream-id layout");
    if (c.memory_mode != QRMC_MEMORY_STORE_CLOUD && c.memory_mode != QRMC_MEMORY_RECOMPUTE)
        fail(QRMC_EINVAL, "unknown memory mode");
}

// ------------------------------------------------------------------ device buffers
template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    void alloc(size_t count) {
        release();
        n = count;
        if (count) cuda_check(cudaMalloc(&p, count * sizeof(T)), "cudaMalloc");
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void upload(const T* h, size_t count, cudaStream_t st) {
        cuda_check(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, st), "H2D");
    }
    ~DevBuf() { release(); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

// K2 work items: every leaf run cut into chunks of <= kProjRun terms, each with
// the per-point table offsets of its prefix (k_0..k_{d-2}) and first leaf value
// (cosine_basis.cpp:58-64 table layout); sorted by length so warps stay in step.
struct ProjectItems {
    std::vector<int32_t> k, len, leaf, pre;  // pre: [d-1][n]
    int n = 0;
};

ProjectItems build_project_items(const Gamma& g, const int* offset) {
    const int d = g.dim;
    const int64_t K = g.size();
    struct It { int32_t k, len, leaf; std::vector<int32_t> pre; };
    std::vector<It> items;
    for (int64_t i = 0; i < K;) {
        int64_t j = i;
        auto same = [&](int64_t r) {
            for (int l = 0; l < d - 1; ++l)
                if (g.rows[static_cast<size_t>(r * d + l)] != g.rows[static_cast<size_t>(i * d + l)]) return false;
            return true;
        };
        while (j < K && same(j)) ++j;
        for (int64_t b0 = i; b0 < j; b0 += kProjRun) {
            It it;
            it.k = static_cast<int32_t>(b0);
            it.len = static_cast<int32_t>(std::min<int64_t>(kProjRun, j - b0));
            it.leaf = offset[d - 1] + g.rows[static_cast<size_t>(b0 * d + d - 1)];
            for (int l = 0; l < d - 1; ++l) it.pre.push_back(offset[l] + g.rows[static_cast<size_t>(b0 * d + l)]);
            items.push_back(std::move(it));
        }
        i = j;
    }
    std::stable_sort(items.begin(), items.end(), [](const It& a, const It& b) { return a.len > b.len; });
    // pad every length class to whole warps (32 items) with empty items, so the
    // kernel's per-warp dispatch on the item length is uniform
    {
        std::vector<It> padded;
        for (size_t i = 0; i < items.size();) {
            size_t j = i;
            while (j < items.size() && items[j].len == items[i].len) padded.push_back(items[j++]);
            while (padded.size() % 32) padded.push_back(It{0, 0, 0, std::vector<int32_t>(static_cast<size_t>(std::max(d - 1, 0)), 0)});
            i = j;
        }
        items.swap(padded);
    }
    ProjectItems out;
    out.n = static_cast<int>(items.size());
    const int np = std::max(d - 1, 1);
    out.pre.assign(static_cast<size_t>(np) * out.n, 0);
    for (int t = 0; t < out.n; ++t) {
        out.k.push_back(items[t].k);
        out.len.push_back(items[t].len);
        out.leaf.push_back(items[t].leaf);
        for (int l = 0; l < d - 1; ++l) out.pre[static_cast<size_t>(l) * out.n + t] = items[t].pre[static_cast<size_t>(l)];
    }
    return out;
}

// Fragment-stream layout of the tensor-core K1 (responses_mma.cu). Groups are
// the upper prefixes u = (k_0..k_{d-3}); each holds a set of (s, b) =
// (k_{d-2}, k_{d-1}) pairs. Pairs are ordered by how many groups contain them
// (then lexicographically); for a chain of sets (full, total-degree and
// hyperbolic index sets) every group is then a prefix of that order, which is
// checked here -- ok = false sends the plan to the series-program K1.
#ifndef QRMC_MMA_BANK_ORDER
#define QRMC_MMA_BANK_ORDER 1  // bank-aware term/group order for the ring kernel too (d=6: K1 -5%)
#endif
struct MmaLayoutOpts {
    int warps = kMmaWarps;      // GEMM warps the units are balanced over
    bool euler_ahead = true;    // the first warps also run the Euler steps (responses_mma.cu)
    bool ring = true;           // steps aligned to W slots and warp segments to the cp.async ring
    int bank_order = QRMC_MMA_BANK_ORDER;
    // the first tail_terms (a multiple of 8) terms of every group go to a transposed GEMM
    // over the groups (units with nb = 8 + tail_terms / 8, responses_ws.cu ws_unit_t): no
    // per-unit epilogue for the hyperbolic tail's many small groups
    int tail_terms = 0;
    int bundle = kMmaBundle;    // max column blocks per unit
};

struct MmaLayout {
    bool ok = false;
    // warp-specialised K1 (responses_ws.cu): swizzled [entry][32 paths] table offsets,
    // relative to the lane's row, per row half (rows 0-3 / 4-7)
    std::vector<uint4> ws_terms;    // [n_terms][2] byte offsets {sA, sB, bA, bB}
    std::vector<uint32_t> ws_gk;    // [2][n_groups][d-2] {A | B << 16}
    std::vector<uint32_t> terms;    // [n_terms] table offsets (s | b << 16)
    std::vector<uint16_t> gk;       // [n_groups][d-2] table offsets of the prefix
    std::vector<int4> units;        // {cb0, nb, c0, c1}, warp-contiguous
    std::vector<int4> warp_info;    // [kMmaWarps] {unit_begin, unit_end, frag_offset, frags}
    std::vector<int32_t> pos;       // k -> position in the per-series stream
    int64_t row_len = 0;
    int64_t frags = 0;              // B fragments per series (useful MACs = K of 256 * frags)
    // K2 on the tensor cores
    int proj_parts = 0;
    std::vector<int4> proj_rects;   // [parts][kProjWarps] {gb0, tb0, ngb | ntb << 8, valid tiles}
    std::vector<int32_t> proj_out;  // [parts][kProjWarps][kProjTiles][32 lanes][2] -> k, or -1
};

// Swizzled table slot of (entry e, path p) in the warp-specialised K1's
// [entry][32 paths] tables: p ^ (4 (e & 3)), so the 4 distinct entries a
// half-warp reads (one per lane column) hit 4 distinct 32-byte bank groups
// whenever they differ mod 4 (the bank-aware term/group order arranges that).
// For the lane's row block r the value sits at e*32 + 8 (r ^ h) + (row ^ 4 (x & 1)),
// x = e & 3, h = x >> 1: two base offsets, A (r = 0, 2) and B (r = 1, 3), each
// relative to the lane's own row; they depend on the row half only.
inline uint32_t ws_off(int e, int half, bool second) {
    const int x = e & 3, h = x >> 1;
    const int rowfix = (x & 1) ? (half ? -4 : 4) : 0;
    return static_cast<uint32_t>(e * 32 + 8 * (second ? 1 - h : h) + rowfix);
}

inline int ws_gk_record(int d) { return (2 * (d - 2) + 3) / 4 * 4; }
// terms of every group the warp-specialised K1 runs as a transposed GEMM (0, 8 or 16;
// QRMC_WS_TAIL overrides)
#ifndef QRMC_WS_TAIL_DEFAULT
#define QRMC_WS_TAIL_DEFAULT 0
#endif
inline int ws_tail_terms() {
    const char* e = std::getenv("QRMC_WS_TAIL");
    const int v = e ? std::atoi(e) : QRMC_WS_TAIL_DEFAULT;
    return v == 16 ? 16 : v == 8 ? 8 : 0;
}
inline size_t ws_gk_index(int d, int n_groups, int half, int g, int l) {
    return (static_cast<size_t>(half) * (n_groups / 2) + g / 2) * ws_gk_record(d) + (g % 2) * (d - 2) + l;
}

MmaLayout build_mma_layout(const Gamma& g, const int* offset, const MmaLayoutOpts& opt = MmaLayoutOpts{}) {
    MmaLayout L;
    const int d = g.dim;
    const int64_t K = g.size();
    if (d < 3 || K == 0) return L;
    const int nu = d - 2;
    auto at = [&](int64_t r, int l) { return g.rows[static_cast<size_t>(r * d + l)]; };
    // groups: maximal runs of rows with equal prefix (rows are lexicographic)
    struct Grp { int64_t r0, n; };
    std::vector<Grp> groups;
    for (int64_t r = 0; r < K;) {
        int64_t e = r + 1;
        auto same = [&](int64_t q) {
            for (int l = 0; l < nu; ++l)
                if (at(q, l) != at(r, l)) return false;
            return true;
        };
        while (e < K && same(e)) ++e;
        groups.push_back({r, e - r});
        r = e;
    }
    const int S = g.kmax[d - 2] + 1, Bn = g.kmax[d - 1] + 1;
    std::vector<int32_t> cnt(static_cast<size_t>(S) * Bn, 0);
    for (int64_t r = 0; r < K; ++r) ++cnt[static_cast<size_t>(at(r, d - 2)) * Bn + at(r, d - 1)];
    std::vector<int32_t> order;
    for (int32_t pr = 0; pr < S * Bn; ++pr)
        if (cnt[static_cast<size_t>(pr)]) order.push_back(pr);
    std::stable_sort(order.begin(), order.end(),
                     [&](int32_t x, int32_t y) { return cnt[static_cast<size_t>(x)] > cnt[static_cast<size_t>(y)]; });
    // Inside a layer of equal count the order is free: arrange each chunk of four
    // terms so that their table rows of c_s and of c_b are distinct mod 4 -- the
    // kernels read 4 terms x 4 paths per half-warp from [entry][path] tables with a
    // row stride = 4 (mod 16) banks, so that makes both operand loads conflict-free.
    if (opt.bank_order) {
        std::vector<int32_t> out;
        out.reserve(order.size());
        size_t i = 0;
        while (i < order.size()) {
            size_t e = i;
            while (e < order.size() && cnt[static_cast<size_t>(order[e])] == cnt[static_cast<size_t>(order[i])]) ++e;
            std::vector<int32_t> pool(order.begin() + static_cast<std::ptrdiff_t>(i), order.begin() + static_cast<std::ptrdiff_t>(e));
            while (!pool.empty()) {
                // rows already in the current chunk, per residue mod 4 (-1: free); a row
                // equal to one already there is a broadcast, not a bank conflict
                const size_t base = out.size() / 4 * 4;
                int row_s[4] = {-1, -1, -1, -1}, row_b[4] = {-1, -1, -1, -1};
                for (size_t q = base; q < out.size(); ++q) {
                    const int es = offset[d - 2] + out[q] / Bn, eb = offset[d - 1] + out[q] % Bn;
                    row_s[es & 3] = es;
                    row_b[eb & 3] = eb;
                }
                size_t best = 0;
                int best_cost = 99;
                for (size_t q = 0; q < pool.size() && best_cost > 0; ++q) {
                    const int es = offset[d - 2] + pool[q] / Bn, eb = offset[d - 1] + pool[q] % Bn;
                    const int cs = row_s[es & 3] >= 0 && row_s[es & 3] != es;
                    const int cb = row_b[eb & 3] >= 0 && row_b[eb & 3] != eb;
                    if (cs + cb < best_cost) {
                        best_cost = cs + cb;
                        best = q;
                    }
                }
                out.push_back(pool[best]);
                pool.erase(pool.begin() + static_cast<std::ptrdiff_t>(best));
            }
            i = e;
        }
        order.swap(out);
    }
    if (std::getenv("QRMC_DEBUG_LAYOUT")) {
        // 4-term chunks whose s (b) rows differ but share a residue mod 4, weighted by the
        // number of groups that read the chunk (the pair count of its first term)
        double w_all = 0, w_s = 0, w_b = 0;
        for (size_t c = 0; c * 4 < order.size(); ++c) {
            int rs[4] = {-1, -1, -1, -1}, rb[4] = {-1, -1, -1, -1};
            bool cs = false, cb = false;
            for (size_t q = 4 * c; q < std::min(order.size(), 4 * c + 4); ++q) {
                const int es = offset[d - 2] + order[q] / Bn, eb = offset[d - 1] + order[q] % Bn;
                cs |= rs[es & 3] >= 0 && rs[es & 3] != es;
                cb |= rb[eb & 3] >= 0 && rb[eb & 3] != eb;
                rs[es & 3] = es;
                rb[eb & 3] = eb;
            }
            const double w = cnt[static_cast<size_t>(order[4 * c])];
            w_all += w;
            w_s += cs ? w : 0;
            w_b += cb ? w : 0;
        }
        std::fprintf(stderr, "terms %zu: weighted chunks with s conflicts %.3f, b conflicts %.3f\n", order.size(),
                     w_s / w_all, w_b / w_all);
    }
    std::vector<int32_t> rank(static_cast<size_t>(S) * Bn, -1);
    for (size_t t = 0; t < order.size(); ++t) rank[static_cast<size_t>(order[t])] = static_cast<int32_t>(t);
    for (const Grp& gr : groups)
        for (int64_t r = gr.r0; r < gr.r0 + gr.n; ++r)
            if (rank[static_cast<size_t>(at(r, d - 2)) * Bn + at(r, d - 1)] >= gr.n) return L;  // not a prefix
    if (static_cast<int64_t>(offset[d - 1] + Bn) * kMmaTabStride > 0xFFFF) return L;
    auto row_of = [](int entry) { return static_cast<uint32_t>(entry * kMmaTabStride); };
    // K1 reads 4-term chunks, K2 8-term blocks, the transposed tail its first tail_terms terms
    const int n_terms = std::max(static_cast<int>((order.size() + 7) & ~size_t{7}), opt.tail_terms);
    L.terms.assign(static_cast<size_t>(n_terms), row_of(offset[d - 2]) | row_of(offset[d - 1]) << 16);
    for (size_t t = 0; t < order.size(); ++t)
        L.terms[t] = row_of(offset[d - 2] + order[t] / Bn) | row_of(offset[d - 1] + order[t] % Bn) << 16;
    L.ws_terms.assign(static_cast<size_t>(n_terms) * 2, make_uint4(0u, 0u, 0u, 0u));
    for (int t = 0; t < n_terms; ++t) {
        const int pr = t < static_cast<int>(order.size()) ? order[t] : 0;  // padding terms read (0, 0)
        const int es = offset[d - 2] + pr / Bn, eb = offset[d - 1] + pr % Bn;
        for (int half = 0; half < 2; ++half)
            L.ws_terms[static_cast<size_t>(t) * 2 + half] =
                make_uint4(8 * ws_off(es, half, false), 8 * ws_off(es, half, true), 8 * ws_off(eb, half, false),
                           8 * ws_off(eb, half, true));
    }

    // groups by size (descending, stable), 8 per column block
    std::vector<int32_t> gi(groups.size());
    for (size_t i = 0; i < gi.size(); ++i) gi[i] = static_cast<int32_t>(i);
    std::stable_sort(gi.begin(), gi.end(), [&](int32_t x, int32_t y) { return groups[x].n > groups[y].n; });
    // Same freedom for groups of equal size: the K1 epilogue reads the prefix
    // rows of groups n = 2 col + h (col = 0..3) of a column block per half-warp,
    // so arrange each such quad to have distinct rows mod 4 on every level.
    if (opt.bank_order) {
        std::vector<int32_t> out;
        out.reserve(gi.size());
        size_t i = 0;
        while (i < gi.size()) {
            size_t e = i;
            while (e < gi.size() && groups[gi[e]].n == groups[gi[i]].n) ++e;
            std::vector<int32_t> pool(gi.begin() + static_cast<std::ptrdiff_t>(i), gi.begin() + static_cast<std::ptrdiff_t>(e));
            while (!pool.empty()) {
                const size_t pos = out.size(), blk = pos / 8 * 8;
                std::vector<int> used(static_cast<size_t>(nu) * 4, -1);  // [level][residue] -> row
                for (size_t q = blk + pos % 2; q < pos; q += 2)
                    for (int l = 0; l < nu; ++l) {
                        const int e = offset[l] + at(groups[out[q]].r0, l);
                        used[static_cast<size_t>(l) * 4 + (e & 3)] = e;
                    }
                size_t best = 0;
                int best_cost = 1 << 20;
                for (size_t q = 0; q < pool.size() && best_cost > 0; ++q) {
                    int cost = 0;
                    for (int l = 0; l < nu; ++l) {
                        const int e = offset[l] + at(groups[pool[q]].r0, l), u = used[static_cast<size_t>(l) * 4 + (e & 3)];
                        cost += u >= 0 && u != e;
                    }
                    if (cost < best_cost) {
                        best_cost = cost;
                        best = q;
                    }
                }
                out.push_back(pool[best]);
                pool.erase(pool.begin() + static_cast<std::ptrdiff_t>(best));
            }
            i = e;
        }
        gi.swap(out);
    }
    const int n_cb = static_cast<int>((gi.size() + 7) / 8);
    L.gk.assign(static_cast<size_t>(n_cb) * 8 * nu, 0);
    for (int c = 0; c < n_cb * 8; ++c)
        for (int l = 0; l < nu; ++l)
            L.gk[static_cast<size_t>(c) * nu + l] = static_cast<uint16_t>(
                row_of(offset[l] + (c < static_cast<int>(gi.size()) ? at(groups[gi[c]].r0, l) : 0)));
    // [half][group pair][R]: the two groups of a pair (2 col, 2 col + 1) in one
    // 16-byte-aligned record of R = 2 (d-2) rounded up to 4 words (ws_gk_index)
    L.ws_gk.assign(static_cast<size_t>(2) * n_cb * 4 * ws_gk_record(d), 0u);
    for (int half = 0; half < 2; ++half)
        for (int c = 0; c < n_cb * 8; ++c)
            for (int l = 0; l < nu; ++l) {
                const int e = offset[l] + (c < static_cast<int>(gi.size()) ? at(groups[gi[c]].r0, l) : 0);
                L.ws_gk[ws_gk_index(d, n_cb * 8, half, c, l)] = ws_off(e, half, false) | ws_off(e, half, true) << 16;
            }
    std::vector<int32_t> cb_chunks;  // chunks of 4 terms per column block (descending)
    for (int cb = 0; cb < n_cb; ++cb) cb_chunks.push_back(static_cast<int32_t>((groups[gi[8 * cb]].n + 3) / 4));

    // units: column blocks of equal chunk count, <= kMmaBundle per unit, chunk
    // range cut into <= kMmaKSplit pieces; balanced over the warps (longest
    // processing time first) with an issue-slot cost model
    struct Unit { int cb0, nb, c0, c1; double cost; };
    std::vector<Unit> units;
    // issue-slot cost model of a unit: per chunk step cost_step + nb cost_nb, per column
    // block epilogue cost_epi (QRMC_COST_STEP / _NB / _EPI override, tuning only)
    auto env_or = [](const char* n, double v) {
        const char* e = std::getenv(n);
        return e ? std::atof(e) : v;
    };
    // (warp-specialised layout: (12, 10, 64) measured 0.705 s vs 0.708-0.710 for (16, 10, 48)
    // at the bench shape, M = 2e6; the ring kernel keeps (16, 10, 48))
    const double cost_step = env_or("QRMC_COST_STEP", opt.ring ? 16.0 : 12.0), cost_nb = env_or("QRMC_COST_NB", 10.0),
                 cost_epi = env_or("QRMC_COST_EPI", opt.ring ? 48.0 : 64.0);
    auto add_units = [&](int cb, int nb, int lo, int hi) {  // chunk range [lo, hi) of cbs cb..cb+nb-1
        if (hi <= lo) return;
        const int np = (hi - lo + kMmaKSplit - 1) / kMmaKSplit;
        for (int q = 0; q < np; ++q) {
            const int c0 = lo + static_cast<int>(static_cast<int64_t>(hi - lo) * q / np);
            const int c1 = lo + static_cast<int>(static_cast<int64_t>(hi - lo) * (q + 1) / np);
            const double len = c1 - c0;
            units.push_back({cb, nb, c0, c1, len * (cost_step + nb * cost_nb) + nb * cost_epi});
        }
    };
#ifndef QRMC_MMA_STAIR
#define QRMC_MMA_STAIR 1
#endif
    // the tail: column blocks whose groups all have <= tail_terms terms (groups are sorted
    // by size) go to the transposed GEMM over their groups; the rest stay here
    const int tnb = opt.tail_terms / 8;  // term blocks of the transposed GEMM (N = 8 terms each)
    int tail_cb = n_cb;
    if (tnb > 0)
        for (int cb = 0; cb < n_cb; ++cb)
            if (4 * cb_chunks[cb] <= opt.tail_terms) {
                tail_cb = cb;
                break;
            }
    for (int cb = 0; cb < tail_cb;) {
        int e = cb;
        if (QRMC_MMA_STAIR) {
            // staircase bundles: kMmaBundle consecutive column blocks share the chunks
            // all of them have; each block's remainder runs in narrower units
            e = std::min(tail_cb, cb + opt.bundle);
            int lo = 0;
            for (int k = e; k > cb; --k) {  // blocks cb..k-1 share [lo, E_{k-1})
                add_units(cb, k - cb, lo, cb_chunks[k - 1]);
                lo = std::max(lo, cb_chunks[k - 1]);
            }
        } else {
            while (e < tail_cb && e - cb < opt.bundle && cb_chunks[e] == cb_chunks[cb]) ++e;
            add_units(cb, e - cb, 0, cb_chunks[cb]);
        }
        cb = e;
    }
    // transposed units: chunks of 4 groups (2 n_cb of them) x tnb blocks of 8 terms,
    // encoded nb = 8 + tnb; cost: A fragments need d-2 table rows per group
    if (tnb > 0 && tail_cb < n_cb) {
        const int tb = 2 * tail_cb, tc = 2 * n_cb - tb;  // chunks of 4 groups: [tb, 2 n_cb)
        const int np = (tc + kMmaKSplit - 1) / kMmaKSplit;
        for (int q = 0; q < np; ++q) {
            const int c0 = tb + static_cast<int>(static_cast<int64_t>(tc) * q / np);
            const int c1 = tb + static_cast<int>(static_cast<int64_t>(tc) * (q + 1) / np);
            units.push_back({-1, 8 + tnb, c0, c1, (c1 - c0) * (16.0 + tnb * 10.0 + 4.0 * nu) + tnb * 48.0});
        }
    }
    std::vector<int32_t> ui(units.size());
    for (size_t i = 0; i < ui.size(); ++i) ui[i] = static_cast<int32_t>(i);
    std::stable_sort(ui.begin(), ui.end(), [&](int32_t x, int32_t y) { return units[x].cost > units[y].cost; });
    const int n_warps = opt.warps;
    std::vector<std::vector<int32_t>> per_warp(n_warps);
    std::vector<double> load(n_warps, 0.0);
    // the first warps also run the next Euler step and x-only parts during the
    // GEMM phase
#ifndef QRMC_MMA_EULER_COST
#define QRMC_MMA_EULER_COST 800
#endif
    // (responses_mma.cu kAheadThreads: the Euler tasks and the x-only parts)
    if (opt.euler_ahead)
        for (int w = 0; w < std::min(n_warps, (std::max(kMmaPaths * d, 3 * kMmaPaths) + 31) / 32); ++w)
            load[w] = QRMC_MMA_EULER_COST;
    // Warp w issues on SM sub-partition w % 4, whose DMMA pipe its warps share:
    // balance the four sub-partitions first (LPT), then the warps inside each.
#ifndef QRMC_MMA_SMSP_BALANCE
#define QRMC_MMA_SMSP_BALANCE 1
#endif
    constexpr int kSub = QRMC_MMA_SMSP_BALANCE ? 4 : 1;
    std::vector<std::vector<int32_t>> per_sub(kSub);
    {
        std::vector<double> sl(kSub, 0.0);
        for (int w = 0; w < n_warps; ++w) sl[w % kSub] += load[w];
        for (int32_t u : ui) {
            const int b = static_cast<int>(std::min_element(sl.begin(), sl.end()) - sl.begin());
            per_sub[b].push_back(u);
            sl[b] += units[u].cost;
        }
    }
    for (int b = 0; b < kSub; ++b) {
        for (int32_t u : per_sub[b]) {  // still in descending cost order
            int w = b;
            for (int v = b; v < n_warps; v += kSub)
                if (load[v] < load[w]) w = v;
            per_warp[w].push_back(u);
            load[w] += units[u].cost;
        }
    }
    if (std::getenv("QRMC_DEBUG_LAYOUT")) {
        for (int w = 0; w < n_warps; ++w) {
            std::fprintf(stderr, "warp %2d load %8.0f:", w, load[w]);
            for (int32_t u : per_warp[w])
                std::fprintf(stderr, " [cb%d nb%d c%d-%d]", units[u].cb0, units[u].nb, units[u].c0, units[u].c1);
            std::fprintf(stderr, "\n");
        }
    }
    std::vector<int64_t> frag_at(static_cast<size_t>(n_cb) * cb_chunks[0], -1);
    const int cstride = cb_chunks[0];
    std::vector<int64_t> tfrag_at(static_cast<size_t>(2 * n_cb) * std::max(tnb, 1), -1);  // [tchunk][term block]
    int64_t woff = 0;
    for (int w = 0; w < n_warps; ++w) {
        std::sort(per_warp[w].begin(), per_warp[w].end(), [&](int32_t x, int32_t y) {
            return units[x].cb0 != units[y].cb0 ? units[x].cb0 < units[y].cb0 : units[x].c0 < units[y].c0;
        });
        const int ub = static_cast<int>(L.units.size());
        int64_t f = 0;
        for (int32_t u : per_warp[w]) {
            const Unit& un = units[u];
            L.units.push_back(make_int4(un.cb0, un.nb, un.c0, un.c1));
            if (un.nb >= 8) {  // transposed: tnb fragments per chunk of 4 groups
                for (int c = un.c0; c < un.c1; ++c, f += tnb)
                    for (int i = 0; i < tnb; ++i) tfrag_at[static_cast<size_t>(c) * tnb + i] = woff + f + i;
                L.frags += static_cast<int64_t>(tnb) * (un.c1 - un.c0);
                continue;
            }
            // a step takes 1, 2 or 4 fragment slots (3 column blocks use 4), aligned,
            // so no step straddles the ring wrap
            const int stride = opt.ring && un.nb == 3 ? 4 : un.nb;
            L.frags += static_cast<int64_t>(un.nb) * (un.c1 - un.c0);
            if (opt.ring) f = (f + stride - 1) / stride * stride;
            for (int c = un.c0; c < un.c1; ++c, f += stride)
                for (int i = 0; i < un.nb; ++i) frag_at[static_cast<size_t>(un.cb0 + i) * cstride + c] = woff + f + i;
        }
        const int64_t fpad = opt.ring ? (f + kMmaRingFrags - 1) / kMmaRingFrags * kMmaRingFrags : f;
        L.warp_info.push_back(make_int4(ub, static_cast<int>(L.units.size()), static_cast<int>(woff), static_cast<int>(fpad)));
        woff += fpad;
    }
    L.row_len = woff * 32;
    if (L.row_len >= (int64_t{1} << 31)) return MmaLayout{};
    // k -> stream position: column n of block cb, term t in chunk t/4 row t%4
    L.pos.assign(static_cast<size_t>(K), 0);
    for (int c = 0; c < static_cast<int>(gi.size()); ++c) {
        const Grp& gr = groups[gi[c]];
        const int cb = c / 8, n = c % 8;
        for (int64_t r = gr.r0; r < gr.r0 + gr.n; ++r) {
            const int t = rank[static_cast<size_t>(at(r, d - 2)) * Bn + at(r, d - 1)];
            if (cb >= tail_cb) {
                // transposed: B[k = group c % 4][n = term t % 8] of chunk c / 4, block t / 8
                const int64_t f = tfrag_at[static_cast<size_t>(c / 4) * tnb + t / 8];
                if (f < 0) fail(QRMC_ELOGIC, "mma layout: tail term outside the fragment stream");
                L.pos[static_cast<size_t>(r)] = static_cast<int32_t>(f * 32 + (((t % 8) << 2) | (c % 4)));
                continue;
            }
            const int64_t f = frag_at[static_cast<size_t>(cb) * cstride + t / 4];
            if (f < 0) fail(QRMC_ELOGIC, "mma layout: term outside the fragment stream");
            L.pos[static_cast<size_t>(r)] = static_cast<int32_t>(f * 32 + ((n << 2) | (t & 3)));
        }
    }
    // K2 (project_mma.cu): output tiles (group block gb, 8-term block tb) of the
    // staircase G[u][t], t < T_u, cut into full rectangles of ng x nt tiles
    // (ng in {1, 2, 4, 8}, ng * nt <= kProjTiles), one per warp, kProjWarps per
    // CTA part. Group blocks are sorted by T_u, so the staircase is a sequence of
    // strips of equal width (term blocks).
    {
        struct Rect { int gb0, ng, tb0, nt, tiles; };
        std::vector<int> ntb(static_cast<size_t>(n_cb));
        for (int cb = 0; cb < n_cb; ++cb) ntb[cb] = static_cast<int>((groups[gi[8 * cb]].n + 7) / 8);
        std::vector<Rect> rects;
        for (int g = 0; g < n_cb;) {
            int h = 1;
            while (g + h < n_cb && ntb[g + h] == ntb[g]) ++h;
            const int w = ntb[g];
            // rows in power-of-two bands; each band cut into ng x (kProjTiles / ng)
            for (int r0 = 0; r0 < h;) {
                int ng = 1;
                while (ng * 2 <= std::min(16, kProjTiles)) ng *= 2;  // a power of two (kernel shapes)
                while (ng > h - r0) ng /= 2;
                const int nt_max = kProjTiles / ng;
                for (int t0 = 0; t0 < w; t0 += nt_max) {
                    const int nt = std::min(nt_max, w - t0);
                    rects.push_back(Rect{g + r0, ng, t0, nt, ng * nt});
                }
                r0 += ng;
            }
            g += h;
        }
        std::stable_sort(rects.begin(), rects.end(), [](const Rect& x, const Rect& y) { return x.tiles > y.tiles; });
        const int parts = static_cast<int>((rects.size() + kProjWarps - 1) / kProjWarps);
        // LPT over parts, at most kProjWarps rectangles each
        std::vector<std::vector<int>> part_r(static_cast<size_t>(parts));
        std::vector<int> part_load(static_cast<size_t>(parts), 0);
        for (size_t i = 0; i < rects.size(); ++i) {
            int best = -1;
            for (int q = 0; q < parts; ++q)
                if (static_cast<int>(part_r[q].size()) < kProjWarps && (best < 0 || part_load[q] < part_load[best])) best = q;
            part_r[best].push_back(static_cast<int>(i));
            part_load[best] += rects[i].tiles;
        }
        L.proj_parts = parts;
        L.proj_rects.assign(static_cast<size_t>(parts) * kProjWarps, make_int4(0, 0, 1, 0));
        L.proj_out.assign(static_cast<size_t>(parts) * kProjWarps * kProjTiles * 64, -1);
        for (int q = 0; q < parts; ++q) {
            for (size_t w = 0; w < part_r[q].size(); ++w) {
                const Rect& r = rects[part_r[q][w]];
                const size_t slot = static_cast<size_t>(q) * kProjWarps + w;
                L.proj_rects[slot] = make_int4(r.gb0, r.tb0, r.ng | r.nt << 8, r.tiles);
                for (int ig = 0; ig < r.ng; ++ig) {
                    for (int n = 0; n < 8; ++n) {  // group row of the tile (lane >> 2)
                        const int c = 8 * (r.gb0 + ig) + n;
                        if (c >= static_cast<int>(gi.size())) continue;
                        const Grp& gr = groups[gi[c]];
                        for (int64_t row = gr.r0; row < gr.r0 + gr.n; ++row) {
                            const int t = rank[static_cast<size_t>(at(row, d - 2)) * Bn + at(row, d - 1)];
                            const int it = t / 8 - r.tb0;
                            if (it < 0 || it >= r.nt) continue;
                            // C[row = lane >> 2][col = 2 (lane & 3) + h]
                            const int col = t % 8, lane = n * 4 + col / 2, h = col % 2;
                            L.proj_out[(slot * kProjTiles + ig * r.nt + it) * 64 + lane * 2 + h] = static_cast<int32_t>(row);
                        }
                    }
                }
            }
        }
    }
    L.ok = true;
    return L;
}

// The series program on the device (tiles + group words).
struct DevProgram {
    DevBuf<int4> tiles;
    DevBuf<uint32_t> prog;
    DevProgram(const Program& p, cudaStream_t st) {
        tiles.alloc(p.tiles.size());
        tiles.upload(p.tiles.data(), p.tiles.size(), st);
        prog.alloc(p.tile_prog.size());
        prog.upload(p.tile_prog.data(), p.tile_prog.size(), st);
    }
    SeriesTiles view() const { return SeriesTiles{tiles.p, static_cast<int>(tiles.n), prog.p}; }
};

// ------------------------------------------------------------------ NCCL (loaded lazily)
struct NcclApi {
    void* handle = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            api.handle = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (api.handle) break;
        }
        if (!api.handle) return;
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(api.handle, "ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(api.handle, "ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(api.handle, "ncclCommDestroy"));
        api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(api.handle, "ncclAllGather"));
        api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(api.handle, "ncclAllReduce"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(dlsym(api.handle, "ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(dlsym(api.handle, "ncclGroupEnd"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(api.handle, "ncclGetErrorString"));
    });
    if (!api.handle || !api.GetUniqueId || !api.CommInitRank || !api.AllGather || !api.AllReduce || !api.GroupStart ||
        !api.GroupEnd)
        fail(QRMC_ENCCL, "libnccl.so.2 could not be loaded");
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        fail(QRMC_ENCCL, fmt("%s: %s", what, nccl().GetErrorString ? nccl().GetErrorString(r) : "error"));
}

}  // namespace

// ------------------------------------------------------------------ session / plan
struct qrmc_gpu_session {
    int device = 0;
    int rank = 0;
    int world = 1;
    cudaStream_t stream = nullptr;
    ncclComm_t comm = nullptr;
};

struct qrmc_gpu_plan {
    qrmc_gpu_session* session = nullptr;
    bool owns_session = false;
    Gamma gamma;
    Program program;
    StepArgs base{};
    ProjArgs proj{};
    int64_t K = 0;
    int steps = 0;
    int lanes_per_rank = kLanes;
    // The ranks whose paths this process computes: its own session rank, or --
    // for qrmc_gpu_replay_ranks_solve -- every rank of a virtual world of G ranks
    // on this one device, each writing its own lanes' partial rows (what the
    // per-step ncclAllGather assembles when the ranks are separate GPUs).
    struct Shard {
        int rank = 0, lane_lo = 0, lane_hi = 0;
        int64_t n_owned = 0;
        DevBuf<double> resp, cloud;
    };
    std::vector<std::unique_ptr<Shard>> shards;
    int shard_world = 1;
    DevBuf<uint32_t> d_tile_prog;
    DevBuf<int4> d_tiles;
    DevBuf<int32_t> d_pack_pos, d_item_k, d_item_len, d_item_leaf, d_item_pre;
    int n_items = 0;
    // tensor-core K1 (responses_mma.cu), when the index set allows it
    bool use_mma = false, use_proj_mma = false;
    bool use_ws = false;  // warp-specialised K1 (responses_ws.cu) in place of k_responses_mma
    WsArgs ws{};
    DevBuf<int4> d_ws_units, d_ws_warps;
    DevBuf<uint4> d_ws_terms;
    DevBuf<int32_t> d_ws_stride;
    DevBuf<uint32_t> d_ws_gk;
    MmaArgs mma{};
    ProjMmaArgs pmma{};
    DevBuf<int4> d_pm_rects;
    DevBuf<int32_t> d_pm_out;
    DevBuf<double> d_pm_scratch;  // K2 split halves (ProjMmaArgs::split)
    DevBuf<int> d_pm_counters;
    DevBuf<double> d_alpha_mma;
    DevBuf<int4> d_mma_units, d_mma_warps;
    DevBuf<uint32_t> d_mma_terms;
    DevBuf<uint16_t> d_mma_gk;
    DevBuf<int32_t> d_mma_pos;
    DevBuf<double> d_pack_scale, d_alpha, d_coef, d_partials;
    DevBuf<unsigned long long> d_counters;
    DevBuf<int> d_flags;
    cudaGraphExec_t graph = nullptr;
    // 3N+1 events: ev[0] before the first kernel, then one after each kernel;
    // step i's kernels (responses, project[+exchange], finish) end at
    // ev[3(N-1-i)+1 .. 3(N-1-i)+3].
    std::vector<cudaEvent_t> ev;
    int launches_per_run = 0;
    uint64_t h2d_bytes = 0, d2h_bytes = 0;

    ~qrmc_gpu_plan() {
        if (graph) cudaGraphExecDestroy(graph);
        for (auto e : ev) cudaEventDestroy(e);
    }
};

namespace {

std::unique_ptr<qrmc_gpu_session> make_session(int device, int rank, int world, const void* id) {
    if (world < 1 || rank < 0 || rank >= world) fail(QRMC_EINVAL, "session: bad rank/world");
    auto s = std::make_unique<qrmc_gpu_session>();
    s->device = device;
    s->rank = rank;
    s->world = world;
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    cuda_check(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    if (world > 1) {
        if (!id) fail(QRMC_EINVAL, "session: world > 1 needs an NCCL unique id");
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof uid);
        nccl_check(nccl().CommInitRank(&s->comm, world, uid, rank), "ncclCommInitRank");
    }
    return s;
}

void destroy_session(qrmc_gpu_session* s) {
    if (!s) return;
    cudaSetDevice(s->device);
    if (s->comm) nccl().CommDestroy(s->comm);
    if (s->stream) cudaStreamDestroy(s->stream);
    delete s;
}

int current_device() {
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    return dev;
}

// Enqueue the whole backward loop on st (captured into a graph when world == 1).
void enqueue_solve(qrmc_gpu_plan& P, cudaStream_t st, bool with_events) {
    const int N = P.steps;
    cuda_check(cudaMemsetAsync(P.d_counters.p, 0, 2 * sizeof(unsigned long long), st), "memset");
    cuda_check(cudaMemsetAsync(P.d_flags.p, 0, sizeof(int), st), "memset");
    // flags[1] = 0x7f7f7f7f: "no SimulationError step yet" for atomicMin
    cuda_check(cudaMemsetAsync(P.d_flags.p + 1, 0x7f, sizeof(int), st), "memset");
    int e = 0;
    auto mark = [&] {
        if (with_events) cuda_check(cudaEventRecordWithFlags(P.ev[e++], st, cudaEventRecordExternal), "event");
    };
    mark();
    const int world = P.session->world;
    auto shard_args = [&](const qrmc_gpu_plan::Shard& sh, int i) {
        StepArgs a = P.base;
        a.step = i;
        a.lane_lo = sh.lane_lo;
        a.owned_lanes = sh.lane_hi - sh.lane_lo;
        a.n_owned = sh.n_owned;
        a.resp = sh.resp.p;
        a.cloud = sh.cloud.p;
        return a;
    };
    for (int i = N - 1; i >= 0; --i) {
        for (const auto& sh : P.shards) {
            const StepArgs a = shard_args(*sh, i);
            if (P.use_ws)
                cuda_check(launch_responses_ws(a, P.ws, st), "k_responses_ws");
            else if (P.use_mma)
                cuda_check(launch_responses_mma(a, P.mma, st), "k_responses_mma");
            else
                cuda_check(launch_responses(a, st), "k_responses");
        }
        mark();
        for (const auto& sh : P.shards) {
            const StepArgs a = shard_args(*sh, i);
            ProjArgs pa = P.proj;
            pa.partials = P.d_partials.p + static_cast<size_t>(sh->lane_lo) * P.K;
            if (P.use_proj_mma) {
                ProjMmaArgs pm = P.pmma;
                pm.partials = pa.partials;
                cuda_check(launch_project_mma(a, pm, st), "k_project_mma");
            } else {
                cuda_check(launch_project(a, pa, st), "k_project");
            }
        }
        if (world > 1) {
            // Every rank must agree on the solve's fate before the partial rows are
            // shared: a SimulationError / NumericError on any rank aborts all of
            // them at the next step's K1 (parallel.cpp:22-43 rethrows the first
            // lane exception for the whole solve). flags = {kind (max: ESIM wins),
            // min SimulationError step}.
            nccl_check(nccl().GroupStart(), "ncclGroupStart");
            nccl_check(nccl().AllReduce(P.d_flags.p, P.d_flags.p, 1, ncclInt32, ncclMax, P.session->comm, st),
                       "ncclAllReduce(flags)");
            nccl_check(nccl().AllReduce(P.d_flags.p + 1, P.d_flags.p + 1, 1, ncclInt32, ncclMin, P.session->comm, st),
                       "ncclAllReduce(step)");
            nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
            const size_t lpr = static_cast<size_t>(P.lanes_per_rank);
            nccl_check(nccl().AllGather(P.d_partials.p + static_cast<size_t>(P.session->rank) * lpr * P.K,
                                        P.d_partials.p, lpr * P.K, ncclDouble, P.session->comm, st),
                       "ncclAllGather");
        }
        mark();
        FinishArgs f{};
        f.all_partials = P.d_partials.p;
        f.basis_size = P.K;
        f.inv_m = 1.0 / static_cast<double>(P.base.paths);
        f.coef_row = P.d_coef.p + static_cast<size_t>(i) * P.K;
        f.pack_pos = P.d_pack_pos.p;
        f.pack_scale = P.d_pack_scale.p;
        if (P.use_mma) {
            f.alpha_mma = P.d_alpha_mma.p;
            f.mma_row_len = P.use_ws ? 0 : P.mma.row_len;
            f.mma_pos = P.d_mma_pos.p;
            f.mma_stride = P.use_ws ? P.d_ws_stride.p : nullptr;
        }
        StepArgs a = P.base;
        a.step = i;
        cuda_check(launch_finish(a, f, st), "k_finish_step");
        mark();
    }
    if (world > 1) {
        // TruncationStats are the sums over all lanes (solver.cpp:220-223): every
        // rank returns the global counters
        nccl_check(nccl().AllReduce(P.d_counters.p, P.d_counters.p, 2, ncclUint64, ncclSum, P.session->comm, st),
                   "ncclAllReduce(counters)");
    }
}

std::unique_ptr<qrmc_gpu_plan> make_plan(qrmc_gpu_session* s, const qrmc_problem_t& prob,
                                         const qrmc_config_t& cfg, int replay_world = 0) {
    validate_config(cfg);
    auto P = std::make_unique<qrmc_gpu_plan>();
    P->session = s;
    cuda_check(cudaSetDevice(s->device), "cudaSetDevice");
    const ProblemDev pd = to_device_problem(prob);
    P->gamma = build_gamma(cfg.gamma_kind, prob.dim, cfg.degrees, cfg.n_degrees);
    if (P->gamma.dim != prob.dim) fail(QRMC_EINVAL, "RunConfig: gamma/measure dims must equal spec.dim");
    const MeasureDev md = to_device_measure(cfg, prob.dim);
    P->program = build_program(P->gamma);
    P->K = P->gamma.size();
    P->steps = cfg.steps;
    const int d = prob.dim;
    cudaStream_t st = s->stream;

    // lane ownership: rank g owns lanes [g*lpr, min(256, (g+1)*lpr))
    if (replay_world < 0 || replay_world > kLanes) fail(QRMC_EINVAL, "replay: world must be in [1, 256]");
    if (replay_world > 0 && s->world != 1) fail(QRMC_EINVAL, "replay: needs a single-process session");
    const int G = replay_world > 0 ? replay_world : s->world;
    P->shard_world = G;
    P->lanes_per_rank = (kLanes + G - 1) / G;
    const int64_t chunks = (cfg.paths + kChunk - 1) / kChunk;
    for (int r = (replay_world > 0 ? 0 : s->rank); r < (replay_world > 0 ? G : s->rank + 1); ++r) {
        auto sh = std::make_unique<qrmc_gpu_plan::Shard>();
        sh->rank = r;
        sh->lane_lo = std::min(kLanes, r * P->lanes_per_rank);
        sh->lane_hi = std::min(kLanes, sh->lane_lo + P->lanes_per_rank);
        for (int lane = sh->lane_lo; lane < sh->lane_hi; ++lane)
            for (int64_t c = lane; c < chunks; c += kLanes)
                sh->n_owned += std::min<int64_t>(kChunk, cfg.paths - c * kChunk);
        sh->resp.alloc(static_cast<size_t>(std::max<int64_t>(sh->n_owned, 1)));
        if (cfg.memory_mode == QRMC_MEMORY_STORE_CLOUD)
            sh->cloud.alloc(static_cast<size_t>(std::max<int64_t>(sh->n_owned, 1)) * d);
        P->shards.push_back(std::move(sh));
    }

    // device tables
    const Program& pg = P->program;
    P->d_tiles.alloc(pg.tiles.size());
    P->d_tiles.upload(pg.tiles.data(), pg.tiles.size(), st);
    P->d_tile_prog.alloc(pg.tile_prog.size());
    P->d_tile_prog.upload(pg.tile_prog.data(), pg.tile_prog.size(), st);
    P->d_pack_pos.alloc(pg.pack_pos.size());
    P->d_pack_pos.upload(pg.pack_pos.data(), pg.pack_pos.size(), st);
    P->d_pack_scale.alloc(pg.pack_scale.size());
    P->d_pack_scale.upload(pg.pack_scale.data(), pg.pack_scale.size(), st);
    P->d_alpha.alloc(static_cast<size_t>(cfg.steps) * pg.kp);
    cuda_check(cudaMemsetAsync(P->d_alpha.p, 0, P->d_alpha.n * sizeof(double), st), "memset");
    P->d_coef.alloc(static_cast<size_t>(cfg.steps) * P->K);
    P->d_partials.alloc(static_cast<size_t>(P->lanes_per_rank) * G * P->K);
    cuda_check(cudaMemsetAsync(P->d_partials.p, 0, P->d_partials.n * sizeof(double), st), "memset");
    P->d_counters.alloc(2);
    P->d_flags.alloc(2);

    StepArgs& a = P->base;
    a.prob = pd;
    a.meas = md;
    a.steps = cfg.steps;
    a.step = cfg.steps - 1;
    a.dt = prob.horizon / cfg.steps;
    a.sqrt_dt = std::sqrt(a.dt);
    a.q = cfg.damping;
    a.seed = cfg.seed;
    a.paths = cfg.paths;
    a.lane_lo = P->shards.front()->lane_lo;  // per shard at launch (enqueue_solve)
    a.owned_lanes = P->shards.front()->lane_hi - P->shards.front()->lane_lo;
    a.n_owned = P->shards.front()->n_owned;
    a.alpha_packed = P->d_alpha.p;
    a.kp = pg.kp;
    a.tiles = SeriesTiles{P->d_tiles.p, static_cast<int>(P->d_tiles.n), P->d_tile_prog.p};
    a.resp = P->shards.front()->resp.p;
    a.cloud = P->shards.front()->cloud.p;
    a.counters = P->d_counters.p;
    a.err_flags = P->d_flags.p;
    a.abort_flag = P->d_flags.p;

    ProjArgs& pa = P->proj;
    int off = 0;
    for (int l = 0; l < d; ++l) {
        pa.offset[l] = off;
        pa.kmax[l] = P->gamma.kmax[l];
        off += (P->gamma.kmax[l] + 2) & ~1;  // even: K2 reads leaf values as 16-byte pairs
    }
    pa.table_len = off;
    const ProjectItems items = build_project_items(P->gamma, pa.offset);
    P->n_items = items.n;
    P->d_item_k.alloc(items.k.size());
    P->d_item_k.upload(items.k.data(), items.k.size(), st);
    P->d_item_len.alloc(items.len.size());
    P->d_item_len.upload(items.len.data(), items.len.size(), st);
    P->d_item_leaf.alloc(items.leaf.size());
    P->d_item_leaf.upload(items.leaf.data(), items.leaf.size(), st);
    P->d_item_pre.alloc(items.pre.size());
    P->d_item_pre.upload(items.pre.data(), items.pre.size(), st);
    pa.item_k = P->d_item_k.p;
    pa.item_len = P->d_item_len.p;
    pa.item_leaf = P->d_item_leaf.p;
    pa.item_pre = P->d_item_pre.p;
    pa.n_items = items.n;
#ifndef QRMC_PROJ_SMEM_KB
#define QRMC_PROJ_SMEM_KB 96
#endif
    const size_t budget = QRMC_PROJ_SMEM_KB * 1024;  // K2 point-table staging
    const size_t per_point = (static_cast<size_t>(off) + 1) * sizeof(double);
    if (per_point > budget)
        fail(QRMC_ENOTIMPL, fmt("per-point basis table of %d entries exceeds shared memory", off));
    pa.batch = static_cast<int>(std::min<size_t>(64, budget / per_point));
    pa.basis_size = P->K;

    // tensor-core K1 when the index set is a chain of (s, b) prefixes and the
    // per-path tables fit shared memory; QRMC_K1=series forces the series program
    {
        const char* k1 = std::getenv("QRMC_K1");
        const bool want = !(k1 && std::strcmp(k1, "series") == 0);
        const size_t smem = responses_mma_smem_bytes(d, off);
        int optin = 0;
        cuda_check(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, s->device), "attr");
        if (want && d >= 3 && smem && smem <= static_cast<size_t>(optin)) {
            MmaLayout L = build_mma_layout(P->gamma, pa.offset);
            if (L.ok) {
                P->use_mma = true;
                P->d_mma_units.alloc(L.units.size());
                P->d_mma_units.upload(L.units.data(), L.units.size(), st);
                P->d_mma_warps.alloc(L.warp_info.size());
                P->d_mma_warps.upload(L.warp_info.data(), L.warp_info.size(), st);
                P->d_mma_terms.alloc(L.terms.size());
                P->d_mma_terms.upload(L.terms.data(), L.terms.size(), st);
                P->d_mma_gk.alloc(L.gk.size());
                P->d_mma_gk.upload(L.gk.data(), L.gk.size(), st);
                P->d_mma_pos.alloc(L.pos.size());
                P->d_mma_pos.upload(L.pos.data(), L.pos.size(), st);
                P->d_alpha_mma.alloc(static_cast<size_t>(cfg.steps) * L.row_len);
                cuda_check(cudaMemsetAsync(P->d_alpha_mma.p, 0, P->d_alpha_mma.n * sizeof(double), st), "memset");
                MmaArgs& m = P->mma;
                m.alpha = P->d_alpha_mma.p;
                m.row_len = L.row_len;
                m.units = P->d_mma_units.p;
                m.warp_info = P->d_mma_warps.p;
                m.terms = P->d_mma_terms.p;
                m.gk = P->d_mma_gk.p;
                m.table_len = off;
                for (int l = 0; l < d; ++l) {
                    m.offset[l] = pa.offset[l];
                    m.kmax[l] = pa.kmax[l];
                }
                cuda_check(configure_responses_mma(d, smem), "k_responses_mma attributes");
                // the warp-specialised K1 when two table buffers fit and d <= 4: with five or
                // more coordinates its four producer warps run two Euler/table rounds per
                // evaluation and the single-buffered k_responses_mma is faster (d=5: 0.111 vs
                // 0.145 s, d=6 Gamma_H(6,64): 1.02 vs 1.23 s at M=2e6; profiles/r02_k1_ws.md).
                // QRMC_K1=mma / QRMC_K1=ws force either.
                const size_t wsmem = responses_ws_smem_bytes(d, off);
                const bool ws_pick = k1 && std::strcmp(k1, "ws") == 0 ? true : (d <= 4 && !(k1 && std::strcmp(k1, "mma") == 0));
                if (ws_pick && wsmem && wsmem <= static_cast<size_t>(optin) &&
                    static_cast<int64_t>(off) * 32 < 0xFFFF) {
                    MmaLayoutOpts o;
                    o.warps = kWsConsumers;
                    o.euler_ahead = false;
                    o.ring = false;
                    o.bank_order = 1;
                    o.tail_terms = ws_tail_terms();
                    o.bundle = QRMC_WS_BUNDLE;
                    MmaLayout W = build_mma_layout(P->gamma, pa.offset, o);
                    if (W.ok) {
                        P->use_ws = true;
                        P->d_ws_units.alloc(W.units.size());
                        P->d_ws_units.upload(W.units.data(), W.units.size(), st);
                        P->d_ws_warps.alloc(W.warp_info.size());
                        P->d_ws_warps.upload(W.warp_info.data(), W.warp_info.size(), st);
                        P->d_ws_terms.alloc(W.ws_terms.size());
                        P->d_ws_terms.upload(W.ws_terms.data(), W.ws_terms.size(), st);
                        P->d_ws_gk.alloc(W.ws_gk.size());
                        P->d_ws_gk.upload(W.ws_gk.data(), W.ws_gk.size(), st);
                        // warp-major fragment streams: warp w's series 0..N-1 back to back,
                        // so a consumer (and its L1 prefetch) walks one linear stream from
                        // alpha_{i+1} to alpha_{N-1}; finish writes alpha_i at pos + i * stride
                        const int N = cfg.steps;
                        std::vector<int4> winfo = W.warp_info;
                        std::vector<int32_t> wpos(W.pos.size()), wstride(W.pos.size());
                        for (size_t k = 0; k < W.pos.size(); ++k) {
                            const int64_t frag = W.pos[k] / 32, lane_slot = W.pos[k] % 32;
                            int w = 0;
                            while (!(frag >= winfo[w].z && frag < winfo[w].z + winfo[w].w)) ++w;
                            wpos[k] = static_cast<int32_t>((static_cast<int64_t>(winfo[w].z) * N + (frag - winfo[w].z)) * 32 + lane_slot);
                            wstride[k] = winfo[w].w * 32;
                        }
                        for (auto& wi : winfo) wi.z *= N;
                        P->d_ws_warps.upload(winfo.data(), winfo.size(), st);
                        P->d_mma_pos.alloc(wpos.size());
                        P->d_mma_pos.upload(wpos.data(), wpos.size(), st);
                        P->d_ws_stride.alloc(wstride.size());
                        P->d_ws_stride.upload(wstride.data(), wstride.size(), st);
                        // + the prefetch distance: the last warp's prefetches stay in bounds
                        P->d_alpha_mma.alloc(static_cast<size_t>(N) * W.row_len + 32 * (kWsPrefetch + 2));
                        cuda_check(cudaMemsetAsync(P->d_alpha_mma.p, 0, P->d_alpha_mma.n * sizeof(double), st), "memset");
                        m.alpha = nullptr;  // k_responses_mma is not launched
                        WsArgs& w = P->ws;
                        w.alpha = P->d_alpha_mma.p;
                        w.units = P->d_ws_units.p;
                        w.warp_info = P->d_ws_warps.p;
                        w.terms = P->d_ws_terms.p;
                        w.gk = P->d_ws_gk.p;
                        w.n_groups = static_cast<int>(W.ws_gk.size() / ws_gk_record(d));
                        w.table_len = off;
                        for (int l = 0; l < d; ++l) {
                            w.offset[l] = pa.offset[l];
                            w.kmax[l] = pa.kmax[l];
                        }
                        cuda_check(configure_responses_ws(d, wsmem), "k_responses_ws attributes");
                        P->h2d_bytes += (W.units.size() + W.warp_info.size()) * sizeof(int4) +
                                        W.ws_terms.size() * sizeof(uint4) + W.ws_gk.size() * sizeof(uint32_t) +
                                        2 * W.pos.size() * sizeof(int32_t);
                    }
                }
                // K2 on the tensor cores (QRMC_K2=series forces the series K2)
                const char* k2 = std::getenv("QRMC_K2");
                // QRMC_K2_BATCH=16 forces the narrow batch (tests: both give the same bits)
                // and QRMC_K2_BATCH=24 the wide one when it fits. Default: 24 paths for d <= 4 (Gamma_H(4,100):
                // K2 -4..6%), 16 beyond (Gamma_H(6,64): 0.338 vs 0.347 s, d = 5, 6 otherwise equal)
                const char* k2b = std::getenv("QRMC_K2_BATCH");
                int pbatch = project_mma_batch(off, static_cast<size_t>(optin));
                const int want = k2b ? std::atoi(k2b) : (d <= 4 ? kProjBatchWide : kProjBatchNarrow);
                if (pbatch && want == kProjBatchNarrow) pbatch = kProjBatchNarrow;
                const size_t psmem = pbatch ? project_mma_smem_bytes(off, pbatch) : 0;
                if (!(k2 && std::strcmp(k2, "series") == 0) && pbatch && L.proj_parts > 0) {
                    P->use_proj_mma = true;
                    P->d_pm_rects.alloc(L.proj_rects.size());
                    P->d_pm_rects.upload(L.proj_rects.data(), L.proj_rects.size(), st);
                    P->d_pm_out.alloc(L.proj_out.size());
                    P->d_pm_out.upload(L.proj_out.data(), L.proj_out.size(), st);
                    ProjMmaArgs& pm = P->pmma;
                    pm.rects = P->d_pm_rects.p;
                    pm.out = P->d_pm_out.p;
                    pm.terms = P->d_mma_terms.p;
                    pm.gk = P->d_mma_gk.p;
                    pm.scale = P->d_pack_scale.p;
                    pm.parts = L.proj_parts;
                    pm.table_len = off;
                    for (int l = 0; l < d; ++l) {
                        pm.offset[l] = pa.offset[l];
                        pm.kmax[l] = pa.kmax[l];
                    }
                    pm.basis_size = P->K;
                    pm.batch = pbatch;
                    // split each lane's chunks over two CTAs when that fills the last wave of
                    // CTAs (one CTA per SM) noticeably better: Gamma_H(4,100) on 148 SMs runs
                    // 2 x 256 CTAs = 3.46 waves (87% of 4 busy), split 6.92 waves (99% of 7)
                    {
                        int sms = 0;
                        cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->device), "attr");
                        const char* ks = std::getenv("QRMC_K2_SPLIT");
                        // decided on the single-GPU grid (all 256 lanes) whatever the world size:
                        // the split changes the rounding of the lane sums, and alpha must be
                        // bitwise independent of the GPU count
                        const double w1 = static_cast<double>(L.proj_parts) * kLanes / std::max(sms, 1);
                        const double e1 = w1 / std::ceil(w1), e2 = 2 * w1 / std::ceil(2 * w1);
                        pm.split = ks ? (std::atoi(ks) == 2 ? 2 : 1) : (e2 > e1 + 0.02 ? 2 : 1);
                        if (pm.split == 2) {
                            P->d_pm_scratch.alloc(static_cast<size_t>(2) * kLanes * L.proj_parts * kProjWarps *
                                                  kProjTiles * 64);
                            P->d_pm_counters.alloc(static_cast<size_t>(kLanes) * L.proj_parts);
                            cuda_check(cudaMemsetAsync(P->d_pm_counters.p, 0, P->d_pm_counters.n * sizeof(int), st),
                                       "memset");
                            pm.scratch = P->d_pm_scratch.p;
                            pm.counters = P->d_pm_counters.p;
                        }
                    }
                    cuda_check(configure_project_mma(d, pbatch, psmem), "k_project_mma attributes");
                    P->base.cloud_cos = 1;  // K1 stores cos(pi F(x)) for this K2
                    P->h2d_bytes += L.proj_rects.size() * sizeof(int4) + L.proj_out.size() * sizeof(int32_t);
                }
                P->h2d_bytes += (L.units.size() + L.warp_info.size()) * sizeof(int4) +
                                L.terms.size() * sizeof(uint32_t) + L.gk.size() * sizeof(uint16_t) +
                                L.pos.size() * sizeof(int32_t);
            }
        }
    }
    cuda_check(configure_project(d, project_smem_bytes(pa)), "k_project attributes");
    cuda_check(configure_series_kernels(), "series kernel attributes");
    P->ev.resize(3 * static_cast<size_t>(cfg.steps) + 1);
    for (auto& e : P->ev) cuda_check(cudaEventCreate(&e), "cudaEventCreate");
    P->launches_per_run = (2 * static_cast<int>(P->shards.size()) + 1) * cfg.steps;
    P->h2d_bytes += (items.k.size() * 3 + items.pre.size()) * sizeof(int32_t) +
                   pg.pack_pos.size() * sizeof(int32_t) + pg.pack_scale.size() * sizeof(double) +
                   pg.tiles.size() * sizeof(int4) + pg.tile_prog.size() * sizeof(uint32_t);
    P->d2h_bytes = static_cast<uint64_t>(cfg.steps) * P->K * sizeof(double) + 2 * sizeof(unsigned long long) +
                   2 * sizeof(int);

    if (s->world == 1) {
        cudaGraph_t g;
        cuda_check(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "capture");
        try {
            enqueue_solve(*P, st, true);
        } catch (...) {
            cudaStreamEndCapture(st, &g);
            throw;
        }
        cuda_check(cudaStreamEndCapture(st, &g), "capture end");
        cuda_check(cudaGraphInstantiate(&P->graph, g, 0), "graph instantiate");
        cudaGraphDestroy(g);
    }
    cuda_check(cudaStreamSynchronize(st), "plan sync");
    return P;
}

void run_plan(qrmc_gpu_plan& P, qrmc_stats_t* stats, double* step_wall) {
    cudaStream_t st = P.session->stream;
    cuda_check(cudaSetDevice(P.session->device), "cudaSetDevice");
    if (P.graph)
        cuda_check(cudaGraphLaunch(P.graph, st), "graph launch");
    else
        enqueue_solve(P, st, true);
    cuda_check(cudaStreamSynchronize(st), "solve");
    unsigned long long counters[2];
    int flags[2];
    cuda_check(cudaMemcpy(counters, P.d_counters.p, sizeof counters, cudaMemcpyDeviceToHost), "D2H");
    cuda_check(cudaMemcpy(flags, P.d_flags.p, sizeof flags, cudaMemcpyDeviceToHost), "D2H");
    float ms = 0.f;
    cuda_check(cudaEventElapsedTime(&ms, P.ev.front(), P.ev.back()), "event time");
    if (step_wall) {
        for (int i = 0; i < P.steps; ++i) {
            const int b = 3 * (P.steps - 1 - i);
            float t = 0.f;
            cuda_check(cudaEventElapsedTime(&t, P.ev[b], P.ev[b + 3]), "event time");
            step_wall[i] = t * 1e-3;
        }
    }
    if (stats) {
        stats->applications = counters[0];
        stats->clipped = counters[1];
        stats->error_step = -1;
        stats->kernel_launches = P.launches_per_run;
        stats->device_seconds = ms * 1e-3;
    }
    if (flags[0] == QRMC_ESIM) {
        Failure f{QRMC_ESIM, fmt("euler_step: state out of range at step %d", flags[1]), flags[1]};
        throw f;
    }
    if (flags[0] == QRMC_ENUMERIC) fail(QRMC_ENUMERIC, "backward_solve: non-finite response or coefficient");
}

void download(qrmc_gpu_plan& P, double* coeffs, size_t len) {
    const size_t need = static_cast<size_t>(P.steps) * P.K;
    if (!coeffs || len < need) fail(QRMC_EINVAL, "coefficient buffer too small");
    cuda_check(cudaMemcpy(coeffs, P.d_coef.p, need * sizeof(double), cudaMemcpyDeviceToHost), "D2H coeffs");
}

// A throwaway single-GPU context for the probe entry points.
struct Scratch {
    std::unique_ptr<qrmc_gpu_session, void (*)(qrmc_gpu_session*)> s{nullptr, destroy_session};
    Scratch() {
        s.reset(make_session(current_device(), 0, 1, nullptr).release());
        cuda_check(configure_series_kernels(), "series kernel attributes");
    }
};

// Minimal StepArgs for probes that only need the problem and measure.
StepArgs probe_args(const qrmc_problem_t* prob, const qrmc_config_t* cfg, int dim) {
    StepArgs a{};
    if (prob) a.prob = to_device_problem(*prob);
    else a.prob.dim = dim;
    a.meas = to_device_measure(*cfg, dim);
    a.steps = cfg->steps;
    const double horizon = prob ? prob->horizon : 1.0;
    a.dt = horizon / std::max(cfg->steps, 1);
    a.sqrt_dt = std::sqrt(a.dt);
    a.q = cfg->damping;
    a.seed = cfg->seed;
    a.paths = cfg->paths;
    return a;
}

}  // namespace

// =================================================================== C ABI
extern "C" {

qrmc_status qrmc_problem_sin_bench(int32_t dim, double kappa, double lambda, double horizon,
                                   qrmc_problem_t* out) {
    if (!out || dim < 1) return QRMC_EINVAL;
    if (!(horizon > 0.0)) return QRMC_EINVAL;
    std::memset(out, 0, sizeof *out);
    const double lam = lambda > 0.0 ? lambda : 1.0 / std::sqrt(static_cast<double>(dim));
    out->dim = dim;
    out->brownian_dim = dim;
    out->horizon = horizon;
    out->terminal_kind = QRMC_TERMINAL_SIN_SUM;
    out->driver_kind = QRMC_DRIVER_SIN_BENCH;
    out->drift_kind = QRMC_DRIFT_ZERO;
    out->diffusion_kind = QRMC_DIFFUSION_IDENTITY;
    out->terminal_params[0] = out->driver_params[0] = kappa;
    out->terminal_params[1] = out->driver_params[1] = lam;
    out->growth_g = 2.0 + kappa;
    out->growth_f = 1.0;
    out->lipschitz_f = 2.0;
    out->moment_ratio = 1.0;
    out->state_bound = 1e15;
    return QRMC_OK;
}

int64_t qrmc_gpu_gamma_size(int32_t kind, int32_t dim, const int32_t* degrees, int32_t n_degrees) {
    int64_t n = 0;
    const qrmc_status st = guarded(nullptr, 0, [&] { n = build_gamma(kind, dim, degrees, n_degrees).size(); });
    return st == QRMC_OK ? n : -static_cast<int64_t>(st);
}

qrmc_status qrmc_gpu_gamma_indices(int32_t kind, int32_t dim, const int32_t* degrees, int32_t n_degrees,
                                   int32_t* out, size_t out_len, char* err, size_t err_len) {
    return guarded(err, err_len, [&] {
        const Gamma g = build_gamma(kind, dim, degrees, n_degrees);
        if (!out || out_len < g.rows.size()) fail(QRMC_EINVAL, "output buffer too small");
        std::memcpy(out, g.rows.data(), g.rows.size() * sizeof(int32_t));
    });
}

qrmc_status qrmc_gpu_mma_layout_check(int32_t kind, int32_t dim, const int32_t* degrees, int32_t n_degrees,
                                      uint64_t seed, int64_t* info, double* max_rel_err, char* err, size_t err_len) {
    return guarded(err, err_len, [&] {
        if (!info || !max_rel_err) fail(QRMC_EINVAL, "null output");
        const Gamma g = build_gamma(kind, dim, degrees, n_degrees);
        const int d = g.dim;
        const int64_t K = g.size();
        int offset[kMaxDim] = {}, off = 0;
        for (int l = 0; l < d; ++l) {  // make_plan's table layout
            offset[l] = off;
            off += (g.kmax[l] + 2) & ~1;
        }
        const MmaLayout L = build_mma_layout(g, offset);
        for (int i = 0; i < 8; ++i) info[i] = 0;
        *max_rel_err = 0.0;
        info[0] = L.ok ? 1 : 0;
        if (!L.ok) return;
        // random point (cosine tables c_k = cos(k theta_l)) and coefficients
        uint64_t st = seed * 0x9E3779B97F4A7C15ull + 1;
        auto rnd = [&] {
            st ^= st << 13;
            st ^= st >> 7;
            st ^= st << 17;
            return static_cast<double>(st >> 11) * 0x1p-53;
        };
        std::vector<double> tab(static_cast<size_t>(off), 0.0);  // entry -> value (one path)
        for (int l = 0; l < d; ++l) {
            const double th = 3.141592653589793 * rnd();
            for (int k = 0; k <= g.kmax[l]; ++k) tab[static_cast<size_t>(offset[l] + k)] = std::cos(k * th);
        }
        std::vector<double> alpha(static_cast<size_t>(K));
        for (auto& a : alpha) a = 2.0 * rnd() - 1.0;
        auto term = [&](int64_t r) {
            double v = 1.0;
            for (int l = 0; l < d; ++l) v *= tab[static_cast<size_t>(offset[l] + g.rows[static_cast<size_t>(r * d + l)])];
            return v;
        };
        double direct = 0.0, scale = 0.0;
        for (int64_t r = 0; r < K; ++r) {
            direct += alpha[static_cast<size_t>(r)] * term(r);
            scale += std::fabs(alpha[static_cast<size_t>(r)] * term(r));
        }
        // K1: scatter alpha into one series' fragment stream, then replay the
        // kernel's traversal (units per warp, step alignment, B lane order,
        // A from the term table rows, epilogue through the group rows)
        std::vector<double> stream(static_cast<size_t>(L.row_len), 0.0);
        std::vector<uint8_t> hit(static_cast<size_t>(L.row_len), 0);
        for (int64_t r = 0; r < K; ++r) {
            const int32_t p = L.pos[static_cast<size_t>(r)];
            if (p < 0 || p >= L.row_len || hit[static_cast<size_t>(p)]) fail(QRMC_ELOGIC, "mma layout: position clash");
            hit[static_cast<size_t>(p)] = 1;
            stream[static_cast<size_t>(p)] = alpha[static_cast<size_t>(r)];
        }
        auto row_val = [&](uint32_t row_x_stride) { return tab[row_x_stride / kMmaTabStride]; };
        const int nu = d - 2;
        double y = 0.0;
        int64_t frags_read = 0;
        for (int w = 0; w < kMmaWarps; ++w) {
            const int4 wi = L.warp_info[static_cast<size_t>(w)];
            int64_t fpos = 0;
            for (int u = wi.x; u < wi.y; ++u) {
                const int4 un = L.units[static_cast<size_t>(u)];
                const int nb = un.y, W = nb == 3 ? 4 : nb;
                fpos = (fpos + W - 1) / W * W;
                std::vector<double> C(static_cast<size_t>(nb) * 8, 0.0);
                for (int c = un.z; c < un.w; ++c, fpos += W) {
                    for (int i = 0; i < nb; ++i) {
                        const double* B = &stream[static_cast<size_t>((wi.z + fpos + i) * 32)];
                        ++frags_read;
                        for (int lane = 0; lane < 32; ++lane) {
                            const int rr = lane & 3, col = lane >> 2;  // B[term rr][group col]
                            const uint32_t tp = L.terms[static_cast<size_t>(4 * c + rr)];
                            const double A = row_val(tp & 0xFFFFu) * row_val(tp >> 16);
                            C[static_cast<size_t>(i * 8 + col)] += A * B[lane];
                        }
                    }
                }
                for (int i = 0; i < nb; ++i)
                    for (int n = 0; n < 8; ++n) {
                        const int grp = 8 * (un.x + i) + n;
                        double U = 1.0;
                        for (int l = 0; l < nu; ++l) U *= row_val(L.gk[static_cast<size_t>(grp * nu + l)]);
                        y += U * C[static_cast<size_t>(i * 8 + n)];
                    }
            }
            if (fpos > wi.w) fail(QRMC_ELOGIC, "mma layout: warp stream overrun");
        }
        // K2: one path with S = 1 through every rectangle's output map
        std::vector<double> part(static_cast<size_t>(K), 0.0);
        std::vector<uint8_t> khit(static_cast<size_t>(K), 0);
        for (size_t slot = 0; slot < L.proj_rects.size(); ++slot) {
            const int4 rc = L.proj_rects[slot];
            const int ng = rc.z & 0xFF, nt = rc.z >> 8;
            if (rc.w == 0) continue;
            for (int ig = 0; ig < ng; ++ig)
                for (int it = 0; it < nt; ++it)
                    for (int lane = 0; lane < 32; ++lane)
                        for (int h = 0; h < 2; ++h) {
                            const int32_t k = L.proj_out[(slot * kProjTiles + ig * nt + it) * 64 + lane * 2 + h];
                            if (k < 0) continue;
                            if (khit[static_cast<size_t>(k)]) fail(QRMC_ELOGIC, "mma layout: K2 output clash");
                            khit[static_cast<size_t>(k)] = 1;
                            const int grp = 8 * (rc.x + ig) + (lane >> 2);
                            const int t = 8 * (rc.y + it) + 2 * (lane & 3) + h;
                            double U = 1.0;
                            for (int l = 0; l < nu; ++l) U *= row_val(L.gk[static_cast<size_t>(grp * nu + l)]);
                            const uint32_t tp = L.terms[static_cast<size_t>(t)];
                            part[static_cast<size_t>(k)] = U * row_val(tp & 0xFFFFu) * row_val(tp >> 16);
                        }
        }
        double e2 = 0.0;
        for (int64_t r = 0; r < K; ++r) {
            if (!khit[static_cast<size_t>(r)]) fail(QRMC_ELOGIC, "mma layout: K2 misses a term");
            e2 = std::max(e2, std::fabs(part[static_cast<size_t>(r)] - term(r)));
        }
        *max_rel_err = std::max(std::fabs(y - direct) / std::max(scale, 1e-300), e2);
        // warp-specialised K1 (responses_ws.cu): 32 paths with their own points in
        // swizzled [entry][32] tables; replay every lane's operand addressing
        // (row-half offsets, row blocks r = 0..3 at A[0], B[0], A[16], B[16]) and the
        // dense per-warp fragment streams, then compare each path's y with the direct sum
        for (int tail : {0, 8, 16}) {
            MmaLayoutOpts o;
            o.warps = kWsConsumers;
            o.euler_ahead = false;
            o.ring = false;
            o.bank_order = 1;
            o.tail_terms = tail;
            o.bundle = QRMC_WS_BUNDLE;
            const MmaLayout W = build_mma_layout(g, offset, o);
            if (!W.ok) fail(QRMC_ELOGIC, "ws layout: not a chain although the mma layout is");
            std::vector<double> wtab(static_cast<size_t>(off) * 32, 0.0);
            std::vector<std::vector<double>> ptab(32, std::vector<double>(static_cast<size_t>(off), 0.0));
            for (int p = 0; p < 32; ++p)
                for (int l = 0; l < d; ++l) {
                    const double th = 3.141592653589793 * rnd();
                    for (int k = 0; k <= g.kmax[l]; ++k) {
                        const int e = offset[l] + k;
                        const double v = std::cos(k * th);
                        ptab[p][static_cast<size_t>(e)] = v;
                        wtab[static_cast<size_t>(e) * 32 + (p ^ ((e & 3) << 2))] = v;
                    }
                }
            std::vector<double> ws(static_cast<size_t>(W.row_len), 0.0);
            std::vector<uint8_t> whit(static_cast<size_t>(W.row_len), 0);
            for (int64_t r = 0; r < K; ++r) {
                const int32_t q = W.pos[static_cast<size_t>(r)];
                if (q < 0 || q >= W.row_len || whit[static_cast<size_t>(q)]) fail(QRMC_ELOGIC, "ws layout: position clash");
                whit[static_cast<size_t>(q)] = 1;
                ws[static_cast<size_t>(q)] = alpha[static_cast<size_t>(r)];
            }
            const int n_groups = static_cast<int>(W.ws_gk.size() / ws_gk_record(d));  // 2 halves x n/2 pairs
            auto at_off = [&](int lane, uint32_t o16, int r16) {  // the kernel's trow + o16 + 16 r16
                return wtab[static_cast<size_t>((lane >> 2) + static_cast<int>(o16) + 16 * r16)];
            };
            std::vector<double> yp(32, 0.0);
            for (int w = 0; w < kWsConsumers; ++w) {
                const int4 wi = W.warp_info[static_cast<size_t>(w)];
                int64_t f = wi.z;
                for (int u = wi.x; u < wi.y; ++u) {
                    const int4 un = W.units[static_cast<size_t>(u)];
                    if (un.y >= 8) {
                        // transposed tail unit: K = 4 groups per chunk, N = 8 terms per block;
                        // A[row][k] = U_{4c+k}(path), B[k][n] at lane n * 4 + k
                        const int tnb = un.y - 8;
                        std::vector<double> C(static_cast<size_t>(tnb) * 4 * 64, 0.0);  // [i][r][row][term col]
                        for (int c = un.z; c < un.w; ++c, f += tnb)
                            for (int i = 0; i < tnb; ++i)
                                for (int lane = 0; lane < 32; ++lane) {
                                    const int row = lane >> 2, col = lane & 3, half = row >> 2;
                                    double uu[4] = {1, 1, 1, 1};
                                    for (int l = 0; l < d - 2; ++l) {
                                        const uint32_t o2 = W.ws_gk[ws_gk_index(d, n_groups, half, 4 * c + col, l)];
                                        uu[0] *= at_off(lane, o2 & 0xFFFFu, 0);
                                        uu[1] *= at_off(lane, o2 >> 16, 0);
                                        uu[2] *= at_off(lane, o2 & 0xFFFFu, 1);
                                        uu[3] *= at_off(lane, o2 >> 16, 1);
                                    }
                                    for (int r = 0; r < 4; ++r)
                                        for (int n = 0; n < 8; ++n)
                                            C[((static_cast<size_t>(i) * 4 + r) * 8 + row) * 8 + n] +=
                                                uu[r] * ws[static_cast<size_t>((f + i) * 32 + n * 4 + col)];
                                }
                        for (int i = 0; i < tnb; ++i)
                            for (int lane = 0; lane < 32; ++lane) {
                                const int row = lane >> 2, col = lane & 3, half = row >> 2;
                                for (int h = 0; h < 2; ++h) {
                                    const int t = 8 * i + 2 * col + h;
                                    const uint4 tw = W.ws_terms[static_cast<size_t>(t) * 2 + half];
                                    double a[4];
                                    a[0] = at_off(lane, tw.x / 8, 0) * at_off(lane, tw.z / 8, 0);
                                    a[1] = at_off(lane, tw.y / 8, 0) * at_off(lane, tw.w / 8, 0);
                                    a[2] = at_off(lane, tw.x / 8, 1) * at_off(lane, tw.z / 8, 1);
                                    a[3] = at_off(lane, tw.y / 8, 1) * at_off(lane, tw.w / 8, 1);
                                    for (int r = 0; r < 4; ++r)
                                        yp[static_cast<size_t>(8 * r + row)] +=
                                            a[r] * C[((static_cast<size_t>(i) * 4 + r) * 8 + row) * 8 + 2 * col + h];
                                }
                            }
                        continue;
                    }
                    const int nb = un.y;
                    std::vector<double> C(static_cast<size_t>(nb) * 4 * 64, 0.0);  // [i][r][path row][group col]
                    for (int c = un.z; c < un.w; ++c, f += nb)
                        for (int i = 0; i < nb; ++i)
                            for (int lane = 0; lane < 32; ++lane) {
                                // A[row][k] for row blocks r: this lane's (row, col = k) value
                                const int row = lane >> 2, col = lane & 3, half = row >> 2;
                                const uint4 tw = W.ws_terms[static_cast<size_t>(4 * c + col) * 2 + half];
                                double a[4];
                                a[0] = at_off(lane, tw.x / 8, 0) * at_off(lane, tw.z / 8, 0);
                                a[1] = at_off(lane, tw.y / 8, 0) * at_off(lane, tw.w / 8, 0);
                                a[2] = at_off(lane, tw.x / 8, 1) * at_off(lane, tw.z / 8, 1);
                                a[3] = at_off(lane, tw.y / 8, 1) * at_off(lane, tw.w / 8, 1);
                                for (int r = 0; r < 4; ++r)
                                    for (int n = 0; n < 8; ++n)  // B[k = col][n] sits at lane n * 4 + col
                                        C[((static_cast<size_t>(i) * 4 + r) * 8 + row) * 8 + n] +=
                                            a[r] * ws[static_cast<size_t>((f + i) * 32 + n * 4 + col)];
                            }
                    for (int i = 0; i < nb; ++i)
                        for (int lane = 0; lane < 32; ++lane) {
                            const int row = lane >> 2, col = lane & 3, half = row >> 2;
                            const int g0 = 8 * (un.x + i) + 2 * col;
                            for (int h = 0; h < 2; ++h) {
                                double uu[4] = {1, 1, 1, 1};
                                for (int l = 0; l < d - 2; ++l) {
                                    const uint32_t o = W.ws_gk[ws_gk_index(d, n_groups, half, g0 + h, l)];
                                    uu[0] *= at_off(lane, o & 0xFFFFu, 0);
                                    uu[1] *= at_off(lane, o >> 16, 0);
                                    uu[2] *= at_off(lane, o & 0xFFFFu, 1);
                                    uu[3] *= at_off(lane, o >> 16, 1);
                                }
                                for (int r = 0; r < 4; ++r)
                                    yp[static_cast<size_t>(8 * r + row)] +=
                                        uu[r] * C[((static_cast<size_t>(i) * 4 + r) * 8 + row) * 8 + 2 * col + h];
                            }
                        }
                }
                if (f != wi.z + wi.w) fail(QRMC_ELOGIC, "ws layout: warp stream length mismatch");
            }
            for (int p = 0; p < 32; ++p) {
                double dp = 0.0, sp = 0.0;
                for (int64_t r = 0; r < K; ++r) {
                    double v = alpha[static_cast<size_t>(r)];
                    for (int l = 0; l < d; ++l) v *= ptab[p][static_cast<size_t>(offset[l] + g.rows[static_cast<size_t>(r * d + l)])];
                    dp += v;
                    sp += std::fabs(v);
                }
                *max_rel_err = std::max(*max_rel_err, std::fabs(yp[static_cast<size_t>(p)] - dp) / std::max(sp, 1e-300));
            }
        }
        info[1] = K;
        info[2] = static_cast<int64_t>(L.units.size());
        info[3] = L.frags;
        info[4] = frags_read;
        info[5] = L.row_len / 32;
        info[6] = L.proj_parts;
        info[7] = static_cast<int64_t>(L.terms.size());
    });
}

qrmc_status qrmc_gpu_nccl_unique_id(void* out128, char* err, size_t err_len) {
    return guarded(err, err_len, [&] {
        ncclUniqueId id;
        nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(out128, &id, sizeof id);
    });
}

qrmc_status qrmc_gpu_session_create(int32_t device, int32_t rank, int32_t world, const void* nccl_unique_id,
                                    qrmc_gpu_session_t** out, char* err, size_t err_len) {
    return guarded(err, err_len, [&] {
        if (!out) fail(QRMC_EINVAL, "session: null output");
        *out = make_session(device, rank, world, nccl_unique_id).release();
    });
}

void qrmc_gpu_session_destroy(qrmc_gpu_session_t* s) { destroy_session(s); }

qrmc_status qrmc_gpu_plan_create(qrmc_gpu_session_t* session, const qrmc_problem_t* problem,
                                 const qrmc_config_t* config, qrmc_gpu_plan_t** out, char* err,
                                 size_t err_len) {
    return guarded(err, err_len, [&] {
        if (!problem || !config || !out) fail(QRMC_EINVAL, "plan: null argument");
        bool owns = false;
        if (!session) {
            session = make_session(current_device(), 0, 1, nullptr).release();
            owns = true;
        }
        try {
            auto P = make_plan(session, *problem, *config);
            P->owns_session = owns;
            *out = P.release();
        } catch (...) {
            if (owns) destroy_session(session);
            throw;
        }
    });
}

qrmc_status qrmc_gpu_plan_run(qrmc_gpu_plan_t* plan, qrmc_stats_t* stats, char* err, size_t err_len) {
    return guarded(err, err_len, [&] {
        if (!plan) fail(QRMC_EINVAL, "plan: null");
        run_plan(*plan, stats, nullptr);
    }, stats);
}

qrmc_status qrmc_gpu_plan_download(qrmc_gpu_plan_t* plan, double* coeffs, size_t coeffs_len, char* err,
                                   size_t err_len) {
    return guarded(err, err_len, [&] {
        if (!plan) fail(QRMC_EINVAL, "plan: null");
        cuda_check(cudaSetDevice(plan->session->device), "cudaSetDevice");
        download(*plan, coeffs, coeffs_len);
    });
}

int64_t qrmc_gpu_plan_basis_size(const qrmc_gpu_plan_t* plan) { return plan ? plan->K : -1; }

qrmc_status qrmc_gpu_plan_kernel_seconds(const qrmc_gpu_plan_t* plan, double* out3, double* per_step,
                                         char* err, size_t err_len) {
    return guarded(err, err_len, [&] {
        if (!plan || !out3) fail(QRMC_EINVAL, "plan_kernel_seconds: null argument");
        const int N = plan->steps;
        out3[0] = out3[1] = out3[2] = 0.0;
        for (int s = 0; s < N; ++s) {
            for (int k = 0; k < 3; ++k) {
                float t = 0.f;
                cuda_check(cudaEventElapsedTime(&t, plan->ev[3 * s + k], plan->ev[3 * s + k + 1]), "event time");
                out3[k] += t * 1e-3;
                // per_step rows are indexed by the cloud step i = N-1-s
                if (per_step) per_step[3 * (N - 1 - s) + k] = t * 1e-3;
            }
        }
    });
}

qrmc_status qrmc_gpu_lane_ownership(int64_t paths, int32_t rank, int32_t world, int32_t* lane_lo,
                                    int32_t* lane_hi, int64_t* n_owned) {
    if (paths < 1 || world < 1 || rank < 0 || rank >= world || !lane_lo || !lane_hi || !n_owned)
        return QRMC_EINVAL;
    const int lpr = (kLanes + world - 1) / world;
    const int lo = std::min(kLanes, rank * lpr);
    const int hi = std::min(kLanes, lo + lpr);
    const int64_t chunks = (paths + kChunk - 1) / kChunk;
    int64_t n = 0;
    for (int lane = lo; lane < hi; ++lane)
        for (int64_t c = lane; c < chunks; c += kLanes) n += std::min<int64_t>(kChunk, paths - c * kChunk);
    *lane_lo = lo;
    *lane_hi = hi;
    *n_owned = n;
    return QRMC_OK;
}

int64_t qrmc_gpu_owned_path(int64_t q, int32_t lane_lo, int32_t owned_lanes) {
    // the device's owned-index -> path map (kernels.cu owned_to_path), exported for host tests
    const int64_t cq = q / kChunk;
    const int64_t r = cq / owned_lanes;
    const int64_t lane = lane_lo + cq % owned_lanes;
    return (r * kLanes + lane) * kChunk + q % kChunk;
}

qrmc_status qrmc_gpu_plan_io_bytes(const qrmc_gpu_plan_t* plan, uint64_t* h2d, uint64_t* d2h) {
    if (!plan || !h2d || !d2h) return QRMC_EINVAL;
    *h2d = plan->h2d_bytes;
    *d2h = plan->d2h_bytes;
    return QRMC_OK;
}

const char* qrmc_gpu_plan_kernel_name(const qrmc_gpu_plan_t* plan, int which) {
    if (!plan) return nullptr;
    switch (which) {
        case 0: return plan->use_ws ? "k_responses_ws" : plan->use_mma ? "k_responses_mma" : "k_responses";
        case 1: return plan->use_proj_mma ? "k_project_mma" : "k_project";
        case 2: return "k_finish_step";
        default: return nullptr;
    }
}

void* qrmc_gpu_plan_stream(const qrmc_gpu_plan_t* plan) {
    return plan ? static_cast<void*>(plan->session->stream) : nullptr;
}

void qrmc_gpu_plan_destroy(qrmc_gpu_plan_t* plan) {
    if (!plan) return;
    qrmc_gpu_session* s = plan->owns_session ? plan->session : nullptr;
    cudaSetDevice(plan->session->device);
    delete plan;
    destroy_session(s);
}

qrmc_status qrmc_gpu_backward_solve(qrmc_gpu_session_t* session, const qrmc_problem_t* problem,
                                    const qrmc_config_t* config, double* coeffs, size_t coeffs_len,
                                    double* step_wall_seconds, qrmc_stats_t* stats, char* err,
                                    size_t err_len) {
    if (stats) {
        std::memset(stats, 0, sizeof *stats);
        stats->error_step = -1;
    }
    return guarded(err, err_len, [&] {
        if (!problem || !config) fail(QRMC_EINVAL, "backward_solve: null argument");
        // validate everything host-side before touching a device, in the
        // reference's order: spec.validate(), config.validate(spec) (solver.cpp:110-111)
        to_device_problem(*problem);
        validate_config(*config);
        const Gamma g = build_gamma(config->gamma_kind, problem->dim, config->degrees, config->n_degrees);
        to_device_measure(*config, problem->dim);
        if (!coeffs || coeffs_len < static_cast<size_t>(g.size()) * static_cast<size_t>(config->steps))
            fail(QRMC_EINVAL, "coefficient buffer too small");
        std::unique_ptr<qrmc_gpu_session, void (*)(qrmc_gpu_session*)> own(nullptr, destroy_session);
        if (!session) {
            own.reset(make_session(current_device(), 0, 1, nullptr).release());
            session = own.get();
        }
        auto P = make_plan(session, *problem, *config);
        run_plan(*P, stats, step_wall_seconds);
        download(*P, coeffs, coeffs_len);
    }, stats);
}

qrmc_status qrmc_gpu_replay_ranks_solve(const qrmc_problem_t* problem, const qrmc_config_t* config, int32_t world,
                                        double* coeffs, size_t coeffs_len, qrmc_stats_t* stats, char* err,
                                        size_t err_len) {
    if (stats) {
        std::memset(stats, 0, sizeof *stats);
        stats->error_step = -1;
    }
    return guarded(err, err_len, [&] {
        if (!problem || !config) fail(QRMC_EINVAL, "replay: null argument");
        if (world < 1 || world > kLanes) fail(QRMC_EINVAL, "replay: world must be in [1, 256]");
        std::unique_ptr<qrmc_gpu_session, void (*)(qrmc_gpu_session*)> own(
            make_session(current_device(), 0, 1, nullptr).release(), destroy_session);
        auto P = make_plan(own.get(), *problem, *config, world);
        run_plan(*P, stats, nullptr);
        download(*P, coeffs, coeffs_len);
    }, stats);
}

qrmc_status qrmc_gpu_evaluate(const qrmc_config_t* config, int32_t dim, const double* coeffs_step,
                              const double* x, int64_t n, double* out, char* err, size_t err_len) {
    return guarded(err, err_len, [&] {
        if (!config || !coeffs_step || (!x && n) || (!out && n)) fail(QRMC_EINVAL, "evaluate: null argument");
        Scratch sc;
        cudaStream_t st = sc.s->stream;
        const Gamma g = build_gamma(config->gamma_kind, dim, config->degrees, config->n_degrees);
        const Program pg = build_program(g);
        StepArgs a = probe_args(nullptr, config, dim);
        std::vector<double> packed(static_cast<size_t>(pg.kp), 0.0);
        for (int64_t k = 0; k < g.size(); ++k) packed[pg.pack_pos[k]] = coeffs_step[k] * pg.pack_scale[k];
        DevBuf<double> d_alpha(packed.size()), d_x(static_cast<size_t>(std::max<int64_t>(n, 1)) * dim),
            d_out(static_cast<size_t>(std::max<int64_t>(n, 1)));
        DevProgram dp(pg, st);
        d_alpha.upload(packed.data(), packed.size(), st);
        if (n) d_x.upload(x, static_cast<size_t>(n) * dim, st);
        a.tiles = dp.view();
        if (n) cuda_check(launch_eval_points(a, d_alpha.p, d_x.p, n, config->damping, 1, d_out.p, st), "k_eval_points");
        cuda_check(cudaStreamSynchronize(st), "evaluate");
        if (n) cuda_check(cudaMemcpy(out, d_out.p, static_cast<size_t>(n) * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    });
}

qrmc_status qrmc_gpu_mse_metrics(const qrmc_config_t* config, int32_t dim, double kappa, double lambda,
                                 double horizon, const double* coeffs, uint64_t eval_seed,
                                 int32_t eval_points, double* out6, double* step_sq, char* err,
                                 size_t err_len) {
    return guarded(err, err_len, [&] {
        if (!config || !coeffs || !out6) fail(QRMC_EINVAL, "mse_metrics: null argument");
        if (eval_points < 1) fail(QRMC_EINVAL, "mse_metrics: eval_points must be >= 1");
        Scratch sc;
        cudaStream_t st = sc.s->stream;
        const Gamma g = build_gamma(config->gamma_kind, dim, config->degrees, config->n_degrees);
        const Program pg = build_program(g);
        qrmc_problem_t prob{};
        qrmc_problem_sin_bench(dim, kappa, lambda, horizon, &prob);
        StepArgs a = probe_args(&prob, config, dim);
        const int N = config->steps;
        std::vector<double> packed(static_cast<size_t>(pg.kp) * N, 0.0);
        for (int i = 0; i < N; ++i)
            for (int64_t k = 0; k < g.size(); ++k)
                packed[static_cast<size_t>(i) * pg.kp + pg.pack_pos[k]] = coeffs[static_cast<size_t>(i) * g.size() + k] * pg.pack_scale[k];
        DevBuf<double> d_alpha(packed.size()), d_sq(static_cast<size_t>(N) * eval_points),
            d_squ(static_cast<size_t>(N) * eval_points);
        DevProgram dp(pg, st);
        d_alpha.upload(packed.data(), packed.size(), st);
        a.tiles = dp.view();
        a.alpha_packed = d_alpha.p;
        a.kp = pg.kp;
        const double lam = prob.terminal_params[1];
        cuda_check(launch_mse(a, kappa, lam, horizon, eval_seed, eval_points, d_sq.p, d_squ.p, st), "k_mse");
        std::vector<double> sq(d_sq.n), squ(d_squ.n);
        cuda_check(cudaStreamSynchronize(st), "mse");
        cuda_check(cudaMemcpy(sq.data(), d_sq.p, sq.size() * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
        cuda_check(cudaMemcpy(squ.data(), d_squ.p, squ.size() * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
        // metrics_from_squared_errors (benchmark.cpp:69-84), in the reference's order
        double mx = 0.0, tot = 0.0, mxu = 0.0, totu = 0.0;
        for (int i = 0; i < N; ++i) {
            double s = 0.0, su = 0.0;
            for (int m = 0; m < eval_points; ++m) {
                s += sq[static_cast<size_t>(i) * eval_points + m];
                su += squ[static_cast<size_t>(i) * eval_points + m];
            }
            mx = std::max(mx, s);
            tot += s;
            mxu = std::max(mxu, su);
            totu += su;
            if (step_sq) step_sq[i] = s;
        }
        const double nn = eval_points, steps = N;
        out6[0] = std::log(mx / nn);
        out6[1] = std::log(tot / (steps * nn));
        out6[2] = std::log(mxu / nn);
        out6[3] = std::log(totu / (steps * nn));
        out6[4] = out6[5] = 0.0;
    });
}

qrmc_status qrmc_gpu_philox(const uint32_t* ctr, const uint32_t* key, int64_t n, uint32_t* out, char* err,
                            size_t err_len) {
    return guarded(err, err_len, [&] {
        if (n <= 0) return;
        Scratch sc;
        cudaStream_t st = sc.s->stream;
        DevBuf<uint32_t> d_ctr(static_cast<size_t>(n) * 4), d_key(static_cast<size_t>(n) * 2), d_out(static_cast<size_t>(n) * 4);
        d_ctr.upload(ctr, d_ctr.n, st);
        d_key.upload(key, d_key.n, st);
        cuda_check(launch_philox(d_ctr.p, d_key.p, n, d_out.p, st), "k_philox");
        cuda_check(cudaStreamSynchronize(st), "philox");
        cuda_check(cudaMemcpy(out, d_out.p, d_out.n * sizeof(uint32_t), cudaMemcpyDeviceToHost), "D2H");
    });
}

qrmc_status qrmc_gpu_stream_draws(uint64_t seed, const uint64_t* stream_ids, int64_t n_streams, int32_t n_draws,
                                  int32_t kind, void* out, char* err, size_t err_len) {
    return guarded(err, err_len, [&] {
        if (n_streams <= 0 || n_draws <= 0) return;
        if (kind < 0 || kind > 2) fail(QRMC_EINVAL, "stream_draws: kind must be 0, 1 or 2");
        Scratch sc;
        cudaStream_t st = sc.s->stream;
        DevBuf<uint64_t> d_sid(static_cast<size_t>(n_streams)), d_out(static_cast<size_t>(n_streams) * n_draws);
        d_sid.upload(stream_ids, d_sid.n, st);
        cuda_check(launch_stream_draws(seed, d_sid.p, n_streams, n_draws, kind, d_out.p, st), "k_stream_draws");
        cuda_check(cudaStreamSynchronize(st), "draws");
        cuda_check(cudaMemcpy(out, d_out.p, d_out.n * sizeof(uint64_t), cudaMemcpyDeviceToHost), "D2H");
    });
}

qrmc_status qrmc_gpu_cloud_paths(const qrmc_problem_t* problem, const qrmc_config_t* config, int32_t step,
                                 int64_t first, int64_t n, double* out, char* err, size_t err_len) {
    return guarded(err, err_len, [&] {
        if (!problem || !config) fail(QRMC_EINVAL, "cloud_paths: null argument");
        if (step < 0 || step > config->steps) fail(QRMC_EINVAL, "cloud_paths: step out of range");
        if (n <= 0) return;
        Scratch sc;
        cudaStream_t st = sc.s->stream;
        StepArgs a = probe_args(problem, config, problem->dim);
        a.step = step;
        const size_t len = static_cast<size_t>(config->steps - step + 1) * problem->dim;
        DevBuf<double> d_out(static_cast<size_t>(n) * len);
        DevBuf<int> d_bad(1);
        cuda_check(cudaMemsetAsync(d_bad.p, 0, sizeof(int), st), "memset");
        cuda_check(launch_cloud_paths(a, first, n, d_out.p, d_bad.p, st), "k_cloud_paths");
        cuda_check(cudaStreamSynchronize(st), "paths");
        int bad = 0;
        cuda_check(cudaMemcpy(&bad, d_bad.p, sizeof bad, cudaMemcpyDeviceToHost), "D2H");
        cuda_check(cudaMemcpy(out, d_out.p, d_out.n * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
        if (bad) {
            Failure f{QRMC_ESIM, fmt("euler_step: state out of range at step %d", bad), bad};
            throw f;
        }
    });
}

}  // extern "C"

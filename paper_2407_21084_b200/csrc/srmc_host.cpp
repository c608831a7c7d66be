// srmc_host.cpp -- host side of the SRMC solver (include/qrmc_srmc.h): the plan that
// keeps every step's tables on the device, runs the backward loop (one kernel launch
// per step, srmc.cu) over this rank's hypercubes and all-gathers each step's table
// over NCCL (north_star item 5: "hypercubes are partitioned and each time step ends with
// an NCCL all-gather of the coefficient table"). No computation happens here.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>

#include "qrmc_gpu.h"
#include "qrmc_srmc.h"
#include "srmc_types.h"

using namespace qrmc_srmc_dev;

namespace {

struct Fail {
    int32_t status;
    std::string msg;
};
[[noreturn]] void fail(int32_t st, const std::string& m) { throw Fail{st, m}; }
void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(QRMC_ECUDA, std::string("CUDA: ") + cudaGetErrorString(e) + " (" + what + ")");
}

// NCCL, loaded lazily (the library itself does not link it; torch ships libnccl.so.2)
struct Nccl {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*Err)(ncclResult_t) = nullptr;
};
Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        for (const char* name : {"libnccl.so.2", "libnccl.so"})
            if ((n.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL))) break;
        if (!n.h) return;
        n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(dlsym(n.h, "ncclGetUniqueId"));
        n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(dlsym(n.h, "ncclCommInitRank"));
        n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(dlsym(n.h, "ncclCommDestroy"));
        n.AllGather = reinterpret_cast<decltype(n.AllGather)>(dlsym(n.h, "ncclAllGather"));
        n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(dlsym(n.h, "ncclAllReduce"));
        n.Err = reinterpret_cast<decltype(n.Err)>(dlsym(n.h, "ncclGetErrorString"));
    });
    if (!n.h || !n.GetUniqueId || !n.CommInitRank || !n.AllGather || !n.AllReduce)
        fail(QRMC_ENCCL, "libnccl.so.2 could not be loaded");
    return n;
}
void nk(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(QRMC_ENCCL, std::string(what) + ": " + (nccl().Err ? nccl().Err(r) : "error"));
}

template <class Fn>
int32_t guarded(char* err, size_t el, Fn&& fn) {
    try {
        fn();
        return QRMC_OK;
    } catch (const Fail& f) {
        set_err(err, el, f.msg.c_str());
        return f.status;
    } catch (const std::bad_alloc&) {
        set_err(err, el, "host allocation failed");
        return QRMC_ECAPACITY;
    }
}

void cell_range(int64_t cells, int rank, int world, int64_t& k0, int64_t& k1) {
    const int64_t per = (cells + world - 1) / world;
    k0 = std::min<int64_t>(cells, rank * per);
    k1 = std::min<int64_t>(cells, k0 + per);
}

}  // namespace

struct qrmc_srmc_plan {
    qrmc_srmc_problem_t prob{};
    qrmc_srmc_config_t cfg{};
    SrmcDev base{};
    int device = 0, rank = 0, world = 1, d = 1, P = 1, N = 1;
    bool zpass = false, keep_z = false, anyz = false;
    int64_t cells = 0, per = 0, rows = 0, k0 = 0, k1 = 0;
    cudaStream_t st = nullptr;
    ncclComm_t comm = nullptr;
    double *dy = nullptr, *dz = nullptr;  // [N][rows][P], [N][rows][d][P]
    int* dbad = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;

    ~qrmc_srmc_plan() {
        cudaSetDevice(device);
        if (dy) cudaFree(dy);
        if (dz) cudaFree(dz);
        if (dbad) cudaFree(dbad);
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
        if (comm) nccl().CommDestroy(comm);
        if (st) cudaStreamDestroy(st);
    }
};

namespace {

std::unique_ptr<qrmc_srmc_plan> make_plan(const qrmc_srmc_problem_t* prob, const qrmc_srmc_config_t* cfg, int device,
                                          int rank, int world, const void* id, bool keep_z) {
    char msg[256] = {0};
    const int rc = validate(prob, cfg, msg, sizeof msg);
    if (rc != QRMC_OK) fail(rc, msg);
    if (world < 1 || rank < 0 || rank >= world) fail(QRMC_EINVAL, "plan: bad rank/world");
    if (world > 1 && !id) fail(QRMC_EINVAL, "plan: world > 1 needs an NCCL unique id");
    auto P = std::make_unique<qrmc_srmc_plan>();
    P->prob = *prob;
    P->cfg = *cfg;
    P->device = device;
    P->rank = rank;
    P->world = world;
    P->d = prob->dim;
    P->P = cfg->basis == QRMC_SRMC_LP1 ? P->d + 1 : 1;
    P->N = cfg->steps;
    P->zpass = needs_z(prob);
    P->keep_z = keep_z;
    P->anyz = P->zpass || keep_z || cfg->want_z;
    P->base = make_dev(prob, cfg);
    {
        // Morton-ordered rows when the grid side is a power of two (srmc_types.h); the
        // download restores the lexicographic layout. QRMC_SRMC_MORTON=0 keeps row = cell.
        const int n = cfg->cells_per_dim;
        const char* e = std::getenv("QRMC_SRMC_MORTON");
        int bits = 0;
        while ((1 << bits) < n) ++bits;
        if (P->d > 1 && n > 1 && (n & (n - 1)) == 0 && bits <= P->d - 1 && P->d * bits <= 30 &&
            !(e && e[0] == '0')) {
            P->base.morton = 1;
            P->base.mbits = bits;
            for (int b = 0; b < bits; ++b) {
                P->base.mmul |= 1u << (b * (P->d - 1));
                P->base.mmask |= 1u << (b * P->d);
            }
        }
    }
    P->cells = P->base.cells;
    P->per = (P->cells + world - 1) / world;
    P->rows = P->per * world;
    cell_range(P->cells, rank, world, P->k0, P->k1);
    ck(cudaSetDevice(device), "cudaSetDevice");
    ck(cudaStreamCreateWithFlags(&P->st, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreate(&P->e0), "event");
    ck(cudaEventCreate(&P->e1), "event");
    const size_t ny = static_cast<size_t>(P->N) * P->rows * P->P;
    ck(cudaMalloc(&P->dy, ny * sizeof(double)), "cudaMalloc y tables");
    ck(cudaMemsetAsync(P->dy, 0, ny * sizeof(double), P->st), "memset");
    if (P->anyz) {
        const size_t nz = ny * P->d;
        ck(cudaMalloc(&P->dz, nz * sizeof(double)), "cudaMalloc z tables");
        ck(cudaMemsetAsync(P->dz, 0, nz * sizeof(double), P->st), "memset");
    }
    ck(cudaMalloc(&P->dbad, sizeof(int)), "cudaMalloc");
    if (world > 1) {
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof uid);
        nk(nccl().CommInitRank(&P->comm, world, uid, rank), "ncclCommInitRank");
    }
    ck(cudaStreamSynchronize(P->st), "plan sync");
    return P;
}

void run_plan(qrmc_srmc_plan& P, qrmc_srmc_stats_t* stats) {
    ck(cudaSetDevice(P.device), "cudaSetDevice");
    const size_t per_y = static_cast<size_t>(P.rows) * P.P, per_z = per_y * P.d;
    ck(cudaMemsetAsync(P.dbad, 0, sizeof(int), P.st), "memset");
    ck(cudaEventRecord(P.e0, P.st), "event");
    SrmcDev s = P.base;
    s.k0 = P.k0;
    s.k1 = P.k1;
    s.bad = P.dbad;
    int launches = 0;
    for (int i = P.N - 1; i >= 0; --i) {
        s.step = i;
        s.last = (i == P.N - 1);
        s.t = (i + 1) * s.dt;  // the driver is evaluated at (t_{i+1}, X_{i+1}, Y1, Zhat_i(X_i))
        s.decay = std::exp(((s.p[1] * s.p[1]) * static_cast<double>(P.d)) * (s.t - s.T) / 2.0);
        double* y = P.dy + per_y * i;
        ck(launch_step(P.d, P.P, s, s.last ? nullptr : P.dy + per_y * (i + 1), y, P.anyz ? P.dz + per_z * i : nullptr,
                       P.zpass, !P.zpass && P.anyz, P.st),
           "k_srmc_step");
        ++launches;
        if (P.world > 1) {
            // every endpoint may land in any rank's cells: the whole step table on every rank
            const size_t chunk = static_cast<size_t>(P.per) * P.P;
            nk(nccl().AllGather(y + chunk * P.rank, y, chunk, ncclDouble, P.comm, P.st), "ncclAllGather(y)");
        }
    }
    if (P.world > 1) {
        if (P.keep_z && P.dz) {
            const size_t chunk = static_cast<size_t>(P.per) * P.P * P.d;
            for (int i = 0; i < P.N; ++i)
                nk(nccl().AllGather(P.dz + per_z * i + chunk * P.rank, P.dz + per_z * i, chunk, ncclDouble, P.comm, P.st),
                   "ncclAllGather(z)");
        }
        nk(nccl().AllReduce(P.dbad, P.dbad, 1, ncclInt32, ncclMax, P.comm, P.st), "ncclAllReduce(flag)");
    }
    ck(cudaEventRecord(P.e1, P.st), "event");
    int bad = 0;
    ck(cudaMemcpyAsync(&bad, P.dbad, sizeof bad, cudaMemcpyDeviceToHost, P.st), "D2H");
    ck(cudaStreamSynchronize(P.st), "solve");
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, P.e0, P.e1), "event time");
    if (stats) {
        stats->path_steps = static_cast<uint64_t>(P.k1 - P.k0) * static_cast<uint64_t>(P.base.M) * P.N;
        stats->path_passes = P.zpass ? 2 : 1;
        stats->device_seconds = ms * 1e-3;
        stats->kernel_launches = launches;
    }
    if (bad) fail(QRMC_ENUMERIC, "non-finite SRMC coefficient");
}

void download(qrmc_srmc_plan& P, double* y, size_t y_len, double* z, size_t z_len) {
    const size_t per_y = static_cast<size_t>(P.cells) * P.P, rows_y = static_cast<size_t>(P.rows) * P.P;
    if (!y || y_len < per_y * P.N) fail(QRMC_EINVAL, "y buffer too small (steps * cells * P)");
    if (z && (!P.dz || z_len < per_y * P.d * P.N))
        fail(QRMC_EINVAL, P.dz ? "z buffer too small (steps * cells * d * P)" : "plan keeps no z tables");
    ck(cudaSetDevice(P.device), "cudaSetDevice");
    if (P.base.morton) {
        // back to lexicographic rows through one step-sized scratch table
        double* tmp = nullptr;
        ck(cudaMalloc(&tmp, per_y * (z ? P.d : 1) * sizeof(double)), "cudaMalloc download scratch");
        try {
            for (int i = 0; i < P.N; ++i) {
                ck(launch_unmorton(P.d, P.base.n, P.base.mbits, P.P, P.dy + rows_y * i, tmp, P.st), "k_unmorton");
                ck(cudaMemcpyAsync(y + per_y * i, tmp, per_y * sizeof(double), cudaMemcpyDeviceToHost, P.st), "D2H y");
                if (z) {
                    ck(launch_unmorton(P.d, P.base.n, P.base.mbits, P.P * P.d, P.dz + rows_y * P.d * i, tmp, P.st),
                       "k_unmorton");
                    ck(cudaMemcpyAsync(z + per_y * P.d * i, tmp, per_y * P.d * sizeof(double), cudaMemcpyDeviceToHost,
                                       P.st),
                       "D2H z");
                }
            }
            ck(cudaStreamSynchronize(P.st), "download");
        } catch (...) {
            cudaFree(tmp);
            throw;
        }
        cudaFree(tmp);
        return;
    }
    for (int i = 0; i < P.N; ++i) {
        ck(cudaMemcpyAsync(y + per_y * i, P.dy + rows_y * i, per_y * sizeof(double), cudaMemcpyDeviceToHost, P.st), "D2H y");
        if (z)
            ck(cudaMemcpyAsync(z + per_y * P.d * i, P.dz + rows_y * P.d * i, per_y * P.d * sizeof(double),
                               cudaMemcpyDeviceToHost, P.st),
               "D2H z");
    }
    ck(cudaStreamSynchronize(P.st), "download");
}

}  // namespace

extern "C" {

int32_t qrmc_srmc_nccl_unique_id(void* out128, char* err, size_t err_len) {
    return guarded(err, err_len, [&] {
        if (!out128) fail(QRMC_EINVAL, "null output");
        ncclUniqueId id;
        nk(nccl().GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(out128, &id, sizeof id);
    });
}

int32_t qrmc_srmc_plan_create(const qrmc_srmc_problem_t* prob, const qrmc_srmc_config_t* cfg, int32_t device,
                              int32_t rank, int32_t world, const void* nccl_unique_id, int32_t keep_z,
                              qrmc_srmc_plan_t** out, char* err, size_t err_len) {
    return guarded(err, err_len, [&] {
        if (!out) fail(QRMC_EINVAL, "null output");
        *out = make_plan(prob, cfg, device, rank, world, nccl_unique_id, keep_z != 0).release();
    });
}

int32_t qrmc_srmc_plan_run(qrmc_srmc_plan_t* plan, qrmc_srmc_stats_t* stats, char* err, size_t err_len) {
    return guarded(err, err_len, [&] {
        if (!plan) fail(QRMC_EINVAL, "null plan");
        run_plan(*plan, stats);
    });
}

int32_t qrmc_srmc_plan_download(qrmc_srmc_plan_t* plan, double* y, size_t y_len, double* z, size_t z_len, char* err,
                                size_t err_len) {
    return guarded(err, err_len, [&] {
        if (!plan) fail(QRMC_EINVAL, "null plan");
        download(*plan, y, y_len, z, z_len);
    });
}

void* qrmc_srmc_plan_stream(const qrmc_srmc_plan_t* plan) { return plan ? static_cast<void*>(plan->st) : nullptr; }

void qrmc_srmc_plan_destroy(qrmc_srmc_plan_t* plan) { delete plan; }

int32_t qrmc_srmc_cell_range(int64_t cells, int32_t rank, int32_t world, int64_t* k0, int64_t* k1) {
    if (cells < 0 || world < 1 || rank < 0 || rank >= world || !k0 || !k1) return QRMC_EINVAL;
    cell_range(cells, rank, world, *k0, *k1);
    return QRMC_OK;
}

int32_t qrmc_srmc_solve(const qrmc_srmc_problem_t* prob, const qrmc_srmc_config_t* cfg, double* y, size_t y_len,
                        double* z, size_t z_len, qrmc_srmc_stats_t* stats, char* err, size_t err_len) {
    return guarded(err, err_len, [&] {
        char msg[256] = {0};
        const int rc = validate(prob, cfg, msg, sizeof msg);
        if (rc != QRMC_OK) fail(rc, msg);
        const int P = cfg->basis == QRMC_SRMC_LP1 ? prob->dim + 1 : 1;
        int64_t cells = 1;
        for (int l = 0; l < prob->dim; ++l) cells *= cfg->cells_per_dim;
        const size_t per_y = static_cast<size_t>(cells) * P;
        if (!y || y_len < per_y * cfg->steps) fail(QRMC_EINVAL, "y buffer too small (steps * cells * P)");
        if (z && z_len < per_y * prob->dim * cfg->steps) fail(QRMC_EINVAL, "z buffer too small (steps * cells * d * P)");
        int dev = 0;
        ck(cudaGetDevice(&dev), "cudaGetDevice");
        auto plan = make_plan(prob, cfg, dev, 0, 1, nullptr, z != nullptr);
        run_plan(*plan, stats);
        download(*plan, y, y_len, z, z_len);
    });
}

}  // extern "C"

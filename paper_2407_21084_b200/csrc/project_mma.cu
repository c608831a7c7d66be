// project_mma.cu -- K2 (phase 2 of backward step i) on the FP64 tensor cores.
//
// Same contract as k_project in kernels.cu (proj/src/solver.cpp:180-199): per
// owned lane, partial[lane][k] = sum over the lane's paths m of S_m phi_k(X_m).
// With k = (u, s, b) as in responses_mma.cu and phi_k = sqrt2^{nnz(k)}
// U_u A_t (plain cosines),
//
//   G[u][t] = sum_m (S_m U_u(X_m)) A_t(X_m),   t < T_u,
//
// is a GEMM [groups x paths] x [paths x terms] with a staircase N extent, run
// as mma.sync.m8n8k4.f64 with M = 8 groups, N = 8 terms, K = 4 paths. Every
// warp owns one rectangle of ng x nt <= kProjTiles output tiles (host.cpp
// build_mma_layout) and keeps it in registers while the CTA streams the lane's
// paths through shared memory in batches of B = 24 (16 when the tables of 24 do not
// fit) paths: per batch, the cosine
// tables c_k(x_l) of every coordinate are built once ([entry][path] layout as in
// K1), then each warp forms its W = S * U fragments (per group block) and A
// fragments (per term block) and issues the DMMAs. The lane's sum over paths is
// thus a fixed-order tensor-core reduction: deterministic and independent of
// the GPU count (lanes never split across GPUs).
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"
#include "mma_common.cuh"
#include "qrmc_device.cuh"

namespace qrmc_dev {

namespace {

constexpr int kThreads = kProjWarps * 32;
#ifndef QRMC_PROJ_BRANCHLESS
#define QRMC_PROJ_BRANCHLESS 1
#endif
#ifndef QRMC_PROJ_TSPLIT
#define QRMC_PROJ_TSPLIT 4
#endif
constexpr int kTabSplit = QRMC_PROJ_TSPLIT;

// The batch loop's CTA barrier. Warps of one CTA run different project_rect shape
// instantiations, so they reach it from different code locations: a named barrier
// (id 1, all kThreads threads) is defined by its id and arrival count, which PTX
// specifies for exactly this case (unlike __syncthreads in divergent call sites).
__device__ __forceinline__ void batch_barrier() {
    asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory");
}

// batch geometry: B paths per batch, table row stride B + 4 (paths, padded). A chunk's
// last batch may be short (B need not divide kChunk): its missing paths read S = 0, so
// they add exact zeros and the path order of the tensor-core sum is the same for every B.
template <int B>
struct BatchGeom {
    static constexpr int kStride = B + 4;
    static constexpr int kPerChunk = (kChunk + B - 1) / B;
};

template <int B>
struct ProjSmem {
    double s[2][B];  // S_m of the batch (0 past the chunk's end)
    int second;      // split = 2: this CTA finished its lane's second half
    // followed by two cosine-table buffers [table_len][B + 4]
};

// batch b of the lane: chunk r = b / kPerChunk, paths [base, base + n)
struct Batch {
    int64_t q0, m0;  // owned index and path number of the first path
    int n;           // paths (<= 0: past the lane's end)
};

template <int B>
__device__ __forceinline__ Batch lane_batch(const StepArgs& a, int lane_rel, int b) {
    constexpr int kPerChunk = BatchGeom<B>::kPerChunk;
    const int64_t r = b / kPerChunk;
    const int base = (b % kPerChunk) * B;
    const int64_t c = static_cast<int64_t>(a.lane_lo + lane_rel) + r * kLanes;
    Batch bt;
    bt.q0 = (r * a.owned_lanes + lane_rel) * kChunk + base;
    bt.m0 = c * kChunk + base;
    int64_t rem = a.paths - bt.m0;
    if (rem > kChunk - base) rem = kChunk - base;
    bt.n = static_cast<int>(rem < B ? (rem < 0 ? 0 : rem) : B);
    return bt;
}

}  // namespace

// The batch loop of one warp shape: NG group blocks x up to 8 / NG term blocks.
template <int D, int NG, bool GEN, int B>
__device__ __forceinline__ void project_rect(const StepArgs& a, const ProjMmaArgs& p, ProjSmem<B>& sm, double* tabs0,
                                             size_t tab_elems, int lane_rel, int slot, int4 rc) {
    constexpr int NT = kProjTiles / NG;
    constexpr int kStride = BatchGeom<B>::kStride;
    constexpr int kProjBatch = B;
    const int tid = threadIdx.x, lane = tid & 31;
    const int gb0 = rc.x, tb0 = rc.y, nt = rc.z >> 8;
    const int row = lane >> 2, col = lane & 3;
    // the lane's fixed operand rows (K1's offsets are rows x kMmaTabStride):
    // group u = 8 (gb0 + ig) + row, term t = 8 (tb0 + it) + row
    int gro[NG][D - 2];
#pragma unroll
    for (int ig = 0; ig < NG; ++ig)
#pragma unroll
        for (int l = 0; l < D - 2; ++l) gro[ig][l] = __ldg(&p.gk[(8 * (gb0 + ig) + row) * (D - 2) + l]) / kMmaTabStride * kStride;
    int ts_[NT], tb_[NT];
#pragma unroll
    for (int it = 0; it < NT; ++it) {
        const uint32_t v = it < nt ? __ldg(&p.terms[8 * (tb0 + it) + row]) : 0u;
        ts_[it] = static_cast<int>(v & 0xFFFFu) / kMmaTabStride * kStride;
        tb_[it] = static_cast<int>(v >> 16) / kMmaTabStride * kStride;
    }
    double acc[NG][NT][2];
#pragma unroll
    for (int ig = 0; ig < NG; ++ig)
#pragma unroll
        for (int it = 0; it < NT; ++it) acc[ig][it][0] = acc[ig][it][1] = 0.0;

    // table task of this thread: path pt, piece q, coordinate l
    constexpr int TS = kTabSplit * kProjBatch * D <= kThreads ? kTabSplit : kThreads / (kProjBatch * D);
    constexpr int kTasks = TS * kProjBatch * D;
    const int pt = tid % kProjBatch, tq = (tid / kProjBatch) % TS, tl = tid / (kProjBatch * TS);
    const int64_t chunks_total = (a.paths + kChunk - 1) / kChunk;
    const int64_t my_chunks = (chunks_total - (a.lane_lo + lane_rel) + kLanes - 1) / kLanes;
    const int n_batches = static_cast<int>(my_chunks) * BatchGeom<B>::kPerChunk;
    // split = 2: half z takes chunks [0, ceil(c/2)) or the rest (a chunk boundary, so the
    // halves -- and the bits -- do not depend on the batch width B)
    const int half = blockIdx.z;
    const int hb = static_cast<int>((my_chunks + 1) / 2) * BatchGeom<B>::kPerChunk;
    const int b_lo = p.split == 2 && half == 1 ? hb : 0;
    const int b_hi = p.split == 2 && half == 0 ? hb : n_batches;
    // cos theta_l (and S) of this thread's task in batch b, fetched a batch ahead
    auto fetch = [&](int b, double& c1, double& sv) {
        c1 = 1.0;
        sv = 0.0;
        if (b >= b_hi || tid >= kTasks) return;
        {
            const Batch bt = lane_batch<B>(a, lane_rel, b);
            if (pt >= bt.n) return;
            if (a.cloud && a.cloud_cos) {
                c1 = a.cloud[tl * a.n_owned + bt.q0 + pt];
            } else {
                double xl;
                if (a.cloud) {
                    xl = a.cloud[tl * a.n_owned + bt.q0 + pt];
                } else {
                    // recompute-from-seeds (solver.cpp:187-193): regenerate X_i
                    xl = measure_inv_cdf<GEN>(a.meas,
                                         u64_to_uniform(stream_u64_at(
                                             a.seed, sid_training(a.step, static_cast<uint64_t>(bt.m0 + pt)), tl)),
                                         tl);
                }
                c1 = cos(DMUL(3.14159265358979323846, measure_cdf<GEN>(a.meas, xl, tl)));
            }
            if (tq == 0 && tl == 0) sv = a.resp[bt.q0 + pt];
        }
    };
    auto build = [&](int buf, double c1, double sv) {
        if (tid >= kTasks) return;
#ifndef QRMC_PROJ_EXP_NOTAB  // timing experiments only (wrong results)
        cos_table_piece_c(c1, p.kmax[tl], tq, TS, tabs0 + buf * tab_elems + p.offset[tl] * kStride + pt, kStride);
#endif
        if (tq == 0 && tl == 0) sm.s[buf][pt] = sv;
    };

    double cn, sn;
    fetch(b_lo, cn, sn);
    build(0, cn, sn);
    fetch(b_lo + 1, cn, sn);
    batch_barrier();
    for (int b = b_lo; b < b_hi; ++b) {
        const int buf = (b - b_lo) & 1;
        // tables of batch b+1 (other buffer) while the tensor cores take batch b
        if (b + 1 < b_hi) {
            build(buf ^ 1, cn, sn);
            fetch(b + 2, cn, sn);
        }
        const double* tb = tabs0 + buf * tab_elems;
        // K = 4 paths per DMMA: path 4 ks + col of the batch
#pragma unroll
        for (int ks = 0; ks < kProjBatch / 4; ++ks) {
            const int m = 4 * ks + col;
            const double* tm = tb + m;
            const double sv = sm.s[buf][m];
            double w[NG];
#pragma unroll
            for (int ig = 0; ig < NG; ++ig) {
                double u = DMUL(sv, tm[gro[ig][0]]);
#pragma unroll
                for (int l = 1; l < D - 2; ++l) u = DMUL(u, tm[gro[ig][l]]);
                w[ig] = u;
            }
#if QRMC_PROJ_BRANCHLESS
            // every tile of the shape runs (tiles past nt read row 0 and are never
            // written out): no data-dependent branch around mma.sync, so no
            // warp re-convergence before each DMMA
#pragma unroll
            for (int it = 0; it < NT; ++it) {
                const double bv = DMUL(tm[ts_[it]], tm[tb_[it]]);
#pragma unroll
                for (int ig = 0; ig < NG; ++ig) dmma(acc[ig][it], w[ig], bv);
            }
#else
#pragma unroll
            for (int it = 0; it < NT; ++it) {
                if (NT == 1 || it < nt) {
                    const double bv = DMUL(tm[ts_[it]], tm[tb_[it]]);
#pragma unroll
                    for (int ig = 0; ig < NG; ++ig) dmma(acc[ig][it], w[ig], bv);
                }
            }
#endif
        }
        batch_barrier();
    }
    // partial[lane][k] = sqrt2^{nnz(k)} G[u][t]
    double* out = p.partials + static_cast<int64_t>(lane_rel) * p.basis_size;
    const int32_t* om = p.out + static_cast<int64_t>(slot) * kProjTiles * 64;
    if (p.split == 2) {
        // both halves park their tiles; the CTA that arrives second writes half 0 + half 1
        const size_t cta_vals = static_cast<size_t>(kProjWarps) * kProjTiles * 64;
        const size_t at = (static_cast<size_t>(lane_rel) * gridDim.x + blockIdx.x) * cta_vals +
                          static_cast<size_t>(threadIdx.x >> 5) * kProjTiles * 64;
        const size_t half_vals = static_cast<size_t>(gridDim.y) * gridDim.x * cta_vals;
        double* mine = p.scratch + half * half_vals + at;
#pragma unroll
        for (int ig = 0; ig < NG; ++ig)
#pragma unroll
            for (int it = 0; it < NT; ++it)
                if (it < nt) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) mine[(ig * nt + it) * 64 + lane * 2 + h] = acc[ig][it][h];
                }
        __threadfence();
        batch_barrier();
        if (threadIdx.x == 0) {
            int* ctr = p.counters + static_cast<size_t>(lane_rel) * gridDim.x + blockIdx.x;
            const int old = atomicAdd(ctr, 1);
            sm.second = old == 1;
            if (old == 1) *ctr = 0;  // both halves are in: ready for the next launch
        }
        batch_barrier();
        if (!sm.second) return;
        __threadfence();
        const double* h0 = p.scratch + at;
        const double* h1 = p.scratch + half_vals + at;
#pragma unroll
        for (int ig = 0; ig < NG; ++ig)
#pragma unroll
            for (int it = 0; it < NT; ++it)
                if (it < nt) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int k = __ldg(&om[(ig * nt + it) * 64 + lane * 2 + h]);
                        const int e = (ig * nt + it) * 64 + lane * 2 + h;
                        if (k >= 0) out[k] = DMUL(DADD(__ldcg(h0 + e), __ldcg(h1 + e)), __ldg(&p.scale[k]));
                    }
                }
        return;
    }
#pragma unroll
    for (int ig = 0; ig < NG; ++ig)
#pragma unroll
        for (int it = 0; it < NT; ++it)
            if (it < nt) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int k = __ldg(&om[(ig * nt + it) * 64 + lane * 2 + h]);
                    if (k >= 0) out[k] = DMUL(acc[ig][it][h], __ldg(&p.scale[k]));
                }
            }
}

template <int D, bool GEN, int B>
#ifndef QRMC_PROJ_MINB
#define QRMC_PROJ_MINB 1
#endif
__global__ void __launch_bounds__(kThreads, QRMC_PROJ_MINB) k_project_mma(const StepArgs a, const ProjMmaArgs p) {
    static_assert(D >= 3, "the tensor-core K2 needs an upper prefix");
    static_assert(B % 4 == 0 && kChunk % 4 == 0, "batches of whole k-steps inside chunks");
    static_assert(B * D <= kThreads, "one table task per thread");
    extern __shared__ __align__(16) unsigned char dsm[];
    ProjSmem<B>& sm = *reinterpret_cast<ProjSmem<B>*>(dsm);
    double* tabs0 = reinterpret_cast<double*>(dsm + ((sizeof(ProjSmem<B>) + 15) & ~size_t{15}));
    const size_t tab_elems = static_cast<size_t>(p.table_len) * BatchGeom<B>::kStride;
    const int warp = threadIdx.x >> 5;
    const int part = blockIdx.x, lane_rel = blockIdx.y;
    const int slot = part * kProjWarps + warp;
    const int4 rc = __ldg(&p.rects[slot]);
    // every warp runs the same batch loop (named barrier batch_barrier); the shape
    // only sets its register tile. Empty slots carry tiles = 0 and write nothing.
    switch (rc.z & 0xFF) {
        case 16:
            if constexpr (kProjTiles >= 16) project_rect<D, 16, GEN, B>(a, p, sm, tabs0, tab_elems, lane_rel, slot, rc);
            break;
        case 8:
            if constexpr (kProjTiles >= 8) project_rect<D, 8, GEN, B>(a, p, sm, tabs0, tab_elems, lane_rel, slot, rc);
            break;
        case 4:
            if constexpr (kProjTiles >= 4) project_rect<D, 4, GEN, B>(a, p, sm, tabs0, tab_elems, lane_rel, slot, rc);
            break;
        case 2:
            if constexpr (kProjTiles >= 2) project_rect<D, 2, GEN, B>(a, p, sm, tabs0, tab_elems, lane_rel, slot, rc);
            break;
        default: project_rect<D, 1, GEN, B>(a, p, sm, tabs0, tab_elems, lane_rel, slot, rc); break;
    }
}

template <int B>
static size_t smem_bytes_b(int table_len) {
    return ((sizeof(ProjSmem<B>) + 15) & ~size_t{15}) +
           2 * static_cast<size_t>(BatchGeom<B>::kStride) * table_len * sizeof(double);
}

size_t project_mma_smem_bytes(int table_len, int batch) {
    return batch == kProjBatchWide ? smem_bytes_b<kProjBatchWide>(table_len) : smem_bytes_b<kProjBatchNarrow>(table_len);
}

int project_mma_batch(int table_len, size_t optin) {
    if (smem_bytes_b<kProjBatchWide>(table_len) <= optin) return kProjBatchWide;
    if (smem_bytes_b<kProjBatchNarrow>(table_len) <= optin) return kProjBatchNarrow;
    return 0;
}

template <int D, int B, class Fn>
static cudaError_t with_project_kernel_b(bool gen, Fn&& fn) {
    return gen ? fn(k_project_mma<D, true, B>) : fn(k_project_mma<D, false, B>);
}

template <class Fn>
static cudaError_t with_project_kernel(int dim, int batch, bool gen, Fn&& fn) {
    const bool wide = batch == kProjBatchWide;
    switch (dim) {
        case 3: return wide ? with_project_kernel_b<3, kProjBatchWide>(gen, fn) : with_project_kernel_b<3, kProjBatchNarrow>(gen, fn);
        case 4: return wide ? with_project_kernel_b<4, kProjBatchWide>(gen, fn) : with_project_kernel_b<4, kProjBatchNarrow>(gen, fn);
        case 5: return wide ? with_project_kernel_b<5, kProjBatchWide>(gen, fn) : with_project_kernel_b<5, kProjBatchNarrow>(gen, fn);
        case 6: return wide ? with_project_kernel_b<6, kProjBatchWide>(gen, fn) : with_project_kernel_b<6, kProjBatchNarrow>(gen, fn);
        case 7: return wide ? with_project_kernel_b<7, kProjBatchWide>(gen, fn) : with_project_kernel_b<7, kProjBatchNarrow>(gen, fn);
        case 8: return wide ? with_project_kernel_b<8, kProjBatchWide>(gen, fn) : with_project_kernel_b<8, kProjBatchNarrow>(gen, fn);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t configure_project_mma(int dim, int batch, size_t smem) {
    auto set = [&](auto kern) {
        return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    };
    const cudaError_t e = with_project_kernel(dim, batch, false, set);
    return e != cudaSuccess ? e : with_project_kernel(dim, batch, true, set);
}

cudaError_t launch_project_mma(const StepArgs& a, const ProjMmaArgs& p, cudaStream_t st) {
    if (a.owned_lanes == 0 || p.parts == 0) return cudaSuccess;
    const dim3 grid(static_cast<unsigned>(p.parts), static_cast<unsigned>(a.owned_lanes),
                    static_cast<unsigned>(p.split == 2 ? 2 : 1));
    return with_project_kernel(a.prob.dim, p.batch, a.meas.form == 3, [&](auto kern) {
        kern<<<grid, kThreads, project_mma_smem_bytes(p.table_len, p.batch), st>>>(a, p);
        return cudaGetLastError();
    });
}

}  // namespace qrmc_dev

// responses_mma.cu -- K1 (phase 1 of backward step i) on the FP64 tensor cores.
//
// Same contract as k_responses in kernels.cu (proj/src/solver.cpp:147-177):
// per path m, draw X_i ~ nu, Euler to N, evaluate every future series
// alpha_{j+1} at X_{j+1}, truncate, accumulate the driver, emit S_m.
//
// The series sum is restructured as a GEMM. Write k = (u, s, b) with u the
// upper prefix (k_0..k_{D-3}), s = k_{D-2}, b = k_{D-1}. For the index sets the
// solver builds (full, total degree, hyperbolic), the (s, b) sets of the groups
// u form a chain, so with one shared order of the (s, b) pairs every group is a
// prefix of length T_u (host.cpp build_mma_layout verifies this). Then
//
//   y(x) = sum_u U_u(x) C_u(x),  U_u = prod_{l<D-2} c_{k_l}(x_l),
//   C_u(x) = sum_{t < T_u} A_t(x) alpha'_{u,t},  A_t = c_{s_t}(x_{D-2}) c_{b_t}(x_{D-1}),
//
// and C = A * alpha' is a dense GEMM [paths x terms] x [terms x groups] with a
// staircase K extent, run as mma.sync.m8n8k4.f64 (8 paths x 8 groups x 4
// terms). The host sorts groups by T_u, cuts them into 8-group column blocks
// of 4-term chunks, and forms units (<= kMmaBundle column blocks of equal chunk
// count x a chunk range of <= kMmaKSplit) balanced over the warps. Each warp
// runs the DMMAs of its units for all the CTA's paths and folds C into y
// through U at the end of every unit (C is linear in the chunk range, so a
// column block can be split across warps with no reduction of C). Each warp
// streams its own B fragments (32 doubles in lane order) through a private
// shared-memory ring with cp.async, so the GEMM phase has no CTA barrier; the
// per-path cosine tables c_k(x_l), k <= kmax_l, live in shared memory.
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>
#include <cstdio>

#include "kernels.cuh"
#include "qrmc_device.cuh"
#include "mma_common.cuh"
#include "series_block.cuh"

namespace qrmc_dev {

namespace {

constexpr int kThreads = kMmaWarps * 32;

// clock read that stays in place relative to barriers (phase timing experiments)
__device__ __forceinline__ long long clk_fenced() {
    long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)::"memory");
    return t;
}
// CTA barrier whose release is observed: the clock read depends on its result
__device__ __forceinline__ long long sync_clk() {
    const int n = __syncthreads_count(1);
    long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t) : "r"(n) : "memory");
    return t;
}
#ifndef QRMC_MMA_AHEAD
#define QRMC_MMA_AHEAD 2
#endif
#ifndef QRMC_MMA_UNROLL4
#define QRMC_MMA_UNROLL4 1
#endif
#ifndef QRMC_MMA_TSPLIT
#define QRMC_MMA_TSPLIT 1
#endif
constexpr int kTabSplit = QRMC_MMA_TSPLIT;  // recurrence pieces per (path, coordinate) table

template <int D>
struct MmaSmem {
    double ring[kMmaWarps][kMmaRingFrags * 32];
    double x[2][kMmaPaths][D];  // X_j and X_{j+1}, alternating
    double theta[kMmaPaths][D];
    double w0[kMmaPaths], dsum[kMmaPaths];
    double wq[2][kMmaPaths], lq[2][kMmaPaths], dpre[2][kMmaPaths], term[kMmaPaths];  // x-only parts, by evaluation parity
    double ypart[kMmaWarps][kMmaPaths];
    int bad[kMmaPaths];
    int abort;
    // followed by the cosine tables [table_len][kTabStride] (c_k(x_l) of path p at
    // (offset_l + k) * kTabStride + p)
};

template <int D>
__device__ __forceinline__ double* mma_tables(unsigned char* base) {
    return reinterpret_cast<double*>(base + ((sizeof(MmaSmem<D>) + 15) & ~size_t{15}));
}

// A warp's private fragment stream: series s = 0..n_series-1 (alpha_{i+1+s}),
// each the warp's `frags` fragments (a multiple of kMmaRingFrags; no unit step
// straddles a ring wrap), copied in batches of kMmaBatch through a ring of
// kMmaRingBatches slots.
struct WarpStream {
    const double* src;  // alpha + (i+1) * row_len + frag_offset * 32
    int64_t row_len;
    double* ring;
    uint32_t per;       // batches per series
    uint32_t total;     // batches over all series
    uint32_t issued, landed;
    uint32_t ready;     // fragments landed: landed * kMmaBatch
    uint32_t refill_at; // stream position that frees the next slot
    uint32_t b_in;      // next batch's index inside its series
    const double* next; // next batch's source
    int lane;

    __device__ __forceinline__ void issue() {
        double* d = ring + (issued % kMmaRingBatches) * (kMmaBatch * 32);
#pragma unroll
        for (int c = 0; c < kMmaBatch * 32 / 2 / 32; ++c)
            cp_async16(d + 2 * (c * 32 + lane), next + 2 * (c * 32 + lane));
        cp_async_commit();
        ++issued;
        refill_at += kMmaBatch;
        next += kMmaBatch * 32;
        if (++b_in == per) {  // next series: alpha_{j+2} of the same warp's stream
            b_in = 0;
            src += row_len;
            next = src;
        }
    }
    // make fragments [.., upto) visible to the whole warp
    __device__ __forceinline__ void land(uint32_t upto) {
        if (upto <= ready) return;
        // batches [0, need) must have landed: allow issued - need to stay in flight
        const uint32_t need = (upto + kMmaBatch - 1) / kMmaBatch;
        switch (issued - need) {
            case 0: cp_async_wait<0>(); break;
            case 1: cp_async_wait<1>(); break;
            case 2: cp_async_wait<2>(); break;
            default: cp_async_wait<3>(); break;
        }
        landed = need;
        ready = need * kMmaBatch;
        __syncwarp();
    }
    // fragments below `consumed` are read: refill the freed slots
    __device__ __forceinline__ void refill(uint32_t consumed) {
        if (consumed >= refill_at && issued < total) {
            __syncwarp();
            do issue(); while (consumed >= refill_at && issued < total);
        }
    }
};

// one unit: NB column blocks x chunks [c0, c1), then y += U * C. Tables are
// laid out [k][path] with stride kTabStride, the ring as [frag][lane].
constexpr int kTabStride = kMmaTabStride;

template <int D, int NB>
__device__ __forceinline__ void run_unit(const MmaArgs& m, int cb0, int c0, int c1, uint32_t& fpos, WarpStream& ws,
                                         const double* tab, int lane, double (&y)[kMmaRowBlocks]) {
    constexpr int RB = kMmaRowBlocks;
    const int row = lane >> 2, col = lane & 3;
    double acc[RB][NB][2];  // written first by the unit's first chunk (C = 0)
    const double* trow = tab + row;
    const double* ring = ws.ring + lane;
    const uint32_t* term = m.terms + 4 * c0 + col;
    auto step = [&](auto first, uint32_t f) {
        const uint32_t tp = __ldg(term);
        term += 4;
        const double* ps = trow + (tp & 0xFFFFu);
        const double* pb = trow + (tp >> 16);
        double a[RB];
#pragma unroll
        for (int r = 0; r < RB; ++r) a[r] = DMUL(ps[8 * r], pb[8 * r]);
        const double* rb = ring + (f % kMmaRingFrags) * 32;
        double b[NB];
#pragma unroll
        for (int i = 0; i < NB; ++i) b[i] = rb[32 * i];
#pragma unroll
        for (int i = 0; i < NB; ++i)
#pragma unroll
            for (int r = 0; r < RB; ++r) {
                if constexpr (decltype(first)::value)
                    dmma0(acc[r][i], a[r], b[i]);
                else
                    dmma(acc[r][i], a[r], b[i]);
            }
    };
    constexpr uint32_t W = NB == 3 ? 4 : NB;  // fragment slots per step (host.cpp build_mma_layout)
    static_assert((QRMC_MMA_UNROLL4 ? 4 : 2) * W + kMmaBatch - 1 <= kMmaRingFrags,
                  "the ring must hold a whole step group past any batch boundary");
    fpos = (fpos + W - 1) / W * W;
    // the first chunk starts the accumulators
    ws.land(fpos + W);
    step(std::true_type{}, fpos);
    fpos += W;
    ws.refill(fpos);
    int c = c0 + 1;
#if QRMC_MMA_UNROLL4
    for (; c + 3 < c1; c += 4) {
        ws.land(fpos + 4 * W);
        step(std::false_type{}, fpos);
        step(std::false_type{}, fpos + W);
        step(std::false_type{}, fpos + 2 * W);
        step(std::false_type{}, fpos + 3 * W);
        fpos += 4 * W;
        ws.refill(fpos);
    }
#endif
    for (; c + 1 < c1; c += 2) {
        ws.land(fpos + 2 * W);
        step(std::false_type{}, fpos);
        step(std::false_type{}, fpos + W);
        fpos += 2 * W;
        ws.refill(fpos);
    }
    if (c < c1) {
        ws.land(fpos + W);
        step(std::false_type{}, fpos);
        fpos += W;
        ws.refill(fpos);
    }
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        // the lane's two groups g, g+1 (g even) have adjacent prefix rows:
        // 2 (D-2) u16 = (D-2) aligned u32 words
        const int g0 = 8 * (cb0 + i) + 2 * col;
        uint32_t wpair[D - 2];
        const uint32_t* gw = reinterpret_cast<const uint32_t*>(m.gk + g0 * (D - 2));
#pragma unroll
        for (int w = 0; w < D - 2; ++w) wpair[w] = __ldg(gw + w);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const double* pu[D - 2];
#pragma unroll
            for (int l = 0; l < D - 2; ++l) {
                const int e = h * (D - 2) + l;  // u16 entry of the pair
                pu[l] = trow + ((wpair[e >> 1] >> (16 * (e & 1))) & 0xFFFFu);
            }
#pragma unroll
            for (int r = 0; r < RB; ++r) {
                double u = pu[0][8 * r];
#pragma unroll
                for (int l = 1; l < D - 2; ++l) u = DMUL(u, pu[l][8 * r]);
                y[r] = fma(u, acc[r][i][h], y[r]);
            }
        }
    }
}

}  // namespace

template <int D, bool GEN>
#ifndef QRMC_MMA_MINB
#define QRMC_MMA_MINB 1
#endif
__global__ void __launch_bounds__(kThreads, QRMC_MMA_MINB) k_responses_mma(const StepArgs a, const MmaArgs m) {
    static_assert(D >= 3, "the tensor-core K1 needs an upper prefix");
    static_assert(kMmaPaths * D <= kThreads, "one (path, coordinate) task per thread");
    static_assert(kMmaPaths <= 32, "warp 0 holds every path's truncation counters");
    // threads that run ahead during the GEMM phase (Euler tasks, x-only parts)
    constexpr int kAheadThreads = ((kMmaPaths * D > 3 * kMmaPaths ? kMmaPaths * D : 3 * kMmaPaths) + 31) / 32 * 32;
    static_assert(kAheadThreads <= kThreads, "ahead group fits the CTA");
    extern __shared__ __align__(16) unsigned char dsm[];
    MmaSmem<D>& sm = *reinterpret_cast<MmaSmem<D>*>(dsm);
    double* tabs = mma_tables<D>(dsm);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) sm.abort = *a.abort_flag;
    __syncthreads();
    if (sm.abort) return;

    const int64_t q0 = static_cast<int64_t>(blockIdx.x) * kMmaPaths;
    const int4 wi = __ldg(&m.warp_info[warp]);  // {unit_begin, unit_end, frag_offset, frags}
    WarpStream ws;
    ws.src = m.alpha + static_cast<int64_t>(a.step + 1) * m.row_len + static_cast<int64_t>(wi.z) * 32;
    ws.row_len = m.row_len;
    ws.ring = sm.ring[warp];
    ws.per = static_cast<uint32_t>(wi.w) / kMmaBatch;
    ws.total = static_cast<uint32_t>(a.steps - 1 - a.step) * ws.per;
    ws.issued = 0;
    ws.landed = 0;
    ws.ready = 0;
    ws.refill_at = 0;
    ws.b_in = 0;
    ws.next = ws.src;
    ws.lane = lane;
    while (ws.issued < ws.total && ws.issued < kMmaRingBatches) ws.issue();
    ws.refill_at = kMmaBatch;  // batch kMmaRingBatches reuses the first slot

    // start points X_i ~ nu: draws 0..D-1 of the path's stream (solver.cpp:150-152)
    const int tp = tid / D, tl = tid % D;
    const bool task = tid < kMmaPaths * D;
    const int64_t tq = q0 + tp;
    const uint64_t tsid = sid_training(a.step, static_cast<uint64_t>(owned_path(a, tq < a.n_owned ? tq : 0)));
    if (task) {
        const double x = measure_inv_cdf<GEN>(a.meas, u64_to_uniform(stream_u64_at(a.seed, tsid, tl)), tl);
        sm.x[0][tp][tl] = x;
        if (a.cloud && tq < a.n_owned)
            a.cloud[tl * a.n_owned + tq] = a.cloud_cos ? cos(DMUL(3.14159265358979323846, measure_cdf<GEN>(a.meas, x, tl))) : x;
    }
    __syncthreads();
    uint32_t apps = 0, clipped = 0;
    if (tid < kMmaPaths) {
        double x[D];
#pragma unroll
        for (int l = 0; l < D; ++l) x[l] = sm.x[0][tid][l];
        sm.w0[tid] = damping_weight<D>(x, a.q);
        sm.dsum[tid] = 0.0;
        sm.bad[tid] = 0;
    }
    __syncthreads();

    // Euler step jj of coordinate tl (sde.cpp:37-73): X_{jj+1} from X_jj, draw
    // D + (jj-i)*D + tl of the path's stream, and theta_l(X_{jj+1}) when alpha_{jj+1}
    // is evaluated there. Independent of the series values: it runs ahead.
    auto euler = [&](int jj) {
        if (task) {
            const int src = (jj - a.step) & 1;
            const double nrm = qrmc_normal_quantile(
                u64_to_uniform(stream_u64_at(a.seed, tsid, static_cast<uint64_t>(D) * (jj - a.step + 1) + tl)));
            const double dw = DMUL(a.sqrt_dt, nrm);
            const double xo = sm.x[src][tp][tl];
            const double v = euler_coord(a.prob, xo, dw, tl, a.dt);
            sm.x[src ^ 1][tp][tl] = v;
            if ((!isfinite(v) || fabs(v) > a.prob.state_bound) && sm.bad[tp] == 0) sm.bad[tp] = jj + 1;
            if (jj + 1 < a.steps) sm.theta[tp][tl] = DMUL(3.14159265358979323846, measure_cdf<GEN>(a.meas, v, tl));
        }
    };
    // x-only parts of evaluation jj (path p), one kind per task so that the
    // transcendental functions run on different warps: 0 weight at X_{jj+1}
    // (terminal value at X_N), 1 truncation bound at X_{jj+1}, 2 the driver's
    // x-part at X_jj
    auto path_part = [&](int jj, int p, int kind) {
        const int c = (jj - a.step) & 1;
        double xv[D];
#pragma unroll
        for (int l = 0; l < D; ++l) xv[l] = sm.x[kind == 2 ? c : c ^ 1][p][l];
        if (kind == 0) {
            if (jj + 1 == a.steps)
                sm.term[p] = terminal<D>(a.prob, xv);
            else
                sm.wq[c][p] = damping_weight<D>(xv, a.q);
        } else if (kind == 1) {
            sm.lq[c][p] = lstar<D>(a.prob, xv);
        } else {
            sm.dpre[c][p] = driver_pre<D>(a.prob, DMUL(static_cast<double>(jj), a.dt), xv);
        }
    };
    // truncation + driver of evaluation jj (solver.cpp:160-172) for path p
    auto finish_eval = [&](int jj, int p) {
        const int c = (jj - a.step) & 1;
        double y;
        if (jj + 1 == a.steps) {
            y = sm.term[p];  // exact initialisation at the terminal step (solver.cpp:69-72)
        } else {
            double ys = 0.0;
#pragma unroll
            for (int w = 0; w < kMmaWarps; ++w) ys += sm.ypart[w][p];
            y = DMUL(ys, sm.wq[c][p]);
        }
        const double cv = truncate_soft(y, sm.lq[c][p]);
        if (q0 + p < a.n_owned) {
            ++apps;
            if (cv != y) ++clipped;
        }
        sm.dsum[p] = DADD(sm.dsum[p], driver_apply(a.prob, sm.dpre[c][p], cv));
    };
    // one phase: finish evaluation jj_fin, the x-only parts of evaluation
    // jj_parts, and the cosine tables c_k(x_l) = cos(k theta_l) of evaluation
    // jj_tab (kTabSplit Chebyshev pieces per (path, coordinate); lanes on
    // consecutive paths: conflict-free [k][path] stores). Every 32-task group is
    // one warp's work.
    auto tables_and_paths = [&](int jj_tab, int jj_fin, int jj_parts) {
        constexpr int kPathTasks = 4 * kMmaPaths;
#ifndef QRMC_MMA_SKIP_TABLES  // timing experiments only
        const int n_tab = jj_tab >= 0 ? kTabSplit * kMmaPaths * D : 0;
#else
        const int n_tab = 0;
#endif
        for (int t = tid; t < kPathTasks + n_tab; t += kThreads) {
            if (t < kPathTasks) {
                // finish on warp 0 (it holds the truncation counters), parts on warps 1-3
                const int p = t % kMmaPaths, kind = t / kMmaPaths;
                if (kind == 0) {
                    if (jj_fin >= 0) finish_eval(jj_fin, p);
                } else if (jj_parts >= 0) {
                    path_part(jj_parts, p, kind - 1);
                }
                continue;
            }
            const int tt = t - kPathTasks;
            const int p = tt % kMmaPaths, q = (tt / kMmaPaths) % kTabSplit, l = tt / (kMmaPaths * kTabSplit);
            cos_table_piece(sm.theta[p][l], m.kmax[l], q, kTabSplit, tabs + m.offset[l] * kTabStride + p, kTabStride);
        }
    };

    euler(a.step);
    __syncthreads();
    tables_and_paths(a.step + 1 < a.steps ? a.step : -1, -1, a.step);
    __syncthreads();
#ifdef QRMC_MMA_PHASE_CLOCKS
    long long acc_own = 0, acc_gemm = 0, acc_tab = 0;
    const long long c_k0 = clk_fenced();
#endif
    for (int j = a.step; j < a.steps; ++j) {
        if (j + 1 < a.steps) {
            // evaluation of alpha_{j+1} at X_{j+1}. The first kAheadThreads threads
            // first run the next Euler step and the x-only parts of the next
            // evaluation (the host gives their warps correspondingly less GEMM work)
#ifdef QRMC_MMA_PHASE_CLOCKS
            const long long c_g0 = clk_fenced();
#endif
#if QRMC_MMA_AHEAD >= 1
            if (tid < kAheadThreads) {
                euler(j + 1);
#if QRMC_MMA_AHEAD >= 2
                asm volatile("bar.sync 1, %0;" ::"n"(kAheadThreads) : "memory");
                if (tid < 3 * kMmaPaths) path_part(j + 1, tid % kMmaPaths, tid / kMmaPaths);
#endif
            }
#endif
            double y[kMmaRowBlocks];
#pragma unroll
            for (int r = 0; r < kMmaRowBlocks; ++r) y[r] = 0.0;
            uint32_t fpos = static_cast<uint32_t>(j - a.step) * static_cast<uint32_t>(wi.w);  // stream position of this series
            ws.refill(fpos);  // the previous series' padding counts as consumed
#ifndef QRMC_MMA_SKIP_GEMM  // timing experiments only: phases without the GEMM
            for (int u = wi.x; u < wi.y; ++u) {
#else
            for (int u = wi.x; u < wi.x; ++u) {
#endif
                const int4 un = __ldg(&m.units[u]);
                if (un.y == 1) {
                    run_unit<D, 1>(m, un.x, un.z, un.w, fpos, ws, tabs, lane, y);
                } else if constexpr (kMmaBundle == 2) {
                    run_unit<D, 2>(m, un.x, un.z, un.w, fpos, ws, tabs, lane, y);
                } else if constexpr (kMmaBundle > 2) {
                    switch (un.y) {
                        case 2: run_unit<D, 2>(m, un.x, un.z, un.w, fpos, ws, tabs, lane, y); break;
                        case 3: run_unit<D, 3>(m, un.x, un.z, un.w, fpos, ws, tabs, lane, y); break;
                        default: run_unit<D, kMmaBundle>(m, un.x, un.z, un.w, fpos, ws, tabs, lane, y); break;
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < kMmaRowBlocks; ++r) {
                y[r] += __shfl_xor_sync(0xffffffffu, y[r], 1);
                y[r] += __shfl_xor_sync(0xffffffffu, y[r], 2);
                if ((lane & 3) == 0) sm.ypart[warp][8 * r + (lane >> 2)] = y[r];
            }
#ifdef QRMC_MMA_PHASE_CLOCKS
            const long long c_w = clk_fenced();
            const long long c_g1 = sync_clk();
#else
            __syncthreads();
#endif
#ifdef QRMC_MMA_PHASE_CLOCKS
            acc_own += c_w - c_g0;
            acc_gemm += c_g1 - c_g0;
            if (blockIdx.x == 100 && a.step == 5 && lane == 0 && j == 10)
                printf("RAW warp=%d g0=%lld w=%lld g1=%lld\n", warp, c_g0, c_w, c_g1);
#endif
        }
#ifdef QRMC_MMA_PHASE_CLOCKS
        const long long c_t0 = clk_fenced();
#endif
        // finish evaluation j; tables and x-only parts of evaluation j+1
#if QRMC_MMA_AHEAD == 0
        if (j + 1 < a.steps) euler(j + 1);
        __syncthreads();
#endif
        tables_and_paths(j + 2 < a.steps ? j + 1 : -1, j, QRMC_MMA_AHEAD >= 2 ? -1 : (j + 1 < a.steps ? j + 1 : -1));
#ifdef QRMC_MMA_PHASE_CLOCKS
        acc_tab += sync_clk() - c_t0;
#else
        __syncthreads();
#endif
    }
#ifdef QRMC_MMA_PHASE_CLOCKS
    if (blockIdx.x == 100 && a.step == 5 && lane == 0)
        printf("PHASE warp=%d own=%lld gemm=%lld tables=%lld total=%lld\n", warp, acc_own, acc_gemm, acc_tab,
               clk_fenced() - c_k0);
#endif
    cp_async_wait<0>();
    const int cur = (a.steps - a.step) & 1;  // X_N
    if (tid < kMmaPaths) {
        const int64_t q = q0 + tid;
        if (q < a.n_owned) {
            if (sm.bad[tid]) {
                // first error kind wins; SimulationError keeps the smallest step
                record_error(a.err_flags, QRMC_ESIM, sm.bad[tid]);
            } else {
                double xN[D];
#pragma unroll
                for (int l = 0; l < D; ++l) xN[l] = sm.x[cur][tid][l];
                const double term = terminal<D>(a.prob, xN);
                const double v = DDIV(DADD(term, DMUL(a.dt, sm.dsum[tid])), sm.w0[tid]);
                if (!isfinite(v)) record_error(a.err_flags, QRMC_ENUMERIC, 0);
                a.resp[q] = v;
            }
        }
    }
    // truncation counters: warp 0 holds them (paths < 32), one atomic per CTA
    if (warp == 0) {
        for (int o = 16; o > 0; o >>= 1) {
            apps += __shfl_down_sync(0xffffffffu, apps, o);
            clipped += __shfl_down_sync(0xffffffffu, clipped, o);
        }
        if (lane == 0 && apps) {
            atomicAdd(a.counters, static_cast<unsigned long long>(apps));
            if (clipped) atomicAdd(a.counters + 1, static_cast<unsigned long long>(clipped));
        }
    }
}

size_t responses_mma_smem_bytes(int dim, int table_len) {
    size_t head = 0;
    switch (dim) {
        case 3: head = sizeof(MmaSmem<3>); break;
        case 4: head = sizeof(MmaSmem<4>); break;
        case 5: head = sizeof(MmaSmem<5>); break;
        case 6: head = sizeof(MmaSmem<6>); break;
        case 7: head = sizeof(MmaSmem<7>); break;
        case 8: head = sizeof(MmaSmem<8>); break;
        default: return 0;
    }
    return ((head + 15) & ~size_t{15}) + static_cast<size_t>(kTabStride) * table_len * sizeof(double);
}

template <class Fn>
static cudaError_t with_kernel(int dim, bool gen, Fn&& fn) {
    switch (dim) {
        case 3: return gen ? fn(k_responses_mma<3, true>) : fn(k_responses_mma<3, false>);
        case 4: return gen ? fn(k_responses_mma<4, true>) : fn(k_responses_mma<4, false>);
        case 5: return gen ? fn(k_responses_mma<5, true>) : fn(k_responses_mma<5, false>);
        case 6: return gen ? fn(k_responses_mma<6, true>) : fn(k_responses_mma<6, false>);
        case 7: return gen ? fn(k_responses_mma<7, true>) : fn(k_responses_mma<7, false>);
        case 8: return gen ? fn(k_responses_mma<8, true>) : fn(k_responses_mma<8, false>);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t configure_responses_mma(int dim, size_t smem) {
    auto set = [&](auto kern) {
        return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    };
    const cudaError_t e = with_kernel(dim, false, set);
    return e != cudaSuccess ? e : with_kernel(dim, true, set);
}

cudaError_t launch_responses_mma(const StepArgs& a, const MmaArgs& m, cudaStream_t st) {
    if (a.n_owned == 0) return cudaSuccess;
    const size_t smem = responses_mma_smem_bytes(a.prob.dim, m.table_len);
    const unsigned blocks = static_cast<unsigned>((a.n_owned + kMmaPaths - 1) / kMmaPaths);
    const cudaError_t e = with_kernel(a.prob.dim, a.meas.form == 3, [&](auto kern) {
        kern<<<blocks, kThreads, smem, st>>>(a, m);
        return cudaGetLastError();
    });
    return e;
}

}  // namespace qrmc_dev

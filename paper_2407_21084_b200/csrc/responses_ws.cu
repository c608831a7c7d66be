// responses_ws.cu -- K1 (phase 1 of backward step i), warp-specialised.
//
// Same contract as k_responses_mma (responses_mma.cu) and k_responses
// (kernels.cu), i.e. proj/src/solver.cpp:147-177 with response_impl
// (solver.cpp:54-88): per path m of cloud i, draw X_i ~ nu, Euler to N,
// evaluate every future series alpha_{j+1} at X_{j+1}, truncate, accumulate the
// driver, emit S_m. The series is the same staircase GEMM on the FP64 tensor
// cores (mma.sync.m8n8k4.f64, see responses_mma.cu for the restructuring); what
// changes is the schedule of one CTA (32 paths, 20 warps):
//
//   * 16 consumer warps only run DMMAs. Evaluation j reads one of two cosine
//     table buffers (j & 1); B fragments come straight from L2 into registers,
//     prefetched to L1 a few fragments ahead along each warp's own stream, so
//     the GEMM has no shared-memory ring and no CTA barrier.
//   * 4 producer warps (one per SM sub-partition) run everything else one
//     evaluation ahead: the Euler step to X_{j+1}, the x-only parts of
//     evaluation j (weight, truncation bound, driver part), the truncation and
//     driver of evaluation j-2 (whose GEMM has finished) and the cosine tables
//     of evaluation j into the buffer the GEMM of j-2 has released.
//   * The hand-off is four named barriers: FULL[b] (producers arrive, consumers
//     wait: tables of buffer b ready) and DONE[b] (consumers arrive, producer
//     warp 0 waits: buffer b and its partial sums free).
//
// Tables are [entry][32 paths] with the path index swizzled by the entry
// (host.cpp ws_off): no padding, so two buffers of the config-2 tables (408
// entries) fit in shared memory.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "kernels.cuh"
#include "mma_common.cuh"
#include "qrmc_device.cuh"

namespace qrmc_dev {

namespace {

constexpr int kThreads = (kWsConsumers + kWsProducers) * 32;
constexpr int kProdThreads = kWsProducers * 32;
constexpr int kConsThreads = kWsConsumers * 32;
constexpr int kRB = kWsPaths / 8;  // row blocks
#ifndef QRMC_WS_CONSUMER_REGS
#define QRMC_WS_CONSUMER_REGS 104
#endif
#ifndef QRMC_WS_PRODUCER_REGS
#define QRMC_WS_PRODUCER_REGS 56
#endif
constexpr int kWsConsumerRegs = QRMC_WS_CONSUMER_REGS;
constexpr int kWsProducerRegs = QRMC_WS_PRODUCER_REGS;
// setmaxnreg only moves registers inside the CTA's launch allocation (ptxas allocates
// 65536 / kThreads rounded down to 8 per thread): a larger total would leave the
// consumers' setmaxnreg.inc waiting forever
constexpr int kLaunchRegs = (65536 / kThreads) / 8 * 8;
static_assert(kWsConsumers * kWsConsumerRegs + kWsProducers * kWsProducerRegs <=
                  (kWsConsumers + kWsProducers) * kLaunchRegs,
              "setmaxnreg budget exceeds the launch allocation");
static_assert(kRB == 4, "the swizzled operand addressing assumes 4 row blocks");
static_assert(kWsConsumers % 4 == 0 && kWsProducers == 4, "one producer warp per SM sub-partition");

// named barriers (0 is __syncthreads)
constexpr int kBarFull = 1;  // + buffer
constexpr int kBarDone = 3;  // + buffer
constexpr int kBarProd = 5;
constexpr int kFullCount = kThreads;             // all producers arrive, all consumers wait
constexpr int kDoneCount = kConsThreads + 32;    // all consumers arrive, producer warp 0 waits

__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// clock read that stays in place relative to the barriers (timing builds only)
__device__ __forceinline__ long long clk() {
    long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)::"memory");
    return t;
}
// clock read ordered after the value v is available (v read from shared memory
// after a barrier: the barrier's completion, which bar.sync may defer)
__device__ __forceinline__ long long clk_dep(double v) {
    long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t) : "d"(v) : "memory");
    return t;
}
__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }
// read-only loads with an L1 eviction priority: the operand tables (terms, group
// rows, units; re-read every evaluation) stay, the streamed B fragments go first
__device__ __forceinline__ uint4 ldg_keep(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::evict_last.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ int4 ldg_keep(const int4* p) {
    int4 v;
    asm volatile("ld.global.nc.L1::evict_last.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ double ldg_stream(const double* p) {
    double v;
    asm volatile("ld.global.nc.L1::evict_first.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

template <int D>
struct WsSmem {
    double ypart[3][kWsConsumers][kWsPaths];  // per consumer warp, slot j % 3
    double x[2][D][kWsPaths];                  // X_j and X_{j+1}, alternating ([l][path]: lanes on consecutive banks)
    double w0[kWsPaths], dsum[kWsPaths], term[kWsPaths];
    double wq[3][kWsPaths], lq[3][kWsPaths], dpre[3][kWsPaths];  // x-only parts, slot j % 3
    int bad[kWsPaths];
    int abort;
    // followed by two table buffers [table_len][32] (swizzled)
};

template <int D>
__device__ __forceinline__ double* ws_tables(unsigned char* base) {
    return reinterpret_cast<double*>(base + ((sizeof(WsSmem<D>) + 15) & ~size_t{15}));
}

// cos(k theta) for k = 0..kmax at entries off + k of path p (swizzled slot,
// host.cpp ws_off), lanes on consecutive paths. Four interleaved Chebyshev
// recurrences of stride 4, c_{k+4} = 2 c_4 c_k - c_{k-4} (T_{n+m} + T_{n-m} =
// 2 T_m T_n), so the dependent FMA chain is a quarter as long: the producers
// share the FP64 pipe with the consumers' DMMAs, where every dependent
// operation waits for a pipe slot.
__device__ __forceinline__ void ws_table(double th, int kmax, int off, int p, double* tab) {
    const double c1 = cos(th);
    const double c2 = fma(DMUL(2.0, c1), c1, -1.0);
    const double c3 = fma(DMUL(2.0, c1), c2, -c1);
    const double c4 = fma(DMUL(2.0, c2), c2, -1.0);
    const double two4 = DMUL(2.0, c4);
    // slots of entries off + 4m + t are (off + 4m + t) * 32 + (p ^ sw[t]): the
    // swizzle depends on (off + t) & 3 only
    int sw[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) sw[t] = p ^ (((off + t) & 3) << 2);
    double prv[4] = {c4, c3, c2, c1};  // c_{t-4} = c_{4-t}
    double cur[4] = {1.0, c1, c2, c3};
    double* base = tab + static_cast<size_t>(off) * 32;
    for (int k = 0; k <= kmax; k += 4, base += 128) {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            if (k + t <= kmax) base[32 * t + sw[t]] = cur[t];
            const double nx = fma(two4, cur[t], -prv[t]);
            prv[t] = cur[t];
            cur[t] = nx;
        }
    }
}

// One unit: NB column blocks x chunks [c0, c1), then y += U * C. B fragments
// come from the warp's linear stream (bsrc), prefetched to L1 kWsPrefetch
// fragments ahead; the next chunk's operand offsets are loaded one step ahead;
// the group rows of the epilogue at the unit's start.
template <int D, int NB>
__device__ __forceinline__ void ws_unit(const WsArgs& m, int cb0, int c0, int c1, const double*& bsrc,
                                        const char* trow, int half, int col, double (&y)[kRB]) {
    double acc[kRB][NB][2];
    constexpr int R = (2 * (D - 2) + 3) / 4 * 4;  // the pair (g0, g0 + 1)'s record (host.cpp ws_gk_index)
    uint32_t wp[NB][R];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const uint4* gw = reinterpret_cast<const uint4*>(
            m.gk + (static_cast<size_t>(half) * (m.n_groups / 2) + 4 * (cb0 + i) + col) * R);
#pragma unroll
        for (int q = 0; q < R / 4; ++q) {
            const uint4 v = ldg_keep(gw + q);
            wp[i][4 * q] = v.x;
            wp[i][4 * q + 1] = v.y;
            wp[i][4 * q + 2] = v.z;
            wp[i][4 * q + 3] = v.w;
        }
    }
    const uint4* tw = m.terms + (4 * c0 + col) * 2 + half;
    uint4 w = ldg_keep(tw);
    auto step = [&](auto first, bool more) {
        const uint4 cw = w;
        tw += 8;
        if (more) w = ldg_keep(tw);
        const double* sA = reinterpret_cast<const double*>(trow + cw.x);
        const double* sB = reinterpret_cast<const double*>(trow + cw.y);
        const double* bA = reinterpret_cast<const double*>(trow + cw.z);
        const double* bB = reinterpret_cast<const double*>(trow + cw.w);
        double a[kRB];
#ifdef QRMC_WS_EXP_NODMUL  // timing experiments only (wrong results)
        a[0] = sA[0];
        a[1] = sB[0];
        a[2] = bA[16];
        a[3] = bB[16];
#else
        a[0] = DMUL(sA[0], bA[0]);
        a[1] = DMUL(sB[0], bB[0]);
        a[2] = DMUL(sA[16], bA[16]);
        a[3] = DMUL(sB[16], bB[16]);
#endif
        double b[NB];
#pragma unroll
        for (int i = 0; i < NB; ++i) {
#ifdef QRMC_WS_EXP_NOB
            b[i] = static_cast<double>(col + i);
#else
            b[i] = ldg_stream(bsrc + 32 * i);
            prefetch_l1(bsrc + 32 * (kWsPrefetch + i));
#endif
        }
        bsrc += 32 * NB;
#pragma unroll
        for (int i = 0; i < NB; ++i)
#pragma unroll
            for (int r = 0; r < kRB; ++r) {
                if constexpr (decltype(first)::value)
                    dmma0(acc[r][i], a[r], b[i]);
                else
                    dmma(acc[r][i], a[r], b[i]);
            }
    };
    step(std::true_type{}, c0 + 1 < c1);
    int c = c0 + 1;
    for (; c + 3 < c1; c += 4) {
        step(std::false_type{}, true);
        step(std::false_type{}, true);
        step(std::false_type{}, true);
        step(std::false_type{}, c + 4 < c1);
    }
    for (; c < c1; ++c) step(std::false_type{}, c + 1 < c1);
    // epilogue: groups g0 = 8 (cb0 + i) + 2 col + h, U = prod_{l < D-2} c_{k_l}
#ifdef QRMC_WS_EXP_NOEPI
#pragma unroll
    for (int i = 0; i < NB; ++i)
#pragma unroll
        for (int r = 0; r < kRB; ++r) y[r] += acc[r][i][0] + acc[r][i][1] + wp[i][0];
    return;
#endif
#pragma unroll
    for (int i = 0; i < NB; ++i) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            double u[kRB];
#pragma unroll
            for (int l = 0; l < D - 2; ++l) {
                const uint32_t o = wp[i][h * (D - 2) + l];
                const double* pA = reinterpret_cast<const double*>(trow) + (o & 0xFFFFu);
                const double* pB = reinterpret_cast<const double*>(trow) + (o >> 16);
                if (l == 0) {
                    u[0] = pA[0];
                    u[1] = pB[0];
                    u[2] = pA[16];
                    u[3] = pB[16];
                } else {
                    u[0] = DMUL(u[0], pA[0]);
                    u[1] = DMUL(u[1], pB[0]);
                    u[2] = DMUL(u[2], pA[16]);
                    u[3] = DMUL(u[3], pB[16]);
                }
            }
#pragma unroll
            for (int r = 0; r < kRB; ++r) y[r] = fma(u[r], acc[r][i][h], y[r]);
        }
    }
}

// A transposed tail unit (host.cpp MmaLayoutOpts::tail_terms): chunks [c0, c1) of 4
// groups, NBT blocks of 8 terms. D_t = sum_u U_u alpha'_{u,t} as DMMAs with the group
// products U (d-2 table rows per group) as the A operand, then y += A_t D_t for the
// unit's 8 NBT terms -- one epilogue for many small groups.
template <int D, int NBT>
__device__ __forceinline__ void ws_unit_t(const WsArgs& m, int c0, int c1, const double*& bsrc, const char* trow,
                                          int half, int col, double (&y)[kRB]) {
    double acc[kRB][NBT][2];
    constexpr int R = (2 * (D - 2) + 3) / 4 * 4;  // group-pair record (host.cpp ws_gk_index)
    const uint4* rec = reinterpret_cast<const uint4*>(m.gk) +
                       (static_cast<size_t>(half) * (m.n_groups / 2) + 2 * c0 + (col >> 1)) * (R / 4);
    const int sub = (col & 1) * (D - 2);
    uint32_t wn[R];
    auto load_rec = [&](uint32_t (&w)[R]) {
#pragma unroll
        for (int q = 0; q < R / 4; ++q) {
            const uint4 v = ldg_keep(rec + q);
            w[4 * q] = v.x;
            w[4 * q + 1] = v.y;
            w[4 * q + 2] = v.z;
            w[4 * q + 3] = v.w;
        }
    };
    load_rec(wn);
    auto step = [&](auto first, bool more) {
        uint32_t w[R];
#pragma unroll
        for (int q = 0; q < R; ++q) w[q] = wn[q];
        rec += 2 * (R / 4);  // next chunk: 4 groups = 2 pair records
        if (more) load_rec(wn);
        double a[kRB];
#pragma unroll
        for (int l = 0; l < D - 2; ++l) {
            const uint32_t o = w[sub + l];
            const double* pA = reinterpret_cast<const double*>(trow) + (o & 0xFFFFu);
            const double* pB = reinterpret_cast<const double*>(trow) + (o >> 16);
            if (l == 0) {
                a[0] = pA[0];
                a[1] = pB[0];
                a[2] = pA[16];
                a[3] = pB[16];
            } else {
                a[0] = DMUL(a[0], pA[0]);
                a[1] = DMUL(a[1], pB[0]);
                a[2] = DMUL(a[2], pA[16]);
                a[3] = DMUL(a[3], pB[16]);
            }
        }
        double b[NBT];
#pragma unroll
        for (int i = 0; i < NBT; ++i) {
            b[i] = ldg_stream(bsrc + 32 * i);
            prefetch_l1(bsrc + 32 * (kWsPrefetch + i));
        }
        bsrc += 32 * NBT;
#pragma unroll
        for (int i = 0; i < NBT; ++i)
#pragma unroll
            for (int r = 0; r < kRB; ++r) {
                if constexpr (decltype(first)::value)
                    dmma0(acc[r][i], a[r], b[i]);
                else
                    dmma(acc[r][i], a[r], b[i]);
            }
    };
    step(std::true_type{}, c0 + 1 < c1);
    int c = c0 + 1;
    for (; c + 3 < c1; c += 4) {
        step(std::false_type{}, true);
        step(std::false_type{}, true);
        step(std::false_type{}, true);
        step(std::false_type{}, c + 4 < c1);
    }
    for (; c < c1; ++c) step(std::false_type{}, c + 1 < c1);
    // epilogue: the lane's terms t = 8 i + 2 col + h, A_t = c_s(x_{d-2}) c_b(x_{d-1})
#pragma unroll
    for (int i = 0; i < NBT; ++i)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint4 tw = ldg_keep(m.terms + (8 * i + 2 * col + h) * 2 + half);
            const double* sA = reinterpret_cast<const double*>(trow + tw.x);
            const double* sB = reinterpret_cast<const double*>(trow + tw.y);
            const double* bA = reinterpret_cast<const double*>(trow + tw.z);
            const double* bB = reinterpret_cast<const double*>(trow + tw.w);
            y[0] = fma(DMUL(sA[0], bA[0]), acc[0][i][h], y[0]);
            y[1] = fma(DMUL(sB[0], bB[0]), acc[1][i][h], y[1]);
            y[2] = fma(DMUL(sA[16], bA[16]), acc[2][i][h], y[2]);
            y[3] = fma(DMUL(sB[16], bB[16]), acc[3][i][h], y[3]);
        }
}

}  // namespace

template <int D, bool GEN>
__global__ void __launch_bounds__(kThreads, 1) k_responses_ws(const StepArgs a, const WsArgs m) {
    static_assert(D >= 3, "the tensor-core K1 needs an upper prefix");
    extern __shared__ __align__(16) unsigned char dsm[];
    WsSmem<D>& sm = *reinterpret_cast<WsSmem<D>*>(dsm);
    double* tabs = ws_tables<D>(dsm);
    const size_t tab_elems = static_cast<size_t>(m.table_len) * 32;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int i0 = a.step, N = a.steps;
    if (tid == 0) sm.abort = *a.abort_flag;
    if (tid < kWsPaths) sm.bad[tid] = 0;
    __syncthreads();
    if (sm.abort) return;
    const int64_t q0 = static_cast<int64_t>(blockIdx.x) * kWsPaths;

    if (warp < kWsConsumers) {
        // ------------------------------------------------------------ consumers
        // registers move from the producer warpgroup to the consumers (the GEMM's
        // accumulators and load pipeline); 16 x 104 + 4 x 56 warps' worth fit 64K
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kWsConsumerRegs));
        const int cw = warp;
        const int row = lane >> 2, col = lane & 3, half = row >> 2;
        const int4 wi = __ldg(&m.warp_info[cw]);  // {unit_begin, unit_end, series-0 fragment, frags per series}
        // the warp's linear stream from alpha_{i+1} on, and its L1 prefetch
        const double* bsrc = m.alpha + (static_cast<int64_t>(wi.z) + static_cast<int64_t>(i0 + 1) * wi.w) * 32 + lane;
        for (int f = 0; f < kWsPrefetch; ++f) prefetch_l1(bsrc + 32 * f);
#ifdef QRMC_WS_CLOCKS
        long long cts[24][3];
#endif
        for (int j = i0; j < N - 1; ++j) {
            // evaluation of alpha_{j+1} at X_{j+1}
            double y[kRB];
#pragma unroll
            for (int r = 0; r < kRB; ++r) y[r] = 0.0;
#ifdef QRMC_WS_CLOCKS
            const long long t0 = clk();
#endif
            bar_sync(kBarFull + (j & 1), kFullCount);
            const char* trow = reinterpret_cast<const char*>(tabs + (j & 1) * tab_elems + row);
#ifdef QRMC_WS_CLOCKS
            const long long t1 = clk_dep(*reinterpret_cast<const volatile double*>(trow));
#endif
            for (int u = wi.x; u < wi.y; ++u) {
                const int4 un = ldg_keep(&m.units[u]);
                if (un.y == 1)
                    ws_unit<D, 1>(m, un.x, un.z, un.w, bsrc, trow, half, col, y);
                else if (un.y == 2)
                    ws_unit<D, 2>(m, un.x, un.z, un.w, bsrc, trow, half, col, y);
#if QRMC_WS_BUNDLE >= 3
                else if (un.y == 3)
                    ws_unit<D, 3>(m, un.x, un.z, un.w, bsrc, trow, half, col, y);
#endif
                else if (un.y == 9)
                    ws_unit_t<D, 1>(m, un.z, un.w, bsrc, trow, half, col, y);
                else
                    ws_unit_t<D, 2>(m, un.z, un.w, bsrc, trow, half, col, y);
            }
#pragma unroll
            for (int r = 0; r < kRB; ++r) {
                y[r] += __shfl_xor_sync(0xffffffffu, y[r], 1);
                y[r] += __shfl_xor_sync(0xffffffffu, y[r], 2);
                if (col == 0) sm.ypart[j % 3][cw][8 * r + row] = y[r];
            }
            bar_arrive(kBarDone + (j & 1), kDoneCount);
#ifdef QRMC_WS_CLOCKS
            cts[j][0] = t0;
            cts[j][1] = t1;
            cts[j][2] = clk_dep(y[0]);
#endif
        }
#ifdef QRMC_WS_CLOCKS
        if ((blockIdx.x == 1000 || blockIdx.x == 30000) && lane == 0 && (cw % 4 == 0))
            for (int j = i0; j < N - 1; ++j)
                printf("B%d C%d j=%d wait=%lld gemm=%lld\n", blockIdx.x, cw, j, cts[j][1] - cts[j][0], cts[j][2] - cts[j][1]);
#endif
        return;
    }

    // ---------------------------------------------------------------- producers
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kWsProducerRegs));
    const int pt = tid - kConsThreads;
    const int p = pt & 31, pw = pt >> 5;  // path (lane), producer warp
    const int64_t q = q0 + p;
    const bool live = q < a.n_owned;
    const uint64_t sid = sid_training(i0, static_cast<uint64_t>(owned_path(a, live ? q : 0)));
    uint32_t apps = 0, clipped = 0;

    // start points X_i ~ nu: draws 0..D-1 of the path's stream (solver.cpp:150-152)
    for (int l = pw; l < D; l += kWsProducers) {
        const double x = measure_inv_cdf<GEN>(a.meas, u64_to_uniform(stream_u64_at(a.seed, sid, l)), l);
        sm.x[0][l][p] = x;
        if (a.cloud && live)
            a.cloud[l * a.n_owned + q] = a.cloud_cos ? cos(DMUL(3.14159265358979323846, measure_cdf<GEN>(a.meas, x, l))) : x;
    }
    bar_sync(kBarProd, kProdThreads);
    if (pw == 0) {
        double x[D];
#pragma unroll
        for (int l = 0; l < D; ++l) x[l] = sm.x[0][l][p];
        sm.w0[p] = damping_weight<D>(x, a.q);
        sm.dsum[p] = 0.0;
    }

    // truncation + driver of evaluation jj (solver.cpp:160-172), producer warp 0
    auto finish = [&](int jj) {
        const int c = jj % 3;
        double yv;
        if (jj + 1 == N) {
            yv = sm.term[p];  // exact initialisation at the terminal step (solver.cpp:69-72)
        } else {
            // fixed-order pairwise sum of the consumer warps' partials (a short
            // dependency chain on the shared FP64 pipe)
            double v[kWsConsumers];
#pragma unroll
            for (int w = 0; w < kWsConsumers; ++w) v[w] = sm.ypart[jj % 3][w][p];
#pragma unroll
            for (int s2 = kWsConsumers / 2; s2 > 0; s2 /= 2)
#pragma unroll
                for (int w = 0; w < s2; ++w) v[w] += v[w + s2];
            yv = DMUL(v[0], sm.wq[c][p]);
        }
        const double cv = truncate_soft(yv, sm.lq[c][p]);
        if (live) {
            ++apps;
            if (cv != yv) ++clipped;
        }
        sm.dsum[p] = DADD(sm.dsum[p], driver_apply(a.prob, sm.dpre[c][p], cv));
    };

#ifdef QRMC_WS_CLOCKS
    long long pts[24][4];
    const long long pstart = clk();
#endif
    for (int j = i0; j < N; ++j) {
        // Euler step j (sde.cpp:37-73): X_{j+1} from X_j, draw D + (j-i)*D + l
        const int src = (j - i0) & 1;
#ifdef QRMC_WS_CLOCKS
        const long long estart = clk();
#endif
        for (int l = pw; l < D; l += kWsProducers) {
#ifndef QRMC_WS_EXP_NOEULER
            const double nrm = normal_quantile_ilp(
                u64_to_uniform(stream_u64_at(a.seed, sid, static_cast<uint64_t>(D) * (j - i0 + 1) + l)));
#else
            const double nrm = 0.001 * (j + l);
#endif
            const double dw = DMUL(a.sqrt_dt, nrm);
            const double xo = sm.x[src][l][p];
            const double v = euler_coord(a.prob, xo, dw, l, a.dt);
            sm.x[src ^ 1][l][p] = v;
            if ((!isfinite(v) || fabs(v) > a.prob.state_bound) && sm.bad[p] == 0) sm.bad[p] = j + 1;
        }
#ifdef QRMC_WS_CLOCKS
        const long long e0 = clk_dep(sm.x[src ^ 1][pw][p]);  // Euler done (own value)
#endif
        bar_sync(kBarProd, kProdThreads);
#ifdef QRMC_WS_CLOCKS
        const long long e1 = clk_dep(*reinterpret_cast<volatile double*>(&sm.x[src ^ 1][(pw + 1) % D][p]));
#endif
        if (pw == 0) {
            // the GEMM of evaluation j-2 has released table buffer j & 1
            if (j - 2 >= i0 && j + 1 < N) bar_sync(kBarDone + (j & 1), kDoneCount);
        } else {
            // x-only parts of evaluation j, one kind per warp: weight at X_{j+1}
            // (terminal value at X_N), truncation bound at X_{j+1}, the driver's
            // x-part at (t_j, X_j)
            const int kind = pw - 1, c = j % 3;
            double xv[D];
#pragma unroll
            for (int l = 0; l < D; ++l) xv[l] = sm.x[kind == 2 ? src : src ^ 1][l][p];
            if (kind == 0) {
                if (j + 1 == N)
                    sm.term[p] = terminal<D>(a.prob, xv);
                else
                    sm.wq[c][p] = damping_weight<D>(xv, a.q);
            } else if (kind == 1) {
                sm.lq[c][p] = lstar<D>(a.prob, xv);
            } else {
                sm.dpre[c][p] = driver_pre<D>(a.prob, DMUL(static_cast<double>(j), a.dt), xv);
            }
        }
#ifdef QRMC_WS_CLOCKS
        const long long e2 = clk_dep(pw == 0 ? 0.0 : (pw == 1 ? sm.wq[j % 3][p] : pw == 2 ? sm.lq[j % 3][p] : sm.dpre[j % 3][p]));
#endif
        if (j + 1 < N) {
            // cosine tables of evaluation j (X_{j+1}) into buffer j & 1
            bar_sync(kBarProd, kProdThreads);
            double* tb = tabs + (j & 1) * tab_elems;
            for (int l = pw; l < D; l += kWsProducers) {
                const double th = DMUL(3.14159265358979323846, measure_cdf<GEN>(a.meas, sm.x[src ^ 1][l][p], l));
#ifndef QRMC_WS_EXP_NOTAB
                ws_table(th, m.kmax[l], m.offset[l], p, tb);
#else
                if (th == 12345.0) tb[p] = th;
#endif
            }
            bar_arrive(kBarFull + (j & 1), kFullCount);
        }
#ifdef QRMC_WS_CLOCKS
        pts[j][0] = e0 - estart;   // Euler compute (incl. iteration start)
        pts[j][1] = e1 - e0;       // wait for the other producers' Euler
        pts[j][2] = e2 - e1;       // parts (warps 1-3) / DONE wait (warp 0)
        pts[j][3] = clk_dep(*reinterpret_cast<volatile double*>(tabs + (j & 1) * tab_elems + p)) - e2;  // sync + tables
#endif
        // truncation + driver of evaluation j-2 off the tables' critical path: its
        // partial sums sit in slot (j-2) % 3, which the consumers rewrite only after
        // the GEMM of evaluation j+1
        if (pw == 0 && j - 2 >= i0) {
            if (j + 1 == N) bar_sync(kBarDone + (j & 1), kDoneCount);
            finish(j - 2);
        }
    }
    if (pw == 0 && N - 2 >= i0) {
        bar_sync(kBarDone + ((N - 2) & 1), kDoneCount);
        finish(N - 2);
    }
#ifdef QRMC_WS_CLOCKS
    if ((blockIdx.x == 1000 || blockIdx.x == 30000) && p == 0)
        for (int j = i0; j < N; ++j)
            printf("B%d P%d j=%d euler=%lld sync1=%lld parts=%lld tables=%lld\n", blockIdx.x, pw, j,
                   pts[j][0], pts[j][1], pts[j][2], pts[j][3]);
#endif
    bar_sync(kBarProd, kProdThreads);  // the terminal parts (warps 1-3) are in place
    if (pw != 0) return;
    finish(N - 1);

    const int cur = (N - i0) & 1;  // X_N
    if (live) {
        if (sm.bad[p]) {
            record_error(a.err_flags, QRMC_ESIM, sm.bad[p]);
        } else {
            const double v = DDIV(DADD(sm.term[p], DMUL(a.dt, sm.dsum[p])), sm.w0[p]);
            if (!isfinite(v)) record_error(a.err_flags, QRMC_ENUMERIC, 0);
            a.resp[q] = v;
        }
    }
    (void)cur;
    for (int o = 16; o > 0; o >>= 1) {
        apps += __shfl_down_sync(0xffffffffu, apps, o);
        clipped += __shfl_down_sync(0xffffffffu, clipped, o);
    }
    if (lane == 0 && apps) {
        atomicAdd(a.counters, static_cast<unsigned long long>(apps));
        if (clipped) atomicAdd(a.counters + 1, static_cast<unsigned long long>(clipped));
    }
}

size_t responses_ws_smem_bytes(int dim, int table_len) {
    size_t head = 0;
    switch (dim) {
        case 3: head = sizeof(WsSmem<3>); break;
        case 4: head = sizeof(WsSmem<4>); break;
        case 5: head = sizeof(WsSmem<5>); break;
        case 6: head = sizeof(WsSmem<6>); break;
        case 7: head = sizeof(WsSmem<7>); break;
        case 8: head = sizeof(WsSmem<8>); break;
        default: return 0;
    }
    return ((head + 15) & ~size_t{15}) + 2 * static_cast<size_t>(table_len) * 32 * sizeof(double);
}

template <class Fn>
static cudaError_t with_ws_kernel(int dim, bool gen, Fn&& fn) {
    switch (dim) {
        case 3: return gen ? fn(k_responses_ws<3, true>) : fn(k_responses_ws<3, false>);
        case 4: return gen ? fn(k_responses_ws<4, true>) : fn(k_responses_ws<4, false>);
        case 5: return gen ? fn(k_responses_ws<5, true>) : fn(k_responses_ws<5, false>);
        case 6: return gen ? fn(k_responses_ws<6, true>) : fn(k_responses_ws<6, false>);
        case 7: return gen ? fn(k_responses_ws<7, true>) : fn(k_responses_ws<7, false>);
        case 8: return gen ? fn(k_responses_ws<8, true>) : fn(k_responses_ws<8, false>);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t configure_responses_ws(int dim, size_t smem) {
    auto set = [&](auto kern) {
        return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    };
    const cudaError_t e = with_ws_kernel(dim, false, set);
    return e != cudaSuccess ? e : with_ws_kernel(dim, true, set);
}

cudaError_t launch_responses_ws(const StepArgs& a, const WsArgs& m, cudaStream_t st) {
    if (a.n_owned == 0) return cudaSuccess;
    const size_t smem = responses_ws_smem_bytes(a.prob.dim, m.table_len);
    const unsigned blocks = static_cast<unsigned>((a.n_owned + kWsPaths - 1) / kWsPaths);
    return with_ws_kernel(a.prob.dim, a.meas.form == 3, [&](auto kern) {
        kern<<<blocks, kThreads, smem, st>>>(a, m);
        return cudaGetLastError();
    });
}

}  // namespace qrmc_dev

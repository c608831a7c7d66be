// kernels.cu -- the sm_100a kernels of one backward step and their launchers.
//
// One backward step i of backward_solve (proj/src/solver.cpp:143-219) is
//   K1 k_responses    phase 1: per path, draw X_i ~ nu, Euler to N, evaluate
//                     every future series alpha_{j+1} at X_{j+1}, truncate,
//                     accumulate the driver, emit S_m (solver.cpp:147-177)
//   K2 k_project      phase 2: per lane, acc[lane][k] = sum_m S_m phi_k(X_i^m)
//                     in the reference's lane/chunk order (solver.cpp:180-199)
//   K3 k_finish_step  coeffs[k] = (sum_{lane=0..255} acc[lane][k]) * (1/M),
//                     finiteness check, and the packed alpha' row the next
//                     steps' K1 reads (solver.cpp:201-213)
// plus the probes behind the C ABI's replay entry points.
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "kernels.cuh"
#include "qrmc_device.cuh"
#include "series_block.cuh"

namespace qrmc_dev {

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ int64_t owned_to_path(const StepArgs& a, int64_t q) {
    // owned index q -> global path m: owned chunk cq = q / 1024 is (round r,
    // lane lo + cq % owned_lanes), chunk c = 256 r + lane (LaneLayout::for_lane,
    // parallel.hpp:28-35, restricted to this rank's lanes).
    const int64_t cq = q / kChunk;
    const int64_t r = cq / a.owned_lanes;
    const int64_t lane = a.lane_lo + cq % a.owned_lanes;
    return (r * kLanes + lane) * kChunk + q % kChunk;
}

__device__ __forceinline__ void sample_start(const MeasureDev& m, int d, Stream& s, double* x) {
    for (int l = 0; l < d; ++l) x[l] = measure_inv_cdf(m, s.next_uniform(), l);
}

// ---------------------------------------------------------------- K1
// P paths per thread, 128 threads per CTA; the CTA walks the backward step's
// future time points in lockstep so that each coefficient row alpha_{j+1}
// streams through shared memory once per CTA (series_block.cuh). P, S2, LT
// per dimension: k1_p / k1_s2 / k1_lt (qrmc_types.h).
constexpr int kK1Threads = 128;

// Per-path state of K1 kept in shared memory between evaluations, so the
// series evaluation has the register file to itself.
template <int D>
struct PathSmem {
    double xj[D];  // X_j
    double xn[D];  // X_{j+1}
    double w0, dsum;
    unsigned long long block, buf1;  // RngStream position
    int pos, bad;
};

// dynamic shared memory of a series kernel: coefficient/program tiles, the
// per-thread sibling table c_{D-2}[0..S2) for P points, and (K1) path state
template <int D>
constexpr size_t series_smem_bytes(int P, bool paths = false) {
    return sizeof(SeriesSmem) + static_cast<size_t>(k1_s2(D)) * P * kK1Threads * sizeof(double) +
           (paths ? sizeof(PathSmem<D>) * P * kK1Threads : 0);
}

template <int D>
#ifndef QRMC_K1_MIN_BLOCKS
#define QRMC_K1_MIN_BLOCKS 1
#endif
__global__ void __launch_bounds__(kK1Threads, QRMC_K1_MIN_BLOCKS) k_responses(const StepArgs a) {
    constexpr int P = k1_p(D), S2 = k1_s2(D), LT = k1_lt(D);
    extern __shared__ __align__(16) unsigned char dsm[];
    SeriesSmem& sm = *reinterpret_cast<SeriesSmem*>(dsm);
    double* t2s = reinterpret_cast<double*>(dsm + sizeof(SeriesSmem));
    PathSmem<D>* ps = reinterpret_cast<PathSmem<D>*>(dsm + sizeof(SeriesSmem) +
                                                    static_cast<size_t>(S2) * P * kK1Threads * sizeof(double));
    __shared__ int s_abort;
    if (threadIdx.x == 0) s_abort = *a.abort_flag;
    __syncthreads();
    if (s_abort) return;  // uniform per CTA

    uint32_t apps = 0, clipped = 0;
    int64_t m_of[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
        PathSmem<D>& st = ps[p * kK1Threads + threadIdx.x];
        const int64_t q = (static_cast<int64_t>(blockIdx.x) * P + p) * kK1Threads + threadIdx.x;
        const bool valid = q < a.n_owned;
        m_of[p] = owned_to_path(a, valid ? q : 0);
        Stream s(a.seed, sid_training(a.step, static_cast<uint64_t>(m_of[p])));
        double x[D];
#pragma unroll
        for (int l = 0; l < D; ++l) x[l] = measure_inv_cdf(a.meas, s.next_uniform(), l);
        if (a.cloud && valid) {
#pragma unroll
            for (int l = 0; l < D; ++l) a.cloud[l * a.n_owned + q] = x[l];
        }
#pragma unroll
        for (int l = 0; l < D; ++l) st.xj[l] = x[l];
        st.w0 = damping_weight<D>(x, a.q);
        st.dsum = 0.0;
        st.block = s.block;
        st.buf1 = s.buf1;
        st.pos = s.pos;
        st.bad = 0;
    }
    for (int j = a.step; j < a.steps; ++j) {
        const bool last = j + 1 == a.steps;
        double c1[P][D];
#pragma unroll
        for (int p = 0; p < P; ++p) {
            PathSmem<D>& st = ps[p * kK1Threads + threadIdx.x];
            Stream s(a.seed, sid_training(a.step, static_cast<uint64_t>(m_of[p])));
            s.block = st.block;
            s.buf1 = st.buf1;
            s.pos = st.pos;
            double x[D];
#pragma unroll
            for (int l = 0; l < D; ++l) x[l] = st.xj[l];
            const int b = euler_step<D>(a.prob, x, a.sqrt_dt, a.dt, s, j);
            if (b && !st.bad) st.bad = b;
            st.block = s.block;
            st.buf1 = s.buf1;
            st.pos = s.pos;
#pragma unroll
            for (int l = 0; l < D; ++l) {
                st.xn[l] = x[l];
                c1[p][l] = last ? 0.0 : cos(DMUL(3.14159265358979323846, measure_cdf(a.meas, x[l], l)));
            }
        }
        double ys[P];
        if (!last)
            series_block<D, P, S2, LT>(sm, t2s, a.tiles, a.alpha_packed + static_cast<int64_t>(j + 1) * a.kp, c1, ys);
#pragma unroll
        for (int p = 0; p < P; ++p) {
            PathSmem<D>& st = ps[p * kK1Threads + threadIdx.x];
            const int64_t q = (static_cast<int64_t>(blockIdx.x) * P + p) * kK1Threads + threadIdx.x;
            double xn[D], xj[D];
#pragma unroll
            for (int l = 0; l < D; ++l) {
                xn[l] = st.xn[l];
                xj[l] = st.xj[l];
            }
            // exact initialisation at the terminal step (solver.cpp:69-72)
            const double y = last ? terminal<D>(a.prob, xn) : DMUL(ys[p], damping_weight<D>(xn, a.q));
            const double c = truncate_soft(y, lstar<D>(a.prob, xn));
            if (q < a.n_owned) {
                ++apps;
                if (c != y) ++clipped;
            }
            st.dsum = DADD(st.dsum, driver<D>(a.prob, DMUL(static_cast<double>(j), a.dt), xj, c));
#pragma unroll
            for (int l = 0; l < D; ++l) st.xj[l] = xn[l];
        }
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
        const int64_t q = (static_cast<int64_t>(blockIdx.x) * P + p) * kK1Threads + threadIdx.x;
        if (q >= a.n_owned) continue;
        const PathSmem<D>& st = ps[p * kK1Threads + threadIdx.x];
        if (st.bad) {
            record_error(a.err_flags, QRMC_ESIM, st.bad);
        } else {
            double xj[D];
#pragma unroll
            for (int l = 0; l < D; ++l) xj[l] = st.xj[l];
            const double term = terminal<D>(a.prob, xj);
            const double v = DDIV(DADD(term, DMUL(a.dt, st.dsum)), st.w0);
            if (!isfinite(v)) record_error(a.err_flags, QRMC_ENUMERIC, 0);
            a.resp[q] = v;
        }
    }
    // truncation counters: warp-aggregate then one atomic per warp
    for (int o = 16; o > 0; o >>= 1) {
        apps += __shfl_down_sync(0xffffffffu, apps, o);
        clipped += __shfl_down_sync(0xffffffffu, clipped, o);
    }
    if ((threadIdx.x & 31) == 0 && apps) {
        atomicAdd(a.counters, static_cast<unsigned long long>(apps));
        if (clipped) atomicAdd(a.counters + 1, static_cast<unsigned long long>(clipped));
    }
}

// ---------------------------------------------------------------- K2
// CTA (item tile, owned lane). A work item is a chunk of <= kProjRun leaf
// indices of one leaf run (host.cpp build_project_items; items sorted by
// length so a warp's lanes stay in step). Each thread owns kProjItems items
// and sums S_m * phi_k(X_m) over the lane's paths in ascending m -- the
// reference's per-lane order (solver.cpp:186-197), deterministic and
// independent of the GPU count -- with the reference's Student-cosine table
// values (cosine_basis.cpp:71-89). The run prefix S_m*((T_0*T_1)*...*T_{d-2})
// is formed once per (item, point); each term is then one FMA.
#ifndef QRMC_PROJ_THREADS
#define QRMC_PROJ_THREADS 256
#endif
constexpr int kProjThreads = QRMC_PROJ_THREADS;
#ifndef QRMC_PROJ_ITEMS
#define QRMC_PROJ_ITEMS 4
#endif
constexpr int kProjItems = QRMC_PROJ_ITEMS;  // items per thread

template <int D>
__global__ void __launch_bounds__(kProjThreads) k_project(const StepArgs a, const ProjArgs p) {
    extern __shared__ double smem[];
    double* tab = smem;                          // [batch][table_len]
    double* sv = smem + p.batch * p.table_len;   // [batch]
    const int lane_rel = blockIdx.y;
    const int lane = a.lane_lo + lane_rel;
    constexpr int NPRE = D > 1 ? D - 1 : 1;

    int pre[kProjItems][NPRE], leaf[kProjItems], len[kProjItems], kfirst[kProjItems];
    double acc[kProjItems][kProjRun];
#pragma unroll
    for (int t = 0; t < kProjItems; ++t) {
        const int it = (blockIdx.x * kProjItems + t) * kProjThreads + threadIdx.x;
        const bool live = it < p.n_items;
        len[t] = live ? p.item_len[it] : 0;
        kfirst[t] = live ? p.item_k[it] : 0;
        leaf[t] = live ? p.item_leaf[it] : 0;
#pragma unroll
        for (int l = 0; l < NPRE; ++l) pre[t][l] = (live && D > 1) ? p.item_pre[l * p.n_items + it] : 0;
#pragma unroll
        for (int b = 0; b < kProjRun; ++b) acc[t][b] = 0.0;
    }

    const int64_t chunks_total = (a.paths + kChunk - 1) / kChunk;
    for (int64_t c = lane; c < chunks_total; c += kLanes) {
        const int64_t r = c / kLanes;
        const int64_t q_chunk = (r * a.owned_lanes + lane_rel) * kChunk;  // owned index of the chunk
        const int64_t m_chunk = c * kChunk;
        const int64_t rem = a.paths - m_chunk;
        const int nlen = static_cast<int>(rem < kChunk ? rem : kChunk);
        for (int base = 0; base < nlen; base += p.batch) {
            const int nb = min(p.batch, nlen - base);
            __syncthreads();
            // tables: one (point, coordinate) recurrence per task (cosine_basis.cpp:67-89);
            // a second task per pair restarts the recurrence at k0 = kmax/2 from directly
            // evaluated cosines, halving the serial chain the CTA waits on
            for (int task = threadIdx.x; task < 2 * nb * D; task += kProjThreads) {
                const int half = task & 1;
                const int pt = (task >> 1) / D, l = (task >> 1) % D;
                const int64_t q = q_chunk + base + pt;
                double xl;
                if (a.cloud) {
                    xl = a.cloud[l * a.n_owned + q];
                } else {
                    // recompute-from-seeds (solver.cpp:187-193): regenerate X_i
                    Stream s(a.seed, sid_training(a.step, static_cast<uint64_t>(m_chunk + base + pt)));
                    double u = 0.0;
                    for (int ll = 0; ll <= l; ++ll) u = s.next_uniform();
                    xl = measure_inv_cdf(a.meas, u, l);
                }
                const double theta = DMUL(3.14159265358979323846, measure_cdf(a.meas, xl, l));
                const double c1 = cos(theta);
                double* t = tab + pt * p.table_len + p.offset[l];
                const int kmax = p.kmax[l];
                const int k0 = kmax >= 8 ? kmax / 2 : kmax + 1;  // second half [k0, kmax]
                const double sqrt2 = 1.4142135623730951;
                const double two_c1 = DMUL(2.0, c1);
                if (half == 0) {
                    t[0] = 1.0;
                    if (kmax >= 1) {
                        double prev = 1.0, cur = c1;
                        t[1] = DMUL(sqrt2, c1);
                        for (int k = 2; k < k0; ++k) {
                            const double nx = DSUB(DMUL(two_c1, cur), prev);
                            prev = cur;
                            cur = nx;
                            t[k] = DMUL(sqrt2, nx);
                        }
                    }
                    if (l == 0) sv[pt] = a.resp[q];
                } else if (k0 <= kmax) {
                    double prev = cos(static_cast<double>(k0 - 1) * theta), cur = cos(static_cast<double>(k0) * theta);
                    t[k0] = DMUL(sqrt2, cur);
                    for (int k = k0 + 1; k <= kmax; ++k) {
                        const double nx = DSUB(DMUL(two_c1, cur), prev);
                        prev = cur;
                        cur = nx;
                        t[k] = DMUL(sqrt2, nx);
                    }
                }
            }
            __syncthreads();
#pragma unroll
            for (int it = 0; it < kProjItems; ++it) {
                // item lengths are uniform per warp (host pads length classes to whole
                // warps): one dispatch per (item slot, batch) into a static-length loop
                auto points = [&](auto len_c) {
                    constexpr int LEN = decltype(len_c)::value;
                    constexpr int NP2 = (LEN + 1) / 2;
                    for (int pt = 0; pt < nb; ++pt) {
                        const double* t = tab + pt * p.table_len;
                        // w = S_m * ((T_0 T_1) ... T_{d-2}); each term one FMA with the leaf
                        // value, read as 16-byte pairs (leaf offsets are even)
                        double w = sv[pt];
                        if constexpr (D > 1) {
                            double prefix = t[pre[it][0]];
#pragma unroll
                            for (int l = 1; l < D - 1; ++l) prefix = DMUL(prefix, t[pre[it][l]]);
                            w = DMUL(w, prefix);
                        }
                        const double2* lv = reinterpret_cast<const double2*>(t + leaf[it]);
#pragma unroll
                        for (int b2 = 0; b2 < NP2; ++b2) {
                            const double2 v = lv[b2];
                            acc[it][2 * b2] = fma(w, v.x, acc[it][2 * b2]);
                            if (2 * b2 + 1 < LEN) acc[it][2 * b2 + 1] = fma(w, v.y, acc[it][2 * b2 + 1]);
                        }
                    }
                };
                switch (len[it]) {
                    case 1: points(std::integral_constant<int, 1>{}); break;
                    case 2: points(std::integral_constant<int, 2>{}); break;
                    case 3: points(std::integral_constant<int, 3>{}); break;
                    case 4: points(std::integral_constant<int, 4>{}); break;
                    case 5: points(std::integral_constant<int, 5>{}); break;
                    case 6: points(std::integral_constant<int, 6>{}); break;
                    case 7: points(std::integral_constant<int, 7>{}); break;
                    case 8: points(std::integral_constant<int, 8>{}); break;
                    default: break;
                }
            }
        }
    }
#pragma unroll
    for (int it = 0; it < kProjItems; ++it) {
        double* out = p.partials + static_cast<int64_t>(lane_rel) * p.basis_size + kfirst[it];
#pragma unroll
        for (int b = 0; b < kProjRun; ++b)
            if (b < len[it]) out[b] = acc[it][b];
    }
}

// ---------------------------------------------------------------- K3
__global__ void k_finish_step(const StepArgs a, const FinishArgs f) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= f.basis_size) return;
    double sum = 0.0;
    for (int lane = 0; lane < kLanes; ++lane) sum = DADD(sum, f.all_partials[static_cast<int64_t>(lane) * f.basis_size + k]);
    const double v = DMUL(sum, f.inv_m);
    if (!isfinite(v)) record_error(a.err_flags, QRMC_ENUMERIC, 0);
    f.coef_row[k] = v;
    const double scaled = DMUL(v, f.pack_scale[k]);
    a.alpha_packed[static_cast<int64_t>(a.step) * a.kp + f.pack_pos[k]] = scaled;
    if (f.alpha_mma)
        f.alpha_mma[static_cast<int64_t>(a.step) * (f.mma_stride ? f.mma_stride[k] : f.mma_row_len) + f.mma_pos[k]] = scaled;
}

// ---------------------------------------------------------------- probes
__global__ void k_philox(const uint4* ctr, const uint2* key, int64_t n, uint4* out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = philox4x32_10(ctr[i], key[i]);
}

__global__ void k_stream_draws(uint64_t seed, const uint64_t* sids, int64_t n, int n_draws, int kind,
                               void* out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Stream s(seed, sids[i]);
    for (int k = 0; k < n_draws; ++k) {
        const int64_t at = i * n_draws + k;
        if (kind == 0)
            static_cast<uint64_t*>(out)[at] = s.next_u64();
        else if (kind == 1)
            static_cast<double*>(out)[at] = s.next_uniform();
        else
            static_cast<double*>(out)[at] = s.next_normal();
    }
}

template <int D>
__global__ void k_cloud_paths(const StepArgs a, int64_t first, int64_t n, double* out, int* bad_out) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int64_t len = static_cast<int64_t>(a.steps - a.step + 1) * D;
    double* path = out + r * len;
    Stream s(a.seed, sid_training(a.step, static_cast<uint64_t>(first + r)));
    double x[D];
#pragma unroll
    for (int l = 0; l < D; ++l) {
        x[l] = measure_inv_cdf(a.meas, s.next_uniform(), l);
        path[l] = x[l];
    }
    for (int j = a.step; j < a.steps; ++j) {
        const int b = euler_step<D>(a.prob, x, a.sqrt_dt, a.dt, s, j);
        if (b) {
            atomicMax(bad_out, b);
            return;
        }
#pragma unroll
        for (int l = 0; l < D; ++l) path[(j + 1 - a.step) * D + l] = x[l];
    }
}

// evaluate_solution / SeriesEvaluator::eval at given points (solver.cpp:228-237),
// one point per thread; every thread of the CTA joins the series walk.
template <int D>
__global__ void __launch_bounds__(kK1Threads) k_eval_points(const StepArgs a, const double* alpha_row,
                                                            const double* x, int64_t n, double q,
                                                            int with_weight, double* out) {
    extern __shared__ __align__(16) unsigned char dsm[];
    SeriesSmem& sm = *reinterpret_cast<SeriesSmem*>(dsm);
    double* t2s = reinterpret_cast<double*>(dsm + sizeof(SeriesSmem));
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t rr = r < n ? r : n - 1;
    double p[D], c1[1][D], y[1];
#pragma unroll
    for (int l = 0; l < D; ++l) {
        p[l] = x[rr * D + l];
        c1[0][l] = cos(DMUL(3.14159265358979323846, measure_cdf(a.meas, p[l], l)));
    }
    series_block<D, 1, k1_s2(D), k1_lt(D)>(sm, t2s, a.tiles, alpha_row, c1, y);
    if (r < n) out[r] = with_weight ? DMUL(y[0], damping_weight<D>(p, q)) : y[0];
}

// mse_metrics (benchmark.cpp:86-151): per (step i, point m) squared errors of
// the damped series against exact_solution/weight (benchmark.cpp:20-28).
template <int D>
__global__ void __launch_bounds__(kK1Threads) k_mse(const StepArgs a, double kappa, double lam, double horizon,
                                                    uint64_t eval_seed, int eval_points, double* sq,
                                                    double* sq_u) {
    extern __shared__ __align__(16) unsigned char dsm[];
    SeriesSmem& sm = *reinterpret_cast<SeriesSmem*>(dsm);
    double* t2s = reinterpret_cast<double*>(dsm + sizeof(SeriesSmem));
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t r = r0 < eval_points ? r0 : eval_points - 1;
    const int i = blockIdx.y;
    Stream s(eval_seed, sid_evaluation(i, static_cast<uint64_t>(r)));
    double p[D], c1[1][D], y[1];
#pragma unroll
    for (int l = 0; l < D; ++l) {
        p[l] = measure_inv_cdf(a.meas, s.next_uniform(), l);
        c1[0][l] = cos(DMUL(3.14159265358979323846, measure_cdf(a.meas, p[l], l)));
    }
    const double w = damping_weight<D>(p, a.q);
    series_block<D, 1, k1_s2(D), k1_lt(D)>(sm, t2s, a.tiles, a.alpha_packed + static_cast<int64_t>(i) * a.kp, c1, y);
    if (r0 >= eval_points) return;
    const double approx = y[0];
    const double t = DMUL(static_cast<double>(i), a.dt);
    const double e_exp = exp(DDIV(DMUL(DMUL(DMUL(lam, lam), static_cast<double>(D)), DSUB(t, horizon)), 2.0));
    const double truth = DADD(DADD(1.0, kappa), DMUL(sin(DMUL(lam, sum_of<D>(p))), e_exp));
    const double e = DSUB(approx, DDIV(truth, w));
    sq[static_cast<int64_t>(i) * eval_points + r] = DMUL(e, e);
    sq_u[static_cast<int64_t>(i) * eval_points + r] = DMUL(DMUL(DMUL(e, e), w), w);
}

// ---------------------------------------------------------------- dispatch
// QRMC_ONLY_DIM=n (tuning builds only) instantiates the kernels for D = n alone.
#if !defined(QRMC_ONLY_DIM) || QRMC_ONLY_DIM == 1
#define QRMC_DCASE1(...) case 1: { constexpr int D = 1; __VA_ARGS__; } break;
#else
#define QRMC_DCASE1(...)
#endif
#if !defined(QRMC_ONLY_DIM) || QRMC_ONLY_DIM == 2
#define QRMC_DCASE2(...) case 2: { constexpr int D = 2; __VA_ARGS__; } break;
#else
#define QRMC_DCASE2(...)
#endif
#if !defined(QRMC_ONLY_DIM) || QRMC_ONLY_DIM == 3
#define QRMC_DCASE3(...) case 3: { constexpr int D = 3; __VA_ARGS__; } break;
#else
#define QRMC_DCASE3(...)
#endif
#if !defined(QRMC_ONLY_DIM) || QRMC_ONLY_DIM == 4
#define QRMC_DCASE4(...) case 4: { constexpr int D = 4; __VA_ARGS__; } break;
#else
#define QRMC_DCASE4(...)
#endif
#if !defined(QRMC_ONLY_DIM) || QRMC_ONLY_DIM == 5
#define QRMC_DCASE5(...) case 5: { constexpr int D = 5; __VA_ARGS__; } break;
#else
#define QRMC_DCASE5(...)
#endif
#if !defined(QRMC_ONLY_DIM) || QRMC_ONLY_DIM == 6
#define QRMC_DCASE6(...) case 6: { constexpr int D = 6; __VA_ARGS__; } break;
#else
#define QRMC_DCASE6(...)
#endif
#if !defined(QRMC_ONLY_DIM) || QRMC_ONLY_DIM == 7
#define QRMC_DCASE7(...) case 7: { constexpr int D = 7; __VA_ARGS__; } break;
#else
#define QRMC_DCASE7(...)
#endif
#if !defined(QRMC_ONLY_DIM) || QRMC_ONLY_DIM == 8
#define QRMC_DCASE8(...) case 8: { constexpr int D = 8; __VA_ARGS__; } break;
#else
#define QRMC_DCASE8(...)
#endif
#define QRMC_DISPATCH_D(dim, ...)                                                     \
    switch (dim) {                                                                     \
        QRMC_DCASE1(__VA_ARGS__) QRMC_DCASE2(__VA_ARGS__) QRMC_DCASE3(__VA_ARGS__)     \
        QRMC_DCASE4(__VA_ARGS__) QRMC_DCASE5(__VA_ARGS__) QRMC_DCASE6(__VA_ARGS__)     \
        QRMC_DCASE7(__VA_ARGS__) QRMC_DCASE8(__VA_ARGS__)                              \
        default: return cudaErrorInvalidValue;                                         \
    }

// Opt every series kernel into > 48 KiB of dynamic shared memory (once per process).
cudaError_t configure_series_kernels() {
    static cudaError_t status = [] {
        cudaError_t e = cudaSuccess;
        auto set = [&](const void* f, size_t bytes) {
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
        };
#define QRMC_CONFIGURE(Dv)                                                                           \
    set(reinterpret_cast<const void*>(&k_responses<Dv>), series_smem_bytes<Dv>(k1_p(Dv), true));          \
    set(reinterpret_cast<const void*>(&k_eval_points<Dv>), series_smem_bytes<Dv>(1));              \
    set(reinterpret_cast<const void*>(&k_mse<Dv>), series_smem_bytes<Dv>(1));
#ifdef QRMC_ONLY_DIM
        QRMC_CONFIGURE(QRMC_ONLY_DIM)
#else
        QRMC_CONFIGURE(1) QRMC_CONFIGURE(2) QRMC_CONFIGURE(3) QRMC_CONFIGURE(4)
        QRMC_CONFIGURE(5) QRMC_CONFIGURE(6) QRMC_CONFIGURE(7) QRMC_CONFIGURE(8)
#endif
#undef QRMC_CONFIGURE
        return e;
    }();
    return status;
}

cudaError_t launch_responses(const StepArgs& a, cudaStream_t st) {
    if (a.n_owned == 0) return cudaSuccess;
    QRMC_DISPATCH_D(a.prob.dim, {
        const int64_t per_cta = static_cast<int64_t>(kK1Threads) * k1_p(D);
        const unsigned blocks = static_cast<unsigned>((a.n_owned + per_cta - 1) / per_cta);
        k_responses<D><<<blocks, kK1Threads, series_smem_bytes<D>(k1_p(D), true), st>>>(a);
    });
    return cudaGetLastError();
}

size_t project_smem_bytes(const ProjArgs& p) {
    return (static_cast<size_t>(p.batch) * p.table_len + p.batch) * sizeof(double);
}

cudaError_t launch_project(const StepArgs& a, const ProjArgs& p, cudaStream_t st) {
    const unsigned tiles = static_cast<unsigned>((p.n_items + kProjThreads * kProjItems - 1) /
                                                 (kProjThreads * kProjItems));
    const dim3 grid(tiles, static_cast<unsigned>(a.owned_lanes));
    const size_t smem = project_smem_bytes(p);
    QRMC_DISPATCH_D(a.prob.dim, (k_project<D><<<grid, kProjThreads, smem, st>>>(a, p)));
    return cudaGetLastError();
}

cudaError_t configure_project(int dim, size_t smem) {
    cudaError_t e = cudaSuccess;
    QRMC_DISPATCH_D(dim, (e = cudaFuncSetAttribute(k_project<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(smem))));
    return e;
}

cudaError_t launch_finish(const StepArgs& a, const FinishArgs& f, cudaStream_t st) {
    const unsigned blocks = static_cast<unsigned>((f.basis_size + 255) / 256);
    k_finish_step<<<blocks, 256, 0, st>>>(a, f);
    return cudaGetLastError();
}

cudaError_t launch_philox(const uint32_t* ctr, const uint32_t* key, int64_t n, uint32_t* out,
                          cudaStream_t st) {
    const unsigned blocks = static_cast<unsigned>((n + 255) / 256);
    k_philox<<<blocks, 256, 0, st>>>(reinterpret_cast<const uint4*>(ctr),
                                     reinterpret_cast<const uint2*>(key), n,
                                     reinterpret_cast<uint4*>(out));
    return cudaGetLastError();
}

cudaError_t launch_stream_draws(uint64_t seed, const uint64_t* sids, int64_t n, int n_draws, int kind,
                                void* out, cudaStream_t st) {
    const unsigned blocks = static_cast<unsigned>((n + 127) / 128);
    k_stream_draws<<<blocks, 128, 0, st>>>(seed, sids, n, n_draws, kind, out);
    return cudaGetLastError();
}

cudaError_t launch_cloud_paths(const StepArgs& a, int64_t first, int64_t n, double* out, int* bad,
                               cudaStream_t st) {
    const unsigned blocks = static_cast<unsigned>((n + 127) / 128);
    QRMC_DISPATCH_D(a.prob.dim, (k_cloud_paths<D><<<blocks, 128, 0, st>>>(a, first, n, out, bad)));
    return cudaGetLastError();
}

cudaError_t launch_eval_points(const StepArgs& a, const double* alpha_row, const double* x, int64_t n,
                               double q, int with_weight, double* out, cudaStream_t st) {
    const unsigned blocks = static_cast<unsigned>((n + 127) / 128);
    QRMC_DISPATCH_D(a.prob.dim, (k_eval_points<D><<<blocks, kK1Threads, series_smem_bytes<D>(1), st>>>(a, alpha_row, x, n, q, with_weight, out)));
    return cudaGetLastError();
}

cudaError_t launch_mse(const StepArgs& a, double kappa, double lam, double horizon, uint64_t eval_seed,
                       int eval_points, double* sq, double* sq_u, cudaStream_t st) {
    const dim3 grid(static_cast<unsigned>((eval_points + 127) / 128), static_cast<unsigned>(a.steps));
    QRMC_DISPATCH_D(a.prob.dim, (k_mse<D><<<grid, kK1Threads, series_smem_bytes<D>(1), st>>>(a, kappa, lam, horizon, eval_seed, eval_points, sq, sq_u)));
    return cudaGetLastError();
}

}  // namespace qrmc_dev

// series_block.cuh -- block-cooperative evaluation of the Student-cosine series
//     y(x) = sum_{k in Gamma} alpha_k prod_l T_l[k_l](x)       (cosine_basis.cpp:67-112)
// for P points per thread, all threads of a CTA on the same coefficient row.
//
// Sum factorisation over Gamma's lexicographic trie. With c_l[v] = cos(v pi u_l)
// and alpha'_k = alpha_k sqrt2^{nnz(k)} (packed by host.cpp):
//     y = sum_{upper prefix} (prod_{l<D-2} c_l) sum_s c_{D-2}[s] sum_b alpha'[.., s, b] c_{D-1}[b]
// Leaf values c_{D-1}[0..LT) live in a per-point REGISTER table (static
// indices: the run length is static inside a segment loop), sibling weights c_{D-2}[0..S2) in a per-thread SHARED
// table (one LDS per run), both computed once per evaluation with the
// reference's three-term recurrence (cosine_basis.cpp:79-86); indices past
// the tables continue that recurrence in registers. Levels above D-2 change
// rarely and carry (2c1, c_prev, c_cur, acc) recurrence state.
//
// Program (host.cpp build_program): a stream of 32-bit words per tile,
//   group header: bits 0..11 number of segments, 12..15 transition level L of
//                 the upper prefix (15: first group), 16..27 first sibling s0,
//                 bit 28: continuation of the previous tile's group
//   segment word: bits 0..9 pair offset of its coefficients in the tile,
//                 10..21 run length R, 22..31 number of runs (consecutive
//                 siblings whose leaf runs all have length R)
// One dispatch per segment into a loop whose body is static for R <= LT, so
// a run costs R FMAs + 1 fold per point and a few loads. Tiles hold <= kTileA
// coefficients and <= kTileW words and stream through shared memory with
// cp.async double buffering. Control flow is uniform across the
// CTA (every thread walks the same program), so it never diverges.
#pragma once

#include <cstdint>

#include "kernels.cuh"

#ifndef QRMC_HYP_JOINT
#define QRMC_HYP_JOINT 1
#endif

namespace qrmc_dev {

constexpr int kTileA = kSeriesTileA;  // coefficients per shared-memory tile
constexpr int kTileW = kSeriesTileW;  // program words per tile
constexpr int kFirstGroup = 15; // transition code of the first group

struct SeriesSmem {
    double alpha[2][kTileA + 8];  // +8: the leaf chain preloads 4 pairs, possibly past a tile's end
    uint32_t prog[2][kTileW + 4];
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

__device__ __forceinline__ void load_tile(SeriesSmem& sm, int buf, const SeriesTiles& st, const double* row,
                                          int t) {
    const int4 d = st.tiles[t];
    const int na = d.w >> 1;  // 16-byte chunks of coefficients
    const double* ga = row + d.z;
    for (int c = threadIdx.x; c < na; c += blockDim.x) cp_async16(&sm.alpha[buf][2 * c], ga + 2 * c);
    const int np = (d.y + 3) >> 2;  // four words per 16-byte chunk
    const uint32_t* gp = st.prog + d.x;
    for (int c = threadIdx.x; c < np; c += blockDim.x) cp_async16(&sm.prog[buf][4 * c], gp + 4 * c);
}

// The sibling runs of one segment: cnt consecutive siblings s, s+1, ... whose
// leaf runs all have length R; coefficients contiguous, each run padded to even.
template <int P, int S2, int LT>
struct SegState {
    const double (&leaf)[P][LT];
    const double (&tl)[P];
    const double (&t2c)[P];
    const double* t2 /* t2s + tid */;
    int nt;
    double (&g2p)[P];
    double (&g2c)[P];
    double (&acc2)[P];
    double (&acc2b)[P];  // second accumulator: odd leaf indices (independent FMA chain)

    // sibling weight c_{D-2}[s]: shared table below S2, recurrence (in order) above
    __device__ __forceinline__ void weight(int s, double (&ts)[P]) {
        if (s < S2) {
#pragma unroll
            for (int p = 0; p < P; ++p) ts[p] = t2[(s * P + p) * nt];
        } else {
#pragma unroll
            for (int p = 0; p < P; ++p) {
                const double c = fma(t2c[p], g2c[p], -g2p[p]);
                g2p[p] = g2c[p];
                g2c[p] = c;
                ts[p] = c;
            }
        }
    }

    // R <= LT: fully static run body, R FMAs + 1 fold per point per run. The
    // siblings below S2 (shared table) and above (recurrence) run as two loops
    // so neither path is predicated into the other.
    template <int R>
    __device__ __forceinline__ void run_fixed(const double2* ra, int s, int cnt) {
        constexpr int NP = (R + 1) / 2;
        auto body = [&](const double (&ts)[P]) {
            // even / odd leaf indices in two independent chains (ILP), folded with
            // two FMAs so no add sits on the critical path
            double z0[P], z1[P];
#pragma unroll
            for (int j = 0; j < NP; ++j) {
                const double2 a = ra[j];
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    z0[p] = j == 0 ? a.x * leaf[p][0] : fma(a.x, leaf[p][2 * j], z0[p]);
                    if (2 * j + 1 < R) z1[p] = j == 0 ? a.y * leaf[p][1] : fma(a.y, leaf[p][2 * j + 1], z1[p]);
                }
            }
#pragma unroll
            for (int p = 0; p < P; ++p) {
                acc2[p] = fma(ts[p], z0[p], acc2[p]);
                if (R > 1) acc2b[p] = fma(ts[p], z1[p], acc2b[p]);
            }
            ra += NP;
        };
        int n_tab = S2 - s;
        n_tab = n_tab < 0 ? 0 : (n_tab > cnt ? cnt : n_tab);
        const double* tp = t2 + s * P * nt;
#pragma unroll 2
        for (int k = 0; k < n_tab; ++k) {
            double ts[P];
#pragma unroll
            for (int p = 0; p < P; ++p) ts[p] = tp[p * nt];
            tp += P * nt;
            body(ts);
        }
        for (int k = n_tab; k < cnt; ++k) {
            double ts[P];
#pragma unroll
            for (int p = 0; p < P; ++p) {
                const double c = fma(t2c[p], g2c[p], -g2p[p]);
                g2p[p] = g2c[p];
                g2c[p] = c;
                ts[p] = c;
            }
            body(ts);
        }
    }

    // R > LT: the register table, then the Chebyshev recurrence (2 FMAs per term)
    __device__ __forceinline__ void run_long(const double2* ra, int R, int s, int cnt) {
        const int np = (R + 1) >> 1;
        for (int k = 0; k < cnt; ++k, ra += np) {
            double ts[P];
            weight(s + k, ts);
            double z[P], cp[P], cc[P];
#pragma unroll
            for (int p = 0; p < P; ++p) z[p] = 0.0;
#pragma unroll
            for (int j = 0; j < LT / 2; ++j) {
                const double2 a = ra[j];
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    z[p] = fma(a.x, leaf[p][2 * j], z[p]);
                    z[p] = fma(a.y, leaf[p][2 * j + 1], z[p]);
                }
            }
#pragma unroll
            for (int p = 0; p < P; ++p) {
                cp[p] = leaf[p][LT - 2];
                cc[p] = leaf[p][LT - 1];
            }
            for (int j = LT / 2; j < np; ++j) {
                const double2 a = ra[j];
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    const double e = fma(tl[p], cc[p], -cp[p]);  // c_{2j}
                    const double o = fma(tl[p], e, -cc[p]);      // c_{2j+1}
                    z[p] = fma(a.x, e, z[p]);
                    z[p] = fma(a.y, o, z[p]);
                    cp[p] = e;
                    cc[p] = o;
                }
            }
#pragma unroll
            for (int p = 0; p < P; ++p) acc2[p] = fma(ts[p], z[p], acc2[p]);
        }
    }
};

// Groups whose sibling runs follow the hyperbolic profile of budget B,
// R_s = floor(B / max(s,1)) + 1 for s = 0..B (every group of a hyperbolic
// index set whose upper prefix leaves budget B), are evaluated by fully static
// straight-line code: no segment dispatch, no loop control, static shared-memory
// offsets, and the c_0 = 1 leaf/sibling products folded away. These small
// groups are the most frequent ones (C2: 50% of the terms for B <= 15, C4: 73%).
// Siblings 0 and 1 share the longest run (B + 1) and are swept together, with
// leaf values past the register table continued by the Chebyshev recurrence
// (computed once for both); siblings past the shared table S2 continue theirs.
__host__ __device__ constexpr int hyp_run(int B, int s) { return B / (s > 1 ? s : 1) + 1; }
__host__ __device__ constexpr int hyp_pairs_before(int B, int s) {
    int o = 0;
    for (int t = 0; t < s; ++t) o += (hyp_run(B, t) + 1) / 2;
    return o;
}
// the device can run profile B with a leaf table of LT entries
__host__ __device__ constexpr bool hyp_supported(int B, int LT) {
    return B >= 1 && B <= kHypMaxB && LT >= 2;
}

template <int B, int P, int S2, int LT>
struct Hyp {
    const double2* ra;
    const double (&leaf)[P][LT];
    const double (&tl)[P];   // 2 c_{D-1}[1]
    const double (&t2c)[P];  // 2 c_{D-2}[1]
    const double* t2;        // t2s + tid
    int nt;
    double (&acc)[P];

    __device__ __forceinline__ void first_two() {
        constexpr int R = B + 1;
        constexpr int NP = (R + 1) / 2;
        double z0[P], z1[P], cp[P], cc[P];
#pragma unroll
        for (int p = 0; p < P; ++p) {
            cp[p] = leaf[p][LT - 2];
            cc[p] = leaf[p][LT - 1];
        }
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            const double2 a0 = ra[j], a1 = ra[NP + j];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int b = 2 * j + h;
                if (b < R) {
#pragma unroll
                    for (int p = 0; p < P; ++p) {
                        double c;
                        if (b < LT) {
                            c = leaf[p][b < LT ? b : 0];
                        } else {
                            c = fma(tl[p], cc[p], -cp[p]);
                            cp[p] = cc[p];
                            cc[p] = c;
                        }
                        const double x0 = h ? a0.y : a0.x, x1 = h ? a1.y : a1.x;
                        z0[p] = b == 0 ? x0 : fma(x0, c, z0[p]);  // c_0 = 1
                        z1[p] = b == 0 ? x1 : fma(x1, c, z1[p]);
                    }
                }
            }
        }
#pragma unroll
        for (int p = 0; p < P; ++p) acc[p] = fma(t2[(1 * P + p) * nt], z1[p], acc[p] + z0[p]);
    }

    // c2p, c2c enter as (c_{S2-2}, c_{S2-1}) of level D-2 (the group's g2p, g2c)
    template <int S>
    __device__ __forceinline__ void sibling(double (&c2p)[P], double (&c2c)[P]) {
        constexpr int R = hyp_run(B, S);
        constexpr int NP = (R + 1) / 2;
        constexpr int OFF = hyp_pairs_before(B, S);
        double z[P], cp[P], cc[P];
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            const double2 a = ra[OFF + j];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int b = 2 * j + h;
                if (b < R) {
#pragma unroll
                    for (int p = 0; p < P; ++p) {
                        double c;
                        if (b < LT) {
                            c = leaf[p][b < LT ? b : 0];
                        } else {  // past the leaf table: Chebyshev recurrence
                            if (b == LT) {
                                cp[p] = leaf[p][LT - 2];
                                cc[p] = leaf[p][LT - 1];
                            }
                            c = fma(tl[p], cc[p], -cp[p]);
                            cp[p] = cc[p];
                            cc[p] = c;
                        }
                        const double x = h ? a.y : a.x;
                        z[p] = b == 0 ? x : fma(x, c, z[p]);  // c_0 = 1
                    }
                }
            }
        }
#pragma unroll
        for (int p = 0; p < P; ++p) {
            if constexpr (S == 0) {
                acc[p] += z[p];
            } else {
                double ts;
                if constexpr (S < S2) {
                    ts = t2[(S * P + p) * nt];
                } else {
                    ts = fma(t2c[p], c2c[p], -c2p[p]);
                    c2p[p] = c2c[p];
                    c2c[p] = ts;
                }
                acc[p] = fma(ts, z[p], acc[p]);
            }
        }
        if constexpr (S < B) sibling<S + 1>(c2p, c2c);
    }

    __device__ __forceinline__ void run(double (&c2p)[P], double (&c2c)[P]) {
#if QRMC_HYP_JOINT
        if constexpr (B + 1 > LT) {  // siblings 0 and 1 share one recurrence past the table
            first_two();
            if constexpr (B >= 2) sibling<2>(c2p, c2c);
            return;
        }
#endif
        sibling<0>(c2p, c2c);
    }
};

template <int P, int S2, int LT>
__device__ __forceinline__ void hyper_group(int B, const double2* ra, const double (&leaf)[P][LT],
                                            const double (&tl)[P], const double (&t2c)[P], const double* t2,
                                            int nt, double (&c2p)[P], double (&c2c)[P], double (&acc)[P]) {
    switch (B) {
#define QRMC_HYP(b)                                                      \
    case b:                                                              \
        if constexpr (hyp_supported((b), LT) && S2 >= 2)                 \
            Hyp<(b), P, S2, LT>{ra, leaf, tl, t2c, t2, nt, acc}.run(c2p, c2c); \
        break;
        QRMC_HYP(1) QRMC_HYP(2) QRMC_HYP(3) QRMC_HYP(4) QRMC_HYP(5) QRMC_HYP(6) QRMC_HYP(7) QRMC_HYP(8)
        QRMC_HYP(9) QRMC_HYP(10) QRMC_HYP(11) QRMC_HYP(12) QRMC_HYP(13) QRMC_HYP(14) QRMC_HYP(15)
#undef QRMC_HYP
        default: break;
    }
}

// Evaluate the series of coefficient row `row` at P points per thread.
// c1[p][l] = cos(pi u_l) of point p; t2s: shared scratch of S2*P*blockDim doubles.
// Must be called by every thread of the CTA.
template <int D, int P, int S2, int LT>
__device__ __forceinline__ void series_block(SeriesSmem& sm, double* t2s, const SeriesTiles& st,
                                             const double* row, const double (&c1)[P][D], double (&y)[P]) {
    static_assert(LT % 2 == 0 && LT >= 4 && LT <= 32 && S2 >= 2, "table sizes");
    constexpr int NU = D > 2 ? D - 2 : 1;  // upper levels 0..D-3
    const int tid = threadIdx.x, nt = blockDim.x;
    double utc[P][NU], ucur[P][NU], uprev[P][NU], uacc[P][NU];
    double leaf[P][LT], tl[P], t2c[P], acc2[P], acc2b[P], g2p[P], g2c[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
#pragma unroll
        for (int l = 0; l < NU; ++l) {
            const double c = D > 2 ? c1[p][l] : 0.0;
            utc[p][l] = 2.0 * c;
            ucur[p][l] = 1.0;
            uprev[p][l] = c;  // c_{-1} = c_1: the first advance yields c_1 exactly
            uacc[p][l] = 0.0;
        }
        // sibling table c_{D-2}[0..S2) -> shared memory, layout [s][p][tid]
        const double cs = D >= 2 ? c1[p][D >= 2 ? D - 2 : 0] : 1.0;
        t2c[p] = 2.0 * cs;
        double a = 1.0, b = cs;
        t2s[(0 * P + p) * nt + tid] = a;
        t2s[(1 * P + p) * nt + tid] = b;
#pragma unroll
        for (int s = 2; s < S2; ++s) {
            const double c = fma(t2c[p], b, -a);
            t2s[(s * P + p) * nt + tid] = c;
            a = b;
            b = c;
        }
        g2p[p] = a;  // (c_{S2-2}, c_{S2-1}): start of the recurrence past the table
        g2c[p] = b;
        const double cl = c1[p][D - 1];
        tl[p] = 2.0 * cl;
        leaf[p][0] = 1.0;
        leaf[p][1] = cl;
#pragma unroll
        for (int k = 2; k < LT; ++k) leaf[p][k] = fma(tl[p], leaf[p][k - 1], -leaf[p][k - 2]);
        acc2[p] = 0.0;
        acc2b[p] = 0.0;
    }
    load_tile(sm, 0, st, row, 0);
    cp_async_commit();
    for (int t = 0; t < st.n_tiles; ++t) {
        const int buf = t & 1;
        if (t + 1 < st.n_tiles) {
            load_tile(sm, buf ^ 1, st, row, t + 1);
            cp_async_commit();
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const int n_words = st.tiles[t].y;
        const uint32_t* pw = sm.prog[buf];
        const double2* pa = reinterpret_cast<const double2*>(sm.alpha[buf]);
        int i = 0;
        while (i < n_words) {
            const uint32_t h = pw[i++];
            const int n_seg = static_cast<int>(h & 0xFFFu);
            int s = static_cast<int>((h >> 16) & 0xFFFu);
            if (!(h & (1u << 28))) {
                // a new group: close the previous one and the upper nodes above it,
                // advance level L of the upper prefix
                const int L = static_cast<int>((h >> 12) & 15u);
                if constexpr (D > 2) {
                    if (L != kFirstGroup) {
#pragma unroll
                        for (int p = 0; p < P; ++p) {
                            uacc[p][D - 3] = fma(ucur[p][D - 3], acc2[p] + acc2b[p], uacc[p][D - 3]);
#pragma unroll
                            for (int l = D - 4; l >= 0; --l) {
                                if (l >= L) {
                                    uacc[p][l] = fma(ucur[p][l], uacc[p][l + 1], uacc[p][l]);
                                    uacc[p][l + 1] = 0.0;
                                }
                            }
#pragma unroll
                            for (int l = 0; l < D - 2; ++l) {
                                if (l == L) {
                                    const double nx = fma(utc[p][l], ucur[p][l], -uprev[p][l]);
                                    uprev[p][l] = ucur[p][l];
                                    ucur[p][l] = nx;
                                } else if (l > L) {
                                    ucur[p][l] = 1.0;
                                    uprev[p][l] = 0.5 * utc[p][l];
                                }
                            }
                        }
                    }
                }
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    acc2[p] = 0.0;
                    acc2b[p] = 0.0;
                    g2p[p] = t2s[((S2 - 2) * P + p) * nt + tid];
                    g2c[p] = t2s[((S2 - 1) * P + p) * nt + tid];
                }
            }
            if (h & (1u << 29)) {
                // hyperbolic-profile group: one word {pair offset, B}, static code
                const uint32_t w = pw[i++];
                hyper_group<P, S2, LT>(static_cast<int>(w >> 16), pa + (w & 0x3FFu), leaf, tl, t2c, t2s + tid, nt, g2p, g2c, acc2);
                continue;
            }
            SegState<P, S2, LT> ss{leaf, tl, t2c, t2s + tid, nt, g2p, g2c, acc2, acc2b};
            for (int g = 0; g < n_seg; ++g) {
                const uint32_t w = pw[i++];
                const double2* ra = pa + (w & 0x3FFu);
                const int R = static_cast<int>((w >> 10) & 0xFFFu);
                const int cnt = static_cast<int>(w >> 22);
                // one dispatch per segment of equal-length runs
                switch (R) {
#define QRMC_SEG(r) \
    case r:         \
        if constexpr ((r) <= LT) ss.template run_fixed<(r)>(ra, s, cnt); \
        break;
                    QRMC_SEG(1) QRMC_SEG(2) QRMC_SEG(3) QRMC_SEG(4) QRMC_SEG(5) QRMC_SEG(6) QRMC_SEG(7)
                    QRMC_SEG(8) QRMC_SEG(9) QRMC_SEG(10) QRMC_SEG(11) QRMC_SEG(12) QRMC_SEG(13) QRMC_SEG(14)
                    QRMC_SEG(15) QRMC_SEG(16) QRMC_SEG(17) QRMC_SEG(18) QRMC_SEG(19) QRMC_SEG(20) QRMC_SEG(21)
                    QRMC_SEG(22) QRMC_SEG(23) QRMC_SEG(24) QRMC_SEG(25) QRMC_SEG(26) QRMC_SEG(27) QRMC_SEG(28)
                    QRMC_SEG(29) QRMC_SEG(30) QRMC_SEG(31) QRMC_SEG(32)
#undef QRMC_SEG
                    default: break;
                }
                if (R > LT) ss.run_long(ra, R, s, cnt);
                s += cnt;
            }
        }
        __syncthreads();  // the buffer is refilled by the next iteration's prefetch
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
        if constexpr (D > 2) {
            uacc[p][D - 3] = fma(ucur[p][D - 3], acc2[p] + acc2b[p], uacc[p][D - 3]);
#pragma unroll
            for (int l = D - 4; l >= 0; --l) uacc[p][l] = fma(ucur[p][l], uacc[p][l + 1], uacc[p][l]);
            y[p] = uacc[p][0];
        } else {
            y[p] = acc2[p] + acc2b[p];
        }
    }
}

}  // namespace qrmc_dev

// series_block.cuh -- block-cooperative evaluation of the Student-cosine series
//     y(x) = sum_{k in Gamma} alpha_k prod_l T_l[k_l](x)       (cosine_basis.cpp:67-112)
// for P points per thread, all threads of a CTA on the same coefficient row.
//
// Sum factorisation over Gamma's lexicographic trie. With c_l[v] = cos(v pi u_l)
// and alpha'_k = alpha_k sqrt2^{nnz(k)} (packed by host.cpp):
//     y = sum_{upper prefix} (prod_{l<D-2} c_l) sum_s c_{D-2}[s] sum_b alpha'[.., s, b] c_{D-1}[b]
// The two deepest levels are evaluated from per-point REGISTER tables,
// c_{D-2}[0..S2) and c_{D-1}[0..LT), computed once per evaluation, so every
// term inside the tables costs exactly one FMA and every leaf run one more
// (its fold into the sibling sum). Indices beyond the tables continue the
// reference's three-term Chebyshev recurrence (cosine_basis.cpp:79-86) in
// registers. Levels above D-2 ("upper" levels) change rarely and carry
// (2c1, c_prev, c_cur, acc) recurrence state.
//
// Program (host.cpp build_program): one GROUP per upper prefix (k_0..k_{D-3}),
//   word 0: bits 0..3  transition level L of the upper prefix vs the previous
//                      group (kFirstGroup for the first, kContGroup when the
//                      group continues from the previous tile),
//           bits 4..17 number of sibling runs n in this chunk,
//           bits 18..31 first sibling index s0 (0, or >= S2 for continuations)
//   words 1..n: leaf run lengths R_s (leaf indices 0..R_s-1)
// and the packed coefficients of each run, padded to even length. Groups are
// cut into tiles (<= kTileA coefficients, <= kTileP words) that stream
// through shared memory with cp.async double buffering; inner loops read
// coefficients as 16-byte shared-memory broadcasts. Control flow is uniform
// across the CTA (every thread walks the same program), so it never diverges.
#pragma once

#include <cstdint>

#include "kernels.cuh"

namespace qrmc_dev {

constexpr int kTileA = 2048;    // coefficients per shared-memory tile (16 KiB)
constexpr int kTileP = 1024;    // program words per tile (4 KiB)
constexpr int kFirstGroup = 15; // transition code of the first group
constexpr int kContGroup = 14;  // continuation of the previous tile's group

struct SeriesSmem {
    double alpha[2][kTileA];
    uint32_t prog[2][kTileP];
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void load_tile(SeriesSmem& sm, int buf, const SeriesTiles& st, const double* row,
                                          int t) {
    const int4 d = st.tiles[t];
    const int na = d.w >> 1;  // 16-byte chunks of coefficients
    const double* ga = row + d.z;
    for (int c = threadIdx.x; c < na; c += blockDim.x) cp_async16(&sm.alpha[buf][2 * c], ga + 2 * c);
    const int np = (d.y + 3) >> 2;
    const uint32_t* gp = st.prog + d.x;
    for (int c = threadIdx.x; c < np; c += blockDim.x) cp_async16(&sm.prog[buf][4 * c], gp + 4 * c);
}

// Leaf run z = sum_{b<R} alpha'[b] c_b for P points; pa advances past the run.
template <int P, int LT>
__device__ __forceinline__ void leaf_run(const double2*& pa, int R, const double (&leaf)[P][LT],
                                         const double (&tl)[P], double (&z0)[P], double (&z1)[P]) {
#pragma unroll
    for (int p = 0; p < P; ++p) z0[p] = z1[p] = 0.0;
#pragma unroll
    for (int b2 = 0; b2 < LT / 2; ++b2) {
        if (2 * b2 < R) {
            const double2 a = pa[b2];
#pragma unroll
            for (int p = 0; p < P; ++p) {
                z0[p] = fma(a.x, leaf[p][2 * b2], z0[p]);
                z1[p] = fma(a.y, leaf[p][2 * b2 + 1], z1[p]);
            }
        }
    }
    if (R > LT) {
        double cp[P], cc[P];
#pragma unroll
        for (int p = 0; p < P; ++p) {
            cp[p] = leaf[p][LT - 2];
            cc[p] = leaf[p][LT - 1];
        }
        const int pairs = (R + 1) >> 1;
        for (int b2 = LT / 2; b2 < pairs; ++b2) {
            const double2 a = pa[b2];
#pragma unroll
            for (int p = 0; p < P; ++p) {
                const double e = fma(tl[p], cc[p], -cp[p]);  // c_{2 b2}
                const double o = fma(tl[p], e, -cc[p]);      // c_{2 b2 + 1}
                z0[p] = fma(a.x, e, z0[p]);
                z1[p] = fma(a.y, o, z1[p]);
                cp[p] = e;
                cc[p] = o;
            }
        }
    }
    pa += (R + 1) >> 1;
}

// Evaluate the series of coefficient row `row` at P points per thread.
// c1[p][l] = cos(pi u_l) of point p. Must be called by every thread of the CTA.
template <int D, int P, int S2, int LT>
__device__ __forceinline__ void series_block(SeriesSmem& sm, const SeriesTiles& st, const double* row,
                                             const double (&c1)[P][D], double (&y)[P]) {
    static_assert(LT % 2 == 0 && LT >= 2 && S2 >= 2, "table sizes");
    constexpr int NU = D > 2 ? D - 2 : 1;  // upper levels 0..D-3
    double utc[P][NU], ucur[P][NU], uprev[P][NU], uacc[P][NU];
    double t2[P][S2], leaf[P][LT], tl[P], t2c[P];
    double acc2[P], g2p[P], g2c[P];  // sibling sum of the current group; recurrence past S2
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
        const double cs = D >= 2 ? c1[p][D >= 2 ? D - 2 : 0] : 1.0;
        t2c[p] = 2.0 * cs;
        t2[p][0] = 1.0;
        t2[p][1] = cs;
#pragma unroll
        for (int s = 2; s < S2; ++s) t2[p][s] = fma(t2c[p], t2[p][s - 1], -t2[p][s - 2]);
        const double cl = c1[p][D - 1];
        tl[p] = 2.0 * cl;
        leaf[p][0] = 1.0;
        leaf[p][1] = cl;
#pragma unroll
        for (int b = 2; b < LT; ++b) leaf[p][b] = fma(tl[p], leaf[p][b - 1], -leaf[p][b - 2]);
        acc2[p] = 0.0;
        g2p[p] = t2[p][S2 - 2];
        g2c[p] = t2[p][S2 - 1];
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
        int wi = 0;
        while (wi < n_words) {
            const uint32_t h = pw[wi];
            const int L = static_cast<int>(h & 15u);
            const int n = static_cast<int>((h >> 4) & 0x3FFFu);
            const int s0 = static_cast<int>(h >> 18);
            const uint32_t* runs = pw + wi + 1;
            wi += 1 + n;
            if (L != kContGroup) {
                if (L != kFirstGroup) {
                    // close the finished group and the upper nodes above it, advance level L
#pragma unroll
                    for (int p = 0; p < P; ++p) {
                        if constexpr (D > 2) {
                            uacc[p][D - 3] = fma(ucur[p][D - 3], acc2[p], uacc[p][D - 3]);
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
                        acc2[p] = 0.0;
                    }
                }
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    g2p[p] = t2[p][S2 - 2];
                    g2c[p] = t2[p][S2 - 1];
                }
            }
            int s = 0;
            if (s0 == 0) {
                // siblings inside the register table: static indices
#pragma unroll
                for (int ss = 0; ss < S2; ++ss) {
                    if (ss < n) {
                        double z0[P], z1[P];
                        leaf_run<P, LT>(pa, static_cast<int>(runs[ss]), leaf, tl, z0, z1);
#pragma unroll
                        for (int p = 0; p < P; ++p) {
                            acc2[p] = fma(t2[p][ss], z0[p], acc2[p]);
                            acc2[p] = fma(t2[p][ss], z1[p], acc2[p]);
                        }
                    }
                }
                s = S2;
            }
            // siblings past the table (relative index ss, absolute s0 + ss >= S2):
            // advance the recurrence (g2p, g2c) = (c_{s-2}, c_{s-1})
            for (int ss = s; ss < n; ++ss) {
                double z0[P], z1[P];
                leaf_run<P, LT>(pa, static_cast<int>(runs[ss]), leaf, tl, z0, z1);
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    const double cs = fma(t2c[p], g2c[p], -g2p[p]);
                    g2p[p] = g2c[p];
                    g2c[p] = cs;
                    acc2[p] = fma(cs, z0[p] + z1[p], acc2[p]);
                }
            }
        }
        __syncthreads();  // the buffer is refilled by the next iteration's prefetch
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
        if constexpr (D > 2) {
            uacc[p][D - 3] = fma(ucur[p][D - 3], acc2[p], uacc[p][D - 3]);
#pragma unroll
            for (int l = D - 4; l >= 0; --l) uacc[p][l] = fma(ucur[p][l], uacc[p][l + 1], uacc[p][l]);
            y[p] = uacc[p][0];
        } else {
            y[p] = acc2[p];
        }
    }
}

}  // namespace qrmc_dev

// series_block.cuh -- block-cooperative evaluation of the Student-cosine series
//     y(x) = sum_{k in Gamma} alpha_k prod_l T_l[k_l](x)       (cosine_basis.cpp:67-112)
// for P points per thread, all threads of a CTA on the same coefficient row.
//
// Layout (built by host.cpp): the packed row alpha'_k = alpha_k sqrt2^{nnz(k)}
// in lexicographic (= depth-first trie) order, each leaf run padded to even
// length; the node program (one word per leaf run: bits 0..3 transition
// level L, 15 = first run of the set; bits 4.. run length R) cut into tiles
// of <= kTileA coefficients and <= kTileP runs, never splitting a run.
// Tiles stream HBM/L2 -> shared memory with cp.async, double-buffered, so
// the inner loops read coefficients as 16-byte shared-memory broadcasts.
//
// Per point the evaluation is sum factorisation over the trie (Horner on
// every level): the leaf level uses a register table of the first LT
// Chebyshev values c_b = cos(b pi u) (one FMA per term), runs longer than LT
// continue the three-term recurrence in registers; internal levels carry
// (c_prev, c_cur, 2c1, acc) in registers. Control flow is uniform across
// the CTA (every thread walks the same program), so branches never diverge.
#pragma once

#include <cstdint>

#include "kernels.cuh"

namespace qrmc_dev {

constexpr int kTileA = 2048;  // coefficients per shared-memory tile (16 KiB)
constexpr int kTileP = 1024;  // run words per tile (4 KiB)
constexpr int kFirstRun = 15; // transition code of a set's first run


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

// Evaluate the series of coefficient row `row` at P points per thread.
// c1[p][l] = cos(pi u_l) of point p. Must be called by every thread of the CTA.
template <int D, int P, int LT>
__device__ __forceinline__ void series_block(SeriesSmem& sm, const SeriesTiles& st, const double* row,
                                             const double (&c1)[P][D], double (&y)[P]) {
    static_assert(LT % 2 == 0 && LT >= 2, "leaf table holds pairs");
    constexpr int NI = D > 1 ? D - 1 : 1;  // internal levels 0..D-2
    double tc[P][NI], cur[P][NI], prev[P][NI], acc[P][NI];
    double leaf[P][LT];
#pragma unroll
    for (int p = 0; p < P; ++p) {
#pragma unroll
        for (int l = 0; l < NI; ++l) {
            const double c = D > 1 ? c1[p][l] : 0.0;
            tc[p][l] = 2.0 * c;
            cur[p][l] = 1.0;
            prev[p][l] = c;  // c_{-1} = c_1, so the first advance yields c_1 exactly
            acc[p][l] = 0.0;
        }
        const double cl = c1[p][D - 1], tl = 2.0 * cl;
        leaf[p][0] = 1.0;
        leaf[p][1] = cl;
#pragma unroll
        for (int b = 2; b < LT; ++b) leaf[p][b] = fma(tl, leaf[p][b - 1], -leaf[p][b - 2]);
        y[p] = 0.0;
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
        const int n_runs = st.tiles[t].y;
        const uint32_t* pw = sm.prog[buf];
        const double2* pa = reinterpret_cast<const double2*>(sm.alpha[buf]);
        for (int n = 0; n < n_runs; ++n) {
            const uint32_t w = pw[n];
            const int L = static_cast<int>(w & 15u);
            const int R = static_cast<int>(w >> 4);
            if constexpr (D >= 2) {
                if (L == D - 2) {
                    // sibling run: advance the deepest internal level
#pragma unroll
                    for (int p = 0; p < P; ++p) {
                        const double nx = fma(tc[p][D - 2], cur[p][D - 2], -prev[p][D - 2]);
                        prev[p][D - 2] = cur[p][D - 2];
                        cur[p][D - 2] = nx;
                    }
                } else if (L != kFirstRun) {
#pragma unroll
                    for (int p = 0; p < P; ++p) {
#pragma unroll
                        for (int l = D - 3; l >= 0; --l) {
                            if (l >= L) {
                                acc[p][l] = fma(cur[p][l], acc[p][l + 1], acc[p][l]);
                                acc[p][l + 1] = 0.0;
                            }
                        }
#pragma unroll
                        for (int l = 0; l < D - 1; ++l) {
                            if (l == L) {
                                const double nx = fma(tc[p][l], cur[p][l], -prev[p][l]);
                                prev[p][l] = cur[p][l];
                                cur[p][l] = nx;
                            } else if (l > L) {
                                cur[p][l] = 1.0;
                                prev[p][l] = 0.5 * tc[p][l];
                            }
                        }
                    }
                }
            }
            // leaf run: z = sum_{b<R} alpha'[b] c_b
            double z0[P], z1[P];
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
                // long run: continue the Chebyshev recurrence from (c_{LT-2}, c_{LT-1})
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
                        const double tl = 2.0 * leaf[p][1];
                        const double e = fma(tl, cc[p], -cp[p]);  // c_{2 b2}
                        const double o = fma(tl, e, -cc[p]);      // c_{2 b2 + 1}
                        z0[p] = fma(a.x, e, z0[p]);
                        z1[p] = fma(a.y, o, z1[p]);
                        cp[p] = e;
                        cc[p] = o;
                    }
                }
            }
            pa += (R + 1) >> 1;
#pragma unroll
            for (int p = 0; p < P; ++p) {
                const double z = z0[p] + z1[p];
                if constexpr (D >= 2)
                    acc[p][D - 2] = fma(cur[p][D - 2], z, acc[p][D - 2]);
                else
                    y[p] += z;
            }
        }
        __syncthreads();  // the buffer is refilled by the next iteration's prefetch
    }
    if constexpr (D >= 2) {
#pragma unroll
        for (int p = 0; p < P; ++p) {
#pragma unroll
            for (int l = D - 3; l >= 0; --l) acc[p][l] = fma(cur[p][l], acc[p][l + 1], acc[p][l]);
            y[p] = acc[p][0];
        }
    }
}

}  // namespace qrmc_dev

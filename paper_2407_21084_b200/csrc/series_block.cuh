// series_block.cuh -- block-cooperative evaluation of the Student-cosine series
//     y(x) = sum_{k in Gamma} alpha_k prod_l T_l[k_l](x)       (cosine_basis.cpp:67-112)
// for P points per thread, all threads of a CTA on the same coefficient row.
//
// Sum factorisation over Gamma's lexicographic trie. With c_l[v] = cos(v pi u_l)
// and alpha'_k = alpha_k sqrt2^{nnz(k)} (packed by host.cpp):
//     y = sum_{upper prefix} (prod_{l<D-2} c_l) sum_s c_{D-2}[s] sum_b alpha'[.., s, b] c_{D-1}[b]
// Leaf values c_{D-1}[0..LT) live in a per-point REGISTER table (static
// indices inside a Duff's-device jump table, so a run of R coefficients costs
// exactly R FMAs), sibling weights c_{D-2}[0..S2) in a per-thread SHARED
// table (one LDS per run), both computed once per evaluation with the
// reference's three-term recurrence (cosine_basis.cpp:79-86); indices past
// the tables continue that recurrence in registers. Levels above D-2 change
// rarely and carry (2c1, c_prev, c_cur, acc) recurrence state.
//
// Program (host.cpp build_program): one 64-bit word per leaf run,
//   x: bits 0..10  pair offset of the run's coefficients inside the tile
//      bits 11..22 run length R
//   y: bits 0..11  sibling index s = k_{D-2}
//      bit  12     first run of a group (upper prefix k_0..k_{D-3} changed)
//      bits 13..16 transition level L of that prefix change (15: first group)
// cut into tiles of <= kTileA coefficients / <= kTileP runs that stream
// through shared memory with cp.async double buffering. The node loop is
// software-pipelined: the next run's word and first coefficient pair are
// loaded while the current run computes. Control flow is uniform across the
// CTA (every thread walks the same program), so it never diverges.
#pragma once

#include <cstdint>

#include "kernels.cuh"
#include "leaf_chain.cuh"

namespace qrmc_dev {

constexpr int kTileA = 2048;    // coefficients per shared-memory tile (16 KiB)
constexpr int kTileP = 1024;    // runs per tile (8 KiB of words)
constexpr int kFirstGroup = 15; // transition code of the first group

struct SeriesSmem {
    double alpha[2][kTileA + 8];  // +8: the leaf chain preloads 4 pairs, possibly past a tile's end
    uint2 prog[2][kTileP + 2];    // + a zero word after the last run (pipelined prefetch)
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
    const int np = (d.y + 2) >> 1;  // two 8-byte words per chunk, incl. the zero pad word
    const uint32_t* gp = st.prog + d.x;
    for (int c = threadIdx.x; c < np; c += blockDim.x) cp_async16(&sm.prog[buf][2 * c], gp + 4 * c);
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
    double leaf[P][LT], tl[P], t2c[P], acc2[P], g2p[P], g2c[P];
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
        const uint2* pw = sm.prog[buf];
        const double2* pa = reinterpret_cast<const double2*>(sm.alpha[buf]);
        uint2 w = pw[0];  // pair offsets are < 1024 (masked 0x3FF)
        const unsigned pa_s = static_cast<unsigned>(__cvta_generic_to_shared(pa));
        for (int n = 0; n < n_runs; ++n) {
            const uint2 wn = pw[n + 1];  // software pipeline: the next run's word
            const int off = static_cast<int>(w.x & 0x3FFu);
            const int R = static_cast<int>((w.x >> 11) & 0xFFFu);
            const int s = static_cast<int>(w.y & 0xFFFu);
            if (w.y & 0x1000u) {
                // first run of a group: close the previous group and the upper nodes
                // above it, advance level L of the upper prefix
                const int L = static_cast<int>((w.y >> 13) & 15u);
                if constexpr (D > 2) {
                    if (L != kFirstGroup) {
#pragma unroll
                        for (int p = 0; p < P; ++p) {
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
                    }
                }
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    acc2[p] = 0.0;
                    g2p[p] = t2s[((S2 - 2) * P + p) * nt + tid];
                    g2c[p] = t2s[((S2 - 1) * P + p) * nt + tid];
                }
            }
            // sibling weight c_{D-2}[s]
            double ts[P];
            if (s < S2) {
#pragma unroll
                for (int p = 0; p < P; ++p) ts[p] = t2s[(s * P + p) * nt + tid];
            } else {
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    const double c = fma(t2c[p], g2c[p], -g2p[p]);
                    g2p[p] = g2c[p];
                    g2c[p] = c;
                    ts[p] = c;
                }
            }
            // leaf run z = sum_{b<R} alpha'[b] c_b: one brx.idx into a PTX Duff chain
            double z0[P], z1[P];
            leaf_chain<P, LT>(pa_s + 16u * static_cast<unsigned>(off), min((R + 1) >> 1, LT / 2), leaf, z0, z1);
            if (R > LT) {
                // long run: continue the Chebyshev recurrence from (c_{LT-2}, c_{LT-1})
                const double2* ra = pa + off;
                double cp[P], cc[P];
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    cp[p] = leaf[p][LT - 2];
                    cc[p] = leaf[p][LT - 1];
                }
                const int pairs = (R + 1) >> 1;
                for (int b2 = LT / 2; b2 < pairs; ++b2) {
                    const double2 aa = ra[b2];
#pragma unroll
                    for (int p = 0; p < P; ++p) {
                        const double e = fma(tl[p], cc[p], -cp[p]);  // c_{2 b2}
                        const double o = fma(tl[p], e, -cc[p]);      // c_{2 b2 + 1}
                        z0[p] = fma(aa.x, e, z0[p]);
                        z1[p] = fma(aa.y, o, z1[p]);
                        cp[p] = e;
                        cc[p] = o;
                    }
                }
            }
#pragma unroll
            for (int p = 0; p < P; ++p) {
                acc2[p] = fma(ts[p], z0[p], acc2[p]);
                acc2[p] = fma(ts[p], z1[p], acc2[p]);
            }
            w = wn;
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

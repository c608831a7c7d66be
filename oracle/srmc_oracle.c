/* srmc_oracle.c -- TEST INFRASTRUCTURE ONLY: plain-C restatement of the SRMC scheme
 * specified in include/qrmc_srmc.h.
 *
 * PARITY UNPINNED against the reference: /root/reference has no SRMC code (SURVEY.md
 * 8(a), last row; PAPER.md:361-366 only summarises the method). This file is the
 * checker for the GPU path under replayed draws; the scheme itself is pinned only
 * statistically, against closed forms (tests/test_srmc.py). The shared pieces follow
 * the reference: Philox4x32-10 stream and stream ids (proj/src/rng.cpp:9-49,
 * proj/include/qrmc/rng.hpp:26-84, reused from qrmc_oracle.c), the SinBenchmark
 * functors (proj/src/benchmark.cpp:30-67), Euler (proj/src/sde.cpp:37-73) and the
 * soft truncation clamp (proj/src/solver.cpp:37-41).
 *
 * Straightforward order: cells one after another (OpenMP over cells), paths m = 0..M-1
 * in order, sequential sums, Cholesky on the normal equations. Only tests/ may load it.
 */
#include "qrmc_oracle.c" /* Philox stream, normal quantile, error helper (static) */

#include <omp.h>

#include "qrmc_srmc.h"

typedef struct {
    int kind, d, n, P, last;
    int64_t cells, M;
    uint64_t seed;
    double lo, hi, h, inv_h, inv2h, dt, inv_dt, sqrt_dt, t, T, L, bdt, sig, theta, inv_sig;
    double p[8];
} srmc_t;

static double s_terminal(const srmc_t* s, const double* x) {
    double sum = 0.0;
    for (int l = 0; l < s->d; ++l) sum += x[l];
    if (s->kind == QRMC_SRMC_SIN_BENCH) return (1.0 + s->p[0]) + sin(s->p[1] * sum);
    const double v = exp(sum * (1.0 / (double)s->d)) - s->p[4]; /* the reciprocal, as the device */
    return v > 0.0 ? v : 0.0;
}

static double s_driver(const srmc_t* s, const double* x, double y, const double* z) {
    if (s->kind == QRMC_SRMC_SIN_BENCH) {
        double sum = 0.0;
        for (int l = 0; l < s->d; ++l) sum += x[l];
        const double lam = s->p[1];
        const double e = exp(((lam * lam) * (double)s->d) * (s->t - s->T) / 2.0);
        const double w = ((y - s->p[0]) - 1.0) - sin(lam * sum) * e;
        const double ww = w * w;
        return ww < 1.0 ? ww : 1.0;
    }
    const double rl = s->p[2], rb = s->p[3];
    double zs = 0.0;
    for (int l = 0; l < s->d; ++l) zs += z[l];
    const double borrow = zs * s->inv_sig - y;
    return ((-rl) * y - s->theta * zs) + (rb - rl) * (borrow > 0.0 ? borrow : 0.0);
}

static double s_eval(const srmc_t* s, const double* tab, const double* x) {
    int64_t k = 0;
    double sl[QRMC_SRMC_MAX_DIM];
    for (int l = 0; l < s->d; ++l) {
        double xc = x[l] < s->lo ? s->lo : x[l];
        xc = xc > s->hi ? s->hi : xc;
        int c = (int)floor((xc - s->lo) * s->inv_h); /* reciprocal of h, as the device */
        c = c < 0 ? 0 : (c >= s->n ? s->n - 1 : c);
        k = k * s->n + c;
        const double centre = s->lo + ((double)c + 0.5) * s->h;
        sl[l] = (xc - centre) * s->inv2h;
    }
    const double* row = tab + k * s->P;
    double v = row[0];
    if (s->P > 1)
        for (int l = 0; l < s->d; ++l) v += row[1 + l] * sl[l];
    return v;
}

static void s_path(const srmc_t* s, const double* next, const int* cc, int step, int64_t k, int64_t m, double* x0,
                   double* phi, double* dw, double* x1, double* y1) {
    stream_t r;
    stream_init(&r, s->seed, sid_training(step, (uint64_t)k * (uint64_t)s->M + (uint64_t)m));
    phi[0] = 1.0;
    for (int l = 0; l < s->d; ++l) {
        const double u = stream_uniform(&r);
        x0[l] = s->lo + ((double)cc[l] + u) * s->h;
        if (s->P > 1) phi[1 + l] = 2.0 * u - 1.0;
    }
    for (int l = 0; l < s->d; ++l) {
        dw[l] = s->sqrt_dt * qrmc_ppnd16(stream_uniform(&r)); /* PPND16 directly, as the device */
        x1[l] = (x0[l] + s->bdt) + s->sig * dw[l];
    }
    if (s->last) {
        *y1 = s_terminal(s, x1);
    } else {
        double v = s_eval(s, next, x1);
        *y1 = v < -s->L ? -s->L : (v > s->L ? s->L : v);
    }
}

/* Cholesky solve with the same zero-pivot rule as the device (degenerate cell) */
static void s_solve(int P, const double* A /* P*P full */, double* b, int nr) {
    double Lm[QRMC_SRMC_MAX_DIM + 1][QRMC_SRMC_MAX_DIM + 1] = {{0}};
    for (int j = 0; j < P; ++j) {
        double dd = A[j * P + j];
        for (int q = 0; q < j; ++q) dd -= Lm[j][q] * Lm[j][q];
        const double ljj = dd > 1e-300 ? sqrt(dd) : 0.0;
        Lm[j][j] = ljj;
        for (int r = j + 1; r < P; ++r) {
            double v = A[r * P + j];
            for (int q = 0; q < j; ++q) v -= Lm[r][q] * Lm[j][q];
            Lm[r][j] = ljj > 0.0 ? v / ljj : 0.0;
        }
    }
    for (int hh = 0; hh < nr; ++hh) {
        double* y = b + hh * P;
        for (int r = 0; r < P; ++r) {
            double v = y[r];
            for (int q = 0; q < r; ++q) v -= Lm[r][q] * y[q];
            y[r] = Lm[r][r] > 0.0 ? v / Lm[r][r] : 0.0;
        }
        for (int r = P - 1; r >= 0; --r) {
            double v = y[r];
            for (int q = r + 1; q < P; ++q) v -= Lm[q][r] * y[q];
            y[r] = Lm[r][r] > 0.0 ? v / Lm[r][r] : 0.0;
        }
    }
}

static void s_cell(const srmc_t* s, int step, const double* next, int64_t k, int zpass, int anyz, double* yout,
                   double* zout) {
    const int d = s->d, P = s->P;
    int cc[QRMC_SRMC_MAX_DIM];
    int64_t r = k;
    for (int l = d - 1; l >= 0; --l) {
        cc[l] = (int)(r % s->n);
        r /= s->n;
    }
    double A[(QRMC_SRMC_MAX_DIM + 1) * (QRMC_SRMC_MAX_DIM + 1)] = {0};
    double by[QRMC_SRMC_MAX_DIM + 1] = {0};
    double bz[QRMC_SRMC_MAX_DIM * (QRMC_SRMC_MAX_DIM + 1)] = {0};
    double x0[QRMC_SRMC_MAX_DIM], x1[QRMC_SRMC_MAX_DIM], phi[QRMC_SRMC_MAX_DIM + 1], dw[QRMC_SRMC_MAX_DIM], y1;
    const double zero[QRMC_SRMC_MAX_DIM] = {0};
    for (int64_t m = 0; m < s->M; ++m) {
        s_path(s, next, cc, step, k, m, x0, phi, dw, x1, &y1);
        for (int a = 0; a < P; ++a)
            for (int b = 0; b < P; ++b) A[a * P + b] += phi[a] * phi[b];
        if (anyz)
            for (int l = 0; l < d; ++l) {
                const double rz = (y1 * dw[l]) * s->inv_dt;
                for (int p = 0; p < P; ++p) bz[l * P + p] += rz * phi[p];
            }
        if (!zpass) {
            const double ry = y1 + s->dt * s_driver(s, x1, y1, zero);
            for (int p = 0; p < P; ++p) by[p] += ry * phi[p];
        }
    }
    if (anyz) s_solve(P, A, bz, d);
    if (zpass) {
        for (int64_t m = 0; m < s->M; ++m) {
            s_path(s, next, cc, step, k, m, x0, phi, dw, x1, &y1);
            double zi[QRMC_SRMC_MAX_DIM];
            for (int l = 0; l < d; ++l) {
                double v = bz[l * P];
                for (int p = 1; p < P; ++p) v += bz[l * P + p] * phi[p];
                zi[l] = v;
            }
            const double ry = y1 + s->dt * s_driver(s, x1, y1, zi);
            for (int p = 0; p < P; ++p) by[p] += ry * phi[p];
        }
    }
    s_solve(P, A, by, 1);
    for (int p = 0; p < P; ++p) yout[p] = by[p];
    if (anyz && zout)
        for (int j = 0; j < d * P; ++j) zout[j] = bz[j];
}

static void s_init(srmc_t* s, const qrmc_srmc_problem_t* prob, const qrmc_srmc_config_t* cfg) {
    memset(s, 0, sizeof *s);
    s->kind = prob->kind;
    s->d = prob->dim;
    s->n = cfg->cells_per_dim;
    s->P = cfg->basis == QRMC_SRMC_LP1 ? s->d + 1 : 1;
    s->cells = 1;
    for (int l = 0; l < s->d; ++l) s->cells *= s->n;
    s->M = cfg->paths_per_cell;
    s->seed = cfg->seed;
    s->lo = cfg->lo;
    s->hi = cfg->hi;
    s->h = (cfg->hi - cfg->lo) / cfg->cells_per_dim;
    s->inv_h = 1.0 / s->h;
    s->inv2h = 2.0 / s->h;
    s->T = prob->horizon;
    s->dt = prob->horizon / cfg->steps;
    s->inv_dt = 1.0 / s->dt;
    s->sqrt_dt = sqrt(s->dt);
    s->L = cfg->truncation;
    for (int j = 0; j < 8; ++j) s->p[j] = prob->params[j];
    if (s->kind == QRMC_SRMC_BERGMAN) {
        s->theta = (prob->params[0] - prob->params[2]) / prob->params[1];
        s->inv_sig = 1.0 / prob->params[1];
        const double drift = prob->params[0] - 0.5 * (prob->params[1] * prob->params[1]);
        s->bdt = drift * s->dt;
        s->sig = prob->params[1];
    } else {
        s->bdt = 0.0;
        s->sig = 1.0;
    }
}

/* one backward step over the cells [k_begin, k_end) (a rank's shard in the sharded tests);
 * y_step / z_step are the full step tables, next = step+1's y table */
int32_t srmc_oracle_step(const qrmc_srmc_problem_t* prob, const qrmc_srmc_config_t* cfg, int32_t step,
                         const double* next, double* y_step, double* z_step, int64_t k_begin, int64_t k_end,
                         int32_t threads) {
    srmc_t s;
    s_init(&s, prob, cfg);
    s.last = (step == cfg->steps - 1);
    s.t = (step + 1) * s.dt; /* f at (t_{i+1}, X_{i+1}, Y1, Zhat_i(X_i)) */
    const int zpass = prob->kind == QRMC_SRMC_BERGMAN;
    const int anyz = zpass || cfg->want_z || z_step != NULL;
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t k = k_begin; k < k_end; ++k)
        s_cell(&s, step, s.last ? NULL : next, k, zpass, anyz, y_step + k * s.P,
               z_step ? z_step + k * s.d * s.P : NULL);
    return 0;
}

int32_t srmc_oracle_solve(const qrmc_srmc_problem_t* prob, const qrmc_srmc_config_t* cfg, double* y, double* z,
                          int32_t threads) {
    srmc_t s;
    s_init(&s, prob, cfg);
    const size_t per_y = (size_t)s.cells * s.P, per_z = per_y * s.d;
    for (int i = cfg->steps - 1; i >= 0; --i)
        srmc_oracle_step(prob, cfg, i, i == cfg->steps - 1 ? NULL : y + per_y * (i + 1), y + per_y * i,
                         z ? z + per_z * i : NULL, 0, s.cells, threads);
    return 0;
}

double srmc_oracle_eval(const qrmc_srmc_problem_t* prob, const qrmc_srmc_config_t* cfg, const double* y_step,
                        const double* x) {
    srmc_t s;
    memset(&s, 0, sizeof s);
    s.d = prob->dim;
    s.n = cfg->cells_per_dim;
    s.P = cfg->basis == QRMC_SRMC_LP1 ? s.d + 1 : 1;
    s.lo = cfg->lo;
    s.hi = cfg->hi;
    s.h = (cfg->hi - cfg->lo) / cfg->cells_per_dim;
    s.inv_h = 1.0 / s.h;
    s.inv2h = 2.0 / s.h;
    return s_eval(&s, y_step, x);
}

/* PPND16 of n uniforms two ways, for the header check (tests/test_srmc.py): whole, and
 * through the split branches the device batches across a warp (srmc.cu srmc_quantiles). */
void srmc_oracle_ppnd16_both(const double* u, int64_t n, double* whole, double* split) {
    for (int64_t i = 0; i < n; ++i) {
        const double q = u[i] - 0.5;
        whole[i] = qrmc_ppnd16(u[i]);
        if ((q < 0 ? -q : q) <= 0.425) {
            split[i] = qrmc_ppnd16_central(q);
        } else {
            const double v = qrmc_ppnd16_tail(q < 0 ? u[i] : 1.0 - u[i]);
            split[i] = q < 0 ? -v : v;
        }
    }
}

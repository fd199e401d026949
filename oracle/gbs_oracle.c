/*
 * gbs_oracle.c -- TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct
 * fp64 CPU implementation of the extrapolated GBS time stepper on the
 * method-of-lines FD right-hand sides of the five BASELINE.json configs.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * table or helper with the CUDA path (paper_1907_11771_b200/csrc); the two
 * meet only at the seeded input bytes (gbs_inputs/) and the fp64 weights.
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC (no intrinsics).
 * OpenMP is used only over the outermost grid loop of pointwise passes, so
 * the result is bit-identical for every thread count (no reductions inside
 * the stepping).
 *
 * What it follows, step by step, in the paper's order (§2.1,
 * Eq. (1) "eq:GBS", lines 85-98, and the combination at lines 109-115,
 * 221-225):
 *
 *   for each macro step (section) of length H, starting from Y:
 *     for each sequence k in the order given (ascending n_k):
 *       h = H / n_k
 *       y_0 = Y
 *       y_1 = y_0 + h f(y_0)                        Eq. (1) row 1 (FE)
 *       y_{n+1} = y_{n-1} + 2h f(y_n), n = 1..N     Eq. (1) row 2 (LF), N = n_k
 *       y*_k = 1/4 (y_{N-1} + 2 y_N + y_{N+1})      Eq. (1) row 3 (averaging)
 *     Y <- sum_k w_k y*_k, summed from 0.0 in the order given
 *
 *
 * f(y) is the MOL right-hand side (BASELINE.json configs; PAPER.md:565 uses
 * a spectral derivative instead):
 *   ADV1D      u_t = -u_x
 *   ACOUSTIC2D p_t = -(u_x + v_y), u_t = -p_x, v_t = -p_y
 *   WAVE3D     u_t = v, v_t = u_xx + u_yy + u_zz
 * ADV1D with order 0 is the paper's own spectral derivative (PAPER.md:565,
 * §4.1): the derivative of the trigonometric interpolant, by its definition
 * -- a forward DFT, multiplication by 2 pi i k for |k| < N/2 (the Nyquist
 * mode of an even-N grid has no odd derivative and is dropped), an inverse
 * DFT -- as plain O(N^2) loops over a cos/sin table of 2 pi m / N.
 * Otherwise the derivatives are
 * centered periodic FD derivatives in the antisymmetric pairing form
 * (SURVEY.md §8(c) item 3), grid spacing 1/N_d on the unit box (S6):
 *   D1 u_i = N_d * sum_{j=1..r} a_j (u_{i+j} - u_{i-j})
 *   D2 u_i = N_d^2 * (b_0 u_i + sum_{j=1..r} b_j (u_{i+j} + u_{i-j}))
 * The standard centered Taylor coefficients are typed in below as exact
 * rationals; tests/test_oracle_fd.py pins them to the Taylor (Vandermonde)
 * conditions solved exactly and to the stencils' order of accuracy.
 *
 * "dims" are the array extents; "scale" are the N_d of the spacing 1/N_d.
 * They coincide on a full periodic grid; they differ only when the tests
 * evaluate a sampled output on a periodically-extracted sub-box (the value
 * at the box centre is then the same arithmetic on the same inputs).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

#define ORACLE_ADV1D 1
#define ORACLE_ACOUSTIC2D 2
#define ORACLE_WAVE3D 3

/* ---- centered FD coefficients (standard Taylor weights) ---------------- */
/* first derivative, D1 u_i = N sum_j a_j (u_{i+j} - u_{i-j}) */
static const double A4[2] = {2.0 / 3.0, -1.0 / 12.0};
static const double A8[4] = {4.0 / 5.0, -1.0 / 5.0, 4.0 / 105.0, -1.0 / 280.0};
/* second derivative, D2 u_i = N^2 (b0 u_i + sum_j b_j (u_{i+j} + u_{i-j})) */
static const double B4_0 = -5.0 / 2.0;
static const double B4[2] = {4.0 / 3.0, -1.0 / 12.0};
static const double B8_0 = -205.0 / 72.0;
static const double B8[4] = {8.0 / 5.0, -1.0 / 5.0, 8.0 / 315.0, -1.0 / 560.0};

static int g_threads = 1;

int oracle_set_threads(int n) {
    g_threads = n < 1 ? 1 : n;
#ifdef _OPENMP
    return g_threads;
#else
    return 1;
#endif
}

/* Exported for the coefficient pin (tests/test_oracle_fd.py). */
int oracle_fd_coeffs(int order, double* a, double* b0, double* b) {
    int r, j;
    const double *pa, *pb;
    double pb0;
    if (order == 4) { r = 2; pa = A4; pb = B4; pb0 = B4_0; }
    else if (order == 8) { r = 4; pa = A8; pb = B8; pb0 = B8_0; }
    else return -1;
    for (j = 0; j < r; ++j) { a[j] = pa[j]; b[j] = pb[j]; }
    *b0 = pb0;
    return r;
}

static int wrap(int64_t i, int64_t n) {
    /* periodic index, valid for |i| < 2n */
    if (i < 0) return (int)(i + n);
    if (i >= n) return (int)(i - n);
    return (int)i;
}

typedef struct {
    int pde, order, r, F;
    int64_t nx, ny, nz, npts;
    double sx, sy, sz;          /* N_d of the spacing 1/N_d */
    const double* a;            /* D1 coefficients */
    const double* b;            /* D2 coefficients */
    double b0;
    double *ct, *st;            /* spectral (order 0): cos, sin of 2 pi m / nx */
    double *re, *im;            /* spectral scratch: DFT of the field */
} grid_t;

static void release(grid_t* g) {
    free(g->ct); free(g->st); free(g->re); free(g->im);
    g->ct = g->st = g->re = g->im = NULL;
}

static int setup(grid_t* g, int pde, int order, const int64_t* dims, const double* scale) {
    memset(g, 0, sizeof(*g));
    g->pde = pde;
    g->order = order;
    if (order == 4) { g->r = 2; g->a = A4; g->b = B4; g->b0 = B4_0; }
    else if (order == 8) { g->r = 4; g->a = A8; g->b = B8; g->b0 = B8_0; }
    else if (order == 0 && pde == ORACLE_ADV1D && dims[0] >= 2 && dims[0] % 2 == 0) {
        int64_t m, n = dims[0];
        g->r = 0;
        g->ct = (double*)malloc(sizeof(double) * (size_t)n);
        g->st = (double*)malloc(sizeof(double) * (size_t)n);
        g->re = (double*)malloc(sizeof(double) * (size_t)n);
        g->im = (double*)malloc(sizeof(double) * (size_t)n);
        if (!g->ct || !g->st || !g->re || !g->im) { release(g); return -7; }
        for (m = 0; m < n; ++m) {
            g->ct[m] = cos(2.0 * M_PI * (double)m / (double)n);
            g->st[m] = sin(2.0 * M_PI * (double)m / (double)n);
        }
    }
    else return -1;
    g->nx = dims[0]; g->ny = dims[1]; g->nz = dims[2];
    g->sx = scale[0]; g->sy = scale[1]; g->sz = scale[2];
    if (pde == ORACLE_ADV1D) g->F = 1;
    else if (pde == ORACLE_ACOUSTIC2D) g->F = 3;
    else if (pde == ORACLE_WAVE3D) g->F = 2;
    else return -2;
    if (g->nx < 1 || g->ny < 1 || g->nz < 1) return -3;
    if (g->nx < g->r + 1) return -3;
    if (pde != ORACLE_ADV1D && g->ny < g->r + 1) return -3;
    if (pde == ORACLE_WAVE3D && g->nz < g->r + 1) return -3;
    g->npts = g->nx * g->ny * g->nz;
    return 0;
}

/* D1 along x of field u at (x, y, z) */
static double d1x(const grid_t* g, const double* u, int64_t x, int64_t y, int64_t z) {
    double s = 0.0;
    int j;
    const double* row = u + (z * g->ny + y) * g->nx;
    for (j = 1; j <= g->r; ++j)
        s += g->a[j - 1] * (row[wrap(x + j, g->nx)] - row[wrap(x - j, g->nx)]);
    return g->sx * s;
}

static double d1y(const grid_t* g, const double* u, int64_t x, int64_t y, int64_t z) {
    double s = 0.0;
    int j;
    const double* pl = u + z * g->ny * g->nx;
    for (j = 1; j <= g->r; ++j)
        s += g->a[j - 1] * (pl[wrap(y + j, g->ny) * g->nx + x] - pl[wrap(y - j, g->ny) * g->nx + x]);
    return g->sy * s;
}

static double d2x(const grid_t* g, const double* u, int64_t x, int64_t y, int64_t z) {
    const double* row = u + (z * g->ny + y) * g->nx;
    double s = g->b0 * row[x];
    int j;
    for (j = 1; j <= g->r; ++j)
        s += g->b[j - 1] * (row[wrap(x + j, g->nx)] + row[wrap(x - j, g->nx)]);
    return g->sx * g->sx * s;
}

static double d2y(const grid_t* g, const double* u, int64_t x, int64_t y, int64_t z) {
    const double* pl = u + z * g->ny * g->nx;
    double s = g->b0 * pl[y * g->nx + x];
    int j;
    for (j = 1; j <= g->r; ++j)
        s += g->b[j - 1] * (pl[wrap(y + j, g->ny) * g->nx + x] + pl[wrap(y - j, g->ny) * g->nx + x]);
    return g->sy * g->sy * s;
}

static double d2z(const grid_t* g, const double* u, int64_t x, int64_t y, int64_t z) {
    int64_t pl = g->ny * g->nx, off = y * g->nx + x;
    double s = g->b0 * u[z * pl + off];
    int j;
    for (j = 1; j <= g->r; ++j)
        s += g->b[j - 1] * (u[wrap(z + j, g->nz) * pl + off] + u[wrap(z - j, g->nz) * pl + off]);
    return g->sz * g->sz * s;
}

/* spectral u_x on the unit periodic interval (order 0): u_hat_k = sum_j u_j
 * e^{-2 pi i j k / N}; u_x(j) = (1/N) sum_{|k| < N/2} 2 pi i k u_hat_k e^{2 pi i j k / N}
 * (k and N - k taken together: the result is real) */
static void spectral_d1(const grid_t* g, const double* u, double* du) {
    const int64_t n = g->nx;
    int64_t k, j;
#pragma omp parallel for num_threads(g_threads) schedule(static)
    for (k = 0; k < n; ++k) {
        double re = 0.0, im = 0.0;
        int64_t jj;
        for (jj = 0; jj < n; ++jj) {
            int64_t m = (jj * k) % n;
            re += u[jj] * g->ct[m];
            im -= u[jj] * g->st[m];
        }
        g->re[k] = re;
        g->im[k] = im;
    }
#pragma omp parallel for num_threads(g_threads) schedule(static)
    for (j = 0; j < n; ++j) {
        double s = 0.0;
        int64_t kk;
        for (kk = 1; kk < n / 2; ++kk) {
            /* mode kk and its conjugate -kk: 2 Re(2 pi i kk u_hat_kk e^{2 pi i j kk / N}) */
            int64_t m = (j * kk) % n;
            double wre = -2.0 * M_PI * (double)kk * g->im[kk];   /* Re(2 pi i kk u_hat) */
            double wim = 2.0 * M_PI * (double)kk * g->re[kk];    /* Im(2 pi i kk u_hat) */
            s += 2.0 * (wre * g->ct[m] - wim * g->st[m]);
        }
        du[j] = s / (double)n;
    }
}

/* f = rhs(y): the MOL right-hand side, SoA [F][nz][ny][nx] */
static void rhs(const grid_t* g, const double* y, double* f) {
    int64_t n = g->npts;
    int64_t z;
    if (g->pde == ORACLE_ADV1D && g->order == 0) {
        int64_t x;
        spectral_d1(g, y, f);
        for (x = 0; x < g->nx; ++x) f[x] = -f[x];
    } else if (g->pde == ORACLE_ADV1D) {
        const double* u = y;
        int64_t x;
#pragma omp parallel for num_threads(g_threads) schedule(static)
        for (x = 0; x < g->nx; ++x) f[x] = -d1x(g, u, x, 0, 0);
    } else if (g->pde == ORACLE_ACOUSTIC2D) {
        const double *p = y, *u = y + n, *v = y + 2 * n;
        int64_t yy;
#pragma omp parallel for num_threads(g_threads) schedule(static)
        for (yy = 0; yy < g->ny; ++yy) {
            int64_t x;
            for (x = 0; x < g->nx; ++x) {
                int64_t i = yy * g->nx + x;
                f[i] = -(d1x(g, u, x, yy, 0) + d1y(g, v, x, yy, 0));
                f[n + i] = -d1x(g, p, x, yy, 0);
                f[2 * n + i] = -d1y(g, p, x, yy, 0);
            }
        }
    } else { /* WAVE3D */
        const double *u = y, *v = y + n;
#pragma omp parallel for num_threads(g_threads) schedule(static)
        for (z = 0; z < g->nz; ++z) {
            int64_t yy, x;
            for (yy = 0; yy < g->ny; ++yy)
                for (x = 0; x < g->nx; ++x) {
                    int64_t i = (z * g->ny + yy) * g->nx + x;
                    f[i] = v[i];
                    f[n + i] = d2x(g, u, x, yy, z) + d2y(g, u, x, yy, z) + d2z(g, u, x, yy, z);
                }
        }
    }
}

/* out = a + c * f   (pointwise) */
static void axpy(int64_t len, double* out, const double* a, double c, const double* f) {
    int64_t i;
#pragma omp parallel for num_threads(g_threads) schedule(static)
    for (i = 0; i < len; ++i) out[i] = a[i] + c * f[i];
}

int oracle_rhs(int pde, int order, const int64_t* dims, const double* scale,
               const double* y, double* f) {
    grid_t g;
    int rc = setup(&g, pde, order, dims, scale);
    if (rc) return rc;
    rhs(&g, y, f);
    release(&g);
    return 0;
}

/*
 * Advance Y (in place, SoA [F][nz][ny][nx]) by M macro steps of length H.
 * Sequences are taken in the order given by n_k[0..m-1] (callers pass them
 * ascending).  Returns 0, or a negative code on invalid input / no memory.
 */
int oracle_advance(int pde, int order, const int64_t* dims, const double* scale,
                   int m, const int32_t* n_k, const double* w_k, double H,
                   int64_t M, double* Y) {
    grid_t g;
    int rc = setup(&g, pde, order, dims, scale);
    int64_t len, step, i;
    int k;
    double *bufs[4], *f, *acc;
    if (rc) return rc;
    if (m < 1) { release(&g); return -4; }
    for (k = 0; k < m; ++k)
        if (n_k[k] < 2 || (n_k[k] % 2) != 0) { release(&g); return -5; }
    if (!(H > 0.0)) { release(&g); return -6; }
    len = g.F * g.npts;
    for (k = 0; k < 4; ++k) bufs[k] = (double*)malloc(sizeof(double) * (size_t)len);
    f = (double*)malloc(sizeof(double) * (size_t)len);
    acc = (double*)malloc(sizeof(double) * (size_t)len);
    if (!bufs[0] || !bufs[1] || !bufs[2] || !bufs[3] || !f || !acc) {
        for (k = 0; k < 4; ++k) free(bufs[k]);
        free(f);
        free(acc);
        release(&g);
        return -7;
    }

    for (step = 0; step < M; ++step) {
        for (i = 0; i < len; ++i) acc[i] = 0.0;
        for (k = 0; k < m; ++k) {
            int N = n_k[k], n;
            double h = H / (double)N;
            /* three rotating levels: ym1 = y_{n-1}, y0 = y_n, yp1 = y_{n+1} */
            double *ym1 = bufs[0], *y0 = bufs[1], *yp1 = bufs[2], *t;
            /* y_0 = Y, y_1 = y_0 + h f(y_0)   (FE) */
            memcpy(ym1, Y, sizeof(double) * (size_t)len);
            rhs(&g, ym1, f);
            axpy(len, y0, ym1, h, f);
            /* LF: y_{n+1} = y_{n-1} + 2h f(y_n), n = 1..N */
            for (n = 1; n <= N; ++n) {
                rhs(&g, y0, f);
                axpy(len, yp1, ym1, 2.0 * h, f);
                if (n < N) { t = ym1; ym1 = y0; y0 = yp1; yp1 = t; }
            }
            /* y* = 1/4 (y_{N-1} + 2 y_N + y_{N+1}); acc += w_k y* */
            {
                double wk = w_k[k];
#pragma omp parallel for num_threads(g_threads) schedule(static)
                for (i = 0; i < len; ++i) {
                    double ystar = 0.25 * ((ym1[i] + 2.0 * y0[i]) + yp1[i]);
                    acc[i] = acc[i] + wk * ystar;
                }
            }
        }
        memcpy(Y, acc, sizeof(double) * (size_t)len);
    }
    for (k = 0; k < 4; ++k) free(bufs[k]);
    free(f);
    free(acc);
    release(&g);
    return 0;
}

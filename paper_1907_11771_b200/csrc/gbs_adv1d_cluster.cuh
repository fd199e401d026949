// gbs_adv1d_cluster.cuh -- the whole run of a small 1-D advection problem in one
// launch: one CTA per GBS sequence, the m CTAs of a
// thread-block cluster run their sequences concurrently (the paper's "separate
// cores") on state held in shared memory, and combine
// through distributed shared memory after every macro step.
//
// Per macro step, CTA k (sequence n_k, h = H/n_k), same arithmetic as the
// per-substep kernels (gbs_kernels.cuh), so results are bit-identical to them:
//   a  = Y + h f(Y)                        FE
//   b  = Y + 2h f(a), then LF in place      LF_1 .. LF_{n-1}
//   t_k = prev + cur + h f(cur)             final step (unweighted)
//   cluster barrier; every CTA forms Y = wh_0 t_0, then Y = fma(wh_k, t_k, Y) for
//   k = 1..m-1 in ascending n_k, reading t_k from CTA k's shared memory (DSMEM);
//   cluster barrier (t_k may be overwritten).
// f(u) = -s sum_j a_j (u_{i+j} - u_{i-j}) with periodic wrap.
#pragma once

#include <cooperative_groups.h>

#include "gbs_kernels.cuh"

namespace gbs {

struct Adv1DClusterArgs {
    double* Y;                // in/out, nx values (global)
    int nx;
    double sx;
    double H;
    long long macro_steps;
    const int* nk;            // m step counts (ascending), device
    const double* wh;         // m half-weights w_k / 2, device
    int* nonfinite;
};

template <int R>
__global__ void __launch_bounds__(256)
adv1d_cluster_run(const Adv1DClusterArgs A) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int k = (int)cluster.block_rank();
    const int m = (int)cluster.num_blocks();
    const int nx = A.nx, tid = threadIdx.x, nt = blockDim.x;
    extern __shared__ double sm[];
    double* Ys = sm;              // combined state
    double* a = sm + nx;          // level buffers
    double* b = sm + 2 * nx;
    double* t = sm + 3 * nx;      // unweighted final-step contribution of this sequence
    const int n = A.nk[k];
    const double h = A.H / (double)n;

    auto rhs = [&](const double* u, int x) {
        double d = 0.0;
#pragma unroll
        for (int j = 1; j <= R; ++j) d = fma(FD<R>::a(j), u[wrap_once(x + j, nx)] - u[wrap_once(x - j, nx)], d);
        return -A.sx * d;
    };

    for (int x = tid; x < nx; x += nt) Ys[x] = A.Y[x];
    __syncthreads();
    for (long long step = 0; step < A.macro_steps; ++step) {
        for (int x = tid; x < nx; x += nt) a[x] = combine<MODE_FE>(0.0, Ys[x], rhs(Ys, x), 0.0, h, 0.0);
        __syncthreads();
        for (int x = tid; x < nx; x += nt) b[x] = combine<MODE_LF>(Ys[x], a[x], rhs(a, x), 0.0, 2.0 * h, 0.0);
        __syncthreads();
        double *prev = a, *cur = b;
        for (int i = 2; i <= n - 1; ++i) {
            for (int x = tid; x < nx; x += nt) prev[x] = combine<MODE_LF>(prev[x], cur[x], rhs(cur, x), 0.0, 2.0 * h, 0.0);
            __syncthreads();
            double* s = prev; prev = cur; cur = s;
        }
        for (int x = tid; x < nx; x += nt) t[x] = prev[x] + cur[x] + h * rhs(cur, x);
        cluster.sync();
        for (int x = tid; x < nx; x += nt) {
            const double* t0 = cluster.map_shared_rank(t, 0);
            double y = A.wh[0] * t0[x];
            for (int r = 1; r < m; ++r) y = fma(A.wh[r], cluster.map_shared_rank(t, r)[x], y);
            Ys[x] = y;
        }
        cluster.sync();
    }
    if (k == 0) {
        bool bad = false;
        for (int x = tid; x < nx; x += nt) {
            A.Y[x] = Ys[x];
            bad |= !isfinite(Ys[x]);
        }
        if (bad && A.nonfinite) *A.nonfinite = 1;
    }
}

// The paper's own spatial discretisation (§4.1): the spectral
// (Fourier collocation) derivative on an even periodic grid.  The derivative of
// the trigonometric interpolant is the circulant pairing sum
//   u_x(x_i) = s sum_{j=1}^{N/2-1} alpha_j (u_{i+j} - u_{i-j}),
//   alpha_j = pi (-1)^{j+1} cot(j pi / N) / N,  s = N / length
// (the Nyquist term vanishes: cot(pi/2) = 0), i.e. the FD pairing form of radius
// N/2 - 1 with these weights, read from shared memory (host-computed in fp64).
// Same per-macro-step structure and combine as adv1d_cluster_run.
__global__ void __launch_bounds__(256)
adv1d_cluster_run_spectral(const Adv1DClusterArgs A, const double* __restrict__ alpha) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int k = (int)cluster.block_rank();
    const int m = (int)cluster.num_blocks();
    const int nx = A.nx, tid = threadIdx.x, nt = blockDim.x;
    const int R = nx / 2 - 1;
    extern __shared__ double sm[];
    double* Ys = sm;
    double* a = sm + nx;
    double* b = sm + 2 * nx;
    double* t = sm + 3 * nx;
    double* al = sm + 4 * nx;     // alpha_1 .. alpha_R
    const int n = A.nk[k];
    const double h = A.H / (double)n;

    auto rhs = [&](const double* u, int x) {
        double d = 0.0;
        for (int j = 1; j <= R; ++j) d = fma(al[j - 1], u[wrap_once(x + j, nx)] - u[wrap_once(x - j, nx)], d);
        return -A.sx * d;
    };

    for (int x = tid; x < nx; x += nt) Ys[x] = A.Y[x];
    for (int j = tid; j < R; j += nt) al[j] = alpha[j];
    __syncthreads();
    for (long long step = 0; step < A.macro_steps; ++step) {
        for (int x = tid; x < nx; x += nt) a[x] = combine<MODE_FE>(0.0, Ys[x], rhs(Ys, x), 0.0, h, 0.0);
        __syncthreads();
        for (int x = tid; x < nx; x += nt) b[x] = combine<MODE_LF>(Ys[x], a[x], rhs(a, x), 0.0, 2.0 * h, 0.0);
        __syncthreads();
        double *prev = a, *cur = b;
        for (int i = 2; i <= n - 1; ++i) {
            for (int x = tid; x < nx; x += nt) prev[x] = combine<MODE_LF>(prev[x], cur[x], rhs(cur, x), 0.0, 2.0 * h, 0.0);
            __syncthreads();
            double* s = prev; prev = cur; cur = s;
        }
        for (int x = tid; x < nx; x += nt) t[x] = prev[x] + cur[x] + h * rhs(cur, x);
        cluster.sync();
        for (int x = tid; x < nx; x += nt) {
            const double* t0 = cluster.map_shared_rank(t, 0);
            double y = A.wh[0] * t0[x];
            for (int r = 1; r < m; ++r) y = fma(A.wh[r], cluster.map_shared_rank(t, r)[x], y);
            Ys[x] = y;
        }
        cluster.sync();
    }
    if (k == 0) {
        bool bad = false;
        for (int x = tid; x < nx; x += nt) {
            A.Y[x] = Ys[x];
            bad |= !isfinite(Ys[x]);
        }
        if (bad && A.nonfinite) *A.nonfinite = 1;
    }
}

}  // namespace gbs

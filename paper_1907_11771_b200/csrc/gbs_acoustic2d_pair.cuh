// gbs_acoustic2d_pair.cuh -- two consecutive leap-frog substeps of 2-D linear
// acoustics in one HBM pass (temporal blocking), TMA-fed.
//
//   p_t = -(u_x + v_y),  u_t = -p_x,  v_t = -p_y          (BASELINE.json configs 2-3)
//
// Two leap-frog steps (Eq. (1) row 2) from P = y_{n-1}, S = y_n:
//   A = P + cfA f(S)  (= y_{n+1}),   B = S + cfB f(A)  (= y_{n+2})
// split into two independent chains -- p feeds only (u, v) and (u, v) feed only p:
//   chain U:  A_p = P_p - cfA (D_x S_u + D_y S_v);   B_u = S_u - cfB D_x A_p,  B_v = S_v - cfB D_y A_p
//   chain P:  A_u = P_u - cfA D_x S_p,  A_v = P_v - cfA D_y S_p;   B_p = S_p - cfB (D_x A_u + D_y A_v)
// Each chain is one kernel that reads three fields (24 B/pt) and writes three
// (24 B/pt): the pair moves 96 B/pt for two substeps instead of 144.  The
// intermediate level is formed in shared memory on the band extended by the
// stencil radius r (A_p on rows [-r, 16+r) x cols [-r, 64+r); A_u on the band rows
// x cols [-r, 64+r); A_v on rows [-r, 16+r) x the band columns), with exactly the
// operations and summation order of the single-step kernels, so the result is
// bit-identical to two single-step launches (tested).
//
// Layout: slab mode only (ghost rows of r on each side of the y axis, refreshed
// before every launch; one slab = a self-exchange), so every box lies inside the
// tensor; x halos are separate column blocks at wrapped coordinates.  A CTA
// covers 64 columns and marches y in AC2_BH = 32-row bands (the intermediate level's
// halo overhead is (32 + 2r) / 32 instead of (16 + 2r) / 16); 16 consumer warps work on
// 2 x 2 point blocks (rows r, r+1 and columns c, c+1: 128-bit shared loads, y windows
// shared by the two rows) in two phases per band -- the intermediate level on the
// extended band, then the band's output (one block per thread) -- with the items of a
// phase spread over all consumer threads; 1 producer warp issues one TMA box per column
// block per field, D = 2 stages (shared memory).
#pragma once

#include "gbs_wave3d_tma.cuh"

namespace gbs {
namespace tma {

__host__ __device__ constexpr int pad16(int x) { return (x + 15) / 16 * 16; }   // 128-byte blocks

constexpr int AC2_BH = 32;                        // rows per band
constexpr int AC2_NW = 16;                        // consumer warps (+ 1 producer warp)

template <int R>
struct Ac2Geom {
    static constexpr int BH = AC2_BH;
    static constexpr int NRU = BH + 2 * R;        // rows [-r, BH + r)
    static constexpr int NRV = BH + 4 * R;        // rows [-2r, BH + 2r)
    static constexpr int WA = TX + 2 * R;         // cols [-r, 64 + r)
};

// chain U stage: S_u (rows [-r,BH+r); blocks at cols -2r, -r, 0, 64, 64+r), S_v (rows
// [-2r,BH+2r); cols -r, 0, 64), P_p (rows [-r,BH+r); cols -r, 0, 64)
template <int R>
struct ChainULayout {
    using G = Ac2Geom<R>;
    static constexpr int BU = pad16(G::NRU * R), CU = G::NRU * TX;     // strip / centre blocks
    static constexpr int BV = pad16(G::NRV * R), CV = G::NRV * TX;
    static constexpr int SU = 0;                                       // L2 | L1 | C | R1 | R2
    static constexpr int SV = SU + 4 * BU + CU;                        // L1 | C | R1
    static constexpr int PP = SV + 2 * BV + CV;                        // L1 | C | R1
    static constexpr int STAGE = PP + 2 * BU + CU;
    static constexpr int D = 2;
    static constexpr int SCR = G::NRU * G::WA;                         // A_p scratch
    static constexpr size_t bytes = ((size_t)D * STAGE + SCR) * 8 + 2 * D * 8;
    static constexpr uint32_t stage_bytes =
        (uint32_t)(4 * G::NRU * R + G::NRU * TX + 2 * G::NRV * R + G::NRV * TX + 2 * G::NRU * R + G::NRU * TX) * 8;
};

// chain P stage: S_p (centre rows [-2r,BH+2r); strips at cols -2r, -r, 64, 64+r on the band
// rows), P_u (band rows; cols -r, 0, 64), P_v (rows [-r,BH+r); band columns)
template <int R>
struct ChainPLayout {
    using G = Ac2Geom<R>;
    static constexpr int BS = pad16(G::BH * R);
    static constexpr int SPC = 0, SPS = G::NRV * TX;                   // centre | L2 L1 R1 R2
    static constexpr int PU = SPS + 4 * BS;                            // L1 | C | R1
    static constexpr int PV = PU + 2 * BS + G::BH * TX;
    static constexpr int STAGE = PV + G::NRU * TX;
    static constexpr int D = 2;
    static constexpr int SCR_U = G::BH * G::WA, SCR_V = G::NRU * TX;   // A_u, A_v scratch
    static constexpr size_t bytes = ((size_t)D * STAGE + SCR_U + SCR_V) * 8 + 2 * D * 8;
    static constexpr uint32_t stage_bytes =
        (uint32_t)(G::NRV * TX + 4 * G::BH * R + 2 * G::BH * R + G::BH * TX + G::NRU * TX) * 8;
};

struct Ac2PairMaps {
    // per field (p, u, v) of the current level S and the previous level P:
    //   [0] 64 x BH, [1] r x BH, [2] 64 x (BH+2r), [3] r x (BH+2r), [4] 64 x (BH+4r), [5] r x (BH+4r)
    CUtensorMap s[3][6];
    CUtensorMap p[3][6];
};

struct Ac2PairArgs {
    double* A[3];            // y_{n+1} (p, u, v)
    double* B[3];            // y_{n+2}
    int nx, ny;              // ny = local slab rows
    int ylo, yhi, ychunk;    // rows [ylo, yhi) of the slab, ychunk rows per CTA (multiples of BH)
    int yskip;               // rows skipped after the first chunk (both face bands in one launch)
    double sx, sy, cfA, cfB;
};

// value pairs of a block-decomposed region: column c (even) of local row rr
template <int R, int NB>
struct Cols {
    int col0[NB], width[NB], base[NB];
    __device__ __forceinline__ const double* at(const double* st, int rr, int c) const {
        // constant indices only (no dynamically indexed local array)
        const double* ptr = st + base[0] + rr * width[0] + (c - col0[0]);
#pragma unroll
        for (int k = 1; k < NB; ++k)
            if (c >= col0[k]) ptr = st + base[k] + rr * width[k] + (c - col0[k]);
        return ptr;
    }
};

// barrier of the consumer warps only (the producer warp has returned)
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;" ::"n"(32 * AC2_NW) : "memory"); }

__device__ __forceinline__ void ldpair(const double* p, double& a, double& b) {
    const double2 t = *reinterpret_cast<const double2*>(p);
    a = t.x; b = t.y;
}

// ---------------------------------------------------------------------------------------
template <int R>
__global__ void __launch_bounds__(32 * (AC2_NW + 1), 1)
acoustic2d_chainU_tma(const __grid_constant__ Ac2PairMaps M, const Ac2PairArgs A, const int ybase) {
    using L = ChainULayout<R>;
    using G = Ac2Geom<R>;
    constexpr int D = L::D, NW = AC2_NW, BH = G::BH;
    extern __shared__ __align__(128) double smem[];
    double* scr = smem + (size_t)D * L::STAGE;
    uint64_t* full = reinterpret_cast<uint64_t*>(scr + L::SCR);
    uint64_t* empty = full + D;
    const int tid = threadIdx.x + 32 * threadIdx.y, warp = threadIdx.y, lane = threadIdx.x;
    const int nx = A.nx;
    const int x0 = blockIdx.x * TX;
    const int ys = A.ylo + blockIdx.y * A.ychunk + (blockIdx.y ? A.yskip : 0);
    const int niter = min(A.ychunk, A.yhi - ys) / BH;
    const Cols<R, 5> su{{-2 * R, -R, 0, TX, TX + R}, {R, R, TX, R, R},
                        {L::SU, L::SU + L::BU, L::SU + 2 * L::BU, L::SU + 2 * L::BU + L::CU, L::SU + 3 * L::BU + L::CU}};
    const Cols<R, 3> sv{{-R, 0, TX}, {R, TX, R}, {L::SV, L::SV + L::BV, L::SV + L::BV + L::CV}};
    const Cols<R, 3> pp{{-R, 0, TX}, {R, TX, R}, {L::PP, L::PP + L::BU, L::PP + L::BU + L::CU}};

    if (tid == 0) {
        for (int s = 0; s < D; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NW); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == NW) {
        // ============================ producer ============================
        if (lane != 0) return;
        const int xl2 = wrap_any(x0 - 2 * R, nx), xl1 = wrap_any(x0 - R, nx);
        const int xr1 = wrap_any(x0 + TX, nx), xr2 = wrap_any(x0 + TX + R, nx);
        for (int i = 0; i < niter; ++i) {
            const int s = i % D;
            if (i >= D) mbar_wait(&empty[s], (uint32_t)(((i / D) - 1) & 1));
            mbar_expect_tx(&full[s], L::stage_bytes);
            double* st = smem + (size_t)s * L::STAGE;
            const int y = ys + i * BH + ybase;             // tensor row of the band's first row
            const int yu = y - R, yv = y - 2 * R;
            tma_load_3d(st + su.base[0], &M.s[1][3], xl2, yu, 0, &full[s]);
            tma_load_3d(st + su.base[1], &M.s[1][3], xl1, yu, 0, &full[s]);
            tma_load_3d(st + su.base[2], &M.s[1][2], x0, yu, 0, &full[s]);
            tma_load_3d(st + su.base[3], &M.s[1][3], xr1, yu, 0, &full[s]);
            tma_load_3d(st + su.base[4], &M.s[1][3], xr2, yu, 0, &full[s]);
            tma_load_3d(st + sv.base[0], &M.s[2][5], xl1, yv, 0, &full[s]);
            tma_load_3d(st + sv.base[1], &M.s[2][4], x0, yv, 0, &full[s]);
            tma_load_3d(st + sv.base[2], &M.s[2][5], xr1, yv, 0, &full[s]);
            tma_load_3d(st + pp.base[0], &M.p[0][3], xl1, yu, 0, &full[s]);
            tma_load_3d(st + pp.base[1], &M.p[0][2], x0, yu, 0, &full[s]);
            tma_load_3d(st + pp.base[2], &M.p[0][3], xr1, yu, 0, &full[s]);
        }
        return;
    }
    // ============================ consumers ============================
    constexpr int NT = 32 * NW;
    for (int i = 0; i < niter; ++i) {
        const int s = i % D;
        mbar_wait(&full[s], (uint32_t)((i / D) & 1));
        const double* st = smem + (size_t)s * L::STAGE;
        // phase 1: A_p on rows [-r, BH+r) x cols [-r, 64+r), 2 x 2 points per item
        constexpr int QR = G::NRU / 2, QC = G::WA / 2;
        for (int it = tid; it < QR * QC; it += NT) {
            const int r = -R + 2 * (it / QC), c = -R + 2 * (it % QC);
            double dxu[2][2] = {{0, 0}, {0, 0}}, dyv[2][2] = {{0, 0}, {0, 0}};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double w[2 * R + 2];
#pragma unroll
                for (int k = 0; k <= R; ++k) ldpair(su.at(st, r + h + R, c - R + 2 * k), w[2 * k], w[2 * k + 1]);
#pragma unroll
                for (int j = 1; j <= R; ++j)
#pragma unroll
                    for (int e = 0; e < 2; ++e) dxu[h][e] = fma(FD<R>::a(j), w[R + e + j] - w[R + e - j], dxu[h][e]);
            }
            double col[2 * R + 2][2];                     // S_v rows r-R .. r+1+R at cols c, c+1
#pragma unroll
            for (int k = 0; k < 2 * R + 2; ++k) ldpair(sv.at(st, r - R + k + 2 * R, c), col[k][0], col[k][1]);
#pragma unroll
            for (int j = 1; j <= R; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        dyv[h][e] = fma(FD<R>::a(j), col[R + h + j][e] - col[R + h - j][e], dyv[h][e]);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double p0, p1;
                ldpair(pp.at(st, r + h + R, c), p0, p1);
                const double pv[2] = {p0, p1};
                double ap[2];
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    ap[e] = combine<MODE_LF>(pv[e], 0.0, -fma(A.sx, dxu[h][e], A.sy * dyv[h][e]), 0.0, A.cfA, 0.0);
                *reinterpret_cast<double2*>(scr + (r + h + R) * G::WA + (c + R)) = make_double2(ap[0], ap[1]);
            }
        }
        consumers_sync();
        // phase 2: B_u, B_v on the band (BH x 64), 2 x 2 items
        for (int it = tid; it < (BH / 2) * (TX / 2); it += NT) {
            const int r = 2 * (it / (TX / 2)), c = 2 * (it % (TX / 2));
            double dxp[2][2] = {{0, 0}, {0, 0}}, dyp[2][2] = {{0, 0}, {0, 0}};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double w[2 * R + 2];
#pragma unroll
                for (int k = 0; k <= R; ++k)
                    ldpair(scr + (r + h + R) * G::WA + (c - R + 2 * k + R), w[2 * k], w[2 * k + 1]);
#pragma unroll
                for (int j = 1; j <= R; ++j)
#pragma unroll
                    for (int e = 0; e < 2; ++e) dxp[h][e] = fma(FD<R>::a(j), w[R + e + j] - w[R + e - j], dxp[h][e]);
            }
            double col[2 * R + 2][2];                     // A_p rows r-R .. r+1+R at cols c, c+1
#pragma unroll
            for (int k = 0; k < 2 * R + 2; ++k)
                ldpair(scr + (r - R + k + R) * G::WA + (c + R), col[k][0], col[k][1]);
#pragma unroll
            for (int j = 1; j <= R; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        dyp[h][e] = fma(FD<R>::a(j), col[R + h + j][e] - col[R + h - j][e], dyp[h][e]);
            const int64_t g0 = (int64_t)(ys + i * BH + r) * nx + x0 + c;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double u0, u1, v0, v1;
                ldpair(su.at(st, r + h + R, c), u0, u1);
                ldpair(sv.at(st, r + h + 2 * R, c), v0, v1);
                const double uu[2] = {u0, u1}, vv[2] = {v0, v1};
                double bu[2], bv[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    bu[e] = combine<MODE_LF>(uu[e], 0.0, -A.sx * dxp[h][e], 0.0, A.cfB, 0.0);
                    bv[e] = combine<MODE_LF>(vv[e], 0.0, -A.sy * dyp[h][e], 0.0, A.cfB, 0.0);
                }
                const int64_t g = g0 + (int64_t)h * nx;
                __stcs(reinterpret_cast<double2*>(A.A[0] + g), make_double2(col[R + h][0], col[R + h][1]));
                __stcs(reinterpret_cast<double2*>(A.B[1] + g), make_double2(bu[0], bu[1]));
                __stcs(reinterpret_cast<double2*>(A.B[2] + g), make_double2(bv[0], bv[1]));
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        consumers_sync();                                  // the scratch is rewritten next band
    }
}

// ---------------------------------------------------------------------------------------
template <int R>
__global__ void __launch_bounds__(32 * (AC2_NW + 1), 1)
acoustic2d_chainP_tma(const __grid_constant__ Ac2PairMaps M, const Ac2PairArgs A, const int ybase) {
    using L = ChainPLayout<R>;
    using G = Ac2Geom<R>;
    constexpr int D = L::D, NW = AC2_NW, BH = G::BH;
    extern __shared__ __align__(128) double smem[];
    double* scru = smem + (size_t)D * L::STAGE;
    double* scrv = scru + L::SCR_U;
    uint64_t* full = reinterpret_cast<uint64_t*>(scrv + L::SCR_V);
    uint64_t* empty = full + D;
    const int tid = threadIdx.x + 32 * threadIdx.y, warp = threadIdx.y, lane = threadIdx.x;
    const int nx = A.nx;
    const int x0 = blockIdx.x * TX;
    const int ys = A.ylo + blockIdx.y * A.ychunk + (blockIdx.y ? A.yskip : 0);
    const int niter = min(A.ychunk, A.yhi - ys) / BH;
    // S_p x windows on the band rows: strips L2 L1 | centre (band rows = centre rows 2r..) | R1 R2
    const Cols<R, 5> spx{{-2 * R, -R, 0, TX, TX + R}, {R, R, TX, R, R},
                         {L::SPS, L::SPS + L::BS, L::SPC + 2 * R * TX, L::SPS + 2 * L::BS, L::SPS + 3 * L::BS}};
    const Cols<R, 3> pu{{-R, 0, TX}, {R, TX, R}, {L::PU, L::PU + L::BS, L::PU + L::BS + BH * TX}};

    if (tid == 0) {
        for (int s = 0; s < D; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NW); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == NW) {
        if (lane != 0) return;
        const int xl2 = wrap_any(x0 - 2 * R, nx), xl1 = wrap_any(x0 - R, nx);
        const int xr1 = wrap_any(x0 + TX, nx), xr2 = wrap_any(x0 + TX + R, nx);
        for (int i = 0; i < niter; ++i) {
            const int s = i % D;
            if (i >= D) mbar_wait(&empty[s], (uint32_t)(((i / D) - 1) & 1));
            mbar_expect_tx(&full[s], L::stage_bytes);
            double* st = smem + (size_t)s * L::STAGE;
            const int y = ys + i * BH + ybase;
            tma_load_3d(st + L::SPC, &M.s[0][4], x0, y - 2 * R, 0, &full[s]);
            tma_load_3d(st + L::SPS, &M.s[0][1], xl2, y, 0, &full[s]);
            tma_load_3d(st + L::SPS + L::BS, &M.s[0][1], xl1, y, 0, &full[s]);
            tma_load_3d(st + L::SPS + 2 * L::BS, &M.s[0][1], xr1, y, 0, &full[s]);
            tma_load_3d(st + L::SPS + 3 * L::BS, &M.s[0][1], xr2, y, 0, &full[s]);
            tma_load_3d(st + pu.base[0], &M.p[1][1], xl1, y, 0, &full[s]);
            tma_load_3d(st + pu.base[1], &M.p[1][0], x0, y, 0, &full[s]);
            tma_load_3d(st + pu.base[2], &M.p[1][1], xr1, y, 0, &full[s]);
            tma_load_3d(st + L::PV, &M.p[2][2], x0, y - R, 0, &full[s]);
        }
        return;
    }
    constexpr int NT = 32 * NW;
    constexpr int QC = G::WA / 2;
    constexpr int N1A = (BH / 2) * QC, N1B = (G::NRU / 2) * (TX / 2);
    for (int i = 0; i < niter; ++i) {
        const int s = i % D;
        mbar_wait(&full[s], (uint32_t)((i / D) & 1));
        const double* st = smem + (size_t)s * L::STAGE;
        // phase 1: A_u on the band rows x cols [-r, 64+r) (items [0, N1A)), then A_v on
        // rows [-r, BH+r) x the band columns (items [N1A, N1A + N1B)), one item space
        for (int it = tid; it < N1A + N1B; it += NT) {
            if (it < N1A) {
                const int r = 2 * (it / QC), c = -R + 2 * (it % QC);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    double w[2 * R + 2], dxp[2] = {0, 0};
#pragma unroll
                    for (int k = 0; k <= R; ++k) ldpair(spx.at(st, r + h, c - R + 2 * k), w[2 * k], w[2 * k + 1]);
#pragma unroll
                    for (int j = 1; j <= R; ++j)
#pragma unroll
                        for (int e = 0; e < 2; ++e) dxp[e] = fma(FD<R>::a(j), w[R + e + j] - w[R + e - j], dxp[e]);
                    double p0, p1;
                    ldpair(pu.at(st, r + h, c), p0, p1);
                    const double pv[2] = {p0, p1};
                    double au[2];
#pragma unroll
                    for (int e = 0; e < 2; ++e) au[e] = combine<MODE_LF>(pv[e], 0.0, -A.sx * dxp[e], 0.0, A.cfA, 0.0);
                    *reinterpret_cast<double2*>(scru + (r + h) * G::WA + (c + R)) = make_double2(au[0], au[1]);
                }
            } else {
                const int jt = it - N1A;
                const int r = -R + 2 * (jt / (TX / 2)), c = 2 * (jt % (TX / 2));
                double col[2 * R + 2][2], dyp[2][2] = {{0, 0}, {0, 0}};
#pragma unroll
                for (int k = 0; k < 2 * R + 2; ++k)
                    ldpair(st + L::SPC + (r - R + k + 2 * R) * TX + c, col[k][0], col[k][1]);
#pragma unroll
                for (int j = 1; j <= R; ++j)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
#pragma unroll
                        for (int e = 0; e < 2; ++e)
                            dyp[h][e] = fma(FD<R>::a(j), col[R + h + j][e] - col[R + h - j][e], dyp[h][e]);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    double p0, p1;
                    ldpair(st + L::PV + (r + h + R) * TX + c, p0, p1);
                    const double pv[2] = {p0, p1};
                    double av[2];
#pragma unroll
                    for (int e = 0; e < 2; ++e) av[e] = combine<MODE_LF>(pv[e], 0.0, -A.sy * dyp[h][e], 0.0, A.cfA, 0.0);
                    *reinterpret_cast<double2*>(scrv + (r + h + R) * TX + c) = make_double2(av[0], av[1]);
                }
            }
        }
        consumers_sync();
        // phase 2: B_p on the band
        for (int it = tid; it < (BH / 2) * (TX / 2); it += NT) {
            const int r = 2 * (it / (TX / 2)), c = 2 * (it % (TX / 2));
            double dxu[2][2] = {{0, 0}, {0, 0}}, dyv[2][2] = {{0, 0}, {0, 0}};
            double cu[2][2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double w[2 * R + 2];
#pragma unroll
                for (int k = 0; k <= R; ++k)
                    ldpair(scru + (r + h) * G::WA + (c - R + 2 * k + R), w[2 * k], w[2 * k + 1]);
                cu[h][0] = w[R]; cu[h][1] = w[R + 1];
#pragma unroll
                for (int j = 1; j <= R; ++j)
#pragma unroll
                    for (int e = 0; e < 2; ++e) dxu[h][e] = fma(FD<R>::a(j), w[R + e + j] - w[R + e - j], dxu[h][e]);
            }
            double col[2 * R + 2][2];
#pragma unroll
            for (int k = 0; k < 2 * R + 2; ++k) ldpair(scrv + (r - R + k + R) * TX + c, col[k][0], col[k][1]);
#pragma unroll
            for (int j = 1; j <= R; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        dyv[h][e] = fma(FD<R>::a(j), col[R + h + j][e] - col[R + h - j][e], dyv[h][e]);
            const int64_t g0 = (int64_t)(ys + i * BH + r) * nx + x0 + c;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double s0, s1;
                ldpair(st + L::SPC + (r + h + 2 * R) * TX + c, s0, s1);
                const double sp[2] = {s0, s1};
                double bp[2];
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    bp[e] = combine<MODE_LF>(sp[e], 0.0, -fma(A.sx, dxu[h][e], A.sy * dyv[h][e]), 0.0, A.cfB, 0.0);
                const int64_t g = g0 + (int64_t)h * nx;
                __stcs(reinterpret_cast<double2*>(A.A[1] + g), make_double2(cu[h][0], cu[h][1]));
                __stcs(reinterpret_cast<double2*>(A.A[2] + g), make_double2(col[R + h][0], col[R + h][1]));
                __stcs(reinterpret_cast<double2*>(A.B[0] + g), make_double2(bp[0], bp[1]));
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        consumers_sync();
    }
}

}  // namespace tma
}  // namespace gbs

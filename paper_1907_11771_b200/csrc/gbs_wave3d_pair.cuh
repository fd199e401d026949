// gbs_wave3d_pair.cuh -- two consecutive GBS substeps of the 3-D wave in one
// HBM pass (temporal blocking), TMA-fed.
//
// Step A is a leap-frog step (Eq. (1) row 2) from (P, S) = (y_{n-1}, y_n):
//     u_a = P_u + cfA S_v                 (pointwise: u_t = v)
//     v_a = P_v + cfA lap(S_u)
// Step B is a leap-frog step (MODE_LF) or the final step fused with the averaging
// and the weighted accumulate (MODE_FIN0 / MODE_FINACC, Eq. (1) row 3 and
// PAPER.md:109-115) from (S, y_a):
//     LF :  u_b = S_u + cfB v_a,                 v_b = S_v + cfB lap(u_a)
//     FIN:  acc (+)= wh (S_u + u_a + cfB v_a),   acc (+)= wh (S_v + v_a + cfB lap(u_a))
// Because u_a is pointwise in (P_u, S_v), lap(u_a) needs only the tiles of P_u
// and S_v: u_a(x') = fma(cfA, S_v(x'), P_u(x')) is exactly the operation the
// single-step kernel performs at x', and every sum is formed in the same order,
// so the pair kernel is bit-identical to two single-step launches (tested)
// while moving 32 B read + 32 B write per point for two substeps instead of 96 B.
//
// Outputs go to buffers distinct from P and S (their halos are read by
// neighbouring CTAs): LF writes y_{n+1} -> (Au, Av) and y_{n+2} -> (Bu, Bv);
// FIN writes only the accumulator (Bu, Bv).
//
// Pipeline (64x16 tile, 16 warps x 2 points; lane 0 of warp 0 also issues TMA):
//   stage i (D-deep ring): S_u tile of plane z = z0+i (x/y stencil of lap(S_u)),
//     S_v and P_u tiles of plane z+R (to build the u_a tile of plane z+R), the
//     S_u centre box of plane z+R (front of the S_u register queue)
//   ua ring (R+2 deep): u_a tiles, the one of plane p built by all warps at
//     iteration p-R and read (x/y stencil of lap(u_a)) at iteration p, so the
//     builder never waits on the readers of the same plane; per-slot full/empty
//     mbarriers (16 warp arrivals) with two iterations of slack
//   own-point streams (S_v and P_v of plane z, the accumulator) by 128-bit loads
//     issued one iteration ahead.
// z neighbours of S_u and u_a live in two register queues of 2R+1 planes.
#pragma once

#include "gbs_wave3d_tma.cuh"

namespace gbs {
namespace tma {

template <int R, int MODEB>
struct PairLayout {
    static constexpr int SH = TY + 2 * R;
    static constexpr int NACC = (MODEB == MODE_FINACC) ? 2 : 0;
    static constexpr int D = 2;                            // TMA stages
    static constexpr int RG = (MODEB == MODE_FINACC) ? R + 1 : R + 2;   // u_a ring
    static constexpr int CENTER = SH * TX;
    static constexpr int STRIP = TY * R;
    static constexpr int TILE = CENTER + 2 * STRIP;
    static constexpr int PWT = TY * TX;
    // stage: S_u tile (z) | S_v tile (z+R) | P_u tile (z+R) | S_u centre (z+R) |
    //        S_v centre (z) | P_v centre (z) | accumulator (z, FINACC)
    static constexpr int STAGE = 3 * TILE + (3 + NACC) * PWT;
    static constexpr size_t stage_doubles = (size_t)D * STAGE;
    static constexpr size_t ring_doubles = (size_t)RG * TILE;
    static constexpr size_t bytes = (stage_doubles + ring_doubles) * 8 + (2 * D + 2 * RG + 1) * 8;
    static constexpr uint32_t stage_bytes = STAGE * 8;
    static constexpr uint32_t tile_bytes = TILE * 8;
};

struct PairMaps {
    CUtensorMap su_a, su_b, su_c;     // S_u: TXxTY, TXxR, RxTY
    CUtensorMap sv_a, sv_b, sv_c;     // S_v
    CUtensorMap pu_a, pu_b, pu_c;     // P_u
    CUtensorMap pv, acc_u, acc_v;     // TXxTY
};

struct PairArgs {
    double* Au; double* Av;           // y_{n+1} (LF)
    double* Bu; double* Bv;           // y_{n+2} (LF) or the accumulator (FIN)
    const double* Su; const double* Sv; const double* Pu; const double* Pv;
    int nx, ny, nz, zchunk;
    int64_t plane;
    double sx2, sy2, sz2;
    double cfA, cfB, wh;
    int* nonfinite;
};

template <int R, int MODEB, bool SLAB>
__global__ void __launch_bounds__(256, 1)
wave3d_pair_tma(const __grid_constant__ PairMaps M, const PairArgs A, const int zbase) {
    using L = PairLayout<R, MODEB>;
    constexpr int D = L::D, RG = L::RG, TILE = L::TILE, STAGE = L::STAGE, PWT = L::PWT;
    constexpr int NW = TY / 2;                 // 8 warps; each thread owns 2 x 2 points
    constexpr int Q = 2 * R + 1;
    extern __shared__ __align__(128) double smem[];
    double* stages = smem;
    double* ring = smem + L::stage_doubles;
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + L::ring_doubles);
    uint64_t* empty = full + D;
    uint64_t* ua_full = empty + D;
    uint64_t* ua_empty = ua_full + RG;
    uint64_t* init = ua_empty + RG;

    const int tx = threadIdx.x, ty = threadIdx.y, lane = tx, t = ty * 32 + tx;
    const int nx = A.nx, ny = A.ny, nz = A.nz;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int z0 = blockIdx.z * A.zchunk;
    const int niter = min(A.zchunk, nz - z0);
    auto zc = [&](int z) -> int {
        if constexpr (SLAB) return z + zbase;
        else return wrap_once(z, nz);
    };
    const int64_t plane = A.plane;
    const int r0 = 2 * ty;                     // the thread's rows r0, r0 + 1 of the tile
    const int64_t own = (int64_t)(y0 + r0) * nx + x0 + 2 * tx;
    auto zoff = [&](int z) -> int64_t {
        if constexpr (SLAB) return (int64_t)z * plane;
        else return (int64_t)wrap_once(z, nz) * plane;
    };
    const bool producer = (ty == 0 && lane == 0);
    const int ytop = wrap_any(y0 - R, ny), ybot = wrap_any(y0 + TY, ny);
    const int xl = wrap_any(x0 - R, nx), xr = wrap_any(x0 + TX, nx);

    auto load_tile = [&](double* dst, const CUtensorMap* a, const CUtensorMap* b, const CUtensorMap* c, int z,
                         uint64_t* bar) {
        tma_load_3d(dst, b, x0, ytop, z, bar);
        tma_load_3d(dst + R * TX, a, x0, y0, z, bar);
        tma_load_3d(dst + (R + TY) * TX, b, x0, ybot, z, bar);
        tma_load_3d(dst + L::CENTER, c, xl, y0, z, bar);
        tma_load_3d(dst + L::CENTER + L::STRIP, c, xr, y0, z, bar);
    };
    auto issue_stage = [&](int i) {
        const int s = i % D;
        if (i >= D) mbar_wait(&empty[s], (uint32_t)(((i / D) - 1) & 1));
        mbar_expect_tx(&full[s], L::stage_bytes);
        double* st = stages + (size_t)s * STAGE;
        const int z = zc(z0 + i), zf = zc(z0 + i + R);
        load_tile(st, &M.su_a, &M.su_b, &M.su_c, z, &full[s]);
        load_tile(st + TILE, &M.sv_a, &M.sv_b, &M.sv_c, zf, &full[s]);
        load_tile(st + 2 * TILE, &M.pu_a, &M.pu_b, &M.pu_c, zf, &full[s]);
        tma_load_3d(st + 3 * TILE, &M.su_a, x0, y0, zf, &full[s]);
        tma_load_3d(st + 3 * TILE + PWT, &M.sv_a, x0, y0, z, &full[s]);
        tma_load_3d(st + 3 * TILE + 2 * PWT, &M.pv, x0, y0, z, &full[s]);
        if constexpr (MODEB == MODE_FINACC) {
            tma_load_3d(st + 3 * TILE + 3 * PWT, &M.acc_u, x0, y0, z, &full[s]);
            tma_load_3d(st + 3 * TILE + 4 * PWT, &M.acc_v, x0, y0, z, &full[s]);
        }
    };
    // u_a tile of relative plane p from S_v / P_u tiles into its ring slot
    auto build = [&](const double* sv, const double* pu, int p) {
        const int slot = p % RG, use = p / RG;
        if (use >= 1) mbar_wait(&ua_empty[slot], (uint32_t)((use - 1) & 1));
        const double2* v2 = reinterpret_cast<const double2*>(sv);
        const double2* p2 = reinterpret_cast<const double2*>(pu);
        double2* o2 = reinterpret_cast<double2*>(ring + (size_t)slot * TILE);
        for (int e = t; e < TILE / 2; e += 32 * NW) {
            const double2 a = v2[e], b = p2[e];
            o2[e] = make_double2(fma(A.cfA, a.x, b.x), fma(A.cfA, a.y, b.y));
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&ua_full[slot]);
    };

    if (producer) {
        for (int s = 0; s < D; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NW); }
        for (int s = 0; s < RG; ++s) { mbar_init(&ua_full[s], NW); mbar_init(&ua_empty[s], NW); }
        mbar_init(init, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // ---- prologue: u_a tiles of planes z0 .. z0+R-1 (S_v, P_u tiles staged in the stage area)
    static_assert(2 * R * TILE <= (int)L::stage_doubles, "prologue tiles must fit the stage area");
    if (producer) {
        prefetch_map(&M.su_a); prefetch_map(&M.su_b); prefetch_map(&M.su_c);
        prefetch_map(&M.sv_a); prefetch_map(&M.sv_b); prefetch_map(&M.sv_c);
        prefetch_map(&M.pu_a); prefetch_map(&M.pu_b); prefetch_map(&M.pu_c); prefetch_map(&M.pv);
        if constexpr (MODEB == MODE_FINACC) { prefetch_map(&M.acc_u); prefetch_map(&M.acc_v); }
        mbar_expect_tx(init, 2 * R * L::tile_bytes);
        for (int p = 0; p < R; ++p) {
            load_tile(stages + (size_t)(2 * p) * TILE, &M.sv_a, &M.sv_b, &M.sv_c, zc(z0 + p), init);
            load_tile(stages + (size_t)(2 * p + 1) * TILE, &M.pu_a, &M.pu_b, &M.pu_c, zc(z0 + p), init);
        }
    }
    // register queues of S_u and u_a at planes z-R .. z+R; point index 2*row + col
    double qs[Q][4], qa[Q][4];
#pragma unroll
    for (int j = 0; j < 2 * R; ++j) {
        const int64_t oz = zoff(z0 - R + j);
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int64_t o = oz + own + (int64_t)r * nx;
            const double2 su = __ldg(reinterpret_cast<const double2*>(A.Su + o));
            const double2 sv = __ldg(reinterpret_cast<const double2*>(A.Sv + o));
            const double2 pu = __ldg(reinterpret_cast<const double2*>(A.Pu + o));
            qs[j][2 * r] = su.x; qs[j][2 * r + 1] = su.y;
            qa[j][2 * r] = fma(A.cfA, sv.x, pu.x); qa[j][2 * r + 1] = fma(A.cfA, sv.y, pu.y);
        }
    }
    mbar_wait(init, 0);
    for (int p = 0; p < R && p < niter; ++p)
        build(stages + (size_t)(2 * p) * TILE, stages + (size_t)(2 * p + 1) * TILE, p);
    __syncthreads();                          // the stage area is free again
    if (producer)
        for (int i = 0; i < D - 1 && i < niter; ++i) issue_stage(i);

    // x-window sources of the thread's two rows: columns 2tx - R + 2k
    int woff[2][R + 1];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int k = 0; k <= R; ++k) {
            const int col = 2 * tx - R + 2 * k, row = r0 + r;
            woff[r][k] = col < 0 ? L::CENTER + row * R + (col + R)
                       : col >= TX ? L::CENTER + L::STRIP + row * R + (col - TX)
                                   : (R + row) * TX + col;
        }
    const int crow0 = (R + r0) * TX + 2 * tx;   // tile offset of (row r0, column 2tx)

    // lap at the 4 points from a tile (x, y) and a queue (z): same sums in the same order as
    // the single-step kernel; the y neighbours are streamed so rows r0 and r0+1 share loads
    auto lap4 = [&](const double* tile, const double (*q)[4], double* lap, double* cen) {
        double lx[4], ly[4], lz[4];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            double xw[2 * R + 2];
#pragma unroll
            for (int k = 0; k <= R; ++k) {
                const double2 a = *reinterpret_cast<const double2*>(tile + woff[r][k]);
                xw[2 * k] = a.x; xw[2 * k + 1] = a.y;
            }
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int p = 2 * r + v;
                cen[p] = xw[R + v];
                lx[p] = FD<R>::b0() * xw[R + v];
#pragma unroll
                for (int j = 1; j <= R; ++j) lx[p] = fma(FD<R>::b(j), xw[R + v + j] + xw[R + v - j], lx[p]);
                ly[p] = FD<R>::b0() * xw[R + v];
                lz[p] = ly[p];
            }
        }
        double prev_up[2], prev_dn[2];          // rows r0-(j-1) and r0+j of the previous j
#pragma unroll
        for (int j = 1; j <= R; ++j) {
            const double2 u = *reinterpret_cast<const double2*>(tile + crow0 - j * TX);          // r0 - j
            const double2 d = *reinterpret_cast<const double2*>(tile + crow0 + (1 + j) * TX);    // r0+1+j
            const double up0[2] = {u.x, u.y}, dn1[2] = {d.x, d.y};
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const double dn0 = (j == 1) ? cen[2 + v] : prev_dn[v];     // row r0 + j
                const double up1 = (j == 1) ? cen[v] : prev_up[v];         // row r0 + 1 - j
                ly[v] = fma(FD<R>::b(j), dn0 + up0[v], ly[v]);
                ly[2 + v] = fma(FD<R>::b(j), dn1[v] + up1, ly[2 + v]);
                prev_up[v] = up0[v];
                prev_dn[v] = dn1[v];
            }
        }
#pragma unroll
        for (int p = 0; p < 4; ++p) {
#pragma unroll
            for (int j = 1; j <= R; ++j) lz[p] = fma(FD<R>::b(j), q[R + j][p] + q[R - j][p], lz[p]);
            lap[p] = fma(A.sx2, lx[p], fma(A.sy2, ly[p], A.sz2 * lz[p]));
        }
    };

    bool bad = false;
    for (int i = 0; i < niter; ++i) {
        const int s = i % D;
        if (producer && i + D - 1 < niter) issue_stage(i + D - 1);
        mbar_wait(&full[s], (uint32_t)((i / D) & 1));
        const double* st = stages + (size_t)s * STAGE;
        if (i + R < niter) build(st + TILE, st + 2 * TILE, i + R);   // u_a tile of plane z+R
        double csv[4], cpv[4], cau[4] = {0, 0, 0, 0}, cav[4] = {0, 0, 0, 0};
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int po = (r0 + r) * TX + 2 * tx;                      // own column in a centre box
            const int to = (R + r0 + r) * TX + 2 * tx;                  // own column in a tile
            const double2 fs = *reinterpret_cast<const double2*>(st + 3 * TILE + po);
            const double2 fv = *reinterpret_cast<const double2*>(st + TILE + to);
            const double2 fp = *reinterpret_cast<const double2*>(st + 2 * TILE + to);
            qs[2 * R][2 * r] = fs.x; qs[2 * R][2 * r + 1] = fs.y;
            qa[2 * R][2 * r] = fma(A.cfA, fv.x, fp.x);
            qa[2 * R][2 * r + 1] = fma(A.cfA, fv.y, fp.y);
            const double2 a = *reinterpret_cast<const double2*>(st + 3 * TILE + PWT + po);
            const double2 b = *reinterpret_cast<const double2*>(st + 3 * TILE + 2 * PWT + po);
            csv[2 * r] = a.x; csv[2 * r + 1] = a.y; cpv[2 * r] = b.x; cpv[2 * r + 1] = b.y;
            if constexpr (MODEB == MODE_FINACC) {
                const double2 c = *reinterpret_cast<const double2*>(st + 3 * TILE + 3 * PWT + po);
                const double2 d = *reinterpret_cast<const double2*>(st + 3 * TILE + 4 * PWT + po);
                cau[2 * r] = c.x; cau[2 * r + 1] = c.y; cav[2 * r] = d.x; cav[2 * r + 1] = d.y;
            }
        }
        double lapS[4], lapA[4], xs_c[4], xa_c[4];
        lap4(st, qs, lapS, xs_c);                               // S_u tile, plane z
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        {
            const int slot = i % RG;
            mbar_wait(&ua_full[slot], (uint32_t)((i / RG) & 1));
            lap4(ring + (size_t)slot * TILE, qa, lapA, xa_c);
            __syncwarp();
            if (lane == 0) mbar_arrive(&ua_empty[slot]);
        }
        double ua[4], va[4], ub[4], vb[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            ua[p] = xa_c[p];                                                    // step A, u
            va[p] = combine<MODE_LF>(cpv[p], csv[p], lapS[p], 0.0, A.cfA, 0.0);     // step A, v
            ub[p] = combine<MODEB>(xs_c[p], ua[p], va[p], cau[p], A.cfB, A.wh);     // step B, u
            vb[p] = combine<MODEB>(csv[p], va[p], lapA[p], cav[p], A.cfB, A.wh);    // step B, v
            if constexpr (MODEB != MODE_LF) bad |= !isfinite(ub[p]) || !isfinite(vb[p]);
        }
        const int64_t oz = zoff(z0 + i);
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int64_t o = oz + own + (int64_t)r * nx;
            if constexpr (MODEB == MODE_LF) {
                *reinterpret_cast<double2*>(A.Au + o) = make_double2(ua[2 * r], ua[2 * r + 1]);
                *reinterpret_cast<double2*>(A.Av + o) = make_double2(va[2 * r], va[2 * r + 1]);
            }
            *reinterpret_cast<double2*>(A.Bu + o) = make_double2(ub[2 * r], ub[2 * r + 1]);
            *reinterpret_cast<double2*>(A.Bv + o) = make_double2(vb[2 * r], vb[2 * r + 1]);
        }
#pragma unroll
        for (int j = 0; j < 2 * R; ++j)
#pragma unroll
            for (int p = 0; p < 4; ++p) { qs[j][p] = qs[j + 1][p]; qa[j][p] = qa[j + 1][p]; }
    }
    if constexpr (MODEB != MODE_LF)
        if (bad && A.nonfinite) *A.nonfinite = 1;
}

}  // namespace tma
}  // namespace gbs

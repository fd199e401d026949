// gbs_wave3d_half.cuh -- the single-stencil-field 3-D wave kernel: one "half" of
// the two-substep pass, or the forward-Euler substep, TMA-fed.
//
// The leap-frog pair of gbs_wave3d_pair.cuh (Eq. (1) row 2, two
// consecutive substeps of one sequence) splits into two computations that share
// no value (u_t = v is pointwise, so the u-level is carried one step ahead):
//   half A:  v_{n+1} = P_v + cfA lap(S_u),   u_{n+2} = S_u + cfB v_{n+1}
//   half B:  v_{n+2} = S_v + cfB lap(U),     u_{n+3} = U   + cfA v_{n+2}
// Each is   O1 = P + c1 lap(X),   O2 = X + c2 O1   with one stencil field X and
// one pointwise field P: 16 B read + 16 B written per point, the same 64 B per
// point for the pair as the coupled kernel, but a CTA carries ONE register
// queue instead of two.  The forward-Euler start (Eq. (1) row 1) has the same
// form with X = u_0, P = v_0, c1 = h, c2 = 2h (O1 = v_1, O2 = u_2, the u-level
// one step ahead) plus the pointwise O3 = u_1 = u_0 + h v_0.  Every value is
// formed by exactly the operation the single-substep kernels use (fma(cf, f, p),
// the Laplacian's sums in the same order), so results are bit-identical to the
// coupled pair and to single substeps (tested).
//
// Why: under the 1 kW power cap the coupled pair kernel is bound
// by its SM side -- 240 registers (two 2r+1-plane queues) leave 8 warps per SM,
// and its shared-memory traffic (TMA fills, 40 128-bit loads per thread-plane,
// front boxes re-read from L2) runs the L1/shared pipeline at ~70%.  With one
// queue per CTA:
//   * the tile is 64 x TYH (TYH = 32 on grids whose ny allows it), halving the
//     relative y-halo (the largest source of excess DRAM reads of the coupled
//     kernel) and the halo loads per point;
//   * the queue front (plane z + R) comes from a ring of R + D tiles instead of a
//     second TMA box of the same data;
//   * the pointwise field P arrives by TMA in the same stage as the tile (a version that
//     read it with register-prefetched global loads exposed their latency: 56% of the
//     stall samples long-scoreboard on the register move at the loop top, ncu; double
//     buffering it in registers spilled);
//   * 16 warps (RPT = 2 rows x 2 columns per thread) or 8 (RPT = 4).
// Producer: lane 0 of warp 0 issues the five boxes of plane z + R + D - 1 (centre
// TX x TYH, y halos TX x R, x strips R x TYH) into a ring of R + D tiles through
// full/empty mbarriers (no extra producer warp: 16 warps keep 128 registers).
#pragma once

#include "gbs_wave3d_tma.cuh"
#include "gbs_wave3d_pair.cuh"      // MODE_FEA

namespace gbs {
namespace tma {

enum { HALF_LF = 0, HALF_FE = 1 };
constexpr int TYH_TALL = 32;           // tile rows on grids with ny % 32 == 0

template <int R, int TYH, int D>
struct HalfLayout {
    static constexpr int SH = TYH + 2 * R;
    static constexpr int CENTER = SH * TX;
    static constexpr int STRIP = TYH * R;
    static constexpr int TILE = CENTER + 2 * STRIP;
    static constexpr int RING = R + D;
    static constexpr int PWT = TYH * TX;                  // one plane of the pointwise field P
    static constexpr size_t ring_doubles = (size_t)RING * TILE;
    static constexpr size_t p_doubles = (size_t)D * PWT;
    static constexpr size_t bytes = (ring_doubles + p_doubles) * 8 + (2 * D + 1) * 8;
    static constexpr uint32_t tile_bytes = TILE * 8;
    static constexpr uint32_t stage_bytes = (TILE + PWT) * 8;
    static_assert((CENTER * 8) % 128 == 0 && (STRIP * 8) % 128 == 0, "TMA destinations need 128 B alignment");
};

struct HalfMaps {
    CUtensorMap x_a, x_b, x_c;        // X: TX x TYH centre, TX x R y halos, R x TYH x strips
    CUtensorMap p;                    // P: TX x TYH
};

struct HalfArgs {
    const double* X;                  // stencil field (its own points seed the queue)
    const double* P;                  // pointwise field
    double* O1; double* O2; double* O3;   // O3: FE only (u_1)
    int nx, ny, nz, zchunk;
    int zlo, zhi, zskip;
    int64_t plane;
    double sx2, sy2, sz2;
    double c1, c2;
    int band;
    int hint;                         // 1 centre boxes evict_last, 2 P box evict_first,
                                      // 4 halo boxes evict_first, 8 streaming stores
};

template <int R, int KIND, bool SLAB, int TYH, int RPT, int D>
__global__ void __launch_bounds__(32 * (TYH / RPT), 1)
wave3d_half_tma(const __grid_constant__ HalfMaps M, const HalfArgs A, const int zbase) {
    using L = HalfLayout<R, TYH, D>;
    constexpr int NW = TYH / RPT;              // warps; lane 0 of warp 0 also issues the TMA boxes
    constexpr int RING = L::RING, TILE = L::TILE;
    extern __shared__ __align__(128) double smem[];
    double* ring = smem;
    double* pst = smem + L::ring_doubles;      // P of plane i in slot i % D
    uint64_t* full = reinterpret_cast<uint64_t*>(pst + L::p_doubles);
    uint64_t* empty = full + D;
    uint64_t* init = empty + D;

    const int tx = threadIdx.x, ty = threadIdx.y, lane = tx;
    const int nx = A.nx, ny = A.ny, nz = A.nz;
    int xt, yt;
    tile_of(blockIdx.x, nx / TX, ny / TYH, A.band, xt, yt);
    const int x0 = xt * TX, y0 = yt * TYH;
    const int z0 = A.zlo + blockIdx.z * A.zchunk + (blockIdx.z ? A.zskip : 0);
    const int niter = min(A.zchunk, A.zhi - z0);
    auto zc = [&](int z) -> int {
        if constexpr (SLAB) return z + zbase;
        else return wrap_once(z, nz);
    };
    const bool producer = (ty == 0 && lane == 0);
    const int ytop = wrap_any(y0 - R, ny), ybot = wrap_any(y0 + TYH, ny);
    const int xl = wrap_any(x0 - R, nx), xr = wrap_any(x0 + TX, nx);
    const uint64_t pol_last = policy_evict_last(), pol_first = policy_evict_first();
    auto ld = [&](void* dst, const CUtensorMap* m, int x, int y, int z, uint64_t* bar, int bit, uint64_t pol) {
        if (A.hint & bit) tma_load_3d_hint(dst, m, x, y, z, bar, pol);
        else tma_load_3d(dst, m, x, y, z, bar);
    };
    // tile of plane p (the x/y stencil at iteration p, the queue front at iteration p - R)
    auto issue_tile = [&](int p, uint64_t* bar) {
        double* t = ring + (size_t)(p % RING) * TILE;
        const int z = zc(z0 + p);
        ld(t, &M.x_b, x0, ytop, z, bar, 4, pol_first);
        ld(t + R * TX, &M.x_a, x0, y0, z, bar, 1, pol_last);
        ld(t + (R + TYH) * TX, &M.x_b, x0, ybot, z, bar, 4, pol_first);
        ld(t + L::CENTER, &M.x_c, xl, y0, z, bar, 4, pol_first);
        ld(t + L::CENTER + L::STRIP, &M.x_c, xr, y0, z, bar, 4, pol_first);
    };
    // stage k = the tile of plane k + R (slot (k + R) % RING, full[k % D]); its slot held
    // plane k + R - RING = k - D, free once every warp is done with iteration k - D
    auto issue_stage = [&](int k) {
        const int s = k % D;
        if (k >= D) mbar_wait(&empty[s], (uint32_t)(((k / D) - 1) & 1));
        mbar_expect_tx(&full[s], L::stage_bytes);
        issue_tile(k + R, &full[s]);
        ld(pst + (size_t)s * L::PWT, &M.p, x0, y0, zc(z0 + k), &full[s], 2, pol_first);   // P of plane k
    };
    if (producer) {
        for (int s = 0; s < D; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NW); }
        mbar_init(init, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (producer) {
        prefetch_map(&M.x_a); prefetch_map(&M.x_b); prefetch_map(&M.x_c); prefetch_map(&M.p);
        mbar_expect_tx(init, R * L::tile_bytes);
        for (int p = 0; p < R; ++p) issue_tile(p, init);
        for (int k = 0; k < D - 1 && k < niter; ++k) issue_stage(k);
    }

    const int64_t plane = A.plane;
    const int r0 = RPT * ty;                   // the thread's rows r0 .. r0 + RPT - 1 of the tile
    const int64_t own = (int64_t)(y0 + r0) * nx + x0 + 2 * tx;
    auto zoff = [&](int z) -> int64_t {
        if constexpr (SLAB) return (int64_t)z * plane;
        else return (int64_t)wrap_once(z, nz) * plane;
    };
    const bool scs = A.hint & 8;
    // register queue of X at planes z - R .. z + R; point (row r, column v) -> [r][v]
    double q[2 * R + 1][RPT][2];
#pragma unroll
    for (int j = 0; j < R; ++j)
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            const double2 t = __ldg(reinterpret_cast<const double2*>(A.X + zoff(z0 - R + j) + own + (int64_t)r * nx));
            q[j][r][0] = t.x; q[j][r][1] = t.y;
        }
    const int crow0 = (R + r0) * TX + 2 * tx;  // tile offset of (row r0, column 2tx)
    mbar_wait(init, 0);
#pragma unroll
    for (int j = 0; j < R; ++j)
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            const double2 t = *reinterpret_cast<const double2*>(ring + (size_t)j * TILE + crow0 + r * TX);
            q[R + j][r][0] = t.x; q[R + j][r][1] = t.y;
        }

    // x-window sources: columns 2tx - R + 2k of row r0 + r (centre column or a strip)
    int woff[RPT][R + 1];
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
        for (int k = 0; k <= R; ++k) {
            const int col = 2 * tx - R + 2 * k, row = r0 + r;
            woff[r][k] = col < 0 ? L::CENTER + row * R + (col + R)
                       : col >= TX ? L::CENTER + L::STRIP + row * R + (col - TX)
                                   : (R + row) * TX + col;
        }

    for (int i = 0; i < niter; ++i) {
        const int s = i % D;
        if (producer && i + D - 1 < niter) issue_stage(i + D - 1);
        mbar_wait(&full[s], (uint32_t)((i / D) & 1));
        const double* tile = ring + (size_t)(i % RING) * TILE;               // plane z
        const double* front = ring + (size_t)((i + R) % RING) * TILE;        // plane z + R
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            const double2 f = *reinterpret_cast<const double2*>(front + crow0 + r * TX);
            q[2 * R][r][0] = f.x; q[2 * R][r][1] = f.y;
        }
        // the three directional sums, each b0 c + sum_j b_j (pair), in the single-step order
        double lx[RPT][2], ly[RPT][2], lz[RPT][2];
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            double xw[2 * R + 2];
#pragma unroll
            for (int k = 0; k <= R; ++k) {
                if (k == R / 2) {                   // the thread's own points: already in the queue
                    xw[2 * k] = q[R][r][0]; xw[2 * k + 1] = q[R][r][1];
                    continue;
                }
                const double2 t = *reinterpret_cast<const double2*>(tile + woff[r][k]);
                xw[2 * k] = t.x; xw[2 * k + 1] = t.y;
            }
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const double c = xw[R + v];
                lx[r][v] = FD<R>::b0() * c;
                ly[r][v] = FD<R>::b0() * c;
                lz[r][v] = FD<R>::b0() * c;
#pragma unroll
                for (int j = 1; j <= R; ++j) {
                    lx[r][v] = fma(FD<R>::b(j), xw[R + v + j] + xw[R + v - j], lx[r][v]);
                    lz[r][v] = fma(FD<R>::b(j), q[R + j][r][v] + q[R - j][r][v], lz[r][v]);
                }
            }
        }
        if constexpr (RPT == 2) {
            // y: rows r0 - j and r0 + 1 + j loaded per j; the other member of each pair is
            // the previous j's load (or the own row)
            double prev_up[2], prev_dn[2];
#pragma unroll
            for (int j = 1; j <= R; ++j) {
                const double2 u = *reinterpret_cast<const double2*>(tile + crow0 - j * TX);          // r0 - j
                const double2 d = *reinterpret_cast<const double2*>(tile + crow0 + (1 + j) * TX);    // r0+1+j
                const double up0[2] = {u.x, u.y}, dn1[2] = {d.x, d.y};
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    const double dn0 = (j == 1) ? q[R][1][v] : prev_dn[v];     // row r0 + j
                    const double up1 = (j == 1) ? q[R][0][v] : prev_up[v];     // row r0 + 1 - j
                    ly[0][v] = fma(FD<R>::b(j), dn0 + up0[v], ly[0][v]);
                    ly[1][v] = fma(FD<R>::b(j), dn1[v] + up1, ly[1][v]);
                    prev_up[v] = up0[v];
                    prev_dn[v] = dn1[v];
                }
            }
        } else {
            // y column: rows r0 - R .. r0 + RPT - 1 + R (own rows from the queue)
            double yc[RPT + 2 * R][2];
#pragma unroll
            for (int k = 0; k < RPT + 2 * R; ++k) {
                if (k >= R && k < R + RPT) {
                    yc[k][0] = q[R][k - R][0]; yc[k][1] = q[R][k - R][1];
                } else {
                    const double2 t = *reinterpret_cast<const double2*>(tile + crow0 + (k - R) * TX);
                    yc[k][0] = t.x; yc[k][1] = t.y;
                }
            }
#pragma unroll
            for (int r = 0; r < RPT; ++r)
#pragma unroll
                for (int v = 0; v < 2; ++v)
#pragma unroll
                    for (int j = 1; j <= R; ++j)
                        ly[r][v] = fma(FD<R>::b(j), yc[R + r + j][v] + yc[R + r - j][v], ly[r][v]);
        }
        double pc[RPT][2];                              // P at the own points of plane z
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            const double2 t = *reinterpret_cast<const double2*>(pst + (size_t)s * L::PWT + (r0 + r) * TX + 2 * tx);
            pc[r][0] = t.x; pc[r][1] = t.y;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);          // this warp is done with stage s
        const int64_t o = zoff(z0 + i) + own;
        auto put = [&](double* p, double a, double b) {
            if (scs) __stcs(reinterpret_cast<double2*>(p), make_double2(a, b));
            else *reinterpret_cast<double2*>(p) = make_double2(a, b);
        };
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            double o1[2], o2[2];
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const double lap = fma(A.sx2, lx[r][v], fma(A.sy2, ly[r][v], A.sz2 * lz[r][v]));
                o1[v] = fma(A.c1, lap, pc[r][v]);                   // combine<LF>(P, -, lap, c1)
                o2[v] = fma(A.c2, o1[v], q[R][r][v]);               // combine<LF>(X, -, O1, c2)
            }
            put(A.O1 + o + (int64_t)r * nx, o1[0], o1[1]);
            put(A.O2 + o + (int64_t)r * nx, o2[0], o2[1]);
            if constexpr (KIND == HALF_FE)                          // u_1 = u_0 + h v_0
                put(A.O3 + o + (int64_t)r * nx, fma(A.c1, pc[r][0], q[R][r][0]), fma(A.c1, pc[r][1], q[R][r][1]));
        }
#pragma unroll
        for (int j = 0; j < 2 * R; ++j)
#pragma unroll
            for (int r = 0; r < RPT; ++r) { q[j][r][0] = q[j + 1][r][0]; q[j][r][1] = q[j + 1][r][1]; }
    }
}

}  // namespace tma
}  // namespace gbs

namespace gbs {
namespace tma {

// ---------------------------------------------------------------------------
// The two-laplacian passes of the 3-D path with both stencil fields fed through rings of
// R + D tiles (the queue fronts, plane z + R, are read from the ring instead of being loaded
// again as separate centre boxes).  The same operations in the same order as
// gbs_wave3d_pair.cuh, so bit-identical to it:
//   MODE_FEA     the forward Euler fused with the first step of chain A: fields u_0, v_0;
//                outputs A2 = v_2, A3 = u_3, A1 = v_1, A4 = u_2 (D = 4, 213 KB)
//   MODE_FIN0/   the last leap-frog step + averaging + weighted accumulate: fields S_u, U and
//   MODE_FINACC  the pointwise boxes S_v, P_v (+ the accumulator) of plane z; outputs the
//                accumulator's u, v (A3, A1 pointers) (D = 2, 224 KB)
// 64 x 16 tiles, 8 warps x 2 x 2 points, two register queues (as the pair kernel).
// ---------------------------------------------------------------------------
struct Ring2Maps {
    HalfMaps u, v;                    // the two stencil fields: centre TX x TY, y halos, x strips
    CUtensorMap sv, pv, acc_u, acc_v; // FIN: TX x TY boxes
};

struct Ring2Args {
    const double* Su; const double* U;   // the two stencil fields (queue seeds)
    double* A1; double* A2; double* A3; double* A4;
    int nx, ny, nz, zchunk;
    int zlo, zhi, zskip;
    int64_t plane;
    double sx2, sy2, sz2;
    double cfA, cfB, wh;
    int* nonfinite;
    int band;
    int hint;                         // 1 centre boxes evict_last, 2 pointwise boxes evict_first,
                                      // 4 halo boxes evict_first, 8 .cs stores
};

template <int R, int MODE>
struct Ring2Layout {
    static constexpr bool FIN = MODE != MODE_FEA;
    static constexpr int NPW = FIN ? (MODE == MODE_FINACC ? 4 : 2) : 0;
    static constexpr int D = FIN ? 2 : 4;
    using T = HalfLayout<R, TY, D>;
    static constexpr int PWT = TY * TX;
    static constexpr size_t pw_doubles = (size_t)D * NPW * PWT;
    static constexpr size_t bytes = (2 * T::ring_doubles + pw_doubles) * 8 + (2 * D + 1) * 8;
    static constexpr uint32_t stage_bytes = 2 * T::tile_bytes + NPW * PWT * 8;
};

template <int R, int MODE, bool SLAB>
__global__ void __launch_bounds__(256, 1)
wave3d_ring2(const __grid_constant__ Ring2Maps M, const Ring2Args A, const int zbase) {
    using RL = Ring2Layout<R, MODE>;
    using L = typename RL::T;
    constexpr int D = RL::D, NPW = RL::NPW, PWT = RL::PWT;
    constexpr int NW = TY / 2;                 // 8 warps, 2 rows x 2 columns per thread
    constexpr int RING = L::RING, TILE = L::TILE;
    constexpr int Q = 2 * R + 1;
    extern __shared__ __align__(128) double smem[];
    double* ringu = smem;
    double* ringv = smem + L::ring_doubles;
    double* pw = smem + 2 * L::ring_doubles;   // [stage][S_v, P_v, acc_u, acc_v]
    uint64_t* full = reinterpret_cast<uint64_t*>(pw + RL::pw_doubles);
    uint64_t* empty = full + D;
    uint64_t* init = empty + D;

    const int tx = threadIdx.x, ty = threadIdx.y, lane = tx;
    const int nx = A.nx, ny = A.ny, nz = A.nz;
    int xt, yt;
    tile_of(blockIdx.x, nx / TX, ny / TY, A.band, xt, yt);
    const int x0 = xt * TX, y0 = yt * TY;
    const int z0 = A.zlo + blockIdx.z * A.zchunk + (blockIdx.z ? A.zskip : 0);
    const int niter = min(A.zchunk, A.zhi - z0);
    auto zc = [&](int z) -> int {
        if constexpr (SLAB) return z + zbase;
        else return wrap_once(z, nz);
    };
    const bool producer = (ty == 0 && lane == 0);
    const int ytop = wrap_any(y0 - R, ny), ybot = wrap_any(y0 + TY, ny);
    const int xl = wrap_any(x0 - R, nx), xr = wrap_any(x0 + TX, nx);
    const uint64_t pol_last = policy_evict_last(), pol_first = policy_evict_first();
    auto ld = [&](void* dst, const CUtensorMap* m, int x, int y, int z, uint64_t* bar, int bit, uint64_t pol) {
        if (A.hint & bit) tma_load_3d_hint(dst, m, x, y, z, bar, pol);
        else tma_load_3d(dst, m, x, y, z, bar);
    };
    auto issue_tile = [&](double* ring, const HalfMaps& m, int p, uint64_t* bar) {
        double* t = ring + (size_t)(p % RING) * TILE;
        const int z = zc(z0 + p);
        ld(t, &m.x_b, x0, ytop, z, bar, 4, pol_first);
        ld(t + R * TX, &m.x_a, x0, y0, z, bar, 1, pol_last);
        ld(t + (R + TY) * TX, &m.x_b, x0, ybot, z, bar, 4, pol_first);
        ld(t + L::CENTER, &m.x_c, xl, y0, z, bar, 4, pol_first);
        ld(t + L::CENTER + L::STRIP, &m.x_c, xr, y0, z, bar, 4, pol_first);
    };
    // stage k: the tiles of plane k + R (both rings) and the pointwise boxes of plane k
    auto issue_stage = [&](int k) {
        const int s = k % D;
        if (k >= D) mbar_wait(&empty[s], (uint32_t)(((k / D) - 1) & 1));
        mbar_expect_tx(&full[s], RL::stage_bytes);
        issue_tile(ringu, M.u, k + R, &full[s]);
        issue_tile(ringv, M.v, k + R, &full[s]);
        if constexpr (RL::FIN) {
            double* p = pw + (size_t)s * NPW * PWT;
            const int z = zc(z0 + k);
            ld(p, &M.sv, x0, y0, z, &full[s], 2, pol_first);
            ld(p + PWT, &M.pv, x0, y0, z, &full[s], 2, pol_first);
            if constexpr (MODE == MODE_FINACC) {
                ld(p + 2 * PWT, &M.acc_u, x0, y0, z, &full[s], 2, pol_first);
                ld(p + 3 * PWT, &M.acc_v, x0, y0, z, &full[s], 2, pol_first);
            }
        }
    };
    if (producer) {
        for (int s = 0; s < D; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NW); }
        mbar_init(init, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (producer) {
        prefetch_map(&M.u.x_a); prefetch_map(&M.u.x_b); prefetch_map(&M.u.x_c);
        prefetch_map(&M.v.x_a); prefetch_map(&M.v.x_b); prefetch_map(&M.v.x_c);
        if constexpr (RL::FIN) { prefetch_map(&M.sv); prefetch_map(&M.pv); }
        if constexpr (MODE == MODE_FINACC) { prefetch_map(&M.acc_u); prefetch_map(&M.acc_v); }
        mbar_expect_tx(init, 2 * R * L::tile_bytes);
        for (int p = 0; p < R; ++p) { issue_tile(ringu, M.u, p, init); issue_tile(ringv, M.v, p, init); }
        for (int k = 0; k < D - 1 && k < niter; ++k) issue_stage(k);
    }

    const int64_t plane = A.plane;
    const int r0 = 2 * ty;
    const int64_t own = (int64_t)(y0 + r0) * nx + x0 + 2 * tx;
    auto zoff = [&](int z) -> int64_t {
        if constexpr (SLAB) return (int64_t)z * plane;
        else return (int64_t)wrap_once(z, nz) * plane;
    };
    // queues of the two fields at planes z - R .. z + R; point index 2*row + col
    double qs[Q][4], qa[Q][4];
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int64_t oz = zoff(z0 - R + j);
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int64_t o = oz + own + (int64_t)r * nx;
            const double2 su = __ldg(reinterpret_cast<const double2*>(A.Su + o));
            const double2 uu = __ldg(reinterpret_cast<const double2*>(A.U + o));
            qs[j][2 * r] = su.x; qs[j][2 * r + 1] = su.y;
            qa[j][2 * r] = uu.x; qa[j][2 * r + 1] = uu.y;
        }
    }
    const int crow0 = (R + r0) * TX + 2 * tx;
    mbar_wait(init, 0);
#pragma unroll
    for (int j = 0; j < R; ++j)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const double2 a = *reinterpret_cast<const double2*>(ringu + (size_t)j * TILE + crow0 + r * TX);
            const double2 b = *reinterpret_cast<const double2*>(ringv + (size_t)j * TILE + crow0 + r * TX);
            qs[R + j][2 * r] = a.x; qs[R + j][2 * r + 1] = a.y;
            qa[R + j][2 * r] = b.x; qa[R + j][2 * r + 1] = b.y;
        }
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
    // lap at the 4 points: the pair kernel's lap4, same sums in the same order
    auto lap4 = [&](const double* tile, const double (*q)[4], double* lap, double* cen) {
        double lx[4], ly[4], lz[4];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            double xw[2 * R + 2];
#pragma unroll
            for (int k = 0; k <= R; ++k) {
                if (k == R / 2) {
                    xw[2 * k] = q[R][2 * r]; xw[2 * k + 1] = q[R][2 * r + 1];
                    continue;
                }
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
        double prev_up[2], prev_dn[2];
#pragma unroll
        for (int j = 1; j <= R; ++j) {
            const double2 u = *reinterpret_cast<const double2*>(tile + crow0 - j * TX);
            const double2 d = *reinterpret_cast<const double2*>(tile + crow0 + (1 + j) * TX);
            const double up0[2] = {u.x, u.y}, dn1[2] = {d.x, d.y};
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const double dn0 = (j == 1) ? cen[2 + v] : prev_dn[v];
                const double up1 = (j == 1) ? cen[v] : prev_up[v];
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

    const bool scs = A.hint & 8;
    auto put = [&](double* p, double a, double b) {
        if (scs) __stcs(reinterpret_cast<double2*>(p), make_double2(a, b));
        else *reinterpret_cast<double2*>(p) = make_double2(a, b);
    };
    bool bad = false;
    for (int i = 0; i < niter; ++i) {
        const int s = i % D;
        if (producer && i + D - 1 < niter) issue_stage(i + D - 1);
        mbar_wait(&full[s], (uint32_t)((i / D) & 1));
        const size_t cur = (size_t)(i % RING) * TILE, fr = (size_t)((i + R) % RING) * TILE;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const double2 a = *reinterpret_cast<const double2*>(ringu + fr + crow0 + r * TX);
            const double2 b = *reinterpret_cast<const double2*>(ringv + fr + crow0 + r * TX);
            qs[2 * R][2 * r] = a.x; qs[2 * R][2 * r + 1] = a.y;
            qa[2 * R][2 * r] = b.x; qa[2 * R][2 * r + 1] = b.y;
        }
        double csv[4] = {0, 0, 0, 0}, cpv[4] = {0, 0, 0, 0}, cau[4] = {0, 0, 0, 0}, cav[4] = {0, 0, 0, 0};
        if constexpr (RL::FIN) {
            const double* p = pw + (size_t)s * NPW * PWT;
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const int po = (r0 + r) * TX + 2 * tx;
                const double2 a = *reinterpret_cast<const double2*>(p + po);
                const double2 b = *reinterpret_cast<const double2*>(p + PWT + po);
                csv[2 * r] = a.x; csv[2 * r + 1] = a.y; cpv[2 * r] = b.x; cpv[2 * r + 1] = b.y;
                if constexpr (MODE == MODE_FINACC) {
                    const double2 c = *reinterpret_cast<const double2*>(p + 2 * PWT + po);
                    const double2 d = *reinterpret_cast<const double2*>(p + 3 * PWT + po);
                    cau[2 * r] = c.x; cau[2 * r + 1] = c.y; cav[2 * r] = d.x; cav[2 * r + 1] = d.y;
                }
            }
        }
        double lapS[4], lapU[4], xs_c[4], xu_c[4];
        lap4(ringu + cur, qs, lapS, xs_c);
        lap4(ringv + cur, qa, lapU, xu_c);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        const int64_t oz = zoff(z0 + i);
        if constexpr (MODE == MODE_FEA) {
            double va[4], ub[4], vb[4], uc[4];
#pragma unroll
            for (int p = 0; p < 4; ++p) {            // as wave3d_pair_tma MODE_FEA
                const double u0 = xs_c[p], v0 = xu_c[p];
                vb[p] = combine<MODE_FE>(0.0, v0, lapS[p], 0.0, A.cfA, 0.0);        // v_1
                const double u1 = combine<MODE_FE>(0.0, u0, v0, 0.0, A.cfA, 0.0);   // u_1
                uc[p] = combine<MODE_LF>(u0, 0.0, vb[p], 0.0, A.cfB, 0.0);         // u_2
                const double lap1 = fma(A.cfA, lapU[p], lapS[p]);                   // lap(u_1)
                va[p] = combine<MODE_LF>(v0, 0.0, lap1, 0.0, A.cfB, 0.0);           // v_2
                ub[p] = combine<MODE_LF>(u1, 0.0, va[p], 0.0, A.cfB, 0.0);          // u_3
            }
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const int64_t o = oz + own + (int64_t)r * nx;
                put(A.A2 + o, va[2 * r], va[2 * r + 1]);
                put(A.A3 + o, ub[2 * r], ub[2 * r + 1]);
                put(A.A1 + o, vb[2 * r], vb[2 * r + 1]);
                put(A.A4 + o, uc[2 * r], uc[2 * r + 1]);
            }
        } else {
            double ub[4], vb[4];
#pragma unroll
            for (int p = 0; p < 4; ++p) {            // as wave3d_pair_tma FIN0 / FINACC
                const double va = combine<MODE_LF>(cpv[p], csv[p], lapS[p], 0.0, A.cfA, 0.0);   // v_N
                ub[p] = combine<MODE>(xs_c[p], xu_c[p], va, cau[p], A.cfB, A.wh);               // acc_u
                vb[p] = combine<MODE>(csv[p], va, lapU[p], cav[p], A.cfB, A.wh);                // acc_v
                bad |= !isfinite(ub[p]) || !isfinite(vb[p]);
            }
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const int64_t o = oz + own + (int64_t)r * nx;
                put(A.A3 + o, ub[2 * r], ub[2 * r + 1]);
                put(A.A1 + o, vb[2 * r], vb[2 * r + 1]);
            }
        }
#pragma unroll
        for (int j = 0; j < 2 * R; ++j)
#pragma unroll
            for (int p = 0; p < 4; ++p) { qs[j][p] = qs[j + 1][p]; qa[j][p] = qa[j + 1][p]; }
    }
    if constexpr (RL::FIN)
        if (bad && A.nonfinite) *A.nonfinite = 1;
}

}  // namespace tma
}  // namespace gbs
